"""ctypes binding of libcpdb.so (the C ABI in include/cpdb.h).

This is the reference-side binding a Python maintainer would add (see
INTEGRATION.md); the C++ drop-in headers in include/cpd/ bind the same ABI.
There is no fallback: if the shared library or a B200 is missing every call
raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcpdb.so")
MAX_ORDER = 8
ROOT_KEY = 0xFFFFFFFF

OK, INVALID_ARGUMENT, STALE_INTERMEDIATE, SINGULAR_TRIANGULAR, LOGIC_ERROR, CUDA_ERROR, \
    NCCL_ERROR, OUT_OF_MEMORY, FILE_ERROR, FORMAT_ERROR, SINGULAR_SYSTEM = range(11)


class TraceRow(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint64),
        ("order", C.c_uint32),
        ("update_order", C.c_uint32 * MAX_ORDER),
        ("pad0", C.c_uint32),
        ("fitness", C.c_double),
        ("raw_radicand", C.c_double),
        ("wall_seconds", C.c_double),
        ("root_ttm_count", C.c_uint64),
        ("flops", C.c_uint64),
        ("beta_used", C.c_double),
        ("regularized", C.c_int32),
        ("pad1", C.c_int32),
    ]


class Config(C.Structure):
    _fields_ = [
        ("rank", C.c_uint64),
        ("max_iterations", C.c_uint64),
        ("fitness_threshold", C.c_double),
        ("strategy", C.c_int32),
        ("extrapolate", C.c_int32),
        ("alpha", C.c_double),
        ("has_beta_override", C.c_int32),
        ("pad0", C.c_int32),
        ("beta_override", C.c_double),
        ("activation_gap", C.c_double),
        ("seed", C.c_uint64),
    ]


class State(C.Structure):
    _fields_ = [
        ("sweeps_done", C.c_uint64),
        ("lam", C.POINTER(C.c_double)),
        ("factors", C.POINTER(C.c_double)),
        ("q0_history", C.POINTER(C.c_double)),
        ("history_mask", C.c_uint32),
        ("has_active_beta", C.c_int32),
        ("active_beta", C.c_double),
        ("has_prev_fitness", C.c_int32),
        ("pad0", C.c_int32),
        ("prev_fitness", C.c_double),
    ]


class Profile(C.Structure):
    _fields_ = [
        ("sweeps", C.c_uint64),
        ("solve_ms", C.c_double),
        ("sweep1_ms", C.c_double),
        ("root_ttms", C.c_uint64),
        ("root_ttm_ms", C.c_double),
        ("root_ttm_flops", C.c_double),
        ("root_ttm_bytes", C.c_double),
        ("branch_ttm_ms", C.c_double),
        ("mode_update_ms", C.c_double),
        ("comm_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
        ("qr_shifted", C.c_uint64),
        ("qr_householder", C.c_uint64),
        ("gate_mispredictions", C.c_uint64),
    ]


Q0Observer = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_double),
                         C.c_uint64, C.c_uint64)

P = C.POINTER(C.c_double)
U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)
CTX = C.c_void_p

# name -> (restype, argtypes)
class ShardStep(C.Structure):
    _fields_ = [("src_layout", C.c_int32), ("src_mode", C.c_int32), ("out_layout", C.c_int32),
                ("out_mode", C.c_int32), ("reduction", C.c_int32), ("scatter_mode", C.c_int32),
                ("words", C.c_uint64)]


class ShardCost(C.Structure):
    _fields_ = [("tflops", C.c_double), ("bus_gbs", C.c_double), ("latency_s", C.c_double)]


SIGNATURES = {
    "cpdb_version": (C.c_char_p, []),
    "cpdb_last_error": (C.c_char_p, []),
    "cpdb_device_ok": (C.c_int, [C.c_int]),
    "cpdb_create": (C.c_int, [C.c_int, C.POINTER(CTX)]),
    "cpdb_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(CTX)]),
    "cpdb_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "cpdb_nccl_selftest": (C.c_int, [C.c_int, P]),
    "cpdb_destroy": (None, [CTX]),
    "cpdb_shard_rows": (C.c_int, [C.c_uint64, C.c_int, C.c_int, U64P, U64P]),
    "cpdb_tensor_set": (C.c_int, [CTX, P, U64P, C.c_uint32]),
    "cpdb_tensor_set_async": (C.c_int, [CTX, P, U64P, C.c_uint32]),
    "cpdb_tensor_set_device": (C.c_int, [CTX, C.c_void_p, U64P, C.c_uint32]),
    "cpdb_tensor_synth": (C.c_int, [CTX, C.c_int32, U64P, C.c_uint32, C.c_uint64, C.c_double,
                                    C.c_uint64]),
    "cpdb_tensor_synth_truth": (C.c_int, [CTX, C.c_int32, U64P, C.c_uint32, C.c_uint64,
                                          C.c_uint64, P]),
    "cpdb_tensor_synth_norms": (C.c_int, [CTX, P]),
    "cpdb_tensor_get": (C.c_int, [CTX, P]),
    "cpdb_shard_plan_ex": (C.c_int, [C.c_uint32, C.c_int32, C.c_uint64, U64P, C.c_uint64, C.c_int,
                                     C.c_int32, C.POINTER(ShardCost), C.POINTER(ShardStep),
                                     C.c_uint64, U64P, C.POINTER(C.c_int32), U64P, C.c_uint64,
                                     U64P, P]),
    "cpdb_set_shard_policy": (C.c_int, [CTX, C.c_int32, C.POINTER(ShardCost)]),
    "cpdb_create_local_group": (C.c_int, [C.c_int, C.c_int, C.POINTER(CTX)]),
    "cpdb_tensor_load_cpdt": (C.c_int, [CTX, C.c_char_p]),
    "cpdb_tensor_save_cpdt": (C.c_int, [CTX, C.c_char_p]),
    "cpdb_cpdt_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint32), U64P]),
    "cpdb_tensor_norm_sq": (C.c_int, [CTX, P]),
    "cpdb_solve": (C.c_int, [CTX, C.POINTER(Config), C.POINTER(State), C.POINTER(TraceRow), U64P,
                             P, P, P, P, Q0Observer, C.c_void_p]),
    "cpdb_session_begin": (C.c_int, [CTX, C.POINTER(Config), C.POINTER(State), C.POINTER(C.c_void_p)]),
    "cpdb_session_run": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(TraceRow), U64P,
                                   C.POINTER(C.c_int32)]),
    "cpdb_session_end": (C.c_int, [C.c_void_p, C.POINTER(State), P, P]),
    "cpdb_session_destroy": (None, [C.c_void_p]),
    "cpdb_profile_get": (C.c_int, [CTX, C.POINTER(Profile)]),
    "cpdb_set_options": (C.c_int, [CTX, C.c_int32, C.c_int32]),
    "cpdb_ttm": (C.c_int, [CTX, P, U64P, C.c_uint32, P, C.c_uint64, C.c_uint32, P]),
    "cpdb_unfold": (C.c_int, [CTX, P, U64P, C.c_uint32, C.c_uint32, P]),
    "cpdb_khatri_rao": (C.c_int, [CTX, C.POINTER(P), U64P, C.c_uint32, C.c_uint64, P]),
    "cpdb_thin_qr": (C.c_int, [CTX, P, C.c_uint64, C.c_uint64, P, P]),
    "cpdb_solve_rows_lower": (C.c_int, [CTX, P, C.c_uint64, P, C.c_uint64, P, I64P]),
    "cpdb_normalize_columns": (C.c_int, [CTX, P, C.c_uint64, C.c_uint64, P, P]),
    "cpdb_extrapolate_q0": (C.c_int, [CTX, P, P, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                      P]),
    "cpdb_fitness_fast_qr": (C.c_int, [CTX, C.c_double, P, P, C.c_uint64, P, P, P, C.c_uint64, P,
                                       P]),
    "cpdb_inner": (C.c_int, [CTX, P, P, C.c_uint64, P]),
    "cpdb_als_solve": (C.c_int, [CTX, C.POINTER(Config), P, P, C.POINTER(TraceRow), U64P, P, P]),
    "cpdb_mttkrp": (C.c_int, [CTX, P, U64P, C.c_uint32, C.POINTER(P), U64P, U64P, C.c_uint32, P]),
    "cpdb_solve_spd": (C.c_int, [CTX, P, C.c_uint64, C.c_uint64, P, C.c_uint64, C.c_uint64, P,
                                 C.POINTER(C.c_int32)]),
    "cpdb_fitness_fast_als": (C.c_int, [CTX, C.c_double, P, P, C.c_uint64, C.c_uint64, P, P,
                                        C.c_uint64, P, P, P]),
    "cpdb_select_beta": (C.c_int, [C.c_double, C.c_double, C.c_double, P]),
    "cpdb_schedule_build": (C.c_int, [C.c_uint32, C.c_int32, C.c_uint64, I64P, C.c_uint64, U64P,
                                      U64P]),
    "cpdb_schedule_validate": (C.c_int, [C.c_uint32, I64P, C.c_uint64, C.c_uint64]),
    "cpdb_retained_keys": (C.c_int, [C.c_uint32, I64P, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.POINTER(C.c_uint32), C.c_uint64, U64P]),
    "cpdb_measured_cost": (C.c_int, [C.c_uint32, C.c_int32, U64P, C.c_uint64, C.c_uint64, U64P,
                                     U64P]),
    "cpdb_closed_form_cost": (C.c_int, [C.c_uint32, C.c_int32, U64P, C.c_uint64, U64P]),
    "cpdb_leading_flop_coefficient": (C.c_int, [C.c_uint32, C.c_int32, U64P]),
    "cpdb_shard_plan": (C.c_int, [C.c_uint32, C.c_int32, C.c_uint64, U64P, C.c_uint64, C.c_int,
                                  C.POINTER(C.c_int32), U64P, C.c_uint64, U64P]),
    "cpdb_exec_step": (C.c_int, [CTX, C.c_uint32, C.c_uint32, C.c_uint32, P, C.c_uint64]),
    "cpdb_cache_dims": (C.c_int, [CTX, C.c_uint32, U64P, C.POINTER(C.c_int32)]),
    "cpdb_cache_get": (C.c_int, [CTX, C.c_uint32, P]),
    "cpdb_cache_drop": (C.c_int, [CTX, C.c_uint32]),
}

_LIB = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libcpdb.so once; raises when it was not built (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g;"
                          f" g.build()'` (make -C paper_2503_18759_b200/csrc)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def exported_symbols():
    return list(SIGNATURES)
