"""ctypes front-end for the CPU checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

Two libraries share one C signature set:
  * ``liboracle.so``       -- the C restatement (oracle/cpd_oracle.c), prefix ``cpdo_``
  * ``_ref/libcpdref.so``  -- the unmodified reference headers behind a C shim
                              (oracle/ref_runner.cpp), prefix ``cpdref_``

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAX_ORDER = 8

STRATEGIES = {"naive": 0, "dim-tree": 1, "dim_tree": 1, "branch-reuse": 2, "branch_reuse": 2}


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


Q0Observer = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_double),
                         C.c_uint64, C.c_uint64)

_P = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_P)


def _u64(vals) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(vals, dtype=np.uint64))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


@dataclass
class SolveOut:
    trace: List[dict]
    lam: np.ndarray
    factors: List[np.ndarray]
    factors_per_sweep: Optional[List[List[np.ndarray]]] = None
    lambda_per_sweep: Optional[np.ndarray] = None
    state: Optional[dict] = None


@dataclass
class SweepState:
    """Sweep-boundary solver state (see oracle/cpd_abi_types.h)."""
    sweeps_done: int
    lam: np.ndarray
    factors: List[np.ndarray]
    q0_history: Optional[List[Optional[np.ndarray]]] = None
    active_beta: Optional[float] = None
    prev_fitness: Optional[float] = None


def trace_to_dicts(rows, n) -> List[dict]:
    out = []
    for i in range(n):
        r = rows[i]
        out.append(dict(iteration=int(r.iteration),
                        update_order=[int(r.update_order[k]) for k in range(r.order)],
                        fitness=float(r.fitness), raw_radicand=float(r.raw_radicand),
                        wall_seconds=float(r.wall_seconds), root_ttm_count=int(r.root_ttm_count),
                        flops=int(r.flops), beta_used=float(r.beta_used),
                        regularized=bool(r.regularized)))
    return out


class Oracle:
    """One of the two CPU checkers.  ``kind`` is "port" (C restatement) or
    "reference" (the reference headers compiled in place)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            path, self.pre = os.path.join(HERE, "liboracle.so"), "cpdo_"
        elif kind == "reference":
            path, self.pre = os.path.join(HERE, "_ref", "libcpdref.so"), "cpdref_"
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.path = path
        self.lib = C.CDLL(path)
        f = self._f
        f("last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._f("last_error")().decode())

    # ---- .cpdt files (reference codec; kind "reference" only) -------------
    def write_tensor_file(self, path: str, x: np.ndarray) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64)
        d = np.asarray(x.shape, dtype=np.uint64)
        self._check(self._f("write_tensor_file")(os.fsencode(path), _dp(x),
                                                  d.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  C.c_uint32(x.ndim)))

    def read_tensor_file(self, path: str, cap: int = 1 << 26):
        """-> (rc, array or None); rc 8 file_error, 9 format_error"""
        order = C.c_uint32()
        dims = np.zeros(8, dtype=np.uint64)
        out = np.empty(cap)
        rc = self._f("read_tensor_file")(os.fsencode(path), C.byref(order),
                                         dims.ctypes.data_as(C.POINTER(C.c_uint64)), _dp(out),
                                         C.c_uint64(cap))
        if rc != 0:
            return rc, None
        shape = [int(v) for v in dims[: order.value]]
        return 0, out[: int(np.prod(shape))].reshape(shape).copy()

    def assemble_noisy(self, dims, rank, collinearity, l1, l2, seed) -> np.ndarray:
        """reference synth.hpp:80-106 (kind "reference" only)"""
        d = np.asarray(dims, dtype=np.uint64)
        c = np.ascontiguousarray(collinearity, dtype=np.float64)
        out = np.empty(int(np.prod(dims)))
        self._check(self._f("assemble_noisy")(d.ctypes.data_as(C.POINTER(C.c_uint64)),
                                              C.c_uint32(len(dims)), C.c_uint64(rank), _dp(c),
                                              C.c_double(l1), C.c_double(l2),
                                              C.c_uint64(seed), _dp(out)))
        return out.reshape([int(v) for v in dims])

    # ---- primitives -------------------------------------------------------
    def rng_normals(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self._check(self._f("rng_normals")(C.c_uint64(seed), C.c_uint64(n), _dp(out)))
        return out

    def ttm(self, t: np.ndarray, b: np.ndarray, mode: int) -> np.ndarray:
        t = np.ascontiguousarray(t, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        dims = _u64(t.shape)
        od = list(t.shape)
        od[mode] = b.shape[0]
        out = np.empty(od)
        if b.shape[1] != t.shape[mode]:
            raise ValueError("ttm: matrix columns do not match mode extent")
        self._check(self._f("ttm")(_dp(t), dims.ctypes.data_as(_U64P), C.c_uint32(t.ndim), _dp(b),
                                   C.c_uint64(b.shape[0]), C.c_uint32(mode), _dp(out)))
        return out

    def unfold(self, t: np.ndarray, mode: int) -> np.ndarray:
        t = np.ascontiguousarray(t, dtype=np.float64)
        out = np.empty((t.shape[mode], t.size // t.shape[mode]))
        dims = _u64(t.shape)
        self._check(self._f("unfold")(_dp(t), dims.ctypes.data_as(_U64P), C.c_uint32(t.ndim),
                                      C.c_uint32(mode), _dp(out)))
        return out

    def khatri_rao(self, mats: Sequence[np.ndarray]) -> np.ndarray:
        ms = [np.ascontiguousarray(m, dtype=np.float64) for m in mats]
        ptrs = (_P * len(ms))(*[_dp(m) for m in ms])
        rows = _u64([m.shape[0] for m in ms])
        out = np.empty((int(np.prod([m.shape[0] for m in ms])), ms[0].shape[1]))
        self._check(self._f("khatri_rao")(ptrs, rows.ctypes.data_as(_U64P), C.c_uint32(len(ms)),
                                          C.c_uint64(ms[0].shape[1]), _dp(out)))
        return out

    def thin_qr(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, n = a.shape
        q, r = np.empty((m, n)), np.empty((n, n))
        self._check(self._f("thin_qr")(_dp(a), C.c_uint64(m), C.c_uint64(n), _dp(q), _dp(r)))
        return q, r

    def solve_rows_lower(self, l: np.ndarray, rhs: np.ndarray):
        l = np.ascontiguousarray(l, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.empty_like(rhs)
        bad = C.c_int64(-1)
        rc = self._f("solve_rows_lower")(_dp(l), C.c_uint64(l.shape[0]), _dp(rhs),
                                         C.c_uint64(rhs.shape[0]), _dp(out), C.byref(bad))
        self._check(rc)
        return out

    def normalize_columns(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out, w = np.empty_like(a), np.empty(a.shape[1])
        self._check(self._f("normalize_columns")(_dp(a), C.c_uint64(a.shape[0]),
                                                 C.c_uint64(a.shape[1]), _dp(out), _dp(w)))
        return out, w

    def extrapolate_q0(self, now, prev, beta, alpha):
        now = np.ascontiguousarray(now, dtype=np.float64)
        prev = np.ascontiguousarray(prev, dtype=np.float64)
        out = np.empty_like(now)
        self._check(self._f("extrapolate_q0")(_dp(now), _dp(prev), C.c_uint64(now.shape[0]),
                                              C.c_uint64(now.shape[1]), C.c_double(beta),
                                              C.c_double(alpha), _dp(out)))
        return out

    def select_beta(self, prev, now, gap):
        b = C.c_double(0)
        on = self._f("select_beta")(C.c_double(prev), C.c_double(now), C.c_double(gap), C.byref(b))
        return b.value if on else None

    def fitness_fast_qr(self, nx2, v, a_hat, r0, r_n, lam):
        v, a_hat, r0, r_n, lam = (np.ascontiguousarray(z, dtype=np.float64)
                                  for z in (v, a_hat, r0, r_n, lam))
        fit, raw = C.c_double(), C.c_double()
        self._check(self._f("fitness_fast_qr")(C.c_double(nx2), _dp(v), _dp(a_hat),
                                               C.c_uint64(v.shape[0]), _dp(r0), _dp(r_n),
                                               _dp(lam), C.c_uint64(lam.size), C.byref(fit),
                                               C.byref(raw)))
        return fit.value, raw.value

    # ---- schedules ----------------------------------------------------------
    def schedule(self, order: int, strategy, iterations: int):
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        cap = 64 * iterations * order
        out = np.zeros((cap, 6), dtype=np.int64)
        n, cyc = C.c_uint64(), (C.c_uint64 * 2)()
        self._check(self._f("schedule")(C.c_uint32(order), C.c_int32(s), C.c_uint64(iterations),
                                        out.ctypes.data_as(C.POINTER(C.c_int64)), C.c_uint64(cap),
                                        C.byref(n), cyc))
        return out[: n.value].copy(), (int(cyc[0]), int(cyc[1]))

    def retained_keys(self, order, strategy, iterations, it, block):
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        out = (C.c_uint32 * 256)()
        n = C.c_uint64()
        self._check(self._f("retained_keys")(C.c_uint32(order), C.c_int32(s),
                                             C.c_uint64(iterations), C.c_uint64(it),
                                             C.c_uint64(block), out, C.c_uint64(256), C.byref(n)))
        return [int(out[i]) for i in range(n.value)]

    def measured_cost(self, order, strategy, dims, rank, iterations):
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        d = _u64(dims)
        fl, ro = C.c_uint64(), C.c_uint64()
        self._check(self._f("measured_cost")(C.c_uint32(order), C.c_int32(s),
                                             d.ctypes.data_as(_U64P), C.c_uint64(rank),
                                             C.c_uint64(iterations), C.byref(fl), C.byref(ro)))
        return fl.value, ro.value

    def execute_run(self, x, rank, strategy, iterations, seed, init_factors):
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        x = np.ascontiguousarray(x, dtype=np.float64)
        dims = list(x.shape)
        order = len(dims)
        init = np.concatenate([np.ascontiguousarray(f, dtype=np.float64).ravel()
                               for f in init_factors])
        sched, _ = self.schedule(order, s, iterations)
        # output sizes: one Y per update (I_mode x R^(N-1))
        ys = []
        for it in range(iterations):
            modes = []
            for row in sched[sched[:, 0] == it]:
                if int(row[2]) not in modes:
                    modes.append(int(row[2]))
            for m in modes:
                shp = [rank] * order
                shp[m] = dims[m]
                ys.append(shp)
        total = sum(int(np.prod(s_)) for s_ in ys)
        out = np.empty(total)
        fl = np.zeros(len(ys), dtype=np.uint64)
        d = _u64(dims)
        self._check(self._f("execute_run")(_dp(x), d.ctypes.data_as(_U64P), C.c_uint32(order),
                                           C.c_uint64(rank), C.c_int32(s), C.c_uint64(iterations),
                                           C.c_uint64(seed), _dp(init), _dp(out),
                                           fl.ctypes.data_as(_U64P)))
        res, off = [], 0
        for shp in ys:
            n = int(np.prod(shp))
            res.append(out[off:off + n].reshape(shp))
            off += n
        return res, [int(v) for v in fl]

    # ---- solver ---------------------------------------------------------------
    def solve(self, x: np.ndarray, rank: int, iterations: int, *, extrapolate: bool = True,
              strategy="branch-reuse", seed: int = 0, alpha: float = 0.1,
              beta_override: Optional[float] = None, activation_gap: float = 0.03,
              fitness_threshold: float = 1.0, state: Optional[SweepState] = None,
              dump_per_sweep: bool = False,
              q0_observer: Optional[Callable[[int, int, np.ndarray], None]] = None) -> SolveOut:
        x = np.ascontiguousarray(x, dtype=np.float64)
        dims = list(x.shape)
        order = len(dims)
        cfg = Config(rank=rank, max_iterations=iterations, fitness_threshold=fitness_threshold,
                     strategy=STRATEGIES[strategy] if isinstance(strategy, str) else strategy,
                     extrapolate=1 if extrapolate else 0, alpha=alpha,
                     has_beta_override=0 if beta_override is None else 1,
                     beta_override=0.0 if beta_override is None else beta_override,
                     activation_gap=activation_gap, seed=seed)
        nfac = sum(d * rank for d in dims)
        zrows = rank ** (order - 1)
        trace = (TraceRow * iterations)()
        tlen = C.c_uint64()
        lam = np.empty(rank)
        fac = np.empty(nfac)
        fps = np.empty((iterations, nfac)) if dump_per_sweep else None
        lps = np.empty((iterations, rank)) if dump_per_sweep else None
        st_ptr = None
        keep = []
        if state is not None:
            s_lam = np.ascontiguousarray(state.lam, dtype=np.float64).copy()
            s_fac = np.concatenate([np.ascontiguousarray(f, dtype=np.float64).ravel()
                                    for f in state.factors])
            s_hist = np.zeros(order * zrows * rank)
            mask = 0
            if state.q0_history is not None:
                for n, h in enumerate(state.q0_history):
                    if h is not None:
                        s_hist[n * zrows * rank:(n + 1) * zrows * rank] = np.asarray(h).ravel()
                        mask |= 1 << n
            keep = [s_lam, s_fac, s_hist]
            st = State(sweeps_done=state.sweeps_done, lam=_dp(s_lam), factors=_dp(s_fac),
                       q0_history=_dp(s_hist), history_mask=mask,
                       has_active_beta=0 if state.active_beta is None else 1,
                       active_beta=0.0 if state.active_beta is None else state.active_beta,
                       has_prev_fitness=0 if state.prev_fitness is None else 1,
                       prev_fitness=0.0 if state.prev_fitness is None else state.prev_fitness)
            st_ptr = C.byref(st)
        cb = None
        if q0_observer is not None:
            def _cb(_u, sweep, mode, ptr, rows, cols):
                q0_observer(int(sweep), int(mode),
                            np.ctypeslib.as_array(ptr, shape=(rows * cols,)).reshape(rows, cols).copy())
            cb = Q0Observer(_cb)
        rc = self._f("solve")(_dp(x), _u64(dims).ctypes.data_as(_U64P), C.c_uint32(order),
                              C.byref(cfg), st_ptr, trace, C.byref(tlen), _dp(lam), _dp(fac),
                              None if fps is None else _dp(fps),
                              None if lps is None else _dp(lps), cb, None)
        self._check(rc)
        n = tlen.value

        def split(flat):
            out, off = [], 0
            for d in dims:
                out.append(flat[off:off + d * rank].reshape(d, rank).copy())
                off += d * rank
            return out

        res = SolveOut(trace=trace_to_dicts(trace, n), lam=lam, factors=split(fac))
        if dump_per_sweep:
            res.factors_per_sweep = [split(fps[i]) for i in range(n)]
            res.lambda_per_sweep = lps[:n].copy()
        if state is not None:
            s_lam, s_fac, s_hist = keep
            res.state = dict(sweeps_done=int(st.sweeps_done), lam=s_lam.copy(),
                             factors=split(s_fac),
                             q0_history=[s_hist[k * zrows * rank:(k + 1) * zrows * rank]
                                         .reshape(zrows, rank).copy()
                                         if st.history_mask & (1 << k) else None
                                         for k in range(order)],
                             active_beta=float(st.active_beta) if st.has_active_beta else None,
                             prev_fitness=float(st.prev_fitness) if st.has_prev_fitness else None)
        return res

    # ---- CP-ALS, normal equations (solvers.hpp:149-208) --------------------
    def cp_als(self, x: np.ndarray, rank: int, iterations: int, *, seed: int = 0,
               fitness_threshold: float = 1.0, init_lam=None, init_factors=None) -> SolveOut:
        x = np.ascontiguousarray(x, dtype=np.float64)
        dims = list(x.shape)
        cfg = Config(rank=rank, max_iterations=iterations, fitness_threshold=fitness_threshold,
                     strategy=0, extrapolate=0, alpha=0.1, has_beta_override=0, beta_override=0.0,
                     activation_gap=0.03, seed=seed)
        trace = (TraceRow * iterations)()
        tlen = C.c_uint64()
        lam = np.empty(rank)
        fac = np.empty(sum(d * rank for d in dims))
        il = None if init_lam is None else np.ascontiguousarray(init_lam, dtype=np.float64)
        ifa = None if init_factors is None else np.concatenate(
            [np.ascontiguousarray(f, dtype=np.float64).ravel() for f in init_factors])
        self._check(self._f("cp_als")(_dp(x), _u64(dims).ctypes.data_as(_U64P), C.c_uint32(len(dims)),
                                      C.byref(cfg), None if il is None else _dp(il),
                                      None if ifa is None else _dp(ifa), trace, C.byref(tlen),
                                      _dp(lam), _dp(fac)))
        out, off = [], 0
        for d in dims:
            out.append(fac[off:off + d * rank].reshape(d, rank).copy())
            off += d * rank
        return SolveOut(trace=trace_to_dicts(trace, tlen.value), lam=lam, factors=out)

    def mttkrp(self, t: np.ndarray, factors, mode: int) -> np.ndarray:
        t = np.ascontiguousarray(t, dtype=np.float64)
        ms = [None if f is None else np.ascontiguousarray(f, dtype=np.float64) for f in factors]
        rank = next(m.shape[1] for k, m in enumerate(ms) if k != mode and m is not None)
        ptrs = (_P * len(ms))(*[None if m is None else _dp(m) for m in ms])
        out = np.empty((t.shape[mode], rank))
        self._check(self._f("mttkrp")(_dp(t), _u64(t.shape).ctypes.data_as(_U64P),
                                      C.c_uint32(t.ndim), ptrs, C.c_uint64(rank),
                                      C.c_uint32(mode), _dp(out)))
        return out

    def solve_spd(self, g: np.ndarray, rhs: np.ndarray):
        g = np.ascontiguousarray(g, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty_like(rhs)
        reg = C.c_int32()
        self._check(self._f("solve_spd")(_dp(g), C.c_uint64(g.shape[0]), _dp(rhs),
                                         C.c_uint64(rhs.shape[0]), _dp(x), C.byref(reg)))
        return x, bool(reg.value)

    def fitness_fast_als(self, nx2, m, a_hat, gamma, lam, s_last):
        m, a_hat, gamma, lam, s_last = (np.ascontiguousarray(z, dtype=np.float64)
                                        for z in (m, a_hat, gamma, lam, s_last))
        fit, raw = C.c_double(), C.c_double()
        self._check(self._f("fitness_fast_als")(C.c_double(nx2), _dp(m), _dp(a_hat),
                                                C.c_uint64(m.shape[0]), C.c_uint64(m.shape[1]),
                                                _dp(gamma), _dp(lam), C.c_uint64(lam.size),
                                                _dp(s_last), C.byref(fit), C.byref(raw)))
        return fit.value, raw.value

    def reconstruct(self, factors, lam=None) -> np.ndarray:
        """kruskal.hpp:54-67 reconstruct."""
        dims = [int(f.shape[0]) for f in factors]
        rank = int(factors[0].shape[1])
        lam = np.ones(rank) if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
        flat = np.ascontiguousarray(np.concatenate([np.ascontiguousarray(f).ravel()
                                                    for f in factors]))
        out = np.empty(dims)
        d = _u64(dims)
        self._check(self._f("reconstruct")(d.ctypes.data_as(_U64P), C.c_uint32(len(dims)),
                                           C.c_uint64(rank), _dp(lam), _dp(flat), _dp(out)))
        return out

    def synth_baseline(self, kind: int, dims, rank: int, rho: float, seed: int,
                       want_truth: bool = False):
        d = _u64(dims)
        out = np.empty([int(v) for v in dims])
        truth = np.empty(sum(int(v) * rank for v in dims)) if want_truth else None
        self._check(self._f("synth_baseline")(C.c_int32(kind), d.ctypes.data_as(_U64P),
                                              C.c_uint32(len(dims)), C.c_uint64(rank),
                                              C.c_double(rho), C.c_uint64(seed), _dp(out),
                                              None if truth is None else _dp(truth)))
        if want_truth:
            fs, off = [], 0
            for v in dims:
                fs.append(truth[off:off + int(v) * rank].reshape(int(v), rank))
                off += int(v) * rank
            return out, fs
        return out


def available(kind: str) -> bool:
    p = os.path.join(HERE, "liboracle.so") if kind == "port" else os.path.join(HERE, "_ref",
                                                                                "libcpdref.so")
    return os.path.exists(p)
