"""B200-native CP-ALS-QR hot path (arXiv 2503.18759) -- Python mirror of the
reference's ``cpd`` C++ interface over the libcpdb C ABI (include/cpdb.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/cpd (file:line cited per function).  All
arithmetic runs in libcpdb.so on an sm_100a device; nothing here computes,
and there is no CPU fallback: a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _cpdb

__all__ = [
    "CpdError", "StaleIntermediateError", "SingularTriangularError", "Context", "default_context",
    "SolverConfig", "TraceRow", "KruskalModel", "SolveResult", "SweepState", "Strategy",
    "cp_als_qr", "als_qr_bre", "ttm", "unfold", "khatri_rao", "thin_qr",
    "solve_rows_lower_triangular", "normalize_columns", "extrapolate_q0", "select_beta",
    "fitness_fast_qr", "inner", "build_schedule", "validate_schedule", "retained_keys",
    "measured_cost", "closed_form_cost", "leading_flop_coefficient", "Schedule",
    "ContractionStep", "ModeUpdate", "FactorState", "IntermediateCache", "execute",
]


# ---------------------------------------------------------------- errors
class CpdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class StaleIntermediateError(CpdError):
    """dim_tree.hpp:21-23"""


class SingularTriangularError(CpdError):
    """linalg.hpp:19-26; ``column`` is the failing diagonal entry."""

    def __init__(self, code, msg, column=-1):
        super().__init__(code, msg)
        self.column = column


class CpdInvalidArgument(CpdError, ValueError):
    """std::invalid_argument"""


class CpdLogicError(CpdError):
    """std::logic_error"""


class CudaError(CpdError):
    pass


class FileError(CpdError, OSError):
    """io.hpp:21-23 file_error (cannot open / read / write)"""


class FormatError(CpdError):
    """io.hpp:25-27 format_error (malformed .cpdt payload)"""


class SingularSystemError(CpdError):
    """linalg.hpp:15-17 singular_system_error (solve_spd failed after the ridge)"""


def _lib():
    return _cpdb.load()


def _raise(rc: int, column: int = -1):
    if rc == _cpdb.OK:
        return
    msg = _lib().cpdb_last_error().decode()
    if rc == _cpdb.INVALID_ARGUMENT:
        raise CpdInvalidArgument(rc, msg)
    if rc == _cpdb.STALE_INTERMEDIATE:
        raise StaleIntermediateError(rc, msg)
    if rc == _cpdb.SINGULAR_TRIANGULAR:
        raise SingularTriangularError(rc, msg, column)
    if rc == _cpdb.LOGIC_ERROR:
        raise CpdLogicError(rc, msg)
    if rc == _cpdb.FILE_ERROR:
        raise FileError(rc, msg)
    if rc == _cpdb.FORMAT_ERROR:
        raise FormatError(rc, msg)
    if rc == _cpdb.SINGULAR_SYSTEM:
        raise SingularSystemError(rc, msg)
    raise CudaError(rc, msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_cpdb.P)


def _u64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64))


def _up(a: np.ndarray):
    return a.ctypes.data_as(_cpdb.U64P)


STRATEGIES = {"naive": 0, "dim-tree": 1, "dim_tree": 1, "branch-reuse": 2, "branch_reuse": 2}


class Strategy:
    naive = 0
    dim_tree = 1
    branch_reuse = 2


def _strategy(s) -> int:
    return STRATEGIES[s] if isinstance(s, str) else int(s)


# ---------------------------------------------------------------- context
class Context:
    """One device, one stream, all device buffers (include/cpdb.h)."""

    def __init__(self, device: int = 0, *, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None):
        lib = _lib()
        h = _cpdb.CTX()
        if world > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("sharded context needs the 128-byte NCCL unique id")
            buf = C.create_string_buffer(nccl_id, 128)
            _raise(lib.cpdb_create_sharded(device, rank, world, buf, C.byref(h)))
        else:
            _raise(lib.cpdb_create(device, C.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    @classmethod
    def local_group(cls, device: int, world: int) -> List["Context"]:
        """`world` mode-0 shard ranks inside this process on one device (each
        must be driven from its own thread); collectives use a shared device
        buffer instead of NCCL -- exercises the sharded path on one GPU."""
        hs = (_cpdb.CTX * world)()
        _raise(_lib().cpdb_create_local_group(device, world, hs))
        out = []
        for r in range(world):
            ctx = cls.__new__(cls)
            ctx._h = _cpdb.CTX(hs[r])
            ctx.device, ctx.rank, ctx.world = device, r, world
            out.append(ctx)
        return out

    @staticmethod
    def nccl_selftest(device: int = 0) -> float:
        """The sharded path's NCCL calls on a one-rank communicator
        (cpdb_nccl_selftest): returns the max error (0.0 when they work)."""
        out = np.zeros(1)
        _raise(_lib().cpdb_nccl_selftest(device, _p(out)))
        return float(out[0])

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _raise(_lib().cpdb_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "_h", None):
            _lib().cpdb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---- X
    def set_tensor(self, x: np.ndarray, dims: Optional[Sequence[int]] = None, wait: bool = True):
        """Upload X (sharded contexts: this rank's slab; ``dims`` = global).
        ``wait=False`` queues the copy and returns (cpdb_tensor_set_async): the
        array is kept alive by the context, must not be modified until the
        next solve / session begin / norm_sq, and should be page-locked for
        the copy to overlap the host side of that call."""
        x = _f64(x)
        d = _u64(dims if dims is not None else x.shape)
        if wait:
            _raise(_lib().cpdb_tensor_set(self._h, _p(x), _up(d), len(d)))
            self._pending_host = None
        else:
            self._pending_host = x  # (the upload reads it until the next synchronising call)
            _raise(_lib().cpdb_tensor_set_async(self._h, _p(x), _up(d), len(d)))
        self.dims = [int(v) for v in d]

    def set_tensor_device(self, ptr: int, dims: Sequence[int]):
        d = _u64(dims)
        _raise(_lib().cpdb_tensor_set_device(self._h, C.c_void_p(ptr), _up(d), len(d)))
        self.dims = [int(v) for v in d]

    def synth_tensor(self, kind: int, dims: Sequence[int], rank: int, rho: float, seed: int):
        d = _u64(dims)
        _raise(_lib().cpdb_tensor_synth(self._h, kind, _up(d), len(d), rank, rho, seed))
        self.dims = [int(v) for v in d]

    def set_shard_policy(self, policy="auto", cost: Optional[dict] = None):
        """Reduction strategy of this context's sharded sessions (shard_plan_ex)."""
        pol = SHARD_POLICIES[policy] if isinstance(policy, str) else int(policy)
        _raise(_lib().cpdb_set_shard_policy(self._h, pol, _shard_cost(cost)))

    def synth_truth(self, kind: int, dims: Sequence[int], rank: int, seed: int) -> List[np.ndarray]:
        """The truth factors synth_tensor builds X from (lambda = 1)."""
        d = _u64(dims)
        flat = np.empty(sum(int(v) * rank for v in dims))
        _raise(_lib().cpdb_tensor_synth_truth(self._h, kind, _up(d), len(d), rank, seed, _p(flat)))
        out, off = [], 0
        for v in dims:
            out.append(flat[off:off + int(v) * rank].reshape(int(v), rank).copy())
            off += int(v) * rank
        return out

    def synth_norms(self):
        """(||X_clean||^2, ||E||^2) of the last synth_tensor (global over ranks)."""
        out = np.zeros(2)
        _raise(_lib().cpdb_tensor_synth_norms(self._h, _p(out)))
        return float(out[0]), float(out[1])

    def load_tensor(self, path: str):
        """Stream a .cpdt file (io.hpp:93-121) straight into HBM; a sharded
        context reads only its mode-0 slab."""
        _raise(_lib().cpdb_tensor_load_cpdt(self._h, os.fsencode(path)))
        self.dims = cpdt_info(path)

    def save_tensor(self, path: str):
        _raise(_lib().cpdb_tensor_save_cpdt(self._h, os.fsencode(path)))

    def get_tensor(self, local_dims: Sequence[int]) -> np.ndarray:
        out = np.empty([int(v) for v in local_dims])
        _raise(_lib().cpdb_tensor_get(self._h, _p(out)))
        return out

    def norm_sq(self) -> float:
        v = C.c_double()
        _raise(_lib().cpdb_tensor_norm_sq(self._h, C.byref(v)))
        return v.value

    def profile(self) -> dict:
        p = _cpdb.Profile()
        _raise(_lib().cpdb_profile_get(self._h, C.byref(p)))
        return {name: getattr(p, name) for name, _ in p._fields_}

    def set_options(self, timing: bool = True, overlap: bool = True):
        """timing: per-kernel CUDA events; overlap: root-TTM prefetch on a
        low-priority stream (off = every TTM in order, the kernel alone)."""
        _raise(_lib().cpdb_set_options(self._h, int(timing), int(overlap)))

    # ---- solver
    def session(self, cfg: "SolverConfig", *, extrapolate: bool) -> "SolverSession":
        """Resumable run_qr (cpdb_session_*): begin now, then run(n) sweeps at a time."""
        return SolverSession(self, cfg, extrapolate)

    def solve(self, cfg: "SolverConfig", *, extrapolate: bool, init: Optional["KruskalModel"] = None,
              state: Optional["SweepState"] = None, dump_per_sweep: bool = False) -> "SolveResult":
        dims = self.dims
        order = len(dims)
        R = int(cfg.rank)
        c = _cpdb.Config(rank=R, max_iterations=int(cfg.max_iterations),
                         fitness_threshold=float(cfg.fitness_threshold),
                         strategy=_strategy(cfg.strategy), extrapolate=1 if extrapolate else 0,
                         alpha=float(cfg.alpha),
                         has_beta_override=0 if cfg.beta_override is None else 1,
                         beta_override=0.0 if cfg.beta_override is None else float(cfg.beta_override),
                         activation_gap=float(cfg.activation_gap), seed=int(cfg.seed))
        nfac = sum(d * R for d in dims)
        zrows = R ** (order - 1)
        iters = int(cfg.max_iterations)
        trace = (_cpdb.TraceRow * iters)()
        tlen = C.c_uint64()
        lam = np.empty(R)
        fac = np.empty(nfac)
        fps = np.empty((iters, nfac)) if dump_per_sweep else None
        lps = np.empty((iters, R)) if dump_per_sweep else None
        st = None
        keep = None
        if state is None and init is not None:
            state = SweepState(0, np.asarray(init.lam, dtype=np.float64), list(init.factors))
        if state is not None:
            check_init_state(state, dims, R)
            s_lam = _f64(state.lam).copy()
            s_fac = np.concatenate([_f64(f).ravel() for f in state.factors])
            s_hist = np.zeros(order * zrows * R)
            mask = 0
            for n, h in enumerate(state.q0_history or []):
                if h is not None:
                    s_hist[n * zrows * R:(n + 1) * zrows * R] = np.asarray(h).ravel()
                    mask |= 1 << n
            keep = (s_lam, s_fac, s_hist)
            st = _cpdb.State(sweeps_done=int(state.sweeps_done), lam=_p(s_lam), factors=_p(s_fac),
                             q0_history=_p(s_hist), history_mask=mask,
                             has_active_beta=0 if state.active_beta is None else 1,
                             active_beta=0.0 if state.active_beta is None else state.active_beta,
                             has_prev_fitness=0 if state.prev_fitness is None else 1,
                             prev_fitness=0.0 if state.prev_fitness is None else state.prev_fitness)
        obs = _cpdb.Q0Observer()
        if cfg.q0_observer is not None:
            user_cb = cfg.q0_observer

            def _cb(_u, sweep, mode, ptr, rows, cols):
                q = np.ctypeslib.as_array(ptr, shape=(rows * cols,)).reshape(rows, cols).copy()
                user_cb(int(sweep), int(mode), q)

            obs = _cpdb.Q0Observer(_cb)
        rc = _lib().cpdb_solve(self._h, C.byref(c), None if st is None else C.byref(st), trace,
                               C.byref(tlen), _p(lam), _p(fac), None if fps is None else _p(fps),
                               None if lps is None else _p(lps), obs, None)
        _raise(rc)
        n = tlen.value

        def split(flat):
            out, off = [], 0
            for d in dims:
                out.append(flat[off:off + d * R].reshape(d, R).copy())
                off += d * R
            return out

        rows = [TraceRow.from_c(trace[i]) for i in range(n)]
        res = SolveResult(model=KruskalModel(lam.copy(), split(fac)), trace=rows)
        if dump_per_sweep:
            res.factors_per_sweep = [split(fps[i]) for i in range(n)]
            res.lambda_per_sweep = lps[:n].copy()
        if st is not None:
            s_lam, s_fac, s_hist = keep
            res.state = SweepState(
                sweeps_done=int(st.sweeps_done), lam=s_lam.copy(), factors=split(s_fac),
                q0_history=[s_hist[k * zrows * R:(k + 1) * zrows * R].reshape(zrows, R).copy()
                            if st.history_mask & (1 << k) else None for k in range(order)],
                active_beta=float(st.active_beta) if st.has_active_beta else None,
                prev_fitness=float(st.prev_fitness) if st.has_prev_fitness else None)
        return res


    def solve_als(self, cfg: "SolverConfig", init: Optional["KruskalModel"] = None) -> "SolveResult":
        """cp_als (solvers.hpp:149-208) on this context's tensor (cpdb_als_solve)."""
        dims = self.dims
        R = int(cfg.rank)
        c = _config(cfg, False)
        iters = int(cfg.max_iterations)
        trace = (_cpdb.TraceRow * iters)()
        tlen = C.c_uint64()
        lam = np.empty(R)
        fac = np.empty(sum(d * R for d in dims))
        il = if_ = None
        if init is not None:
            if len(init.factors) != len(dims) or init.rank() != R:
                raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT,
                                         "solver: init model does not match tensor/config")
            for f, d in zip(init.factors, dims):
                if np.asarray(f).shape[0] != d:
                    raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT,
                                             "solver: init factor rows do not match tensor")
            il = _f64(init.lam).copy()
            if_ = np.concatenate([_f64(f).ravel() for f in init.factors])
        _raise(_lib().cpdb_als_solve(self._h, C.byref(c), None if il is None else _p(il),
                                     None if if_ is None else _p(if_), trace, C.byref(tlen),
                                     _p(lam), _p(fac)))
        out, off = [], 0
        for d in dims:
            out.append(fac[off:off + d * R].reshape(d, R).copy())
            off += d * R
        rows = [TraceRow.from_c(trace[i]) for i in range(tlen.value)]
        return SolveResult(model=KruskalModel(lam.copy(), out), trace=rows)


def _config(cfg: "SolverConfig", extrapolate: bool) -> _cpdb.Config:
    return _cpdb.Config(rank=int(cfg.rank), max_iterations=int(cfg.max_iterations),
                        fitness_threshold=float(cfg.fitness_threshold),
                        strategy=_strategy(cfg.strategy), extrapolate=1 if extrapolate else 0,
                        alpha=float(cfg.alpha),
                        has_beta_override=0 if cfg.beta_override is None else 1,
                        beta_override=0.0 if cfg.beta_override is None else float(cfg.beta_override),
                        activation_gap=float(cfg.activation_gap), seed=int(cfg.seed))


def check_init_state(state: "SweepState", dims: Sequence[int], rank: int) -> None:
    """initial_factors' guard (solvers.hpp:105-112) for a given model or
    sweep-boundary state, BEFORE any buffer reaches the C ABI (which copies
    order x I_k x R factors, R weights and R^(N-1) x R Q0 histories blindly):
    order / rank mismatch -> "init model does not match tensor/config", row
    mismatch -> "init factor rows do not match tensor"."""
    order, R = len(dims), int(rank)
    facs = list(state.factors)
    lam = np.asarray(state.lam)
    if (len(facs) != order or lam.ndim != 1 or lam.shape[0] != R
            or any(np.asarray(f).ndim != 2 or np.asarray(f).shape[1] != R for f in facs)):
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT,
                                 "solver: init model does not match tensor/config")
    for f, d in zip(facs, dims):
        if np.asarray(f).shape[0] != d:
            raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT,
                                     "solver: init factor rows do not match tensor")
    if state.q0_history is not None:
        zrows = R ** (order - 1)
        hist = list(state.q0_history)
        if len(hist) > order or any(h is not None and np.asarray(h).shape != (zrows, R)
                                    for h in hist):
            raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT,
                                     "solver: Q0 history does not match tensor/config")


class SolverSession:
    """begin / run(n) / end over the context's tensor (include/cpdb.h)."""

    def __init__(self, ctx: Context, cfg: "SolverConfig", extrapolate: bool):
        self.ctx, self.cfg = ctx, cfg
        self._c = _config(cfg, extrapolate)
        h = C.c_void_p()
        _raise(_lib().cpdb_session_begin(ctx.handle, C.byref(self._c), None, C.byref(h)))
        self._h = h
        self.finished = False

    def run(self, sweeps: int) -> List["TraceRow"]:
        rows = (_cpdb.TraceRow * max(int(sweeps), 1))()
        n = C.c_uint64()
        fin = C.c_int32()
        _raise(_lib().cpdb_session_run(self._h, int(sweeps), rows, C.byref(n), C.byref(fin)))
        self.finished = bool(fin.value)
        return [TraceRow.from_c(rows[i]) for i in range(n.value)]

    def end(self) -> "KruskalModel":
        R = int(self.cfg.rank)
        lam = np.empty(R)
        fac = np.empty(sum(d * R for d in self.ctx.dims))
        _raise(_lib().cpdb_session_end(self._h, None, _p(lam), _p(fac)))
        out, off = [], 0
        for d in self.ctx.dims:
            out.append(fac[off:off + d * R].reshape(d, R).copy())
            off += d * R
        return KruskalModel(lam, out)

    def close(self):
        if getattr(self, "_h", None):
            _lib().cpdb_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(0)
    return _DEFAULT


# ---------------------------------------------------------------- value types
@dataclass
class SolverConfig:
    """solvers.hpp:25-50"""
    rank: int = 1
    max_iterations: int = 1
    fitness_threshold: float = 1.0
    algorithm: str = "als-qr"
    strategy: object = "naive"
    extrapolation_enabled: bool = False
    alpha: float = 0.1
    beta_override: Optional[float] = None
    activation_gap: float = 0.03
    seed: int = 0
    q0_observer: Optional[Callable[[int, int, np.ndarray], None]] = None


@dataclass
class TraceRow:
    """solvers.hpp:56-66"""
    iteration: int
    update_order: List[int]
    fitness: float
    raw_radicand: float
    wall_seconds: float
    root_ttm_count: int
    flops: int
    beta_used: float
    regularized: bool

    @staticmethod
    def from_c(r) -> "TraceRow":
        return TraceRow(int(r.iteration), [int(r.update_order[k]) for k in range(r.order)],
                        float(r.fitness), float(r.raw_radicand), float(r.wall_seconds),
                        int(r.root_ttm_count), int(r.flops), float(r.beta_used),
                        bool(r.regularized))

    def as_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class KruskalModel:
    """kruskal.hpp:16-31"""
    lam: np.ndarray
    factors: List[np.ndarray]

    def rank(self) -> int:
        return len(self.lam)

    def order(self) -> int:
        return len(self.factors)


@dataclass
class SweepState:
    """Sweep-boundary state for resume / teacher forcing (include/cpdb.h cpdb_state)."""
    sweeps_done: int
    lam: np.ndarray
    factors: List[np.ndarray]
    q0_history: Optional[List[Optional[np.ndarray]]] = None
    active_beta: Optional[float] = None
    prev_fitness: Optional[float] = None


@dataclass
class SolveResult:
    """solvers.hpp:68-71"""
    model: KruskalModel
    trace: List[TraceRow]
    factors_per_sweep: Optional[List[List[np.ndarray]]] = None
    lambda_per_sweep: Optional[np.ndarray] = None
    state: Optional[SweepState] = None


# ---------------------------------------------------------------- solvers
def _solve(x, cfg: SolverConfig, init, extrapolate: bool, ctx: Optional[Context], **kw):
    ctx = ctx or default_context()
    x = _f64(x)
    ctx.set_tensor(x)
    return ctx.solve(cfg, extrapolate=extrapolate, init=init, **kw)


def cp_als_qr(x, cfg: SolverConfig, init: Optional[KruskalModel] = None,
              ctx: Optional[Context] = None, **kw) -> SolveResult:
    """solvers.hpp:317-322"""
    if cfg.algorithm not in ("als-qr", "als_qr"):
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "cp_als_qr: config algorithm must be als-qr")
    return _solve(x, cfg, init, False, ctx, **kw)


def als_qr_bre(x, cfg: SolverConfig, init: Optional[KruskalModel] = None,
               ctx: Optional[Context] = None, **kw) -> SolveResult:
    """solvers.hpp:329-336 (forces branch reuse and extrapolation)"""
    return _solve(x, cfg, init, True, ctx, **kw)


def cp_als(x, cfg: SolverConfig, init: Optional[KruskalModel] = None,
           ctx: Optional[Context] = None) -> SolveResult:
    """solvers.hpp:149-208 (normal equations + MTTKRP)"""
    if cfg.algorithm not in ("als",):
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "cp_als: config algorithm must be als")
    ctx = ctx or default_context()
    ctx.set_tensor(_f64(x))
    return ctx.solve_als(cfg, init)


# ---------------------------------------------------------------- primitives
def mttkrp(t, factors: Sequence[Optional[np.ndarray]], mode: int,
           ctx: Optional[Context] = None) -> np.ndarray:
    """tensor.hpp:453-488 (factors[mode] is not read)"""
    ctx = ctx or default_context()
    t = _f64(t)
    order = t.ndim
    if len(factors) != order:
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "mttkrp: need one factor per mode")
    mats = [None if f is None else _f64(f) for f in factors]
    ptrs = (_cpdb.P * order)(*[None if m is None else _p(m) for m in mats])
    rows = _u64([0 if m is None else m.shape[0] for m in mats])
    cols = _u64([0 if m is None else (m.shape[1] if m.ndim == 2 else 1) for m in mats])
    rank = next((int(c) for k, c in enumerate(cols) if k != mode and mats[k] is not None), 0)
    out = np.empty((t.shape[mode] if 0 <= mode < order else 0, max(rank, 1)))
    _raise(_lib().cpdb_mttkrp(ctx.handle, _p(t.ravel()), _up(_u64(t.shape)), order, ptrs,
                              _up(rows), _up(cols), mode, _p(out)))
    return out


def solve_spd(g, rhs, ctx: Optional[Context] = None) -> Tuple[np.ndarray, bool]:
    """linalg.hpp:132-187 -> (x, regularized) with x G = rhs"""
    ctx = ctx or default_context()
    g, rhs = _f64(g), _f64(rhs)
    x = np.empty_like(rhs)
    reg = C.c_int32()
    _raise(_lib().cpdb_solve_spd(ctx.handle, _p(g), g.shape[0], g.shape[1], _p(rhs), rhs.shape[0],
                                 rhs.shape[1], _p(x), C.byref(reg)))
    return x, bool(reg.value)


def fitness_fast_als(norm_x_sq, m_last, a_hat_last, gamma_last, lam, s_last,
                     ctx: Optional[Context] = None):
    """kruskal.hpp:88-104 -> (fitness, raw_radicand)"""
    ctx = ctx or default_context()
    m, a, g, lam, s = (_f64(z) for z in (m_last, a_hat_last, gamma_last, lam, s_last))
    if not norm_x_sq > 0.0:
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "fitness_fast_als: zero-norm tensor")
    if m.shape != a.shape:
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "dot: dimension mismatch")
    r = lam.size
    if g.shape[0] != r or s.shape[0] != r:
        raise CpdInvalidArgument(_cpdb.INVALID_ARGUMENT, "fitness_fast_als: dimension mismatch")
    fit, raw = C.c_double(), C.c_double()
    _raise(_lib().cpdb_fitness_fast_als(ctx.handle, float(norm_x_sq), _p(m), _p(a), m.shape[0],
                                        m.shape[1], _p(g), _p(lam), r, _p(s), C.byref(fit),
                                        C.byref(raw)))
    return fit.value, raw.value


def ttm(t, b, mode: int, ctx: Optional[Context] = None) -> np.ndarray:
    """tensor.hpp:288-315: Y = t x_mode b, b is (rows x I_mode)."""
    ctx = ctx or default_context()
    t, b = _f64(t), _f64(b)
    if mode >= t.ndim:
        raise CpdInvalidArgument(1, "ttm: mode out of range")
    if b.ndim != 2 or b.shape[1] != t.shape[mode]:
        raise CpdInvalidArgument(1, "ttm: matrix columns do not match mode extent")
    od = list(t.shape)
    od[mode] = b.shape[0]
    out = np.empty(od)
    d = _u64(t.shape)
    _raise(_lib().cpdb_ttm(ctx.handle, _p(t), _up(d), t.ndim, _p(b), b.shape[0], mode, _p(out)))
    return out


def unfold(t, mode: int, ctx: Optional[Context] = None) -> np.ndarray:
    """tensor.hpp:217-250"""
    ctx = ctx or default_context()
    t = _f64(t)
    if mode >= t.ndim:
        raise CpdInvalidArgument(1, "unfold: mode out of range")
    out = np.empty((t.shape[mode], t.size // t.shape[mode]))
    d = _u64(t.shape)
    _raise(_lib().cpdb_unfold(ctx.handle, _p(t), _up(d), t.ndim, mode, _p(out)))
    return out


def khatri_rao(mats: Sequence[np.ndarray], ctx: Optional[Context] = None) -> np.ndarray:
    """tensor.hpp:343-368 (last argument's row index fastest)"""
    ctx = ctx or default_context()
    if len(mats) == 0:
        raise CpdInvalidArgument(1, "khatri_rao: empty list")
    ms = [_f64(m) for m in mats]
    cols = ms[0].shape[1]
    if any(m.shape[1] != cols for m in ms):
        raise CpdInvalidArgument(1, "khatri_rao: mismatched column counts")
    ptrs = (_cpdb.P * len(ms))(*[_p(m) for m in ms])
    rows = _u64([m.shape[0] for m in ms])
    out = np.empty((int(np.prod([m.shape[0] for m in ms])), cols))
    _raise(_lib().cpdb_khatri_rao(ctx.handle, ptrs, _up(rows), len(ms), cols, _p(out)))
    return out


def thin_qr(a, ctx: Optional[Context] = None) -> Tuple[np.ndarray, np.ndarray]:
    """linalg.hpp:39-99"""
    ctx = ctx or default_context()
    a = _f64(a)
    m, n = a.shape
    q, r = np.empty((m, n)), np.empty((n, n))
    _raise(_lib().cpdb_thin_qr(ctx.handle, _p(a), m, n, _p(q), _p(r)))
    return q, r


def solve_rows_lower_triangular(l, rhs, ctx: Optional[Context] = None) -> np.ndarray:
    """linalg.hpp:192-216"""
    ctx = ctx or default_context()
    l, rhs = _f64(l), _f64(rhs)
    if l.shape[0] != l.shape[1]:
        raise CpdInvalidArgument(1, "solve_rows_lower_triangular: L must be square")
    if rhs.shape[1] != l.shape[0]:
        raise CpdInvalidArgument(1, "solve_rows_lower_triangular: RHS columns must match L")
    out = np.empty_like(rhs)
    bad = C.c_int64(-1)
    rc = _lib().cpdb_solve_rows_lower(ctx.handle, _p(l), l.shape[0], _p(rhs), rhs.shape[0],
                                      _p(out), C.byref(bad))
    _raise(rc, int(bad.value))
    return out


def normalize_columns(a, ctx: Optional[Context] = None) -> Tuple[np.ndarray, np.ndarray]:
    """linalg.hpp:225-242"""
    ctx = ctx or default_context()
    a = _f64(a)
    out, w = np.empty_like(a), np.empty(a.shape[1])
    _raise(_lib().cpdb_normalize_columns(ctx.handle, _p(a), a.shape[0], a.shape[1], _p(out),
                                         _p(w)))
    return out, w


def extrapolate_q0(now, prev, beta: float, alpha: float, ctx: Optional[Context] = None):
    """solvers.hpp:75-86"""
    ctx = ctx or default_context()
    now, prev = _f64(now), _f64(prev)
    if now.shape != prev.shape:
        raise CpdInvalidArgument(1, "extrapolate_q0: shape mismatch")
    out = np.empty_like(now)
    _raise(_lib().cpdb_extrapolate_q0(ctx.handle, _p(now), _p(prev), now.shape[0], now.shape[1],
                                      beta, alpha, _p(out)))
    return out


def select_beta(fitness_prev: float, fitness_now: float, gap: float) -> Optional[float]:
    """solvers.hpp:92-101"""
    b = C.c_double()
    on = _lib().cpdb_select_beta(fitness_prev, fitness_now, gap, C.byref(b))
    return b.value if on else None


def fitness_fast_qr(norm_x_sq, v, a_hat, r0, r_n, lam, ctx: Optional[Context] = None):
    """kruskal.hpp:109-128 -> (fitness, raw_radicand)"""
    ctx = ctx or default_context()
    v, a_hat, r0, r_n, lam = (_f64(z) for z in (v, a_hat, r0, r_n, lam))
    if v.shape != a_hat.shape:
        raise CpdInvalidArgument(1, "fitness_fast_qr: V and A_hat dimensions differ")
    r = lam.size
    if r0.shape != (r, r) or r_n.shape != (r, r):
        raise CpdInvalidArgument(1, "fitness_fast_qr: triangular factor dimension mismatch")
    fit, raw = C.c_double(), C.c_double()
    _raise(_lib().cpdb_fitness_fast_qr(ctx.handle, float(norm_x_sq), _p(v), _p(a_hat), v.shape[0],
                                       _p(r0), _p(r_n), _p(lam), r, C.byref(fit), C.byref(raw)))
    return fit.value, raw.value


def inner(a, b, ctx: Optional[Context] = None) -> float:
    """tensor.hpp:394-399"""
    ctx = ctx or default_context()
    a, b = _f64(a), _f64(b)
    if a.shape != b.shape:
        raise CpdInvalidArgument(1, "inner: shape mismatch")
    out = C.c_double()
    _raise(_lib().cpdb_inner(ctx.handle, _p(a.ravel()), _p(b.ravel()), a.size, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- scheduler
@dataclass(frozen=True)
class ContractionStep:
    """dim_tree.hpp:59-63"""
    source: int
    contract_mode: int
    produces: int


@dataclass
class ModeUpdate:
    """dim_tree.hpp:67-70"""
    mode: int
    steps: List[ContractionStep]


@dataclass
class Schedule:
    """dim_tree.hpp:80-107"""
    order: int
    strategy: int
    iterations: List[List[ModeUpdate]]
    cycle_start: int
    cycle_length: int

    def num_iterations(self) -> int:
        return len(self.iterations)

    def iteration(self, i: int) -> List[ModeUpdate]:
        return self.iterations[i]

    def update_order(self, i: int) -> List[int]:
        return [u.mode for u in self.iterations[i]]

    def flat(self) -> np.ndarray:
        rows = []
        for i, it in enumerate(self.iterations):
            for b, u in enumerate(it):
                for s in u.steps:
                    rows.append((i, b, u.mode, s.source, s.contract_mode, s.produces))
        return np.ascontiguousarray(np.array(rows, dtype=np.int64).reshape(-1, 6))


def step(source: int, contract: int) -> ContractionStep:
    """dim_tree.hpp:196-199"""
    return ContractionStep(source, contract, source & ~(1 << contract))


def build_schedule(order: int, strategy, iterations: int) -> Schedule:
    """dim_tree.hpp:386-426"""
    s = _strategy(strategy)
    n = C.c_uint64()
    cyc = (C.c_uint64 * 2)()
    _raise(_lib().cpdb_schedule_build(order, s, iterations, None, 0, C.byref(n), cyc))
    flat = np.zeros((max(n.value, 1), 6), dtype=np.int64)
    _raise(_lib().cpdb_schedule_build(order, s, iterations, flat.ctypes.data_as(_cpdb.I64P),
                                      n.value, C.byref(n), cyc))
    its: List[List[ModeUpdate]] = [[] for _ in range(iterations)]
    for i, b, mode, src, c, prod in flat[: n.value]:
        ups = its[int(i)]
        while len(ups) <= b:
            ups.append(ModeUpdate(-1, []))
        ups[int(b)].mode = int(mode)
        ups[int(b)].steps.append(ContractionStep(int(src), int(c), int(prod)))
    return Schedule(order, s, its, int(cyc[0]), int(cyc[1]))


def validate_schedule(s: Schedule):
    """dim_tree.hpp:335-379 (raises on a stale or malformed plan)"""
    flat = s.flat()
    _raise(_lib().cpdb_schedule_validate(s.order, flat.ctypes.data_as(_cpdb.I64P), flat.shape[0],
                                         s.num_iterations()))


def retained_keys(s: Schedule, iteration: int, block: int) -> List[int]:
    """dim_tree.hpp:433-465"""
    flat = s.flat()
    keys = (C.c_uint32 * 256)()
    n = C.c_uint64()
    _raise(_lib().cpdb_retained_keys(s.order, flat.ctypes.data_as(_cpdb.I64P), flat.shape[0],
                                     s.num_iterations(), s.cycle_start, s.cycle_length, iteration,
                                     block, keys, 256, C.byref(n)))
    return [int(keys[i]) for i in range(n.value)]


def shard_rows(extent0: int, rank: int, world: int) -> Tuple[int, int]:
    """(begin, count) of the leading-mode rows `rank` owns (host only)."""
    b, n = C.c_uint64(), C.c_uint64()
    _raise(_lib().cpdb_shard_rows(extent0, rank, world, C.byref(b), C.byref(n)))
    return int(b.value), int(n.value)


def cpdt_info(path: str) -> List[int]:
    """Extents from a .cpdt header (host only, no device)."""
    order = C.c_uint32()
    dims = np.zeros(8, dtype=np.uint64)
    _raise(_lib().cpdb_cpdt_info(os.fsencode(path), C.byref(order), _up(dims)))
    return [int(v) for v in dims[: order.value]]


def measured_cost(order: int, strategy, dims: Sequence[int], rank: int,
                  iterations: int = 3) -> Tuple[int, int]:
    """dim_tree.hpp:549-570 -> (total_flops, root_ttm_count)"""
    d = _u64(dims)
    fl, ro = C.c_uint64(), C.c_uint64()
    _raise(_lib().cpdb_measured_cost(order, _strategy(strategy), _up(d), rank, iterations,
                                     C.byref(fl), C.byref(ro)))
    return fl.value, ro.value


SHARD_SRC_SHARDED, SHARD_ALLREDUCE, SHARD_OUT_SHARDED, SHARD_GATHER_V = 1, 2, 4, 8


def shard_plan(order: int, strategy, iterations: int, dims: Sequence[int], rank: int,
               world: int) -> Tuple[np.ndarray, np.ndarray]:
    """Mode-0 sharding plan the device session follows: per
    scheduled step (cpdb_schedule_build order) the SHARD_* flags and the number
    of doubles exchanged (all-reduce of a partial sum / all-gather of V)."""
    d = _u64(dims)
    n = C.c_uint64()
    _raise(_lib().cpdb_shard_plan(order, _strategy(strategy), iterations, _up(d), rank, world,
                                  None, None, 0, C.byref(n)))
    flags = np.zeros(n.value, dtype=np.int32)
    payload = np.zeros(n.value, dtype=np.uint64)
    _raise(_lib().cpdb_shard_plan(order, _strategy(strategy), iterations, _up(d), rank, world,
                                  flags.ctypes.data_as(C.POINTER(C.c_int32)), _up(payload),
                                  n.value, C.byref(n)))
    return flags, payload


SHARD_POLICIES = {"eager": 0, "scatter": 1, "lazy": 2, "auto": 3}
LAYOUTS = {0: "replicated", 1: "sharded", 2: "partial"}
REDUCTIONS = {0: None, 1: "allreduce", 2: "scatter"}
V_OPS = {0: None, 1: "gather", 2: "allreduce"}


def _shard_cost(cost):
    if cost is None:
        return None
    c = _cpdb.ShardCost(float(cost.get("tflops", 0.0)), float(cost.get("bus_gbs", 0.0)),
                        float(cost.get("latency_s", -1.0)))
    return C.byref(c)


def shard_plan_ex(order: int, strategy, iterations: int, dims: Sequence[int], rank: int,
                  world: int, policy="auto", cost: Optional[dict] = None) -> dict:
    """The sharded session's layouts and reductions (csrc/shard.cpp,
    cpdb_shard_plan_ex): per scheduled step {src, out: (layout, mode),
    reduction, scatter_mode, words}; per mode update the V collective and its
    size; the cost model's per-rank compute / communication seconds."""
    d = _u64(dims)
    pol = SHARD_POLICIES[policy] if isinstance(policy, str) else int(policy)
    ns, nu = C.c_uint64(), C.c_uint64()
    cst = _shard_cost(cost)
    _raise(_lib().cpdb_shard_plan_ex(order, _strategy(strategy), iterations, _up(d), rank, world,
                                     pol, cst, None, 0, C.byref(ns), None, None, 0, C.byref(nu),
                                     None))
    steps = (_cpdb.ShardStep * max(ns.value, 1))()
    vop = np.zeros(max(nu.value, 1), dtype=np.int32)
    vw = np.zeros(max(nu.value, 1), dtype=np.uint64)
    est = np.zeros(2)
    _raise(_lib().cpdb_shard_plan_ex(order, _strategy(strategy), iterations, _up(d), rank, world,
                                     pol, cst, steps, ns.value, C.byref(ns),
                                     vop.ctypes.data_as(C.POINTER(C.c_int32)), _up(vw), nu.value,
                                     C.byref(nu), _p(est)))
    out = []
    for i in range(ns.value):
        s_ = steps[i]
        out.append({"src": (LAYOUTS[s_.src_layout], s_.src_mode),
                    "out": (LAYOUTS[s_.out_layout], s_.out_mode),
                    "reduction": REDUCTIONS[s_.reduction], "scatter_mode": s_.scatter_mode,
                    "words": int(s_.words)})
    return {"steps": out, "v_ops": [V_OPS[int(v)] for v in vop[:nu.value]],
            "v_words": [int(v) for v in vw[:nu.value]],
            "est_compute_s": float(est[0]), "est_comm_s": float(est[1])}


def closed_form_cost(order: int, strategy, dims: Sequence[int], rank: int) -> int:
    """dim_tree.hpp:579-621"""
    d = _u64(dims)
    out = C.c_uint64()
    _raise(_lib().cpdb_closed_form_cost(order, _strategy(strategy), _up(d), rank, C.byref(out)))
    return out.value


def leading_flop_coefficient(order: int, strategy) -> int:
    """dim_tree.hpp:625-634"""
    out = C.c_uint64()
    _raise(_lib().cpdb_leading_flop_coefficient(order, _strategy(strategy), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- execute()
class FactorState:
    """factor_state.hpp:18-48 (host copy; thin_qr runs on the device)."""

    def __init__(self, factors: Sequence[np.ndarray], ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.factors = [_f64(f).copy() for f in factors]
        self.qr = [thin_qr(f, self.ctx) for f in self.factors]
        self.versions = [1] * len(self.factors)
        self.lam = np.ones(self.factors[0].shape[1])

    @staticmethod
    def from_factors(factors, ctx: Optional[Context] = None) -> "FactorState":
        return FactorState(factors, ctx)

    def order(self) -> int:
        return len(self.factors)

    def version(self, mode: int) -> int:
        return self.versions[mode]

    def q(self, mode: int) -> np.ndarray:
        return self.qr[mode][0]

    def r(self, mode: int) -> np.ndarray:
        return self.qr[mode][1]

    def update(self, mode: int, factor: np.ndarray):
        self.qr[mode] = thin_qr(factor, self.ctx)
        self.factors[mode] = _f64(factor).copy()
        self.versions[mode] += 1


class IntermediateCache:
    """dim_tree.hpp:112-139; tensors live in the context's HBM slots, the
    stamps stay on the host like the reference keeps them."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.stamps: Dict[int, Dict[int, int]] = {}
        self._x_id = None

    def size(self) -> int:
        return len(self.stamps)

    def find(self, key: int):
        return self.stamps.get(key)

    def clear(self):
        for k in list(self.stamps):
            _lib().cpdb_cache_drop(self.ctx.handle, k)
        self.stamps.clear()


def _mode_set_name(s: int, order: int) -> str:
    return "Y(" + ",".join(str(m + 1) for m in range(order) if s & (1 << m)) + ")"


def execute(schedule: Schedule, x, state: FactorState, cache: IntermediateCache, iteration: int,
            mode: int) -> Tuple[np.ndarray, dict]:
    """dim_tree.hpp:473-544: run one update's steps on the device, checking
    freshness and evicting exactly like the reference.  Returns (Y, cost)."""
    ctx = cache.ctx
    x = _f64(x)
    order = schedule.order
    if x.ndim != order or state.order() != order:
        raise CpdInvalidArgument(1, "execute: order mismatch")
    key = (x.__array_interface__["data"][0], x.shape, float(x.ravel()[0]), float(x.ravel()[-1]))
    if cache._x_id != key:
        ctx.set_tensor(x)
        cache._x_id = key
        cache.stamps.clear()
    it = schedule.iteration(iteration)
    block = next((b for b, u in enumerate(it) if u.mode == mode), None)
    if block is None:
        raise CpdInvalidArgument(1, "execute: mode not in iteration")
    root = (1 << order) - 1
    cost = {"categories": {}, "root_ttm_count": 0, "total_flops": 0}
    result = None
    for s in it[block].steps:
        if s.source == root:
            stamp: Dict[int, int] = {}
            src_key = _cpdb.ROOT_KEY
            src_dims = list(x.shape)
        else:
            entry = cache.stamps.get(s.source)
            if entry is None:
                raise CpdLogicError(_cpdb.LOGIC_ERROR, "execute: scheduled source " +
                                    _mode_set_name(s.source, order) + " missing from cache")
            for m, v in entry.items():
                if v != state.version(m):
                    raise StaleIntermediateError(
                        _cpdb.STALE_INTERMEDIATE,
                        f"execute: stale intermediate {_mode_set_name(s.source, order)} (mode "
                        f"{m + 1} stamped v{v}, current v{state.version(m)}) at iteration "
                        f"{iteration + 1}, update of mode {mode + 1}")
            stamp = dict(entry)
            src_key = s.source
            dims = (C.c_uint64 * 8)()
            present = C.c_int32()
            _raise(_lib().cpdb_cache_dims(ctx.handle, s.source, dims, C.byref(present)))
            src_dims = [int(dims[k]) for k in range(order)]
        c = s.contract_mode
        q = _f64(state.q(c))
        R = q.shape[1]
        _raise(_lib().cpdb_exec_step(ctx.handle, src_key, c, s.produces, _p(q), R))
        out_dims = list(src_dims)
        out_dims[c] = R
        flops = 2 * int(np.prod(out_dims)) * src_dims[c]
        r_power = order - bin(s.source).count("1") + 1
        cat = cost["categories"].setdefault((r_power, s.source), {"count": 0, "flops": 0})
        cat["count"] += 1
        cat["flops"] += flops
        cost["total_flops"] += flops
        if s.source == root:
            cost["root_ttm_count"] += 1
        stamp[c] = state.version(c)
        if s.produces == (1 << mode):
            result = np.empty(out_dims)
            _raise(_lib().cpdb_cache_get(ctx.handle, s.produces, _p(result)))
            _lib().cpdb_cache_drop(ctx.handle, s.produces)
        else:
            cache.stamps[s.produces] = stamp
    keep = retained_keys(schedule, iteration, block)
    for k in list(cache.stamps):
        if k not in keep:
            del cache.stamps[k]
            _lib().cpdb_cache_drop(ctx.handle, k)
    return result, cost
