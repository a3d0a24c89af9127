"""Teacher-forced parity of one device sweep against the oracle.

The device runs k ALS-QR-BRE sweeps from the reference's initial factors and
dumps the sweep-boundary state (factors, lambda, per-mode Q0 history, frozen
beta, previous fitness).  From that SAME state
  * the oracle (tests' checker: the C restatement, bit-identical to the
    reference compiled from /root/reference) runs one sweep,
  * the device runs one sweep twice: resumed from the dumped state (cache
    rebuilt from X), and as sweep k+1 of an uninterrupted k+1-sweep run (the
    steady path, no resume),
so the comparison isolates one sweep's kernel error from trajectory drift.

    python tools/teacher_forced.py c5 [k] [--dims 64x64x64x64] [--out file.json]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json configs (kind, dims, rank, rho)
    "c2": (0, (512, 512, 512), 32, 1e-3),
    "c3": (0, (128, 128, 128, 128), 16, 1e-2),
    "c4": (1, (256, 256, 256), 20, 1e-4),
    "c5": (0, (256, 256, 256, 256), 64, 1e-3),
}
TRUTH_SEED = {"c1": 20250001, "c2": 20250002, "c3": 20250003, "c4": 20250004, "c5": 20250005}
INIT_SEED = 7


def reference_init(port, dims, rank, seed):
    """initial_factors (solvers.hpp:116-122): N(0,1) draws mode by mode, normalised."""
    draws = port.rng_normals(seed, sum(d * rank for d in dims))
    out, off = [], 0
    for d in dims:
        out.append(port.normalize_columns(draws[off:off + d * rank].reshape(d, rank))[0])
        off += d * rank
    return out


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(kind, dims, rank, rho, truth_seed, k, port=None, ctx=None, log=print):
    import paper_2503_18759_b200 as cpd
    from oracle.pyoracle import Oracle, SweepState as OState
    port = port or Oracle("port")
    t0 = time.perf_counter()
    ctx = ctx or cpd.Context(0)
    ctx.synth_tensor(kind, list(dims), rank, rho, truth_seed)
    x = ctx.get_tensor(list(dims))
    log(f"tensor {dims} on the host ({x.nbytes / 1e9:.2f} GB) {time.perf_counter() - t0:.1f}s")
    init = reference_init(port, dims, rank, INIT_SEED)

    def cfg(n):
        return cpd.SolverConfig(rank=rank, max_iterations=n, seed=INIT_SEED)

    start = cpd.SweepState(0, np.ones(rank), [f.copy() for f in init])
    g0 = ctx.solve(cfg(k), extrapolate=True, state=start)
    st = g0.state
    g_cont = ctx.solve(cfg(k + 1), extrapolate=True,
                       state=cpd.SweepState(0, np.ones(rank), [f.copy() for f in init]))
    g_res = ctx.solve(cfg(1), extrapolate=True, state=dataclasses.replace(st))
    t1 = time.perf_counter()
    o = port.solve(x, rank, 1, extrapolate=True, seed=INIT_SEED,
                   state=OState(**dataclasses.asdict(st)))
    t_or = time.perf_counter() - t1
    log(f"oracle sweep {k + 1}: {t_or:.1f}s")
    ot = o.trace[0]
    out = {"dims": list(dims), "rank": rank, "rho": rho, "k": k,
           "oracle_sweep_seconds": t_or,
           "beta_active_at_k": st.active_beta is not None,
           "history_modes": sum(h is not None for h in (st.q0_history or []))}
    for name, g, row in (("continued", g_cont, g_cont.trace[-1]),
                         ("resumed", g_res, g_res.trace[0])):
        out[name] = {
            "iteration": row.iteration, "oracle_iteration": ot["iteration"],
            "fitness": row.fitness, "oracle_fitness": ot["fitness"],
            "rel_fitness_err": abs(row.fitness - ot["fitness"]) / abs(ot["fitness"]),
            "rel_factor_err": [rel(fg, fo) for fg, fo in zip(g.model.factors, o.factors)],
            "rel_lambda_err": rel(g.model.lam, o.lam),
            "flops": int(row.flops), "oracle_flops": int(ot["flops"]),
            "root_ttms": int(row.root_ttm_count), "oracle_root_ttms": int(ot["root_ttm_count"]),
            "update_order": list(row.update_order), "oracle_update_order": list(ot["update_order"]),
            "beta_used": row.beta_used, "oracle_beta_used": ot["beta_used"],
        }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("k", type=int, nargs="?", default=4)
    ap.add_argument("--dims", default=None, help="override extents, e.g. 64x64x64x64")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    kind, dims, rank, rho = CONFIGS[a.config]
    if a.dims:
        dims = tuple(int(v) for v in a.dims.split("x"))
    res = run(kind, dims, rank, rho, TRUTH_SEED[a.config], a.k,
              log=lambda *m: print(*m, file=sys.stderr, flush=True))
    res["config"] = a.config
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
