"""Full-length parity at a BASELINE size: the device solver vs the reference
compiled here (oracle/_ref, single host core) on the same device-generated
tensor, every sweep of the BASELINE sweep count.  Writes a JSON summary.

    python tools/full_parity.py c4 [--sweeps N] [--floor] [--out profiles/...json]

--floor also runs the reference on X perturbed by 1e-15 (relative, one draw
per element) to show the oracle's own sensitivity next to the GPU-vs-oracle
difference.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402
from oracle.pyoracle import Oracle, available  # noqa: E402


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--sweeps", type=int, default=0)
    ap.add_argument("--floor", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = bench.CONFIGS[a.config]
    sweeps = a.sweeps or c["sweeps"]
    dims = list(c["dims"])
    ctx = cpd.Context(0)
    ctx.synth_tensor(c["kind"], dims, c["rank"], c["rho"], bench.TRUTH_SEED[a.config])
    x = ctx.get_tensor(dims)
    cfg = cpd.SolverConfig(rank=c["rank"], max_iterations=sweeps, seed=bench.INIT_SEED)
    t0 = time.perf_counter()
    g = ctx.solve(cfg, extrapolate=True)
    t_gpu = time.perf_counter() - t0
    kind = "reference" if available("reference") else "port"
    ora = Oracle(kind)
    t0 = time.perf_counter()
    o = ora.solve(x, c["rank"], sweeps, extrapolate=True, seed=bench.INIT_SEED)
    t_cpu = time.perf_counter() - t0
    assert len(g.trace) == len(o.trace)
    fit_rel = [rel(gr.fitness, orow["fitness"]) for gr, orow in zip(g.trace, o.trace)]
    exact = all(gr.flops == orow["flops"] and gr.root_ttm_count == orow["root_ttm_count"]
                and gr.update_order == orow["update_order"] and gr.beta_used == orow["beta_used"]
                for gr, orow in zip(g.trace, o.trace))
    first_beta_g = next((r.iteration for r in g.trace if r.beta_used != 0.0), None)
    first_beta_o = next((r["iteration"] for r in o.trace if r["beta_used"] != 0.0), None)
    fac = [float(np.linalg.norm(fg - fo) / np.linalg.norm(fo))
           for fg, fo in zip(g.model.factors, o.factors)]
    out = {
        "config": a.config, "dims": dims, "rank": c["rank"], "sweeps": sweeps,
        "oracle": kind, "data": "device generator (BASELINE construction), downloaded to host",
        "gpu_vs_oracle": {
            "max_rel_fitness": max(fit_rel), "median_rel_fitness": float(np.median(fit_rel)),
            "worst_sweep": int(np.argmax(fit_rel)) + 1,
            "final_factor_rel": fac, "final_lambda_rel":
                float(np.linalg.norm(g.model.lam - o.lam) / np.linalg.norm(o.lam)),
            "integer_trace_identical": bool(exact),
            "beta_activation_sweep": [first_beta_g, first_beta_o],
            "final_fitness": [g.trace[-1].fitness, o.trace[-1]["fitness"]],
        },
        "wall_seconds": {"gpu_solve": t_gpu, "oracle_solve": t_cpu},
        "tolerance": "north star: relative fitness and factor error <= 1e-10 per sweep",
    }
    if a.floor:
        rng = np.random.default_rng(2025)
        xp = x * (1.0 + 1e-15 * rng.standard_normal(x.shape))
        op = ora.solve(xp, c["rank"], sweeps, extrapolate=True, seed=bench.INIT_SEED)
        fr = [rel(p["fitness"], q["fitness"]) for p, q in zip(op.trace, o.trace)]
        out["oracle_vs_perturbed_oracle"] = {
            "perturbation": "x * (1 + 1e-15 N(0,1))", "max_rel_fitness": max(fr),
            "median_rel_fitness": float(np.median(fr)), "worst_sweep": int(np.argmax(fr)) + 1}
    print(json.dumps(out, indent=1))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
