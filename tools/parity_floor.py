"""Measure, per GPU parity case of tests/test_gpu_solver.py, the device-vs-
oracle error next to the oracle's own perturbation floor (the oracle run on
X * (1 + 1e-15 N(0,1)) vs the oracle on X).  Prints JSON lines.

    python tools/parity_floor.py [--out gpurun_out/parity_floor.jsonl]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2503_18759_b200 as cpd  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

META = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")))


def errs(tr_a, fa, lam_a, tr_b, fb, lam_b):
    fit = max(abs(a - b) / abs(b) for a, b in zip(tr_a, tr_b))
    fac = max(float(np.linalg.norm(x - y) / np.linalg.norm(y)) for x, y in zip(fa, fb))
    lam = float(np.linalg.norm(lam_a - lam_b) / np.linalg.norm(lam_b))
    return fit, fac, lam


def case(ctx, port, name, x, rank, iters, seed, strategy="branch-reuse", extrap=True):
    cfg = cpd.SolverConfig(rank=rank, max_iterations=iters, seed=seed, strategy=strategy)
    g = cpd.als_qr_bre(x, cfg, ctx=ctx) if extrap else cpd.cp_als_qr(x, cfg, ctx=ctx)
    o = port.solve(x, rank, iters, extrapolate=extrap, strategy=strategy, seed=seed)
    rng = np.random.default_rng(12345)
    xp = x * (1.0 + 1e-15 * rng.standard_normal(x.shape))
    p = port.solve(xp, rank, iters, extrapolate=extrap, strategy=strategy, seed=seed)
    fo = [t["fitness"] for t in o.trace]
    gf = [t.fitness for t in g.trace]
    pf = [t["fitness"] for t in p.trace]
    ge = errs(gf, g.model.factors, g.model.lam, fo, o.factors, o.lam)
    pe = errs(pf, p.factors, p.lam, fo, o.factors, o.lam) if len(pf) == len(fo) else (None,) * 3
    return {"case": name, "gpu_fit": ge[0], "gpu_factor": ge[1], "gpu_lambda": ge[2],
            "floor_fit": pe[0], "floor_factor": pe[1], "floor_lambda": pe[2],
            "final_fitness": fo[-1]}


def als_case(ctx, ora, name, x, rank, iters, seed):
    cfg = cpd.SolverConfig(rank=rank, max_iterations=iters, seed=seed, algorithm="als")
    g = cpd.cp_als(x, cfg, ctx=ctx)
    o = ora.cp_als(x, rank, iters, seed=seed)
    rng = np.random.default_rng(12345)
    p = ora.cp_als(x * (1.0 + 1e-15 * rng.standard_normal(x.shape)), rank, iters, seed=seed)
    fo = [t["fitness"] for t in o.trace]
    ge = errs([t.fitness for t in g.trace], g.model.factors, g.model.lam, fo, o.factors, o.lam)
    pe = errs([t["fitness"] for t in p.trace], p.factors, p.lam, fo, o.factors, o.lam)
    return {"case": name, "gpu_fit": ge[0], "gpu_factor": ge[1], "gpu_lambda": ge[2],
            "floor_fit": pe[0], "floor_factor": pe[1], "floor_lambda": pe[2],
            "final_fitness": fo[-1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--als-only", action="store_true")
    a = ap.parse_args()
    ctx = cpd.default_context()
    port = Oracle("port")
    rows = []
    for dims, rank in [] if a.als_only else [((9, 8, 7), 3), ((7, 6, 5, 4), 3), ((10, 10, 10), 4), ((16, 24, 20), 5),
                       ((12, 10, 8, 16), 4)]:
        x = port.rng_normals(31, int(np.prod(dims))).reshape(dims)
        for variant in ("naive", "dim-tree", "branch-reuse", "bre"):
            strat = "branch-reuse" if variant == "bre" else variant
            rows.append(case(ctx, port, f"small{dims}R{rank}-{variant}", x, rank, 12, 3, strat,
                             variant == "bre"))
    for dims, rank in [] if a.als_only else [((9, 8, 7), 1), ((20, 18, 16), 7), ((30, 28, 26), 13), ((40, 38, 36), 33),
                       ((70, 66, 65), 64), ((12, 11, 10, 9), 9), ((10, 9, 8, 8, 7), 5)]:
        x = port.rng_normals(4242 + rank, int(np.prod(dims))).reshape(dims)
        if len(dims) == 5:
            rows.append(case(ctx, port, f"rank{dims}R{rank}", x, rank, 4, 5, "naive", False))
        else:
            rows.append(case(ctx, port, f"rank{dims}R{rank}", x, rank, 6, 5))
    if not a.als_only:
        x = port.synth_baseline(1, (48, 48, 48), 20, 1e-4, META["truth_seeds"]["c4"])
        rows.append(case(ctx, port, "c4_48^3", x, 20, 60, META["init_seed"]))
        x = port.synth_baseline(0, (40, 36, 34, 33), 32, 1e-3, META["truth_seeds"]["c5"])
        rows.append(case(ctx, port, "tallz", x, 32, 8, META["init_seed"]))
        x = port.synth_baseline(0, (64, 64, 64), 16, 1e-3, META["truth_seeds"]["c2"])
        rows.append(case(ctx, port, "variants64", x, 16, 24, META["init_seed"]))
    ora = Oracle("reference")
    for dims, rank, kind in [((12, 11, 10), 4, 0), ((9, 8, 7), 3, 0), ((8, 7, 6, 5), 3, 0),
                             ((40, 30, 20), 8, 0), ((16, 12, 10, 8), 5, 0), ((30, 2, 20), 2, 0),
                             ((50, 60), 7, 0), ((64, 64, 64), 20, 1)]:
        x = ora.synth_baseline(kind, dims, rank, 1e-2, 777 + rank)
        rows.append(als_case(ctx, ora, f"als{dims}R{rank}k{kind}", x, rank, 25, 9))
    for dims, rank in [((12, 11, 10), 4), ((7, 6, 5, 4), 3)]:
        x = np.random.default_rng(sum(dims)).standard_normal(dims)
        rows.append(als_case(ctx, ora, f"als_random{dims}R{rank}", x, rank, 15, 31))
    out = open(a.out, "w") if a.out else None
    for r in rows:
        line = json.dumps(r)
        print(line)
        if out:
            out.write(line + "\n")


if __name__ == "__main__":
    main()
