"""SURVEY.md 8f row 3 on the B200: naive vs dim-tree vs branch-reuse CP-ALS-QR
sweeps (no extrapolation) on the same device kernels, against the
reference's C12 acceptance ordering (acceptance_test.cpp:390-406: mean sweep
time qr-br < qr-dt < qr-naive, br <= 0.8 naive; 200^3 random tensor, R 20,
10 sweeps -- make_config(alg, strategy, rank, iters, seed), :44-54) and the paper's leading-flop ratio 8 : 12 : 18
(dim_tree.hpp:623-634).  Writes one JSON document.

    python tools/strategy_bench.py [--out profiles/r02_strategies.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import paper_2503_18759_b200 as cpd  # noqa: E402

STRATS = ("naive", "dim-tree", "branch-reuse")


def run(ctx, dims, rank, sweeps, strategy):
    cfg = cpd.SolverConfig(rank=rank, max_iterations=sweeps, seed=1212, strategy=strategy)
    s = ctx.session(cfg, extrapolate=False)
    rows = s.run(sweeps)
    s.close()
    w = [r.wall_seconds for r in rows]
    flops = [rows[0].flops] + [rows[i].flops - rows[i - 1].flops for i in range(1, len(rows))]
    return {"mean_sweep_s": w[-1] / len(w),  # the reference's C12 measure
            "steady_sweeps_per_s": (len(w) - 2) / (w[-1] - w[1]),
            "steady_flops_per_sweep": float(np.mean(flops[2:])),
            "flops_first_three": int(rows[2].flops)}


def case(name, dims, rank, sweeps, tensor=None, synth=None):
    ctx = cpd.Context(0)
    if tensor is not None:
        ctx.set_tensor(tensor)
    else:
        ctx.synth_tensor(*synth)
    for st in STRATS:  # warm the kernels
        run(ctx, dims, rank, 3, st)
    res = {st: run(ctx, dims, rank, sweeps, st) for st in STRATS}
    ctx.close()
    t = {st: res[st]["mean_sweep_s"] for st in STRATS}
    lead = {st: cpd.leading_flop_coefficient(len(dims), st) for st in STRATS}
    return {
        "case": name, "dims": list(dims), "rank": rank, "sweeps": sweeps, "results": res,
        "c12_order_holds": t["branch-reuse"] < t["dim-tree"] < t["naive"],
        "br_over_naive": t["branch-reuse"] / t["naive"],
        "c12_br_le_0.8_naive": t["branch-reuse"] <= 0.8 * t["naive"],
        "leading_flop_coefficients": lead,
        "time_ratio_vs_naive": {st: t[st] / t["naive"] for st in STRATS},
        "leading_ratio_vs_naive": {st: lead[st] / lead["naive"] for st in STRATS},
        "first3_flop_ratio_vs_naive": {st: res[st]["flops_first_three"] /
                                       res["naive"]["flops_first_three"] for st in STRATS},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    x = np.random.default_rng(1212).standard_normal((200, 200, 200))
    out = [case("c12_200^3_R20_random", (200, 200, 200), 20, 10, tensor=x),
           case("c2_512^3_R32", (512, 512, 512), 32, 20,
                synth=(0, [512, 512, 512], 32, 1e-3, 20250002)),
           case("c3_128^4_R16", (128, 128, 128, 128), 16, 20,
                synth=(0, [128] * 4, 16, 1e-2, 20250003))]
    doc = json.dumps(out, indent=1)
    print(doc)
    if a.out:
        open(a.out, "w").write(doc)


if __name__ == "__main__":
    main()
