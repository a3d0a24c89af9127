"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers (compiled in place into
oracle/_ref/libcpdref.so by oracle/Makefile) -- not the restatement -- so the
fixtures pin both the C restatement (tests/test_golden.py) and the GPU path.
The reference has no golden files of its own (every vector is
seed-regenerated), so these are produced here, once, and committed.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Oracle  # noqa: E402

# BASELINE.json configs: kind, dims, rank, rho, sweeps.
CONFIGS = {
    "c1": (0, (100, 100, 100), 10, 1e-2, 50),
    "c2": (0, (512, 512, 512), 32, 1e-3, 100),
    "c3": (0, (128, 128, 128, 128), 16, 1e-2, 100),
    "c4": (1, (256, 256, 256), 20, 1e-4, 500),
    "c5": (0, (256, 256, 256, 256), 64, 1e-3, 50),
}
TRUTH_SEED = {k: 20250000 + i + 1 for i, k in enumerate(CONFIGS)}
INIT_SEED = 7


def trace_arrays(trace):
    return dict(
        fitness=np.array([r["fitness"] for r in trace]),
        raw=np.array([r["raw_radicand"] for r in trace]),
        flops=np.array([r["flops"] for r in trace], dtype=np.uint64),
        roots=np.array([r["root_ttm_count"] for r in trace], dtype=np.uint64),
        beta=np.array([r["beta_used"] for r in trace]),
        order=np.array([r["update_order"] for r in trace], dtype=np.int64),
    )


def main():
    ref = Oracle("reference")
    out = {}
    meta = {"source": "oracle/_ref/libcpdref.so (reference headers, -O3 -DNDEBUG "
                      "-ffp-contract=off)", "truth_seeds": TRUTH_SEED, "init_seed": INIT_SEED}

    # rng.hpp draw order
    for seed in (0, 7, 20250001):
        out[f"rng_normals_{seed}"] = ref.rng_normals(seed, 64)

    # ttm / unfold / khatri-rao / qr primitives on a 9x8x7 tensor
    x = ref.rng_normals(101, 9 * 8 * 7).reshape(9, 8, 7)
    out["prim_x"] = x
    for m, n in enumerate(x.shape):
        b = ref.rng_normals(200 + m, 3 * n).reshape(3, n)
        out[f"prim_b{m}"] = b
        out[f"prim_ttm{m}"] = ref.ttm(x, b, m)
        out[f"prim_unfold{m}"] = ref.unfold(x, m)
    a = ref.rng_normals(301, 50 * 6).reshape(50, 6)
    out["prim_qr_a"] = a
    out["prim_qr_q"], out["prim_qr_r"] = ref.thin_qr(a)
    t1 = np.triu(ref.rng_normals(302, 16).reshape(4, 4))
    t2 = np.triu(ref.rng_normals(303, 16).reshape(4, 4))
    t1[0, 0], t2[0, 0] = abs(t1[0, 0]) + 0.5, abs(t2[0, 0]) + 0.5
    out["prim_kr_a"], out["prim_kr_b"] = t1, t2
    out["prim_kr"] = ref.khatri_rao([t1, t2])
    out["prim_kr_q"], out["prim_kr_r"] = ref.thin_qr(out["prim_kr"])

    # schedules and cost anchors
    for order in (3, 4):
        for s in ("naive", "dim-tree", "branch-reuse"):
            steps, cyc = ref.schedule(order, s, 7)
            out[f"sched_{order}_{s}"] = steps
            out[f"sched_{order}_{s}_cycle"] = np.array(cyc, dtype=np.int64)
    anchors = {}
    for k, (_, dims, rank, _, sweeps) in CONFIGS.items():
        fl, ro = ref.measured_cost(len(dims), "branch-reuse", dims, rank, sweeps)
        f1, _ = ref.measured_cost(len(dims), "branch-reuse", dims, rank, 1)
        anchors[k] = {"flops": fl, "roots": ro, "sweep1_flops": f1}
    meta["cost_anchors"] = anchors

    # solver trajectories
    small = {
        "s3": ((9, 8, 7), 3, 12),
        "s4": ((7, 6, 5, 4), 3, 12),
        "s10": ((10, 10, 10), 4, 12),
    }
    for name, (dims, rank, iters) in small.items():
        x = ref.rng_normals(400 + len(name), int(np.prod(dims))).reshape(dims)
        out[f"{name}_x"] = x
        for strat in ("naive", "dim-tree", "branch-reuse"):
            r = ref.solve(x, rank, iters, extrapolate=False, strategy=strat, seed=3)
            for key, val in trace_arrays(r.trace).items():
                out[f"{name}_{strat}_{key}"] = val
        r = ref.solve(x, rank, iters, extrapolate=True, seed=3)
        for key, val in trace_arrays(r.trace).items():
            out[f"{name}_bre_{key}"] = val
        for k, f in enumerate(r.factors):
            out[f"{name}_bre_factor{k}"] = f
        out[f"{name}_bre_lambda"] = r.lam

    # C1 (full BASELINE config 1) and a reduced C4-style ill-conditioned run
    kind, dims, rank, rho, sweeps = CONFIGS["c1"]
    x = ref.synth_baseline(kind, dims, rank, rho, TRUTH_SEED["c1"])
    out["c1_x_checksum"] = np.array([x.sum(), (x * x).sum(), x.ravel()[0], x.ravel()[-1]])
    r = ref.solve(x, rank, sweeps, extrapolate=True, seed=INIT_SEED)
    for key, val in trace_arrays(r.trace).items():
        out[f"c1_{key}"] = val
    for k, f in enumerate(r.factors):
        out[f"c1_factor{k}"] = f
    out["c1_lambda"] = r.lam

    x4 = ref.synth_baseline(1, (32, 32, 32), 5, 1e-4, TRUTH_SEED["c4"])
    out["c4s_x_checksum"] = np.array([x4.sum(), (x4 * x4).sum(), x4.ravel()[0], x4.ravel()[-1]])
    r = ref.solve(x4, 5, 100, extrapolate=True, seed=INIT_SEED)
    for key, val in trace_arrays(r.trace).items():
        out[f"c4s_{key}"] = val

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
