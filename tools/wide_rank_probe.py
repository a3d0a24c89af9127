"""Ranks above 64 (widerank.cu): device sweeps/s of ALS-QR-BRE against the CPU
oracle port on the same tensor, with the per-sweep parity of the two (diagnostic).

    python tools/wide_rank_probe.py [dims=192x192x192] [rank=128] [sweeps=6] [cpu_sweeps=2]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2503_18759_b200 as cpd  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402  (checker / CPU baseline only)

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "192x192x192").split("x"))
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 128
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
cpu_sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
port = Oracle("port")
x = port.synth_baseline(0, dims, rank, 1e-3, 4242)
ctx = cpd.Context(0)
cfg = cpd.SolverConfig(rank=rank, max_iterations=sweeps, seed=7)
cpd.als_qr_bre(x, cfg, ctx=ctx)  # warm-up (allocations, module load)
g = cpd.als_qr_bre(x, cfg, ctx=ctx)
w = [t.wall_seconds for t in g.trace]
dev = (sweeps - 2) / (w[-1] - w[1])
out = {"dims": dims, "rank": rank, "device_sweeps_per_s": dev,
       "kernel_launches": ctx.profile()["kernel_launches"]}
if cpu_sweeps > 0:
    t0 = time.perf_counter()
    o = port.solve(x, rank, cpu_sweeps, extrapolate=True, seed=7)
    cpu = cpu_sweeps / (time.perf_counter() - t0)
    out["cpu_port_sweeps_per_s"] = cpu
    out["speedup"] = dev / cpu
    out["max_rel_fitness_gap_first_sweeps"] = max(
        abs(a.fitness - b["fitness"]) / abs(b["fitness"]) for a, b in zip(g.trace, o.trace))
print(json.dumps(out))
