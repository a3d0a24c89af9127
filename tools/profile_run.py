"""Minimal driver for ncu captures: synthesise a BASELINE config on the device
and run W warm-up + K sweeps of ALS-QR-BRE (no CPU baseline, no e2e)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--no-timing", action="store_true")
a = ap.parse_args()
c = bench.CONFIGS[a.config]
ctx = cpd.Context(0)
if a.no_timing:
    ctx.set_options(timing=False)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[a.config])
s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=a.warmup + a.sweeps,
                                 seed=bench.INIT_SEED), extrapolate=True)
w = s.run(a.warmup)
r = s.run(a.sweeps)
p = ctx.profile()
print("sweep ms", (r[-1].wall_seconds - w[-1].wall_seconds) / a.sweeps * 1e3, "fit", r[-1].fitness,
      "launches", p["kernel_launches"])
