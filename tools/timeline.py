"""Per-launch device timeline of a few steady-state sweeps (diagnostic).

    python tools/timeline.py c2 [--warmup 4] [--sweeps 3] [--out gpurun_out/tl_c2.csv]

Sets CPDB_TIMELINE (an event pair around every launch site; the events cost
the PDL overlap between kernels, so sweeps run a little slower than in the
bench) and prints, for each recorded sweep, every launch's stream, start and
end relative to the sweep's first launch, in microseconds.
"""
import argparse
import os
import sys
import tempfile

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--warmup", type=int, default=4)
ap.add_argument("--sweeps", type=int, default=3)
ap.add_argument("--out", default="")
a = ap.parse_args()
path = a.out or os.path.join(tempfile.mkdtemp(), "tl.csv")
if os.path.exists(path):
    os.remove(path)

import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

c = bench.CONFIGS[a.config]
ctx = cpd.Context(0)
ctx.set_options(timing=False)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[a.config])
os.environ["CPDB_TIMELINE"] = path  # read by the session at begin()
s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=a.warmup + a.sweeps,
                                 seed=bench.INIT_SEED), extrapolate=True)
rows = s.run(a.warmup + a.sweeps)
s.close()
names = {0: "main", 1: "side", 2: "lo", 3: "mid", 4: "aux", 5: "zq", 6: "tail"}
recs = []
for line in open(path):
    lab, st, sw, mode, t0, t1 = line.strip().split(",")
    recs.append((lab, int(st), int(sw), int(mode), float(t0), float(t1)))
last = max(r[2] for r in recs)
for sw in range(last - a.sweeps + 1, last + 1):
    rs = sorted((r for r in recs if r[2] == sw), key=lambda r: r[4])
    if not rs:
        continue
    base = rs[0][4]
    end = max(r[5] for r in rs)
    print(f"sweep {sw}: {end - base:.1f} us from its first launch")
    for lab, st, _, mode, t0, t1 in rs:
        print(f"  {names[st]:4s} m{mode} {lab:14s} {t0 - base:8.1f} -> {t1 - base:8.1f}  ({t1 - t0:6.1f})")
w = [r.wall_seconds for r in rows]
print("ms/sweep (with timeline events):",
      " ".join(f"{(w[i] - w[i - 1]) * 1e3:.3f}" for i in range(len(w) - a.sweeps, len(w))))
