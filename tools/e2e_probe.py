"""Where does the e2e (host-buffer) time of a bench job go?  Times each phase
of the public-API job with wall clocks (diagnostic only)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
c = bench.CONFIGS[name]
dims = list(c["dims"])
ctx = cpd.Context(0)
ctx.synth_tensor(c["kind"], dims, c["rank"], c["rho"], bench.TRUTH_SEED[name])
x = ctx.get_tensor(dims)
pinned = torch.empty(x.size, dtype=torch.float64, pin_memory=True).numpy()
pinned[:] = x.ravel()
xh = pinned.reshape(dims)
for rep in range(3):
    t = [time.perf_counter()]
    ctx.set_tensor(xh, dims)
    t.append(time.perf_counter())
    s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=K, seed=7), extrapolate=True)
    t.append(time.perf_counter())
    r1 = s.run(1)
    t.append(time.perf_counter())
    r = s.run(K - 1)
    t.append(time.perf_counter())
    m = s.end()
    t.append(time.perf_counter())
    s.close()
    d = np.diff(t) * 1e3
    print(f"rep {rep}: set_tensor {d[0]:.1f} ms  begin {d[1]:.1f}  sweep1 {d[2]:.1f}  "
          f"sweeps2..K {d[3]:.1f} ({d[3]/(K-1):.3f}/sweep)  end {d[4]:.1f}  total {t[-1]-t[0]:.3f}s")
