"""Per-sweep device times across a run(W) / run(K) boundary (diagnostic)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 5
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
c = bench.CONFIGS[name]
ctx = cpd.Context(0)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[name])
for split in (True, False):
    s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=W + K, seed=bench.INIT_SEED),
                    extrapolate=True)
    rows = (s.run(W) + s.run(K)) if split else s.run(W + K)
    s.close()
    w = [r.wall_seconds for r in rows]
    d = [(w[i] - w[i - 1]) * 1e3 for i in range(1, len(w))]
    print(name, "split" if split else "whole", "K/s=%.1f" % (K / (w[-1] - w[W - 1])),
          "ms/sweep:", " ".join(f"{v:.3f}" for v in d))
