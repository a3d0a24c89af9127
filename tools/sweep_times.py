"""Per-sweep device times of one run (diagnostic for run-to-run variance)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
c = bench.CONFIGS[name]
ctx = cpd.Context(0)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[name])
s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=n, seed=7), extrapolate=True)
rows = s.run(n)
s.close()
w = [r.wall_seconds for r in rows]
d = [(w[i] - w[i - 1]) * 1e3 for i in range(1, len(w))]
print(name, "ms/sweep:", " ".join(f"{v:.3f}" for v in d[2:]))
