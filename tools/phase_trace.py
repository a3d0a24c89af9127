import os, sys
sys.path.insert(0, ".")
import bench
import paper_2503_18759_b200 as cpd
name = sys.argv[1]
c = bench.CONFIGS[name]
ctx = cpd.Context(0)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[name])
s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=12, seed=7), extrapolate=True)
s.run(12)
s.close()
