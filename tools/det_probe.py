"""Determinism check: the same BASELINE config solved repeatedly in one
context must give bit-identical traces (diagnostic)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_18759_b200 as cpd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
c = dict(bench.CONFIGS[name]) if name in bench.CONFIGS else None
if c is None:  # "d1xd2x...:R"
    ds, r = name.split(":")
    c = dict(kind=0, dims=tuple(int(v) for v in ds.split("x")), rank=int(r), rho=1e-2)
    bench.TRUTH_SEED[name] = 12345
ctx = cpd.Context(0)
ctx.synth_tensor(c["kind"], list(c["dims"]), c["rank"], c["rho"], bench.TRUTH_SEED[name])
ref = None
bad = 0
for rep in range(reps):
    s = ctx.session(cpd.SolverConfig(rank=c["rank"], max_iterations=sweeps, seed=7),
                    extrapolate=True)
    rows = s.run(sweeps)
    s.end()
    s.close()
    tr = [(r.fitness, r.raw_radicand) for r in rows]
    if ref is None:
        ref = tr
    elif tr != ref:
        bad += 1
        first = next(i for i in range(len(tr)) if tr[i] != ref[i])
        print("rep", rep, "differs from sweep", first + 1, tr[first], ref[first])
print(name, "reps", reps, "mismatching", bad)
