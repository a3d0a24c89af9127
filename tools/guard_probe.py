"""Small runs of the round-2 additions for the allocator guard zones (CPDB_GUARD=1):
a wide-rank ALS-QR-BRE solve, a wide-rank CP-ALS
solve, a branch-reuse solve whose sweep boundary reuses the previous update,
a split-run session and a sharded run in slabs (diagnostic).

    CPDB_GUARD=1 python tools/sanitize_probe.py [wide|als|reuse|shard]
"""
import sys
import threading

import numpy as np

sys.path.insert(0, ".")
import paper_2503_18759_b200 as cpd  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "wide"
rng = np.random.default_rng(3)
if what == "wide":
    x = rng.standard_normal((70, 68, 66))
    r = cpd.als_qr_bre(x, cpd.SolverConfig(rank=65, max_iterations=3, seed=5))
    print("wide", r.trace[-1].fitness)
elif what == "als":
    x = rng.standard_normal((40, 30, 20))
    r = cpd.cp_als(x, cpd.SolverConfig(rank=80, max_iterations=3, seed=5, algorithm="als"))
    print("als", r.trace[-1].fitness)
elif what == "reuse":
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, [48, 40, 32], 8, 1e-2, 99)
    s = ctx.session(cpd.SolverConfig(rank=8, max_iterations=8, seed=3), extrapolate=True)
    rows = s.run(3) + s.run(3)
    s.end()
    s.close()
    print("reuse", rows[-1].fitness)
else:
    import os
    os.environ["CPDB_RS_MIN_FLOPS"] = "0"
    group = cpd.Context.local_group(0, 2)
    out = [None, None]

    def body(rk):
        c = group[rk]
        c.set_shard_policy("scatter", None)
        c.synth_tensor(0, [64, 64, 64], 64, 1e-3, 7)
        out[rk] = c.solve(cpd.SolverConfig(rank=64, max_iterations=3, seed=7), extrapolate=True)

    ts = [threading.Thread(target=body, args=(k,)) for k in range(2)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    print("shard", out[0].trace[-1].fitness)
