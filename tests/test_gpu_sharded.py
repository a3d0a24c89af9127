"""The mode-0 sharded solver on ONE GPU: `world` ranks run in
this process (one host thread each) through Context.local_group, whose
collectives (all-reduce of the partial sums of mode-0 contractions, all-gather
of V for the mode-0 update) use a shared device buffer instead of NCCL.  The
session, slab geometry, shard plan and replicated tail are the production
code; only the transport differs.  Results must match the unsharded run
(summation order of the partials differs -> 1e-10 tolerance), integer costs
exactly."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_ranks(ctxs, fn):
    out, errs = [None] * len(ctxs), []

    def body(r):
        try:
            out[r] = fn(r, ctxs[r])
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("policy", ["eager", "scatter", "lazy", "auto"])
@pytest.mark.parametrize("dims,rank,world,variant", [
    ((16, 12, 10), 3, 2, "bre"),
    ((24, 20, 16), 5, 4, "bre"),
    ((12, 10, 8, 6), 3, 2, "bre"),
    ((16, 12, 10), 3, 2, "naive"),
    ((12, 10, 8, 6), 3, 2, "dim-tree"),
    ((128, 96, 64), 16, 4, "bre"),
    ((32, 24, 24, 20), 8, 8, "bre"),
    ((16, 16, 16, 16), 64 // 4, 4, "bre"),
    ((132, 70, 68), 66, 2, "bre"),  # a rank above 64: the rank-generic tail, blocked Q packing
])
def test_sharded_matches_unsharded(ctx, port, dims, rank, world, variant, policy):
    """Every reduction strategy of the sharded session (csrc/shard.cpp: eager
    all-reduce, reduce-scatter onto a free mode, lazy reduction at V, and the
    cost model's per-step choice) gives the unsharded trajectory."""
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(0, dims, rank, 1e-2, 20250003)
    strategy = "branch-reuse" if variant == "bre" else variant
    cfg = cpd.SolverConfig(rank=rank, max_iterations=10, seed=7, strategy=strategy)
    ext = variant == "bre"
    ctx.set_tensor(x)
    ref = ctx.solve(cfg, extrapolate=ext)
    rows = dims[0] // world
    group = cpd.Context.local_group(0, world)
    # slow modelled links make "auto" mix all three strategies on these sizes
    cost = {"bus_gbs": 0.05} if policy == "auto" else None

    def rank_run(r, c):
        c.set_shard_policy(policy, cost)
        c.set_tensor(np.ascontiguousarray(x[r * rows:(r + 1) * rows]), dims)
        return c.solve(cfg, extrapolate=ext)

    res = run_ranks(group, rank_run)
    for g in res:
        assert len(g.trace) == len(ref.trace)
        for a, b in zip(g.trace, ref.trace):
            assert a.update_order == b.update_order and a.flops == b.flops
            assert a.root_ttm_count == b.root_ttm_count and a.beta_used == b.beta_used
            assert abs(a.fitness - b.fitness) <= 1e-10 * b.fitness
        for fa, fb in zip(g.model.factors, ref.model.factors):
            assert np.linalg.norm(fa - fb) <= 1e-10 * np.linalg.norm(fb)
    # the replicated tail: every rank holds the same model
    for g in res[1:]:
        for fa, fb in zip(g.model.factors, res[0].model.factors):
            assert np.array_equal(fa, fb)
    for c in group:
        c.close()


def test_sharded_synth_matches_unsharded(ctx):
    """Device generator on slabs: the counter-based values do not depend on
    the shard layout; the noise scale is all-reduced."""
    import paper_2503_18759_b200 as cpd
    dims, world = [32, 24, 20], 4
    ctx.synth_tensor(0, dims, 6, 1e-2, 99)
    full = ctx.get_tensor(dims)
    group = cpd.Context.local_group(0, world)

    def rank_run(r, c):
        c.synth_tensor(0, dims, 6, 1e-2, 99)
        return c.get_tensor([dims[0] // world] + dims[1:])

    slabs = run_ranks(group, rank_run)
    got = np.concatenate(slabs, axis=0)
    assert np.allclose(got, full, rtol=1e-13, atol=1e-13 * np.abs(full).max())
    for c in group:
        c.close()


def test_nccl_calls_execute_on_one_rank():
    """The NCCL operations the sharded session issues -- in-place all-reduce,
    all-gather, and the grouped per-slice reduce-scatter -- run on a one-rank
    communicator of this B200 and return their input (a multi-rank NCCL run
    needs more than the one GPU this environment has)."""
    import paper_2503_18759_b200 as cpd
    assert cpd.Context.nccl_selftest(0) == 0.0


def test_nccl_library_available():
    """The multi-GPU transport: libnccl.so.2 resolves (dlopen, comm.cpp) and
    hands out a unique id; one rank per GPU then calls cpdb_create_sharded."""
    import paper_2503_18759_b200 as cpd
    uid = cpd.Context.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)


@pytest.mark.parametrize("dims,world", [((24, 20, 16), 2), ((12, 10, 8, 6), 2)])
def test_sharded_stop_test_undoes_speculative_update(ctx, port, dims, world):
    """Sharded runs also issue the next sweep's first update (its collectives
    included) before reading the fitness; when the stop test fires every rank
    undoes it and returns the unsharded run's model."""
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(0, dims, 3, 1e-2, 20250013)
    ctx.set_tensor(x)
    tr = ctx.solve(cpd.SolverConfig(rank=3, max_iterations=6, seed=7), extrapolate=True).trace
    # midway between sweeps 5 and 6: the stop sweep does not hinge on last bits
    assert tr[-1].fitness - tr[-2].fitness > 1e-8
    thr = 0.5 * (tr[-2].fitness + tr[-1].fitness)
    cfg = cpd.SolverConfig(rank=3, max_iterations=30, seed=7, fitness_threshold=thr)
    ref = ctx.solve(cfg, extrapolate=True)
    assert len(ref.trace) == 6
    rows = dims[0] // world
    group = cpd.Context.local_group(0, world)

    def rank_run(r, c):
        c.set_tensor(np.ascontiguousarray(x[r * rows:(r + 1) * rows]), dims)
        return c.solve(cfg, extrapolate=True)

    res = run_ranks(group, rank_run)
    for g in res:
        assert len(g.trace) == len(ref.trace)
        for a, b in zip(g.trace, ref.trace):
            assert abs(a.fitness - b.fitness) <= 1e-10 * b.fitness
        for fa, fb in zip(g.model.factors, ref.model.factors):
            assert np.linalg.norm(fa - fb) <= 1e-10 * np.linalg.norm(fb)
        assert np.linalg.norm(g.model.lam - ref.model.lam) <= 1e-10 * np.linalg.norm(ref.model.lam)
    for c in group:
        c.close()


@pytest.mark.parametrize("policy", ["eager", "scatter", "lazy", "auto"])
@pytest.mark.parametrize("k", [3, 4, 5])
def test_sharded_resume_rebuilds_planned_layouts(ctx, port, policy, k):
    """A sharded session resumed from a sweep-boundary state rebuilds every
    retained intermediate in the layout the plan gave it (split, replicated
    or partial sums) and continues the unsharded trajectory."""
    import paper_2503_18759_b200 as cpd
    from test_gpu_solver import port_init
    dims, rank, world = (16, 12, 8, 8), 4, 4
    x = port.synth_baseline(0, dims, rank, 1e-2, 20250021)
    init = cpd.SweepState(0, np.ones(rank), port_init(port, dims, rank, 7))
    cfg = cpd.SolverConfig(rank=rank, max_iterations=k + 3, seed=7)
    ctx.set_tensor(x)
    ref = ctx.solve(cfg, extrapolate=True, state=init)
    first = ctx.solve(cpd.SolverConfig(rank=rank, max_iterations=k, seed=7), extrapolate=True,
                      state=init)
    assert first.state.sweeps_done == k
    rows = dims[0] // world
    group = cpd.Context.local_group(0, world)
    cost = {"bus_gbs": 0.05} if policy == "auto" else None

    def rank_run(r, c):
        c.set_shard_policy(policy, cost)
        c.set_tensor(np.ascontiguousarray(x[r * rows:(r + 1) * rows]), dims)
        return c.solve(cpd.SolverConfig(rank=rank, max_iterations=3, seed=7), extrapolate=True,
                       state=first.state)

    res = run_ranks(group, rank_run)
    for g in res:
        assert len(g.trace) == 3
        for a, b in zip(g.trace, ref.trace[k:]):
            assert a.iteration == b.iteration and a.flops == b.flops
            assert abs(a.fitness - b.fitness) <= 1e-10 * b.fitness
        for fa, fb in zip(g.model.factors, ref.model.factors):
            assert np.linalg.norm(fa - fb) <= 1e-10 * np.linalg.norm(fb)
    for c in group:
        c.close()


@pytest.mark.parametrize("policy", ["eager", "scatter", "lazy", "auto"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_c5_proxy_matches_unsharded(ctx, port, policy, world):
    """Config 5's path sharded: fourth order, R = 64 (tall multi-kernel Z-QR
    of Z = 262144 x 64, the wide V-GEMM, the 3-cycle branch reuse) at the
    64^4 proxy, every reduction strategy, against the unsharded run."""
    import paper_2503_18759_b200 as cpd
    dims, rank = (64, 64, 64, 64), 64
    x = port.synth_baseline(0, dims, rank, 1e-3, 20250005)
    cfg = cpd.SolverConfig(rank=rank, max_iterations=5, seed=7)
    ctx.set_tensor(x)
    ref = ctx.solve(cfg, extrapolate=True)
    rows = dims[0] // world
    group = cpd.Context.local_group(0, world)
    cost = {"bus_gbs": 0.05} if policy == "auto" else None

    def rank_run(r, c):
        c.set_shard_policy(policy, cost)
        c.set_tensor(np.ascontiguousarray(x[r * rows:(r + 1) * rows]), dims)
        return c.solve(cfg, extrapolate=True)

    res = run_ranks(group, rank_run)
    for g in res:
        assert len(g.trace) == len(ref.trace)
        for a, b in zip(g.trace, ref.trace):
            assert a.update_order == b.update_order and a.flops == b.flops
            assert abs(a.fitness - b.fitness) <= 1e-10 * b.fitness
        for fa, fb in zip(g.model.factors, ref.model.factors):
            assert np.linalg.norm(fa - fb) <= 1e-10 * np.linalg.norm(fb)
    for c in group:
        c.close()


@pytest.mark.parametrize("policy", ["eager", "scatter", "auto"])
@pytest.mark.parametrize("dims,rank,world", [((64, 64, 64, 64), 64, 2), ((128, 72, 64), 64, 4),
                                             ((32, 24, 24, 20), 8, 2)])
def test_reduced_steps_in_slabs_bit_identical(monkeypatch, policy, dims, rank, world):
    """A reduced TTM step runs in slabs whose collectives overlap the next
    slab's kernel (Session::ttm_step): column halves of Q when it contracts
    the leading (split) mode at R = 64, outer slices otherwise.  Every output
    element is accumulated and reduced in the same order as in one launch and
    one collective: bit-identical runs."""
    import paper_2503_18759_b200 as cpd
    rows = dims[0] // world
    cfg = cpd.SolverConfig(rank=rank, max_iterations=5, seed=7)
    monkeypatch.setenv("CPDB_RS_MIN_FLOPS", "0")
    outs = []
    for chunks in ("1", "4"):
        monkeypatch.setenv("CPDB_RS_CHUNKS", chunks)
        group = cpd.Context.local_group(0, world)
        cost = {"bus_gbs": 0.05} if policy == "auto" else None

        def rank_run(r, c):
            c.set_shard_policy(policy, cost)
            c.synth_tensor(0, list(dims), rank, 1e-3, 31337)
            res = c.solve(cfg, extrapolate=True)
            return res, c.profile()["kernel_launches"]

        outs.append(run_ranks(group, rank_run))
        for c in group:
            c.close()
    one, four = outs
    # (auto may pick lazy everywhere, and eager at R < 64 only reduces
    # leading-mode contractions, which stay whole: no slabs there)
    if policy == "scatter" or (policy == "eager" and rank == 64):
        assert four[0][1] > one[0][1]  # the slabs did launch
    for (a, _), (b, _) in zip(one, four):
        assert [(t.fitness, t.raw_radicand) for t in a.trace] == \
               [(t.fitness, t.raw_radicand) for t in b.trace]
        for fa, fb in zip(a.model.factors, b.model.factors):
            assert np.array_equal(fa, fb)
