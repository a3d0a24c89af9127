"""Multi-GPU path on CPU: the mode-0 sharding plan that the
device session follows (csrc/schedule.hpp shard_flags, ABI cpdb_shard_plan),
executed by two gloo ranks with numpy TTMs standing in for the device kernels.

Each rank holds a contiguous slab of mode-0 rows of X.  Following the
reference schedules (dim_tree.hpp:386-426) and the plan's flags, it keeps its
own intermediate cache, all-reduces the partial sums of mode-0 contractions
and all-gathers V's rows for the mode-0 update; every final Y(n) must equal
the unsharded X x_{k != n} Q_k^T.
"""
import os
import socket

import numpy as np
import pytest

import paper_2503_18759_b200 as cpd

STRATS = ["naive", "dim-tree", "branch-reuse"]


def ttm(t, q, mode):
    """Y = T x_mode Q^T (tensor.hpp:288-315 semantics), numpy."""
    y = np.tensordot(q.T, t, axes=([1], [mode]))
    return np.moveaxis(y, 0, mode)


@pytest.mark.parametrize("order", [3, 4])
@pytest.mark.parametrize("strategy", STRATS)
def test_plan_rule_and_world1(order, strategy):
    sched = cpd.build_schedule(order, strategy, 6)
    dims = [8, 6, 5, 4][:order]
    f1, p1 = cpd.shard_plan(order, strategy, 6, dims, 3, 1)
    assert not f1.any() and not p1.any()  # one rank: nothing is sharded or exchanged
    f2, p2 = cpd.shard_plan(order, strategy, 6, dims, 3, 2)
    flat = sched.flat()
    assert len(f2) == flat.shape[0]
    for (it, b, mode, src, c, prod), f, p in zip(flat, f2, p2):
        assert bool(f & cpd.SHARD_SRC_SHARDED) == bool(src & 1)
        assert bool(f & cpd.SHARD_ALLREDUCE) == bool((src & 1) and c == 0)
        assert bool(f & cpd.SHARD_OUT_SHARDED) == bool(prod & 1)
        words = 0
        if f & cpd.SHARD_ALLREDUCE:
            words = int(np.prod([dims[k] if prod >> k & 1 else 3 for k in range(order)]))
        if f & cpd.SHARD_GATHER_V:
            assert mode == 0 and prod == 1
            words += dims[0] * 3
        assert p == words


def test_eager_allreduce_payloads_match_survey():
    """C2 2,0 reductions per steady sweep (71 MB, 0);
    C5 2,0,3 (10.7 GB, 0, 3.2 GB), largest single 8.59 GB."""
    for dims, rank, cyc, want in (((512,) * 3, 32, 2, [(2, 71e6), (0, 0)]),
                                  ((256,) * 4, 64, 3, [(2, 10.7e9), (0, 0), (3, 3.2e9)])):
        order = len(dims)
        sched = cpd.build_schedule(order, "branch-reuse", 12)
        flags, pay = cpd.shard_plan(order, "branch-reuse", 12, dims, rank, 2)
        flat = sched.flat()
        per = {}
        for (it, *_), f, p in zip(flat, flags, pay):
            if f & cpd.SHARD_ALLREDUCE:
                n, b = per.get(int(it), (0, 0))
                per[int(it)] = (n + 1, b + int(p) * 8)
        start = sched.cycle_start
        got = [per.get(i, (0, 0)) for i in range(start, start + cyc)]
        # the cycle phase is fixed by the schedule; compare as a rotation
        rots = [got[i:] + got[:i] for i in range(cyc)]
        assert any(all(g[0] == w[0] and abs(g[1] - w[1]) <= 0.02 * max(w[1], 1)
                       for g, w in zip(r, want)) for r in rots), got
    # largest single exchange at C5: the root X x_1 Q_1^T -> Y(2,3,4), 64 x 256^3 doubles
    flags, pay = cpd.shard_plan(4, "branch-reuse", 12, (256,) * 4, 64, 2)
    assert int(pay.max()) * 8 == 64 * 256 ** 3 * 8  # 8.59 GB


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, order, strategy, sweeps, errq):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = [8, 6, 5, 4][:order]
        R = 3
        rng = np.random.default_rng(11)
        x = rng.standard_normal(dims)
        qs = [np.linalg.qr(rng.standard_normal((d, R)))[0] for d in dims]
        rows = dims[0] // world
        lo = rank * rows
        xl = x[lo:lo + rows]
        sched = cpd.build_schedule(order, strategy, sweeps)
        flags, pay = cpd.shard_plan(order, strategy, sweeps, dims, R, world)
        root = (1 << order) - 1
        cache = {}
        i = 0
        for it in range(sweeps):
            for up in sched.iteration(it):
                y = None
                for st in up.steps:
                    f = int(flags[i])
                    i += 1
                    src = xl if st.source == root else cache[st.source]
                    assert bool(f & cpd.SHARD_SRC_SHARDED) == (src.shape[0] == rows and
                                                               st.source & 1 == 1)
                    q = qs[st.contract_mode]
                    if st.contract_mode == 0 and f & cpd.SHARD_SRC_SHARDED:
                        q = q[lo:lo + rows]
                    out = ttm(src, q, st.contract_mode)
                    if f & cpd.SHARD_ALLREDUCE:
                        t = torch.from_numpy(np.ascontiguousarray(out))
                        dist.all_reduce(t)
                        out = t.numpy()
                    if st.produces == (1 << up.mode):
                        y = out
                        if f & cpd.SHARD_GATHER_V:  # V = Y_(0) Q0: gather rows
                            parts = [torch.zeros_like(torch.from_numpy(out))
                                     for _ in range(world)]
                            dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(out)))
                            y = np.concatenate([p.numpy() for p in parts], axis=0)
                    else:
                        cache[st.produces] = out
                want = x
                for k in range(order):
                    if k != up.mode:
                        want = ttm(want, qs[k], k)
                np.testing.assert_allclose(y, want, rtol=1e-12, atol=1e-12)
                # the factor update changes Q_n (versions advance): new Q_n,
                # identical on every rank (replicated tail)
                qs[up.mode] = np.linalg.qr(
                    np.random.default_rng(100 * it + up.mode).standard_normal(
                        (dims[up.mode], R)))[0]
                # entries that absorbed the old Q_n are now stale and, by the
                # schedule's freshness invariant, never read again
                cache = {k: v for k, v in cache.items() if k >> up.mode & 1}
        assert i == len(flags)
    except Exception as e:  # surfaced to the parent
        errq.put(f"rank {rank}: {e!r}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("order,strategy", [(3, "branch-reuse"), (4, "branch-reuse"),
                                            (3, "dim-tree"), (4, "naive")])
def test_sharded_chain_gloo_world2(order, strategy):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, order, strategy, 5, errq))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), errs
