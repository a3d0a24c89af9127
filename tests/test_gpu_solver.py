"""GPU: the device-resident CP-ALS-QR solver against the CPU oracle.

Tolerances (BASELINE.json north star): relative fitness and factor error
<= 1e-10 per sweep, identical trace length, update order, beta-activation
sweep and integer flops / root-TTM counts.
"""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
META = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")))
FIT_TOL = 1e-10
FACTOR_TOL = 1e-10


def cfg_of(rank, iters, seed=0, strategy="branch-reuse", **kw):
    import paper_2503_18759_b200 as cpd
    return cpd.SolverConfig(rank=rank, max_iterations=iters, seed=seed, strategy=strategy, **kw)


def compare(gpu, ora, *, fit_tol=FIT_TOL, factor_tol=FACTOR_TOL, check_factors=True):
    assert len(gpu.trace) == len(ora.trace)
    for g, o in zip(gpu.trace, ora.trace):
        assert g.iteration == o["iteration"]
        assert g.update_order == o["update_order"]
        assert g.flops == o["flops"] and g.root_ttm_count == o["root_ttm_count"]
        assert g.beta_used == o["beta_used"], (g.iteration, g.beta_used, o["beta_used"])
        assert abs(g.fitness - o["fitness"]) <= fit_tol * max(abs(o["fitness"]), 1e-300), \
            (g.iteration, g.fitness, o["fitness"])
    if check_factors:
        for k, (fg, fo) in enumerate(zip(gpu.model.factors, ora.factors)):
            err = np.linalg.norm(fg - fo) / np.linalg.norm(fo)
            assert err <= factor_tol, (k, err)
        assert np.linalg.norm(gpu.model.lam - ora.lam) / np.linalg.norm(ora.lam) <= factor_tol


@pytest.mark.parametrize("dims,rank", [((9, 8, 7), 3), ((7, 6, 5, 4), 3), ((10, 10, 10), 4),
                                       ((16, 24, 20), 5), ((12, 10, 8, 16), 4)])
@pytest.mark.parametrize("variant", ["naive", "dim-tree", "branch-reuse", "bre"])
def test_small_trajectories(ctx, port, dims, rank, variant):
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(31, int(np.prod(dims))).reshape(dims)
    if variant == "bre":
        g = cpd.als_qr_bre(x, cfg_of(rank, 12, seed=3), ctx=ctx)
        o = port.solve(x, rank, 12, extrapolate=True, seed=3)
    else:
        g = cpd.cp_als_qr(x, cfg_of(rank, 12, seed=3, strategy=variant), ctx=ctx)
        o = port.solve(x, rank, 12, extrapolate=False, strategy=variant, seed=3)
    # measured (tools/parity_floor.py, profiles/r02_parity_floor.jsonl): fit
    # <= 1.9e-14, factors <= 8e-15, the oracle's own 1e-15-perturbation floor
    # is the same order -- the north-star bar holds with 4 digits to spare
    compare(g, o)


def test_c1_full_config(ctx, port, golden):
    """BASELINE config 1: 100^3 R10 + 1e-2 noise, 50 sweeps ALS-QR-BRE."""
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(0, (100, 100, 100), 10, 1e-2, META["truth_seeds"]["c1"])
    g = cpd.als_qr_bre(x, cfg_of(10, 50, seed=META["init_seed"]), ctx=ctx, dump_per_sweep=True)
    o = port.solve(x, 10, 50, extrapolate=True, seed=META["init_seed"], dump_per_sweep=True)
    compare(g, o)
    first = next(t.iteration for t in g.trace if t.beta_used != 0.0)
    assert first == 8
    for s in range(50):
        for k in range(3):
            fo = o.factors_per_sweep[s][k]
            assert np.linalg.norm(g.factors_per_sweep[s][k] - fo) / np.linalg.norm(fo) <= FACTOR_TOL
    assert np.array_equal(np.array([t["fitness"] for t in o.trace]), golden["c1_fitness"])


def test_c4_ill_conditioned_reduced(ctx, port):
    """C4 construction (congruence 0.9, log-scaled columns, 1e-4 noise) at 48^3 R20."""
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(1, (48, 48, 48), 20, 1e-4, META["truth_seeds"]["c4"])
    g = cpd.als_qr_bre(x, cfg_of(20, 60, seed=META["init_seed"]), ctx=ctx)
    o = port.solve(x, 20, 60, extrapolate=True, seed=META["init_seed"])
    # measured: fit 1.5e-11 (oracle floor 1.3e-11), factors 1.1e-12
    compare(g, o)


def test_c3_shape_4th_order_reduced(ctx, port):
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(0, (24, 24, 24, 24), 16, 1e-2, META["truth_seeds"]["c3"])
    g = cpd.als_qr_bre(x, cfg_of(16, 20, seed=META["init_seed"]), ctx=ctx)
    o = port.solve(x, 16, 20, extrapolate=True, seed=META["init_seed"])
    compare(g, o)


def test_q0_structure_observed(ctx, port):
    """solver_test.cpp:182-195"""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(557, 9 * 8 * 7).reshape(9, 8, 7)
    seen = []

    def obs(sweep, mode, q0):
        seen.append((sweep, mode))
        assert abs(q0[0, 0] - 1.0) <= 1e-12
        assert np.abs(q0[0, 1:]).max() <= 1e-12
        assert np.abs(q0[1:, 0]).max() <= 1e-12

    cpd.cp_als_qr(x, cfg_of(3, 4, seed=11, q0_observer=obs), ctx=ctx)
    assert len(seen) == 12


def test_beta_zero_and_gate(ctx, port):
    """solver_test.cpp:226-249: beta 0 == plain branch reuse; gap 0 never fires."""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(577, 8 * 7 * 6).reshape(8, 7, 6)
    a = cpd.als_qr_bre(x, cfg_of(3, 6, seed=21, beta_override=0.0), ctx=ctx)
    b = cpd.cp_als_qr(x, cfg_of(3, 6, seed=21), ctx=ctx)
    assert [t.fitness for t in a.trace] == [t.fitness for t in b.trace]
    for fa, fb in zip(a.model.factors, b.model.factors):
        assert np.array_equal(fa, fb)
    c = cpd.als_qr_bre(x, cfg_of(3, 6, seed=23, activation_gap=0.0), ctx=ctx)
    assert all(t.beta_used == 0.0 for t in c.trace)


def test_deterministic(ctx, port):
    """solver_test.cpp:272-282: bit-identical traces across runs."""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(593, 7 * 6 * 5).reshape(7, 6, 5)
    r1 = cpd.cp_als_qr(x, cfg_of(2, 6, seed=77), ctx=ctx)
    r2 = cpd.cp_als_qr(x, cfg_of(2, 6, seed=77), ctx=ctx)
    assert [(t.fitness, t.raw_radicand) for t in r1.trace] == \
        [(t.fitness, t.raw_radicand) for t in r2.trace]


def test_rejections(ctx, port):
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(571, 6 * 5 * 2).reshape(6, 5, 2)
    with pytest.raises(ValueError):
        cpd.cp_als_qr(x, cfg_of(3, 3), ctx=ctx)
    with pytest.raises(ValueError):
        cpd.cp_als_qr(np.zeros((4, 4, 4)), cfg_of(2, 3), ctx=ctx)
    with pytest.raises(ValueError):
        cpd.cp_als_qr(x, cfg_of(2, 0), ctx=ctx)


def test_early_stop_on_threshold(ctx, port):
    """solver_test.cpp:284-294: an exact low-rank tensor stops early."""
    import paper_2503_18759_b200 as cpd
    a = [port.rng_normals(600 + k, d * 2).reshape(d, 2) for k, d in enumerate((6, 5, 4))]
    x = np.einsum("ir,jr,kr->ijk", *a)
    r = cpd.cp_als_qr(x, cfg_of(2, 50, seed=3, fitness_threshold=0.999), ctx=ctx)
    assert len(r.trace) < 50 and r.trace[-1].fitness >= 0.999


def test_teacher_forced_one_sweep(ctx, port):
    """load the oracle state at sweep k, run one GPU sweep, compare
    with the oracle's sweep k+1 -- separates kernel error from drift."""
    import paper_2503_18759_b200 as cpd
    from oracle.pyoracle import SweepState
    x = port.synth_baseline(1, (40, 40, 40), 8, 1e-4, 77)
    for k in (1, 2, 5, 9):
        s0 = port.solve(x, 8, k, extrapolate=True, seed=7, state=SweepState(
            0, np.ones(8), port_init(port, x.shape, 8, 7)))
        st = s0.state
        o = port.solve(x, 8, 1, extrapolate=True, seed=7, state=SweepState(**st))
        g = ctx_solve_state(ctx, x, 8, st)
        assert g.trace[0].iteration == k + 1
        assert g.trace[0].flops == o.trace[0]["flops"]
        # one sweep from identical state: only kernel rounding separates the
        # two; the radicand cancels ~3 digits at fit 0.999 (SURVEY.md 8c floor)
        assert abs(g.trace[0].fitness - o.trace[0]["fitness"]) <= FIT_TOL * o.trace[0]["fitness"]
        for fg, fo in zip(g.model.factors, o.factors):
            assert np.linalg.norm(fg - fo) / np.linalg.norm(fo) <= 1e-11


def port_init(port, dims, rank, seed):
    draws = port.rng_normals(seed, sum(d * rank for d in dims))
    out, off = [], 0
    for d in dims:
        out.append(port.normalize_columns(draws[off:off + d * rank].reshape(d, rank))[0])
        off += d * rank
    return out


def ctx_solve_state(ctx, x, rank, st):
    import paper_2503_18759_b200 as cpd
    ctx.set_tensor(x)
    state = cpd.SweepState(**st)
    return ctx.solve(cfg_of(rank, 1, seed=7), extrapolate=True, state=state)


# ---------------------------------------------------------------- full BASELINE sizes
FULL = {  # (kind, dims, rank, rho)  BASELINE.json configs 2, 3, 5
    "c2": (0, (512, 512, 512), 32, 1e-3),
    "c3": (0, (128, 128, 128, 128), 16, 1e-2),
    "c5": (0, (256, 256, 256, 256), 64, 1e-3),
}


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_full_size_sweep_properties(name):
    """Size-independent properties at BASELINE's full sizes (C5: 34 GB in HBM):
    integer flops / root counts equal the scheduler's dry run (bit-exact),
    update orders follow the plan, factors have unit columns and Q has
    orthonormal columns, fitness in [0, 1], and a second run is bit-identical."""
    import paper_2503_18759_b200 as cpd
    kind, dims, rank, rho = FULL[name]
    sweeps = 4
    ctx = cpd.Context(0)
    ctx.synth_tensor(kind, list(dims), rank, rho, META["truth_seeds"][name])
    cfg = cfg_of(rank, sweeps, seed=META["init_seed"])
    runs = []
    for _ in range(2):
        s = ctx.session(cfg, extrapolate=True)
        rows = s.run(sweeps)
        model = s.end()
        s.close()
        runs.append((rows, model))
    rows, model = runs[0]
    sched = cpd.build_schedule(len(dims), "branch-reuse", sweeps)
    for i, r in enumerate(rows):
        fl, roots = cpd.measured_cost(len(dims), "branch-reuse", dims, rank, i + 1)
        assert r.flops == fl and r.root_ttm_count == roots
        assert r.update_order == sched.update_order(i)
        assert 0.0 <= r.fitness <= 1.0
    for f in model.factors:
        assert np.allclose(np.linalg.norm(f, axis=0), 1.0, atol=1e-12)
        assert np.linalg.matrix_rank(f) == rank
    assert [(r.fitness, r.raw_radicand) for r in runs[1][0]] == \
        [(r.fitness, r.raw_radicand) for r in rows]
    for fa, fb in zip(runs[1][1].factors, model.factors):
        assert np.array_equal(fa, fb)


@pytest.mark.parametrize("name,k", [("c2", 2), ("c3", 3)])
def test_full_size_teacher_forced(port, name, k):
    """Teacher-forced sweep at BASELINE's full C2 / C3 size: the oracle's state
    after sweep k (restated C port, single core) -> one device sweep vs the
    oracle's sweep k+1.  Fitness <= 1e-10 relative, factors
    <= 1e-10, identical integer flops."""
    import paper_2503_18759_b200 as cpd
    from oracle.pyoracle import SweepState
    kind, dims, rank, rho = FULL[name]
    ctx = cpd.Context(0)
    ctx.synth_tensor(kind, list(dims), rank, rho, META["truth_seeds"][name])
    x = ctx.get_tensor(list(dims))
    init = port_init(port, x.shape, rank, META["init_seed"])
    s0 = port.solve(x, rank, k, extrapolate=True, seed=META["init_seed"],
                    state=SweepState(0, np.ones(rank), init))
    st = s0.state
    o = port.solve(x, rank, 1, extrapolate=True, seed=META["init_seed"], state=SweepState(**st))
    g = ctx.solve(cfg_of(rank, 1, seed=META["init_seed"]), extrapolate=True,
                  state=cpd.SweepState(**st))
    assert g.trace[0].iteration == k + 1
    assert g.trace[0].flops == o.trace[0]["flops"]
    assert g.trace[0].root_ttm_count == o.trace[0]["root_ttm_count"]
    assert abs(g.trace[0].fitness - o.trace[0]["fitness"]) <= FIT_TOL * o.trace[0]["fitness"]
    for fg, fo in zip(g.model.factors, o.factors):
        assert np.linalg.norm(fg - fo) / np.linalg.norm(fo) <= FACTOR_TOL


def test_repeated_solves_bit_identical_with_root_prefetch():
    """Steady branch-reuse sweeps overlap the root TTM (low-priority stream)
    with the preceding update.  Repeated solves in one context must stay
    bit-identical (this shape exposed the TMA TTM's early stage release beside
    DSMEM cluster CTAs; tools/det_probe.py)."""
    import paper_2503_18759_b200 as cpd
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, [96, 96, 96, 96], 16, 1e-2, 12345)
    ref = None
    for _ in range(6):
        s = ctx.session(cfg_of(16, 4, seed=7), extrapolate=True)
        rows = s.run(4)
        model = s.end()
        s.close()
        got = ([(r.fitness, r.raw_radicand) for r in rows], [f.copy() for f in model.factors])
        if ref is None:
            ref = got
        else:
            assert got[0] == ref[0]
            for a, b in zip(got[1], ref[1]):
                assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,rank", [((9, 8, 7), 1), ((20, 18, 16), 7), ((30, 28, 26), 13),
                                       ((40, 38, 36), 33), ((70, 66, 65), 64),
                                       ((12, 11, 10, 9), 9), ((10, 9, 8, 8, 7), 5)])
def test_rank_edges_vs_oracle(ctx, port, dims, rank):
    """Rank 1, ranks that are not multiples of 8 (padding of the DMMA
    fragments and the packed Q), R = 33 (the RM = 64 templates with one
    padding block), R = 64 (largest supported), 4th order with R = I_n, and a
    5th-order tensor (naive plan only; the tree plans are orders 3-4)."""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(4242 + rank, int(np.prod(dims))).reshape(dims)
    if len(dims) == 5:
        g = cpd.cp_als_qr(x, cfg_of(rank, 4, seed=5, strategy="naive"), ctx=ctx)
        o = port.solve(x, rank, 4, extrapolate=False, strategy="naive", seed=5)
    else:
        g = cpd.als_qr_bre(x, cfg_of(rank, 6, seed=5), ctx=ctx)
        o = port.solve(x, rank, 6, extrapolate=True, seed=5)
    compare(g, o)  # measured: fit <= 1.3e-14, factors <= 4.2e-15


@pytest.mark.parametrize("early", ["1", "0"])
@pytest.mark.parametrize("overlap_sms", ["", "0", "16"])
def test_schedule_variants_match_oracle(ctx, port, monkeypatch, early, overlap_sms):
    """The event-driven sweep-boundary front (CPDB_EARLY_FRONT: the next
    update's Z-QR and chain run under the previous update's V-GEMM/finisher)
    and the SM budget of updates beside the prefetched root (CPDB_OVERLAP_SMS)
    only reorder launches: trajectories match the oracle and repeat bit for
    bit.  C2 construction at 64^3 R16 (Z-QR 256 x 16)."""
    import paper_2503_18759_b200 as cpd
    monkeypatch.setenv("CPDB_EARLY_FRONT", early)
    if overlap_sms:
        monkeypatch.setenv("CPDB_OVERLAP_SMS", overlap_sms)
    x = port.synth_baseline(0, (64, 64, 64), 16, 1e-3, META["truth_seeds"]["c2"])
    g = cpd.als_qr_bre(x, cfg_of(16, 24, seed=META["init_seed"]), ctx=ctx)
    o = port.solve(x, 16, 24, extrapolate=True, seed=META["init_seed"])
    compare(g, o)  # measured: fit 9.4e-12, factors 2.6e-16
    g2 = cpd.als_qr_bre(x, cfg_of(16, 24, seed=META["init_seed"]), ctx=ctx)
    assert [t.fitness for t in g2.trace] == [t.fitness for t in g.trace]
    for a, b in zip(g.model.factors, g2.model.factors):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("speculate", ["1", "0"])
@pytest.mark.parametrize("dims", [(40, 36, 32), (20, 18, 16, 14)])
def test_stop_test_undoes_speculative_update(ctx, port, monkeypatch, speculate, dims):
    """The next sweep's first update is issued before the host reads the
    fitness (beta decided on the device).  When the stop test fires, that
    update is undone: trace, factors and lambda equal the oracle's, which
    never ran it (solvers.hpp:301)."""
    import paper_2503_18759_b200 as cpd
    monkeypatch.setenv("CPDB_SPECULATE", speculate)
    x = port.synth_baseline(0, dims, 3, 1e-2, 20250011)
    # threshold midway between the oracle's fitness at sweeps k-1 and k (the
    # last sweep <= 10 that still gains > 1e-9): the run stops at sweep k
    # whatever the last bits of either side's fitness
    f = [t["fitness"] for t in port.solve(x, 3, 10, extrapolate=True, seed=5).trace]
    k = max(i + 1 for i in range(2, 10) if f[i] - f[i - 1] > 1e-9)
    thr = 0.5 * (f[k - 2] + f[k - 1])
    o = port.solve(x, 3, 40, extrapolate=True, seed=5, fitness_threshold=thr)
    assert len(o.trace) == k
    g = cpd.als_qr_bre(x, cfg_of(3, 40, seed=5, fitness_threshold=thr), ctx=ctx)
    compare(g, o)


def test_tall_z_fourth_order_vs_oracle(ctx, port):
    """The tall-Z Z-QR (multi-kernel form, C5's path: Z = 32768 x 32 does not
    fit the 8-CTA cluster) on a fourth-order tensor, BRE, against the oracle."""
    import paper_2503_18759_b200 as cpd
    dims = (40, 36, 34, 33)
    x = port.synth_baseline(0, dims, 32, 1e-3, META["truth_seeds"]["c5"])
    g = cpd.als_qr_bre(x, cfg_of(32, 8, seed=META["init_seed"]), ctx=ctx)
    o = port.solve(x, 32, 8, extrapolate=True, seed=META["init_seed"])
    compare(g, o)  # measured: fit 1.5e-13, factors 1.7e-14
    assert any(t.beta_used != 0.0 for t in g.trace)  # the history path runs too


# ---------------------------------------------------------------- C5 (north star config 5)
@pytest.mark.parametrize("k", [3, 4, 5, 12])
def test_c5_proxy_teacher_forced(port, k):
    """BASELINE config 5's device path -- fourth order, R = 64: the tall
    multi-kernel Z-QR of Z = 262144 x 64 (zqr_rows/apply/fin<64>),
    vgemm<64>, finish_cluster<64>, the 3-cycle branch reuse -- at the 64^4
    proxy of the 256^4 tensor (Z and every R-sized operand keep their C5
    size).  The device's state after sweep k -> one oracle sweep (the
    reference's Householder thin_qr on that Z, linalg.hpp:39-99) vs the
    device's sweep k+1, both uninterrupted and resumed from the state.  k =
    3, 4, 5 cover the three phases of the cycle (dim_tree.hpp:411-422); k =
    12 runs with the Q0 history in use.  Fitness, factors and lambda <= 1e-10
    relative; integer flops, root counts, update order and beta identical."""
    from tools.teacher_forced import CONFIGS, TRUTH_SEED, run
    kind, _, rank, rho = CONFIGS["c5"]
    r = run(kind, (64, 64, 64, 64), rank, rho, TRUTH_SEED["c5"], k, port=port)
    for name in ("continued", "resumed"):
        g = r[name]
        assert g["iteration"] == g["oracle_iteration"] == k + 1
        assert g["flops"] == g["oracle_flops"] and g["root_ttms"] == g["oracle_root_ttms"]
        assert g["update_order"] == g["oracle_update_order"]
        assert g["beta_used"] == g["oracle_beta_used"]
        assert g["rel_fitness_err"] <= FIT_TOL, (name, g)
        assert max(g["rel_factor_err"]) <= FACTOR_TOL, (name, g)
        assert g["rel_lambda_err"] <= FACTOR_TOL, (name, g)


# ---------------------------------------------------------------- full-length BASELINE parity
FULL_LENGTH = {  # (kind, dims, rank, rho, sweeps): BASELINE.json configs 2, 3, 4
    "c2": (0, (512, 512, 512), 32, 1e-3, 100),
    "c3": (0, (128, 128, 128, 128), 16, 1e-2, 100),
    "c4": (1, (256, 256, 256), 20, 1e-4, 500),
}


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_length_parity(port, name):
    """Every sweep of BASELINE configs 2-4 at full size and full sweep count,
    device vs the oracle (the C restatement, bit-identical to the reference:
    tests/test_oracle.py) on the same device-generated tensor: fitness and
    final factors / lambda <= 1e-10 relative on every sweep, identical trace
    length, update order, integer flops / root counts and beta-activation
    sweep (solver_test.cpp:168-180).  Measured round 1 on the
    reference itself: C2 1.7e-13, C3 4.0e-11, C4 5.1e-11 (its own 1e-15
    perturbation floor 1.7e-11)."""
    import paper_2503_18759_b200 as cpd
    kind, dims, rank, rho, sweeps = FULL_LENGTH[name]
    ctx = cpd.Context(0)
    ctx.synth_tensor(kind, list(dims), rank, rho, META["truth_seeds"][name])
    x = ctx.get_tensor(list(dims))
    g = ctx.solve(cfg_of(rank, sweeps, seed=META["init_seed"]), extrapolate=True)
    o = port.solve(x, rank, sweeps, extrapolate=True, seed=META["init_seed"])
    compare(g, o)
    fb = [t.iteration for t in g.trace if t.beta_used != 0.0]
    ob = [t["iteration"] for t in o.trace if t["beta_used"] != 0.0]
    assert fb[:1] == ob[:1] and len(fb) == len(ob)
    ctx.close()


@pytest.mark.parametrize("dims", [(40, 36, 32), (20, 18, 16, 14)])
def test_breakdown_in_undone_update_is_not_reported(ctx, port, monkeypatch, dims):
    """The next sweep's first update runs speculatively before the host reads
    this sweep's fitness; its status word is its own (one per sweep parity).
    A breakdown there (CPDB_FAULT_SWEEP injects one) after the stop test
    fired is discarded with the undone update -- the converged model comes
    back -- while the same breakdown in a sweep that is consumed raises, as
    the reference would (linalg.hpp:199-203)."""
    import paper_2503_18759_b200 as cpd
    x = port.synth_baseline(0, dims, 3, 1e-2, 20250011)
    f = [t["fitness"] for t in port.solve(x, 3, 10, extrapolate=True, seed=5).trace]
    k = max(i + 1 for i in range(2, 10) if f[i] - f[i - 1] > 1e-9)
    thr = 0.5 * (f[k - 2] + f[k - 1])
    o = port.solve(x, 3, 40, extrapolate=True, seed=5, fitness_threshold=thr)
    assert len(o.trace) == k
    monkeypatch.setenv("CPDB_FAULT_SWEEP", str(k + 1))
    g = cpd.als_qr_bre(x, cfg_of(3, 40, seed=5, fitness_threshold=thr), ctx=ctx)
    compare(g, o)
    monkeypatch.setenv("CPDB_FAULT_SWEEP", str(k - 1))
    with pytest.raises(cpd.SingularTriangularError):
        cpd.als_qr_bre(x, cfg_of(3, 40, seed=5, fitness_threshold=thr), ctx=ctx)


@pytest.mark.parametrize("delta", [1e-8, 1e-10])
def test_ill_conditioned_factors_do_not_break_down(ctx, port, delta):
    """Two nearly collinear rank-1 terms (columns equal to `delta` in two
    modes) drive kappa(A_n) to ~2e9 (delta 1e-8) / ~7e12 (1e-10): the
    CholeskyQR2 Gram is numerically indefinite there.  The reference's
    Householder QR carries on (linalg.hpp:39-99); so must we -- the first
    pass retries with a shifted Gram (rowalg.cuh chol_first_pass) and the
    second restores orthogonality.  The fitness (well conditioned) agrees
    with the oracle's to within the oracle's own sensitivity, measured here
    with a 1e-15 relative perturbation of X."""
    import paper_2503_18759_b200 as cpd
    rng = np.random.default_rng(5)
    dims, R = (30, 28, 26), 3
    a = [rng.standard_normal((d, R)) for d in dims]
    a[0][:, 1] = a[0][:, 0] + delta * rng.standard_normal(dims[0])
    a[1][:, 1] = a[1][:, 0] + delta * rng.standard_normal(dims[1])
    x = np.einsum("ir,jr,kr->ijk", *a)
    o = port.solve(x, R, 15, extrapolate=True, seed=7)
    xp = x * (1.0 + 1e-15 * np.random.default_rng(6).standard_normal(x.shape))
    op = port.solve(xp, R, 15, extrapolate=True, seed=7)
    g = cpd.als_qr_bre(x, cfg_of(R, 15, seed=7), ctx=ctx)
    assert ctx.profile()["qr_shifted"] > 0  # the retry did run
    assert len(g.trace) == len(o.trace) == 15
    floor = max(abs(a_["fitness"] - b["fitness"]) for a_, b in zip(op.trace, o.trace))
    err = max(abs(t.fitness - b["fitness"]) for t, b in zip(g.trace, o.trace))
    print(f"delta {delta}: fitness gap {err:.2e}, oracle floor {floor:.2e}")
    assert err <= max(1e-9, 100 * floor), (err, floor)
    for t, b in zip(g.trace, o.trace):
        assert t.flops == b["flops"] and t.update_order == b["update_order"]


@pytest.mark.parametrize("dims,rank", [((40, 36, 32), 8), ((20, 18, 16, 14), 6),
                                       ((512, 512, 512), 32), ((128, 128, 128, 128), 16)])
def test_split_runs_keep_the_pipeline_and_the_results(dims, rank):
    """A resumable session issues the next sweep's first update ahead of the
    host sync even on the last sweep of a run() call.  run(a) + run(b) must be
    bit-identical to run(a + b); end() after run(a) takes the work issued
    ahead back and returns the state after a sweeps (a fresh a-sweep run's,
    bit for bit), after which the session accepts no further run()."""
    import paper_2503_18759_b200 as cpd
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, list(dims), rank, 1e-3, 4711)  # (beta gate opens mid-run)

    def go(parts, iters):
        s = ctx.session(cfg_of(rank, iters, seed=11), extrapolate=True)
        rows = []
        for n in parts:
            rows += s.run(n)
        m = s.end()
        return s, [(r.iteration, r.fitness, r.raw_radicand, r.flops, r.beta_used) for r in rows], m

    s0, whole, m_whole = go([12], 12)
    s0.close()
    s1, split, m_split = go([1, 4, 2, 5], 12)
    s1.close()
    assert split == whole
    assert np.array_equal(m_split.lam, m_whole.lam)
    for a, b in zip(m_split.factors, m_whole.factors):
        assert np.array_equal(a, b)
    # end() in the middle of a longer session == a run that stops there
    s2, part, m_part = go([7], 12)
    s3, short, m_short = go([7], 7)
    s3.close()
    assert part == short == whole[:7]
    assert np.array_equal(m_part.lam, m_short.lam)
    for a, b in zip(m_part.factors, m_short.factors):
        assert np.array_equal(a, b)
    with pytest.raises(cpd.CpdLogicError):
        s2.run(1)
    s2.close()


@pytest.mark.parametrize("dims,rank,variant,sweeps", [
    ((70, 68, 66), 65, "bre", 8),
    ((100, 96, 98), 96, "bre", 6),
    ((140, 132, 136), 130, "dim-tree", 3),
    ((132, 131, 130), 130, "naive", 2),
    ((66, 65, 67, 65), 65, "bre", 3),
])
def test_wide_ranks_vs_oracle(ctx, port, dims, rank, variant, sweeps):
    """Ranks above 64 (the reference accepts any rank up to the smallest
    extent, solvers.hpp:221-224): the rank-generic tail (widerank.cu --
    Khatri-Rao + cooperative Householder QR, row solves, exact normalisation)
    behind the same session, against the oracle at the north-star bar."""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(900 + rank, int(np.prod(dims))).reshape(dims)
    if variant == "bre":
        g = cpd.als_qr_bre(x, cfg_of(rank, sweeps, seed=5), ctx=ctx)
        o = port.solve(x, rank, sweeps, extrapolate=True, seed=5)
    else:
        g = cpd.cp_als_qr(x, cfg_of(rank, sweeps, seed=5, strategy=variant), ctx=ctx)
        o = port.solve(x, rank, sweeps, extrapolate=False, strategy=variant, seed=5)
    compare(g, o)


@pytest.mark.parametrize("dims,rank,variant", [((9, 8, 7), 3, "bre"), ((16, 24, 20), 5, "dim-tree"),
                                               ((12, 10, 8, 16), 4, "bre"), ((40, 38, 36), 33, "bre"),
                                               ((70, 66, 65), 64, "naive")])
def test_householder_kernels_at_small_ranks(ctx, port, monkeypatch, dims, rank, variant):
    """CPDB_HOUSEHOLDER=1 swaps the CholeskyQR kernels for the rank-generic
    Householder ones (widerank.cu) at any rank: same trajectories."""
    import paper_2503_18759_b200 as cpd
    monkeypatch.setenv("CPDB_HOUSEHOLDER", "1")
    x = port.rng_normals(61, int(np.prod(dims))).reshape(dims)
    if variant == "bre":
        g = cpd.als_qr_bre(x, cfg_of(rank, 10, seed=3), ctx=ctx)
        o = port.solve(x, rank, 10, extrapolate=True, seed=3)
    else:
        g = cpd.cp_als_qr(x, cfg_of(rank, 10, seed=3, strategy=variant), ctx=ctx)
        o = port.solve(x, rank, 10, extrapolate=False, strategy=variant, seed=3)
    compare(g, o)


def test_breakdown_restarts_on_householder(ctx, port, monkeypatch):
    """A CholeskyQR breakdown that the shifted retry cannot cure does not end
    the solve where the reference's Householder QR carries on
    (linalg.hpp:39-99): cpdb_solve starts the run again on the Householder
    kernels.  The test hook injects the breakdown into the CholeskyQR attempt
    only; the restarted run matches the oracle."""
    import paper_2503_18759_b200 as cpd
    dims, rank = (40, 36, 32), 6
    x = port.synth_baseline(0, dims, rank, 1e-2, 20250017)
    o = port.solve(x, rank, 12, extrapolate=True, seed=5)
    monkeypatch.setenv("CPDB_FAULT_SWEEP", "4")
    monkeypatch.setenv("CPDB_FAULT_ONCE", "1")
    g = cpd.als_qr_bre(x, cfg_of(rank, 12, seed=5), ctx=ctx)
    assert ctx.profile()["qr_householder"] == 1
    compare(g, o)


@pytest.mark.parametrize("dims,rank,extrap", [((40, 36, 32), 8, True), ((40, 36, 32), 8, False),
                                              ((20, 18, 16, 14), 6, True),
                                              ((256, 256, 256), 20, True),
                                              ((64, 64, 64, 64), 16, True)])
def test_boundary_repetition_elided_bit_identical(monkeypatch, dims, rank, extrap):
    """The permuted update orders end one sweep and begin the next with the
    same mode, whose Z-QR and TTM chain inputs have not changed in between:
    the session takes the previous update's Y_(n) / Q0 / R0 instead of
    launching the kernels again (mode_update_front).  Same bits as
    recomputing (CPDB_REUSE_BOUNDARY=0), same integer cost report, also when
    the stop test undoes a speculative update that reused."""
    import paper_2503_18759_b200 as cpd
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, list(dims), rank, 1e-2, 99)

    def go(reuse, iters, thr=1.0):
        monkeypatch.setenv("CPDB_REUSE_BOUNDARY", reuse)
        cfg = cfg_of(rank, iters, seed=3, fitness_threshold=thr)
        ctx.profile()
        r = ctx.solve(cfg, extrapolate=extrap)
        return r, ctx.profile()["kernel_launches"]

    (a, la), (b, lb) = go("1", 14), go("0", 14)
    assert la < lb  # launches were elided
    assert [(t.fitness, t.raw_radicand, t.flops, t.root_ttm_count, t.beta_used) for t in a.trace] == \
           [(t.fitness, t.raw_radicand, t.flops, t.root_ttm_count, t.beta_used) for t in b.trace]
    for fa, fb in zip(a.model.factors, b.model.factors):
        assert np.array_equal(fa, fb)
    assert np.array_equal(a.model.lam, b.model.lam)
    # early stop in the middle: the undone speculative update had reused
    f = [t.fitness for t in a.trace]
    k = max(i for i in range(3, 12) if f[i] > f[i - 1])
    thr = 0.5 * (f[k - 1] + f[k])
    (c, _), (d, _) = go("1", 14, thr), go("0", 14, thr)
    assert len(c.trace) == len(d.trace) == k + 1
    for fa, fb in zip(c.model.factors, d.model.factors):
        assert np.array_equal(fa, fb)


@pytest.mark.parametrize("dims,rank", [((40, 36, 32), 8), ((20, 18, 16, 14), 6), ((256, 256, 256), 20),
                                       ((64, 64, 64, 64), 16)])
def test_gate_prediction_bit_identical(monkeypatch, dims, rank):
    """Before the beta gate opens, the next sweep's first update is issued on
    the prediction that it stays closed; on the sweep where it opens the
    update is taken back and issued again with beta (once per run).  Same
    bits as waiting for the gate on the device (CPDB_PREDICT_GATE=0), with
    and without the boundary reuse, also when the stop test fires on the
    activation sweep itself."""
    import paper_2503_18759_b200 as cpd
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, list(dims), rank, 1e-2, 99)

    def go(predict, reuse, iters, thr=1.0):
        monkeypatch.setenv("CPDB_PREDICT_GATE", predict)
        monkeypatch.setenv("CPDB_REUSE_BOUNDARY", reuse)
        r = ctx.solve(cfg_of(rank, iters, seed=3, fitness_threshold=thr), extrapolate=True)
        return r, ctx.profile()["gate_mispredictions"]

    def key(r):
        return [(t.fitness, t.raw_radicand, t.flops, t.beta_used) for t in r.trace]

    base, m0 = go("0", "0", 16)
    assert m0 == 0
    act = next(i for i, t in enumerate(base.trace) if t.beta_used != 0.0)  # first extrapolated sweep
    for reuse in ("0", "1"):
        got, m = go("1", reuse, 16)
        assert m == 1  # the gate opened once
        assert key(got) == key(base)
        for fa, fb in zip(got.model.factors, base.model.factors):
            assert np.array_equal(fa, fb)
    # stop on the sweep whose fitness opens the gate (the one before `act`)
    f = [t.fitness for t in base.trace]
    stop = act - 1
    if stop >= 1 and f[stop] > f[stop - 1]:
        thr = 0.5 * (f[stop - 1] + f[stop])
        a, _ = go("1", "1", 16, thr)
        b, _ = go("0", "0", 16, thr)
        assert len(a.trace) == len(b.trace) == stop + 1
        for fa, fb in zip(a.model.factors, b.model.factors):
            assert np.array_equal(fa, fb)
