"""SURVEY.md 8f row 1 on the device: the BASELINE generator and the sharded
.cpdt loader, pinned against the reference.

* Generator (csrc/synth.cu): the truth factors it exports rebuild X_clean
  through the reference's own reconstruct (kruskal.hpp:54-67, oracle/_ref) to
  1e-13; the noise has ||E|| = rho ||X_clean|| (BASELINE construction); the
  factor draws have the BASELINE distributions (i.i.d. N(0,1); C4's
  congruence-0.9 columns with log-uniform scales in [1e-3, 1]).
* Loader: each rank of a mode-0 sharded context reads exactly its slab
  (cpdb_shard_rows, ragged included) of a file written by the reference's own
  codec (io.hpp:93-121), bit for bit.
"""
import threading

import numpy as np
import pytest

import paper_2503_18759_b200 as cpd

pytestmark = pytest.mark.gpu


def checkers(port):
    from oracle.pyoracle import Oracle, available
    out = [port]
    if available("reference"):
        out.append(Oracle("reference"))
    return out


@pytest.mark.parametrize("kind,dims,rank", [
    (0, (20, 18, 16), 5), (0, (10, 9, 8, 7), 4), (0, (64, 48, 40), 20),
    (1, (30, 28, 26), 20), (1, (12, 11, 10, 9), 6),
])
def test_generator_truth_reconstructs_x_clean(ctx, port, kind, dims, rank):
    seed = 20250100 + rank
    ctx.synth_tensor(kind, list(dims), rank, 0.0, seed)
    x = ctx.get_tensor(list(dims))
    truth = ctx.synth_truth(kind, list(dims), rank, seed)
    for o in checkers(port):
        want = o.reconstruct(truth)
        err = np.linalg.norm(x - want) / np.linalg.norm(want)
        assert err <= 1e-13, (o.kind, err)
    n0, n1 = ctx.synth_norms()
    assert n1 == 0.0
    assert abs(n0 - np.sum(want * want)) <= 1e-13 * n0


@pytest.mark.parametrize("kind,dims,rank,rho", [
    (0, (40, 36, 32), 10, 1e-2), (0, (24, 20, 18, 16), 16, 1e-2), (0, (48, 44, 40), 32, 1e-3),
    (1, (48, 48, 48), 20, 1e-4),
])
def test_generator_noise_level(ctx, kind, dims, rank, rho):
    """X = X_clean + E with ||E|| = rho ||X_clean||: the difference of the rho
    and rho = 0 tensors of one seed (same factors, same X_clean bytes) carries
    rounding of ~eps/rho relative, hence the tolerance max(1e-12, 50 eps/rho)."""
    seed = 777 + rank
    ctx.synth_tensor(kind, list(dims), rank, 0.0, seed)
    clean = ctx.get_tensor(list(dims))
    ctx.synth_tensor(kind, list(dims), rank, rho, seed)
    noisy = ctx.get_tensor(list(dims))
    n0, n1 = ctx.synth_norms()
    assert n1 > 0
    e = noisy - clean
    got = np.linalg.norm(e) / np.linalg.norm(clean)
    tol = max(1e-12, 50 * np.finfo(float).eps / rho)
    assert abs(got - rho) <= tol * rho, (got, rho)
    # and the exported norms are what was used
    assert abs(np.sqrt(n0) - np.linalg.norm(clean)) <= 1e-13 * np.sqrt(n0)
    # E is Gaussian noise: mean ~ 0, no correlation with X_clean
    z = e.ravel() / np.std(e)
    assert abs(z.mean()) <= 6 / np.sqrt(z.size)
    c = np.dot(z, clean.ravel()) / (np.linalg.norm(z) * np.linalg.norm(clean))
    assert abs(c) <= 6 / np.sqrt(z.size)


def test_generator_factor_distributions(ctx):
    """kind 0 (C1/C2/C3/C5): i.i.d. N(0,1) entries.  kind 1 (C4): per mode
    column j = s_j (sqrt(.9) g + sqrt(.1) h_j): unit-scaled columns have
    pairwise cosine ~0.9 and the scales s_j = 10^(-3U) lie in [1e-3, 1]."""
    f0 = ctx.synth_truth(0, [256, 256, 256, 256], 64, 20250005)
    v = np.concatenate([f.ravel() for f in f0])
    n = v.size
    assert abs(v.mean()) <= 6 / np.sqrt(n)
    assert abs(v.var() - 1.0) <= 6 * np.sqrt(2.0 / n)
    kurt = np.mean(v ** 4) / v.var() ** 2
    assert abs(kurt - 3.0) <= 0.1
    # different modes / columns are independent streams
    assert abs(np.corrcoef(f0[0][:, 0], f0[1][:, 0])[0, 1]) <= 0.3
    f1 = ctx.synth_truth(1, [4096, 4096, 4096], 20, 20250004)
    for f in f1:
        g = f / np.linalg.norm(f, axis=0)
        cos = g.T @ g
        off = cos[~np.eye(20, dtype=bool)]
        assert abs(off.mean() - 0.9) <= 0.02, off.mean()
        s = np.linalg.norm(f, axis=0) / np.sqrt(f.shape[0])  # ~ s_j (E|col|^2 = s_j^2 I)
        assert s.min() >= 1e-3 * 0.9 and s.max() <= 1.0 * 1.1
        assert np.log10(s).max() - np.log10(s).min() >= 1.0  # log-uniform spread over 3 decades


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


@pytest.mark.parametrize("dims,world", [((16, 12, 10), 2), ((12, 7, 6, 5), 4), ((8, 40, 33), 4),
                                        ((64, 32, 32), 8), ((9, 9, 7), 3)])
def test_sharded_cpdt_load_slabs(port, tmp_path, dims, world):
    """io.hpp:93-121: a file the reference's codec wrote; every rank of a
    world-`world` group loads its mode-0 slab bit for bit, and the slabs tile
    the reference reader's tensor.  (Slabs are equal: a leading extent that
    does not divide by the world size is rejected, see below.)"""
    from oracle.pyoracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    ref = Oracle("reference")
    x = port.rng_normals(4711 + world, int(np.prod(dims))).reshape(dims)
    p = str(tmp_path / "x.cpdt")
    ref.write_tensor_file(p, x)
    rc, back = ref.read_tensor_file(p)
    assert rc == 0 and np.array_equal(back, x)
    group = cpd.Context.local_group(0, world)

    def rank_run(r, c):
        c.load_tensor(p)
        b, n = cpd.shard_rows(dims[0], r, world)
        return b, n, c.get_tensor([n] + list(dims[1:]))

    slabs = run_ranks(group, rank_run)
    nxt = 0
    for r, (b, n, got) in enumerate(slabs):
        assert b == nxt
        assert np.array_equal(got, back[b:b + n]), r
        nxt = b + n
    assert nxt == dims[0]
    # the sharded context also rejects what decode_tensor rejects
    bad = str(tmp_path / "trunc.cpdt")
    with open(p, "rb") as f:
        raw = f.read()
    with open(bad, "wb") as f:
        f.write(raw[:-8])

    def rank_bad(r, c):
        with pytest.raises(cpd.FormatError):
            c.load_tensor(bad)
        return True

    assert all(run_ranks(group, rank_bad))
    for c in group:
        c.close()


def test_sharded_load_rejects_ragged_leading_extent(port, tmp_path):
    """Equal mode-0 slabs are the sharding contract (cpdb_shard_rows): a
    leading extent that does not divide by the world size is an
    invalid_argument on every rank, before any device allocation."""
    from oracle.pyoracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    x = port.rng_normals(4712, 13 * 7 * 6).reshape(13, 7, 6)
    p = str(tmp_path / "r.cpdt")
    Oracle("reference").write_tensor_file(p, x)
    with pytest.raises(ValueError):
        cpd.shard_rows(13, 1, 4)
    group = cpd.Context.local_group(0, 4)

    def rank_run(r, c):
        with pytest.raises(ValueError):
            c.load_tensor(p)
        return True

    assert all(run_ranks(group, rank_run))
    for c in group:
        c.close()


def test_async_upload_matches_synchronous(port):
    """cpdb_tensor_set_async queues the upload of X on the context's stream;
    every later call is ordered behind it and the solver's host-side set-up
    (the reference's Rng draw of the initial factors) runs under it.  Same
    bits as the synchronous upload, from pinned and from pageable memory."""
    import ctypes
    import numpy as np
    import paper_2503_18759_b200 as cpd
    dims, rank = (96, 80, 72), 8
    x = port.synth_baseline(0, dims, rank, 1e-2, 20250021)
    cfg = cpd.SolverConfig(rank=rank, max_iterations=6, seed=7)
    ctx = cpd.Context(0)
    ctx.set_tensor(x)
    ref = ctx.solve(cfg, extrapolate=True)
    # page-locked host memory straight from the CUDA runtime (no torch here:
    # importing it after libnccl.so.2 has been loaded by the NCCL tests of
    # this process would clash with its bundled NCCL)
    srcs = [x]
    try:
        rt = ctypes.CDLL("libcudart.so.12")
        ptr = ctypes.c_void_p()
        if rt.cudaMallocHost(ctypes.byref(ptr), ctypes.c_size_t(x.nbytes)) == 0:
            pinned = np.ctypeslib.as_array((ctypes.c_double * x.size).from_address(ptr.value))
            pinned = pinned.reshape(dims)
            pinned[:] = x
            srcs.insert(0, pinned)
    except OSError:
        pass
    for src in srcs:
        ctx.set_tensor(src, wait=False)
        assert ctx.norm_sq() == float(ref_norm(ctx, x))
        ctx.set_tensor(src, wait=False)
        got = ctx.solve(cfg, extrapolate=True)
        assert [(t.fitness, t.flops) for t in got.trace] == [(t.fitness, t.flops) for t in ref.trace]
        for a, b in zip(got.model.factors, ref.model.factors):
            assert np.array_equal(a, b)


def ref_norm(ctx, x):
    import paper_2503_18759_b200 as cpd
    c2 = cpd.Context(0)
    c2.set_tensor(x)
    return c2.norm_sq()
