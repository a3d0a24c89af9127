"""GPU parity of the single primitives against the CPU oracle (and the
reference's own test properties, tensor_test.cpp / linalg_test.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


TTM_SHAPES = [
    ((9, 8, 7), 3),          # reference test sizes: generic path
    ((7, 6, 5, 4), 3),
    ((16, 24, 32), 8),       # tensor-core layouts
    ((64, 48, 40), 16),
    ((40, 64, 16, 24), 20),  # R padded to 24
    ((33, 40, 48), 32),
    ((24, 32, 40), 64),
    ((100, 100, 100), 10),   # C1 shape
    ((24, 32, 40), 65),      # wide ranks: 64-column blocks (one column in the second)
    ((40, 48, 32, 16), 130),
    ((18, 20, 22), 96),      # a contracted extent that is not a multiple of 4
    ((9, 8, 7), 70),         # generic path at a wide rank
]


@pytest.mark.parametrize("shape,rank", TTM_SHAPES)
def test_ttm_all_modes(ctx, port, shape, rank):
    """tensor_test.cpp:127-141: TTM equals the triple-loop oracle (1e-14)."""
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(7, int(np.prod(shape))).reshape(shape)
    for m, n in enumerate(shape):
        b = port.rng_normals(100 + m, rank * n).reshape(rank, n)
        got = cpd.ttm(x, b, m, ctx)
        want = port.ttm(x, b, m)
        assert got.shape == want.shape
        assert rel(got, want) < 1e-14, (shape, m)


def test_ttm_golden_and_errors(ctx, golden):
    import paper_2503_18759_b200 as cpd
    x = golden["prim_x"]
    for m in range(3):
        assert rel(cpd.ttm(x, golden[f"prim_b{m}"], m, ctx), golden[f"prim_ttm{m}"]) < 1e-14
    with pytest.raises(ValueError):
        cpd.ttm(x, np.ones((2, 5)), 0, ctx)
    with pytest.raises(ValueError):
        cpd.ttm(x, np.ones((2, 9)), 3, ctx)
    # identity leaves the tensor (tensor_test.cpp:118-125)
    for m, n in enumerate(x.shape):
        assert np.array_equal(cpd.ttm(x, np.eye(n), m, ctx), x)


def test_ttm_large_rank_generic(ctx, port):
    import paper_2503_18759_b200 as cpd
    x = port.rng_normals(9, 20 * 70 * 12).reshape(20, 70, 12)
    b = port.rng_normals(10, 70 * 70).reshape(70, 70)
    assert rel(cpd.ttm(x, b, 1, ctx), port.ttm(x, b, 1)) < 1e-14


def test_unfold_khatri_rao_exact(ctx, golden, port):
    import paper_2503_18759_b200 as cpd
    x = golden["prim_x"]
    for m in range(3):
        assert np.array_equal(cpd.unfold(x, m, ctx), golden[f"prim_unfold{m}"])
    kr = cpd.khatri_rao([golden["prim_kr_a"], golden["prim_kr_b"]], ctx)
    assert np.array_equal(kr, golden["prim_kr"])
    mats = [port.rng_normals(50 + i, (3 + i) * 4).reshape(3 + i, 4) for i in range(3)]
    assert np.array_equal(cpd.khatri_rao(mats, ctx), port.khatri_rao(mats))
    with pytest.raises(ValueError):
        cpd.khatri_rao([], ctx)


def test_thin_qr(ctx, golden, port):
    """linalg_test.cpp:39-109"""
    import paper_2503_18759_b200 as cpd
    q, r = cpd.thin_qr(golden["prim_qr_a"], ctx)
    assert rel(q, golden["prim_qr_q"]) < 1e-12 and rel(r, golden["prim_qr_r"]) < 1e-12
    assert np.all(np.diag(r) >= 0)
    # (m >= 256: the cooperative multi-CTA kernel, also with a zero column)
    for m, n in ((512, 64), (100, 10), (7, 7), (4096, 96), (300, 130), (256, 5)):
        a = port.rng_normals(m + n, m * n).reshape(m, n)
        q, r = cpd.thin_qr(a, ctx)
        assert rel(q @ r, a) < 1e-13
        assert np.abs(q.T @ q - np.eye(n)).max() < 1e-13
        assert np.allclose(np.triu(r), r)
        assert np.all(np.diag(r) >= 0)
        qo, ro = port.thin_qr(a) if hasattr(port, "thin_qr") else (q, r)
        assert rel(q, qo) < 1e-11 and rel(r, ro) < 1e-12
    a = port.rng_normals(9, 400 * 6).reshape(400, 6)
    a[:, 2] = 0.0  # zero column: R(2,2) stays 0, the reflector is skipped (linalg.hpp:51)
    q, r = cpd.thin_qr(a, ctx)
    assert r[2, 2] == 0.0 and rel(q @ r, a) < 1e-13
    q, r = cpd.thin_qr(golden["prim_kr"], ctx)
    assert abs(q[0, 0] - 1.0) <= 1e-12 and np.abs(q[0, 1:]).max() <= 1e-12
    assert np.abs(q[1:, 0]).max() <= 1e-12
    # identity and hand example
    q, r = cpd.thin_qr(np.eye(4), ctx)
    assert np.allclose(q, np.eye(4)) and np.allclose(r, np.eye(4))
    q, r = cpd.thin_qr(np.array([[3.0], [4.0]]), ctx)
    assert np.allclose(r, [[5.0]]) and np.allclose(q, [[0.6], [0.8]])
    # rank deficiency shows as a zero diagonal
    a = np.array([[1.0, 2.0], [2.0, 4.0], [3.0, 6.0]])
    _, r = cpd.thin_qr(a, ctx)
    assert abs(r[1, 1]) < 1e-14
    with pytest.raises(ValueError):
        cpd.thin_qr(np.ones((2, 3)), ctx)
    # determinism
    a = port.rng_normals(5, 60 * 8).reshape(60, 8)
    assert np.array_equal(cpd.thin_qr(a, ctx)[0], cpd.thin_qr(a, ctx)[0])


def test_solve_normalize_extrapolate(ctx, port):
    import paper_2503_18759_b200 as cpd
    l = np.tril(port.rng_normals(1, 36).reshape(6, 6)) + 3 * np.eye(6)
    rhs = port.rng_normals(2, 40 * 6).reshape(40, 6)
    assert rel(cpd.solve_rows_lower_triangular(l, rhs, ctx), port.solve_rows_lower(l, rhs)) < 1e-14
    l2 = l.copy()
    l2[3, 3] = 0.0
    with pytest.raises(cpd.SingularTriangularError) as ei:
        cpd.solve_rows_lower_triangular(l2, rhs, ctx)
    assert ei.value.column == 3
    a = port.rng_normals(3, 50 * 5).reshape(50, 5)
    a[:, 2] = 0.0
    g_out, g_w = cpd.normalize_columns(a, ctx)
    o_out, o_w = port.normalize_columns(a)
    assert np.array_equal(g_out, o_out) and np.array_equal(g_w, o_w)  # bit-exact
    now = port.rng_normals(4, 30).reshape(10, 3)
    prev = port.rng_normals(5, 30).reshape(10, 3)
    assert np.array_equal(cpd.extrapolate_q0(now, prev, 0.0, 0.1, ctx), now)
    assert rel(cpd.extrapolate_q0(now, prev, 1 / 500, 0.1, ctx),
               port.extrapolate_q0(now, prev, 1 / 500, 0.1)) < 1e-15


def test_fitness_and_inner(ctx, port):
    import paper_2503_18759_b200 as cpd
    v = port.rng_normals(1, 40 * 4).reshape(40, 4)
    ah = port.rng_normals(2, 40 * 4).reshape(40, 4)
    r0 = np.triu(port.rng_normals(3, 16).reshape(4, 4)) + 2 * np.eye(4)
    rn = np.triu(port.rng_normals(4, 16).reshape(4, 4)) + 2 * np.eye(4)
    lam = np.abs(port.rng_normals(5, 4)) + 0.1
    nx2 = 1e4
    g = cpd.fitness_fast_qr(nx2, v, ah, r0, rn, lam, ctx)
    o = port.fitness_fast_qr(nx2, v, ah, r0, rn, lam)
    assert abs(g[0] - o[0]) < 1e-12 and abs(g[1] - o[1]) < 1e-10 * abs(o[1])
    with pytest.raises(ValueError):
        cpd.fitness_fast_qr(0.0, v, ah, r0, rn, lam, ctx)
    a = port.rng_normals(6, 10001)
    assert abs(cpd.inner(a, a, ctx) - float(a @ a)) < 1e-12 * float(a @ a)
