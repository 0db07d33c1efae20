"""GPU parity of the building blocks against the oracle / reference golden vectors.

Tolerances (FP64): the DMMA contractions sum in a blocked order instead of the
reference's sequential order, so products agree to a few ulps of the operand
norms: ‖Δ‖ ≤ 1e-13·‖ref‖ (kernels); the 7-point stencil gradient uses
round-to-nearest intrinsics in the oracle's order and must be BITWISE equal.
"""
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("shape", [(37, 5, 4), (1000, 20, 20), (333, 7, 13), (4096, 128, 128),
                                   (2048, 256, 200), (16, 1, 1)])
def test_matmul_at_b(pcal, orc, shape):
    n, pa, pb = shape
    a = orc.random_normal(n, pa, 11)
    b = orc.random_normal(n, pb, 12)
    got = pcal.matmul_at_b(a, b)
    want = orc.matmul_at_b(a, b)
    assert got.shape == want.shape
    assert rel(got, want) <= 1e-13


@pytest.mark.parametrize("shape", [(37, 5), (1000, 20), (1001, 33), (8192, 64), (2048, 256)])
def test_gram_exactly_symmetric(pcal, orc, shape):
    n, p = shape
    x = orc.random_normal(n, p, 21)
    g = pcal.gram(x)
    assert np.array_equal(g, g.T)  # gram mirrors the upper triangle (kernels.cpp:150-151)
    assert rel(g, orc.gram(x)) <= 1e-13


@pytest.mark.parametrize("shape", [(37, 5, 6), (1000, 20, 40), (513, 17, 3), (4096, 128, 256)])
def test_matmul(pcal, orc, shape):
    m, k, nc = shape
    a = orc.random_normal(m, k, 31)
    b = orc.random_normal(k, nc, 32)
    assert rel(pcal.matmul(a, b), orc.matmul(a, b)) <= 1e-13


def test_kernels_vs_reference_golden(pcal, gold):
    assert rel(pcal.matmul_at_b(gold["k_a"], gold["k_b"]), gold["k_matmul_at_b"]) <= 1e-14
    assert rel(pcal.gram(gold["k_a"]), gold["k_gram"]) <= 1e-14
    assert rel(pcal.matmul(gold["k_a"], gold["k_c"]), gold["k_matmul"]) <= 1e-14


def test_orthonormalize(pcal, orc, gold):
    q = pcal.orthonormalize(gold["k_orth_x"])
    assert np.abs(q - gold["k_orth_q"]).max() <= 1e-13
    x = orc.random_normal(5000, 64, 41)
    q = pcal.orthonormalize(x)
    assert np.linalg.norm(q.T @ q - np.eye(64)) <= 1e-12  # acceptance_main.cpp:101
    assert rel(q, orc.orthonormalize(x)) <= 1e-12
    # X = Q·R with R = QᵀX upper triangular (span preserved)
    r = q.T @ x
    assert np.abs(np.tril(r, -1)).max() <= 1e-10 * np.abs(r).max()


@pytest.mark.parametrize("n,p", [(3000, 129), (4000, 300), (6000, 777), (4096, 1024)])
def test_orthonormalize_wide_p(pcal, orc, n, p):
    """CholeskyQR2 for 128 < p ≤ 2048 (k_cholesky_wide + k_trinv_wide: transposed
    factor, warp-per-row dots; warp-per-column inverse) against the oracle's
    orthonormalize (kernels.cpp:250-265) and the acceptance feasibility bar, for
    p off and on the 32-column grid."""
    x = orc.random_normal(n, p, 43)
    q = pcal.orthonormalize(x)
    assert pcal.last_orthonormalize_path() == "cholqr2"  # no MGS2 fallback
    assert np.linalg.norm(q.T @ q - np.eye(p)) <= 1e-12  # acceptance_main.cpp:101
    assert rel(q, orc.orthonormalize(x)) <= 1e-11
    r = q.T @ x
    assert np.abs(np.tril(r, -1)).max() <= 1e-10 * np.abs(r).max()


def test_orthonormalize_rank_deficient(pcal, orc):
    x = orc.random_normal(40, 4, 42)
    x[:, 3] = x[:, 0] + x[:, 1]  # exactly dependent column (test_kernels.cpp:150-181)
    with pytest.raises(pcal.RankError):
        pcal.orthonormalize(x)
    with pytest.raises(np.linalg.LinAlgError):
        orc.orthonormalize(x)


def test_orthonormalize_fixed_point(pcal):
    x = np.zeros((6, 3), order="F")
    x[0, 0] = x[1, 1] = x[2, 2] = 1.0
    assert np.abs(pcal.orthonormalize(x) - x).max() <= 1e-15


def test_pcal_step_known_answers(pcal, orc, gold):
    col = np.array([[3.0], [4.0]])
    out, deg = pcal.pcal_step(col, np.zeros((2, 1)), 5.0)  # (3,4) → (0.6,0.8)
    assert deg == 0 and abs(out[0, 0] - 0.6) < 1e-15 and abs(out[1, 0] - 0.8) < 1e-15
    out, _ = pcal.pcal_step(gold["ps_x"], gold["ps_g"], 2.0)
    assert np.abs(out - gold["ps_out"]).max() <= 1e-15
    assert np.abs(np.linalg.norm(out, axis=0) - 1.0).max() <= 1e-14
    # grad_l = eta·X ⇒ zero update ⇒ every column degenerate, previous column kept
    x = gold["ps_x"]
    out, deg = pcal.pcal_step(x, 2.0 * x, 2.0)
    assert deg == 5
    assert np.abs(out - x / np.linalg.norm(x, axis=0)).max() <= 1e-15
    with pytest.raises(pcal.ParameterError):
        pcal.pcal_step(x, x, 0.0)


def test_pcal_step_divergence(pcal):
    x = np.ones((8, 2), order="F")
    g = np.zeros((8, 2), order="F")
    g[0, 0] = np.inf
    with pytest.raises(pcal.DivergenceError):
        pcal.pcal_step(x, g, 1.0)


def test_spectral_norm(pcal, orc, gold):
    s = pcal.spectral_norm_estimate(gold["k_spec_a"], 11)
    assert abs(s - gold["k_spec_s"]) <= 1e-9 * gold["k_spec_s"]


def test_dense_gradient(pcal, orc):
    n, p = 1000, 20
    m = orc.dense_trace_min(n, p, 5, s=10.0)
    x = orc.initial_point_qr(n, p, 6)
    f_ref, g_ref = orc.evaluate(m, x)
    f, g = pcal.evaluate(pcal.QuadraticModel(m.a, p, m.s), x)
    assert rel(g, g_ref) <= 1e-13
    assert abs(f - f_ref) <= 1e-12 * abs(f_ref)


def test_dense_gradient_with_linear_term(pcal, orc):
    from oracle.oracle import Model, MODEL_DENSE
    n, p = 300, 7
    a = orc.sym_part(orc.random_normal(n, n, 8))
    g0 = orc.random_normal(n, p, 9)
    x = orc.random_normal(n, p, 10)
    f_ref, g_ref = orc.evaluate(Model(MODEL_DENSE, n, p, 1.0, a=a, g0=g0), x)
    f, g = pcal.evaluate(pcal.QuadraticModel(a, p, 1.0, g0=g0), x)
    assert rel(g, g_ref) <= 1e-13
    assert abs(f - f_ref) <= 1e-12 * abs(f_ref)


@pytest.mark.parametrize("grid,p", [((6, 5, 4), 3), ((64, 64, 64), 4), ((16, 16, 16), 33)])
def test_stencil_gradient_bitwise(pcal, orc, grid, p):
    from oracle.oracle import Model, MODEL_STENCIL
    n = grid[0] * grid[1] * grid[2]
    v = orc.random_uniform(n, 3)
    x = orc.random_normal(n, p, 4)
    f_ref, g_ref = orc.evaluate(Model(MODEL_STENCIL, n, p, 13.0, grid=grid, v=v), x)
    f, g = pcal.evaluate(pcal.StencilModel(grid, v, p, 13.0), x)
    assert np.array_equal(g, g_ref)  # same op order, no contraction
    assert abs(f - f_ref) <= 1e-12 * abs(f_ref)


@pytest.mark.parametrize("grid,p", [((6, 6, 6), 4), ((48, 48, 48), 3), ((8, 6, 10), 5),
                                    ((96, 16, 5), 3), ((72, 8, 4), 2)])
def test_kohn_sham_gradient(pcal, orc, grid, p):
    from oracle.oracle import Model, MODEL_KOHN_SHAM
    n = grid[0] * grid[1] * grid[2]
    v = -orc.random_uniform(n, 5)
    x = orc.initial_point_qr(n, p, 6)
    mo = Model(MODEL_KOHN_SHAM, n, p, 12.0, grid=grid, v=v)
    f_ref, g_ref = orc.evaluate(mo, x)
    f, g = pcal.evaluate(pcal.KohnShamModel(grid, v, p, 12.0), x)
    assert rel(g, g_ref) <= 1e-14  # only the device cbrt may differ by an ulp
    assert abs(f - f_ref) <= 1e-12 * abs(f_ref)


@pytest.mark.parametrize("grid,p", [((32, 8, 5), 3), ((48, 16, 7), 2), ((128, 16, 4), 2),
                                    ((64, 64, 64), 2), ((40, 24, 3), 5),
                                    ((96, 16, 5), 3), ((72, 8, 4), 2), ((100, 8, 3), 2)])
def test_stencil_march_bitwise(pcal, orc, grid, p):
    """z-marching kernel (nx ≤ 128, ny % 8 == 0): same bits as the oracle.
    (96,16,5) / (72,8,4) / (100,8,3) take the full-row march with 4 points per
    lane and idle lanes (nx % 4 == 0, 64 < nx < 128: L = nx/4 < 32 — the x wrap
    over the active lanes and the masked stores)."""
    from oracle.oracle import Model, MODEL_STENCIL
    n = grid[0] * grid[1] * grid[2]
    v = orc.random_uniform(n, 13)
    x = orc.random_normal(n, p, 14)
    f_ref, g_ref = orc.evaluate(Model(MODEL_STENCIL, n, p, 13.0, grid=grid, v=v), x)
    f, g = pcal.evaluate(pcal.StencilModel(grid, v, p, 13.0), x)
    assert np.array_equal(g, g_ref)
    assert abs(f - f_ref) <= 1e-12 * abs(f_ref)


@pytest.mark.parametrize("kind,grid,p", [("stencil", (64, 16, 6), 3), ("stencil", (128, 8, 5), 2),
                                         ("stencil", (32, 16, 3), 4), ("kohn_sham", (48, 8, 6), 3),
                                         ("kohn_sham", (96, 16, 4), 2)])
def test_tma_stencil_is_bitwise_the_register_march(pcal, orc, kind, grid, p, monkeypatch):
    """The TMA-staged stencil (k_stencil_tma, rows of a multiple of 16 points)
    against the register-pipelined full-row march: same G bits, same f to
    rounding; and both against the oracle's G."""
    from oracle.oracle import Model, MODEL_STENCIL, MODEL_KOHN_SHAM
    n = grid[0] * grid[1] * grid[2]
    v = orc.random_uniform(n, 21) if kind == "stencil" else -orc.random_uniform(n, 21)
    x = orc.random_normal(n, p, 22)
    cls = pcal.StencilModel if kind == "stencil" else pcal.KohnShamModel
    f1, g1 = pcal.evaluate(cls(grid, v, p, 13.0), x)
    monkeypatch.setenv("PCAL_NO_TMA_STENCIL", "1")
    f2, g2 = pcal.evaluate(cls(grid, v, p, 13.0), x)
    assert np.array_equal(g1, g2)
    assert abs(f1 - f2) <= 1e-13 * abs(f2)
    mk = MODEL_STENCIL if kind == "stencil" else MODEL_KOHN_SHAM
    f_ref, g_ref = orc.evaluate(Model(mk, n, p, 13.0, grid=grid, v=v), x)
    if kind == "stencil":
        assert np.array_equal(g1, g_ref)
    else:
        assert rel(g1, g_ref) <= 1e-14


def test_tma_stencil_slot_release_under_load(pcal, monkeypatch):
    """Regression: the TMA stencil released its first ring slot (plane z0 − 1)
    right after issuing the shared-memory loads, and under full load the next
    TMA fill of that slot overtook them — a few rows of plane z0 took plane
    z0 + 3's values (seen at config 5, p = 1024, a few rows per evaluation).
    Slots are now released after the plane's arithmetic has consumed them.
    A 128 × 128 × 16 grid with p = 512 (8192 blocks, the same XP = 4 kernel)
    evaluated repeatedly must give the register march's G every time."""
    grid, p = (128, 128, 16), 512
    n = grid[0] * grid[1] * grid[2]
    rng = np.random.default_rng(5)
    v = rng.uniform(size=n)
    x = np.asfortranarray(rng.standard_normal((n, p)))
    m = pcal.StencilModel(grid, v, p, 13.0)
    monkeypatch.setenv("PCAL_NO_TMA_STENCIL", "1")
    f_ref, g_ref = pcal.evaluate(m, x)
    monkeypatch.delenv("PCAL_NO_TMA_STENCIL")
    for _ in range(8):  # the old release failed 2 of 3 runs of 4 evaluations
        f, g = pcal.evaluate(m, x)
        assert np.array_equal(g, g_ref)


@pytest.mark.parametrize("case", ["stencil", "dense", "sharded", "gram"])
def test_triangular_diagonal_tiles_are_bitwise(pcal, orc, case, monkeypatch):
    """The Gram's diagonal tiles compute only their upper-triangle sub-blocks
    (mma_stage_tri, 17 instead of 32 DMMAs per warp and k-step) with the same
    k order as the full tile.  Every used value of a tile owned by one CTA is
    bitwise the full tile's; stream-K re-balances its CTA ranges by tile cost,
    which moves the K boundaries of split tiles, so single-GPU Grams agree to
    rounding.  The sharded path keeps its fixed K segments: bitwise there."""
    from paper_1810_03930_b200 import report_io
    if case == "gram":
        x = orc.random_normal(5000, 300, 31)
        g1 = pcal.gram(x)
        monkeypatch.setenv("PCAL_NO_TRI_TILES", "1")
        g2 = pcal.gram(x)
        assert np.abs(g1 - g2).max() <= 1e-12 * np.abs(g2).max()
        assert np.array_equal(g1, g1.T)
        return
    if case == "dense":
        n, p = 2000, 256
        m = pcal.QuadraticModel(pcal.gen_dense_operator(n, 5), p, 90.0)
    else:
        grid, p = (16, 16, 12), 256
        n = 16 * 16 * 12
        m = pcal.StencilModel(grid, orc.random_uniform(n, 6), p, 13.0)
    x0 = orc.initial_point_qr(n, p, 7)
    cfg = pcal.SolverConfig(tol_rel_kkt=1e-300, max_iter=12)
    run = (lambda: pcal.solve_emulated(m, cfg, x0, 2)) if case == "sharded" else \
        (lambda: pcal.solve(m, cfg, x0))
    r1 = run()
    monkeypatch.setenv("PCAL_NO_TRI_TILES", "1")
    r2 = run()
    if case == "sharded":
        assert report_io.same_numerics(r1, r2)
    else:
        w = r1.trace.shape[0]
        assert w == r2.trace.shape[0]
        for col in (1, 2, 5):
            assert np.all(np.abs(r1.trace[:, col] - r2.trace[:, col]) <=
                          1e-10 * np.abs(r2.trace[:, col])), col


@pytest.mark.parametrize("name,mode", [("qr", "qr"), ("a2i", "a2-i"), ("a2ii", "a2-ii"),
                                       ("a2ii_p1", "a2-ii")])
def test_initial_point_modes_match_reference(pcal, name, mode):
    """initial_point(InitialPointSpec) for Qr / A2TypeI / A2TypeII against the
    reference's own output (tests/golden/reference_init.npz): the column scale
    factors come from the same random stream, the Q factor agrees to rounding."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_init.npz"))
    ref = g[name]
    m, sigma, n, p, seed = g[name + "_args"]
    x = pcal.initial_point(int(n), int(p), int(seed), mode=mode, sigma_lower=float(sigma))
    assert x.shape == ref.shape
    assert np.abs(x - ref).max() <= 1e-12
    assert np.allclose(np.linalg.norm(x, axis=0), np.linalg.norm(ref, axis=0), rtol=1e-14, atol=0)
