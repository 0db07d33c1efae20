"""CPU: the C restatement (oracle/pcal_oracle.c) pinned BITWISE to golden vectors
produced by the unmodified reference (oracle/make_golden.py → tests/golden/),
plus the operator definitions of configs 3–5 (no reference implementation)
checked by finite differences and by dense cross-checks on tiny grids."""
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle import Config, Model, MODEL_DENSE, MODEL_KOHN_SHAM, MODEL_STENCIL

HERE = os.path.dirname(__file__)
GOLD = os.path.join(HERE, "golden", "reference_small.npz")
GRID = os.path.join(HERE, "golden", "reference_grid.npz")
CFG2 = os.path.join(HERE, "golden", "reference_cfg2.npz")
TINY = np.finfo(float).tiny
INIT_SALT = 0x1235713


def sha(a):
    return hashlib.sha256(np.asfortranarray(a, dtype="<f8").tobytes(order="F")).hexdigest()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_rng_stream(orc, gold):
    assert np.array_equal(orc.random_normal(1001, 1, 1)[:, 0], gold["normal_seed1"])
    assert np.array_equal(orc.random_normal(1001, 1, 1, threads=4)[:, 0], gold["normal_seed1"])
    assert np.array_equal(orc.random_normal(21, 1, 1 ^ INIT_SALT)[:, 0], gold["normal_seed_init1"])
    big1 = orc.random_normal(300001, 1, 9, threads=1)
    big4 = orc.random_normal(300001, 1, 9, threads=4)  # checkpointed states are bitwise neutral
    assert np.array_equal(big1, big4)


def test_kernels_bitwise(orc, gold):
    assert np.array_equal(orc.matmul_at_b(gold["k_a"], gold["k_b"]), gold["k_matmul_at_b"])
    assert np.array_equal(orc.gram(gold["k_a"]), gold["k_gram"])
    assert np.array_equal(orc.matmul(gold["k_a"], gold["k_c"]), gold["k_matmul"])
    assert np.array_equal(orc.orthonormalize(gold["k_orth_x"]), gold["k_orth_q"])
    assert orc.spectral_norm_estimate(gold["k_spec_a"], 11) == gold["k_spec_s"]
    out, deg = orc.pcal_step(gold["ps_x"], gold["ps_g"], 2.0)
    assert np.array_equal(out, gold["ps_out"]) and deg == 0


def test_stepsize_closed_forms(orc, gold):
    x = np.array([[1.0], [1.0]]); xp = np.zeros((2, 1))
    g = np.array([[1.0], [3.0]]); gp = np.zeros((2, 1))
    got = [orc.stepsize_select(Config(eta_kind=k), it, 0.5, 0.25, x, xp, g, gp)
           for k, it in [(2, 1), (3, 1), (4, 1), (4, 2), (1, 2)]]
    assert np.array_equal(got, gold["ss_etas"])
    assert got[:4] == [2.0, 2.5, 2.0, 2.5]  # test_solver.cpp:167-190
    # fallbacks (test_solver.cpp:191-224)
    g2 = np.array([[1.0], [-1.0]])
    assert orc.stepsize_select(Config(eta_kind=2), 1, 0.5, 0.25, x, xp, g2, gp) == 0.5
    assert orc.stepsize_select(Config(eta_kind=4), 0, 0.0, 0.125, x, None, g, None) == 0.125
    assert orc.stepsize_select(Config(eta_kind=0, gamma=1e12), 3, 0.5, 0.25, x, xp, g, gp) == 1e10


def test_cfg1_full_run_bitwise(orc, gold):
    m = orc.dense_trace_min(1000, 20, 1, s=float(gold["cfg1_s"]), threads=8)
    assert sha(m.a) == str(gold["cfg1_a_sha"])
    x0 = orc.initial_point_qr(1000, 20, 1 ^ INIT_SALT)
    assert sha(x0) == str(gold["cfg1_x0_sha"])
    r = orc.solve(m, Config(tol_rel_kkt=TINY, max_iter=200, threads=8), x0)
    assert np.array_equal(r.trace[:, :6], gold["cfg1_trace"])
    assert np.array_equal(r.final_pre, gold["cfg1_final_pre"])
    assert np.array_equal(r.final_post, gold["cfg1_final_post"])
    assert sha(r.final_x) == str(gold["cfg1_final_x_sha"])
    assert sha(r.stop_x) == str(gold["cfg1_stop_x_sha"])
    # SURVEY.md §8(c) known answer
    assert r.final_pre[0] == -418.65544567286281 and r.final_post[3] == 2.0011764530960394e-15


def test_cfg1_spectral_scale(orc, gold):
    m = orc.dense_trace_min(1000, 20, 1, threads=4)  # s from Rng(seed ^ 0x73706563)
    assert m.s == float(gold["cfg1_s"])


@pytest.mark.parametrize("name,n,p", [("c40", 40, 5), ("c12", 12, 2), ("c20", 20, 4),
                                      ("c14plam", 14, 3), ("c200", 200, 10)])
def test_small_cases_bitwise(orc, gold, name, n, p):
    r = orc.random_normal(n, n, int(gold[name + "_a_seed"]))
    a = np.asfortranarray(0.5 * (r + r.T))
    s = orc.spectral_norm_estimate(a, 0x73706563)
    assert s == float(gold[name + "_s"])
    x0 = orc.initial_point_qr(n, p, int(gold[name + "_x0_seed"]))
    kw = {"c20": dict(max_iter=40, final_orth=False), "c14plam": dict(multiplier_rule=0)}.get(name, {})
    rep = orc.solve(Model(MODEL_DENSE, n, p, s, a=a), Config(**kw), x0)
    assert np.array_equal(rep.trace[:, :6], gold[name + "_trace"])
    assert rep.status == str(gold[name + "_status"])
    assert np.array_equal(rep.final_x, gold[name + "_final_x"])


def test_stationary_start(orc, gold):
    a = np.asfortranarray(np.diag([1.0, 2.0, 3.0, 4.0]))
    x = np.zeros((4, 2), order="F"); x[0, 0] = x[1, 1] = 1.0
    r = orc.solve(Model(MODEL_DENSE, 4, 2, 4.0, a=a), Config(), x)
    assert r.status == "converged" and r.iterations == 0 and r.trace.shape[0] == 1
    assert np.array_equal(r.trace[:, :6], gold["stat_trace"])


@pytest.mark.parametrize("name,grid,kind", [("st6", (6, 5, 4), MODEL_STENCIL),
                                            ("ks6", (6, 6, 6), MODEL_KOHN_SHAM)])
def test_grid_models_loop_bitwise(orc, name, grid, kind):
    """The restated PCAL loop around the grid operators equals the reference
    solve() driving the same operators, bit for bit."""
    g = np.load(GRID)
    n = grid[0] * grid[1] * grid[2]
    x0 = orc.initial_point_qr(n, 4, 3 ^ INIT_SALT)
    m = Model(kind, n, 4, float(g[name + "_s"]), grid=grid, v=g[name + "_v"])
    r = orc.solve(m, Config(tol_rel_kkt=TINY, max_iter=60), x0)
    assert np.array_equal(r.trace[:, :6], g[name + "_trace"])
    assert np.array_equal(r.final_x, g[name + "_final_x"])


# ---------------------------------------------------------------------------
# operators of configs 3–5: unpinned by the reference
# ---------------------------------------------------------------------------
def dense_laplacian(grid):
    nx, ny, nz = grid
    n = nx * ny * nz
    L = np.zeros((n, n))
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                i = x + nx * (y + ny * z)
                L[i, i] += 6.0
                for j in [((x - 1) % nx) + nx * (y + ny * z), ((x + 1) % nx) + nx * (y + ny * z),
                          x + nx * (((y - 1) % ny) + ny * z), x + nx * (((y + 1) % ny) + ny * z),
                          x + nx * (y + ny * ((z - 1) % nz)), x + nx * (y + ny * ((z + 1) % nz))]:
                    L[i, j] -= 1.0
    return L


@pytest.mark.parametrize("grid", [(4, 4, 4), (5, 3, 6), (6, 6, 6)])
def test_stencil_matches_dense_operator(orc, grid):
    n = grid[0] * grid[1] * grid[2]
    L = dense_laplacian(grid)
    assert np.allclose(L, L.T) and np.linalg.eigvalsh(L)[0] > -1e-12  # L = −Δ_h is PSD
    x = orc.random_normal(n, 3, 1)
    assert np.abs(orc.laplacian(x, grid) - L @ x).max() <= 1e-13
    v = orc.random_uniform(n, 2)
    f, g = orc.evaluate(Model(MODEL_STENCIL, n, 3, 1.0, grid=grid, v=v), x)
    gd = L @ x + v[:, None] * x
    assert np.abs(g - gd).max() <= 1e-13
    assert abs(f - 0.5 * np.sum(x * gd)) <= 1e-12 * abs(f)


@pytest.mark.parametrize("grid", [(4, 4, 4), (6, 5, 4), (3, 4, 5)])
def test_pinv_laplacian_matches_dense_pseudoinverse(orc, grid):
    n = grid[0] * grid[1] * grid[2]
    L = dense_laplacian(grid)
    rho = orc.random_uniform(n, 4)
    m = Model(MODEL_KOHN_SHAM, n, 2, 1.0, grid=grid, v=np.zeros(n))
    got = orc.pinv_laplacian(m, rho)
    want = np.linalg.pinv(L) @ rho
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 48])
def test_fourier_basis_orthonormal_eigenbasis(orc, N):
    q, lam = orc.fourier_basis(N)
    assert np.abs(q.T @ q - np.eye(N)).max() <= 1e-13
    L1 = 2.0 * np.eye(N) - np.roll(np.eye(N), 1, axis=0) - np.roll(np.eye(N), -1, axis=0)
    if N == 1:
        L1 = np.zeros((1, 1))
    elif N == 2:
        L1 = np.array([[2.0, -2.0], [-2.0, 2.0]])
    assert np.abs(L1 @ q - q * lam).max() <= 1e-12


def ks_energy_dense(x, L, v):
    c = (3.0 / np.pi) ** (1.0 / 3.0)
    rho = np.sum(x * x, axis=1)
    h = np.linalg.pinv(L) @ rho
    e = 0.25 * np.sum(x * (L @ x)) + 0.5 * np.sum(v * rho) + 0.25 * rho @ h \
        - 0.375 * c * np.sum(rho ** (4.0 / 3.0))
    g = 0.5 * (L @ x) + (v + h - c * np.cbrt(rho))[:, None] * x
    return e, g


@pytest.mark.parametrize("grid", [(4, 4, 4), (6, 5, 4)])
def test_kohn_sham_matches_dense_restatement(orc, grid):
    n = grid[0] * grid[1] * grid[2]
    L = dense_laplacian(grid)
    v = -orc.random_uniform(n, 5)
    x = orc.initial_point_qr(n, 3, 7)
    f, g = orc.evaluate(Model(MODEL_KOHN_SHAM, n, 3, 1.0, grid=grid, v=v), x)
    fd, gd = ks_energy_dense(x, L, v)
    assert abs(f - fd) <= 1e-12 * abs(fd)
    assert np.abs(g - gd).max() <= 1e-12


@pytest.mark.parametrize("kind,h,tol", [(MODEL_STENCIL, 1e-3, 1e-9), (MODEL_KOHN_SHAM, 1e-5, 1e-6)])
def test_fd_gradient_check(orc, kind, h, tol):
    """acceptance_main.cpp:115-149 tolerances: quadratics 1e-9, density families 1e-6."""
    grid = (6, 5, 4)
    n = 120
    v = orc.random_uniform(n, 3) if kind == MODEL_STENCIL else -orc.random_uniform(n, 3)
    m = Model(kind, n, 6, 1.0, grid=grid, v=v)
    worst = 0.0
    for s in range(5):
        x = orc.random_normal(n, 6, 300 + s)
        worst = max(worst, orc.fd_gradient_check(m, x, h))
    assert worst <= tol


def test_fd_gradient_check_flags_a_wrong_gradient(orc):
    """test_problems.cpp:187-194: a perturbed gradient must be detected."""
    grid = (4, 4, 4)
    n = 64
    m = Model(MODEL_STENCIL, n, 2, 1.0, grid=grid, v=orc.random_uniform(n, 3))
    x = orc.random_normal(n, 2, 1)
    f, g = orc.evaluate(m, x)
    # central difference of the true f at a coordinate vs the perturbed gradient
    i, j, hh = 5, 1, 1e-4 * (1 + abs(x[5, 1]))
    xp, xm = x.copy(order="F"), x.copy(order="F")
    xp[i, j] += hh; xm[i, j] -= hh
    fd = (orc.evaluate(m, xp)[0] - orc.evaluate(m, xm)[0]) / (2 * hh)
    bad = g[i, j] + 1e-3 * (1 + abs(g[i, j]))  # PerturbedModel-style offset
    assert abs(fd - g[i, j]) / (1 + abs(g[i, j])) <= 1e-9
    assert abs(fd - bad) / (1 + abs(g[i, j])) >= 5e-4


@pytest.mark.skipif(not os.path.exists(CFG2) or not os.environ.get("PCAL_SLOW"),
                    reason="config-2 fixture check is slow (set PCAL_SLOW=1)")
def test_cfg2_instance(orc):
    g = np.load(CFG2)
    m = orc.dense_trace_min(16384, 128, 1, s=float(g["cfg2_s"]), threads=8)
    assert sha(m.a) == str(g["cfg2_a_sha"])
    x0 = orc.initial_point_qr(16384, 128, 1 ^ INIT_SALT)
    assert sha(x0) == str(g["cfg2_x0_sha"])


ALGS = {"plam": (0, 1), "plamda": (4, 1), "pcalda": (5, 1), "moptqr": (3, 1), "pcalplamf": (1, 0)}


@pytest.mark.parametrize("name", list(ALGS))
def test_algorithm_variants_bitwise(orc, name):
    """PLAM / PLAM-DA / PCAL-DA / MOptQR / PCAL-PlamFormula (solver.cpp:320-474)."""
    g = np.load(os.path.join(HERE, "golden", "reference_algorithms.npz"))
    alg, mult = ALGS[name]
    m1 = orc.dense_trace_min(1000, 20, 1, s=44.26282919872377, threads=8)
    x01 = orc.initial_point_qr(1000, 20, 1 ^ INIT_SALT)
    r = orc.solve(m1, Config(tol_rel_kkt=TINY, max_iter=60, threads=8, algorithm=alg,
                             multiplier_rule=mult), x01)
    assert np.array_equal(r.trace[:, :6], g[f"a1_{name}_trace"])
    assert sha(r.final_x) == str(g[f"a1_{name}_final_x_sha"])
    rr = orc.random_normal(40, 40, 24)
    a40 = np.asfortranarray(0.5 * (rr + rr.T))
    m40 = Model(MODEL_DENSE, 40, 5, orc.spectral_norm_estimate(a40, 0x73706563), a=a40)
    r = orc.solve(m40, Config(algorithm=alg, multiplier_rule=mult), orc.initial_point_qr(40, 5, 25))
    assert np.array_equal(r.trace[:, :6], g[f"a40_{name}_trace"])
    assert r.status == str(g[f"a40_{name}_status"]) and r.beta == float(g[f"a40_{name}_beta"])
