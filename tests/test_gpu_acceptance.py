"""GPU: the reference's end-to-end acceptance checks (acceptance_main.cpp)
restated for the device models — #1 Rayleigh–Ritz against an eigensolver
oracle, #2 post-orthonormalisation feasibility across the model zoo and both
multiplier formulas, #4 penalty insensitivity of the normalised solver."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SPEC_SALT = 0x73706563


def _dense(pcal, orc, n, p, seed_a):
    a = pcal.gen_dense_operator(n, seed_a)
    return pcal.QuadraticModel(a, p, orc.spectral_norm_estimate(a, seed_a ^ SPEC_SALT)), a


@pytest.mark.parametrize("n,p", [(200, 10), (2000, 40)])
def test_rayleigh_ritz_against_eigensolver(pcal, orc, n, p):
    """Acceptance #1 (acceptance_main.cpp:50-73): ½·(sum of the p smallest
    eigenvalues) to 1e-6, converged, post-orth feasibility ≤ 1e-12."""
    m, a = _dense(pcal, orc, n, p, 101)
    x0 = pcal.initial_point(n, p, 102)
    rep = pcal.solve(m, pcal.SolverConfig(), x0)
    expected = 0.5 * np.sort(np.linalg.eigvalsh(a))[:p].sum()
    assert rep.status == "converged"
    assert abs(rep.final_post_orth.fval - expected) <= 1e-6
    assert rep.final_post_orth.feas <= 1e-12


def _zoo(pcal, orc, kind, seed):
    if kind == "dense":
        return _dense(pcal, orc, 500, 10, seed)[0]
    # p = 5: the periodic Laplacian's lowest cluster (1 + 4 modes on a 16×16 plane)
    # ends at a spectral gap, so the invariant subspace is well defined
    grid = (16, 16, 8)
    n = 16 * 16 * 8
    v = orc.random_uniform(n, seed)
    if kind == "stencil":
        return pcal.StencilModel(grid, v, 5, 12.0 + v.max())
    return pcal.KohnShamModel(grid, -v, 5, 6.0 + v.max())


@pytest.mark.parametrize("kind", ["dense", "stencil", "kohn-sham"])
@pytest.mark.parametrize("alg", ["plam", "pcal"])
def test_post_orth_feasibility_across_models(pcal, orc, kind, alg):
    """Acceptance #2 (acceptance_main.cpp:77-111): every converged run ends with
    post-orth feasibility ≤ 1e-12; at least one run converges."""
    converged = 0
    for seed in range(1, 6):
        m = _zoo(pcal, orc, kind, seed)
        x0 = pcal.initial_point(m.n, m.p, seed)
        rep = pcal.solve(m, pcal.SolverConfig(algorithm=alg, max_iter=3000), x0)
        if rep.status != "converged":
            continue
        converged += 1
        assert rep.final_post_orth is not None and rep.final_post_orth.feas <= 1e-12
    assert converged >= 1


def test_penalty_insensitivity(pcal, orc):
    """Acceptance #4 (acceptance_main.cpp:153-178): the normalised solver
    converges for β ∈ {0, 0.01s, 0.1s, s + 0.1, 10s + 1}."""
    m, _ = _dense(pcal, orc, 500, 10, 41)
    s = m.s
    x0 = pcal.initial_point(500, 10, 41)
    for beta in (0.0, 0.01 * s, 0.1 * s, s + 0.1, 10.0 * s + 1.0):
        rep = pcal.solve(m, pcal.SolverConfig(beta=beta), x0)
        assert rep.status == "converged", beta
