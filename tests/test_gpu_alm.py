"""GPU: ALM (alm_outer, solver.cpp:478-624) — the outer multiplier loop around
inner gradient steps — against the reference's own solve() (golden traces and
counters from oracle/_ref, oracle/make_golden.py ALM_CASES) and the reference's
ALM unit tests (test_solver.cpp:318-331, 463-498)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TINY = np.finfo(float).tiny
INIT_SALT = 0x1235713
GOLD = os.path.join(os.path.dirname(__file__), "golden")

# oracle/make_golden.py ALM_CASES: instance, AlmOptions, config overrides
CASES = {
    "a40_default": ("a40", (500, 50, 0.1), {}),
    "a40_tight_caps": ("a40", (6, 5, 0.1), {}),
    "a40_budget": ("a40", (500, 50, 0.01), {"max_iter": 25}),
    "a40_beta0": ("a40", (500, 50, 0.1), {"beta": 0.0, "max_iter": 300}),
    "c1_caps": ("c1", (7, 50, 0.1), {"max_iter": 60}),
}


def close(a, b, tol, floor=0.0):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= tol * np.abs(b) + floor)


def _instance(pcal, orc, which):
    if which == "a40":
        r = orc.random_normal(40, 40, 24)
        a = np.asfortranarray(0.5 * (r + r.T))
        return pcal.QuadraticModel(a, 5, orc.spectral_norm_estimate(a, 0x73706563)), \
            orc.initial_point_qr(40, 5, 25)
    a = pcal.gen_dense_operator(1000, 1)
    return pcal.QuadraticModel(a, 20, 44.26282919872377), orc.initial_point_qr(1000, 20, 1 ^ INIT_SALT)


@pytest.mark.parametrize("name", list(CASES))
def test_alm_matches_reference(pcal, orc, name):
    """Status, iteration count, outer / cap counters, the trace window and the
    final metrics (pre-orth: the inner loop's best iterate with the last
    recorded kkt_rel, as the reference reports them)."""
    g = np.load(os.path.join(GOLD, "reference_alm.npz"))
    which, (imax, omax, scale), over = CASES[name]
    model, x0 = _instance(pcal, orc, which)
    cfg = pcal.SolverConfig(algorithm="alm", alm=pcal.AlmOptions(imax, omax, scale), **over)
    rep = pcal.solve(model, cfg, x0)
    tr = g[f"{name}_trace"]
    assert rep.status == str(g[f"{name}_status"])
    assert rep.beta == float(g[f"{name}_beta"])
    outer, caps = (int(v) for v in g[f"{name}_counts"])
    it_ref = int(g[f"{name}_iterations"])
    if rep.status == "converged":
        # BB steps inside ALM's best-iterate restarts are chaotic: rounding-level
        # differences grow over ~50 steps and move the later restarts (measured:
        # restarts at rows 23, 33 identical, then 129 vs 130, ...), so the
        # run is held to the same optimum rather than the same step count
        assert rep.outer_iterations >= 1 and outer >= 1
        assert rep.inner_cap_hits == caps == 0
    else:
        assert rep.iterations == it_ref and rep.trace.shape[0] == tr.shape[0]
        assert (rep.outer_iterations, rep.inner_cap_hits) == (outer, caps)
    w = min(25, tr.shape[0], rep.trace.shape[0])
    for col in (1, 2, 5):
        assert close(rep.trace[:w, col], tr[:w, col], 1e-9), col
    assert close(rep.trace[:w, 4], tr[:w, 4], 1e-9, 1e-13)
    fp = g[f"{name}_final_pre"]
    if rep.status != "converged" and np.all(np.isfinite(fp)):
        # the reported iterate is the best of the last inner loop (solver.cpp:570)
        assert close([rep.final_pre_orth.fval, rep.final_pre_orth.kkt_abs], fp[:2], 1e-8)
    if name == "a40_beta0":  # test_solver.cpp:463-479: the penalty-free inner problem is
        assert rep.status != "converged"  # unbounded, the iterates flee the manifold
        if rep.status == "max_iter":
            assert rep.trace[-1, 4] > 100.0 * rep.trace[0, 4] + 1.0
    fpost = g[f"{name}_final_post"]
    if np.all(np.isfinite(fpost)) and rep.final_post_orth is not None:
        assert abs(rep.final_post_orth.fval - fpost[0]) <= 1e-8 * abs(fpost[0]) + 1e-12
        assert rep.final_post_orth.feas <= 1e-12


def test_alm_converges_and_counts_both_loops(pcal):
    """test_solver.cpp:488-498: gen_problem2(30, 3, 1, 1.01, 1.01, 1, 31) from the
    QR start with seed 32 converges with ≥ 1 multiplier update."""
    from paper_1810_03930_b200 import harness as H
    m = H.make_problem(H.ProblemSpec(kind="p2", n=30, p=3, kappa=1.0, theta=1.01, zeta=1.01,
                                     xi=1.0, seed=31))
    rep = pcal.solve(m, pcal.SolverConfig(algorithm="alm"), pcal.initial_point(30, 3, 32))
    assert rep.status == "converged"
    assert rep.outer_iterations >= 1 and rep.iterations >= rep.outer_iterations
    assert rep.final_post_orth.feas <= 1e-12


def test_alm_stationary_start(pcal):
    """test_solver.cpp:318-331 for ALM: a stationary start terminates at once."""
    a = np.diag([1.0, 2.0, 3.0, 4.0])
    x = np.zeros((4, 2))
    x[0, 0] = x[1, 1] = 1.0
    rep = pcal.solve(pcal.QuadraticModel(a, 2, 4.0), pcal.SolverConfig(algorithm="alm"), x)
    assert rep.status == "converged" and rep.iterations == 0 and rep.outer_iterations == 0
    assert rep.trace.shape[0] == 1 and rep.trace[0, 3] == 0.0


def test_alm_report_json_counters(pcal, orc):
    """to_json carries outer_iterations / inner_cap_hits (report_io.cpp:100-101)."""
    import json
    from paper_1810_03930_b200 import report_io as R
    model, x0 = _instance(pcal, orc, "a40")
    rep = pcal.solve(model, pcal.SolverConfig(algorithm="alm", alm=pcal.AlmOptions(6, 5, 0.1)), x0)
    echo = R.echo_for(model, pcal.SolverConfig(algorithm="alm"), rep, problem="p3", seed=0)
    j = json.loads(R.to_json(rep, echo))
    assert (j["outer_iterations"], j["inner_cap_hits"]) == (5, 5)
    assert j["config"]["solver"] == "alm"


@pytest.mark.parametrize("kind", ["stencil", "p4"])
def test_alm_on_every_model_family(pcal, orc, kind):
    """ALM runs on the grid and bilinear device models as on the dense one (the
    engine is model-agnostic): converges, post-orth feasible, at PLAM's optimum.
    (p = 5 on the 8×8×6 grid: the lowest Laplacian cluster, 1 + 4 modes, ends
    at a spectral gap, so the subspace is well defined.)"""
    from paper_1810_03930_b200 import harness as H
    if kind == "stencil":
        grid, n, p = (8, 8, 6), 8 * 8 * 6, 5
        v = orc.random_uniform(n, 3)
        m = pcal.StencilModel(grid, v, p, 12.0 + v.max())
    else:
        n, p = 60, 4
        m = H.make_problem(H.ProblemSpec(kind=kind, n=n, p=p, seed=51))
    x0 = pcal.initial_point(n, p, 52)
    ra = pcal.solve(m, pcal.SolverConfig(algorithm="alm", max_iter=5000), x0)
    rp = pcal.solve(m, pcal.SolverConfig(algorithm="plam", max_iter=5000), x0)
    assert ra.status == "converged" and rp.status == "converged"
    assert ra.final_post_orth.feas <= 1e-12 and ra.outer_iterations >= 1
    assert abs(ra.final_post_orth.fval - rp.final_post_orth.fval) <= 1e-6 * abs(rp.final_post_orth.fval)


def test_alm_sharded_bitwise_across_rank_counts(pcal, orc):
    """ALM on the row-sharded path (emulated ranks): every rank takes the same
    outer decisions from the allreduced ‖∇L‖, and 1–3 ranks give bitwise
    identical reports; the run also matches the reference's
    golden counters and the single-GPU trace window."""
    from paper_1810_03930_b200 import report_io
    g = np.load(os.path.join(GOLD, "reference_alm.npz"))
    model, x0 = _instance(pcal, orc, "c1")
    cfg = pcal.SolverConfig(algorithm="alm", alm=pcal.AlmOptions(7, 50, 0.1), max_iter=60)
    reps = [pcal.solve_emulated(model, cfg, x0, R) for R in (1, 2, 3)]
    outer, caps = (int(v) for v in g["c1_caps_counts"])
    assert reps[0].status == "max_iter" and reps[0].iterations == 60
    assert (reps[0].outer_iterations, reps[0].inner_cap_hits) == (outer, caps)
    for r in reps[1:]:
        assert report_io.same_numerics(reps[0], r)
        assert (r.outer_iterations, r.inner_cap_hits) == (outer, caps)
    single = pcal.solve(model, cfg, x0)
    assert close(reps[0].trace[:25, 1], single.trace[:25, 1], 1e-9)
