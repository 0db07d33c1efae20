"""GPU: the reference's Bilinear (P4) and Density (P1 α > 0, P6) models on the
device (PCAL_MODEL_BILINEAR / PCAL_MODEL_DENSITY) — evaluation against the
reference's own ``evaluate`` (golden values from oracle/_ref), the central
difference gradient check of acceptance #3, and acceptance #2 / #4 exactly as
the reference runs them (run_single over the problem zoo)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

# oracle/make_golden.py MODEL_EVAL_CASES
EVAL_CASES = {
    "p1": dict(kind="p1", n=60, p=6, alpha=1.0, seed=31),
    "p6": dict(kind="p6", n=60, p=6, seed=32),
    "p4": dict(kind="p4", n=60, p=6, seed=35),
    "p1_block": dict(kind="p1", n=45, p=4, alpha=2.0, mode="block-tridiag", seed=36),
    "p6_block": dict(kind="p6", n=45, p=4, mode="block-tridiag", seed=37),
}


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_model_evaluate_matches_reference(pcal, name):
    """f and G = ∇f of gen_problem{1,4,6} (problems.cpp:143-206) at a seeded point:
    the device models agree with the reference's evaluate to 1e-12 (the Hartree
    solve goes through L⁻¹ instead of the triangular solves: rounding only)."""
    from paper_1810_03930_b200 import harness as H
    g = np.load(os.path.join(GOLD, "reference_models.npz"))
    m = H.make_problem(H.ProblemSpec(**EVAL_CASES[name]))
    x = g[name + "_x"]
    f, grad = pcal.evaluate(m, x)
    fr, gr = float(g[name + "_f"]), g[name + "_g"]
    assert abs(f - fr) <= 1e-12 * abs(fr)
    assert np.linalg.norm(grad - gr) <= 1e-12 * np.linalg.norm(gr)


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_fd_gradient_check_matches_reference(pcal, name):
    """fd_gradient_check (problems.cpp:296-325) with the reference defaults
    (h = 1e-5, seed 0x5eedc0de: the same 50 coordinates) through the device
    evaluation, against the reference's own value at the same point.  At these
    sizes the value is rounding noise (ε·|f|/h; the central difference is exact
    or O(h²) small), and the device's tree-ordered sums are no noisier than
    the reference's sequential ones."""
    from paper_1810_03930_b200 import harness as H
    g = np.load(os.path.join(GOLD, "reference_models.npz"))
    m = H.make_problem(H.ProblemSpec(**EVAL_CASES[name]))
    got, ref = pcal.fd_gradient_check(m, g[name + "_x"]), float(g[name + "_fd"])
    assert got <= max(4.0 * ref, 1e-8), (got, ref)
    with pytest.raises(pcal.ParameterError):
        pcal.fd_gradient_check(m, g[name + "_x"], h=0.0)


def test_gradient_central_differences(pcal):
    """Acceptance #3 (acceptance_main.cpp:115-149): density families ≤ 1e-6 with
    h = 1e-5, the bilinear family ≤ 1e-9 with h = 1e-4 (positive density start
    points for P6)."""
    from paper_1810_03930_b200 import harness as H
    rng = np.random.default_rng(3)
    for name, h, tol in (("p1", 1e-5, 1e-6), ("p6", 1e-5, 1e-6), ("p4", 1e-4, 1e-9)):
        m = H.make_problem(H.ProblemSpec(**EVAL_CASES[name]))
        for probe in range(5):
            x = np.asfortranarray(rng.standard_normal((m.n, m.p)))
            while name == "p6" and (x * x).sum(axis=1).min() < 1e-3:
                x = np.asfortranarray(rng.standard_normal((m.n, m.p)))
            assert pcal.fd_gradient_check(m, x, h) <= tol, (name, probe)


@pytest.mark.parametrize("alg", ["plam", "pcal"])
@pytest.mark.parametrize("kind", ["p1", "p2", "p3", "p4"])
def test_acceptance_post_orth_feasibility_zoo(pcal, kind, alg):
    """Acceptance #2 (acceptance_main.cpp:77-111) as the reference runs it:
    run_single(P1–P4 defaults, n = 500, p = 10, seeds 1–5, QR start); every
    converged run ends with post-orth feasibility ≤ 1e-12, at least one converges."""
    from paper_1810_03930_b200 import harness as H
    converged = 0
    for seed in range(1, 6):
        rep, _ = H.run_single(H.ProblemSpec(kind=kind, n=500, p=10, seed=seed),
                              pcal.SolverConfig(algorithm=alg), H.InitialPointSpec())
        if rep.status != "converged":
            continue
        converged += 1
        assert rep.final_post_orth is not None and rep.final_post_orth.feas <= 1e-12
    assert converged >= 1


def test_acceptance_penalty_insensitivity_p1(pcal):
    """Acceptance #4 (acceptance_main.cpp:153-178) exactly: P1 (α = 1) n = 500,
    p = 10, seed 41; PCAL converges for β ∈ {0, 0.01s, 0.1s, s + 0.1, 10s + 1}."""
    from paper_1810_03930_b200 import harness as H
    spec = H.ProblemSpec(kind="p1", n=500, p=10, seed=41)
    s = H.make_problem(spec).s
    for beta in (0.0, 0.01 * s, 0.1 * s, s + 0.1, 10.0 * s + 1.0):
        rep, _ = H.run_single(spec, pcal.SolverConfig(beta=beta), H.InitialPointSpec())
        assert rep.status == "converged", beta


def test_density_model_sharded_layouts(pcal):
    """The sharded session takes the L and L⁻¹ row slabs (pcal_b200.h); a model
    whose linv is missing is a parameter error, not a crash."""
    from paper_1810_03930_b200 import harness as H
    m = H.make_problem(H.ProblemSpec(kind="p6", n=60, p=6, seed=32))
    bad = pcal.DensityModel(m.a, m.p, m.coeff, m.s, variant="p6", linv=m.linv)
    bad.linv = None
    with pytest.raises(pcal.ParameterError):
        pcal.evaluate(bad, np.eye(60, 6, order="F"))


@pytest.mark.parametrize("name", ["p1_near", "p4_far", "p6_near"])
def test_diagnostics_match_reference(pcal, name):
    """kkt_violation, feasibility_violation, merit_h and feasibility_bound_check
    (diagnostics.cpp:21-98) on the device against the reference's values."""
    from paper_1810_03930_b200 import diagnostics as D
    from paper_1810_03930_b200 import harness as H
    spec = {"p1_near": dict(kind="p1", n=60, p=6, alpha=1.0, seed=31, beta=30.0),
            "p4_far": dict(kind="p4", n=60, p=6, seed=35, beta=1.0),
            "p6_near": dict(kind="p6", n=45, p=4, mode="block-tridiag", seed=37, beta=20.0)}[name]
    beta = spec.pop("beta")
    g = np.load(os.path.join(GOLD, "reference_diagnostics.npz"))
    ref = g[name + "_out"]
    x = g[name + "_x"]
    m = H.make_problem(H.ProblemSpec(**spec))
    assert abs(D.kkt_violation(m, x) - ref[0]) <= 1e-11 * ref[0]
    assert abs(D.feasibility_violation(x) - ref[1]) <= 1e-11 * ref[1]
    assert abs(D.merit_h(m, x, beta) - ref[2]) <= 1e-11 * abs(ref[2])
    b = D.feasibility_bound_check(m, x, beta)
    assert b.applicable == bool(ref[3]) and b.holds == bool(ref[7])
    for v, r in ((b.delta, ref[4]), (b.lhs, ref[5]), (b.rhs, ref[6]), (b.slack, ref[8])):
        assert abs(v - r) <= 1e-10 * abs(r) + 1e-14
