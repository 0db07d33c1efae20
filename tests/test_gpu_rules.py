"""GPU parity of the stepsize rules and of orthonormalize's MGS2 branch
(VERDICT r01 item 4).

* stepsize_select (solver.cpp:212-251): Constant, Differential, BB1, BB2 (ABB
  is the default every other test runs) and the clamp to [eta_min, eta_max]
  drive a config-1 solve; the GPU's trace window — η in particular — must
  match the oracle's (the reference's closed forms are pinned on the CPU by
  tests/test_oracle_golden.py against test_solver.cpp:167-224's shapes).
* orthonormalize (kernels.cpp:250-261): a start whose Cholesky pass hits the
  pivot floor 1e-14·‖XᵀX‖_F although the columns are independent, so the MGS2
  fallback runs and succeeds (a nearly parallel column, the condition-1e6
  family of test_kernels.cpp:183-195 pushed to the floor), and one far under
  the floor that raises rank_error.
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TINY = float(np.finfo(float).tiny)
INIT_SALT = 0x1235713
S_CFG1 = 44.26282919872377  # the reference's s for config 1 (tests/golden/reference_small.npz)


def close(a, b, tol, floor=0.0):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return bool(np.all(np.abs(a - b) <= tol * np.abs(b) + floor))


@pytest.fixture(scope="module")
def inst(pcal, orc):
    a = pcal.gen_dense_operator(1000, 1)
    x0 = orc.initial_point_qr(1000, 20, 1 ^ INIT_SALT)
    return a, x0


RULES = {  # name: (kind, gamma, eta_min, eta_max)
    "constant": (0, S_CFG1 + 2.0, 1e-10, 1e10),
    "differential": (1, 1.0, 1e-10, 1e10),
    "bb1": (2, 1.0, 1e-10, 1e10),
    "bb2": (3, 1.0, 1e-10, 1e10),
    "abb_clamped": (4, 1.0, 40.0, 47.0),
}


@pytest.mark.parametrize("name", list(RULES))
def test_stepsize_rule_trace_matches_oracle(pcal, orc, inst, name):
    from oracle.oracle import Config, Model, MODEL_DENSE
    a, x0 = inst
    kind, gamma, lo, hi = RULES[name]
    ref = orc.solve(Model(MODEL_DENSE, 1000, 20, S_CFG1, a=a),
                    Config(eta_kind=kind, gamma=gamma, eta_min=lo, eta_max=hi,
                           tol_rel_kkt=TINY, max_iter=60, threads=8), x0)
    rule = pcal.StepsizeRule(kind=kind, gamma=gamma, eta_min=lo, eta_max=hi)
    rep = pcal.solve(pcal.QuadraticModel(a, 20, S_CFG1),
                     pcal.SolverConfig(eta_rule=rule, tol_rel_kkt=TINY, max_iter=60), x0)
    assert rep.status == ref.status and rep.trace.shape == (ref.trace.shape[0], 7)
    w = 30
    assert close(rep.trace[:w, 5], ref.trace[:w, 5], 1e-9)   # η: the rule itself
    assert close(rep.trace[:w, 1], ref.trace[:w, 1], 1e-9)
    assert close(rep.trace[:w, 2], ref.trace[:w, 2], 1e-9)
    assert close(rep.trace[:w, 4], ref.trace[:w, 4], 1e-9, 1e-14)
    if name == "constant":
        assert np.all(rep.trace[:, 5] == gamma)
    if name == "abb_clamped":
        assert np.all((rep.trace[:, 5] >= lo) & (rep.trace[:, 5] <= hi))
        assert np.any(rep.trace[1:, 5] == lo) or np.any(rep.trace[1:, 5] == hi)
    assert abs(rep.final_post_orth.fval - ref.final_post[0]) <= 1e-9 * abs(ref.final_post[0])


def _near_parallel(orc, n, eps_scale):
    """Three columns: u, w and u + α·q (q ⟂ u, w) with α² just above the pivot
    floor — independent, but the Cholesky pivot of the third column suffers
    the cancellation a_33 − l_31² and can land under 1e-14·‖XᵀX‖_F."""
    q = orc.orthonormalize(orc.random_normal(n, 3, 4242))
    a2 = 1e-14 * math.sqrt(5.0) * eps_scale  # ‖XᵀX‖_F ≈ √5
    return np.asfortranarray(np.stack([q[:, 0], q[:, 1], q[:, 0] + math.sqrt(a2) * q[:, 2]],
                                      axis=1))


def test_orthonormalize_mgs2_fallback_succeeds(pcal, orc):
    """orthonormalize falls back to MGS2 exactly when a Cholesky pivot lands on
    or under 1e-14·‖XᵀX‖_F; MGS2 then tests the SAME quantity (the column's
    squared distance to the span of the previous ones) against the same floor,
    so 'Cholesky fails, MGS2 succeeds' only happens within rounding of the floor
    — which side a start lands on depends on summation order, in the reference
    as on the GPU.  Scan α upward from the floor until the DEVICE takes the
    MGS2 branch and succeeds; the result must be the oracle's MGS2 of the same
    matrix (kernels.cpp:212-246) and an orthonormal basis of X's column flag."""
    hit = None
    for k in range(800):
        x = _near_parallel(orc, 50, 1.0 + 0.05 * k / 800)
        try:
            q = pcal.orthonormalize(x)
        except np.linalg.LinAlgError:
            continue  # α still under the floor for MGS2 as well
        if pcal.last_orthonormalize_path().startswith("mgs2"):
            floor = 1e-14 * np.linalg.norm(orc.gram(x))
            try:
                qo = orc.mgs2(x, floor)
            except np.linalg.LinAlgError:
                continue  # the oracle's sums put this start under the floor
            hit = (x, q, qo)
            break
    assert hit is not None, "no start took (and passed) the MGS2 branch"
    x, q, qo = hit
    assert np.linalg.norm(q.T @ q - np.eye(3)) <= 1e-12
    s = np.sign(np.sum(q * qo, axis=0))
    assert np.all(s > 0)  # MGS keeps each column's direction (positive R diagonal)
    assert np.abs(q[:, :2] - qo[:, :2]).max() <= 1e-13
    assert np.abs(q[:, 2] - qo[:, 2]).max() <= 1e-6  # the ~1e-7-sized residual's direction
    r = q.T @ x  # X = Q·R with R upper triangular
    assert np.abs(np.tril(r, -1)).max() <= 1e-12


def test_orthonormalize_rank_deficient_raises(pcal, orc):
    x = _near_parallel(orc, 50, 1e-6)  # α² far under the floor: MGS2 fails as well
    with pytest.raises(np.linalg.LinAlgError):
        pcal.orthonormalize(x)
    assert pcal.last_orthonormalize_path() == "rank"
