"""GPU: caller-defined objectives (PCAL_MODEL_DEVICE_CALLBACK) — the device-side
counterpart of subclassing orthopt::ObjectiveModel (problems.hpp:24-51).  The
example model (examples/device_model_example.cu) computes f = ½tr(XᵀAX) with
its own naive kernels; PCAL around it must follow the built-in dense model."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXAMPLE = os.path.join(ROOT, "build", "libpcal_device_model_example.so")
TINY = np.finfo(float).tiny


class _QuadCtx(C.Structure):
    _fields_ = [("a", C.c_void_p), ("lda", C.c_int64), ("shift", C.c_double)]


def _close(a, b, tol, floor=0.0):
    return np.all(np.abs(np.asarray(a) - np.asarray(b)) <= tol * np.abs(np.asarray(b)) + floor)


@pytest.fixture(scope="module")
def example():
    lib = C.CDLL(EXAMPLE)
    return C.cast(lib.pcal_example_quadratic_grad, C.c_void_p).value


def test_device_callback_model_follows_dense_model(pcal, orc, example):
    import torch
    n, p = 300, 8
    a = pcal.gen_dense_operator(n, 5)
    s = orc.spectral_norm_estimate(a, 5 ^ 0x73706563)
    a_dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()  # column-major A
    ctx = _QuadCtx(a_dev.data_ptr(), n)
    x0 = pcal.initial_point(n, p, 6)
    cfg = pcal.SolverConfig(tol_rel_kkt=TINY, max_iter=60)
    m_cb = pcal.DeviceCallbackModel(n, p, s, grad=example, ctx=C.addressof(ctx))
    r_cb = pcal.solve(m_cb, cfg, x0)
    r_ref = pcal.solve(pcal.QuadraticModel(a, p, s), cfg, x0)
    assert r_cb.status == r_ref.status == "max_iter"
    for col in (1, 2, 4, 5):
        assert _close(r_cb.trace[:40, col], r_ref.trace[:40, col], 1e-9, 1e-14)
    assert abs(r_cb.final_post_orth.fval - r_ref.final_post_orth.fval) <= \
        1e-9 * abs(r_ref.final_post_orth.fval)
    # converges like the built-in model
    rc = pcal.solve(m_cb, pcal.SolverConfig(), x0)
    rr = pcal.solve(pcal.QuadraticModel(a, p, s), pcal.SolverConfig(), x0)
    assert rc.status == rr.status == "converged"
    assert abs(rc.final_post_orth.fval - rr.final_post_orth.fval) <= 1e-9 * abs(rr.final_post_orth.fval)
    del a_dev


def test_fd_gradient_check_flags_a_perturbed_callback(pcal, example):
    """fd_gradient_check on a caller-defined model (problems.cpp:296-325): the exact
    gradient passes at the quadratic tolerance, a gradient shifted by 1e-3 (the
    reference's PerturbedModel fault injection, test_problems.cpp:27-42,187-194)
    is flagged at ≥ 5e-4."""
    import torch
    n, p = 120, 5
    a = pcal.gen_dense_operator(n, 8) / np.sqrt(n)
    a_dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    x = pcal.initial_point(n, p, 9)
    ctx = _QuadCtx(a_dev.data_ptr(), n, 0.0)
    m = pcal.DeviceCallbackModel(n, p, 1.0, grad=example, ctx=C.addressof(ctx))
    assert pcal.fd_gradient_check(m, x, 1e-4) <= 1e-9
    ctx.shift = 1e-3
    assert pcal.fd_gradient_check(m, x, 1e-4) >= 5e-4
    del a_dev


def test_device_callback_nonfinite_gradient_is_evaluation_error(pcal):
    """check_finite (problems.cpp:27-30) ⇒ evaluation_error ⇒ status Diverged
    with no trace row for that point (solver.cpp:460-466)."""
    cudart = C.CDLL("libcudart.so.12")
    cudart.cudaMemsetAsync.argtypes = [C.c_void_p, C.c_int, C.c_size_t, C.c_void_p]

    def grad(x, ld, n, p, g, f, stream, ctx):
        # 0xFF bytes are NaNs; memset nodes are capturable like kernels
        cudart.cudaMemsetAsync(g, 0xFF, 8 * ld * p, stream)
        cudart.cudaMemsetAsync(f, 0, 8, stream)
        return 0

    fn = pcal.GRADIENT_FN(grad)
    x0 = pcal.initial_point(64, 2, 1)
    rep = pcal.solve(pcal.DeviceCallbackModel(64, 2, 1.0, grad=fn), pcal.SolverConfig(), x0)
    assert rep.status == "diverged" and rep.trace.shape[0] == 0


def test_device_callback_failure_is_reported(pcal):
    fn = pcal.GRADIENT_FN(lambda *args: 7)
    with pytest.raises(pcal.EvaluationError):
        pcal.solve(pcal.DeviceCallbackModel(64, 2, 1.0, grad=fn), pcal.SolverConfig(),
                   pcal.initial_point(64, 2, 1))
    with pytest.raises(RuntimeError):  # PCAL_E_UNSUPPORTED: device-callback models are single-GPU
        pcal.solve_emulated(pcal.DeviceCallbackModel(64, 2, 1.0, grad=fn), pcal.SolverConfig(),
                            pcal.initial_point(64, 2, 1), 2)
