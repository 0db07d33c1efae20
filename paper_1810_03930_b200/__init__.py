"""B200-native PCAL iteration — Python mirror of the reference ``orthopt`` API.

The reference is a C++ library (``orthopt::solve``, solver.hpp:120-121); this
package is a thin ctypes layer over the C ABI of ``libpcal_b200.so``
(``include/pcal_b200.h``) with the same names, argument meanings and error
behaviour:

* ``SolverConfig`` / ``StepsizeRule`` / ``MultiplierRule``  (solver.hpp:13-42)
* ``QuadraticModel`` / ``make_quadratic`` / ``StencilModel`` / ``KohnShamModel``
  (problems.hpp:28-111; the grid models are DESIGN.md §3)
* ``solve(model, config, x0, timers=None) -> RunReport``   (report.hpp:51-64)
* building blocks: ``gram``, ``matmul_at_b``, ``matmul``, ``orthonormalize``,
  ``pcal_step``, ``spectral_norm_estimate``, ``initial_point``, ``evaluate``.

Errors: ``ParameterError`` / ``DimensionError`` (reference parameter_error /
dimension_error) are raised before iterating; divergence inside a run is
reported as ``status == "diverged"`` with a partial trace, not raised.  There
is no CPU fallback: if the native library or a CUDA device is missing, calls
raise ``NativeUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "SolverConfig", "StepsizeRule", "MultiplierRule", "RunReport", "FinalMetrics",
    "CategoryTimers", "AlmOptions", "QuadraticModel", "StencilModel", "KohnShamModel", "make_quadratic",
    "BilinearModel", "DensityModel", "density_inverse",
    "solve", "Session", "gram", "matmul_at_b", "matmul", "orthonormalize", "pcal_step",
    "spectral_norm_estimate", "initial_point", "evaluate", "fd_gradient_check", "random_normal", "random_uniform",
    "gen_dense_operator", "flops_estimate", "ParameterError", "DimensionError", "RankError",
    "DivergenceError", "EvaluationError", "NativeUnavailable", "lib", "LIB_PATH",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpcal_b200.so")

OK, E_PARAMETER, E_DIMENSION, E_RANK, E_UNSUPPORTED, E_CUDA, E_STATE = 0, -1, -2, -3, -4, -5, -6
E_DIVERGENCE, E_EVALUATION = -7, -8
STATUS = {0: "converged", 1: "max_iter", 2: "diverged"}
TRACE_COLS = 7
HOST, DEVICE, X0_SEED = 0, 1, 2
MODEL_DENSE, MODEL_STENCIL, MODEL_KOHN_SHAM, MODEL_DEVICE_CALLBACK = 1, 2, 3, 4
MODEL_BILINEAR, MODEL_DENSITY = 5, 6
DENSITY_P1, DENSITY_P6 = 0, 1


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or no B200 is visible (no CPU fallback)."""


class ParameterError(ValueError):
    """orthopt::parameter_error (errors.hpp:24-28)."""


class DimensionError(ValueError):
    """orthopt::dimension_error (errors.hpp:9-13)."""


class RankError(np.linalg.LinAlgError):
    """orthopt::rank_error (errors.hpp:15-19)."""


class DivergenceError(FloatingPointError):
    """orthopt::divergence_error (errors.hpp:33-45)."""


class EvaluationError(FloatingPointError):
    """orthopt::evaluation_error (errors.hpp:27-31)."""


_dp = C.POINTER(C.c_double)


class _Model(C.Structure):
    _fields_ = [("kind", C.c_int32), ("location", C.c_int32), ("n", C.c_int64), ("p", C.c_int64),
                ("s", C.c_double), ("a", C.c_void_p), ("g0", C.c_void_p), ("nx", C.c_int64),
                ("ny", C.c_int64), ("nz", C.c_int64), ("v", C.c_void_p), ("grad", C.c_void_p),
                ("grad_ctx", C.c_void_p), ("b", C.c_void_p), ("linv", C.c_void_p),
                ("coeff", C.c_double), ("density_variant", C.c_int32)]


# pcal_gradient_fn (include/pcal_b200.h): enqueue G = ∇f(X) and f(X) on `stream`
GRADIENT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_void_p)


class _Config(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("beta", C.c_double), ("eta_kind", C.c_int32),
                ("gamma", C.c_double), ("eta_min", C.c_double), ("eta_max", C.c_double),
                ("eta0", C.c_double), ("multiplier_rule", C.c_int32),
                ("tol_rel_kkt", C.c_double), ("max_iter", C.c_int64),
                ("final_orth", C.c_int32), ("device", C.c_int32),
                ("alm_inner_max", C.c_int32), ("alm_outer_max", C.c_int32),
                ("alm_inner_tol_scale", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("trace", _dp), ("trace_capacity", C.c_int64), ("trace_len", C.c_int64),
                ("final_pre", C.c_double * 4), ("final_post", C.c_double * 4),
                ("has_post", C.c_int32), ("stop_x", _dp), ("final_x", _dp), ("has_x", C.c_int32),
                ("iterations", C.c_int64), ("degenerate_steps", C.c_int64),
                ("wall_time", C.c_double), ("status", C.c_int32), ("beta", C.c_double),
                ("eta0", C.c_double), ("outer_iterations", C.c_int64),
                ("inner_cap_hits", C.c_int64)]


class _Timers(C.Structure):
    _fields_ = [("blas3", C.c_double), ("func", C.c_double), ("orth", C.c_double)]


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libpcal_b200.so (built in-tree by ``__graft_entry__.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(f"{LIB_PATH} not built; run python -m paper_1810_03930_b200.build")
    L = C.CDLL(LIB_PATH)
    i64, i32, dbl, vp, u64 = C.c_int64, C.c_int32, C.c_double, C.c_void_p, C.c_uint64
    L.pcal_last_error.restype = C.c_char_p
    L.pcal_config_default.argtypes = [C.POINTER(_Config)]
    L.pcal_solve.argtypes = [C.POINTER(_Model), C.POINTER(_Config), vp, i32, C.POINTER(_Report),
                             C.POINTER(_Timers)]
    L.pcal_session_create.argtypes = [C.POINTER(_Model), C.POINTER(_Config), vp, i32,
                                      C.POINTER(vp)]
    L.pcal_session_run.argtypes = [vp, i64]
    L.pcal_session_sync.argtypes = [vp]
    L.pcal_session_stream.argtypes = [vp]
    L.pcal_session_stream.restype = vp
    L.pcal_session_finish.argtypes = [vp, C.POINTER(_Report)]
    L.pcal_session_destroy.argtypes = [vp]
    L.pcal_session_set_state.argtypes = [vp, vp, vp, i64, dbl]
    L.pcal_session_get_x.argtypes = [vp, vp, C.POINTER(dbl), C.POINTER(i64)]
    L.pcal_session_device_x.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
    L.pcal_session_kernel_launches.argtypes = [vp]
    L.pcal_session_kernel_launches.restype = i64
    L.pcal_session_profile.argtypes = [vp, i64, _dp]
    L.pcal_session_profile_kernels.argtypes = [vp, i64, C.c_char_p, i64]
    L.pcal_session_kernels_per_iteration.argtypes = [vp]
    L.pcal_session_kernels_per_iteration.restype = i64
    L.pcal_session_xm_mode.argtypes = [vp, C.POINTER(i64)]
    L.pcal_session_xm_mode.restype = C.c_int
    L.pcal_matmul_at_b.argtypes = [vp, vp, i64, i64, i64, vp, i32]
    L.pcal_matmul.argtypes = [vp, vp, i64, i64, i64, vp, i32]
    L.pcal_gram.argtypes = [vp, i64, i64, vp, i32]
    L.pcal_orthonormalize.argtypes = [vp, i64, i64, vp, i32]
    L.pcal_evaluate.argtypes = [C.POINTER(_Model), vp, C.POINTER(dbl), vp, i32]
    L.pcal_fd_gradient_check.argtypes = [C.POINTER(_Model), vp, dbl, u64, i32, C.POINTER(dbl)]
    L.pcal_pcal_step.argtypes = [vp, vp, i64, i64, dbl, vp, C.POINTER(i64), i32]
    L.pcal_spectral_norm_estimate.argtypes = [vp, i64, u64, C.POINTER(dbl), i32]
    L.pcal_flops_estimate.argtypes = [i64, i64]
    L.pcal_flops_estimate.restype = dbl
    L.pcal_random_normal.argtypes = [i64, i64, u64, vp, i32]
    L.pcal_random_uniform.argtypes = [i64, u64, vp]
    L.pcal_spectral_norm_estimate_host.argtypes = [vp, i64, u64, i32, C.POINTER(dbl)]
    L.pcal_gen_dense_operator.argtypes = [i64, u64, vp, i32]
    L.pcal_density_inverse.argtypes = [vp, i64, vp, i32]
    L.pcal_initial_point_qr.argtypes = [i64, i64, u64, vp, i32]
    L.pcal_initial_point.argtypes = [i64, i64, i32, dbl, u64, vp, i32]
    L.pcal_partition.argtypes = [C.POINTER(_Model), i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.pcal_nccl_unique_id.argtypes = [vp]
    L.pcal_comm_create_nccl.argtypes = [i32, i32, vp, i32, C.POINTER(vp)]
    L.pcal_comm_destroy.argtypes = [vp]
    L.pcal_session_create_sharded.argtypes = [C.POINTER(_Model), C.POINTER(_Config), vp, i32, vp,
                                              C.POINTER(vp)]
    L.pcal_solve_sharded.argtypes = [C.POINTER(_Model), C.POINTER(_Config), vp, i32, vp,
                                     C.POINTER(_Report), C.POINTER(_Timers)]
    L.pcal_solve_emulated.argtypes = [C.POINTER(_Model), C.POINTER(_Config), vp, i32,
                                      C.POINTER(_Report), C.POINTER(_Timers)]
    L.pcal_row_chunks.argtypes = [C.POINTER(_Model), C.POINTER(i64), C.POINTER(i64)]
    L.pcal_device_count.argtypes = [C.POINTER(i32)]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().pcal_last_error().decode(errors="replace")
    if rc == E_PARAMETER:
        raise ParameterError(msg)
    if rc == E_DIMENSION:
        raise DimensionError(msg)
    if rc == E_RANK:
        raise RankError(msg)
    if rc == E_DIVERGENCE:
        raise DivergenceError(msg)
    if rc == E_EVALUATION:
        raise EvaluationError(msg)
    if rc == E_CUDA:
        raise NativeUnavailable(msg)
    raise RuntimeError(f"pcal error {rc}: {msg}")


def _f64(a) -> np.ndarray:
    """Column-major FP64 host matrix (DenseMatrix layout, matrix.hpp:38-45)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):  # torch tensor already on the device
        return a.data_ptr()
    raise TypeError(type(a))


# --------------------------------------------------------------------------- #
# configuration and results (solver.hpp:13-42, report.hpp:13-72)
# --------------------------------------------------------------------------- #
class StepsizeKind:
    CONSTANT, DIFFERENTIAL, BB1, BB2, ABB = range(5)


class MultiplierRule:
    PLAM_FORMULA, PCAL_FORMULA = 0, 1


@dataclass
class StepsizeRule:
    kind: int = StepsizeKind.ABB
    gamma: float = 1.0
    eta_min: float = 1e-10
    eta_max: float = 1e10
    eta0: float = 0.0


@dataclass
class AlmOptions:
    """AlmOptions (solver.hpp:24-28)."""
    inner_max: int = 500          # gradient steps per multiplier update
    outer_max: int = 50           # multiplier updates
    inner_tol_scale: float = 0.1  # inner target: max(scale·tol, scale^k)·kkt0


@dataclass
class SolverConfig:
    """orthopt::SolverConfig; ``device`` replaces the explicit thread count.
    ``algorithm``: "pcal" (default), "plam", "alm", "moptqr", "plam-da", "pcal-da"."""
    beta: float = -1.0
    eta_rule: StepsizeRule = field(default_factory=StepsizeRule)
    multiplier_rule: int = MultiplierRule.PCAL_FORMULA
    tol_rel_kkt: float = 1e-8
    max_iter: int = 3000
    final_orth: bool = True
    device: int = 0
    algorithm: str = "pcal"
    alm: AlmOptions = field(default_factory=AlmOptions)

    ALGORITHMS = {"plam": 0, "pcal": 1, "alm": 2, "moptqr": 3, "plam-da": 4, "pcal-da": 5}

    def _c(self) -> _Config:
        if self.algorithm not in self.ALGORITHMS:
            raise ParameterError(f"unknown algorithm {self.algorithm!r} "
                                 f"({', '.join(self.ALGORITHMS)})")
        r = self.eta_rule
        return _Config(self.ALGORITHMS[self.algorithm], self.beta, r.kind, r.gamma, r.eta_min, r.eta_max, r.eta0,
                       self.multiplier_rule, self.tol_rel_kkt, self.max_iter,
                       int(self.final_orth), self.device, int(self.alm.inner_max),
                       int(self.alm.outer_max), float(self.alm.inner_tol_scale))


@dataclass
class FinalMetrics:
    fval: float
    kkt_abs: float
    kkt_rel: float
    feas: float


@dataclass
class CategoryTimers:
    blas3: float = 0.0
    func: float = 0.0
    orth: float = 0.0


@dataclass
class RunReport:
    trace: np.ndarray              # (rows, 7): iter, fval, kkt_abs, kkt_rel, feas, eta, elapsed
    final_pre_orth: FinalMetrics
    final_post_orth: Optional[FinalMetrics]
    stop_iterate: Optional[np.ndarray]
    final_x: Optional[np.ndarray]
    iterations: int
    degenerate_steps: int
    wall_time: float
    status: str
    beta: float
    eta0: float
    outer_iterations: int = 0      # ALM multiplier updates (report.hpp:59)
    inner_cap_hits: int = 0        # ALM inner loops stopped by a cap (report.hpp:60)


# --------------------------------------------------------------------------- #
# models (problems.hpp:28-111; grid models: DESIGN.md §3)
# --------------------------------------------------------------------------- #
class _ModelBase:
    kind: int
    n: int
    p: int
    s: float

    def curvature_scale(self) -> float:
        return self.s

    def _c(self) -> tuple:
        raise NotImplementedError


class QuadraticModel(_ModelBase):
    """f(X) = ½tr(XᵀAX) + tr(G0ᵀX) with dense symmetric A (problems.cpp:125-141).
    ``a`` may be a host numpy array or a CUDA torch tensor (column-major)."""

    def __init__(self, a, p: int, s: float, g0=None, n: Optional[int] = None):
        self.kind = MODEL_DENSE
        on_dev = hasattr(a, "data_ptr") and not isinstance(a, np.ndarray)
        self.a = a if on_dev else _f64(a)
        self.g0 = None if g0 is None else (g0 if on_dev else _f64(g0))
        self.location = DEVICE if on_dev else HOST
        # n: global size (a may be the local row slab of a sharded session)
        self.n = int(a.shape[1]) if n is None else int(n)
        self.p = int(p)
        self.s = float(s)

    def _c(self) -> tuple:
        return _Model(self.kind, self.location, self.n, self.p, self.s, _ptr(self.a),
                      _ptr(self.g0), 0, 0, 0, None), (self.a, self.g0)


class StencilModel(_ModelBase):
    """f(X) = ½tr(XᵀLX) + ½tr(XᵀVX), L = −Δ_h 7-point periodic (configs 3 and 5).
    ``v`` is the potential of the owned rows (all rows on a single GPU)."""

    def __init__(self, grid, v, p: int, s: float):
        self.kind = MODEL_STENCIL
        self.grid = tuple(int(g) for g in grid)
        self.v = np.ascontiguousarray(v, dtype=np.float64)
        self.n = self.grid[0] * self.grid[1] * self.grid[2]
        self.p = int(p)
        self.s = float(s)

    def _c(self) -> tuple:
        return _Model(self.kind, HOST, self.n, self.p, self.s, None, None, *self.grid,
                      _ptr(self.v)), (self.v,)


class KohnShamModel(StencilModel):
    """E(X) = ¼tr(XᵀLX) + ½tr(XᵀV_ion X) + ¼ρᵀL†ρ + ½ρᵀε_xc(ρ) (config 4)."""

    def __init__(self, grid, v_ion, p: int, s: float):
        super().__init__(grid, v_ion, p, s)
        self.kind = MODEL_KOHN_SHAM


class DeviceCallbackModel(_ModelBase):
    """A caller-defined objective evaluated by the caller's own device code
    (PCAL_MODEL_DEVICE_CALLBACK): the device-side counterpart of subclassing
    ``orthopt::ObjectiveModel`` (problems.hpp:24-51).  ``grad`` is a
    ``pcal_gradient_fn`` — a C function address (int) or a ``GRADIENT_FN``
    object — that enqueues G = ∇f(X) and f(X) on the stream it is given;
    ``ctx`` is passed through (int address or None).  Single GPU."""

    def __init__(self, n: int, p: int, s: float, grad, ctx=None):
        self.kind = MODEL_DEVICE_CALLBACK
        self.n, self.p, self.s = int(n), int(p), float(s)
        self.grad = grad
        self.ctx = ctx

    def _c(self) -> tuple:
        g = self.grad if isinstance(self.grad, int) else C.cast(self.grad, C.c_void_p).value
        return _Model(self.kind, HOST, self.n, self.p, self.s, None, None, 0, 0, 0, None, g,
                      self.ctx), (self.grad,)


class BilinearModel(_ModelBase):
    """f(X) = ½tr(XᵀAXB), A n×n and B p×p symmetric (BilinearModel, problems.cpp:143-156;
    problem P4).  ``a`` may be the local row slab of a sharded session (then pass n)."""

    def __init__(self, a, b, s: float, n: Optional[int] = None):
        self.kind = MODEL_BILINEAR
        self.a = _f64(a)
        self.b = _f64(b)
        if self.b.ndim != 2 or self.b.shape[0] != self.b.shape[1]:
            raise DimensionError("BilinearModel: b must be p-by-p")
        self.location = HOST
        self.n = int(self.a.shape[1]) if n is None else int(n)
        self.p = int(self.b.shape[0])
        self.s = float(s)

    def _c(self) -> tuple:
        return _Model(self.kind, HOST, self.n, self.p, self.s, _ptr(self.a), None, 0, 0, 0, None,
                      None, None, _ptr(self.b)), (self.a, self.b)


def density_inverse(l, threads: int = 8) -> np.ndarray:
    """L⁻¹ by the reference's LinearSolver (linsolve.cpp:30-102: Cholesky, else LU
    with partial pivoting); raises ParameterError (generation_error) if singular."""
    l = _f64(l)
    out = np.empty_like(l, order="F")
    rc = lib().pcal_density_inverse(_ptr(l), l.shape[0], _ptr(out), threads)
    if rc == E_PARAMETER:
        raise ParameterError("LinearSolver: matrix is numerically singular")
    _check(rc)
    return out


class DensityModel(_ModelBase):
    """DensityModel (problems.cpp:158-206): f = ½tr(XᵀLX) plus, with ρ = rowsq(X)
    and h = L⁻¹ρ, ¼·coeff·ρᵀh (P1) or ½ρᵀh − ¾·coeff·Σρ^{4/3} (P6).  L⁻¹ is
    formed at construction, as the reference builds its LinearSolver there.
    ``l`` / ``linv`` may be the local row slabs of a sharded session (pass n)."""

    def __init__(self, l, p: int, coeff: float, s: float, variant: str = "p1", linv=None,
                 n: Optional[int] = None, mode: str = "random-sym"):
        self.kind = MODEL_DENSITY
        self.mode = mode  # OperatorMode of L (recorded in the container form)
        if int(p) < 1 or 2 * int(p) > (l.shape[1] if n is None else n):
            raise ParameterError("DensityModel: dimensions must satisfy 2p <= n")
        self.a = _f64(l)
        self.linv = density_inverse(self.a) if linv is None else _f64(linv)
        self.variant = variant.lower()
        if self.variant not in ("p1", "p6"):
            raise ParameterError(f"DensityModel: unknown variant {variant!r}")
        self.coeff = float(coeff)
        self.location = HOST
        self.n = int(self.a.shape[1]) if n is None else int(n)
        self.p = int(p)
        self.s = float(s)

    def _c(self) -> tuple:
        return _Model(self.kind, HOST, self.n, self.p, self.s, _ptr(self.a), None, 0, 0, 0, None,
                      None, None, None, _ptr(self.linv), self.coeff,
                      DENSITY_P6 if self.variant == "p6" else DENSITY_P1), (self.a, self.linv)


def make_quadratic(a, p: int, s: float, g0=None) -> QuadraticModel:
    """make_quadratic (problems.cpp:289-294); s must be given (use
    ``spectral_norm_estimate`` to compute it on the device)."""
    return QuadraticModel(a, p, s, g0)


# --------------------------------------------------------------------------- #
# solve (solver.hpp:120-121)
# --------------------------------------------------------------------------- #
def _report_from(rep: _Report, trace: np.ndarray, stop_x, final_x) -> RunReport:
    fp = FinalMetrics(*rep.final_pre[:])
    post = FinalMetrics(*rep.final_post[:]) if rep.has_post else None
    return RunReport(trace=trace[: rep.trace_len].copy(), final_pre_orth=fp, final_post_orth=post,
                     stop_iterate=stop_x if rep.has_x else None,
                     final_x=final_x if rep.has_x else None, iterations=rep.iterations,
                     degenerate_steps=rep.degenerate_steps, wall_time=rep.wall_time,
                     status=STATUS[rep.status], beta=rep.beta, eta0=rep.eta0,
                     outer_iterations=rep.outer_iterations, inner_cap_hits=rep.inner_cap_hits)


def _out_matrix(buf, n: int, p: int) -> np.ndarray:
    if buf is None:
        return np.zeros((n, p), order="F")
    if buf.shape != (n, p) or buf.dtype != np.float64 or not buf.flags.f_contiguous:
        raise DimensionError("report output buffers must be Fortran-ordered float64 n x p")
    return buf


def _new_report(n: int, p: int, max_iter: int, want_x: bool = True, out=None) -> tuple:
    """Report buffers; `out` = (stop_x, final_x): caller-owned host matrices
    (e.g. pinned memory) that receive the iterates instead of fresh arrays."""
    trace = np.zeros((max_iter + 1, TRACE_COLS))
    o_stop, o_final = out if out is not None else (None, None)
    stop_x = _out_matrix(o_stop, n, p) if want_x else None
    final_x = _out_matrix(o_final, n, p) if want_x else None
    rep = _Report()
    rep.trace = trace.ctypes.data_as(_dp)
    rep.trace_capacity = max_iter + 1
    rep.stop_x = stop_x.ctypes.data_as(_dp) if want_x else None
    rep.final_x = final_x.ctypes.data_as(_dp) if want_x else None
    return rep, trace, stop_x, final_x


def solve(model: _ModelBase, config: SolverConfig, x0,
          timers: Optional[CategoryTimers] = None, out=None) -> RunReport:
    """orthopt::solve for PCAL on the B200 (host buffers in, host report out).
    out: optional (stop_x, final_x) host buffers the report's iterates are
    written into (n×p, Fortran order; pinned memory makes the copy-out a DMA)."""
    L = lib()
    cm, keep = model._c()
    cc = config._c()
    on_dev = hasattr(x0, "data_ptr") and not isinstance(x0, np.ndarray)
    if not on_dev:
        x0 = _f64(x0)
    if tuple(x0.shape) != (model.n, model.p):
        raise DimensionError("solve: start point shape mismatch")
    rep, trace, stop_x, final_x = _new_report(model.n, model.p, config.max_iter, out=out)
    tm = _Timers() if timers is not None else None
    _check(L.pcal_solve(C.byref(cm), C.byref(cc), _ptr(x0), DEVICE if on_dev else HOST,
                        C.byref(rep), C.byref(tm) if tm is not None else None))
    if timers is not None:
        timers.blas3 += tm.blas3
        timers.func += tm.func
        timers.orth += tm.orth
    del keep
    return _report_from(rep, trace, stop_x, final_x)


def _x0_arg(x0) -> tuple:
    """(pointer, location, keep-alive) of a start point: a host array, a device
    tensor, or an int seed (PCAL_X0_SEED: initial_point({Qr}, seed) built by the
    library on the device, solver.cpp:136-142)."""
    if isinstance(x0, (int, np.integer)) and not isinstance(x0, bool):
        seed = C.c_uint64(int(x0))
        return C.cast(C.byref(seed), C.c_void_p).value, X0_SEED, seed
    if hasattr(x0, "data_ptr") and not isinstance(x0, np.ndarray):
        return _ptr(x0), DEVICE, x0
    x0 = _f64(x0)
    return _ptr(x0), HOST, x0


class Session:
    """Device-resident run split into create / run / finish (pcal_session_*).
    x0: host array, device tensor, or an int seed (library-built initial point)."""

    def __init__(self, model: _ModelBase, config: SolverConfig, x0):
        self._L = lib()
        self.model, self.config = model, config
        cm, self._keep = model._c()
        cc = config._c()
        ptr, loc, self._x0 = _x0_arg(x0)
        h = C.c_void_p()
        _check(self._L.pcal_session_create(C.byref(cm), C.byref(cc), ptr, loc, C.byref(h)))
        self._h = h
        self.n_local = model.n

    def run(self, iters: int) -> None:
        _check(self._L.pcal_session_run(self._h, iters))

    def sync(self) -> None:
        _check(self._L.pcal_session_sync(self._h))

    @property
    def stream(self) -> int:
        return self._L.pcal_session_stream(self._h) or 0

    def set_state(self, x_prev, x, k: int, eta_prev: float) -> None:
        xp = None if x_prev is None else _f64(x_prev)
        xx = _f64(x)
        _check(self._L.pcal_session_set_state(self._h, _ptr(xp), _ptr(xx), k, eta_prev))

    def get_x(self, out=None) -> tuple:
        """(X_k, η_{k−1}, k) of the current iterate (this rank's rows); `out`: an
        optional preallocated Fortran-ordered host array (e.g. pinned memory)."""
        x = np.zeros((self.n_local, self.model.p), order="F") if out is None else out
        if x.shape != (self.n_local, self.model.p) or not x.flags.f_contiguous:
            raise DimensionError("get_x: out must be a Fortran-ordered n_local x p array")
        eta = C.c_double()
        k = C.c_int64()
        _check(self._L.pcal_session_get_x(self._h, _ptr(x), C.byref(eta), C.byref(k)))
        return x, eta.value, k.value

    def device_x(self) -> tuple:
        p = C.c_void_p()
        ld = C.c_int64()
        _check(self._L.pcal_session_device_x(self._h, C.byref(p), C.byref(ld)))
        return p.value, ld.value

    def finish(self, want_x: bool = True) -> RunReport:
        rep, trace, stop_x, final_x = _new_report(self.model.n, self.model.p,
                                                  self.config.max_iter, want_x)
        _check(self._L.pcal_session_finish(self._h, C.byref(rep)))
        return _report_from(rep, trace, stop_x, final_x)

    def profile(self, iters: int) -> dict:
        """Mean ms per iteration of each phase (CUDA events, no graphs)."""
        out = (C.c_double * 4)()
        _check(self._L.pcal_session_profile(self._h, iters, C.cast(out, _dp)))
        return {"step": out[0], "gradient": out[1], "gram": out[2], "xm": out[3]}

    def profile_kernels(self, iters: int) -> dict:
        """Mean ms per iteration of every kernel (event after each launch, no graphs)."""
        buf = C.create_string_buffer(1 << 16)
        _check(self._L.pcal_session_profile_kernels(self._h, iters, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms = line.split()
            out[name] = float(ms)
        return out

    @property
    def kernel_launches(self) -> int:
        return self._L.pcal_session_kernel_launches(self._h)

    @property
    def kernels_per_iteration(self) -> int:
        return self._L.pcal_session_kernels_per_iteration(self._h)

    def xm_mode(self) -> tuple:
        """("single_block" | "two_block", gated fallbacks so far): the form of the
        X·[W|C] product (pcal_session_xm_mode)."""
        fb = C.c_int64(0)
        m = self._L.pcal_session_xm_mode(self._h, C.byref(fb))
        return ("single_block" if m else "two_block", int(fb.value))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.pcal_session_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------- #
# building blocks (kernels.hpp, solver.hpp:74-113)
# --------------------------------------------------------------------------- #
def matmul_at_b(a, b, device: int = 0) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    if a.shape[0] != b.shape[0]:
        raise DimensionError("matmul_at_b: row counts do not agree")
    c = np.zeros((a.shape[1], b.shape[1]), order="F")
    _check(lib().pcal_matmul_at_b(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(c),
                                  device))
    return c


def matmul(a, b, device: int = 0) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionError("matmul: inner dimensions do not agree")
    c = np.zeros((a.shape[0], b.shape[1]), order="F")
    _check(lib().pcal_matmul(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(c),
                             device))
    return c


def gram(x, device: int = 0) -> np.ndarray:
    x = _f64(x)
    g = np.zeros((x.shape[1], x.shape[1]), order="F")
    _check(lib().pcal_gram(_ptr(x), x.shape[0], x.shape[1], _ptr(g), device))
    return g


def orthonormalize(x, device: int = 0) -> np.ndarray:
    x = _f64(x)
    q = np.zeros_like(x, order="F")
    _check(lib().pcal_orthonormalize(_ptr(x), x.shape[0], x.shape[1], _ptr(q), device))
    return q


def pcal_step(x, grad_l, eta: float, device: int = 0) -> tuple:
    x, g = _f64(x), _f64(grad_l)
    if x.shape != g.shape:
        raise DimensionError("pcal_step: shape mismatch")
    out = np.zeros_like(x, order="F")
    deg = C.c_int64()
    _check(lib().pcal_pcal_step(_ptr(x), _ptr(g), x.shape[0], x.shape[1], eta, _ptr(out),
                                C.byref(deg), device))
    return out, deg.value


def evaluate(model: _ModelBase, x, device: int = 0) -> tuple:
    x = _f64(x)
    cm, keep = model._c()
    f = C.c_double()
    g = np.zeros_like(x, order="F")
    _check(lib().pcal_evaluate(C.byref(cm), _ptr(x), C.byref(f), _ptr(g), device))
    del keep
    return f.value, g


def fd_gradient_check(model: _ModelBase, x, h: float = 1e-5, seed: int = 0x5EEDC0DE,
                      device: int = 0) -> float:
    """fd_gradient_check (problems.cpp:296-325) through the device evaluation."""
    x = _f64(x)
    cm, keep = model._c()
    w = C.c_double()
    _check(lib().pcal_fd_gradient_check(C.byref(cm), _ptr(x), h, seed, device, C.byref(w)))
    del keep
    return w.value


def spectral_norm_estimate(a, seed: int, device: int = 0) -> float:
    a = _f64(a)
    s = C.c_double()
    _check(lib().pcal_spectral_norm_estimate(_ptr(a), a.shape[0], seed, C.byref(s), device))
    return s.value


INIT_MODES = {"qr": 0, "a2-i": 1, "a2-ii": 2}  # InitMode (solver.hpp:47), harness names


ORTH_PATHS = {0: "cholqr2", 1: "mgs2-after-first", 2: "mgs2-after-second", -1: "rank"}


def last_orthonormalize_path() -> str:
    """Branch of orthonormalize (kernels.cpp:250-261) this thread's last device
    orthonormalisation took (diagnostic)."""
    return ORTH_PATHS[lib().pcal_last_orthonormalize_path()]


def initial_point(n: int, p: int, seed: int, device: int = 0, mode: str = "qr",
                  sigma_lower: float = 0.5) -> np.ndarray:
    """initial_point(InitialPointSpec{mode, sigma_lower, seed}, n, p)
    (solver.cpp:136-170): "qr", or the Assumption-A2 starts "a2-i" / "a2-ii"."""
    if mode not in INIT_MODES:
        raise ParameterError(f"initial_point: unknown mode {mode!r}")
    x = np.zeros((n, p), order="F")
    _check(lib().pcal_initial_point(n, p, INIT_MODES[mode], sigma_lower, seed, _ptr(x), device))
    return x


def random_normal(rows: int, cols: int, seed: int, threads: int = 8) -> np.ndarray:
    out = np.empty((rows, cols), order="F")
    _check(lib().pcal_random_normal(rows, cols, seed, _ptr(out), threads))
    return out


def spectral_norm_estimate_host(a, seed: int, threads: int = 8) -> float:
    """spectral_norm_estimate (kernels.cpp:267-293) on the host, bitwise the reference's."""
    a = _f64(a)
    s = C.c_double()
    _check(lib().pcal_spectral_norm_estimate_host(_ptr(a), a.shape[0], seed, threads, C.byref(s)))
    return s.value


def random_uniform(count: int, seed: int) -> np.ndarray:
    out = np.empty(count)
    _check(lib().pcal_random_uniform(count, seed, _ptr(out)))
    return out


def gen_dense_operator(n: int, seed: int, threads: int = 8) -> np.ndarray:
    """sym_part(random_normal(n, n, Rng(seed))) — configs 1–2 (problems.cpp:45-48)."""
    a = np.empty((n, n), order="F")
    _check(lib().pcal_gen_dense_operator(n, seed, _ptr(a), threads))
    return a


def flops_estimate(n: int, p: int) -> float:
    return lib().pcal_flops_estimate(n, p)


# --------------------------------------------------------------------------- #
# row-sharded multi-GPU
# --------------------------------------------------------------------------- #
def partition(model: _ModelBase, nranks: int, rank: int) -> tuple:
    """(row0, nrows) owned by `rank` of `nranks` (z-slabs / row blocks)."""
    cm, keep = model._c()
    r0, nr = C.c_int64(), C.c_int64()
    _check(lib().pcal_partition(C.byref(cm), nranks, rank, C.byref(r0), C.byref(nr)))
    return r0.value, nr.value


def _timed_call(timers, fn):
    tm = _Timers() if timers is not None else None
    fn(C.byref(tm) if tm is not None else None)
    if timers is not None:
        timers.blas3 += tm.blas3
        timers.func += tm.func
        timers.orth += tm.orth


def device_count() -> int:
    """Visible CUDA devices (0 without a GPU)."""
    c = C.c_int32()
    lib().pcal_device_count(C.byref(c))
    return c.value


def row_chunks(model: _ModelBase) -> tuple:
    """(rows per chunk, chunk count) of the sharded path's fixed row chunking."""
    cm, keep = model._c()
    q, nc = C.c_int64(), C.c_int64()
    _check(lib().pcal_row_chunks(C.byref(cm), C.byref(q), C.byref(nc)))
    return q.value, nc.value


def solve_emulated(model: _ModelBase, config: SolverConfig, x0, nranks: int,
                   timers: Optional[CategoryTimers] = None) -> RunReport:
    """The sharded algorithm with `nranks` emulated ranks on one GPU (loopback
    collectives); global host data in, global report out.  `timers` receives
    rank 0's blas3 / func / orth categories."""
    cm, keep = model._c()
    cc = config._c()
    x0 = _f64(x0)
    rep, trace, stop_x, final_x = _new_report(model.n, model.p, config.max_iter)
    _timed_call(timers, lambda t: _check(lib().pcal_solve_emulated(
        C.byref(cm), C.byref(cc), _ptr(x0), nranks, C.byref(rep), t)))
    return _report_from(rep, trace, stop_x, final_x)


def solve_sharded(model: _ModelBase, config: SolverConfig, x0_local, comm: "Comm",
                  n_local: int, timers: Optional[CategoryTimers] = None, out=None) -> RunReport:
    """Row-sharded pcal_solve on this rank (host buffers: local slabs in, local rows out)."""
    cm, keep = model._c()
    cc = config._c()
    x0_local = _f64(x0_local)
    rep, trace, stop_x, final_x = _new_report(n_local, model.p, config.max_iter, out=out)
    _timed_call(timers, lambda t: _check(lib().pcal_solve_sharded(
        C.byref(cm), C.byref(cc), _ptr(x0_local), HOST, comm._h, C.byref(rep), t)))
    return _report_from(rep, trace, stop_x, final_x)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().pcal_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """NCCL communicator of one rank (one process per GPU)."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes, device: int):
        self.nranks, self.rank = nranks, rank
        h = C.c_void_p()
        uid = C.create_string_buffer(bytes(unique_id), 128)
        _check(lib().pcal_comm_create_nccl(nranks, rank, uid, device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().pcal_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedSession(Session):
    """Session over the local rows of a row-sharded problem (model carries the
    global sizes and the LOCAL slabs; x0 = owned rows)."""

    def __init__(self, model: _ModelBase, config: SolverConfig, x0_local, comm: Comm,
                 n_local: int):
        self._L = lib()
        self.model, self.config = model, config
        self.n_local = n_local
        cm, self._keep = model._c()
        cc = config._c()
        ptr, loc, self._x0 = _x0_arg(x0_local)
        h = C.c_void_p()
        _check(self._L.pcal_session_create_sharded(C.byref(cm), C.byref(cc), ptr, loc, comm._h,
                                                   C.byref(h)))
        self._h = h

    def finish(self, want_x: bool = True) -> RunReport:
        rep, trace, stop_x, final_x = _new_report(self.n_local, self.model.p,
                                                  self.config.max_iter, want_x)
        _check(self._L.pcal_session_finish(self._h, C.byref(rep)))
        return _report_from(rep, trace, stop_x, final_x)
