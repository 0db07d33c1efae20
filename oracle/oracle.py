"""ctypes front-end to the parity CHECKERS (test infrastructure only).

Two back-ends with one API:

* ``Restatement`` — ``oracle/build/liboracle.so``, the C restatement of the
  reference PCAL path (``oracle/pcal_oracle.c``).
* ``Reference``   — ``oracle/_ref/libref_driver.so``, the unmodified reference
  core (``/root/reference/proj/core``) compiled from its own sources, driven
  through ``oracle/ref_driver.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module.  The product package never does.
Matrices are numpy float64 arrays in column-major (Fortran) order, the
reference's ``DenseMatrix`` layout (matrix.hpp:38-45).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "build", "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libref_driver.so")

TRACE_COLS = 7
MODEL_DENSE, MODEL_STENCIL, MODEL_KOHN_SHAM = 1, 2, 3
ETA_CONSTANT, ETA_DIFFERENTIAL, ETA_BB1, ETA_BB2, ETA_ABB = range(5)
MULT_PLAM, MULT_PCAL = 0, 1
ALG_PLAM, ALG_PCAL, ALG_ALM, ALG_MOPTQR, ALG_PLAMDA, ALG_PCALDA = range(6)
STATUS_NAMES = {0: "converged", 1: "max_iter", 2: "diverged"}
E_PARAM, E_DIM, E_RANK, E_EVAL, E_DIVERGE = -1, -2, -3, -4, -5

_dp = C.POINTER(C.c_double)


class OrcConfig(C.Structure):
    _fields_ = [("beta", C.c_double), ("eta_kind", C.c_int), ("gamma", C.c_double),
                ("eta_min", C.c_double), ("eta_max", C.c_double), ("eta0", C.c_double),
                ("multiplier_rule", C.c_int), ("tol_rel_kkt", C.c_double),
                ("max_iter", C.c_int64), ("threads", C.c_int), ("final_orth", C.c_int),
                ("algorithm", C.c_int)]


class OrcReport(C.Structure):
    _fields_ = [("trace", _dp), ("trace_len", C.c_int64), ("final_pre", C.c_double * 4),
                ("final_post", C.c_double * 4), ("has_post", C.c_int), ("stop_x", _dp),
                ("final_x", _dp), ("has_x", C.c_int), ("iterations", C.c_int64),
                ("degenerate_steps", C.c_int64), ("wall_time", C.c_double), ("status", C.c_int),
                ("beta_used", C.c_double), ("eta0_used", C.c_double),
                ("snap_iters", C.POINTER(C.c_int64)), ("nsnap", C.c_int), ("snaps", _dp),
                ("snap_eta", _dp)]


class OrcModel(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int64), ("p", C.c_int64), ("s", C.c_double),
                ("a", _dp), ("g0", _dp), ("nx", C.c_int64), ("ny", C.c_int64),
                ("nz", C.c_int64), ("v", _dp), ("work", C.c_void_p)]


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and (a.flags.f_contiguous or a.ndim == 1), "need F-order f64"
    return a.ctypes.data_as(_dp)


def fmat(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


@dataclass
class Model:
    """Problem descriptor shared by both back-ends (problems.hpp:28-111)."""
    kind: int
    n: int
    p: int
    s: float
    a: Optional[np.ndarray] = None      # dense n×n
    g0: Optional[np.ndarray] = None     # dense n×p
    grid: Sequence[int] = (0, 0, 0)
    v: Optional[np.ndarray] = None      # n


@dataclass
class Config:
    """SolverConfig (solver.hpp:13-42), PCAL algorithm."""
    beta: float = -1.0
    eta_kind: int = ETA_ABB
    gamma: float = 1.0
    eta_min: float = 1e-10
    eta_max: float = 1e10
    eta0: float = 0.0
    multiplier_rule: int = MULT_PCAL
    tol_rel_kkt: float = 1e-8
    max_iter: int = 3000
    threads: int = 1
    final_orth: bool = True
    algorithm: int = 1  # ALG_PCAL

    def c(self) -> OrcConfig:
        return OrcConfig(self.beta, self.eta_kind, self.gamma, self.eta_min, self.eta_max,
                         self.eta0, self.multiplier_rule, self.tol_rel_kkt, self.max_iter,
                         self.threads, int(self.final_orth), self.algorithm)


@dataclass
class Report:
    trace: np.ndarray
    final_pre: np.ndarray
    final_post: Optional[np.ndarray]
    stop_x: Optional[np.ndarray]
    final_x: Optional[np.ndarray]
    iterations: int
    degenerate_steps: int
    wall_time: float
    status: str
    beta: float
    eta0: float
    snaps: dict = field(default_factory=dict)
    snap_eta: dict = field(default_factory=dict)
    timers: Optional[np.ndarray] = None


def ensure_built() -> None:
    """Build the checkers with oracle/Makefile (reference part only if present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Base:
    lib: C.CDLL

    def _report(self, model: Model, cfg: Config, snaps: Sequence[int]) -> tuple:
        n, p = model.n, model.p
        trace = np.zeros((cfg.max_iter + 1, TRACE_COLS))
        stop_x = np.zeros((n, p), order="F")
        final_x = np.zeros((n, p), order="F")
        rep = OrcReport()
        rep.trace = trace.ctypes.data_as(_dp)
        rep.stop_x = _ptr(stop_x)
        rep.final_x = _ptr(final_x)
        keep = [trace, stop_x, final_x]
        if snaps:
            it = np.asarray(snaps, dtype=np.int64)
            buf = np.zeros((len(snaps), p, n))
            etas = np.zeros(len(snaps))
            rep.snap_iters = it.ctypes.data_as(C.POINTER(C.c_int64))
            rep.nsnap = len(snaps)
            rep.snaps = buf.ctypes.data_as(_dp)
            rep.snap_eta = etas.ctypes.data_as(_dp)
            keep += [it, buf, etas]
        return rep, keep

    @staticmethod
    def _finish(rep: OrcReport, keep, snaps) -> Report:
        trace, stop_x, final_x = keep[:3]
        out = Report(
            trace=trace[: rep.trace_len].copy(),
            final_pre=np.array(rep.final_pre[:]),
            final_post=np.array(rep.final_post[:]) if rep.has_post else None,
            stop_x=stop_x if rep.has_x else None,
            final_x=final_x if rep.has_x else None,
            iterations=rep.iterations, degenerate_steps=rep.degenerate_steps,
            wall_time=rep.wall_time, status=STATUS_NAMES[rep.status], beta=rep.beta_used,
            eta0=rep.eta0_used)
        if snaps:
            buf, etas = keep[4], keep[5]
            for q, k in enumerate(snaps):
                out.snaps[int(k)] = np.asfortranarray(buf[q].T)
                out.snap_eta[int(k)] = float(etas[q])
        return out


class Restatement(_Base):
    """The C restatement (oracle/pcal_oracle.c)."""
    kind = "port"

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            ensure_built()
        L = self.lib = C.CDLL(path)
        i64, dbl, u64 = C.c_int64, C.c_double, C.c_uint64
        L.orc_random_normal.argtypes = [i64, u64, _dp, C.c_int]
        L.orc_random_uniform.argtypes = [i64, u64, _dp]
        L.orc_sym_part.argtypes = [_dp, i64, _dp]
        L.orc_matmul.argtypes = [_dp, i64, i64, _dp, i64, _dp, C.c_int]
        L.orc_matmul_at_b.argtypes = [_dp, i64, i64, _dp, i64, _dp, C.c_int]
        L.orc_gram.argtypes = [_dp, i64, i64, _dp, C.c_int]
        L.orc_orthonormalize.argtypes = [_dp, i64, i64, _dp]
        L.orc_mgs2.argtypes = [_dp, i64, i64, dbl, _dp]
        L.orc_spectral_norm_estimate.argtypes = [_dp, i64, u64, C.c_int]
        L.orc_spectral_norm_estimate.restype = dbl
        L.orc_model_prepare.argtypes = [C.POINTER(OrcModel)]
        L.orc_model_release.argtypes = [C.POINTER(OrcModel)]
        L.orc_evaluate.argtypes = [C.POINTER(OrcModel), _dp, _dp, _dp, C.c_int]
        L.orc_laplacian_apply.argtypes = [_dp, i64, i64, i64, i64, _dp]
        L.orc_pseudo_inverse_laplacian.argtypes = [C.POINTER(OrcModel), _dp, _dp]
        L.orc_fourier_basis.argtypes = [i64, _dp, _dp]
        L.orc_fd_gradient_check.argtypes = [C.POINTER(OrcModel), _dp, dbl, u64]
        L.orc_fd_gradient_check.restype = dbl
        L.orc_solve_pcal.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcConfig), _dp,
                                     C.POINTER(OrcReport)]
        L.orc_solve.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcConfig), _dp,
                                C.POINTER(OrcReport)]
        L.orc_stepsize_select.argtypes = [C.POINTER(OrcConfig), i64, dbl, dbl, _dp, _dp, _dp,
                                          _dp, i64]
        L.orc_stepsize_select.restype = dbl
        L.orc_pcal_step.argtypes = [_dp, _dp, i64, i64, dbl, _dp, C.POINTER(i64), C.c_int]
        L.orc_pcal_grad_l.argtypes = [C.POINTER(OrcModel), _dp, dbl, C.c_int, _dp, _dp, _dp, _dp,
                                      C.c_int]
        L.orc_flops_estimate_pcal.argtypes = [i64, i64]
        L.orc_flops_estimate_pcal.restype = dbl

    # -- models ------------------------------------------------------------
    def _cmodel(self, m: Model) -> tuple:
        om = OrcModel(m.kind, m.n, m.p, m.s, _ptr(m.a), _ptr(m.g0), m.grid[0], m.grid[1],
                      m.grid[2], _ptr(m.v), None)
        rc = self.lib.orc_model_prepare(C.byref(om))
        if rc:
            raise ValueError(f"orc_model_prepare failed ({rc})")
        return om

    def _release(self, om: OrcModel) -> None:
        self.lib.orc_model_release(C.byref(om))

    # -- setup ---------------------------------------------------------------
    def random_normal(self, rows: int, cols: int, seed: int, threads: int = 1) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        self.lib.orc_random_normal(rows * cols, seed, _ptr(out), threads)
        return out

    def random_uniform(self, count: int, seed: int) -> np.ndarray:
        out = np.empty(count)
        self.lib.orc_random_uniform(count, seed, _ptr(out))
        return out

    def sym_part(self, m: np.ndarray) -> np.ndarray:
        m = fmat(m)
        out = np.empty_like(m, order="F")
        self.lib.orc_sym_part(_ptr(m), m.shape[0], _ptr(out))
        return out

    def spectral_norm_estimate(self, a: np.ndarray, seed: int, threads: int = 1) -> float:
        a = fmat(a)
        return self.lib.orc_spectral_norm_estimate(_ptr(a), a.shape[0], seed, threads)

    def orthonormalize(self, x: np.ndarray) -> np.ndarray:
        x = fmat(x)
        q = np.empty_like(x, order="F")
        rc = self.lib.orc_orthonormalize(_ptr(x), x.shape[0], x.shape[1], _ptr(q))
        if rc == E_RANK:
            raise np.linalg.LinAlgError("orthonormalize: numerically rank-deficient input")
        return q

    def mgs2(self, x, floor: float) -> np.ndarray:
        """mgs2 (kernels.cpp:212-246), the fallback of orthonormalize."""
        x = fmat(x)
        q = np.empty_like(x, order="F")
        if self.lib.orc_mgs2(_ptr(x), x.shape[0], x.shape[1], floor, _ptr(q)) == E_RANK:
            raise np.linalg.LinAlgError("mgs2: numerically rank-deficient input")
        return q

    def initial_point_qr(self, n: int, p: int, seed: int, threads: int = 1) -> np.ndarray:
        """initial_point({Qr}, n, p) (solver.cpp:136-142)."""
        return self.orthonormalize(self.random_normal(n, p, seed, threads))

    def dense_trace_min(self, n: int, p: int, seed: int, s: Optional[float] = None,
                        threads: int = 1) -> Model:
        """gen_problem1(α=0, RandomSym) ≡ make_quadratic (probe 5)."""
        a = self.sym_part(self.random_normal(n, n, seed, threads))
        if s is None:
            s = self.spectral_norm_estimate(a, seed ^ 0x73706563, threads)
        return Model(MODEL_DENSE, n, p, float(s), a=a)

    # -- kernels -------------------------------------------------------------
    def matmul(self, a, b, threads: int = 1) -> np.ndarray:
        a, b = fmat(a), fmat(b)
        c = np.empty((a.shape[0], b.shape[1]), order="F")
        self.lib.orc_matmul(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c), threads)
        return c

    def matmul_at_b(self, a, b, threads: int = 1) -> np.ndarray:
        a, b = fmat(a), fmat(b)
        c = np.empty((a.shape[1], b.shape[1]), order="F")
        self.lib.orc_matmul_at_b(_ptr(a), a.shape[0], a.shape[1], _ptr(b), b.shape[1], _ptr(c),
                                 threads)
        return c

    def gram(self, x, threads: int = 1) -> np.ndarray:
        x = fmat(x)
        g = np.empty((x.shape[1], x.shape[1]), order="F")
        self.lib.orc_gram(_ptr(x), x.shape[0], x.shape[1], _ptr(g), threads)
        return g

    def laplacian(self, x, grid) -> np.ndarray:
        x = fmat(x)
        out = np.empty_like(x, order="F")
        self.lib.orc_laplacian_apply(_ptr(x), grid[0], grid[1], grid[2], x.shape[1], _ptr(out))
        return out

    def pinv_laplacian(self, model: Model, rho: np.ndarray) -> np.ndarray:
        om = self._cmodel(model)
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        out = np.empty_like(rho)
        try:
            self.lib.orc_pseudo_inverse_laplacian(C.byref(om), _ptr(rho), _ptr(out))
        finally:
            self._release(om)
        return out

    def fourier_basis(self, N: int) -> tuple:
        q = np.empty((N, N), order="F")
        lam = np.empty(N)
        self.lib.orc_fourier_basis(N, _ptr(q), _ptr(lam))
        return q, lam

    def evaluate(self, model: Model, x, threads: int = 1) -> tuple:
        x = fmat(x)
        om = self._cmodel(model)
        f = C.c_double()
        g = np.empty_like(x, order="F")
        try:
            rc = self.lib.orc_evaluate(C.byref(om), _ptr(x), C.byref(f), _ptr(g), threads)
        finally:
            self._release(om)
        if rc == E_EVAL:
            raise FloatingPointError("evaluation_error: non-finite objective or gradient")
        return f.value, g

    def fd_gradient_check(self, model: Model, x, h: float = 1e-5, seed: int = 0x5EEDC0DE) -> float:
        x = fmat(x)
        om = self._cmodel(model)
        try:
            return self.lib.orc_fd_gradient_check(C.byref(om), _ptr(x), h, seed)
        finally:
            self._release(om)

    def pcal_grad_l(self, model: Model, x, beta: float = 1.0, mult: int = MULT_PCAL,
                    threads: int = 1) -> tuple:
        x = fmat(x)
        om = self._cmodel(model)
        gl = np.empty_like(x, order="F")
        f, k, fe = C.c_double(), C.c_double(), C.c_double()
        try:
            rc = self.lib.orc_pcal_grad_l(C.byref(om), _ptr(x), beta, mult, _ptr(gl), C.byref(f),
                                          C.byref(k), C.byref(fe), threads)
        finally:
            self._release(om)
        if rc:
            raise FloatingPointError(f"pcal_grad_l failed ({rc})")
        return gl, f.value, k.value, fe.value

    def stepsize_select(self, cfg: Config, it: int, eta_prev: float, eta0: float, x, xp, gl,
                        glp) -> float:
        x, gl = fmat(x), fmat(gl)
        xp = fmat(xp) if xp is not None else None
        glp = fmat(glp) if glp is not None else None
        c = cfg.c()
        return self.lib.orc_stepsize_select(C.byref(c), it, eta_prev, eta0, _ptr(x), _ptr(xp),
                                            _ptr(gl), _ptr(glp), x.size)

    def pcal_step(self, x, gl, eta: float, threads: int = 1) -> tuple:
        x, gl = fmat(x), fmat(gl)
        out = np.empty_like(x, order="F")
        deg = C.c_int64()
        rc = self.lib.orc_pcal_step(_ptr(x), _ptr(gl), x.shape[0], x.shape[1], eta, _ptr(out),
                                    C.byref(deg), threads)
        if rc == E_PARAM:
            raise ValueError("pcal_step: eta must be positive")
        if rc == E_DIVERGE:
            raise FloatingPointError("divergence_error: non-finite iterate")
        return out, deg.value

    def flops_estimate_pcal(self, n: int, p: int) -> float:
        return self.lib.orc_flops_estimate_pcal(n, p)

    # -- solve ---------------------------------------------------------------
    def solve(self, model: Model, cfg: Config, x0, snaps: Sequence[int] = ()) -> Report:
        x0 = fmat(x0)
        om = self._cmodel(model)
        c = cfg.c()
        rep, keep = self._report(model, cfg, snaps)
        try:
            rc = self.lib.orc_solve(C.byref(om), C.byref(c), _ptr(x0), C.byref(rep))
        finally:
            self._release(om)
        if rc == E_PARAM:
            raise ValueError("parameter_error")
        if rc:
            raise RuntimeError(f"orc_solve failed ({rc})")
        return self._finish(rep, keep, snaps)


class Reference(_Base):
    """The unmodified reference core (oracle/_ref/libref_driver.so)."""
    kind = "reference"

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            ensure_built()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (reference sources absent at build time)")
        L = self.lib = C.CDLL(path)
        i64, dbl, u64, vp = C.c_int64, C.c_double, C.c_uint64, C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_dense_trace_min.argtypes = [i64, i64, u64, dbl, C.c_int, _dp, _dp]
        L.ref_make_dense_trace_min.restype = vp
        L.ref_make_quadratic.argtypes = [_dp, _dp, i64, i64, dbl]
        L.ref_make_quadratic.restype = vp
        L.ref_make_grid_model.argtypes = [C.c_int, i64, i64, i64, i64, _dp, dbl]
        L.ref_make_grid_model.restype = vp
        L.ref_free_model.argtypes = [vp]
        L.ref_evaluate.argtypes = [vp, _dp, _dp, _dp]
        L.ref_fd_gradient_check.argtypes = [vp, _dp, dbl, u64]
        L.ref_fd_gradient_check.restype = dbl
        L.ref_random_normal.argtypes = [i64, i64, u64, _dp]
        L.ref_initial_point.argtypes = [C.c_int, dbl, u64, i64, i64, _dp]
        L.ref_spectral_norm_estimate.argtypes = [_dp, i64, u64, C.c_int]
        L.ref_spectral_norm_estimate.restype = dbl
        L.ref_orthonormalize.argtypes = [_dp, i64, i64, _dp]
        L.ref_gram.argtypes = [_dp, i64, i64, _dp]
        L.ref_matmul_at_b.argtypes = [_dp, _dp, i64, i64, i64, _dp]
        L.ref_matmul.argtypes = [_dp, _dp, i64, i64, i64, _dp, C.c_int]
        L.ref_pcal_step.argtypes = [_dp, _dp, i64, i64, dbl, _dp, C.POINTER(i64)]
        L.ref_stepsize_select.argtypes = [C.POINTER(OrcConfig), i64, dbl, dbl, _dp, _dp, _dp, _dp,
                                          i64, i64]
        L.ref_stepsize_select.restype = dbl
        L.ref_kkt_violation.argtypes = [vp, _dp]
        L.ref_kkt_violation.restype = dbl
        L.ref_feasibility_violation.argtypes = [_dp, i64, i64]
        L.ref_feasibility_violation.restype = dbl
        L.ref_flops_estimate_pcal.argtypes = [i64, i64]
        L.ref_flops_estimate_pcal.restype = dbl
        L.ref_solve.argtypes = [vp, C.POINTER(OrcConfig), _dp, C.POINTER(OrcReport), _dp]

    def _err(self) -> str:
        return self.lib.ref_last_error().decode()

    def _handle(self, m: Model):
        if m.kind == MODEL_DENSE:
            h = self.lib.ref_make_quadratic(_ptr(fmat(m.a)), _ptr(m.g0), m.n, m.p, m.s)
        else:
            v = np.ascontiguousarray(m.v, dtype=np.float64)
            h = self.lib.ref_make_grid_model(m.kind, m.grid[0], m.grid[1], m.grid[2], m.p,
                                             _ptr(v), m.s)
        if not h:
            raise RuntimeError(self._err())
        return h

    def random_normal(self, rows: int, cols: int, seed: int) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        self.lib.ref_random_normal(rows, cols, seed, _ptr(out))
        return out

    def initial_point_qr(self, n: int, p: int, seed: int) -> np.ndarray:
        out = np.empty((n, p), order="F")
        rc = self.lib.ref_initial_point(0, 0.5, seed, n, p, _ptr(out))
        if rc:
            raise RuntimeError(self._err())
        return out

    def dense_trace_min(self, n: int, p: int, seed: int, s: Optional[float] = None,
                        threads: int = 1) -> Model:
        a = np.empty((n, n), order="F")
        s_out = C.c_double()
        h = self.lib.ref_make_dense_trace_min(n, p, seed, -1.0 if s is None else s, threads,
                                              _ptr(a), C.byref(s_out))
        if not h:
            raise RuntimeError(self._err())
        self.lib.ref_free_model(h)
        return Model(MODEL_DENSE, n, p, s_out.value, a=a)

    def spectral_norm_estimate(self, a, seed: int, threads: int = 1) -> float:
        a = fmat(a)
        return self.lib.ref_spectral_norm_estimate(_ptr(a), a.shape[0], seed, threads)

    def orthonormalize(self, x) -> np.ndarray:
        x = fmat(x)
        q = np.empty_like(x, order="F")
        rc = self.lib.ref_orthonormalize(_ptr(x), x.shape[0], x.shape[1], _ptr(q))
        if rc == E_RANK:
            raise np.linalg.LinAlgError(self._err())
        return q

    def gram(self, x) -> np.ndarray:
        x = fmat(x)
        g = np.empty((x.shape[1], x.shape[1]), order="F")
        self.lib.ref_gram(_ptr(x), x.shape[0], x.shape[1], _ptr(g))
        return g

    def matmul_at_b(self, a, b) -> np.ndarray:
        a, b = fmat(a), fmat(b)
        c = np.empty((a.shape[1], b.shape[1]), order="F")
        self.lib.ref_matmul_at_b(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(c))
        return c

    def matmul(self, a, b, threads: int = 1) -> np.ndarray:
        a, b = fmat(a), fmat(b)
        c = np.empty((a.shape[0], b.shape[1]), order="F")
        self.lib.ref_matmul(_ptr(a), _ptr(b), a.shape[0], a.shape[1], b.shape[1], _ptr(c), threads)
        return c

    def evaluate(self, model: Model, x) -> tuple:
        x = fmat(x)
        h = self._handle(model)
        f = C.c_double()
        g = np.empty_like(x, order="F")
        try:
            rc = self.lib.ref_evaluate(h, _ptr(x), C.byref(f), _ptr(g))
        finally:
            self.lib.ref_free_model(h)
        if rc == E_EVAL:
            raise FloatingPointError(self._err())
        return f.value, g

    def fd_gradient_check(self, model: Model, x, h: float = 1e-5, seed: int = 0x5EEDC0DE) -> float:
        x = fmat(x)
        hd = self._handle(model)
        try:
            return self.lib.ref_fd_gradient_check(hd, _ptr(x), h, seed)
        finally:
            self.lib.ref_free_model(hd)

    def pcal_step(self, x, gl, eta: float) -> tuple:
        x, gl = fmat(x), fmat(gl)
        out = np.empty_like(x, order="F")
        deg = C.c_int64()
        rc = self.lib.ref_pcal_step(_ptr(x), _ptr(gl), x.shape[0], x.shape[1], eta, _ptr(out),
                                    C.byref(deg))
        if rc == E_PARAM:
            raise ValueError(self._err())
        if rc == E_DIVERGE:
            raise FloatingPointError(self._err())
        return out, deg.value

    def stepsize_select(self, cfg: Config, it: int, eta_prev: float, eta0: float, x, xp, gl,
                        glp) -> float:
        x, gl = fmat(x), fmat(gl)
        xp = fmat(xp) if xp is not None else None
        glp = fmat(glp) if glp is not None else None
        c = cfg.c()
        return self.lib.ref_stepsize_select(C.byref(c), it, eta_prev, eta0, _ptr(x), _ptr(xp),
                                            _ptr(gl), _ptr(glp), x.shape[0], x.shape[1])

    def kkt_violation(self, model: Model, x) -> float:
        h = self._handle(model)
        try:
            return self.lib.ref_kkt_violation(h, _ptr(fmat(x)))
        finally:
            self.lib.ref_free_model(h)

    def feasibility_violation(self, x) -> float:
        x = fmat(x)
        return self.lib.ref_feasibility_violation(_ptr(x), x.shape[0], x.shape[1])

    def flops_estimate_pcal(self, n: int, p: int) -> float:
        return self.lib.ref_flops_estimate_pcal(n, p)

    def solve(self, model: Model, cfg: Config, x0, with_timers: bool = False) -> Report:
        x0 = fmat(x0)
        h = self._handle(model)
        c = cfg.c()
        rep, keep = self._report(model, cfg, ())
        timers = np.zeros(3)
        try:
            rc = self.lib.ref_solve(h, C.byref(c), _ptr(x0), C.byref(rep),
                                    _ptr(timers) if with_timers else None)
        finally:
            self.lib.ref_free_model(h)
        if rc == E_PARAM:
            raise ValueError(self._err())
        if rc:
            raise RuntimeError(f"ref_solve failed ({rc}): {self._err()}")
        out = self._finish(rep, keep, ())
        out.timers = timers if with_timers else None
        return out


def available_reference() -> bool:
    return os.path.exists(LIB_REF)
