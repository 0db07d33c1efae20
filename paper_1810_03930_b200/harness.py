"""The reference harness's single-run entry point on the device path.

``run_single(ProblemSpec, SolverConfig, InitialPointSpec)`` (harness.cpp:62-73,
harness.hpp:16-33): generate the seeded instance, build the start point, solve,
and echo the cell configuration into the report (``fill_config_echo``,
harness.cpp:48-60).  The problem kinds whose model is the dense quadratic are
generated here with the reference's random stream and solved on the B200:

* P1 with α = 0 — ``DensityModel`` degenerates to ½tr(XᵀLX) (problems.cpp:166-206);
  L = ``gen_operator`` (problems.cpp:32-48): ``sym_part(random_normal)`` or the
  5×5 block-tridiagonal operator;
* P2 / P3 — ``gen_problem2`` / ``gen_problem3`` (problems.cpp:219-265): an
  eigenbasis from the orthonormalised uniform matrix, eigenvalues ±θ^{−i} with a
  ξ-biased sign coin, linear-term columns of norm κ·ζ^j (κ = 0 for P3).
  The basis and the product are formed on the device, so the instance agrees
  with the reference's to rounding, not bitwise.

* P1 with α > 0 and P6 — ``DensityModel`` (problems.cpp:158-206, 208-217,
  276-285): L = ``gen_operator``, the Hartree solve through L⁻¹ formed by the
  reference's LinearSolver; P6 takes γ = 2·(3/π)^{1/3};
* P4 — ``gen_problem4`` (problems.cpp:267-274): A = sym_part(random_normal(n, n)),
  B = sym_part(random_normal(p, p)) from one stream, s = s_A·s_B.

The instances of P1, P4 and P6 are bitwise the reference's.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

import paper_1810_03930_b200 as P
from paper_1810_03930_b200.report_io import ConfigEcho, UnsupportedModel, eta_rule_name

INIT_SALT = 0x1235713       # harness.cpp:18 init_seed
SPECTRAL_SALT = 0x73706563  # problems.cpp:19 kSpectralSalt


@dataclass
class ProblemSpec:
    """ProblemSpec (harness.hpp:16-24)."""
    kind: str = "p2"            # "p1" | "p2" | "p3" | "p4" | "p6"
    n: int = 100
    p: int = 5
    alpha: float = 1.0          # p1
    kappa: float = 1.0          # p2
    theta: float = 1.01
    zeta: float = 1.01
    xi: float = 1.0
    mode: str = "random-sym"    # p1/p6 operator: "random-sym" | "block-tridiag"
    seed: int = 0


@dataclass
class InitialPointSpec:
    """InitialPointSpec (solver.hpp:53-57); seed 0 ⇒ init_seed(problem.seed)."""
    mode: str = "qr"            # "qr" | "a2-i" | "a2-ii"
    sigma_lower: float = 0.5
    seed: int = 0


def _require_stiefel(n: int, p: int) -> None:
    if n < 1 or p < 1 or 2 * p > n:  # require_stiefel_dims (problems.cpp)
        raise P.ParameterError("problem: dimensions must satisfy 2p <= n")


def _operator(spec: ProblemSpec, device: int) -> np.ndarray:
    """gen_operator (problems.cpp:32-48)."""
    n = spec.n
    if spec.mode == "block-tridiag":
        if n % 5:
            raise P.ParameterError(f"block operator mode requires n divisible by 5, got n={n}")
        a = np.zeros((n, n), order="F")
        for b in range(0, n, 5):
            for i in range(5):
                a[b + i, b + i] = 2.0
                if i + 1 < 5:
                    a[b + i, b + i + 1] = a[b + i + 1, b + i] = -1.0
        return a
    if spec.mode != "random-sym":
        raise P.ParameterError(f"unknown operator mode {spec.mode!r}")
    return P.gen_dense_operator(n, spec.seed)


def _quadratic_p2(spec: ProblemSpec, device: int) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """gen_problem2 (problems.cpp:219-258): A = sym(P·diag(λ)·Pᵀ), G = scaled uniforms."""
    n, p = spec.n, spec.p
    if spec.theta < 1.0 or spec.zeta < 1.0:
        raise P.ParameterError("gen_problem2: theta and zeta must be at least 1")
    if spec.kappa < 0.0:
        raise P.ParameterError("gen_problem2: kappa must be nonnegative")
    if spec.xi < 0.0 or spec.xi > 1.0:
        raise P.ParameterError("gen_problem2: xi must lie in [0,1]")
    # one stream: n² uniforms for the basis, n sign coins, n·p uniforms for G
    u = P.random_uniform(n * n + n + n * p, spec.seed)
    basis = P.orthonormalize(np.asfortranarray(u[: n * n].reshape((n, n), order="F")),
                             device=device)
    coins = u[n * n: n * n + n]
    mag = spec.theta ** (-np.arange(n, dtype=np.float64))
    lam = np.where(coins < spec.xi, mag, -mag)
    pl = np.asfortranarray(basis * lam[None, :])
    m = P.matmul(pl, np.asfortranarray(basis.T), device=device)
    a = np.asfortranarray(0.5 * (m + m.T))  # sym_part
    g = np.asfortranarray(u[n * n + n:].reshape((n, p), order="F"))
    nrm = np.linalg.norm(g, axis=0)
    scale = np.where(nrm > 0.0, spec.kappa * spec.zeta ** np.arange(p, dtype=np.float64) / nrm, 0.0)
    g = np.asfortranarray(g * scale[None, :])
    return a, (g if spec.kappa != 0.0 else None)


def make_problem(spec: ProblemSpec, device: int = 0):
    """make_problem (harness.cpp:31-46) for the device-evaluated kinds."""
    _require_stiefel(spec.n, spec.p)
    kind = spec.kind.lower()
    if kind == "p1":
        if spec.alpha < 0.0:
            raise P.ParameterError("gen_problem1: alpha must be nonnegative")
        a = _operator(spec, device)
        g0 = None
        if spec.alpha != 0.0:  # gen_problem1 (problems.cpp:208-217)
            s = P.spectral_norm_estimate_host(a, spec.seed ^ SPECTRAL_SALT)
            return P.DensityModel(a, spec.p, spec.alpha, s, variant="p1", mode=spec.mode)
    elif kind == "p6":  # gen_problem6 (problems.cpp:276-285)
        a = _operator(spec, device)
        s = P.spectral_norm_estimate_host(a, spec.seed ^ SPECTRAL_SALT)
        gamma = 2.0 * np.cbrt(3.0 / 3.14159265358979323846)
        return P.DensityModel(a, spec.p, gamma, s, variant="p6", mode=spec.mode)
    elif kind == "p4":  # gen_problem4 (problems.cpp:267-274): A then B from one stream
        n, p = spec.n, spec.p
        z = P.random_normal(n * n + p * p, 1, spec.seed)[:, 0]
        an = z[: n * n].reshape((n, n), order="F")
        bn = z[n * n:].reshape((p, p), order="F")
        a = np.asfortranarray(0.5 * (an + an.T))
        b = np.asfortranarray(0.5 * (bn + bn.T))
        sa = P.spectral_norm_estimate_host(a, spec.seed ^ SPECTRAL_SALT)
        sb = P.spectral_norm_estimate_host(b, spec.seed ^ (SPECTRAL_SALT + 1))
        return P.BilinearModel(a, b, sa * sb)
    elif kind in ("p2", "p3"):
        if kind == "p3":  # gen_problem3 = gen_problem2(κ = 0, ζ = 1)
            spec = ProblemSpec(**{**spec.__dict__, "kappa": 0.0, "zeta": 1.0})
        a, g0 = _quadratic_p2(spec, device)
    else:
        raise UnsupportedModel(f"problem kind {spec.kind!r} has no device model here")
    s = P.spectral_norm_estimate_host(a, spec.seed ^ SPECTRAL_SALT)  # bitwise the reference's
    return P.QuadraticModel(a, spec.p, s, g0=g0)


def run_single(problem: ProblemSpec, config: P.SolverConfig,
               init: InitialPointSpec = InitialPointSpec(),
               timers: Optional[P.CategoryTimers] = None) -> Tuple[P.RunReport, ConfigEcho]:
    """run_single (harness.cpp:62-73): the report and its configuration echo."""
    t0 = time.perf_counter()
    model = make_problem(problem, device=config.device)
    seed = init.seed if init.seed != 0 else problem.seed ^ INIT_SALT
    x0 = P.initial_point(problem.n, problem.p, seed, device=config.device, mode=init.mode,
                         sigma_lower=init.sigma_lower)
    rep = P.solve(model, config, x0, timers=timers)
    echo = ConfigEcho(problem=problem.kind.lower(), n=problem.n, p=problem.p,
                      solver=config.algorithm, beta=rep.beta, eta_rule=eta_rule_name(config.eta_rule),
                      tol_rel_kkt=config.tol_rel_kkt, max_iter=config.max_iter, threads=1,
                      init=init.mode, seed=problem.seed, alpha=problem.alpha, kappa=problem.kappa,
                      theta=problem.theta, zeta=problem.zeta, xi=problem.xi,
                      curvature_scale=model.s)
    rep.wall_time = time.perf_counter() - t0
    return rep, echo


@dataclass
class MatrixSpec:
    """MatrixSpec (harness.hpp:35-43): problems × solvers × seeds."""
    problems: list
    solvers: list                      # algorithm names ("pcal", "plam", "alm", ...)
    seeds: list
    base: Optional[P.SolverConfig] = None  # algorithm overridden per cell
    init: str = "qr"
    sigma_lower: float = 0.5


def run_matrix(spec: MatrixSpec, csv_out) -> None:
    """run_matrix (harness.cpp:75-104): one summary CSV row per cell; a cell whose
    generation fails is recorded as diverged and never aborts the matrix."""
    import dataclasses
    import sys
    from paper_1810_03930_b200 import report_io as R
    if not spec.problems or not spec.solvers or not spec.seeds:
        raise P.ParameterError("run_matrix: empty problem/solver/seed list")
    base = spec.base if spec.base is not None else P.SolverConfig()
    R.write_summary_header(csv_out)
    for prob in spec.problems:
        for alg in spec.solvers:
            for seed in spec.seeds:
                cell = dataclasses.replace(prob, seed=seed)
                cfg = dataclasses.replace(base, algorithm=alg)
                init = InitialPointSpec(mode=spec.init, sigma_lower=spec.sigma_lower)
                try:
                    rep, echo = run_single(cell, cfg, init)
                except (P.ParameterError, P.DimensionError, P.RankError, UnsupportedModel,
                        ValueError) as e:
                    sys.stderr.write(f"cell {cell.kind}/{alg}/{seed} failed: {e}\n")
                    rep = P.RunReport(trace=np.zeros((0, 7)),
                                      final_pre_orth=P.FinalMetrics(0.0, 0.0, 0.0, 0.0),
                                      final_post_orth=None, stop_iterate=None, final_x=None,
                                      iterations=0, degenerate_steps=0, wall_time=0.0,
                                      status="diverged", beta=0.0, eta0=0.0)
                    # fill_config_echo + the solver name; beta / eta_rule stay unset
                    echo = R.ConfigEcho(problem=cell.kind.lower(), n=cell.n, p=cell.p, solver=alg,
                                        beta=0.0, eta_rule="", tol_rel_kkt=0.0, max_iter=0,
                                        init=spec.init, seed=seed, alpha=cell.alpha,
                                        kappa=cell.kappa, theta=cell.theta, zeta=cell.zeta,
                                        xi=cell.xi)
                R.write_summary_row(rep, echo, csv_out)
