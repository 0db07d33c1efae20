"""The reference's diagnostics (diagnostics.hpp / diagnostics.cpp:21-98) on the
device: every n×p product (the gradient, GᵀX, XᵀX, GᵀG, X·W) is a DMMA GEMM
through the C ABI; only p×p quantities are finished on the host — the power
iterations for the spectral bounds use the reference's own
``spectral_norm_estimate`` (bitwise, ``spectral_norm_estimate_host``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import paper_1810_03930_b200 as P

_SEED_LMAX, _SEED_LMIN, _SEED_GRAD = 0x5CA1E, 0x5CA1F, 0x5CA20  # diagnostics.cpp:65-76


def _sym(m: np.ndarray) -> np.ndarray:
    return 0.5 * (m + m.T)  # sym_part: (m_ij + m_ji)/2, the same value on both sides


def _c_of(x, device: int) -> np.ndarray:
    c = P.gram(x, device=device)
    return c - np.eye(c.shape[0])


def kkt_violation_grad(grad_f, x, device: int = 0) -> float:
    """‖G − X·Ψ(GᵀX)‖_F (diagnostics.cpp:21-26)."""
    g, x = P._f64(grad_f), P._f64(x)
    if g.shape != x.shape:
        raise P.DimensionError("kkt_violation: shape mismatch")
    w = _sym(P.matmul_at_b(g, x, device=device))
    return float(np.linalg.norm(g - P.matmul(x, np.asfortranarray(w), device=device)))


def kkt_violation(model, x, device: int = 0) -> float:
    """kkt_violation(model, X) (diagnostics.cpp:28-30)."""
    _, g = P.evaluate(model, x, device=device)
    return kkt_violation_grad(g, x, device=device)


def feasibility_violation(x, device: int = 0) -> float:
    """‖XᵀX − I‖_F (diagnostics.cpp:32-36)."""
    return float(np.linalg.norm(_c_of(P._f64(x), device)))


def merit_h(model, x, beta: float, device: int = 0) -> float:
    """f(X) − ½⟨Ψ(GᵀX), XᵀX − I⟩ + β/4‖XᵀX − I‖² (diagnostics.cpp:38-47)."""
    x = P._f64(x)
    f, g = P.evaluate(model, x, device=device)
    w = _sym(P.matmul_at_b(g, x, device=device))
    c = _c_of(x, device)
    return float(f - 0.5 * np.sum(w * c) + 0.25 * beta * np.sum(c * c))


@dataclass
class FeasibilityBoundResult:
    """FeasibilityBoundResult (diagnostics.hpp:31-38)."""
    applicable: bool = False
    delta: float = 0.0
    lhs: float = 0.0
    rhs: float = 0.0
    holds: bool = False
    slack: float = 0.0


def feasibility_bound_check(model, x, beta: float, device: int = 0) -> FeasibilityBoundResult:
    """Lemma-2 feasibility bound (diagnostics.cpp:58-98): with
    δ = β·σ_min(X)² − ‖∇f‖₂‖X‖₂ > 0, ‖XᵀX − I‖_F ≤ (‖X‖₂/δ)·‖∇L_β‖_F."""
    x = P._f64(x)
    out = FeasibilityBoundResult()
    b = P.gram(x, device=device)
    lmax = P.spectral_norm_estimate_host(b, _SEED_LMAX)
    if not lmax > 0.0:
        return out
    shift = lmax * (1.0 + 1e-8) + 1e-300
    shifted = np.asfortranarray(np.where(np.eye(b.shape[0], dtype=bool), shift - b, -b))
    lmin = max(shift - P.spectral_norm_estimate_host(shifted, _SEED_LMIN), 0.0)
    if not lmin > 0.0:
        return out
    _, g = P.evaluate(model, x, device=device)
    grad_2 = float(np.sqrt(P.spectral_norm_estimate_host(P.gram(g, device=device), _SEED_GRAD)))
    x_2 = float(np.sqrt(lmax))
    out.delta = beta * lmin - grad_2 * x_2
    if not out.delta > 0.0:
        return out
    out.applicable = True
    w = _sym(P.matmul_at_b(g, x, device=device))
    c = b - np.eye(b.shape[0])
    grad_l = g + P.matmul(x, np.asfortranarray(beta * c - w), device=device)
    out.lhs = float(np.linalg.norm(c))
    out.rhs = x_2 / out.delta * float(np.linalg.norm(grad_l))
    out.slack = out.rhs - out.lhs
    out.holds = out.lhs <= out.rhs
    return out
