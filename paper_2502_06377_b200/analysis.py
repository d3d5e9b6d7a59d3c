"""Convergence diagnostics on the GPU (reference ``ibmi.analysis``, analysis.py:56-188).

Same functions and return values as the reference; the dense work (SPD
inverses, products, spectral norms) runs in ``libibmi_b200.so``
(``ibmi_spd_inverse``, the DMMA NT GEMM, the Gram power iteration).  The
products are written X·Yᵀ, so a plain product ``X @ Z`` passes ``Zᵀ``.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .exceptions import DimensionMismatch
from .partition import overlap_depth

__all__ = ["contraction_factor", "spectral_radius_condition", "condition_number_2", "newton_schultz",
           "flop_cost", "CostBreakdown", "lemma_error_recurrence_check"]

POWER_RTOL = 1e-9
POWER_MAX_ITERS = 5000
MAX_CHECK_DIM = 512


def _torch():
    import torch

    return torch


def _dev(a):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _mm(x, z):
    """x @ z on the device through the NT kernel (z transposed once)."""
    from .linalg import dgemm_nt

    return dgemm_nt(x.contiguous(), z.t().contiguous())


def _pieces(a, i1, i2):
    """analysis.py:43-53 — inverses of both diagonal blocks and the couplings."""
    from .linalg import spd_inverse

    a = np.asarray(a, dtype=np.float64)
    i1 = np.asarray(i1, dtype=np.intp)
    i2 = np.asarray(i2, dtype=np.intp)
    if i1.size + i2.size != a.shape[0] or np.intersect1d(i1, i2).size:
        raise ValueError("index sets must partition the matrix without overlap")
    inv1 = spd_inverse(_dev(a[np.ix_(i1, i1)]))
    inv2 = spd_inverse(_dev(a[np.ix_(i2, i2)]))
    a12 = _dev(a[np.ix_(i1, i2)])
    a21 = _dev(a[np.ix_(i2, i1)])
    return a, i1, i2, inv1, inv2, a12, a21


def contraction_factor(a, i1, i2) -> float:
    """‖inv(A_2) A_21 inv(A_1) A_12‖₂ (analysis.py:56-59); its square is the per-sweep rate."""
    from .linalg import two_norm

    _, _, _, inv1, inv2, a12, a21 = _pieces(a, i1, i2)
    t = _mm(_mm(_mm(inv2, a21), inv1), a12)
    return two_norm(t)


def spectral_radius_condition(a, i1, i2, rtol: float = POWER_RTOL, max_iters: int = POWER_MAX_ITERS) -> float:
    """Spectral radius of A_12 inv(A_2) A_21 inv(A_1) by the reference's Rayleigh
    power iteration (analysis.py:62-82); the operator is formed on the GPU."""
    torch = _torch()
    _, _, _, inv1, inv2, a12, a21 = _pieces(a, i1, i2)
    t = _mm(_mm(_mm(a12, inv2), a21), inv1)
    n = t.shape[0]
    v = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.float64, device=t.device)
    prev, rho = -1.0, 0.0
    for _ in range(max_iters):
        y = t @ v
        ny = float(torch.linalg.vector_norm(y))
        if ny == 0.0:
            return 0.0
        rho = float(v @ y)
        if abs(rho - prev) <= rtol * abs(rho):
            break
        prev = rho
        v = y / ny
    return abs(rho)


def condition_number_2(a, rtol: float = POWER_RTOL, max_iters: int = POWER_MAX_ITERS) -> float:
    """λ_max · ‖A⁻¹‖₂ (reference linalg.py:277-303): the power iteration on A and
    on A⁻¹ is the same sequence as two_norm of A and of its inverse."""
    from .linalg import spd_inverse, two_norm

    d = _dev(a)
    if d.shape[0] != d.shape[1]:
        raise DimensionMismatch(f"expected a square matrix, got shape {tuple(d.shape)}")
    lam = two_norm(d, rtol, max_iters)
    inv = spd_inverse(np.asarray(a, dtype=np.float64))
    return lam * two_norm(inv, rtol, max_iters)


def newton_schultz(a, x0, tol: float = 1e-8, max_iters: int = 100):
    """X ← X + X(I − AX) (analysis.py:169-188) with DMMA products; returns
    ``(X, iterations, converged)`` (numpy X)."""
    from .linalg import two_norm

    torch = _torch()
    a = np.asarray(a, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    if a.shape != x0.shape or a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"shapes differ: {a.shape} vs {x0.shape}")
    da, x = _dev(a), _dev(x0)
    eye = torch.eye(a.shape[0], dtype=torch.float64, device=da.device)
    for it in range(1, max_iters + 1):
        r = eye - _mm(da, x)
        if not bool(torch.isfinite(r).all()):
            return x.cpu().numpy(), it, False
        if two_norm(r) <= tol:
            return x.cpu().numpy(), it, True
        x = x + _mm(x, r)
    return x.cpu().numpy(), max_iters, False


@dataclass(frozen=True)
class CostBreakdown:
    """Per-sweep flop model (analysis.py:117-135), exact rationals."""

    k: int
    m: int
    h: int
    per_step_flops: tuple
    total_flops: Fraction
    direct_flops: Fraction


def flop_cost(p: int, k: int, overlap_fraction: float = 0.0) -> CostBreakdown:
    """analysis.py:138-166: edge sets (m+h), interior (m+2h); step cost
    (1/3)s³ + 2k²m²s; direct (7/3)p³."""
    if k < 2:
        raise ValueError(f"need at least 2 blocks, got {k}")
    if p < 2 * k:
        raise ValueError(f"p={p} is too small for {k} blocks")
    m = p // k
    h = overlap_depth(m, overlap_fraction)

    def cost(size):
        return Fraction(1, 3) * size ** 3 + 2 * k * k * m * m * size

    steps = (cost(m + h),) + (cost(m + 2 * h),) * (k - 2) + (cost(m + h),)
    return CostBreakdown(k=k, m=m, h=h, per_step_flops=steps, total_flops=sum(steps, Fraction(0)),
                         direct_flops=Fraction(7, 3) * (k * m) ** 3)


def lemma_error_recurrence_check(a, i1, i2, guess, r: int) -> float:
    """Relative Frobenius gap between r simulated two-block sweeps (GPU
    block_update) and the closed-form congruence Tʳ(guess − Σ₂)Tʳᵀ
    (analysis.py:85-114)."""
    from .linalg import spd_inverse
    from .solver import block_update

    if np.asarray(a).shape[0] > MAX_CHECK_DIM:
        raise ValueError(f"recurrence check forms exact inverses; refusing p > {MAX_CHECK_DIM}")
    a, i1, i2, inv1, inv2, a12, a21 = _pieces(a, i1, i2)
    guess = np.asarray(guess, dtype=np.float64)
    if guess.shape != (i2.size, i2.size):
        raise DimensionMismatch(f"guess shape {guess.shape} does not match second block size {i2.size}")
    sig2 = spd_inverse(a)[np.ix_(i2, i2)]
    sigma = np.eye(a.shape[0])
    sigma[np.ix_(i2, i2)] = guess
    for _ in range(r):
        block_update(a, sigma, i1, i2)
        block_update(a, sigma, i2, i1)
    direct = sigma[np.ix_(i2, i2)] - sig2
    t = _mm(_mm(_mm(inv2, a21), inv1), a12)
    tr = _torch().eye(t.shape[0], dtype=t.dtype, device=t.device)
    base, e = t, r
    while e:                                   # Tʳ by repeated squaring on the DMMA GEMM
        if e & 1:
            tr = _mm(tr, base)
        base, e = _mm(base, base), e >> 1
    closed = _mm(_mm(tr, _dev(guess - sig2)), tr.t().contiguous()).cpu().numpy()
    scale = max(np.linalg.norm(direct), np.linalg.norm(closed))
    if scale == 0.0:
        return 0.0
    return float(np.linalg.norm(direct - closed) / scale)
