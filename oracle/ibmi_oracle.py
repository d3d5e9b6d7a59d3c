"""CPU oracle for the IBMI sweep — TEST INFRASTRUCTURE ONLY.

This is a NumPy/SciPy restatement of the reference algorithm
(`/root/reference/pkg/src/ibmi/solver.py`, `linalg.py`).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it, and only as the checker or the timed CPU baseline.  The
product path (``paper_2502_06377_b200``) never imports it: it fails loudly
when the CUDA library is missing.

Pinned against the reference itself: ``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/ibmi`` (only possible in the build container) and
checks every function below against the reference's own on the same inputs,
then freezes the reference outputs as fixtures under ``tests/golden/``;
``tests/test_oracle_golden.py`` re-checks this module against those fixtures
on every CPU test run.

The arithmetic lives in OpenBLAS/LAPACK exactly as in the reference: dpotrf
(linalg.py:104), dpotrs via ``cho_solve`` (linalg.py:119), dgemm through
``@`` (solver.py:120, :124-125, :154) and dgemv in the power iteration
(linalg.py:265).  The one extension is the starting Σ₀: BASELINE c1/c2 seed
``Σ₀[c₁,c₁] = diag(1/A_ii)`` (``guess="jacobi"``), which the reference lacks
(solver.py:55-59); with the identity guess the loop is the reference's
``solve`` verbatim in order (solver.py:241-270).
"""

from __future__ import annotations

import time

import numpy as np
import scipy.linalg as sla
from scipy.linalg.lapack import dpotrf

from paper_2502_06377_b200.exceptions import DimensionMismatch, NotPositiveDefinite

POWER_RTOL = 1e-9          # linalg.py:47
POWER_MAX_ITERS = 5000     # linalg.py:48
RESTART_SEED = 0x5EED      # linalg.py:49
SYMMETRY_RTOL = 1e-12      # linalg.py:43


def check_symmetric(a: np.ndarray, rtol: float = SYMMETRY_RTOL) -> None:
    """linalg.py:68-77 — max|a - aᵀ| must not exceed rtol · max|a|."""
    big = float(np.max(np.abs(a)))
    if big == 0.0:
        return
    skew = float(np.max(np.abs(a - a.T)))
    if skew > rtol * big:
        raise ValueError(f"matrix is not symmetric: max |a - a.T| = {skew:.3e}")


def spd_inverse(a: np.ndarray) -> np.ndarray:
    """linalg.py:122-130 via :96-119 — dpotrf (lower), dpotrs against I, then ½(X + Xᵀ)."""
    a = np.asarray(a, dtype=np.float64)
    check_symmetric(a)
    l, info = dpotrf(a, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise NotPositiveDefinite(info - 1)
    if info < 0:
        raise ValueError(f"dpotrf illegal argument {-info}")
    x = sla.cho_solve((l, True), np.eye(a.shape[0]), check_finite=False)
    return 0.5 * (x + x.T)


def power_sigma_max(b: np.ndarray, rtol: float = POWER_RTOL, max_iters: int = POWER_MAX_ITERS):
    """linalg.py:223-253 applied to ``B`` (two_norm, :256-274).

    Returns ``(sigma, converged, iterations)``.
    """
    n = b.shape[1]
    bt = b.T
    v = np.full(n, 1.0 / np.sqrt(n))
    prev, sigma, restarted = -1.0, 0.0, False
    for it in range(1, max_iters + 1):
        y = b @ v
        sigma = float(np.linalg.norm(y))
        if sigma == 0.0:
            if restarted:
                return 0.0, True, it
            v = np.random.default_rng(RESTART_SEED).standard_normal(n)
            v = v / np.linalg.norm(v)
            restarted, prev = True, -1.0
            continue
        if abs(sigma - prev) <= rtol * sigma:
            return sigma, True, it
        prev = sigma
        w = bt @ y
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return sigma, True, it
        v = w / nw
    return sigma, False, max_iters


def estimate_matrix(a, sigma, idx, comp) -> np.ndarray:
    """solver.py:154 — ``Σ_II A_Ic + Σ_Ic A_cc`` (the (1,2) block of ΣA)."""
    ii = np.ix_(idx, idx)
    ic = np.ix_(idx, comp)
    cc = np.ix_(comp, comp)
    return sigma[ii] @ a[ic] + sigma[ic] @ a[cc]


def error_estimate(a, sigma, idx, comp, rtol=POWER_RTOL, max_iters=POWER_MAX_ITERS):
    """solver.py:147-155. Returns ``(err, power_iterations, converged)``."""
    s, conv, it = power_sigma_max(estimate_matrix(a, sigma, idx, comp), rtol, max_iters)
    return s, it, conv


class BlockOp:
    """solver.py:109-129 — cached ``ainv = A_II⁻¹``, ``W = ainv A_Ic``; ``apply``
    does ``M = W Σ_cc``, ``Σ_II = sym(ainv + M Wᵀ)``, ``Σ_Ic = -M``, ``Σ_cI = -Mᵀ``."""

    def __init__(self, a, idx, comp):
        self.idx = np.asarray(idx, dtype=np.intp)
        self.comp = np.asarray(comp, dtype=np.intp)
        self.ainv = spd_inverse(a[np.ix_(self.idx, self.idx)])
        self.w = self.ainv @ a[np.ix_(self.idx, self.comp)]

    def apply(self, sigma):
        m = self.w @ sigma[np.ix_(self.comp, self.comp)]
        top = self.ainv + m @ self.w.T
        sigma[np.ix_(self.idx, self.idx)] = 0.5 * (top + top.T)
        sigma[np.ix_(self.idx, self.comp)] = -m
        sigma[np.ix_(self.comp, self.idx)] = -m.T


def frobenius_residual(a, sigma) -> float:
    """BASELINE c2's stopping norm ``‖I − AΣ‖_F`` (no reference counterpart;
    nearest is analysis.py:182-186)."""
    r = a @ sigma
    r[np.diag_indices_from(r)] -= 1.0
    return float(np.linalg.norm(r))


def complement(p: int, idx) -> np.ndarray:
    keep = np.ones(p, dtype=bool)
    keep[np.asarray(idx, dtype=np.intp)] = False
    return np.nonzero(keep)[0].astype(np.intp)


def guess_monte_carlo(a, comp, n_samples: int = 100, seed: int = 0) -> np.ndarray:
    """solver.py:167-181 — cov of L⁻ᵀw restricted to comp (dpotrf + dtrsm, same calls)."""
    a = np.asarray(a, dtype=np.float64)
    l, info = dpotrf(a, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise NotPositiveDefinite(info - 1)
    w = np.random.default_rng(seed).standard_normal((a.shape[0], n_samples))
    z = sla.solve_triangular(l, w, lower=True, trans="T", check_finite=False)
    zc = z[np.asarray(comp, dtype=np.intp)]
    return (zc @ zc.T) / n_samples


def guess_takahashi(a, comp) -> np.ndarray:
    """solver.py:184-212 — unpivoted LDLᵀ of A reordered [rest, comp], then the
    backward recurrence h[i,j] = δ_ij/d_i − Σ_{k>i} l_ki h_kj over the comp corner."""
    a = np.asarray(a, dtype=np.float64)
    comp = np.asarray(comp, dtype=np.intp)
    p = a.shape[0]
    keep = np.ones(p, dtype=bool)
    keep[comp] = False
    order = np.concatenate([np.nonzero(keep)[0], comp])
    w = a[np.ix_(order, order)].copy()
    lower = np.eye(p)
    d = np.zeros(p)
    for j in range(p):                       # right-looking unblocked LDLᵀ
        d[j] = w[j, j]
        col = w[j + 1:, j] / d[j]
        lower[j + 1:, j] = col
        w[j + 1:, j + 1:] -= d[j] * np.outer(col, col)
    c = comp.size
    off = p - c
    h = np.zeros((c, c))
    for i in range(p - 1, off - 1, -1):
        ii = i - off
        lcol = lower[i + 1:, i]
        row = -(lcol @ h[ii + 1:, ii + 1:])
        h[ii, ii + 1:] = row
        h[ii + 1:, ii] = row
        h[ii, ii] = 1.0 / d[i] - lcol @ row
    return 0.5 * (h + h.T)


def initial_sigma(a, comp0, guess: str = "identity", sigma0=None, mc_samples: int = 100,
                  mc_seed: int = 0) -> np.ndarray:
    """solver.py:244-251 (identity) plus the BASELINE ``jacobi`` seed."""
    p = a.shape[0]
    sigma = np.eye(p)
    if sigma0 is not None:
        g = np.asarray(sigma0, dtype=np.float64)
        if g.shape == (p, p):
            g = g[np.ix_(comp0, comp0)]
    elif guess == "identity":
        g = np.eye(comp0.size)
    elif guess == "jacobi":
        g = np.diag(1.0 / np.diag(a)[comp0])
    elif guess == "local":
        g = spd_inverse(a[np.ix_(comp0, comp0)])
    elif guess == "mc":
        g = guess_monte_carlo(a, comp0, mc_samples, mc_seed)
    elif guess == "takahashi":
        g = guess_takahashi(a, comp0)
    else:
        raise ValueError(f"oracle has no guess {guess!r}")
    if g.shape != (comp0.size, comp0.size):
        raise DimensionMismatch(f"initial guess shape {g.shape} vs complement {comp0.size}")
    sigma[np.ix_(comp0, comp0)] = g
    return sigma


def solve(a, sets, *, tol=1e-8, max_iterations=500, guess="identity", sigma0=None,
          stopping="estimate", norm_rtol=POWER_RTOL, norm_max_iters=POWER_MAX_ITERS,
          record_frobenius=False, callback=None, mc_samples=100, mc_seed=0):
    """solver.py:225-278 with the stopping-rule and Σ₀ extensions.

    ``stopping="estimate"``: stop when the reference estimate ≤ tol
    (solver.py:268).  ``stopping="frobenius"``: stop when ‖I − AΣ‖_F < tol
    (BASELINE c2).  Returns a dict with the reference ``SolveReport`` fields
    plus ``power_iters``, ``frobenius_trace`` and ``setup_seconds``.
    """
    a = np.asarray(a, dtype=np.float64)
    p = a.shape[0]
    sets = [np.asarray(s, dtype=np.intp) for s in sets]
    comps = [complement(p, s) for s in sets]
    t0 = time.perf_counter()
    ops = [BlockOp(a, s, c) for s, c in zip(sets, comps)]
    setup_s = time.perf_counter() - t0
    sigma = initial_sigma(a, comps[0], guess, sigma0, mc_samples, mc_seed)
    err_trace, walls, pits, frob = [], [], [], []
    converged, it = False, 0
    while it < max_iterations:
        t = time.perf_counter()
        it += 1
        for op in ops:
            op.apply(sigma)
        err, pi, _ = error_estimate(a, sigma, ops[-1].idx, ops[-1].comp, norm_rtol, norm_max_iters)
        walls.append(time.perf_counter() - t)
        err_trace.append(err)
        pits.append(pi)
        fr = None
        if record_frobenius or stopping == "frobenius":
            fr = frobenius_residual(a, sigma)
            frob.append(fr)
        if callback is not None:
            callback(it, err, fr, sigma)
        done = (fr < tol) if stopping == "frobenius" else (err <= tol)
        if done:
            converged = True
            break
    return dict(iterations=it, converged=converged, error_trace=err_trace, wall_times=walls,
                power_iters=pits, frobenius_trace=frob, setup_seconds=setup_s, result=sigma)
