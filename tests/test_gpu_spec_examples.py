"""The reference specification's worked examples for the hot path, on the GPU
path through the C ABI.  The reference states them in SPEC.md (block_update
:351-354, error_estimate :361-364, solve :371-375) but its own test suite never
runs them, so they are pinned here:

* block_update: block-diagonal A gives Σ_I = A_I⁻¹ and zero off-diagonal
  blocks; A = I keeps Σ = I; an exact Σ_{I^c} = (A⁻¹)_{cc} makes one update
  return A⁻¹ (checked against an independent Gauss–Jordan inverse, the
  reference conftest's second oracle).
* error_estimate: Σ = A⁻¹ gives ≈ 0; A = Σ = I gives exactly 0; otherwise it is
  the spectral norm of the (1,2) block of Σ·A formed by brute force.
* solve: A = I converges in one sweep to I; the paper's 1-D kernel examples
  (RBF p = 2⁸ with 20% overlap; Matérn-5/2 two blocks, here p = 2¹¹ over 30
  sweeps) give the same sweep count, trace and Σ as the CPU oracle, the
  reference's algorithm.

Kernel matrices restate the reference's kernels.py formulas (grid_1d
:74-79, kernel_matrix :100-123, _evaluate :126-140) with its default
hyper-parameters (σ = 0.5, τ = 3.0)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import random_spd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU hosts)")
    import paper_2502_06377_b200 as pkg

    pkg.load_library()


def gauss_jordan_inverse(a: np.ndarray) -> np.ndarray:
    """Gauss–Jordan elimination with partial pivoting (independent of Cholesky)."""
    n = a.shape[0]
    m = np.hstack([a.astype(np.float64).copy(), np.eye(n)])
    for c in range(n):
        r = c + int(np.argmax(np.abs(m[c:, c])))
        if r != c:
            m[[c, r]] = m[[r, c]]
        m[c] /= m[c, c]
        for i in range(n):
            if i != c:
                m[i] -= m[i, c] * m[c]
    return m[:, n:]


def kernel_1d(p: int, family: str, sigma: float = 0.5, tau: float = 3.0) -> np.ndarray:
    x = np.linspace(0.0, float(p) ** 0.9, p)
    d2 = (x[:, None] - x[None, :]) ** 2
    if family == "rbf":
        a = np.exp(-d2 / (2.0 * sigma ** 2))
    elif family == "matern52":
        s = math.sqrt(5.0) * np.sqrt(d2) / tau
        a = (1.0 + s + s ** 2 / 3.0) * np.exp(-s)
    else:
        raise ValueError(family)
    a = np.maximum(a, a.T)
    np.fill_diagonal(a, 1.0)
    return a


def _sets(p, lo, hi):
    idx = np.arange(lo, hi, dtype=np.int64)
    comp = np.setdiff1d(np.arange(p, dtype=np.int64), idx)
    return idx, comp


# ------------------------------------------------------------ block_update

def test_block_update_block_diagonal_gives_exact_block_inverse():
    import paper_2502_06377_b200 as pkg

    p, b = 96, 40
    a = np.zeros((p, p))
    a[:b, :b] = random_spd(b, seed=1)
    a[b:, b:] = random_spd(p - b, seed=2)
    idx, comp = _sets(p, 0, b)
    sigma = np.eye(p)
    pkg.block_update(a, sigma, idx, comp)
    np.testing.assert_allclose(sigma[:b, :b], np.linalg.inv(a[:b, :b]), rtol=0, atol=1e-13)
    assert np.all(sigma[:b, b:] == 0.0) and np.all(sigma[b:, :b] == 0.0)
    # one update per block yields the exact inverse
    idx2, comp2 = _sets(p, b, p)
    pkg.block_update(a, sigma, idx2, comp2)
    ref = gauss_jordan_inverse(a)
    assert np.linalg.norm(sigma - ref) / np.linalg.norm(ref) < 1e-12


def test_block_update_identity_is_a_fixed_point():
    import paper_2502_06377_b200 as pkg

    p = 64
    a = np.eye(p)
    sigma = np.eye(p)
    for lo, hi in ((0, 24), (16, 48), (40, 64)):
        idx, comp = _sets(p, lo, hi)
        pkg.block_update(a, sigma, idx, comp)
        assert np.array_equal(sigma, np.eye(p))


@pytest.mark.parametrize("p,lo,hi", [(4, 0, 2), (4, 1, 3), (130, 17, 83)])
def test_block_update_with_exact_complement_returns_inverse(p, lo, hi):
    import paper_2502_06377_b200 as pkg

    a = random_spd(p, seed=p + lo)
    ainv = gauss_jordan_inverse(a)
    idx, comp = _sets(p, lo, hi)
    sigma = np.eye(p)
    sigma[np.ix_(comp, comp)] = ainv[np.ix_(comp, comp)]
    sigma = 0.5 * (sigma + sigma.T)
    pkg.block_update(a, sigma, idx, comp)
    assert np.linalg.norm(sigma - ainv) / np.linalg.norm(ainv) < 1e-12


# --------------------------------------------------------- error_estimate

def test_error_estimate_at_exact_inverse_is_zero():
    import paper_2502_06377_b200 as pkg

    p = 80
    a = random_spd(p, seed=3)
    sigma = np.linalg.inv(a)
    sigma = 0.5 * (sigma + sigma.T)
    idx, comp = _sets(p, 50, 80)
    assert pkg.error_estimate(a, sigma, idx, comp) <= 1e-10
    eye = np.eye(p)
    assert pkg.error_estimate(eye, eye, idx, comp) == 0.0


@pytest.mark.parametrize("p,lo,hi", [(4, 2, 4), (4, 0, 1), (150, 60, 110)])
def test_error_estimate_equals_brute_force_block_norm(p, lo, hi):
    import paper_2502_06377_b200 as pkg

    a = random_spd(p, seed=7 * p + lo)
    sigma = np.eye(p)
    idx, comp = _sets(p, lo, hi)
    block = (sigma @ a)[np.ix_(idx, comp)]
    ref = np.linalg.norm(block, 2)
    got = pkg.error_estimate(a, sigma, idx, comp)
    assert abs(got - ref) <= 1e-6 * ref


# ------------------------------------------------------------------ solve

def test_solve_identity_converges_in_one_sweep():
    import paper_2502_06377_b200 as pkg

    p = 16
    for part in (pkg.contiguous_partition(p, 2, 0.0), pkg.contiguous_partition(p, 4, 0.25),
                 pkg.red_black_partition(p)):
        rep = pkg.solve(np.eye(p), part)
        assert rep.converged and rep.iterations == 1
        assert np.array_equal(rep.result, np.eye(p))


@pytest.mark.parametrize("case", ["rbf_256_k2_f02", "matern52_2048_k2_f0"])
def test_solve_paper_1d_kernel_examples_match_oracle(case):
    """RBF p = 2⁸, 20% overlap: one sweep, as the paper's Table 2 row.  The
    Matérn-5/2 two-block case does not converge in ~11 sweeps in the reference
    (its counts differ from Table 6), so it is compared over the
    first 30 sweeps, where it is still unconverged on both sides."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    if case == "rbf_256_k2_f02":
        a, part, cap = kernel_1d(256, "rbf"), pkg.contiguous_partition(256, 2, 0.2), 500
    else:
        a, part, cap = kernel_1d(2048, "matern52"), pkg.contiguous_partition(2048, 2, 0.0), 30
    rep = pkg.solve(a, part, pkg.IbmiConfig(max_iterations=cap))
    ref = orc.solve(a, part.sets, max_iterations=cap)
    assert rep.converged == ref["converged"]
    assert rep.iterations == ref["iterations"]
    rel = np.linalg.norm(rep.result - ref["result"]) / np.linalg.norm(ref["result"])
    assert rel <= 1e-10, rel
    err_ref = np.asarray(ref["error_trace"])
    tol = 1e-8
    assert np.all(np.abs(np.asarray(rep.error_trace) - err_ref) <= 1e-6 * err_ref + 5e-2 * tol)
