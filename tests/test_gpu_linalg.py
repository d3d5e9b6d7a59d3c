"""The linalg seam on the device (reference linalg.py:80-211): cholesky,
chol_solve, CholeskyFactor, gather, scatter_add_assign, with the reference
test suite's cases (pkg/tests/test_linalg.py:30-69, :113-139, :234-275) and
the reference outputs frozen in tests/golden/pins.npz; plus block_update /
error_estimate on a non-symmetric Σ (solver.py:132-155)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden, random_spd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU hosts)")
    import paper_2502_06377_b200 as pkg

    pkg.load_library()


def L():
    from paper_2502_06377_b200 import linalg

    return linalg


# ----------------------------------------------------------------- cholesky
def test_cholesky_identity_and_hand_values():
    f = L().cholesky(np.eye(3))
    np.testing.assert_array_equal(f.l, np.eye(3))
    f = L().cholesky([[4.0, 2.0], [2.0, 3.0]])
    np.testing.assert_allclose(f.l, [[2.0, 0.0], [1.0, math.sqrt(2.0)]], rtol=1e-15)
    assert f.dim == 2


@pytest.mark.parametrize("p", [5, 17, 64, 65, 200, 1000])
def test_cholesky_reconstruction_and_strict_lower(p):
    a = random_spd(p, p)
    f = L().cholesky(a)
    assert np.linalg.norm(f.l @ f.l.T - a) / np.linalg.norm(a) <= 1e-10
    assert np.all(np.triu(f.l, 1) == 0.0)
    assert np.all(np.diag(f.l) > 0)
    ref = np.linalg.cholesky(a)
    assert np.linalg.norm(f.l - ref) / np.linalg.norm(ref) <= 1e-13


def test_cholesky_matches_reference_pin():
    pins = golden("pins.npz")
    f = L().cholesky(pins["case1_a"])
    ref = pins["chol_l"]
    assert np.linalg.norm(f.l - ref) / np.linalg.norm(ref) <= 1e-14


def test_cholesky_errors():
    from paper_2502_06377_b200 import DimensionMismatch, NotPositiveDefinite

    a = np.eye(4)
    a[2, 2] = -1.0
    with pytest.raises(NotPositiveDefinite) as info:
        L().cholesky(a)
    assert info.value.index == 2
    big = random_spd(300, 3)
    big[170, 170] = -1e6          # fails inside the blocked factorisation (third 64-block)
    with pytest.raises(NotPositiveDefinite) as info:
        L().cholesky(big)
    from scipy.linalg.lapack import dpotrf

    assert info.value.index == dpotrf(big, lower=1)[1] - 1
    with pytest.raises(DimensionMismatch):
        L().cholesky(np.ones((2, 3)))
    with pytest.raises(ValueError):
        L().cholesky([[1.0, 2.0], [0.5, 3.0]])


def test_cholesky_device_tensor_stays_on_device():
    a = torch.as_tensor(random_spd(96, 2), device="cuda")
    f = L().cholesky(a)
    assert f.l.is_cuda
    assert torch.linalg.norm(f.l @ f.l.T - a) / torch.linalg.norm(a) <= 1e-12


# ----------------------------------------------------------------- chol_solve
def test_chol_solve_reference_cases():
    rng = np.random.default_rng(0)
    f = L().cholesky(np.eye(3))
    b = rng.standard_normal((3, 2))
    np.testing.assert_array_equal(L().chol_solve(f, b), b)
    f = L().cholesky([[4.0, 2.0], [2.0, 3.0]])
    np.testing.assert_allclose(L().chol_solve(f, [[1.0], [0.0]]), [[0.375], [-0.25]], rtol=1e-14)
    f = L().cholesky(np.diag([2.0, 4.0]))
    np.testing.assert_allclose(L().chol_solve(f, np.eye(2)), np.diag([0.5, 0.25]))
    from paper_2502_06377_b200 import DimensionMismatch

    with pytest.raises(DimensionMismatch):
        L().chol_solve(L().cholesky(np.eye(3)), np.ones((4, 1)))


@pytest.mark.parametrize("p,nrhs", [(40, 5), (257, 3), (1000, 64)])
def test_chol_solve_residual(p, nrhs):
    a = random_spd(p, 3 + p)
    b = np.random.default_rng(p).standard_normal((p, nrhs))
    x = L().chol_solve(L().cholesky(a), b)
    assert np.linalg.norm(a @ x - b) / np.linalg.norm(b) <= 1e-10


def test_chol_solve_matches_reference_pin():
    pins = golden("pins.npz")
    f = L().CholeskyFactor(l=pins["chol_l"], dim=96)
    x = L().chol_solve(f, pins["chol_rhs"])
    assert np.linalg.norm(x - pins["chol_x"]) / np.linalg.norm(pins["chol_x"]) <= 1e-12


# ----------------------------------------------------------------- gather / scatter
def test_gather_reference_cases():
    from paper_2502_06377_b200 import IndexOutOfRange

    rng = np.random.default_rng(1)
    a = rng.standard_normal((4, 4))
    np.testing.assert_array_equal(L().gather(a, np.arange(4), np.arange(4)), a)
    np.testing.assert_array_equal(L().gather(np.eye(4), [0, 2], [0, 2]), np.eye(2))
    assert L().gather([[1.0, 2.0], [3.0, 4.0]], [1], [0]) == np.array([[3.0]])
    with pytest.raises(IndexOutOfRange):
        L().gather(np.eye(3), [0, 3], [0])


def test_gather_large_unsorted_repeats():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((700, 900))
    r = rng.integers(0, 700, 333)
    c = rng.integers(0, 900, 517)
    np.testing.assert_array_equal(L().gather(a, r, c), a[np.ix_(r, c)])
    ad = torch.as_tensor(a, device="cuda")
    out = L().gather(ad, r, c)
    assert out.is_cuda and np.array_equal(out.cpu().numpy(), a[np.ix_(r, c)])


def test_scatter_reference_cases():
    from paper_2502_06377_b200 import DimensionMismatch

    rng = np.random.default_rng(3)
    src = rng.standard_normal((3, 3))
    target = np.zeros((3, 3))
    L().scatter_add_assign(target, np.arange(3), np.arange(3), src)
    np.testing.assert_array_equal(target, src)
    target = np.zeros((2, 2))
    L().scatter_add_assign(target, [1], [1], [[9.0]])
    np.testing.assert_array_equal(target, [[0.0, 0.0], [0.0, 9.0]])
    a = rng.standard_normal((6, 6))
    before = a.copy()
    rows, cols = np.array([1, 3, 4]), np.array([0, 2])
    L().scatter_add_assign(a, rows, cols, L().gather(a, rows, cols))
    np.testing.assert_array_equal(a, before)
    target = np.ones((2, 2))
    L().scatter_add_assign(target, [0], [0], [[2.0]], add=True)
    np.testing.assert_array_equal(target, [[3.0, 1.0], [1.0, 1.0]])
    with pytest.raises(DimensionMismatch):
        L().scatter_add_assign(np.zeros((3, 3)), [0, 1], [0], np.ones((1, 1)))


@pytest.mark.parametrize("add", [False, True])
def test_scatter_repeated_indices_follow_numpy(add):
    rng = np.random.default_rng(4)
    t0 = rng.standard_normal((50, 60))
    r = np.array([3, 7, 3, 10, 7, 3])
    c = np.array([5, 5, 9, 1])
    src = rng.standard_normal((r.size, c.size))
    want = t0.copy()
    if add:
        want[np.ix_(r, c)] += src
    else:
        want[np.ix_(r, c)] = src
    got = t0.copy()
    L().scatter_add_assign(got, r, c, src, add=add)
    np.testing.assert_array_equal(got, want)
    td = torch.as_tensor(t0, device="cuda")
    L().scatter_add_assign(td, r, c, src, add=add)
    np.testing.assert_array_equal(td.cpu().numpy(), want)


# ----------------------------------------------------------------- non-symmetric Σ
def test_block_update_and_estimate_nonsymmetric_sigma_match_reference():
    import paper_2502_06377_b200 as pkg

    pins = golden("pins.npz")
    a = pins["case2_a"]
    part = pkg.contiguous_partition(128, 4, 0.125)
    idx, comp = part.sets[1], pkg.complement(part, 1)
    s = pins["nonsym_sigma0"].copy()
    e = pkg.error_estimate(a, s, idx, comp)
    assert abs(e - pins["nonsym_ee"][0]) <= 1e-12 * pins["nonsym_ee"][0]
    pkg.block_update(a, s, idx, comp)
    ref = pins["nonsym_bu"]
    assert np.linalg.norm(s - ref) / np.linalg.norm(ref) <= 1e-13


def test_block_update_nonsymmetric_sigma_noncontiguous_set():
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 90
    a = random_spd(p, 9)
    s = np.eye(p) + 0.03 * np.random.default_rng(9).standard_normal((p, p))
    idx = np.arange(1, p, 3)
    comp = np.setdiff1d(np.arange(p), idx)
    want = s.copy()
    orc.BlockOp(a, idx, comp).apply(want)
    e_ref = orc.error_estimate(a, s, idx, comp)[0]
    assert abs(pkg.error_estimate(a, s, idx, comp) - e_ref) <= 1e-12 * e_ref
    pkg.block_update(a, s, idx, comp)
    assert np.linalg.norm(s - want) / np.linalg.norm(want) <= 1e-13
