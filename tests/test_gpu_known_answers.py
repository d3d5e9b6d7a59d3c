"""Known-answer tests of the device linalg seam, after the classes of the reference's own
dense-core tests (pkg/tests/test_linalg.py: TestSpdInverse :135-161, TestMatmul :164-188,
TestTwoNorm :191-231, TestGatherScatter :234-275, TestConditionNumber :278-296).  The cases
are restated here (hand values, a Gauss-Jordan second oracle, SVD, a triple loop); everything
runs through libibmi_b200.so."""

import warnings

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


def gauss_jordan_inverse(a):
    """Second oracle: Gauss-Jordan with partial pivoting in plain Python loops (small n only)."""
    n = len(a)
    m = np.hstack([np.array(a, dtype=np.float64), np.eye(n)])
    for col in range(n):
        piv = col + int(np.argmax(np.abs(m[col:, col])))
        m[[col, piv]] = m[[piv, col]]
        m[col] /= m[col, col]
        for r in range(n):
            if r != col:
                m[r] -= m[r, col] * m[col]
    return m[:, n:]


# ------------------------------------------------------------------ spd_inverse
def test_spd_inverse_identity_diagonal_and_adjugate():
    from paper_2502_06377_b200.linalg import spd_inverse

    assert np.array_equal(spd_inverse(np.eye(5)), np.eye(5))
    d = np.array([0.5, 2.0, 4.0, 8.0])
    np.testing.assert_allclose(spd_inverse(np.diag(d)), np.diag(1.0 / d), rtol=0, atol=1e-15)
    a = np.array([[4.0, 1.0], [1.0, 3.0]])
    adj = np.array([[3.0, -1.0], [-1.0, 4.0]]) / 11.0
    np.testing.assert_allclose(spd_inverse(a), adj, rtol=1e-14)


@pytest.mark.parametrize("p", [3, 17, 64, 130])
def test_spd_inverse_against_gauss_jordan(p):
    from paper_2502_06377_b200.linalg import spd_inverse

    a = random_spd(p, 100 + p)
    inv = spd_inverse(a)
    np.testing.assert_allclose(inv, gauss_jordan_inverse(a), rtol=1e-8, atol=1e-12)
    assert np.array_equal(inv, inv.T)                                  # exactly symmetric
    assert np.linalg.norm(a @ inv - np.eye(p)) <= 1e-8


# ------------------------------------------------------------------ matmul
def test_matmul_identity_hand_values_and_ones(rng):
    from paper_2502_06377_b200.linalg import matmul

    x = rng.standard_normal((7, 7))
    np.testing.assert_allclose(matmul(np.eye(7), x), x, rtol=0, atol=1e-15)
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert np.array_equal(matmul(a, b), np.array([[19.0, 22.0], [43.0, 50.0]]))
    row = np.arange(1.0, 6.0).reshape(1, 5)
    assert matmul(row, np.ones((5, 1)))[0, 0] == 15.0


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 2), (17, 9, 23), (40, 33, 64)])
def test_matmul_against_triple_loop(rng, shape):
    from paper_2502_06377_b200.linalg import matmul

    m, k, n = shape
    a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    ref = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            s = 0.0
            for t in range(k):
                s += a[i, t] * b[t, j]
            ref[i, j] = s
    np.testing.assert_allclose(matmul(a, b), ref, rtol=0, atol=1e-13 * max(1.0, np.abs(ref).max()))


def test_matmul_dimension_mismatch():
    from paper_2502_06377_b200 import DimensionMismatch
    from paper_2502_06377_b200.linalg import matmul

    with pytest.raises(DimensionMismatch):
        matmul(np.ones((2, 3)), np.ones((4, 2)))


# ------------------------------------------------------------------ two_norm
def test_two_norm_identity_diagonal_nilpotent_zero():
    from paper_2502_06377_b200.linalg import two_norm

    assert abs(two_norm(np.eye(6)) - 1.0) <= 1e-9
    assert abs(two_norm(np.diag([1.0, -7.0, 3.0])) - 7.0) <= 1e-6 * 7.0
    nil = np.array([[0.0, 5.0], [0.0, 0.0]])                            # spectral radius 0, 2-norm 5
    assert abs(two_norm(nil) - 5.0) <= 1e-9
    assert two_norm(np.zeros((4, 3))) == 0.0


@pytest.mark.parametrize("seed,shape", [(0, (30, 30)), (1, (12, 40)), (2, (55, 21)), (3, (900, 700))])
def test_two_norm_against_svd(seed, shape):
    """A well-separated top singular value (5 against ≤ 2), so that the reference's stop rule
    |Δσ| ≤ 1e-9·σ leaves σ within 1e-6 of the SVD value; both Gram forms, all three kernels
    (cluster, flag exchange)."""
    from paper_2502_06377_b200.linalg import two_norm

    rng = np.random.default_rng(seed)
    m, n = shape
    k = min(m, n)
    u, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v, _ = np.linalg.qr(rng.standard_normal((n, k)))
    sv = np.concatenate([[5.0], rng.uniform(0.1, 2.0, k - 1)])
    b = (u * sv) @ v.T
    s = two_norm(b)
    smax = np.linalg.svd(b, compute_uv=False)[0]
    assert abs(s - smax) <= 1e-6 * smax
    for _ in range(5):                                                  # a lower bound never exceeds it
        x = rng.standard_normal(n)
        assert np.linalg.norm(b @ x) / np.linalg.norm(x) <= s + 1e-6


def test_two_norm_rectangular_gaussian(rng):
    from paper_2502_06377_b200.linalg import two_norm

    b = rng.standard_normal((12, 30))
    assert abs(two_norm(b) - np.linalg.svd(b, compute_uv=False)[0]) <= 1e-5 * np.linalg.norm(b, 2)


def test_two_norm_cap_warns_and_returns(rng):
    from paper_2502_06377_b200 import NoConvergenceWarning
    from paper_2502_06377_b200.linalg import two_norm

    b = rng.standard_normal((25, 25))
    with pytest.warns(NoConvergenceWarning):
        s = two_norm(b, rtol=1e-300, max_iters=2)
    assert 0.0 < s <= np.linalg.svd(b, compute_uv=False)[0] * (1 + 1e-12)


# ------------------------------------------------------------------ gather / scatter
def test_gather_scatter_known_answers(rng):
    from paper_2502_06377_b200 import DimensionMismatch, IndexOutOfRange
    from paper_2502_06377_b200.linalg import gather, scatter_add_assign

    a = rng.standard_normal((6, 6))
    every = np.arange(6)
    assert np.array_equal(gather(a, every, every), a)
    assert np.array_equal(gather(np.eye(6), [1, 4], [1, 4]), np.eye(2))
    assert gather(a, [2], [5])[0, 0] == a[2, 5]
    with pytest.raises(IndexOutOfRange):
        gather(a, [0, 6], [0])
    t = np.zeros((6, 6))
    scatter_add_assign(t, every, every, a)
    assert np.array_equal(t, a)
    t = np.zeros((4, 4))
    scatter_add_assign(t, [3], [0], np.array([[2.5]]))
    assert t[3, 0] == 2.5 and np.count_nonzero(t) == 1
    rows, cols = np.array([4, 1]), np.array([0, 3, 5])
    t = rng.standard_normal((6, 6))
    blk = rng.standard_normal((2, 3))
    scatter_add_assign(t, rows, cols, blk)
    assert np.array_equal(gather(t, rows, cols), blk)                   # round trip
    t2 = np.ones((3, 3))
    scatter_add_assign(t2, [0, 2], [1], np.array([[1.0], [2.0]]), add=True)
    assert t2[0, 1] == 2.0 and t2[2, 1] == 3.0 and t2[1, 1] == 1.0
    with pytest.raises(DimensionMismatch):
        scatter_add_assign(np.zeros((3, 3)), [0, 1], [0, 1], np.zeros((3, 2)))


# ------------------------------------------------------------------ condition number
def test_condition_number_known_answers():
    from paper_2502_06377_b200 import NotPositiveDefinite
    from paper_2502_06377_b200.analysis import condition_number_2

    assert abs(condition_number_2(np.eye(8)) - 1.0) <= 1e-9
    assert abs(condition_number_2(np.diag([1.0, 10.0, 100.0])) - 100.0) <= 1e-6 * 100.0
    for p in (5, 40):
        a = random_spd(p, 300 + p)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            c = condition_number_2(a)
        assert abs(c - np.linalg.cond(a, 2)) <= 0.01 * c
    with pytest.raises(NotPositiveDefinite):
        condition_number_2(np.array([[1.0, 2.0], [2.0, 1.0]]))
