"""The SuperMann Anderson least squares (proj/src/solver.cpp:67-76) as the
device computes it -- double-double Gram, column-pivoted Cholesky with Eigen's
pivot order and rank rules (csrc/aa.cuh, host entry spock_anderson_lstsq) --
against the oracle's restatement of Eigen's ColPivHouseholderQR with
threshold 1e-12 (oracle/orc_la.cpp).  CPU only: the entry needs no device."""
import numpy as np
import pytest

from oracle import oracle
from paper_2505_12078_b200.capi import anderson_lstsq
from paper_2505_12078_b200.rng import Philox


def _mat(rows, scales, seed):
    rng = Philox(seed)
    A = rng.normal_matrix(rows, len(scales), 0.0, 1.0)
    return A * np.asarray(scales)[None, :]


def _check(A, b, tol):
    k1 = anderson_lstsq(A, b)
    k2 = oracle.colpiv_qr_solve(A, b)
    assert np.array_equal(k1 == 0.0, k2 == 0.0), (k1, k2)  # same dropped columns
    sc = max(1.0, float(np.abs(k2).max()))
    assert float(np.abs(k1 - k2).max()) <= tol * sc, (k1, k2)
    r1, r2 = b - A @ k1, b - A @ k2
    assert abs(np.linalg.norm(r1) - np.linalg.norm(r2)) <= 1e-10 * max(1.0, np.linalg.norm(b))
    return k1


def _exact(A, b):
    """Least squares in 50-digit arithmetic (normal equations; A has full rank)."""
    import mpmath
    mpmath.mp.dps = 50
    Am, bm = mpmath.matrix(A.tolist()), mpmath.matrix(b.tolist())
    return np.array([float(x) for x in mpmath.lu_solve(Am.T * Am, Am.T * bm)])


@pytest.mark.parametrize("cols", [1, 2, 3, 5, 10])
def test_well_conditioned_matches_householder(cols):
    A = _mat(2000, [1.0] * cols, 3 + cols)
    b = Philox(50 + cols).normal_array(2000)
    k = _check(A, b, 1e-12)
    np.testing.assert_allclose(k, np.linalg.lstsq(A, b, rcond=None)[0], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("small", [1e-4, 1e-7, 1e-9, 1e-11])
def test_graded_columns_kept_down_to_the_threshold(small):
    """Columns far below sqrt(eps) relative but above the 1e-12 threshold are
    kept by the reference's Householder QR -- and by the double-double Gram
    (a plain-double Gram would lose them below ~1e-8)."""
    A = _mat(3000, [1.0, 0.3, small, 0.5], 11)
    b = Philox(12).normal_array(3000)
    k = _check(A, b, 1e-6)
    assert np.all(k != 0.0)


def test_nearly_dependent_column_kept():
    """cond(M_d) ~ 1e9: the Householder solve (oracle) is accurate to ~cond eps
    (2e-6 relative here), the double-double one to ~1e-13 of the exact solution."""
    A = _mat(300, [1.0, 1.0, 1.0], 21)
    A[:, 2] = A[:, 0] + 1e-9 * Philox(22).normal_array(300)
    b = Philox(23).normal_array(300)
    k = _check(A, b, 1e-5)
    assert np.all(k != 0.0)
    ex = _exact(A, b)
    assert float(np.abs(k - ex).max()) <= 1e-11 * float(np.abs(ex).max())


@pytest.mark.parametrize("tiny", [1e-14, 1e-16])
def test_columns_below_threshold_dropped(tiny):
    A = _mat(1000, [1.0, 2.0, tiny], 31)
    b = Philox(32).normal_array(1000)
    k = _check(A, b, 1e-10)
    assert k[2] == 0.0


def test_exact_duplicate_and_zero_columns():
    A = _mat(800, [1.0, 1.0, 1.0, 1.0], 41)
    A[:, 2] = A[:, 0]
    A[:, 3] = 0.0
    b = Philox(42).normal_array(800)
    k = _check(A, b, 1e-10)
    assert np.count_nonzero(k) == 2


def test_anderson_kat_scalar_history():
    """test_solver.cpp:247-263: history r = 1 after r = 2 gives M_d = [-1],
    kappa = -1 (psi = 1)."""
    k = anderson_lstsq(np.array([[-1.0]]), np.array([1.0]))
    assert k[0] == pytest.approx(-1.0, rel=1e-15)
    assert anderson_lstsq(np.zeros((3, 1)), np.full(3, 0.7))[0] == 0.0
