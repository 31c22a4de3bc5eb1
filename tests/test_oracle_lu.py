"""Pins for the oracle's LU (numerics.md s.5; Eq. 2; BJ:11) -- special cases,
closed forms and invariants (SURVEY.md s.8(c.3) LU row). CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import ddqd_inputs as gen
from tests.util import EPS_DD, frac


def _b_of_ones(orc, A):
    n = A.shape[1]
    ones = np.zeros((2, n, 1)); ones[0] = 1.0
    return orc.gemm(A, ones, "block")[:, :, 0]


def _perm_rows(A, ipiv):
    PA = A.copy()
    for k, r in enumerate(ipiv):
        if r != k:
            PA[:, [k, r], :] = PA[:, [r, k], :]
    return PA


def _split_LU(LU):
    n = LU.shape[1]
    L = np.zeros_like(LU); U = np.zeros_like(LU)
    tri = np.tril(np.ones((n, n), bool), -1)
    L[:, tri] = LU[:, tri]; L[0, np.arange(n), np.arange(n)] = 1.0
    U[:, ~tri] = LU[:, ~tri]
    return L, U


def _residual_ok(orc, A, LU, ipiv, factor=100):
    """||PA - LU||_inf <= factor n eps ||A||_inf, with L*U formed exactly (long accumulator)."""
    n = A.shape[1]
    L, U = _split_LU(LU)
    PA = _perm_rows(A, ipiv)
    rows, cols = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ex, err = orc.exact_entries(L, U, PA, rows.ravel(), cols.ravel())   # err = LU - PA exactly
    resid = np.abs(err).reshape(n, n).sum(axis=1).max()
    normA = np.abs(A[0]).sum(axis=1).max()
    return resid <= factor * n * 2.0 ** -104 * normA, resid / normA


def test_identity(orc):
    """A = I -> L = U = I, x = b, no interchanges."""
    n = 12
    A = np.zeros((2, n, n)); A[0] = np.eye(n)
    b = gen.dd_matrix(1, n, 3, 1)[:, 0, :]
    x, LU, ipiv, info = orc.solve(A, b, panel=4, algo="strassen", threshold=1)
    assert info == 0 and np.array_equal(ipiv, np.arange(n))
    assert np.array_equal(LU, A) and np.array_equal(x, b)


def test_2x2_pivoting_example(orc):
    """From S:313 with partial pivoting: [[4,3],[6,3]] swaps rows; L21 = 2/3 (DD); U = [[6,3],[0,1]]."""
    A = np.zeros((2, 2, 2)); A[0] = [[4, 3], [6, 3]]
    LU, ipiv, info = orc.lu(A, panel=1, algo="block")
    assert info == 0 and list(ipiv) == [1, 1]
    assert LU[0, 0, 0] == 6 and LU[0, 0, 1] == 3
    assert abs(frac(LU[:, 1, 0]) - Fraction(2, 3)) <= 2 * EPS_DD
    assert abs(frac(LU[:, 1, 1]) - 1) <= 4 * EPS_DD


def test_panel_1_block_update_equals_unblocked_bitwise(orc):
    """K = 1 with Block update: T = l*u from +0 is exactly dd_mul(l,u), so the factorisation
    is bitwise the unblocked (K >= n) one."""
    A = gen.dd_matrix(40, 40, 6, 0)
    LU1, p1, _ = orc.lu(A, panel=1, algo="block")
    LUn, pn, _ = orc.lu(A, panel=64, algo="block")
    assert np.array_equal(LU1, LUn) and np.array_equal(p1, pn)


@pytest.mark.parametrize("algo,T", [("block", 32), ("strassen", 8), ("winograd", 8)])
def test_c4_like_diagonally_dominant(orc, algo, T):
    """BJ:11 recipe at n = 96: A = R + n I is column diagonally dominant, so partial pivoting
    performs no interchanges (ipiv = identity); PA = LU within 100 n eps |A|; x ~ 1."""
    n = 96
    A = gen.lu_matrix(n, 5)
    b = _b_of_ones(orc, A)
    x, LU, ipiv, info = orc.solve(A, b, panel=32, algo=algo, threshold=T)
    assert info == 0 and np.array_equal(ipiv, np.arange(n))
    ok, rel = _residual_ok(orc, A, LU, ipiv)
    assert ok, rel
    err = np.abs((x[0] - 1.0) + x[1]).max()
    assert err <= 2.0 ** -96 * n * 3 * 18


def test_pivoting_path_random_matrix(orc):
    """Non-dominant random matrix: interchanges happen, |l_ij| <= 1, PA = LU within bound."""
    n = 64
    A = gen.dd_matrix(n, n, 12, 0)
    LU, ipiv, info = orc.lu(A, panel=16, algo="strassen", threshold=4)
    assert info == 0
    assert np.any(ipiv != np.arange(n))
    tri = np.tril(np.ones((n, n), bool), -1)
    assert np.all(np.abs(LU[0][tri]) <= 1.0)
    ok, rel = _residual_ok(orc, A, LU, ipiv)
    assert ok, rel
    # pivot choice is the max magnitude: the first column's pivot row is argmax |a_i0|
    assert ipiv[0] == int(np.argmax(np.abs(A[0, :, 0])))


def test_update_algorithms_agree(orc):
    """P:164 'cannot determine the increase in relative errors': Block vs Strassen vs Winograd
    updates give solutions within the same bound."""
    n = 80
    A = gen.lu_matrix(n, 7)
    b = _b_of_ones(orc, A)
    runs = [orc.solve(A, b, panel=16, algo=a, threshold=4) for a in ("block", "strassen", "winograd")]
    for x, LU, ipiv, info in runs:
        assert np.abs((x[0] - 1.0) + x[1]).max() <= 2.0 ** -90
        assert _residual_ok(orc, A, LU, ipiv)[0]
    assert not np.array_equal(runs[0][1], runs[1][1])    # different summation trees


def test_zero_pivot_info(orc):
    """Exactly singular structure: info = k+1 for the first zero pivot (LAPACK convention)."""
    n = 6
    A = gen.dd_matrix(n, n, 2, 0)
    A[:, :, 2] = 0.0                      # column 2 zero -> pivot at k = 2 is zero
    LU, ipiv, info = orc.lu(A, panel=4, algo="block")
    assert info == 3


def test_tie_lowest_index(orc):
    A = np.zeros((2, 3, 3)); A[0] = [[1, 0, 0], [-2, 1, 0], [2, 0, 1]]
    _, ipiv, _ = orc.lu(A, panel=3, algo="block")
    assert ipiv[0] == 1


# ---- QD LU and the paper's pivot-free mode ---------------------
def test_qd_div(orc):
    """mul(div(1,7),7) within 16 eps_qd of 1; random quotients (calibrated 2^-205)."""
    from tests.util import EPS_QD
    one = np.zeros((4, 1)); one[0] = 1.0
    seven = np.zeros((4, 1)); seven[0] = 7.0
    q = orc.qd_div(one, seven)
    assert abs(frac(orc.qd_op("mul", q, seven)[:, 0]) - 1) <= 16 * EPS_QD
    assert abs(frac(q[:, 0]) - Fraction(1, 7)) <= 4 * EPS_QD
    x = gen.qd_matrix(1, 400, 3, 0).reshape(4, -1)
    y = gen.qd_matrix(1, 400, 4, 0).reshape(4, -1)
    z = orc.qd_div(x, y)
    for i in range(400):
        X, Y = frac(x[:, i]), frac(y[:, i])
        assert abs(frac(z[:, i]) - X / Y) <= Fraction(1, 2 ** 205) * abs(X / Y)


def _qd_lu_matrix(n, seed, shift=True):
    A = gen.qd_matrix(n, n, seed, 0)
    if shift:
        A[0, np.arange(n), np.arange(n)] += n     # exact: |w0| < 1 and n a small integer
    return A


def test_qd_lu_identity_and_2x2(orc):
    n = 9
    A = np.zeros((4, n, n)); A[0] = np.eye(n)
    b = gen.qd_matrix(1, n, 3, 1)[:, 0, :]
    x, LU, ipiv, info = orc.solve(A, b, panel=4, algo="winograd", threshold=1)
    assert info == 0 and np.array_equal(x, b)
    A2 = np.zeros((4, 2, 2)); A2[0] = [[4, 3], [6, 3]]
    LU, ipiv, info = orc.lu(A2, panel=1, algo="block")
    assert list(ipiv) == [1, 1]
    from tests.util import EPS_QD
    assert abs(frac(LU[:, 1, 0]) - Fraction(2, 3)) <= 2 * EPS_QD


def test_qd_lu_residual_and_solution(orc):
    """QD LU with a Winograd update: ||PA - LU|| (exact) <= 100 n eps_qd ||A||; x = 1 within
    2^-200 n kappa 18."""
    n = 48
    A = _qd_lu_matrix(n, 7)
    ones = np.zeros((4, n, 1)); ones[0] = 1.0
    b = orc.gemm(A, ones, "block")[:, :, 0].copy()
    x, LU, ipiv, info = orc.solve(A, b, panel=16, algo="winograd", threshold=4)
    assert info == 0 and np.array_equal(ipiv, np.arange(n))
    L, U = _split_LU(LU)
    L[1:, np.arange(n), np.arange(n)] = 0.0
    r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    _, err = orc.exact_entries(L, U, _perm_rows(A, ipiv), r.ravel(), c.ravel())
    normA = np.abs(A[0]).sum(axis=1).max()
    assert np.abs(err).reshape(n, n).sum(axis=1).max() <= 100 * n * 2.0 ** -209 * normA
    err_x = max(abs(frac(x[:, i]) - 1) for i in range(n))
    assert err_x <= Fraction(1, 2 ** 200) * n * 3 * 18


def test_pivot_free_mode(orc):
    """P:121 pivot-free LU: ipiv = identity always; on a diagonally dominant matrix it equals
    the pivoted factorisation bitwise (no interchange happens there either)."""
    for W in (2, 4):
        n = 40
        A = gen.lu_matrix(n, 3) if W == 2 else _qd_lu_matrix(n, 3)
        LUp, pp, _ = orc.lu(A, panel=8, algo="strassen", threshold=4, pivot=True)
        LUf, pf, _ = orc.lu(A, panel=8, algo="strassen", threshold=4, pivot=False)
        assert np.array_equal(pf, np.arange(n)) and np.array_equal(LUp, LUf)
    # a random (non-dominant) matrix: pivot-free still factors it, with |l_ij| > 1 somewhere
    A = gen.dd_matrix(30, 30, 12, 0)
    LU, piv, info = orc.lu(A, panel=8, algo="block", pivot=False)
    assert info == 0 and np.array_equal(piv, np.arange(30))
    assert np.abs(LU[0][np.tril(np.ones((30, 30), bool), -1)]).max() > 1.0
    assert _residual_ok(orc, A, LU, piv, factor=1e6)[0]
