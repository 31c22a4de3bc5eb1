"""Pins for the oracle's LU (numerics.md s.5; Eq. 2; BJ:11) -- special cases,
closed forms and invariants (SURVEY.md s.8(c.3) LU row). CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import ddqd_inputs as gen
from tests.util import EPS_DD, frac, frac_mat


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


# ---- pivot order with signs and y := P b on systems that do interchange --
def _round_expansion(F, W):
    """A W-word expansion of the rational F (each word the correctly rounded remainder)."""
    out = []
    for _ in range(W):
        w = float(F)
        out.append(w)
        F -= Fraction(w)
    return out


def _signed_qd(rng, n):
    """Random normalised QD values with mixed signs (leading words negative for ~half)."""
    A = gen.qd_matrix(1, n, int(rng.integers(1, 1 << 30)), 0).reshape(4, n)
    return A * rng.choice([-1.0, 1.0], n)


def test_qd_abs_order_unit_table(orc):
    """numerics.md s.3 QD magnitude order: the sign is folded on the leading word, then all four
    words are compared lexicographically. Each row would fail a plausible mistake: no sign
    fold (rows 1-2), a per-word fabs instead of a fold (rows 3-4), comparing only the leading
    word(s) (rows 5-6), '>=' instead of '>' (row 7)."""
    q = lambda *w: list(w) + [0.0] * (4 - len(w))
    t = 2.0 ** -60
    table = [
        (q(-0.75), q(0.5), True),                                   # negative but larger
        (q(0.5), q(-0.75), False),
        (q(0.75, -2.0 ** -55), q(0.75, t), False),                 # |.| = 0.75 - 2^-55 < 0.75 + 2^-60
        (q(-0.75, 2.0 ** -55), q(0.75, t), False),                 # folded: (0.75, -2^-55)
        (q(-0.75, -t, -2.0 ** -115), q(0.75, t, 2.0 ** -116), True),   # third word decides
        (q(0.75, t, 2.0 ** -115, -2.0 ** -170), q(-0.75, -t, -2.0 ** -115, -2.0 ** -171), False),
        (q(-0.75, -t, 2.0 ** -115, 2.0 ** -170), q(0.75, t, -2.0 ** -115, -2.0 ** -170), False),
    ]
    for x, y, want in table:
        assert orc.qd_abs_gt(x, y) == want, (x, y)
        assert abs(frac(x)) > abs(frac(y)) if want else abs(frac(x)) <= abs(frac(y))
    # random mixed-sign pairs sharing 1, 2 or 3 leading words: the order is |Fraction| order
    rng = np.random.default_rng(31)
    X = _signed_qd(rng, 600)
    Y = _signed_qd(rng, 600)
    for i in range(600):
        share = i % 4                       # 0: independent; 1..3: copy the leading words
        if share:
            s = np.sign(X[0, i]) * np.sign(Y[0, i])
            Y[:share, i] = X[:share, i] * s
        x, y = X[:, i], Y[:, i]
        assert orc.qd_abs_gt(x, y) == (abs(frac(x)) > abs(frac(y))), (x, y)


def _exact_pivots(A):
    """Partial pivoting in exact rationals (ties -> lowest row): the pivot sequence of the
    textbook elimination on the represented values of A [W, n, n]."""
    M = frac_mat(A)
    n = len(M)
    piv = []
    for k in range(n):
        r = max(range(k, n), key=lambda i: (abs(M[i][k]), -i))
        piv.append(r)
        M[k], M[r] = M[r], M[k]
        for i in range(k + 1, n):
            f = M[i][k] / M[k][k]
            for j in range(k, n):
                M[i][j] -= f * M[k][j]
    return piv


@pytest.mark.parametrize("W", [2, 4])
def test_pivot_sequence_matches_exact_elimination(orc, W):
    """Mixed-sign random matrices (about half the entries negative, and the QD ones sharing
    leading words across a column so lower words and signs decide): every pivot the oracle
    picks equals the exact-rational partial-pivoting choice (brute force, n = 12). The
    DD/QD elimination perturbs the reduced columns only at 2^-100 relative, far below the
    gaps between candidates of a random matrix."""
    n = 12
    rng = np.random.default_rng(7 + W)
    A = (gen.dd_matrix(n, n, 21, 0) if W == 2 else gen.qd_matrix(n, n, 21, 0))
    A = A * rng.choice([-1.0, 1.0], (1, n, n))
    if W == 4:   # column 0: equal leading words up to sign, the pivot decided below them
        A[:2, 1:6, 0] = A[:2, 0:1, 0] * rng.choice([-1.0, 1.0], 5)
    LU, ipiv, info = orc.lu(A, panel=4, algo="block")
    assert info == 0
    want = _exact_pivots(A)
    assert list(ipiv) == want
    assert any(r != k for k, r in enumerate(want))
    assert any(A[0, r, k] < 0 for k, r in enumerate(want))      # some pivots are negative


def test_column0_pivot_negative_entry(orc):
    """ipiv[0] = argmax |a_i0| where the largest magnitude is a negative entry."""
    for W in (2, 4):
        n = 6
        A = np.zeros((W, n, n))
        A[0] = np.eye(n)
        A[0, :, 0] = [0.25, 0.5, -0.875, 0.75, -0.125, 0.5]
        A[0, 0, 1] = 1.0
        LU, ipiv, info = orc.lu(A, panel=2, algo="block")
        assert ipiv[0] == 2 and info == 0


@pytest.mark.parametrize("W,algo,T", [(2, "strassen", 4), (2, "winograd", 3), (4, "winograd", 4),
                                      (4, "block", 16)])
def test_solve_nondominant_system_exact_rhs(orc, W, algo, T):
    """P:144 setting on a system that interchanges rows: x = [0..n-1], b := A x formed
    exactly (Fractions, rounded to a W-word expansion); the solve (y := P b with the swaps in
    ipiv order, then the two substitutions) returns x within 100 n kappa eps ||x||. Applying
    the swaps in reverse (or not at all) gives O(1) errors."""
    n = 24
    rng = np.random.default_rng(100 + W + T)
    A = (gen.dd_matrix(n, n, 40 + T, 0) if W == 2 else gen.qd_matrix(n, n, 40 + T, 0))
    A = A * rng.choice([-1.0, 1.0], (1, n, n))
    Fa = frac_mat(A)
    b = np.zeros((W, n))
    for i in range(n):
        b[:, i] = _round_expansion(sum((Fa[i][j] * j for j in range(n)), Fraction(0)), W)
    x, LU, ipiv, info = orc.solve(A, b, panel=8, algo=algo, threshold=T)
    assert info == 0
    swaps = [(k, int(r)) for k, r in enumerate(ipiv) if r != k]
    assert len(swaps) >= 3
    # the order of the swaps matters on this system (a reversed application differs)
    y_fwd, y_rev = list(range(n)), list(range(n))
    for k, r in swaps:
        y_fwd[k], y_fwd[r] = y_fwd[r], y_fwd[k]
    for k, r in reversed(swaps):
        y_rev[k], y_rev[r] = y_rev[r], y_rev[k]
    assert y_fwd != y_rev
    kappa = np.linalg.cond(A[0], np.inf)
    eps = 2.0 ** -104 if W == 2 else 2.0 ** -209
    err = max(abs(float(frac(x[:, i]) - i)) for i in range(n))
    assert err <= 100 * n * kappa * eps * (n - 1), (err, kappa)
