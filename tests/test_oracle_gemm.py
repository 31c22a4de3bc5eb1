"""Pins for the oracle's GEMM layer (numerics.md s.4): Simple/Block/Strassen/Winograd
against exact rationals, closed forms, special cases and count laws
(SURVEY.md s.8(c.3) rows 4-6). CPU only."""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import ddqd_inputs as gen
from tests.util import exact_product, frac, is_normalised, rec_depth

ALGOS = ("block", "strassen", "winograd")


def _int_mat(W, rows, cols, rng, lo=-9, hi=10):
    M = np.zeros((W, rows, cols))
    M[0] = rng.integers(lo, hi, (rows, cols))
    return M


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ALGOS)
def test_2x2_integer_product(orc, W, algo):
    """[[1,2],[3,4]] [[5,6],[7,8]] = [[19,22],[43,50]] exactly, every algorithm."""
    A = np.zeros((W, 2, 2)); A[0] = [[1, 2], [3, 4]]
    B = np.zeros((W, 2, 2)); B[0] = [[5, 6], [7, 8]]
    C = orc.gemm(A, B, algo, threshold=1)
    assert C[0].tolist() == [[19, 22], [43, 50]]
    assert np.all(C[1:] == 0)


@pytest.mark.parametrize("W,bound_exp", [(2, -96), (4, -200)])
def test_simple_vs_exact_small_shapes(orc, W, bound_exp):
    """Exact Fraction product for every m,l,n in 1..5: max-norm error <= 2^e l |A| |B| (BJ:5)."""
    rng = 0
    for m, l, n in itertools.product(range(1, 6), repeat=3):
        rng += 1
        A = gen.matrix(W, m, l, rng, 0)
        B = gen.matrix(W, l, n, rng, 1)
        C = orc.gemm(A, B, "block")
        assert is_normalised(C)
        E = exact_product(A, B)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(2) ** bound_exp * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound


def test_exact_accumulator_matches_fractions(orc):
    """The long accumulator (oracle/exact.c) agrees with Python Fractions exactly (to rounding)."""
    for W in (2, 4):
        A = gen.matrix(W, 6, 7, 3, 0)
        B = gen.matrix(W, 7, 5, 3, 1)
        C = orc.gemm(A, B, "block")
        E = exact_product(A, B)
        rows, cols = np.meshgrid(np.arange(6), np.arange(5), indexing="ij")
        ex, err = orc.exact_entries(A, B, C, rows.ravel(), cols.ravel())
        for t, (i, j) in enumerate(zip(rows.ravel(), cols.ravel())):
            assert ex[t] == float(E[i][j])
            assert err[t] == float(E[i][j] - frac(C[:, i, j]))


@pytest.mark.parametrize("W", [2, 4])
def test_block_equals_simple_bitwise(orc, W):
    """Block(bs) tiles only the loop nest; bitwise equal to Simple."""
    for (m, l, n) in [(33, 17, 29), (64, 64, 64), (5, 70, 3)]:
        A = gen.matrix(W, m, l, 7, 0)
        B = gen.matrix(W, l, n, 7, 1)
        C0 = orc.gemm(A, B, "block")
        for bs in (1, 4, 16, 32, 100):
            assert np.array_equal(orc.gemm(A, B, "block", bs=bs), C0)


@pytest.mark.parametrize("W", [2, 4])
def test_identity_and_permutation_exact(orc, W):
    """BJ:5: identity/permutation products are exact (Block/Simple)."""
    n = 37
    A = gen.matrix(W, n, n, 5, 0)
    I = np.zeros((W, n, n)); I[0] = np.eye(n)
    assert np.array_equal(orc.gemm(A, I, "block"), A)
    assert np.array_equal(orc.gemm(I, A, "block"), A)
    perm = np.random.default_rng(1).permutation(n)
    P = np.zeros((W, n, n)); P[0, np.arange(n), perm] = 1.0
    assert np.array_equal(orc.gemm(P, A, "block"), A[:, perm, :])


def test_power_of_two_scaling_bitwise(orc):
    A = gen.dd_matrix(20, 30, 1, 0)
    B = gen.dd_matrix(30, 25, 1, 1)
    for algo in ALGOS:
        C = orc.gemm(A, B, algo, threshold=4)
        C2 = orc.gemm(A * 2.0 ** 5, B * 2.0 ** -3, algo, threshold=4)
        assert np.array_equal(C2, C * 4.0)


@pytest.mark.parametrize("W", [2, 4])
def test_paper_benchmark_pair_closed_form(orc, W):
    """P:61 pair: c_ij = sqrt15 * S(i,n), S from exact integers;
    columns bitwise identical since B's columns are equal."""
    n = 48
    A, B = gen.bench_pair(n, W)
    # examples of S:176-177
    assert gen.bench_pair_exact(2, 1) == 1 and gen.bench_pair_exact(3, 2) == 7
    eps = Fraction(1, 2 ** 104) if W == 2 else Fraction(1, 2 ** 209)
    r15 = Fraction(math.isqrt(15 << 1200), 1 << 600)     # sqrt(15) to 2^-600
    for algo in ALGOS:
        C = orc.gemm(A, B, algo, threshold=5)
        if algo == "block":
            assert np.all(C == C[:, :, :1])
        for i in range(n):
            ex = r15 * gen.bench_pair_exact(n, i + 1)
            got = frac(C[:, i, 0])
            depth = rec_depth(n, n, n, 5) if algo != "block" else 0
            assert abs(got - ex) <= 4 * n * eps * abs(ex) * 18 ** depth + Fraction(1, 2 ** 500)


def test_benchmark_pair_dd_n128_1e28(orc):
    """DD bench pair at n = 128 matches the closed form within 1e-28 (relative)."""
    n = 128
    A, B = gen.bench_pair(n, 2)
    r15 = Fraction(math.isqrt(15 << 1200), 1 << 600)
    for algo in ALGOS:
        C = orc.gemm(A, B, algo, threshold=32)
        for i in range(n):
            ex = r15 * gen.bench_pair_exact(n, i + 1)
            assert abs(frac(C[:, i, 7]) - ex) <= Fraction(1, 10 ** 28) * abs(ex)


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_threshold_ge_dims_is_block(orc, W, algo):
    """BJ:5: threshold >= min(m,l,n) degenerates to Block, bitwise."""
    A = gen.matrix(W, 19, 23, 2, 0)
    B = gen.matrix(W, 23, 21, 2, 1)
    assert np.array_equal(orc.gemm(A, B, algo, threshold=19), orc.gemm(A, B, "block"))


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_recursive_vs_exact_forced_depth(orc, algo):
    """m,l,n <= 16 with T in {1,2,3} (odd padding at several levels) within
    18^d 2^-96 l |A| |B| of the exact product (BJ:5)."""
    cases = [(16, 16, 16), (7, 9, 5), (13, 11, 15), (3, 16, 9), (10, 3, 12)]
    for (m, l, n), T in itertools.product(cases, (1, 2, 3)):
        A = gen.dd_matrix(m, l, m * 100 + T, 0)
        B = gen.dd_matrix(l, n, m * 100 + T, 1)
        C = orc.gemm(A, B, algo, threshold=T)
        E = exact_product(A, B)
        d = rec_depth(m, l, n, T)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(18) ** d * Fraction(1, 2 ** 96) * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ALGOS)
def test_integer_inputs_exact(orc, W, algo):
    """Small-integer inputs: every intermediate sum is exact, so every algorithm is exact
    (SURVEY c.3: identity products exact only on exact-sum inputs for S/W)."""
    rng = np.random.default_rng(3)
    for (m, l, n) in [(17, 9, 13), (32, 32, 32), (5, 31, 6)]:
        A = _int_mat(W, m, l, rng)
        B = _int_mat(W, l, n, rng)
        C = orc.gemm(A, B, algo, threshold=2)
        assert np.array_equal(C[0], A[0] @ B[0])
        assert np.all(C[1:] == 0)


def test_strassen_identity_inexact_on_general_dd(orc):
    """Documented qualification of BJ:5: Strassen(T=1)*I on random DD need not be exact."""
    n = 16
    A = gen.dd_matrix(n, n, 8, 0)
    I = np.zeros((2, n, n)); I[0] = np.eye(n)
    C = orc.gemm(A, I, "strassen", threshold=1)
    nA = float(np.abs(A[0]).max())
    assert np.max(np.abs((C[0] - A[0]) + (C[1] - A[1]))) <= 18 ** 4 * 2.0 ** -96 * n * nA


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_padding_transparency(orc, algo):
    """odd-size result equals the explicitly zero-padded even-size run, cropped."""
    m, l, n, T = 37, 29, 33, 4
    A = gen.dd_matrix(m, l, 4, 0)
    B = gen.dd_matrix(l, n, 4, 1)
    Ap = np.zeros((2, m + 1, l + 1)); Ap[:, :m, :l] = A
    Bp = np.zeros((2, l + 1, n + 1)); Bp[:, :l, :n] = B
    C = orc.gemm(A, B, algo, threshold=T)
    Cp = orc.gemm(Ap, Bp, algo, threshold=T)
    assert np.array_equal(C, Cp[:, :m, :n])


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_count_law(orc, algo):
    """leaf madds = 7^d T^3 at n = T 2^d; 18 vs 15 block adds per level."""
    A = gen.dd_matrix(64, 64, 1, 0)
    B = gen.dd_matrix(64, 64, 1, 1)
    orc.reset_counters()
    orc.gemm(A, B, algo, threshold=32)
    madds, adds = orc.counters()
    assert madds == 7 * 32 ** 3 == 229376
    assert adds == (18 if algo == "strassen" else 15)
    A = gen.dd_matrix(256, 256, 1, 0)
    B = gen.dd_matrix(256, 256, 1, 1)
    orc.reset_counters()
    orc.gemm(A, B, algo, threshold=32)
    madds, adds = orc.counters()
    assert madds == 7 ** 3 * 32 ** 3 == 11239424
    assert adds == (18 if algo == "strassen" else 15) * (1 + 7 + 49)
    orc.reset_counters()
    orc.gemm(A, B, "block")
    assert orc.counters()[0] == 256 ** 3


def test_zero_sizes(orc):
    A = np.zeros((2, 3, 0)); B = np.zeros((2, 0, 4))
    assert np.array_equal(orc.gemm(A, B, "block"), np.zeros((2, 3, 4)))
    assert orc.gemm(np.zeros((2, 0, 5)), np.zeros((2, 5, 2)), "strassen", 1).shape == (2, 0, 2)
    with pytest.raises(ValueError):
        orc.gemm(np.zeros((2, 3, 4)), np.zeros((2, 5, 2)))


def test_strassen_c1_shape_error_vs_exact_sampled(orc):
    """c1-like shape at reduced size: Strassen/Winograd error vs the exact product on sampled
    entries within 18^d 2^-96 l |A| |B|, and the measured error-to-bound ratio is tiny."""
    n, T = 256, 32
    A = gen.dd_matrix(n, n, 2, 0)
    B = gen.dd_matrix(n, n, 2, 1)
    rng = np.random.default_rng(0)
    rows, cols = rng.integers(0, n, 300), rng.integers(0, n, 300)
    nA, nB = float(np.abs(A[0]).max()), float(np.abs(B[0]).max())
    for algo in ALGOS:
        C = orc.gemm(A, B, algo, threshold=T)
        _, err = orc.exact_entries(A, B, C, rows, cols)
        d = 0 if algo == "block" else rec_depth(n, n, n, T)
        bound = 18.0 ** d * 2.0 ** -96 * n * nA * nB
        assert np.max(np.abs(err)) <= bound
        assert np.max(np.abs(err)) <= bound * 2.0 ** -8


@pytest.mark.parametrize("algo", ALGOS)
def test_fused_madd_gemm_vs_exact(orc, algo):
    """Fused-madd variant (row f3): every algorithm within 18^d 2^-96 l |A||B| of the exact
    product; integer inputs still exact; it changes bits relative to the canonical madd."""
    cases = [(13, 11, 15, 3), (16, 16, 16, 2), (7, 9, 5, 1)]
    for (m, l, n, T) in cases:
        A = gen.dd_matrix(m, l, m + 7, 0)
        B = gen.dd_matrix(l, n, m + 7, 1)
        C = orc.gemm(A, B, algo, threshold=T, madd="fused")
        E = exact_product(A, B)
        d = 0 if algo == "block" else rec_depth(m, l, n, T)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(18) ** d * Fraction(1, 2 ** 96) * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound
    A = gen.dd_matrix(40, 40, 3, 0)
    assert not np.array_equal(orc.gemm(A, A, algo, 8, madd="fused"), orc.gemm(A, A, algo, 8))
    rng = np.random.default_rng(3)
    Ai = _int_mat(2, 17, 9, rng)
    Bi = _int_mat(2, 9, 13, rng)
    assert np.array_equal(orc.gemm(Ai, Bi, algo, 2, madd="fused")[0], Ai[0] @ Bi[0])


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ALGOS)
def test_accurate_add_gemm_vs_exact(orc, W, algo):
    """Accurate-add variant (row f3; every addition of the madd and of the Strassen/Winograd
    combinations is the accurate add): within 18^d 2^-96 l |A||B| (QD: 2^-200) of the exact
    product; Block == Simple bitwise; threshold >= dims is Block; integer inputs exact; it
    changes bits relative to the canonical arithmetic."""
    cases = [(13, 11, 15, 3), (16, 16, 16, 2), (7, 9, 5, 1)]
    base = 96 if W == 2 else 200
    for (m, l, n, T) in cases:
        A = gen.matrix(W, m, l, m + 9, 0)
        B = gen.matrix(W, l, n, m + 9, 1)
        C = orc.gemm(A, B, algo, threshold=T, madd="accurate")
        E = exact_product(A, B)
        d = 0 if algo == "block" else rec_depth(m, l, n, T)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(18) ** d * Fraction(1, 2 ** base) * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound
    A = gen.matrix(W, 40, 40, 5, 0)
    assert not np.array_equal(orc.gemm(A, A, algo, 8, madd="accurate"), orc.gemm(A, A, algo, 8))
    if algo == "block":
        for bs in (1, 3, 16):
            assert np.array_equal(orc.gemm(A, A, "block", bs=bs, madd="accurate"), orc.gemm(A, A, "block", madd="accurate"))
    else:
        assert np.array_equal(orc.gemm(A, A, algo, 40, madd="accurate"), orc.gemm(A, A, "block", madd="accurate"))
    rng = np.random.default_rng(4)
    Ai = _int_mat(W, 17, 9, rng)
    Bi = _int_mat(W, 9, 13, rng)
    assert np.array_equal(orc.gemm(Ai, Bi, algo, 2, madd="accurate")[0], Ai[0] @ Bi[0])


def test_accurate_variant_rejections(orc):
    """The accurate-add variant is a GEMM variant: the LU (whose panel/TRSM/solve arithmetic
    is canonical) rejects it; fused + accurate together are rejected."""
    A = gen.dd_matrix(8, 8, 1, 0)
    with pytest.raises(ValueError):
        orc.lu(A, panel=4, madd="accurate")
    with pytest.raises(ValueError):
        orc.gemm(A, A, orc.BLOCK | orc.MADD_FUSED | orc.ADD_ACCURATE)


@pytest.mark.parametrize("algo", ALGOS)
def test_fused_madd_qd_gemm_vs_exact(orc, algo):
    """Fused QD madd variant (row f3): every algorithm within 18^d 2^-200 l |A||B| of the
    exact product; integer inputs exact; Block == Simple."""
    for (m, l, n, T) in [(13, 11, 15, 3), (9, 16, 7, 1)]:
        A = gen.qd_matrix(m, l, m + 11, 0)
        B = gen.qd_matrix(l, n, m + 11, 1)
        C = orc.gemm(A, B, algo, threshold=T, madd="fused")
        E = exact_product(A, B)
        d = 0 if algo == "block" else rec_depth(m, l, n, T)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(18) ** d * Fraction(1, 2 ** 200) * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound
    rng = np.random.default_rng(5)
    Ai = _int_mat(4, 17, 9, rng)
    Bi = _int_mat(4, 9, 13, rng)
    assert np.array_equal(orc.gemm(Ai, Bi, algo, 2, madd="fused")[0], Ai[0] @ Bi[0])
    if algo == "block":
        A = gen.qd_matrix(20, 20, 2, 0)
        assert np.array_equal(orc.gemm(A, A, "block", bs=3, madd="fused"), orc.gemm(A, A, "block", madd="fused"))


def test_splitk_tree_order_pin(orc):
    """Split-k (numerics.md s.4, row a4): 1x4 . 4x1 DD products p = (1, 0, 2^-60 + 2^-120,
    -2^-60). The pairwise tree (p0+p1)+(p2+p3) keeps the 2^-120 (1 + 2^-120 is a DD value);
    the canonical k-ascending fold loses it when 2^-60 + 2^-120 meets 1 (121 bits). So
    s = 2, 4, 8 give exactly 1 + 2^-120 and the canonical Block exactly 1."""
    A = np.zeros((2, 1, 4)); A[0] = 1.0
    B = np.zeros((2, 4, 1))
    B[0, :, 0] = [1.0, 0.0, 2.0 ** -60, -2.0 ** -60]
    B[1, 2, 0] = 2.0 ** -120
    assert frac(orc.gemm(A, B, "block")[:, 0, 0]) == 1
    for s in (2, 4, 8):
        C = orc.gemm(A, B, "block", splitk=s)
        assert list(C[:, 0, 0]) == [1.0, 2.0 ** -120], s


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ALGOS)
def test_splitk_vs_exact(orc, W, algo):
    """Split-k leaves within 18^d 2^-96 l |A||B| (QD 2^-200) of the exact product for s = 2,
    4, 8 including slices that are empty (l < s); integer inputs exact; s = 1 is the canonical
    result; the count law is unchanged."""
    base = 96 if W == 2 else 200
    for (m, l, n, T, s) in [(9, 13, 7, 4, 4), (6, 3, 5, 2, 8), (16, 16, 16, 3, 2), (5, 1, 4, 1, 8)]:
        A = gen.matrix(W, m, l, m + 13, 0)
        B = gen.matrix(W, l, n, m + 13, 1)
        C = orc.gemm(A, B, algo, threshold=T, splitk=s)
        E = exact_product(A, B)
        d = 0 if algo == "block" else rec_depth(m, l, n, T)
        nA = max(abs(frac(A[:, i, k])) for i in range(m) for k in range(l))
        nB = max(abs(frac(B[:, k, j])) for k in range(l) for j in range(n))
        bound = Fraction(18) ** d * Fraction(1, 2 ** base) * l * nA * nB
        for i in range(m):
            for j in range(n):
                assert abs(frac(C[:, i, j]) - E[i][j]) <= bound, (m, l, n, s)
        assert np.array_equal(orc.gemm(A, B, algo, threshold=T, splitk=1), orc.gemm(A, B, algo, threshold=T))
    rng = np.random.default_rng(8)
    Ai = _int_mat(W, 17, 9, rng)
    Bi = _int_mat(W, 9, 13, rng)
    assert np.array_equal(orc.gemm(Ai, Bi, algo, 2, splitk=4)[0], Ai[0] @ Bi[0])
    orc.reset_counters()
    orc.gemm(gen.matrix(W, 16, 16, 1, 0), gen.matrix(W, 16, 16, 1, 1), algo, threshold=4, splitk=4)
    madds, _ = orc.counters()
    d = 0 if algo == "block" else rec_depth(16, 16, 16, 4)
    assert madds == 7 ** d * (16 // 2 ** d) ** 3
