"""Test helpers: exact rationals of DD/QD words, norms, bounds (no method arithmetic)."""
from fractions import Fraction

import numpy as np

EPS_DD = Fraction(1, 2 ** 104)
EPS_QD = Fraction(1, 2 ** 209)


def frac(words):
    """Exact value of an expansion given as a sequence of doubles."""
    return sum((Fraction(float(w)) for w in words), Fraction(0))


def frac_mat(M):
    """[W, r, c] -> list of lists of Fractions."""
    W, r, c = M.shape
    return [[frac(M[:, i, j]) for j in range(c)] for i in range(r)]


def exact_product(A, B):
    Fa, Fb = frac_mat(A), frac_mat(B)
    m, l, n = A.shape[1], A.shape[2], B.shape[2]
    return [[sum((Fa[i][k] * Fb[k][j] for k in range(l)), Fraction(0)) for j in range(n)] for i in range(m)]


def maxabs_words(M):
    """max-norm of the represented values (|sum of words|), as a float upper estimate."""
    return float(np.max(np.abs(M.sum(axis=0)))) if M.size else 0.0


def is_normalised(M):
    """Non-overlap: fl(w_i + w_{i+1}) == w_i for all adjacent words."""
    W = M.shape[0]
    ok = True
    for w in range(W - 1):
        ok &= bool(np.all(M[w] + M[w + 1] == M[w]))
    return ok


def rec_depth(m, l, n, T):
    d = 0
    while min(m, l, n) > T:
        m, l, n = (m + 1) // 2, (l + 1) // 2, (n + 1) // 2
        d += 1
    return d


def rand_dd(rng, n, scale_exp=(-20, 20)):
    """Random normalised DD numbers with varied exponents (for arithmetic pins)."""
    hi = rng.uniform(-1, 1, n) * np.exp2(rng.integers(scale_exp[0], scale_exp[1], n))
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, n)
    s = hi + lo
    bb = s - hi
    e = (hi - (s - bb)) + (lo - bb)
    return np.stack([s, e])
