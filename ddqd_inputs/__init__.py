"""Seeded synthetic inputs shared by the oracle tests, the GPU tests, smoke() and bench.py.

Harness data only: this module holds none of the method's arithmetic (no GEMM,
no DD/QD multiply, no LU). It writes out the input recipes of BASELINE.json
configs (BJ:7 DD entries, BJ:9 QD entries, BJ:11 LU matrix) and the paper's
benchmark pair, as specified in docs/numerics.md section 6.
Neither `oracle/` nor the CUDA package imports it; callers pass its arrays to
both sides.

Layout: planar row-major float64, shape [W, rows, cols] (W = 2 for DD, 4 for QD).
"""
from __future__ import annotations

from fractions import Fraction
from math import isqrt

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M52 = 2.0 ** -52
_TWO_M53 = 2.0 ** -53
TAG_A, TAG_B = 0, 1
_CHUNK = 1 << 22


def mix64(z):
    """SplitMix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def _key(seed: int, tag: int) -> np.uint64:
    with np.errstate(over="ignore"):
        t = mix64(np.array([tag], dtype=np.uint64))[0]
        return mix64(np.array([np.uint64(seed) ^ t], dtype=np.uint64))[0]


def uniform(seed: int, tag: int, draws) -> np.ndarray:
    """U(-1,1) draws number `draws` (uint64 array) of stream (seed, tag); exact."""
    key = _key(seed, tag)
    d = np.asarray(draws, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = mix64(key + (d + np.uint64(1)) * GAMMA)
    return (x >> np.uint64(11)).astype(np.float64) * _TWO_M52 - 1.0


def _two_sum(a, b):
    s = a + b
    bb = s - a
    e = (a - (s - bb)) + (b - bb)
    return s, e


def _fast_two_sum(a, b):
    s = a + b
    e = b - (s - a)
    return s, e


def _renorm4(c0, c1, c2, c3, c4):
    """Input-side renormalisation of a 5-word expansion to 4 non-overlapping words
    (docs/numerics.md s.3 qd_renorm, evaluated on all branches and selected with masks)."""
    s, t4 = _fast_two_sum(c3, c4)
    s, t3 = _fast_two_sum(c2, s)
    s, t2 = _fast_two_sum(c1, s)
    t0, t1 = _fast_two_sum(c0, s)
    z = np.zeros_like(t0)
    # case s1 != 0
    a1, a2 = _fast_two_sum(t1, t2)
    b2, b3 = _fast_two_sum(a2, t3)
    c1_, c2_ = _fast_two_sum(a1, t3)
    d2, d3 = _fast_two_sum(c2_, t4)
    e1, e2 = _fast_two_sum(c1_, t4)
    A_a2 = a2 != 0
    A_b3 = b3 != 0
    A_c2 = c2_ != 0
    A1 = np.where(A_a2, a1, np.where(A_c2, c1_, e1))
    A2 = np.where(A_a2, np.where(A_b3, b2, b2 + t4), np.where(A_c2, d2, e2))
    A3 = np.where(A_a2, np.where(A_b3, b3 + t4, z), np.where(A_c2, d3, z))
    # case s1 == 0
    f0, f1 = _fast_two_sum(t0, t2)
    g1, g2 = _fast_two_sum(f1, t3)
    h2, h3 = _fast_two_sum(g2, t4)
    i1, i2 = _fast_two_sum(g1, t4)
    j0, j1 = _fast_two_sum(f0, t3)
    k1, k2 = _fast_two_sum(j1, t4)
    l0, l1 = _fast_two_sum(j0, t4)
    B_f1 = f1 != 0
    B_g2 = g2 != 0
    B_j1 = j1 != 0
    B0 = np.where(B_f1, f0, np.where(B_j1, j0, l0))
    B1 = np.where(B_f1, np.where(B_g2, g1, i1), np.where(B_j1, k1, l1))
    B2 = np.where(B_f1, np.where(B_g2, h2, i2), np.where(B_j1, k2, z))
    B3 = np.where(B_f1 & B_g2, h3, z)
    nz = t1 != 0
    return (np.where(nz, t0, B0), np.where(nz, A1, B1),
            np.where(nz, A2, B2), np.where(nz, A3, B3))


def _words(rows: int, cols: int, seed: int, tag: int, W: int) -> np.ndarray:
    """Raw draws: returns array [W, rows*cols] of U(-1,1), draw d = e*W + w."""
    n = rows * cols
    out = np.empty((W, n), dtype=np.float64)
    for lo in range(0, n, _CHUNK):
        hi = min(n, lo + _CHUNK)
        e = np.arange(lo, hi, dtype=np.uint64)
        for w in range(W):
            out[w, lo:hi] = uniform(seed, tag, e * np.uint64(W) + np.uint64(w))
    return out


def dd_matrix(rows: int, cols: int, seed: int, tag: int) -> np.ndarray:
    """BJ:7: hi ~ U(-1,1), lo = hi*2^-53*U(-1,1), then (hi,lo) := TwoSum(hi,lo)."""
    u = _words(rows, cols, seed, tag, 2)
    hi = u[0]
    lo = (hi * _TWO_M53) * u[1]
    hi, lo = _two_sum(hi, lo)
    out = np.empty((2, rows, cols), dtype=np.float64)
    out[0] = hi.reshape(rows, cols)
    out[1] = lo.reshape(rows, cols)
    return out


def qd_matrix(rows: int, cols: int, seed: int, tag: int) -> np.ndarray:
    """BJ:9: w0 ~ U(-1,1), w_k = w_{k-1}*2^-53*U(-1,1), renormalised."""
    u = _words(rows, cols, seed, tag, 4)
    w = [u[0]]
    for k in range(1, 4):
        w.append((w[k - 1] * _TWO_M53) * u[k])
    s = _renorm4(w[0], w[1], w[2], w[3], np.zeros_like(w[0]))
    out = np.empty((4, rows, cols), dtype=np.float64)
    for k in range(4):
        out[k] = s[k].reshape(rows, cols)
    return out


def matrix(W: int, rows: int, cols: int, seed: int, tag: int) -> np.ndarray:
    if W == 2:
        return dd_matrix(rows, cols, seed, tag)
    if W == 4:
        return qd_matrix(rows, cols, seed, tag)
    raise ValueError("W must be 2 (DD) or 4 (QD)")


def lu_matrix(n: int, seed: int) -> np.ndarray:
    """BJ:11: DD entries as BJ:7 (tag 0) plus n*I, i.e. dd_add(a_ii, (n, 0)) written out."""
    a = dd_matrix(n, n, seed, TAG_A)
    idx = np.arange(n)
    hi = a[0, idx, idx].copy()
    lo = a[1, idx, idx].copy()
    s, e = _two_sum(hi, np.full(n, float(n)))
    e = e + lo
    s, e = _fast_two_sum(s, e)
    a[0, idx, idx] = s
    a[1, idx, idx] = e
    return a


def _round_expansion(x: Fraction, W: int) -> list:
    words = []
    r = x
    for _ in range(W):
        f = float(r)
        words.append(f)
        r = r - Fraction(f)
    return words


def _sqrt_frac(N: int, bits: int = 400) -> Fraction:
    return Fraction(isqrt(N << (2 * bits)), 1 << bits)


def bench_pair(n: int, W: int):
    """Paper benchmark pair: A = [sqrt5 (i+j-1)], B = [sqrt3 (n-i)], 1-based.

    Each entry is the W-word round-to-nearest expansion of the exact real value.
    """
    av = {}
    for k in range(1, 2 * n):
        av[k] = _round_expansion(_sqrt_frac(5 * k * k), W)
    bv = {}
    for k in range(0, n):
        bv[k] = _round_expansion(_sqrt_frac(3 * k * k), W) if k else [0.0] * W
    A = np.empty((W, n, n))
    B = np.empty((W, n, n))
    i = np.arange(1, n + 1)
    ksum = i[:, None] + i[None, :] - 1
    for w in range(W):
        lut = np.zeros(2 * n)
        for k, v in av.items():
            lut[k] = v[w]
        A[w] = lut[ksum]
        lutb = np.array([bv[n - r][w] for r in range(1, n + 1)])
        B[w] = np.repeat(lutb[:, None], n, axis=1)
    return A, B


def bench_pair_exact(n: int, i: int) -> Fraction:
    """Integer part S(i,n) of c_ij = sqrt(15) * S(i,n), exact; 1-based i."""
    return Fraction(sum((i + k - 1) * (n - k) for k in range(1, n + 1)))
