"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding for oracle/ddqd_oracle.c (DD/QD arithmetic, Simple/Block/Strassen/
Winograd GEMM, blocked LU with partial pivoting, following docs/numerics.md) and
oracle/exact.c (exact long accumulator). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package; the
product path (paper_1510_08642_b200) never does.

Parity status: see the header of ddqd_oracle.c ("QD op sequences: parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "ddqd_oracle.c"), os.path.join(_HERE, "exact.c")]
CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-shared", "-fPIC"]

BLOCK, STRASSEN, WINOGRAD = 0, 1, 2
ALGOS = {"block": BLOCK, "strassen": STRASSEN, "winograd": WINOGRAD}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no contraction, no fast-math)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, *_SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER(ctypes.c_double)
        PI = ctypes.POINTER(ctypes.c_int64)
        i64 = ctypes.c_int64
        for name in ("or_two_sum", "or_fast_two_sum", "or_two_prod"):
            getattr(L, name).argtypes = [i64, P, P, P, P]
        L.or_dd_op.argtypes = [ctypes.c_int, i64, P, P, P, P]
        L.or_qd_op.argtypes = [ctypes.c_int, i64, P, P, P, P]
        L.or_qd_renorm.argtypes = [i64, P, P]
        L.or_dd_abs_gt.argtypes = [P, P]
        L.or_qd_abs_gt.argtypes = [P, P]
        L.or_gemm.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, i64, i64, i64, P, P, P, ctypes.c_int]
        L.or_lu.argtypes = [ctypes.c_int, ctypes.c_int, i64, P, PI, i64, ctypes.c_int, i64, ctypes.c_int]
        L.or_lu_solve.argtypes = [ctypes.c_int, i64, P, PI, P, P]
        L.or_lu_panel.argtypes = [ctypes.c_int, ctypes.c_int, i64, P, PI, i64, i64]
        L.or_qd_div.argtypes = [i64, P, P, P]
        L.or_counter_madds.restype = i64
        L.or_counter_block_adds.restype = i64
        L.or_exact_entries.argtypes = [ctypes.c_int, i64, i64, i64, P, P, P, i64, PI, PI, P, P]
        L.or_exact_diff.argtypes = [ctypes.c_int, i64, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pi(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- EFTs and scalar ops (vectorised over arrays) ----------------------------
def _eft(name, a, b):
    a, b = _f64(a), _f64(b)
    s, e = np.empty_like(a), np.empty_like(a)
    getattr(lib(), name)(a.size, _p(a), _p(b), _p(s), _p(e))
    return s, e


def two_sum(a, b):
    return _eft("or_two_sum", a, b)


def fast_two_sum(a, b):
    return _eft("or_fast_two_sum", a, b)


def two_prod(a, b):
    return _eft("or_two_prod", a, b)


_OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "madd": 4, "madd_fused": 5,
        "add_acc": 6, "sub_acc": 7, "madd_acc": 8}
MADD_FUSED = 0x100
ADD_ACCURATE = 0x200
_VARIANT = {"canonical": 0, "fused": MADD_FUSED, "accurate": ADD_ACCURATE}


def dd_op(op: str, x, y, w=None):
    """x, y, w: arrays [2, n]. madd computes x + y*w."""
    x, y = _f64(x), _f64(y)
    w = _f64(w) if w is not None else np.zeros_like(x)
    z = np.empty_like(x)
    lib().or_dd_op(_OPS[op], x.shape[1], _p(x), _p(y), _p(w), _p(z))
    return z


def qd_op(op: str, x, y, w=None):
    """x, y, w: arrays [4, n]. madd computes x + y*w. (no div for QD)."""
    assert op != "div"
    x, y = _f64(x), _f64(y)
    w = _f64(w) if w is not None else np.zeros_like(x)
    z = np.empty_like(x)
    lib().or_qd_op(_OPS[op], x.shape[1], _p(x), _p(y), _p(w), _p(z))
    return z


def qd_renorm(c):
    """c: [5, n] -> [4, n]."""
    c = _f64(c)
    out = np.empty((4, c.shape[1]))
    lib().or_qd_renorm(c.shape[1], _p(c), _p(out))
    return out


def dd_abs_gt(x, y) -> bool:
    return bool(lib().or_dd_abs_gt(_p(_f64(x)), _p(_f64(y))))


def qd_abs_gt(x, y) -> bool:
    """|x| > |y| in the QD magnitude order (numerics.md s.3: sign folded on the leading
    word, then the four words compared lexicographically) -- the LU's pivot order."""
    return bool(lib().or_qd_abs_gt(_p(_f64(x)), _p(_f64(y))))


# ---- GEMM --------------------------------------------------------------------
def splitk_flag(s: int) -> int:
    """DDQD_SPLITK(s) algo bits (s in 1, 2, 4, 8)."""
    return {1: 0, 2: 0x1000, 4: 0x2000, 8: 0x3000}[s]


def depth_flag(d) -> int:
    """DDQD_DEPTH(d) algo bits: recurse exactly d levels (reading R21)."""
    return 0 if d is None else (int(d) + 1) << 16


def gemm(A, B, algo="block", threshold=32, bs=0, nthreads=0, madd="canonical", splitk=1, depth=None):
    """C := A B for planar [W, m, l] x [W, l, n] arrays (numerics.md s.4); madd='fused'
    selects the fused DD multiply-add variant (numerics.md s.2), madd='accurate' the
    accurate-add variant (every DD/QD addition accurate, numerics.md s.2-3); depth = d forces
    exactly d recursion levels instead of the threshold stop rule (reading R21)."""
    A, B = _f64(A), _f64(B)
    W, m, l = A.shape
    W2, l2, n = B.shape
    if W != W2 or l != l2:
        raise ValueError("dimension mismatch")
    C = np.empty((W, m, n))
    a = (ALGOS[algo] if isinstance(algo, str) else algo) | _VARIANT[madd] | splitk_flag(splitk) | depth_flag(depth)
    rc = lib().or_gemm(W, a, threshold, bs,
                       m, l, n, _p(A), _p(B), _p(C), nthreads)
    if rc:
        raise ValueError("or_gemm: invalid arguments")
    return C


def counters():
    L = lib()
    return L.or_counter_madds(), L.or_counter_block_adds()


def reset_counters():
    lib().or_counter_reset()


# ---- LU ----------------------------------------------------------------------
def lu(A, panel=256, algo="strassen", threshold=128, nthreads=0, pivot=True, madd="canonical"):
    """Blocked right-looking LU (numerics.md s.5) of a [W,n,n] DD (W=2) or QD (W=4) matrix,
    with partial pivoting or (pivot=False) the paper's pivot-free variant.
    Returns (LU [W,n,n], ipiv int64[n], info)."""
    LU = _f64(A).copy()
    W, n = LU.shape[0], LU.shape[1]
    ipiv = np.zeros(n, dtype=np.int64)
    a = ALGOS[algo] | _VARIANT[madd]
    info = lib().or_lu(W, 1 if pivot else 0, n, _p(LU), _pi(ipiv), panel, a, threshold, nthreads)
    if info < 0:
        raise ValueError("or_lu: invalid arguments")
    return LU, ipiv, info


def lu_panel(A, ipiv, p, kb, pivot=True):
    """Steps 1-2 of numerics.md s.5 for the panel of columns [p, p+kb), in place on the
    contiguous [W,n,n] array A and int64 ipiv[n]. Returns this panel's info (0 or k+1)."""
    assert A.dtype == np.float64 and A.flags.c_contiguous and ipiv.dtype == np.int64
    return lib().or_lu_panel(A.shape[0], 1 if pivot else 0, A.shape[1], _p(A), _pi(ipiv), p, kb)


def lu_solve(LU, ipiv, b):
    LU, b = _f64(LU), _f64(b)
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    x = np.empty_like(b)
    lib().or_lu_solve(LU.shape[0], LU.shape[1], _p(LU), _pi(ipiv), _p(b), _p(x))
    return x


def solve(A, b, panel=256, algo="strassen", threshold=128, nthreads=0, pivot=True, madd="canonical"):
    LU, ipiv, info = lu(A, panel, algo, threshold, nthreads, pivot, madd)
    return lu_solve(LU, ipiv, b), LU, ipiv, info


def qd_div(x, y):
    """QD division (numerics.md s.3) on [4, n] arrays."""
    x, y = _f64(x), _f64(y)
    z = np.empty_like(x)
    lib().or_qd_div(x.shape[1], _p(x), _p(y), _p(z))
    return z


# ---- exact reference -----------------------------------------------------------
def exact_entries(A, B, C, rows, cols):
    """Exact value and exact error (exact - sum(C words)) of sampled entries, rounded to double."""
    A, B, C = _f64(A), _f64(B), _f64(C)
    W, m, l = A.shape
    n = B.shape[2]
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    ex = np.empty(rows.size)
    err = np.empty(rows.size)
    bad = lib().or_exact_entries(W, m, l, n, _p(A), _p(B), _p(C), rows.size, _pi(rows), _pi(cols),
                                 _p(ex), _p(err))
    if bad:
        raise ArithmeticError("exact accumulator window violated")
    return ex, err


def exact_diff(x, y):
    """Exact (sum x words - sum y words) rounded to double; x, y [W, n]."""
    x, y = _f64(x), _f64(y)
    out = np.empty(x.shape[1])
    if lib().or_exact_diff(x.shape[0], x.shape[1], _p(x), _p(y), _p(out)):
        raise ArithmeticError("exact accumulator window violated")
    return out
