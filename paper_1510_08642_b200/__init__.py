"""paper_1510_08642_b200 -- B200-native DD/QD GEMM (Block / Strassen / Winograd) and DD LU.

Thin ctypes binding over the C ABI of libddqd.so (include/ddqd.h): argument marshalling
only -- every step of the path runs in the library's sm_100a kernels. PyTorch supplies
device memory and the current stream. There is no CPU fallback: importing this package
fails loudly when libddqd.so is missing, and calls fail when no CUDA device is present.

Layout: planar float64 tensors, shape [2, rows, cols] for DD and [4, rows, cols] for QD
(word 0 = leading word). Method: arXiv 1510.08642.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["dd_gemm", "qd_gemm", "gemm", "gemm_ex", "dd_lu_solve", "qd_lu_solve", "lu_solve", "elementwise", "lib",
           "workspace_bytes", "set_workspace_limit", "launch_count", "release",
           "profile_start", "profile_stop", "fp64_peak",
           "BLOCK", "STRASSEN", "WINOGRAD", "DDQDError"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libddqd.so")

BLOCK, STRASSEN, WINOGRAD = 0, 1, 2
MADD_FUSED = 0x100   # DDQD_MADD_FUSED: fused DD multiply-add in the leaf (docs/numerics.md s.2)
ADD_ACCURATE = 0x200   # DDQD_ADD_ACCURATE: every GEMM addition accurate (docs/numerics.md s.2-3)
_VARIANTS = {"canonical": 0, "fused": MADD_FUSED, "accurate": ADD_ACCURATE}
_ALGOS = {"block": BLOCK, "strassen": STRASSEN, "winograd": WINOGRAD}
_CODES = {-1: "EINVAL", -2: "EALIAS", -3: "ENOMEM", -4: "ECUDA", -5: "ENOTSUP"}


class DDQDError(RuntimeError):
    pass


class Mat(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("ld", ctypes.c_int64), ("ps", ctypes.c_int64), ("bs", ctypes.c_int64)]


class GemmDesc(ctypes.Structure):
    _fields_ = [("prec", ctypes.c_int), ("algo", ctypes.c_int), ("threshold", ctypes.c_int64),
                ("m", ctypes.c_int64), ("l", ctypes.c_int64), ("n", ctypes.c_int64),
                ("batch", ctypes.c_int64),
                ("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("psA", ctypes.c_int64), ("bsA", ctypes.c_int64),
                ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("psB", ctypes.c_int64), ("bsB", ctypes.c_int64),
                ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64), ("psC", ctypes.c_int64), ("bsC", ctypes.c_int64),
                ("beta", ctypes.c_int)]


def _load():
    if not os.path.exists(_SO):
        raise ImportError(
            "libddqd.so not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(_SO)
    i64, vp, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    for f in (L.dd_gemm, L.qd_gemm):
        f.argtypes = [i64, i64, i64, vp, vp, vp, i32, i64]
        f.restype = i32
    L.ddqd_gemm_ex.argtypes = [ctypes.POINTER(GemmDesc)]
    L.dd_lu_solve.argtypes = [i64, vp, vp, vp, vp, i64, i32, i64]
    L.qd_lu_solve.argtypes = [i64, vp, vp, vp, vp, i64, i32, i64]
    L.ddqd_lu_solve.argtypes = [i32, i32, i64, vp, vp, vp, vp, i64, i32, i64]
    L.ddqd_elementwise.argtypes = [i32, i32, i64, vp, vp, vp, vp]
    L.ddqd_lu_panel.argtypes = [i32, i32, i64, vp, vp, i64, i64]
    L.ddqd_band_copy.argtypes = [i32, i32, i64, i64, vp, vp, ctypes.POINTER(Mat), ctypes.POINTER(Mat)]
    L.ddqd_post_add_ptrs.argtypes = [i32, i32, i64, vp, i64, i64, i64, i64, i64, i64, ctypes.POINTER(Mat), i32]
    L.ddqd_ipc_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    L.ddqd_ipc_free.argtypes = [vp]
    L.ddqd_ipc_handle.argtypes = [vp, ctypes.c_char_p]
    L.ddqd_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.ddqd_ipc_close.argtypes = [vp]
    L.ddqd_lu_trsv.argtypes = [i32, i64, vp, vp, vp, vp]
    L.ddqd_set_stream.argtypes = [vp]
    L.ddqd_workspace_bytes.argtypes = [i32, i64, i64, i64, i32, i64]
    L.ddqd_workspace_bytes.restype = ctypes.c_size_t
    L.ddqd_set_workspace.argtypes = [vp, ctypes.c_size_t]
    L.ddqd_set_workspace_limit.argtypes = [ctypes.c_size_t]
    L.ddqd_launch_count.restype = i64
    L.ddqd_last_error.restype = ctypes.c_char_p
    L.ddqd_pre_add.argtypes = [i32, i32, i32, i64, ctypes.POINTER(Mat), ctypes.POINTER(Mat)]
    L.ddqd_pre_add_range.argtypes = [i32, i32, i32, i64, ctypes.POINTER(Mat), ctypes.POINTER(Mat), i64, i64]
    L.ddqd_post_add.argtypes = [i32, i32, i64, ctypes.POINTER(Mat), ctypes.POINTER(Mat), i32]
    L.ddqd_profile_stop.argtypes = [ctypes.POINTER(ctypes.c_double), i32]
    L.ddqd_fp64_peak.argtypes = [i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.ddqd_profile_kernels.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    return L


lib = _load()

EXPORTED = ["dd_gemm", "qd_gemm", "ddqd_gemm_ex", "dd_lu_solve", "qd_lu_solve", "ddqd_lu_solve",
            "ddqd_lu_panel", "ddqd_lu_trsv", "ddqd_post_add_ptrs", "ddqd_ipc_alloc", "ddqd_ipc_free",
            "ddqd_ipc_handle", "ddqd_ipc_open", "ddqd_ipc_close", "ddqd_elementwise", "ddqd_set_stream",
            "ddqd_workspace_bytes", "ddqd_set_workspace", "ddqd_set_workspace_limit",
            "ddqd_launch_count", "ddqd_release", "ddqd_last_error", "ddqd_version",
            "ddqd_profile_start", "ddqd_profile_stop", "ddqd_fp64_peak", "ddqd_pre_add", "ddqd_post_add",
            "ddqd_band_copy", "ddqd_profile_kernels", "ddqd_pre_add_range"]


def _check(rc: int, what: str) -> int:
    if rc < 0:
        msg = lib.ddqd_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise DDQDError(f"{what}: {_CODES.get(rc, rc)}: {msg}")
    return rc


def _torch():
    import torch
    return torch


def _set_stream(t):
    """Make the library use torch's current stream (of t's device; of the current device for
    host tensors, whose staging copies then run on that stream)."""
    torch = _torch()
    idx = t.device.index if t.is_cuda else torch.cuda.current_device()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)   # no Stream object per call
    ptr = raw(idx) if raw is not None else torch.cuda.current_stream(idx).cuda_stream
    lib.ddqd_set_stream(ctypes.c_void_p(ptr))


_SPLITK = {1: 0, 2: 0x1000, 4: 0x2000, 8: 0x3000}   # DDQD_SPLITK(s)


def depth_flag(d) -> int:
    """DDQD_DEPTH(d): recurse exactly d levels (the band schedule's compact problems)."""
    if d is None:
        return 0
    if not 0 <= int(d) <= 254:
        raise ValueError("depth must be in 0..254")
    return (int(d) + 1) << 16


def _algo(a, madd="canonical", splitk=1) -> int:
    """'block' | 'strassen' | 'winograd' (or the int); madd='fused' ORs in DDQD_MADD_FUSED,
    madd='accurate' DDQD_ADD_ACCURATE."""
    v = _ALGOS[a] if isinstance(a, str) else int(a)
    if madd not in _VARIANTS:
        raise ValueError("madd must be 'canonical', 'fused' or 'accurate'")
    if splitk not in _SPLITK:
        raise ValueError("splitk must be 1, 2, 4 or 8")
    return v | _VARIANTS[madd] | _SPLITK[splitk]


def _check_mat(x, W, name):
    torch = _torch()
    if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or x.dim() != 3 or x.shape[0] != W:
        raise ValueError(f"{name} must be a float64 tensor of shape [{W}, rows, cols]")
    if not x.is_contiguous():
        raise ValueError(f"{name} must be contiguous (planar row-major)")


def gemm(A, B, algo="block", threshold=128, out=None, madd="canonical", splitk=1):
    """C := A B with A [W,m,l], B [W,l,n] float64 CUDA tensors, W = 2 (DD) or 4 (QD).
    Pinned/ordinary CPU tensors for A, B and `out` use the library's host-staging path
    (copies inside the call, synchronous)."""
    torch = _torch()
    W = A.shape[0] if A.dim() == 3 else -1
    _check_mat(A, W, "A")
    _check_mat(B, W, "B")
    if W not in (2, 4):
        raise ValueError("leading dimension must be 2 (DD) or 4 (QD)")
    m, l = A.shape[1], A.shape[2]
    if B.shape[1] != l:
        raise ValueError("dimension mismatch")
    n = B.shape[2]
    if out is None:
        out = torch.empty((W, m, n), dtype=torch.float64, device=A.device,
                          pin_memory=(not A.is_cuda and A.is_pinned()))
    _check_mat(out, W, "out")
    if tuple(out.shape) != (W, m, n):
        raise ValueError("out has the wrong shape")
    _set_stream(A)
    f = lib.dd_gemm if W == 2 else lib.qd_gemm
    _check(f(m, l, n, A.data_ptr(), B.data_ptr(), out.data_ptr(), _algo(algo, madd, splitk), threshold), "gemm")
    return out


def dd_gemm(A, B, algo="block", threshold=128, out=None, madd="canonical", splitk=1):
    if A.shape[0] != 2:
        raise ValueError("dd_gemm takes [2, rows, cols] tensors")
    return gemm(A, B, algo, threshold, out, madd, splitk)


def qd_gemm(A, B, algo="block", threshold=128, out=None, madd="canonical", splitk=1):
    if A.shape[0] != 4:
        raise ValueError("qd_gemm takes [4, rows, cols] tensors")
    return gemm(A, B, algo, threshold, out, madd, splitk)


def gemm_ex(prec, algo, threshold, m, l, n, batch, A, lda, psA, bsA, B, ldb, psB, bsB,
            C, ldc, psC, bsC, beta=0, madd="canonical", depth=None):
    """Strided/batched form (ddqd_gemm_ex); A, B, C are device addresses (ints); depth = d ORs in
    DDQD_DEPTH(d) (exactly d recursion levels, threshold unused)."""
    d = GemmDesc(prec, _algo(algo, madd) | depth_flag(depth), threshold, m, l, n, batch, A, lda, psA, bsA, B, ldb, psB, bsB,
                 C, ldc, psC, bsC, beta)
    return _check(lib.ddqd_gemm_ex(ctypes.byref(d)), "gemm_ex")


def batch_mat(t):
    """Mat descriptor of a [batch, W, rows, cols] (or [W, rows, cols]) CUDA tensor whose rows are
    unit-stride (strided views such as the LU's trailing block are allowed)."""
    if t.stride(-1) != 1:
        raise ValueError("rows must be unit-stride")
    r, c = t.shape[-2], t.shape[-1]
    ld, ps = t.stride(-2), t.stride(-3)
    bs = t.stride(0) if t.dim() == 4 else ps * t.shape[0]
    return Mat(t.data_ptr(), r, c, ld, ps, bs)


def _add_algo(algo, madd):
    # the additions follow the accurate variant; the fused variant only changes the leaf madd
    return _algo(algo) | (ADD_ACCURATE if madd == "accurate" else 0)


def pre_add(algo, side, X, Y, madd="canonical", keep=None):
    """One level's fused pre-additions: X [P,W,r,c] -> Y [7P,W,ceil(r/2),ceil(c/2)]; keep = (lo, hi)
    stores only children 7b + c in [lo, hi)."""
    P = 1 if X.dim() == 3 else X.shape[0]
    W = X.shape[-3]
    _set_stream(X)
    x, y = batch_mat(X), batch_mat(Y)
    lo, hi = keep if keep is not None else (0, 7 * P)
    _check(lib.ddqd_pre_add_range(W, _add_algo(algo, madd), side, P, ctypes.byref(x), ctypes.byref(y), lo, hi),
           "pre_add")


def post_add(algo, M, C, beta=0, madd="canonical"):
    """One level's fused post-additions: M [7P,W,h,h'] -> C [P,W,r,c]."""
    P = 1 if C.dim() == 3 else C.shape[0]
    W = C.shape[-3]
    _set_stream(C)
    mm, cc = batch_mat(M), batch_mat(C)
    _check(lib.ddqd_post_add(W, _add_algo(algo, madd), P, ctypes.byref(mm), ctypes.byref(cc), beta), "post_add")


def post_add_ptrs(algo, children, C, r0=0, r1=None, beta=0, madd="canonical"):
    """One level's post-additions reading the 7P children through device pointers
    (ddqd_post_add_ptrs): children = list of 7P CUDA tensors [W, hm, hn] (same shape and strides;
    they may be IPC mappings of other GPUs' memory), C = [P, W, r, c] or [W, r, c]; position rows
    [r0, r1) only."""
    torch = _torch()
    P = 1 if C.dim() == 3 else C.shape[0]
    if len(children) != 7 * P:
        raise ValueError("need 7 children per parent")
    W, hm, hn = children[0].shape
    ld, ps = children[0].stride(1), children[0].stride(0)
    ptrs = torch.tensor([t.data_ptr() for t in children], dtype=torch.int64, device=C.device)
    _set_stream(C)
    cc = batch_mat(C)
    rc = lib.ddqd_post_add_ptrs(W, _add_algo(algo, madd), P, ptrs.data_ptr(), hm, hn, ld, ps, r0,
                                hm if r1 is None else r1, ctypes.byref(cc), beta)
    _check(rc, "post_add_ptrs")
    return ptrs   # keep alive until the kernel ran (caller synchronises)


class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (for torch.as_tensor)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def ipc_alloc(shape, device):
    """A float64 CUDA tensor in its own cudaMalloc allocation (exportable with ipc_handle);
    returns (tensor, raw pointer). Free with ipc_free(pointer) after the tensor is dropped."""
    torch = _torch()
    n = 1
    for d in shape:
        n *= int(d)
    p = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(lib.ddqd_ipc_alloc(8 * max(n, 1), ctypes.byref(p)), "ipc_alloc")
        t = torch.as_tensor(_CudaArray(p.value, shape), device=device)
    return t, p.value


def ipc_free(ptr):
    _check(lib.ddqd_ipc_free(ctypes.c_void_p(ptr)), "ipc_free")


def ipc_handle(ptr) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib.ddqd_ipc_handle(ctypes.c_void_p(ptr), buf), "ipc_handle")
    return buf.raw


def ipc_open(handle: bytes, shape, device):
    """Map another process's ipc_alloc buffer; returns (tensor view, raw pointer)."""
    torch = _torch()
    p = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(lib.ddqd_ipc_open(handle, ctypes.byref(p)), "ipc_open")
        t = torch.as_tensor(_CudaArray(p.value, shape), device=device)
    return t, p.value


def ipc_close(ptr):
    _check(lib.ddqd_ipc_close(ctypes.c_void_p(ptr)), "ipc_close")


def gemm_batched(A, B, C, algo, threshold, beta=0, madd="canonical", depth=None):
    """C[b] := A[b] B[b] for contiguous [batch, W, .., ..] CUDA tensors (one library schedule)."""
    batch, W, m, l = A.shape
    n = B.shape[3]
    _set_stream(A)
    return gemm_ex(W, algo, threshold, m, l, n, batch,
                   A.data_ptr(), l, m * l, W * m * l,
                   B.data_ptr(), n, l * n, W * l * n,
                   C.data_ptr(), n, m * n, W * m * n, beta, madd, depth)


def band_copy(direction, full, compact, rmap=None, cmap=None):
    """ddqd_band_copy: direction 'pack' (compact := full[rmap][:, cmap]) or 'unpack'
    (full[rmap][:, cmap] := compact) for [W, r, c] CUDA tensors with unit-stride rows; rmap /
    cmap: int64 CUDA tensors (None = identity). The compact extent is compact's shape."""
    W, rows, cols = compact.shape
    if full.shape[0] != W:
        raise ValueError("word counts differ")
    dirv = {"pack": 0, "unpack": 1}[direction]
    for mp, k in ((rmap, rows), (cmap, cols)):
        if mp is not None and (mp.dtype != _torch().int64 or mp.numel() != k or not mp.is_contiguous()):
            raise ValueError("maps must be contiguous int64 of the compact extent")
    _set_stream(compact)
    f, c = batch_mat(full), batch_mat(compact)
    _check(lib.ddqd_band_copy(W, dirv, rows, cols, rmap.data_ptr() if rmap is not None else None,
                              cmap.data_ptr() if cmap is not None else None, ctypes.byref(f), ctypes.byref(c)),
           "band_copy")


def lu_solve(A, b, panel=256, algo="strassen", threshold=128, pivot=True, overwrite=False,
             madd="canonical"):
    """Blocked right-looking DD/QD LU (partial pivoting, or the paper's pivot-free variant with
    pivot=False) + solve (Eq. 2). A: [W,n,n] CUDA float64, b: [W,n], W = 2 or 4.
    Returns (x, LU, ipiv, info)."""
    torch = _torch()
    W = A.shape[0]
    if W not in (2, 4):
        raise ValueError("A must be [2|4, n, n]")
    _check_mat(A, W, "A")
    n = A.shape[1]
    if A.shape[2] != n or tuple(b.shape) != (W, n) or b.dtype != torch.float64 or not b.is_contiguous():
        raise ValueError("A must be [W,n,n] and b [W,n] contiguous float64")
    LU = A if overwrite else A.clone()
    x = torch.empty_like(b)
    ipiv = torch.empty(n, dtype=torch.int64, device=A.device)
    _set_stream(A)
    info = _check(lib.ddqd_lu_solve(W, 1 if pivot else 0, n, LU.data_ptr(), b.data_ptr(), x.data_ptr(),
                                    ipiv.data_ptr(), panel, _algo(algo, madd), threshold), "lu_solve")
    return x, LU, ipiv, info


def lu_panel(LU, ipiv, p, kb, pivot=True):
    """Steps 1-2 of the LU for the panel [p, p+kb) of the [W,n,n] CUDA tensor LU, in place
    (ddqd_lu_panel); ipiv: int64 [n] CUDA tensor. Returns this panel's info (0 or k+1)."""
    W, n = LU.shape[0], LU.shape[1]
    _set_stream(LU)
    return _check(lib.ddqd_lu_panel(W, 1 if pivot else 0, n, LU.data_ptr(), ipiv.data_ptr(), p, kb), "lu_panel")


def lu_trsv(LU, ipiv, b):
    """x with LU x = P b from the factors (ddqd_lu_trsv); returns x [W,n]."""
    torch = _torch()
    x = torch.empty_like(b)
    _set_stream(LU)
    _check(lib.ddqd_lu_trsv(LU.shape[0], LU.shape[1], LU.data_ptr(), ipiv.data_ptr(), b.data_ptr(),
                            x.data_ptr()), "lu_trsv")
    return x


def dd_lu_solve(A, b, panel=256, algo="strassen", threshold=128, overwrite=False):
    """DD LU with partial pivoting + solve (BJ:11). Returns (x, LU, ipiv, info)."""
    if A.shape[0] != 2:
        raise ValueError("dd_lu_solve takes [2, n, n]")
    return lu_solve(A, b, panel, algo, threshold, True, overwrite)


def qd_lu_solve(A, b, panel=256, algo="strassen", threshold=128, overwrite=False):
    """QD LU with partial pivoting + solve. Returns (x, LU, ipiv, info)."""
    if A.shape[0] != 4:
        raise ValueError("qd_lu_solve takes [4, n, n]")
    return lu_solve(A, b, panel, algo, threshold, True, overwrite)


_OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "madd": 4, "madd_fused": 5,
        "add_acc": 6, "sub_acc": 7, "madd_acc": 8}


def elementwise(op, x, y, w=None):
    """Device DD/QD arithmetic on planar [W, count] tensors (parity tests of the arithmetic layer)."""
    torch = _torch()
    W = x.shape[0]
    z = torch.empty_like(x)
    w = w if w is not None else torch.zeros_like(x)
    _set_stream(x)
    _check(lib.ddqd_elementwise(W, _OPS[op], x.shape[1], x.data_ptr(), y.data_ptr(), w.data_ptr(),
                                z.data_ptr()), "elementwise")
    return z


def workspace_bytes(prec, m, l, n, algo, threshold):
    return lib.ddqd_workspace_bytes(prec, m, l, n, _algo(algo), threshold)


def set_workspace_limit(nbytes: int):
    lib.ddqd_set_workspace_limit(nbytes)


def launch_count() -> int:
    return lib.ddqd_launch_count()


def release():
    lib.ddqd_release()


def profile_start():
    lib.ddqd_profile_start()


def profile_stop():
    """-> {"leaf": (ms, launches, madds), "pre": (ms, launches, bytes), "post": (...)}"""
    buf = (ctypes.c_double * 18)()
    _check(lib.ddqd_profile_stop(buf, 18), "profile_stop")
    v = list(buf)
    names = ["leaf", "pre", "post", "lu_panel", "lu_trsm", "lu_solve"]
    return {nm: tuple(v[3 * i:3 * i + 3]) for i, nm in enumerate(names)}


def profile_kernels():
    """Per-kernel totals of the last profile_stop(): {name: (class, ms, launches, work)}."""
    need = lib.ddqd_profile_kernels(None, 0)
    buf = ctypes.create_string_buffer(max(int(need), 1))
    lib.ddqd_profile_kernels(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cls, ms, launches, work = line.split("\t")
        out[name] = (int(cls), float(ms), int(float(launches)), float(work))
    return out


def fp64_peak(op="dfma"):
    """Measured FP64-pipe lane-operations per second (DFMA or DADD stream)."""
    r, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib.ddqd_fp64_peak(0 if op == "dfma" else 1, ctypes.byref(r), ctypes.byref(ms)), "fp64_peak")
    return r.value, ms.value
