"""GPU parity tests: the CUDA path (through the C ABI of libddqd.so) against the CPU
oracle on the same seeded inputs. Bit-exact wherever the kernel reproduces the oracle's
summation order (everything here: docs/numerics.md), plus exact-error bounds (BJ:5) at
the BASELINE.json full sizes where only sampled entries are checkable."""
import json
import os

import numpy as np
import pytest

import ddqd_inputs as gen
from tests.util import rec_depth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1510_08642_b200 as ddqd  # noqa: E402

DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def np_(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def same(a, b):
    """bitwise equality of float64 arrays (incl. signed zeros)"""
    return np.array_equal(a.view(np.int64), b.view(np.int64))


# ---- arithmetic layer ---------------------------------------------------------
def _dd_samples(n, seed):
    rng = np.random.default_rng(seed)
    hi = rng.uniform(-1, 1, n) * np.exp2(rng.integers(-30, 30, n))
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, n)
    s = hi + lo
    e = lo - (s - hi)
    x = np.stack([s, e])
    x[:, :50] = 0.0
    return x


@pytest.mark.parametrize("op", ["add", "sub", "mul", "div", "madd"])
def test_dd_elementwise_bitwise(orc, op):
    x, y, w = _dd_samples(100000, 1), _dd_samples(100000, 2), _dd_samples(100000, 3)
    y[:, 1000:2000] = -x[:, 1000:2000]          # exact cancellation
    if op == "div":
        y[:, :50] = 1.0
        y[1, :50] = 0.0
    ref = orc.dd_op(op, x, y, w)
    got = np_(ddqd.elementwise(op, cu(x), cu(y), cu(w)))
    assert same(got, ref)


@pytest.mark.parametrize("op", ["add", "sub", "mul", "madd", "div"])
def test_qd_elementwise_bitwise(orc, op):
    q = [gen.qd_matrix(1, 50000, s, 0).reshape(4, -1) for s in (4, 5, 6)]
    if op != "div":
        q[1][:, :500] = -q[0][:, :500]
    ref = orc.qd_div(q[0], q[1]) if op == "div" else orc.qd_op(op, *q)
    got = np_(ddqd.elementwise(op, *(cu(a) for a in q)))
    assert same(got, ref)


# ---- leaf GEMM (Block) ----------------------------------------------------------
@pytest.mark.parametrize("W", [2, 4])
def test_block_small_and_ragged_bitwise(orc, W):
    shapes = [(1, 1, 1), (3, 5, 2), (7, 1, 9), (33, 17, 65), (64, 64, 64), (65, 63, 129),
              (130, 17, 3), (2, 300, 2), (100, 200, 70)]
    for (m, l, n) in shapes:
        A = gen.matrix(W, m, l, m + l, 0)
        B = gen.matrix(W, l, n, m + l, 1)
        ref = orc.gemm(A, B, "block")
        got = np_(ddqd.gemm(cu(A), cu(B), "block"))
        assert same(got, ref), (m, l, n)


def test_block_large_tiles_bitwise(orc):
    """Shape that selects the 64x64 4x4 kernel (>= 296 tiles) with ragged edges on all sides."""
    A = gen.dd_matrix(1100, 301, 9, 0)
    B = gen.dd_matrix(301, 1090, 9, 1)
    assert same(np_(ddqd.dd_gemm(cu(A), cu(B), "block")), orc.gemm(A, B, "block"))


def test_c0_dd_block_128(orc):
    """BJ:7 (config 0): DD Block 128^3, seed 1: bit-exact vs oracle, and within
    2^-96 l |A| |B| of the exact product on every entry."""
    A = gen.dd_matrix(128, 128, 1, 0)
    B = gen.dd_matrix(128, 128, 1, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), "block"))
    assert same(got, orc.gemm(A, B, "block"))
    r, c = np.meshgrid(np.arange(128), np.arange(128), indexing="ij")
    _, err = orc.exact_entries(A, B, got, r.ravel(), c.ravel())
    bound = 2.0 ** -96 * 128 * np.abs(A[0]).max() * np.abs(B[0]).max()
    assert np.abs(err).max() <= bound


def test_zero_and_degenerate_sizes(orc):
    A = cu(np.zeros((2, 5, 0))); B = cu(np.zeros((2, 0, 4)))
    C = ddqd.dd_gemm(A, B, "strassen", 1)
    assert np_(C).shape == (2, 5, 4) and np.all(np_(C) == 0)
    A = cu(np.zeros((2, 0, 3))); B = cu(np.zeros((2, 3, 4)))
    assert np_(ddqd.dd_gemm(A, B)).shape == (2, 0, 4)


def test_errors():
    A = cu(gen.dd_matrix(4, 4, 1, 0))
    with pytest.raises(ValueError):
        ddqd.dd_gemm(A, cu(gen.dd_matrix(5, 4, 1, 0)))
    with pytest.raises(ValueError):
        ddqd.dd_gemm(A, A, "strassen", 0)          # threshold < 1 -> EINVAL
    with pytest.raises(ddqd.DDQDError):
        ddqd.dd_gemm(A, A, out=A)                  # aliasing -> EALIAS


def test_abi_errors_of_the_newer_entry_points():
    """Argument errors of the LU step, peer-memory combine and IPC entry points come back as
    status codes (no crash, no exception across the ABI), with a message."""
    import ctypes
    L = ddqd.lib
    A = cu(gen.dd_matrix(8, 8, 1, 0))
    ipiv = torch.empty(8, dtype=torch.int64, device=DEV)
    assert L.ddqd_lu_panel(2, 1, 8, A.data_ptr(), ipiv.data_ptr(), 4, 8) == -1    # p + kb > n
    assert L.ddqd_lu_panel(3, 1, 8, A.data_ptr(), ipiv.data_ptr(), 0, 4) == -1    # bad precision
    assert L.ddqd_lu_panel(2, 1, 8, None, ipiv.data_ptr(), 0, 4) == -1             # null pointer
    assert L.ddqd_last_error()
    assert L.ddqd_lu_trsv(2, 8, None, None, None, None) == -1
    M = ddqd.Mat(A.data_ptr(), 8, 8, 8, 64, 128)
    assert L.ddqd_post_add_ptrs(2, 1, 1, None, 4, 4, 4, 16, 0, 4, ctypes.byref(M), 0) == -1   # no pointer table
    assert L.ddqd_post_add_ptrs(2, 3, 1, A.data_ptr(), 4, 4, 4, 16, 0, 4, ctypes.byref(M), 0) == -1  # bad algo
    assert L.ddqd_post_add_ptrs(2, 1, 1, A.data_ptr(), 3, 4, 4, 16, 0, 3, ctypes.byref(M), 0) == -1  # hm != ceil(8/2)
    assert L.ddqd_ipc_handle(None, None) == -1
    assert L.ddqd_ipc_open(None, None) == -1
    with pytest.raises(ValueError):
        ddqd.dd_gemm(A, A, "block", splitk=3)           # split-k must be 1, 2, 4 or 8
    with pytest.raises(ValueError):
        ddqd.gemm(A, A, 0x4000 | 0, 8)                   # unknown algo flag -> EINVAL


# ---- recursion --------------------------------------------------------------------
@pytest.mark.parametrize("algo", ["strassen", "winograd"])
@pytest.mark.parametrize("W", [2, 4])
def test_recursion_odd_shapes_bitwise(orc, algo, W):
    """Odd/rectangular shapes with virtual zero padding at several levels (T small)."""
    for (m, l, n, T) in [(37, 29, 33, 4), (64, 64, 64, 8), (65, 66, 67, 16), (101, 45, 77, 10),
                         (9, 130, 11, 2)]:
        A = gen.matrix(W, m, l, 3 * m + T, 0)
        B = gen.matrix(W, l, n, 3 * m + T, 1)
        ref = orc.gemm(A, B, algo, threshold=T)
        got = np_(ddqd.gemm(cu(A), cu(B), algo, T))
        assert same(got, ref), (m, l, n, T)


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_threshold_ge_dims_equals_block(algo):
    A = cu(gen.dd_matrix(70, 80, 3, 0)); B = cu(gen.dd_matrix(80, 90, 3, 1))
    assert same(np_(ddqd.dd_gemm(A, B, algo, 70)), np_(ddqd.dd_gemm(A, B, "block")))


def test_c1_dd_strassen_1024(orc):
    """BJ:8 (config 1): DD Strassen 1024^3, T = 128 (depth 3), seed 2; Block on the same
    inputs; both bit-exact vs the oracle."""
    A = gen.dd_matrix(1024, 1024, 2, 0)
    B = gen.dd_matrix(1024, 1024, 2, 1)
    gA, gB = cu(A), cu(B)
    got = np_(ddqd.dd_gemm(gA, gB, "strassen", 128))
    assert same(got, orc.gemm(A, B, "strassen", 128))
    got_b = np_(ddqd.dd_gemm(gA, gB, "block"))
    assert same(got_b, orc.gemm(A, B, "block"))
    rng = np.random.default_rng(1)
    r, c = rng.integers(0, 1024, 2048), rng.integers(0, 1024, 2048)
    _, err = orc.exact_entries(A, B, got, r, c)
    bound = 18.0 ** 3 * 2.0 ** -96 * 1024 * np.abs(A[0]).max() * np.abs(B[0]).max()
    assert np.abs(err).max() <= bound


def test_c2_qd_winograd_1024_sampled_and_512_bitwise(orc):
    """BJ:9 (config 2): QD Winograd 1024^3, T = 128, seed 3: sampled exact errors within
    18^3 2^-200 l |A||B|; bit-exact vs the oracle at 512^3 (depth 2) with the same recipe."""
    A = gen.qd_matrix(1024, 1024, 3, 0)
    B = gen.qd_matrix(1024, 1024, 3, 1)
    got = np_(ddqd.qd_gemm(cu(A), cu(B), "winograd", 128))
    rng = np.random.default_rng(2)
    r, c = rng.integers(0, 1024, 512), rng.integers(0, 1024, 512)
    _, err = orc.exact_entries(A, B, got, r, c)
    bound = 18.0 ** 3 * 2.0 ** -200 * 1024 * np.abs(A[0]).max() * np.abs(B[0]).max()
    assert np.abs(err).max() <= bound
    A5, B5 = A[:, :512, :512].copy(), B[:, :512, :512].copy()
    assert same(np_(ddqd.qd_gemm(cu(A5), cu(B5), "winograd", 128)), orc.gemm(A5, B5, "winograd", 128))


def test_c3_shape_reduced_bitwise(orc):
    """BJ:10 recipe (odd m, l, n) at 1023 x 1025 x 1021, T = 128 (depth 3): bit-exact."""
    A = gen.dd_matrix(1023, 1025, 4, 0)
    B = gen.dd_matrix(1025, 1021, 4, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", 128))
    assert same(got, orc.gemm(A, B, "winograd", 128))


def test_c3_full_size_sampled(orc):
    """BJ:10 (config 3): DD Winograd 8191 x 8193 x 8190, T = 256 (depth 5), seed 4, in the
    launch configuration bench.py times: >= 4096 sampled entries, including every padded
    border row/column class, within 18^5 2^-96 l |A| |B| of the exact product."""
    m, l, n, T = 8191, 8193, 8190, 256
    A = gen.dd_matrix(m, l, 4, 0)
    B = gen.dd_matrix(l, n, 4, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", T))
    assert rec_depth(m, l, n, T) == 5
    rng = np.random.default_rng(3)
    r = np.concatenate([rng.integers(0, m, 4000), [0, m - 1, 4095, 4096, m - 1, 0, 2047, 6143]])
    c = np.concatenate([rng.integers(0, n, 4000), [0, n - 1, 4094, 4095, 0, n - 1, 6142, 2047]])
    _, err = orc.exact_entries(A, B, got, r, c)
    bound = 18.0 ** 5 * 2.0 ** -96 * l * np.abs(A[0]).max() * np.abs(B[0]).max()
    assert np.abs(err).max() <= bound
    assert np.abs(err).max() <= bound * 2.0 ** -10     # typical error is far inside the bound


def test_c3_full_size_bitwise(orc):
    """BJ:10 (config 3) at its full size, DD Winograd 8191 x 8193 x 8190, T = 256 (depth 5),
    seed 4, as bench.py runs it: the whole product bit-identical to the oracle's recursion
    (~2 minutes of the oracle on the host cores)."""
    m, l, n, T = 8191, 8193, 8190, 256
    A = gen.dd_matrix(m, l, 4, 0)
    B = gen.dd_matrix(l, n, 4, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", T))
    ref = orc.gemm(A, B, "winograd", threshold=T)
    assert same(got, ref)


def test_host_pointer_path_matches_device(orc):
    A = gen.dd_matrix(300, 257, 7, 0)
    B = gen.dd_matrix(257, 301, 7, 1)
    hA = torch.from_numpy(A).pin_memory(); hB = torch.from_numpy(B).pin_memory()
    hC = ddqd.dd_gemm(hA, hB, "winograd", 64)
    assert same(hC.numpy(), np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", 64)))
    assert same(hC.numpy(), orc.gemm(A, B, "winograd", 64))


@pytest.mark.parametrize("algo", ["block", "strassen", "winograd"])
def test_gemm_ex_strided_beta1(orc, algo):
    """C := C - A B on strided sub-blocks (the LU Schur update form)."""
    N = 200
    big = gen.dd_matrix(N, N, 11, 0)
    m, l, n = 120, 40, 130
    A = big[:, 50:50 + m, 10:10 + l].copy()
    B = big[:, 5:5 + l, 60:60 + n].copy()
    C0 = big[:, 70:70 + m, 65:65 + n].copy()
    T = orc.gemm(A, B, algo, threshold=16)
    ref = orc.dd_op("sub", C0.reshape(2, -1), T.reshape(2, -1)).reshape(2, m, n)
    g = cu(big)
    base, ps = g.data_ptr(), N * N
    ddqd.gemm_ex(2, algo, 16, m, l, n, 1,
                 base + 8 * (50 * N + 10), N, ps, 0,
                 base + 8 * (5 * N + 60), N, ps, 0,
                 base + 8 * (70 * N + 65), N, ps, 0, beta=1)
    assert same(np_(g)[:, 70:70 + m, 65:65 + n], ref)


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_gemm_ex_beta1_fused_last_level(orc, W, algo):
    """C := C - A B where the fused last level is the top level (its beta = 1 epilogue): the
    unrolled 17^3 DD kernel (34^3, T = 32), run-time leaves (30 x 20 x 31, T = 16), and a
    fused level below an unfused one (60 x 40 x 62, T = 16), strided sub-blocks, DD and QD."""
    N = 140
    big = gen.matrix(W, N, N, 12, 0)
    for (m, l, n, T) in ((34, 34, 34, 32), (30, 20, 31, 16), (60, 40, 62, 16)):
        A = big[:, 3:3 + m, 70:70 + l].copy()
        B = big[:, 72:72 + l, 1:1 + n].copy()
        C0 = big[:, 75:75 + m, 71:71 + n].copy()
        Tm = orc.gemm(A, B, algo, threshold=T)
        op = orc.dd_op if W == 2 else orc.qd_op
        ref = op("sub", C0.reshape(W, -1), Tm.reshape(W, -1)).reshape(W, m, n)
        g = cu(big)
        base, ps = g.data_ptr(), N * N
        ddqd.gemm_ex(W, algo, T, m, l, n, 1,
                     base + 8 * (3 * N + 70), N, ps, 0,
                     base + 8 * (72 * N + 1), N, ps, 0,
                     base + 8 * (75 * N + 71), N, ps, 0, beta=1)
        assert same(np_(g)[:, 75:75 + m, 71:71 + n], ref), (m, l, n, T)


# ---- paper benchmark pair ----------------------------------------------------
@pytest.mark.parametrize("n", [1023, 1024, 1025])
def test_paper_pair_columns_and_parity(orc, n):
    """P:60-61 inputs at the paper's sizes, Strassen(32)/Winograd(32) bit-exact vs the
    oracle run on the same inputs; Block's columns bitwise identical (B has equal columns)."""
    A, B = gen.bench_pair(n, 2)
    gA, gB = cu(A), cu(B)
    Cb = np_(ddqd.dd_gemm(gA, gB, "block"))
    assert np.all(Cb == Cb[:, :, :1])
    for algo in ("strassen", "winograd"):
        for T in ((128, 32) if n == 1025 else (128,)):     # the paper's n_min = 32 too
            got = np_(ddqd.dd_gemm(gA, gB, algo, T))
            assert same(got, orc.gemm(A, B, algo, threshold=T))


# ---- LU ---------------------------------------------------------------------------
def _b_ones(orc, A):
    n = A.shape[1]
    ones = np.zeros((2, n, 1)); ones[0] = 1.0
    return orc.gemm(A, ones, "block")[:, :, 0]


@pytest.mark.parametrize("algo,T,K", [("strassen", 32, 64), ("block", 128, 48), ("winograd", 16, 100)])
def test_lu_bitwise_vs_oracle(orc, algo, T, K):
    n = 300
    A = gen.lu_matrix(n, 5)
    b = _b_ones(orc, A)
    x_ref, LU_ref, piv_ref, info_ref = orc.solve(A, b, panel=K, algo=algo, threshold=T)
    x, LU, piv, info = ddqd.dd_lu_solve(cu(A), cu(b), panel=K, algo=algo, threshold=T)
    assert info == info_ref == 0
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref)
    assert same(np_(x), x_ref)


def test_lu_pivoting_path_bitwise(orc):
    """Non-dominant matrix: row interchanges happen; still bit-exact."""
    n = 200
    A = gen.dd_matrix(n, n, 13, 0)
    b = gen.dd_matrix(1, n, 13, 1)[:, 0, :].copy()
    x_ref, LU_ref, piv_ref, _ = orc.solve(A, b, panel=32, algo="strassen", threshold=16)
    x, LU, piv, info = ddqd.dd_lu_solve(cu(A), cu(b), panel=32, algo="strassen", threshold=16)
    assert np.any(piv_ref != np.arange(n))
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref) and same(np_(x), x_ref)


def test_lu_zero_pivot_info():
    A = gen.dd_matrix(40, 40, 2, 0)
    A[:, :, 7] = 0.0
    b = np.zeros((2, 40)); b[0] = 1.0
    _, _, _, info = ddqd.dd_lu_solve(cu(A), cu(b), panel=16, algo="block")
    assert info == 8


def test_c4_lu_1024_bitwise(orc):
    """BJ:11 recipe at n = 1024 (panel 256, Strassen update T = 128): bit-exact vs oracle."""
    n = 1024
    A = gen.lu_matrix(n, 5)
    b = _b_ones(orc, A)
    x_ref, LU_ref, piv_ref, _ = orc.solve(A, b, panel=256, algo="strassen", threshold=128)
    x, LU, piv, info = ddqd.dd_lu_solve(cu(A), cu(b), panel=256, algo="strassen", threshold=128)
    assert info == 0 and same(np_(LU), LU_ref) and same(np_(x), x_ref)


def test_c4_lu_full_size_properties():
    """BJ:11 (config 4): n = 4096, panel 256, Strassen update: ipiv = identity (column
    diagonal dominance), x = 1 within 2^-96 n kappa 18."""
    n = 4096
    A = gen.lu_matrix(n, 5)
    gA = cu(A)
    ones = torch.zeros((2, n, 1), dtype=torch.float64, device=DEV); ones[0] = 1.0
    b = ddqd.dd_gemm(gA, ones, "block")[:, :, 0].contiguous()
    x, LU, piv, info = ddqd.dd_lu_solve(gA, b, panel=256, algo="strassen", threshold=128)
    assert info == 0
    assert np.array_equal(np_(piv), np.arange(n))
    xx = np_(x)
    err = np.abs((xx[0] - 1.0) + xx[1]).max()
    assert err <= 2.0 ** -96 * n * 3 * 18


def test_c4_lu_full_size_bitwise(orc):
    """BJ:11 (config 4) at its full size, n = 4096, panel 256, Strassen update (T = 128), in the
    launch configuration bench.py times: factors, pivots and x bit-identical to the oracle's
    (the LU cannot be sampled entry by entry, so the whole oracle LU runs on the host cores)."""
    n = 4096
    A = gen.lu_matrix(n, 5)
    b = _b_ones(orc, A).copy()
    x_ref, LU_ref, piv_ref, info_ref = orc.solve(A, b, panel=256, algo="strassen", threshold=128)
    x, LU, piv, info = ddqd.dd_lu_solve(cu(A), cu(b), panel=256, algo="strassen", threshold=128)
    assert info == info_ref == 0
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref) and same(np_(x), x_ref)


def test_c2_qd_winograd_full_size_bitwise(orc):
    """BJ:9 (config 2) at its full size, QD Winograd 1024^3, T = 128, seed 3, as bench.py runs
    it: every entry bit-identical to the oracle's recursion."""
    A = gen.qd_matrix(1024, 1024, 3, 0)
    B = gen.qd_matrix(1024, 1024, 3, 1)
    got = np_(ddqd.qd_gemm(cu(A), cu(B), "winograd", 128))
    assert same(got, orc.gemm(A, B, "winograd", threshold=128))


# ---- multi-GPU schedule's CUDA backend, world size 1 (one GPU available) ---------------
@pytest.mark.parametrize("algo,k", [("winograd", 2), ("strassen", 1), ("block", 0)])
def test_mgpu_schedule_cuda_backend_world1(orc, algo, k):
    """The depth-k product schedule (pre-adds, batched slice GEMM, gather, post-adds) through
    the library's ddqd_pre_add / ddqd_gemm_ex / ddqd_post_add on one GPU: bit-exact."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1510_08642_b200.mgpu import DistributedGemm
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        m, l, n, T = 301, 257, 299, 32
        A = gen.dd_matrix(m, l, 17, 0); B = gen.dd_matrix(l, n, 17, 1)
        C = torch.empty((2, m, n), dtype=torch.float64, device=DEV)
        dg = DistributedGemm(2, algo, T, m, l, n, dist, DEV, k=k)
        dg(cu(A), cu(B), C)
        assert same(np_(C), orc.gemm(A, B, algo, threshold=T))
    finally:
        dist.destroy_process_group()


def test_lu_per_column_path_bitwise(tmp_path):
    """The per-column two-kernel panel schedule (DDQD_LU_PANEL=steps) gives the same bits as
    the cooperative panel kernel (run in a subprocess: the switch is read once per process)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "A = gen.dd_matrix(300, 300, 13, 0); b = gen.dd_matrix(1, 300, 13, 1)[:, 0, :].copy()\n"
        "x, LU, piv, info = d.dd_lu_solve(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), 64, 'strassen', 32)\n"
        "q = gen.qd_matrix(200, 200, 3, 0); qb = gen.qd_matrix(1, 200, 3, 1)[:, 0, :].copy()\n"
        "qx, qLU, qp, qi = d.qd_lu_solve(torch.from_numpy(q).cuda(), torch.from_numpy(qb).cuda(), 48, 'winograd', 16)\n"
        "np.save(r'%s', np.concatenate([LU.cpu().numpy().ravel(), x.cpu().numpy().ravel(), piv.cpu().numpy().astype(np.float64),"
        " qLU.cpu().numpy().ravel(), qx.cpu().numpy().ravel()]))\n")
    outs = []
    for mode in ("steps", "coop"):
        f = tmp_path / f"{mode}.npy"
        env = dict(os.environ, DDQD_LU_PANEL=mode)
        subprocess.check_call([sys.executable, "-c", code % f], env=env, cwd=ROOT)
        outs.append(np.load(f))
    assert same(outs[0], outs[1])


# ---- QD LU and the paper's pivot-free LU -----------------------
def _qd_lu_matrix(n, seed):
    A = gen.qd_matrix(n, n, seed, 0)
    A[0, np.arange(n), np.arange(n)] += n
    return A


@pytest.mark.parametrize("pivot", [True, False])
@pytest.mark.parametrize("W", [2, 4])
def test_lu_qd_and_pivot_free_bitwise(orc, W, pivot):
    """DD/QD LU with and without pivoting (the paper's pivot-free LU), Winograd update,
    on a random non-dominant matrix (pivoting path) and bit-exact vs the oracle."""
    n = 200
    A = gen.matrix(W, n, n, 23, 0)
    b = gen.matrix(W, 1, n, 23, 1)[:, 0, :].copy()
    x_ref, LU_ref, piv_ref, info_ref = orc.solve(A, b, panel=48, algo="winograd", threshold=16, pivot=pivot)
    x, LU, piv, info = ddqd.lu_solve(cu(A), cu(b), panel=48, algo="winograd", threshold=16, pivot=pivot)
    assert info == info_ref == 0
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref) and same(np_(x), x_ref)


@pytest.mark.parametrize("W", [2, 4])
def test_lu_pivot_ties_below_leading_word_bitwise(orc, W):
    """Pivot candidates whose leading words are equal up to sign, so the sign fold and the
    lower words decide the pivot (the oracle's order is pinned against exact elimination,
    tests/test_oracle_lu.py); the device picks the same rows and produces the same bits."""
    n = 160
    rng = np.random.default_rng(5 + W)
    A = gen.matrix(W, n, n, 29, 0) * rng.choice([-1.0, 1.0], (1, n, n))
    for k in range(0, n, 7):                      # copy the leading word(s) down each 7th column
        rows = rng.choice(np.arange(k, n), size=min(12, n - k), replace=False)
        A[:W // 2, rows, k] = A[:W // 2, rows[:1], k] * rng.choice([-1.0, 1.0], rows.size)
    b = gen.matrix(W, 1, n, 29, 1)[:, 0, :].copy()
    x_ref, LU_ref, piv_ref, info_ref = orc.solve(A, b, panel=32, algo="strassen", threshold=16)
    x, LU, piv, info = ddqd.lu_solve(cu(A), cu(b), panel=32, algo="strassen", threshold=16)
    assert info == info_ref
    assert np.any(piv_ref != np.arange(n))
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref) and same(np_(x), x_ref)


def test_qd_lu_c4_recipe_512_bitwise(orc):
    n = 512
    A = _qd_lu_matrix(n, 5)
    ones = np.zeros((4, n, 1)); ones[0] = 1.0
    b = orc.gemm(A, ones, "block")[:, :, 0].copy()
    x_ref, LU_ref, _, _ = orc.solve(A, b, panel=128, algo="strassen", threshold=64)
    x, LU, piv, info = ddqd.qd_lu_solve(cu(A), cu(b), panel=128, algo="strassen", threshold=64)
    assert info == 0 and same(np_(LU), LU_ref) and same(np_(x), x_ref)


# ---- fused DD madd variant (DDQD_MADD_FUSED) --------------------
def test_dd_madd_fused_elementwise_bitwise(orc):
    x, y, w = _dd_samples(100000, 4), _dd_samples(100000, 5), _dd_samples(100000, 6)
    assert same(np_(ddqd.elementwise("madd_fused", cu(x), cu(y), cu(w))), orc.dd_op("madd_fused", x, y, w))


@pytest.mark.parametrize("algo", ["block", "strassen", "winograd"])
def test_fused_madd_gemm_bitwise(orc, algo):
    for (m, l, n, T) in [(65, 66, 67, 16), (301, 257, 299, 64), (1024, 1024, 1024, 128)]:
        A = gen.dd_matrix(m, l, 31, 0)
        B = gen.dd_matrix(l, n, 31, 1)
        got = np_(ddqd.gemm(cu(A), cu(B), algo, T, madd="fused"))
        assert same(got, orc.gemm(A, B, algo, threshold=T, madd="fused")), (m, l, n)


def test_fused_madd_lu_and_qd(orc):
    """Fused-madd LU (DD) and the fused QD multiply-add (elementwise and GEMM), bitwise."""
    n = 160
    A = gen.lu_matrix(n, 5)
    b = _b_ones(orc, A)
    x_ref, LU_ref, _, _ = orc.solve(A, b, panel=32, algo="strassen", threshold=16, madd="fused")
    x, LU, piv, info = ddqd.lu_solve(cu(A), cu(b), panel=32, algo="strassen", threshold=16, madd="fused")
    assert info == 0 and same(np_(LU), LU_ref) and same(np_(x), x_ref)
    qx, qy, qw = (_qd_samples(orc, 50000, s) for s in (61, 62, 63))
    qx[:, :5000] = -orc.qd_op("mul", qy[:, :5000], qw[:, :5000])
    assert same(np_(ddqd.elementwise("madd_fused", cu(qx), cu(qy), cu(qw))), orc.qd_op("madd_fused", qx, qy, qw))
    for algo, (m, l, n_, T) in (("block", (65, 70, 61, 8)), ("winograd", (130, 129, 131, 16)),
                                ("strassen", (300, 257, 299, 64))):
        Q1, Q2 = gen.qd_matrix(m, l, 3, 0), gen.qd_matrix(l, n_, 3, 1)
        got = np_(ddqd.gemm(cu(Q1), cu(Q2), algo, T, madd="fused"))
        assert same(got, orc.gemm(Q1, Q2, algo, threshold=T, madd="fused")), algo


# ---- schedule / plumbing robustness ---------------------------------------------------------
def test_batch_beyond_grid_z_limit(orc):
    """> 65535 problems in one batched call (the leaf splits grid.z)."""
    batch, m = 70000, 3
    A = gen.dd_matrix(batch * m, m, 41, 0).reshape(2, batch, m, m).transpose(1, 0, 2, 3).copy()
    B = gen.dd_matrix(batch * m, m, 41, 1).reshape(2, batch, m, m).transpose(1, 0, 2, 3).copy()
    C = torch.empty((batch, 2, m, m), dtype=torch.float64, device=DEV)
    ddqd.gemm_batched(cu(A), cu(B), C, "block", 1)
    got = np_(C)
    for b in (0, 1, 65534, 65535, 65536, batch - 1):
        assert same(got[b], orc.gemm(A[b], B[b], "block"))


@pytest.mark.parametrize("limit_mb", [1, 40])
def test_depth_first_schedule_same_bits(orc, limit_mb):
    """A small workspace limit forces depth-first top levels (chunked batches); results are
    bitwise those of the breadth-first schedule and the oracle."""
    A = gen.dd_matrix(515, 517, 43, 0)
    B = gen.dd_matrix(517, 513, 43, 1)
    ref = orc.gemm(A, B, "winograd", threshold=32)
    try:
        ddqd.set_workspace_limit(limit_mb << 20)
        got = np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", 32))
    finally:
        ddqd.set_workspace_limit(0)
        ddqd.release()
    assert same(got, ref)


def test_caller_workspace_and_stream(orc):
    """Caller-owned workspace (ddqd_set_workspace) and a non-default torch stream."""
    import ctypes
    A = gen.dd_matrix(300, 280, 44, 0)
    B = gen.dd_matrix(280, 290, 44, 1)
    need = ddqd.workspace_bytes(2, 300, 280, 290, "strassen", 40)
    assert need > 0
    ws = torch.empty(need // 8 + 1, dtype=torch.float64, device=DEV)
    s = torch.cuda.Stream()
    try:
        ddqd.lib.ddqd_set_workspace(ctypes.c_void_p(ws.data_ptr()), need)
        with torch.cuda.stream(s):
            gA, gB = cu(A), cu(B)
            C = ddqd.dd_gemm(gA, gB, "strassen", 40)
        s.synchronize()
        got = C.cpu().numpy()
        # too small a caller workspace -> ENOMEM, not a crash
        ddqd.lib.ddqd_set_workspace(ctypes.c_void_p(ws.data_ptr()), 1024)
        with pytest.raises(ddqd.DDQDError):
            ddqd.dd_gemm(gA, gB, "strassen", 40)
    finally:
        ddqd.lib.ddqd_set_workspace(None, 0)
    assert same(got, orc.gemm(A, B, "strassen", threshold=40))


def test_launch_count_and_profile():
    A = cu(gen.dd_matrix(256, 256, 1, 0))
    n0 = ddqd.launch_count()
    ddqd.profile_start()
    ddqd.dd_gemm(A, A, "strassen", 64)
    prof = ddqd.profile_stop()
    # depth 2, breadth-first: the two levels of additions run fused (one pre-add per side,
    # one post-add) around ONE batched leaf launch of the 49 products
    assert ddqd.launch_count() - n0 == 4
    assert prof["leaf"][1] == 1 and prof["leaf"][2] == 49 * 64 ** 3
    assert prof["pre"][1] == 2 and prof["post"][1] == 1


@pytest.mark.parametrize("W", [2, 4])
def test_exhaustive_small_shapes_all_algorithms(orc, W):
    """Every m, l, n in 1..7 with every algorithm at thresholds 1 and 2 (forcing recursion,
    padding at every odd level): bit-exact vs the oracle."""
    import itertools
    for m, l, n in itertools.product(range(1, 8), repeat=3):
        A = gen.matrix(W, m, l, 100 * m + 10 * l + n, 0)
        B = gen.matrix(W, l, n, 100 * m + 10 * l + n, 1)
        gA, gB = cu(A), cu(B)
        for algo, T in (("block", 1), ("strassen", 1), ("winograd", 1), ("strassen", 2), ("winograd", 2)):
            got = np_(ddqd.gemm(gA, gB, algo, T))
            assert same(got, orc.gemm(A, B, algo, threshold=T)), (m, l, n, algo, T)


@pytest.mark.parametrize("W", [2, 4])
def test_lu_tiny_and_ragged_panels(orc, W):
    """n in {1, 2, 3, 17, 70} with panels {1, 4, 64} (n < panel, ragged last panel, K = 1):
    bit-exact vs the oracle, pivoted and pivot-free."""
    for n in (1, 2, 3, 17, 70):
        A = gen.matrix(W, n, n, 50 + n, 0)
        A[0, np.arange(n), np.arange(n)] += 2.0
        b = gen.matrix(W, 1, n, 50 + n, 1)[:, 0, :].copy()
        for K in (1, 4, 64):
            for piv in (True, False):
                xr, LUr, pr, ir = orc.solve(A, b, panel=K, algo="winograd", threshold=2, pivot=piv)
                x, LU, p, info = ddqd.lu_solve(cu(A), cu(b), panel=K, algo="winograd", threshold=2, pivot=piv)
                assert info == ir
                assert np.array_equal(np_(p), pr) and same(np_(LU), LUr) and same(np_(x), xr), (n, K, piv)


def test_qd_host_pointer_path(orc):
    A = gen.qd_matrix(90, 77, 61, 0)
    B = gen.qd_matrix(77, 85, 61, 1)
    hC = ddqd.qd_gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), "strassen", 16)
    assert same(hC.numpy(), orc.gemm(A, B, "strassen", threshold=16))


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
def test_two_level_fused_additions_same_bits(orc, algo, tmp_path):
    """The two-level fused pre/post-additions (recursion.cu, DD) against the one-level
    kernels (DDQD_FUSE2=0 in a fresh process) and the oracle: odd shapes at depth 2..5 so
    the skipped level and the grandchildren are padded, DFS-chunked and BFS schedules."""
    import subprocess, sys, textwrap
    cases = [(37, 29, 33, 4), (65, 66, 67, 16), (101, 45, 77, 10), (515, 517, 513, 32), (9, 130, 11, 2)]
    outs = {}
    for fuse in ("1", "0"):
        code = textwrap.dedent(f"""
            import numpy as np, torch, sys
            sys.path.insert(0, {ROOT!r})
            import ddqd_inputs as gen, paper_1510_08642_b200 as ddqd
            res = []
            for (m, l, n, T) in {cases!r}:
                A = gen.dd_matrix(m, l, 7 * m + T, 0); B = gen.dd_matrix(l, n, 7 * m + T, 1)
                C = ddqd.dd_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), {algo!r}, T)
                res.append(C.cpu().numpy())
            np.savez(sys.argv[1], *res)
        """)
        path = str(tmp_path / f"fuse2_{algo}_{fuse}.npz")
        env = dict(os.environ, DDQD_FUSE2=fuse)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env)
        z = np.load(path)
        outs[fuse] = [z["arr_%d" % i] for i in range(len(cases))]
    for i, (m, l, n, T) in enumerate(cases):
        A = gen.dd_matrix(m, l, 7 * m + T, 0); B = gen.dd_matrix(l, n, 7 * m + T, 1)
        ref = orc.gemm(A, B, algo, threshold=T)
        assert same(outs["1"][i], ref), (m, l, n, T)
        assert same(outs["0"][i], ref), (m, l, n, T)


# ---- accurate-add variant (row f3, DDQD_ADD_ACCURATE) ----------------------------------------
def _qd_samples(orc, n, seed, cancel=True):
    rng = np.random.default_rng(seed)
    raw = [rng.uniform(-1, 1, n) * np.exp2(rng.integers(-20, 20, n))]
    for _ in range(3):
        raw.append(raw[-1] * 2.0 ** -53 * rng.uniform(-1, 1, n))
    raw.append(np.zeros(n))
    return orc.qd_renorm(np.stack(raw))


def test_accurate_add_elementwise_bitwise(orc):
    """Device accurate DD/QD add, sub and madd (numerics.md s.2-3) vs the oracle, bitwise,
    including exact and leading-word cancellation (the merge / ThreeAccum branches)."""
    x, y, w = _dd_samples(100000, 41), _dd_samples(100000, 42), _dd_samples(100000, 43)
    y[:, :20000] = -x[:, :20000]
    y[1, 10000:20000] = _dd_samples(10000, 44)[1]
    y[:, 10000:20000] = orc.dd_op("add", y[:, 10000:20000], np.zeros((2, 10000)))
    for op in ("add_acc", "sub_acc", "madd_acc"):
        got = np_(ddqd.elementwise(op, cu(x), cu(y), cu(w)))
        assert same(got, orc.dd_op(op, x, y, w)), op
    qx, qy, qw = (_qd_samples(orc, 40000, s) for s in (45, 46, 47))
    qy[:, :8000] = -qx[:, :8000]
    qy[1:, 4000:8000] = _qd_samples(orc, 4000, 48)[1:]
    qy[:, 4000:8000] = orc.qd_renorm(np.vstack([qy[:, 4000:8000], np.zeros((1, 4000))]))
    qy[:, 8000:9000] = 0.0
    for op in ("add_acc", "sub_acc", "madd_acc"):
        got = np_(ddqd.elementwise(op, cu(qx), cu(qy), cu(qw)))
        assert same(got, orc.qd_op(op, qx, qy, qw)), op


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("algo", ["block", "strassen", "winograd"])
def test_accurate_add_gemm_bitwise(orc, W, algo):
    """GEMM with every addition accurate: bit-exact vs the oracle's accurate variant on odd
    shapes at several depths (DD up to 1024^3 at depth 3)."""
    cases = [(37, 29, 33, 4), (65, 66, 67, 16), (301, 257, 299, 64)]
    if W == 2:
        cases.append((1024, 1024, 1024, 128))
    for (m, l, n, T) in cases:
        A = gen.matrix(W, m, l, 51 + m, 0)
        B = gen.matrix(W, l, n, 51 + m, 1)
        got = np_(ddqd.gemm(cu(A), cu(B), algo, T, madd="accurate"))
        assert same(got, orc.gemm(A, B, algo, threshold=T, madd="accurate")), (m, l, n, T)


def test_accurate_add_rejections():
    A = cu(gen.dd_matrix(16, 16, 1, 0))
    b = torch.zeros(2, 16, dtype=torch.float64, device=DEV)
    with pytest.raises(ddqd.DDQDError):
        ddqd.lu_solve(A.clone(), b, panel=8, algo="strassen", threshold=4, madd="accurate")
    with pytest.raises(ValueError):   # DDQD_EINVAL: the two variants are exclusive
        ddqd.gemm(A, A, ddqd.MADD_FUSED | ddqd.ADD_ACCURATE | 1, 4)


# ---- LU steps as separate calls + the distributed LU (row f4) --------------------------------
@pytest.mark.parametrize("W", [2, 4])
def test_lu_panel_and_trsv_entry_points(orc, W):
    """ddqd_lu_panel per panel + the caller's Schur update (ddqd_gemm_ex, beta = 1) +
    ddqd_lu_trsv reproduce the one-call LU and the oracle bitwise (ragged last panel)."""
    n, K, T = 150, 32, 8
    A0 = gen.lu_matrix(n, 12) if W == 2 else gen.matrix(4, n, n, 12, 0)
    ones = np.zeros((W, n, 1)); ones[0] = 1.0
    b = orc.gemm(A0, ones, "block")[:, :, 0].copy()
    xr, LUr, pr, ir = orc.solve(A0, b, panel=K, algo="winograd", threshold=T)
    A = cu(A0)
    ipiv = torch.empty(n, dtype=torch.int64, device=DEV)
    info = 0
    for p in range(0, n, K):
        kb = min(K, n - p)
        info = info or ddqd.lu_panel(A, ipiv, p, kb)
        n2 = n - p - kb
        if n2 > 0:
            base = A.data_ptr()
            ddqd.gemm_ex(W, "winograd", T, n2, kb, n2, 1,
                         base + 8 * ((p + kb) * n + p), n, n * n, 0,
                         base + 8 * (p * n + p + kb), n, n * n, 0,
                         base + 8 * ((p + kb) * n + p + kb), n, n * n, 0, beta=1)
    x = ddqd.lu_trsv(A, ipiv, cu(b))
    assert info == ir
    assert same(np_(A), LUr) and np.array_equal(np_(ipiv), pr) and same(np_(x), xr)


@pytest.mark.parametrize("algo", ["strassen", "block"])
def test_distributed_lu_cuda_backend_world1(orc, algo):
    """DistributedLU through the library (ddqd_lu_panel, DistributedGemm with beta = 1 on the
    strided trailing block, ddqd_lu_trsv) on one GPU over NCCL: bitwise the single-GPU LU."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1510_08642_b200.mgpu import DistributedLU
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        n, K, T = 300, 64, 16
        A0 = gen.lu_matrix(n, 13)
        b = _b_ones(orc, A0).copy()
        A = cu(A0)
        x, ipiv, info = DistributedLU(2, n, K, algo, T, dist)(A, cu(b))
        xr, LUr, pr, ir = orc.solve(A0, b, panel=K, algo=algo, threshold=T)
        assert info == ir and same(np_(A), LUr) and same(np_(x), xr)
        assert np.array_equal(np_(ipiv), pr)
    finally:
        dist.destroy_process_group()


# ---- fused p2p combine over CUDA IPC mappings (row e) -------------------------------------------
@pytest.mark.parametrize("cfg,world", [
    ((2, "winograd", 32, 301, 257, 299, 1), 2),
    ((2, "strassen", 16, 200, 203, 190, 2), 3),
    ((4, "winograd", 16, 130, 129, 131, 2), 2),
])
def test_p2p_combine_cuda_ipc_bitwise(orc, cfg, world):
    """DistributedGemm(combine='p2p') with 2-3 processes on this GPU: every process computes its
    depth-k products into its own cudaMalloc buffer, the post-addition levels read them through
    CUDA IPC mappings (ddqd_post_add_ptrs), split over the processes, and each writes its rows
    of C into rank 0's buffer: bit-identical to the single-GPU recursion and the oracle."""
    import multiprocessing as pymp
    import socket
    from tests import _p2p_worker
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = pymp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker.run, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    k, C = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert k != "error", C
    assert all(p.exitcode == 0 for p in procs)
    W, algo, T, m, l, n, _ = cfg
    ref = orc.gemm(gen.matrix(W, m, l, 31, 0), gen.matrix(W, l, n, 31, 1), algo, threshold=T)
    assert k >= 1 and same(C, ref)


# ---- split-k leaf: clusters of CTAs reducing through distributed shared memory (row a4) ---------
def test_splitk_tree_pin_on_device(orc):
    """The oracle's tree-order pin (1 + 2^-120 kept only by the pairwise tree) on the device."""
    A = np.zeros((2, 1, 4)); A[0] = 1.0
    B = np.zeros((2, 4, 1))
    B[0, :, 0] = [1.0, 0.0, 2.0 ** -60, -2.0 ** -60]
    B[1, 2, 0] = 2.0 ** -120
    for s in (2, 4, 8):
        got = np_(ddqd.dd_gemm(cu(A), cu(B), "block", splitk=s))
        assert list(got[:, 0, 0]) == [1.0, 2.0 ** -120]
        assert same(got, orc.gemm(A, B, "block", splitk=s))


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("s", [2, 4, 8])
def test_splitk_bitwise(orc, W, s):
    """Split-k leaves bit-identical to the oracle: ragged tiles, l < s (empty slices), l not a
    multiple of s or of the 16-deep k chunk, Block and recursion leaves, the accurate variant."""
    cases = [("block", 37, 29, 33, 1), ("block", 5, 3, 7, 1), ("block", 64, 100, 70, 1),
             ("winograd", 67, 66, 65, 16), ("strassen", 40, 41, 42, 8)]
    for algo, m, l, n, T in cases:
        A = gen.matrix(W, m, l, 5 * m + s, 0)
        B = gen.matrix(W, l, n, 5 * m + s, 1)
        got = np_(ddqd.gemm(cu(A), cu(B), algo, T, splitk=s))
        assert same(got, orc.gemm(A, B, algo, threshold=T, splitk=s)), (algo, m, l, n)
    A = gen.matrix(W, 45, 50, 9, 0); B = gen.matrix(W, 50, 40, 9, 1)
    got = np_(ddqd.gemm(cu(A), cu(B), "block", madd="accurate", splitk=s))
    assert same(got, orc.gemm(A, B, "block", madd="accurate", splitk=s))


def test_c0_splitk8(orc):
    """BJ:7 (config 0) with the split-k leaf (8-CTA clusters, 128 CTAs for the 16 tiles):
    bit-exact vs the oracle's split-k and within 2^-96 l |A||B| of the exact product."""
    A = gen.dd_matrix(128, 128, 1, 0)
    B = gen.dd_matrix(128, 128, 1, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), "block", splitk=8))
    assert same(got, orc.gemm(A, B, "block", splitk=8))
    r, c = np.meshgrid(np.arange(128), np.arange(128), indexing="ij")
    _, err = orc.exact_entries(A, B, got, r.ravel(), c.ravel())
    assert np.abs(err).max() <= 2.0 ** -96 * 128 * np.abs(A[0]).max() * np.abs(B[0]).max()


def test_two_lane_schedule_same_bits(orc, tmp_path):
    """DDQD_LANES=2 (the last depth-first level's chunks alternate between two streams with
    separate workspace): bit-identical to the oracle, under a workspace limit that forces
    depth-first levels."""
    import subprocess, sys, textwrap
    code = textwrap.dedent(f"""
        import numpy as np, torch, sys
        sys.path.insert(0, {ROOT!r})
        import ddqd_inputs as gen, paper_1510_08642_b200 as ddqd
        A = gen.dd_matrix(515, 517, 43, 0); B = gen.dd_matrix(517, 513, 43, 1)
        ddqd.set_workspace_limit(60 << 20)   # depth-first top 2 levels (37 MB), second lane fits (51 MB)
        C = ddqd.dd_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), "winograd", 32)
        Q = gen.qd_matrix(260, 250, 5, 0); R = gen.qd_matrix(250, 270, 5, 1)
        D = ddqd.qd_gemm(torch.from_numpy(Q).cuda(), torch.from_numpy(R).cuda(), "strassen", 16)
        np.savez(sys.argv[1], C.cpu().numpy(), D.cpu().numpy())
    """)
    path = str(tmp_path / "lanes.npz")
    subprocess.run([sys.executable, "-c", code, path], check=True, env=dict(os.environ, DDQD_LANES="2"))
    z = np.load(path)
    A = gen.dd_matrix(515, 517, 43, 0); B = gen.dd_matrix(517, 513, 43, 1)
    assert same(z["arr_0"], orc.gemm(A, B, "winograd", threshold=32))
    Q = gen.qd_matrix(260, 250, 5, 0); R = gen.qd_matrix(250, 270, 5, 1)
    assert same(z["arr_1"], orc.gemm(Q, R, "strassen", threshold=16))


@pytest.mark.parametrize("algo,madd", [("strassen", "canonical"), ("winograd", "canonical"),
                                       ("strassen", "fused"), ("winograd", "accurate")])
def test_leaf_tail_split_bitwise(orc, algo, madd):
    """The DD leaf tail split (whole waves on 64x64 tiles, the remaining leaves on 32x32
    tiles): 557^3 with T = 64 gives 343 ragged 70x70 leaves = 1372 CTAs, 4.6 waves -- the
    c1 situation with ragged tiles; bit-identical to the oracle for every madd variant."""
    m, l, n = 557, 556, 558
    A = gen.dd_matrix(m, l, 31, 0)
    B = gen.dd_matrix(l, n, 31, 1)
    got = np_(ddqd.dd_gemm(cu(A), cu(B), algo, 64, madd=madd))
    assert same(got, orc.gemm(A, B, algo, threshold=64, madd=madd))


@pytest.mark.parametrize("W", [2, 4])
def test_host_streamed_winograd_bitwise(orc, W):
    """The overlapped host path (Winograd: A11, B11 copied first and M1 = A11 B11 computed
    while the rest of A and B is copied; then the top level's pre-adds, M2..M7 as a batch,
    the post-adds): bitwise the device-pointer call and the oracle -- odd and even
    dimensions (ragged quadrants), depth 1 to 3, pinned and pageable host memory, the
    arithmetic variants."""
    gemm = ddqd.dd_gemm if W == 2 else ddqd.qd_gemm
    cases = [(129, 130, 131, 64, "canonical", True), (200, 201, 199, 32, "canonical", False),
             (97, 64, 65, 16, "accurate", True), (66, 67, 68, 32, "fused", True)]
    for m, l, n, T, madd, pin in cases:
        A = gen.matrix(W, m, l, m + T, 0)
        B = gen.matrix(W, l, n, m + T, 1)
        hA, hB = torch.from_numpy(A), torch.from_numpy(B)
        if pin:
            hA, hB = hA.pin_memory(), hB.pin_memory()
        hC = gemm(hA, hB, "winograd", T, madd=madd).numpy()
        assert same(hC, np_(gemm(cu(A), cu(B), "winograd", T, madd=madd))), (m, l, n, madd)
        assert same(hC, orc.gemm(A, B, "winograd", threshold=T, madd=madd)), (m, l, n, madd)


@pytest.mark.parametrize("madd", ["canonical", "accurate"])
def test_host_streamed_winograd_quadrant_copies(madd):
    """The quadrant-by-quadrant host path (C quadrants >= 32 MB: each formed by its own
    post-addition pass and copied back while the next products run): bitwise the
    device-pointer call, ragged quadrants (odd m and n), pinned and pageable C."""
    m, l, n, T = 2901, 130, 2899, 64
    A = gen.dd_matrix(m, l, 77, 0)
    B = gen.dd_matrix(l, n, 77, 1)
    dev = np_(ddqd.dd_gemm(cu(A), cu(B), "winograd", T, madd=madd))
    for pin in (True, False):
        hA, hB = torch.from_numpy(A), torch.from_numpy(B)
        if pin:
            hA, hB = hA.pin_memory(), hB.pin_memory()
        assert same(ddqd.dd_gemm(hA, hB, "winograd", T, madd=madd).numpy(), dev), pin


@pytest.mark.parametrize("algo,T", [("block", 128), ("winograd", 32)])
def test_cuda_graph_capture(orc, algo, T):
    """Library calls captured into a CUDA graph (the workspace warmed by one eager call first)
    replay to the oracle's bits -- the c0 bench's graph variant relies on this."""
    A = gen.dd_matrix(128, 128, 1, 0)
    B = gen.dd_matrix(128, 128, 1, 1)
    dA, dB = cu(A), cu(B)
    C = torch.empty((2, 128, 128), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ddqd.dd_gemm(dA, dB, algo, T, out=C)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    C.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ddqd.dd_gemm(dA, dB, algo, T, out=C)
    torch.cuda.synchronize()
    assert not C.abs().sum().item()   # capture does not execute
    g.replay()
    torch.cuda.synchronize()
    assert same(np_(C), orc.gemm(A, B, algo, threshold=T))


def test_randomized_shapes_all_paths(orc):
    """Seeded random sweep over shapes (1..300, ragged), thresholds, algorithms, DD/QD and the
    arithmetic variants, device and host pointers: every result bit-identical to the oracle.
    Exercises the leaf selection (small-output / 32x32 / 64x64 / TMA / tail split), the
    recursion's padding and the overlapped host path together."""
    rng = np.random.default_rng(20261019)
    for case in range(80):
        W = int(rng.choice([2, 2, 2, 4]))
        m, l, n = (int(x) for x in rng.integers(1, 301, 3))
        algo = str(rng.choice(["block", "strassen", "winograd"]))
        T = int(rng.choice([8, 16, 32, 64, 128]))
        madd = str(rng.choice(["canonical", "canonical", "fused", "accurate"]))
        host = bool(rng.integers(0, 4) == 0)
        A = gen.matrix(W, m, l, 1000 + case, 0)
        B = gen.matrix(W, l, n, 1000 + case, 1)
        gemm = ddqd.dd_gemm if W == 2 else ddqd.qd_gemm
        if host:
            got = gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), algo, T,
                       madd=madd).numpy()
        else:
            got = np_(gemm(cu(A), cu(B), algo, T, madd=madd))
        assert same(got, orc.gemm(A, B, algo, threshold=T, madd=madd)), (case, W, m, l, n, algo, T, madd, host)


def test_randomized_lu_sweep(orc):
    """Seeded random LU solves (n 1..400, panel widths incl. ragged last panels, every update
    algorithm, DD/QD, pivoting on non-dominant matrices or the paper's pivot-free mode on
    dominant ones): factors, pivots and solution bit-identical to the oracle."""
    rng = np.random.default_rng(4096)
    for case in range(16):
        W = int(rng.choice([2, 2, 4]))
        n = int(rng.integers(1, 401))
        K = int(rng.choice([16, 32, 48, 64, 100, 128, 256]))
        algo = str(rng.choice(["block", "strassen", "winograd"]))
        T = int(rng.choice([8, 16, 32, 64]))
        pivot = bool(rng.integers(0, 3) > 0)
        A = gen.matrix(W, n, n, 500 + case, 0)
        if not pivot:   # the pivot-free LU needs non-zero leading minors: make A dominant
            A[0][np.arange(n), np.arange(n)] += n
        b = gen.matrix(W, 1, n, 500 + case, 1)[:, 0, :].copy()
        ref = orc.solve(A, b, panel=K, algo=algo, threshold=T, pivot=pivot)
        got = ddqd.lu_solve(cu(A), cu(b), panel=K, algo=algo, threshold=T, pivot=pivot)
        tag = (case, W, n, K, algo, T, pivot)
        assert got[3] == ref[3] == 0, tag
        assert np.array_equal(np_(got[2]), ref[2]), tag
        assert same(np_(got[1]), ref[1]) and same(np_(got[0]), ref[0]), tag


# ---- band schedule (BandGemm) and the DDQD_DEPTH flag on one GPU -----------------------------
@pytest.mark.parametrize("W,algo,m,l,n,d", [(2, "winograd", 37, 29, 33, 3), (2, "strassen", 70, 65, 66, 2),
                                              (4, "winograd", 21, 18, 25, 2), (2, "winograd", 200, 190, 170, 0)])
def test_forced_depth_bitwise(orc, W, algo, m, l, n, d):
    """DDQD_DEPTH(d): exactly d levels whatever the shape, bit-identical to the oracle's forced
    depth (reading R21)."""
    A, B = gen.matrix(W, m, l, 43, 0), gen.matrix(W, l, n, 43, 1)
    C = torch.empty((W, m, n), dtype=torch.float64, device=DEV)
    a, b = cu(A), cu(B)
    ddqd._set_stream(a)
    ddqd.gemm_ex(W, algo, 1, m, l, n, 1, a.data_ptr(), l, m * l, 0, b.data_ptr(), n, l * n, 0,
                 C.data_ptr(), n, m * n, 0, 0, depth=d)
    assert same(np_(C), orc.gemm(A, B, algo, threshold=1, depth=d))


def test_band_copy_pack_unpack(orc):
    from paper_1510_08642_b200.mgpu import band_index_map
    rng = np.random.default_rng(3)
    for W in (2, 4):
        F = gen.matrix(W, 301, 257, 44, 0)
        rows = sorted(rng.choice(301, 77, replace=False).tolist())
        cols = band_index_map([257, 129, 65, 33], 5, 20)
        f = cu(F)
        c = torch.empty((W, len(rows), len(cols)), dtype=torch.float64, device=DEV)
        rm = torch.tensor(rows, dtype=torch.int64, device=DEV)
        cm = torch.tensor(cols, dtype=torch.int64, device=DEV)
        ddqd.band_copy("pack", f, c, rm, cm)
        assert same(np_(c), np.ascontiguousarray(F[:, np.array(rows)[:, None], np.array(cols)[None, :]]))
        g = torch.zeros_like(f)
        ddqd.band_copy("unpack", g, c, rm, cm)
        want = np.zeros_like(F)
        want[:, np.array(rows)[:, None], np.array(cols)[None, :]] = F[:, np.array(rows)[:, None], np.array(cols)[None, :]]
        assert same(np_(g), want)
        c2 = torch.empty((W, 301, len(cols)), dtype=torch.float64, device=DEV)
        ddqd.band_copy("pack", f, c2, None, cm)     # identity row map
        assert same(np_(c2), np.ascontiguousarray(F[:, :, cols]))


@pytest.mark.parametrize("W,algo,T,m,l,n,world,beta", [
    (2, "winograd", 64, 1023, 1025, 1021, 8, 0),    # c3-shaped, 2 x 4 grid
    (2, "strassen", 32, 301, 257, 299, 4, 0),
    (4, "winograd", 16, 200, 190, 170, 2, 0),       # QD
    (2, "strassen", 64, 768, 256, 768, 3, 1),       # the LU update form C := C - A B
    (2, "block", 64, 300, 200, 250, 4, 0),
])
def test_band_schedule_emulated_bitwise(orc, W, algo, T, m, l, n, world, beta):
    """Every rank's share of the band schedule run in turn on this GPU (pack -> DDQD_DEPTH GEMM
    -> unpack, the library's kernels): bit-identical to the one-GPU call, so the N-GPU result is
    too (the ranks' kernels are these; only the transport differs)."""
    from paper_1510_08642_b200.mgpu import BandGemm
    A, B = gen.matrix(W, m, l, 45, 0), gen.matrix(W, l, n, 45, 1)
    C0 = gen.matrix(W, m, n, 45, 2)
    C = cu(C0)
    BandGemm(W, algo, T, m, l, n, None, world=world, beta=beta).emulate(cu(A), cu(B), C)
    a, b = cu(A), cu(B)
    ref = cu(C0)
    ddqd._set_stream(a)
    ddqd.gemm_ex(W, algo, T, m, l, n, 1, a.data_ptr(), l, m * l, 0, b.data_ptr(), n, l * n, 0,
                 ref.data_ptr(), n, m * n, 0, beta)
    assert same(np_(C), np_(ref))
    if m <= 400 and not beta:
        assert same(np_(C), orc.gemm(A, B, algo, threshold=T))


def test_band_schedule_nccl_world1(orc):
    import socket
    import torch.distributed as dist
    from paper_1510_08642_b200.mgpu import BandGemm
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        m, l, n, T = 301, 257, 299, 32
        A = gen.dd_matrix(m, l, 17, 0); B = gen.dd_matrix(l, n, 17, 1)
        C = torch.empty((2, m, n), dtype=torch.float64, device=DEV)
        BandGemm(2, "winograd", T, m, l, n, dist)(cu(A), cu(B), C)
        assert same(np_(C), orc.gemm(A, B, "winograd", threshold=T))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [((2, "winograd", 64, 701, 513, 650), 2),
                                       ((2, "strassen", 32, 300, 257, 299), 3),
                                       ((4, "winograd", 32, 190, 170, 201), 2)])
def test_multiprocess_schedules_staged_bitwise(orc, cfg, world):
    """2-3 processes on this GPU run every multi-GPU schedule through the library (exchanges
    over gloo staged through host memory): bands, products (rank-0 combine), products with the
    p2p combine over CUDA IPC, the automatic choice, and bands with beta = 1 -- all
    bit-identical to the one-GPU call."""
    import multiprocessing as pymp
    import socket
    from tests import _p2p_worker
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = pymp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker.run_schedules, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert "error" not in out, out
    assert all(p.exitcode == 0 for p in procs)
    W, algo, T, m, l, n = cfg
    A, B = gen.matrix(W, m, l, 33, 0), gen.matrix(W, l, n, 33, 1)
    ref = np_(ddqd.gemm(cu(A), cu(B), algo, T))
    for name in ("bands", "products", "products_p2p", "products_rows", "auto"):
        assert same(out[name], ref), name
    C0 = cu(gen.matrix(W, m, n, 33, 2))
    a, b = cu(A), cu(B)
    ddqd._set_stream(a)
    ddqd.gemm_ex(W, algo, T, m, l, n, 1, a.data_ptr(), l, m * l, 0, b.data_ptr(), n, l * n, 0,
                 C0.data_ptr(), n, m * n, 0, 1)
    assert same(out["bands_beta1"], np_(C0))
    assert same(out["rows_beta1"], np_(C0))


# ---- ragged leaves: interior / strip split and the flat leaf ------------
@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("w", [17, 65, 129, 257])
def test_ragged_leaf_widths_bitwise(orc, W, w):
    """Leaves of width 17, 65, 129, 257 (n = 1025-type recursions): Block leaves directly, a
    batch of such leaves through one recursion level (Strassen with threshold w so the seven
    children are w x w), and a non-square ragged leaf; bit-identical to the oracle."""
    A, B = gen.matrix(W, w, w + 3, 47, 0), gen.matrix(W, w + 3, w, 47, 1)
    assert same(np_(ddqd.gemm(cu(A), cu(B), "block", 128)), orc.gemm(A, B, "block"))
    m = 2 * w - 1
    A2, B2 = gen.matrix(W, m, m, 48, 0), gen.matrix(W, m, m, 48, 1)
    for algo in ("strassen", "winograd"):
        got = np_(ddqd.gemm(cu(A2), cu(B2), algo, w))
        assert same(got, orc.gemm(A2, B2, algo, threshold=w)), algo
    A3, B3 = gen.matrix(W, w + 40, 33, 49, 0), gen.matrix(W, 33, w, 49, 1)
    assert same(np_(ddqd.gemm(cu(A3), cu(B3), "block", 128)), orc.gemm(A3, B3, "block"))


def test_ragged_split_same_bits_as_unsplit(tmp_path):
    """DDQD_LEAF_RAGGED=0 (whole leaves on padded CTA tiles) and the default interior / strip
    split give the same bits (subprocesses: the switch is read once per process)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "out = []\n"
        "for W, n, T in ((2, 1025, 128), (2, 1025, 32), (4, 517, 64), (4, 263, 16)):\n"
        "    A, B = gen.bench_pair(n, W)\n"
        "    for algo in ('strassen', 'winograd'):\n"
        "        out.append(d.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), algo, T).cpu().numpy().ravel())\n"
        "np.save(r'%s', np.concatenate(out))\n")
    outs = []
    for mode in ("0", "1"):
        f = tmp_path / f"r{mode}.npy"
        env = dict(os.environ, DDQD_LEAF_RAGGED=mode)
        subprocess.check_call([sys.executable, "-c", code % f], env=env, cwd=ROOT)
        outs.append(np.load(f))
    assert same(outs[0], outs[1])


# ---- ABI hardening: aliasing / stride checks, threads and streams, graph capture ----
def test_gemm_ex_alias_and_stride_checks(orc):
    """ddqd_gemm_ex rejects C overlapping A or B (EALIAS) and impossible strides (EINVAL), and
    accepts disjoint sub-blocks of one matrix (the LU's form)."""
    import ctypes
    n = 96
    M = cu(gen.dd_matrix(n, n, 51, 0))
    base = M.data_ptr()
    ps = n * n

    def call(a_off, b_off, c_off, m, l, k, psA=ps, beta=1):
        return ddqd.lib.ddqd_gemm_ex(ctypes.byref(ddqd.GemmDesc(
            2, 1, 16, m, l, k, 1, base + 8 * a_off, n, psA, 0, base + 8 * b_off, n, ps, 0,
            base + 8 * c_off, n, ps, 0, beta)))
    ddqd._set_stream(M)
    # LU-like disjoint blocks: L21 = rows 32.., cols 0..32; U12 = rows 0..32, cols 32..; A22
    assert call(32 * n, 32, 32 * n + 32, 64, 32, 64) == 0
    # C overlapping A (C's block starts inside A's block)
    assert call(0, 32, 16 * n + 16, 48, 32, 48) == -2
    # C overlapping B in the second plane only region still overlaps (same rectangles)
    assert call(32 * n, 32, 32, 32, 32, 32) == -2
    # plane stride smaller than rows * ld
    assert call(32 * n, 32, 32 * n + 32, 64, 32, 64, psA=10) == -1
    torch.cuda.synchronize()
    # panels wider than the TRSM kernels take are refused before anything runs
    assert ddqd.lib.ddqd_lu_panel(2, 1, 4000, M.data_ptr(), M.data_ptr(), 0, 1100) == -5


def test_threads_and_streams_share_the_workspace(orc):
    """Strassen/Winograd calls from two host threads, each on its own stream, with the
    library-owned workspace: every result bit-exact (the call lock + cross-stream events)."""
    import threading
    A, B = gen.dd_matrix(300, 280, 52, 0), gen.dd_matrix(280, 310, 52, 1)
    refs = {a: orc.gemm(A, B, a, threshold=32) for a in ("strassen", "winograd")}
    out, errs = {}, []

    def work(algo):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                a, b = cu(A), cu(B)
                res = [ddqd.gemm(a, b, algo, 32) for _ in range(6)]
                st.synchronize()
                out[algo] = [r.cpu().numpy() for r in res]
        except Exception as e:   # noqa: BLE001
            errs.append(repr(e))
    ts = [threading.Thread(target=work, args=(a,)) for a in ("strassen", "winograd")]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for algo, res in out.items():
        assert all(same(r, refs[algo]) for r in res), algo


def test_graph_capture_workspace_rules(orc):
    """A captured Strassen call whose workspace is already large enough replays correctly even
    after a later, larger call grows the workspace (the old buffer is retired, not freed)."""
    A, B = gen.dd_matrix(200, 200, 53, 0), gen.dd_matrix(200, 200, 53, 1)
    a, b = cu(A), cu(B)
    C = ddqd.gemm(a, b, "strassen", 32)                 # sizes the workspace outside capture
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ddqd.gemm(a, b, "strassen", 32, out=C)
    A2, B2 = gen.dd_matrix(700, 700, 54, 0), gen.dd_matrix(700, 700, 54, 1)
    big = ddqd.gemm(cu(A2), cu(B2), "strassen", 32)     # grows the workspace
    C.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert same(np_(C), orc.gemm(A, B, "strassen", threshold=32))
    assert same(np_(big), orc.gemm(A2, B2, "strassen", threshold=32))


def test_fused_last_level_same_bits(tmp_path, orc):
    """The last recursion level fused with its tiny leaves (fused_last_kernel, and the default
    fused_last_s_kernel / fused_last_q_kernel) gives the bits of the unfused schedule
    (DDQD_FUSE_LAST=0), DD and QD, Strassen and Winograd, canonical and the fused/accurate
    variants (17^3 unrolled, 18^3 and 4^3 run-time leaves), and matches the oracle on a small case."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "out = []\n"
        "for W, n, T in ((2, 1025, 32), (4, 517, 16), (2, 99, 6), (4, 70, 5), (2, 1100, 32), (4, 1025, 32)):\n"
        "    A, B = gen.bench_pair(n, W) if n > 500 else (gen.matrix(W, n, n - 3, 61, 0), gen.matrix(W, n - 3, n + 2, 61, 1))\n"
        "    for algo in ('strassen', 'winograd'):\n"
        "        for madd in ('canonical', 'fused', 'accurate'):\n"
        "            out.append(d.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), algo, T, madd=madd).cpu().numpy().ravel())\n"
        "np.save(r'%s', np.concatenate(out))\n")
    outs = []
    # unfused / the first fused kernel / the default (DD: one position per thread, 17^3
    # unrolled; QD: one product chain per thread)
    for i, extra in enumerate(({"DDQD_FUSE_LAST": "0"}, {"DDQD_FUSED_S": "0"}, {})):
        f = tmp_path / f"f{i}.npy"
        env = dict(os.environ, **extra)
        subprocess.check_call([sys.executable, "-c", code % f], env=env, cwd=ROOT)
        outs.append(np.load(f))
    assert same(outs[0], outs[1]) and same(outs[0], outs[2])
    A, B = gen.matrix(2, 99, 96, 61, 0), gen.matrix(2, 96, 101, 61, 1)
    for algo in ("strassen", "winograd"):
        assert same(np_(ddqd.gemm(cu(A), cu(B), algo, 6)), orc.gemm(A, B, algo, threshold=6))
    A, B = gen.matrix(4, 71, 68, 62, 0), gen.matrix(4, 68, 73, 62, 1)   # QD, 9 x 9 x 9 leaves
    for algo in ("strassen", "winograd"):
        assert same(np_(ddqd.gemm(cu(A), cu(B), algo, 8)), orc.gemm(A, B, algo, threshold=8))


def test_host_streamed_two_stage_bitwise(tmp_path, orc):
    """Host-pointer Winograd with M1 streamed one level deeper (DDQD_HOST_DEEP=2: A11's and B11's
    leading quadrants copied first, M1's first product overlapping the rest): bit-identical to
    the device-pointer call and the oracle, DD and QD, odd shapes."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "out = []\n"
        "for W, m, l, n, T in ((2, 301, 277, 263, 32), (4, 150, 133, 141, 16), (2, 517, 515, 513, 64)):\n"
        "    A, B = gen.matrix(W, m, l, 71, 0), gen.matrix(W, l, n, 71, 1)\n"
        "    h = d.gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), 'winograd', T).numpy()\n"
        "    g = d.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 'winograd', T).cpu().numpy()\n"
        "    out += [h.ravel(), g.ravel()]\n"
        "np.save(r'%s', np.concatenate(out))\n")
    f = tmp_path / "deep.npy"
    env = dict(os.environ, DDQD_HOST_DEEP="2")
    subprocess.check_call([sys.executable, "-c", code % f], env=env, cwd=ROOT)
    v = np.load(f)
    refs = []
    for W, m, l, n, T in ((2, 301, 277, 263, 32), (4, 150, 133, 141, 16), (2, 517, 515, 513, 64)):
        A, B = gen.matrix(W, m, l, 71, 0), gen.matrix(W, l, n, 71, 1)
        r = orc.gemm(A, B, "winograd", threshold=T).ravel()
        refs += [r, r]
    assert same(v, np.concatenate(refs))


def test_host_streamed_tail_blocks_bitwise(tmp_path):
    """Host-pointer Winograd large enough for the block-by-block copy-back (C quadrants >= 32 MB):
    the last product M4 runs one or more levels deeper and C21 is formed and copied back block
    by block; M1 streamed as deep as the recursion allows with DDQD_HOST_DEEP=2. Bit-identical
    to the device-pointer call and to DDQD_HOST_TAIL=0 / DDQD_HOST_DEEP=0 (M4 in one pass, M1
    on one copy stage), DD and QD, odd shapes (ragged halves at every level)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "out = []\n"
        "for W, m, l, n, T in ((2, 3001, 263, 2999, 64), (4, 2049, 133, 2051, 32)):\n"
        "    A, B = gen.matrix(W, m, l, 73, 0), gen.matrix(W, l, n, 73, 1)\n"
        "    h = d.gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), 'winograd', T).numpy()\n"
        "    g = d.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 'winograd', T).cpu().numpy()\n"
        "    out += [h.ravel(), g.ravel()]\n"
        "np.save(r'%s', np.concatenate(out))\n")
    outs = []
    for i, extra in enumerate(({}, {"DDQD_HOST_TAIL": "0", "DDQD_HOST_DEEP": "0"},
                               {"DDQD_HOST_TAIL": "2", "DDQD_HOST_DEEP": "2"})):
        f = tmp_path / f"t{i}.npy"
        subprocess.check_call([sys.executable, "-c", code % f], env=dict(os.environ, **extra), cwd=ROOT)
        outs.append(np.load(f))
    assert same(outs[0], outs[1]) and same(outs[0], outs[2])
    v = outs[0]
    k = 0
    for W, m, n in ((2, 3001, 2999), (4, 2049, 2051)):
        sz = W * m * n
        assert same(v[k:k + sz], v[k + sz:k + 2 * sz])   # host == device pointers
        k += 2 * sz


@pytest.mark.parametrize("m,l", [(128, 257), (192, 129), (127, 257)])
def test_row_pair_tma_leaf_bitwise(orc, m, l):
    """Batched Block leaves whose A rows are not 16-byte aligned (odd ld) but whose B rows are:
    even row counts take the row-pair TMA view (c3's leaf path), an odd row count falls back to
    the cp.async leaf; both bit-identical to the oracle, element by element, for every leaf."""
    batch, n = 80, 128
    A = np.stack([gen.dd_matrix(m, l, 81, b) for b in range(batch)])
    B = np.stack([gen.dd_matrix(l, n, 82, b) for b in range(batch)])
    C = torch.empty((batch, 2, m, n), dtype=torch.float64, device=DEV)
    ddqd.gemm_batched(cu(A), cu(B), C, "block", 1)
    got = np_(C)
    for b in range(0, batch, 9):
        assert same(got[b], orc.gemm(A[b], B[b], "block")), b


def test_lu_split_panel_bitwise(orc, tmp_path):
    """The split panel (the diagonal block on one thread-block cluster, the rows below
    eliminated warp by warp, committed only when the speculated pivots all hold) gives the
    bits of the cooperative panel (DDQD_LU_SPLIT=0) and of the oracle: panels where the
    speculation holds and panels where it misses in the same solve (the gated fallback factors
    those), a ragged last panel, K < 256, QD (16-CTA cluster), pivot-free, and an exactly zero
    pivot (info). Subprocesses: the switch is read once per process."""
    import subprocess
    import sys
    code = (
        "import json, numpy as np, torch, ddqd_inputs as gen, paper_1510_08642_b200 as d\n"
        "def dom_first(W, n, seed, cols):\n"
        "    A = gen.matrix(W, n, n, seed, 0); A[0, np.arange(cols), np.arange(cols)] += n; return A\n"
        "cases = [(2, dom_first(2, 600, 31, 256), 256, 'strassen', 64, True),\n"
        "         (2, gen.lu_matrix(700, 5), 256, 'winograd', 64, True),\n"
        "         (4, dom_first(4, 400, 32, 400), 256, 'strassen', 64, True),\n"
        "         (2, gen.dd_matrix(300, 300, 33, 0), 128, 'block', 1, False),\n"
        "         (2, gen.dd_matrix(300, 300, 34, 0), 100, 'winograd', 32, True)]\n"
        "z = gen.lu_matrix(100, 6); z[:, :, 7] = 0.0\n"
        "cases.append((2, z, 64, 'strassen', 16, True))\n"
        "out, infos = [], []\n"
        "d.profile_start()\n"
        "for W, A, K, algo, T, piv in cases:\n"
        "    n = A.shape[1]; b = gen.matrix(W, 1, n, 35, 1)[:, 0, :].copy()\n"
        "    x, LU, p, info = d.lu_solve(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), panel=K, algo=algo,\n"
        "                                threshold=T, pivot=piv)\n"
        "    out += [LU.cpu().numpy().ravel(), x.cpu().numpy().ravel(), p.cpu().numpy().astype(np.float64)]\n"
        "    infos.append(int(info))\n"
        "d.profile_stop()\n"
        "np.save(r'%s', np.concatenate(out))\n"
        "json.dump({'info': infos, 'kernels': sorted(d.profile_kernels())}, open(r'%s.json', 'w'))\n")
    outs, meta = [], []
    for mode in ("1", "0"):
        f = tmp_path / f"s{mode}.npy"
        subprocess.check_call([sys.executable, "-c", code % (f, f)], env=dict(os.environ, DDQD_LU_SPLIT=mode), cwd=ROOT)
        outs.append(np.load(f))
        meta.append(json.load(open(f"{f}.json")))
    assert same(outs[0], outs[1])
    assert meta[0]["info"] == meta[1]["info"] and meta[0]["info"][-1] == 8 and meta[0]["info"][:-1] == [0] * 5
    assert any("split panel" in k for k in meta[0]["kernels"])
    assert not any("split panel" in k for k in meta[1]["kernels"])
    # the first case (speculation holds in panel 0, misses later) and the QD case vs the oracle
    v, k = outs[0], 0
    A1 = gen.matrix(2, 600, 600, 31, 0); A1[0, np.arange(256), np.arange(256)] += 600
    b1 = gen.matrix(2, 1, 600, 35, 1)[:, 0, :].copy()
    x_ref, LU_ref, piv_ref, _ = orc.solve(A1, b1, panel=256, algo="strassen", threshold=64)
    assert np.any(piv_ref[256:] != np.arange(256, 600)) and np.array_equal(piv_ref[:256], np.arange(256))
    assert same(v[k:k + LU_ref.size], LU_ref.ravel()); k += LU_ref.size
    assert same(v[k:k + x_ref.size], x_ref.ravel()); k += x_ref.size
    assert np.array_equal(v[k:k + 600], piv_ref.astype(np.float64))


@pytest.mark.parametrize("W,n,K", [(2, 1000, 128), (4, 800, 256), (2, 1280, 256)])
def test_lu_backward_lookahead_bitwise(orc, W, n, K):
    """The backward solve's look-ahead (block J's columns folded into the next diagonal block's
    rows on the caller's stream, into the rows above on a side stream; DDQD_LU_BWD_OVERLAP) on
    several 256-row blocks: a ragged bottom block (n = 1000: 232 rows, the per-element path),
    a 32-row bottom block (QD n = 800), whole blocks (n = 1280); non-dominant random matrices
    so the rows are interchanged. Bit-exact vs the oracle's factors and solution."""
    A = gen.matrix(W, n, n, 41 + n, 0)
    b = gen.matrix(W, 1, n, 42 + n, 1)[:, 0, :].copy()
    x_ref, LU_ref, piv_ref, info_ref = orc.solve(A, b, panel=K, algo="strassen", threshold=64)
    x, LU, piv, info = ddqd.lu_solve(cu(A), cu(b), panel=K, algo="strassen", threshold=64)
    assert info == info_ref == 0
    assert np.any(piv_ref != np.arange(n))
    assert np.array_equal(np_(piv), piv_ref)
    assert same(np_(LU), LU_ref) and same(np_(x), x_ref)
