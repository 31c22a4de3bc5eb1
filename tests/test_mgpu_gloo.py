"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU schedule's host logic
(paper_1510_08642_b200/mgpu.py): depth-k product distribution and C row-slab tiling must
reproduce the single-process recursion bit for bit. The compute backend here is built
from the oracle (tests only); on GPUs the same schedule drives libddqd.so over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ddqd_inputs as gen

# mgpu.py imports nothing from the CUDA package at module level
from paper_1510_08642_b200 import mgpu as _mgpu_probe  # noqa: F401  (needs libddqd.so built)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend:
    """CPU stand-in for the library kernels, written from docs/numerics.md s.4 with oracle ops."""

    def __init__(self, W):
        import oracle
        self.o = oracle
        self.W = W
        self.op = oracle.dd_op if W == 2 else oracle.qd_op
        # one OpenMP thread per rank (omp_set_num_threads persists for this thread): several
        # ranks each spinning a team over every core make the oracle ~1000x slower
        oracle.gemm(np.zeros((W, 1, 1)), np.zeros((W, 1, 1)), nthreads=1)

    def empty(self, shape, like):
        return torch.empty(shape, dtype=torch.float64)

    def empty_i64(self, n, like):
        return torch.empty(n, dtype=torch.int64)

    # "peer memory" for the p2p combine: files in /dev/shm mapped by every process
    _count = 0

    def sync(self):
        pass

    def ipc_alloc(self, shape, like):
        OracleBackend._count += 1
        path = f"/dev/shm/ddqd_p2p_{os.getpid()}_{OracleBackend._count}"
        n = int(np.prod(shape))
        t = torch.from_file(path, shared=True, size=n, dtype=torch.float64).view(*shape)
        return t, (path, n), path

    def ipc_open(self, handle, shape, like):
        path, n = handle
        return torch.from_file(path, shared=True, size=n, dtype=torch.float64).view(*shape), None

    def ipc_close(self, c):
        pass

    def ipc_free(self, path):
        os.remove(path)

    # CPU: every backend call completes before it returns, so events are no-ops
    def ipc_event(self, like):
        return None, b""

    def open_event(self, handle, like):
        return None

    def record(self, e):
        pass

    def wait(self, e):
        pass

    def post_add_ptrs(self, algo, children, C, r0, r1):
        """Position rows [r0, r1) of the one-level post-addition, children given as tensors."""
        add = lambda a, b: self._ew("add", a, b)   # noqa: E731
        sub = lambda a, b: self._ew("sub", a, b)   # noqa: E731
        Cv = C if C.dim() == 4 else C.unsqueeze(0)
        hm, hn = children[0].shape[-2], children[0].shape[-1]
        r1 = hm if r1 is None else r1
        rr, cc = Cv.shape[-2], Cv.shape[-1]
        for b in range(Cv.shape[0]):
            p = [np.ascontiguousarray(children[7 * b + c].numpy()[:, r0:r1, :]) for c in range(7)]
            if algo == "strassen":
                q = [add(sub(add(p[0], p[3]), p[4]), p[6]), add(p[2], p[4]), add(p[1], p[3]),
                     add(add(sub(p[0], p[1]), p[2]), p[5])]
            else:
                u2 = add(p[0], p[5]); u3 = add(u2, p[6]); u4 = add(u2, p[4])
                q = [add(p[0], p[1]), add(u4, p[2]), sub(u3, p[3]), add(u3, p[4])]
            for quad, (dr, dc) in enumerate(((0, 0), (0, hn), (hm, 0), (hm, hn))):
                ra, rb = r0 + dr, min(r1 + dr, rr)
                ca, cb = dc, min(hn + dc, cc)
                if rb > ra and cb > ca:
                    Cv[b, :, ra:rb, ca:cb] = torch.from_numpy(np.ascontiguousarray(q[quad][:, : rb - ra, : cb - ca]))
        return None

    def lu_panel(self, A, ipiv, p, kb, pivot):
        return self.o.lu_panel(A.numpy(), ipiv.numpy(), p, kb, pivot)

    def lu_trsv(self, A, ipiv, b):
        return torch.from_numpy(self.o.lu_solve(A.numpy(), ipiv.numpy(), b.numpy()))

    def _ew(self, name, x, y):
        W = self.W
        shp = x.shape
        return self.op(name, x.reshape(W, -1), y.reshape(W, -1)).reshape(shp)

    def _quads(self, X, hr, hc):
        W, r, c = X.shape
        P = np.zeros((W, 2 * hr, 2 * hc))
        P[:, :r, :c] = X
        return P[:, :hr, :hc], P[:, :hr, hc:], P[:, hr:, :hc], P[:, hr:, hc:]

    def pre_add(self, algo, side, X, Y, keep=None):   # (forms every child; `keep` only saves work)
        Xn = X.numpy().reshape((-1,) + tuple(X.shape[-3:]))
        hr, hc = Y.shape[-2], Y.shape[-1]
        add = lambda a, b: self._ew("add", a, b)   # noqa: E731
        sub = lambda a, b: self._ew("sub", a, b)   # noqa: E731
        for b in range(Xn.shape[0]):
            x11, x12, x21, x22 = self._quads(Xn[b], hr, hc)
            if algo == "strassen" and side == 0:
                o = [add(x11, x22), add(x21, x22), x11, x22, add(x11, x12), sub(x21, x11), sub(x12, x22)]
            elif algo == "strassen":
                o = [add(x11, x22), x11, sub(x12, x22), sub(x21, x11), x22, add(x11, x12), add(x21, x22)]
            elif side == 0:
                s1 = add(x21, x22); s2 = sub(s1, x11); s3 = sub(x11, x21); s4 = sub(x12, s2)
                o = [x11, x12, s4, x22, s1, s2, s3]
            else:
                t1 = sub(x12, x11); t2 = sub(x22, t1); t3 = sub(x22, x12); t4 = sub(t2, x21)
                o = [x11, x21, x22, t4, t1, t2, t3]
            for c in range(7):
                Y[7 * b + c] = torch.from_numpy(np.ascontiguousarray(o[c]))

    def post_add(self, algo, M, C, beta=0):
        add = lambda a, b: self._ew("add", a, b)   # noqa: E731
        sub = lambda a, b: self._ew("sub", a, b)   # noqa: E731
        Cv = C if C.dim() == 4 else C.unsqueeze(0)
        hm, hn = M.shape[-2], M.shape[-1]
        for b in range(Cv.shape[0]):
            p = [M[7 * b + c].numpy() for c in range(7)]
            if algo == "strassen":
                c11 = add(sub(add(p[0], p[3]), p[4]), p[6]); c12 = add(p[2], p[4])
                c21 = add(p[1], p[3]); c22 = add(add(sub(p[0], p[1]), p[2]), p[5])
            else:
                u2 = add(p[0], p[5]); u3 = add(u2, p[6]); u4 = add(u2, p[4])
                c11 = add(p[0], p[1]); c12 = add(u4, p[2]); c21 = sub(u3, p[3]); c22 = add(u3, p[4])
            full = np.zeros((self.W, 2 * hm, 2 * hn))
            full[:, :hm, :hn] = c11; full[:, :hm, hn:] = c12; full[:, hm:, :hn] = c21; full[:, hm:, hn:] = c22
            r, c = Cv.shape[-2], Cv.shape[-1]
            t = np.ascontiguousarray(full[:, :r, :c])
            if beta:
                t = sub(np.ascontiguousarray(Cv[b].numpy()), t)
            Cv[b] = torch.from_numpy(t)

    def gemm_batched(self, A, B, C, algo, T):
        for b in range(A.shape[0]):
            C[b] = torch.from_numpy(self.o.gemm(A[b].numpy(), B[b].numpy(), algo, threshold=T))

    def index(self, values, like):
        return torch.tensor(values, dtype=torch.int64)

    def band_copy(self, direction, full, compact, rmap, cmap):
        W, r, c = compact.shape
        ri = rmap if rmap is not None else torch.arange(r)
        ci = cmap if cmap is not None else torch.arange(c)
        if direction == "pack":
            compact[:] = full[:, ri[:, None], ci[None, :]]
        else:
            full[:, ri[:, None], ci[None, :]] = compact

    def gemm_depth(self, A, B, C, algo, depth, beta=0):
        t = self.o.gemm(np.ascontiguousarray(A.numpy()), np.ascontiguousarray(B.numpy()), algo, threshold=1,
                        depth=None if algo == "block" else depth)
        if beta:
            t = self._ew("sub", np.ascontiguousarray(C.numpy()), t)
        C[:] = torch.from_numpy(t)

    def gemm_rows(self, A, B, r0, r1, out, algo, T, beta=0):
        t = self.o.gemm(np.ascontiguousarray(A[:, r0:r1, :].numpy()), B.numpy(), algo, threshold=T)
        if beta:
            t = self._ew("sub", np.ascontiguousarray(out[:, : r1 - r0, :].numpy()), t)
        out[:, : r1 - r0, :] = torch.from_numpy(t)


def _worker(rank, world, port, cfg, q, chunk=None, combine="nccl"):
    # one OpenMP thread per rank: several ranks spinning on all cores crawl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08642_b200.mgpu import DistributedGemm
        W, algo, T, m, l, n, k = cfg
        A = torch.from_numpy(gen.matrix(W, m, l, 21, 0)) if rank == 0 else torch.zeros((W, m, l), dtype=torch.float64)
        B = torch.from_numpy(gen.matrix(W, l, n, 21, 1)) if rank == 0 else torch.zeros((W, l, n), dtype=torch.float64)
        C = torch.zeros((W, m, n), dtype=torch.float64)
        dg = DistributedGemm(W, algo, T, m, l, n, dist, k=k, backend=OracleBackend(W), chunk=chunk,
                             combine=combine)
        dg(A, B, C)
        dg(A, B, C)    # buffers are reused across steps
        if rank == 0:
            q.put((dg.k, C.numpy().copy()))
        if combine == "p2p":
            dg.release()
    finally:
        dist.destroy_process_group()


def _run(cfg, world=2, chunk=None, combine="nccl"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q, chunk, combine)) for r in range(world)]
    for p in procs:
        p.start()
    k, C = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return k, C


@pytest.mark.parametrize("cfg", [
    (2, "winograd", 4, 37, 29, 33, None),     # odd shapes, k chosen by the balancer (k = 2)
    (2, "strassen", 5, 40, 41, 42, 1),
    (4, "winograd", 3, 19, 23, 17, 2),       # QD
    (2, "block", 8, 31, 20, 25, None),       # C row-slab tiling
])
def test_distributed_matches_single_process(orc, cfg):
    W, algo, T, m, l, n, _ = cfg
    k, C = _run(cfg)
    ref = orc.gemm(gen.matrix(W, m, l, 21, 0), gen.matrix(W, l, n, 21, 1), algo, threshold=T)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))
    if algo != "block":
        assert k >= 1


def test_three_ranks_uneven_chunks(orc):
    """world size 3: 49 depth-2 products split 17/16/16, sent in chunks of 5 (uneven rounds),
    pre-additions pruned per rank; still bit-identical to the single-process recursion."""
    cfg = (2, "winograd", 3, 30, 27, 29, 2)
    k, C = _run(cfg, world=3, chunk=5)
    ref = orc.gemm(gen.matrix(2, 30, 27, 21, 0), gen.matrix(2, 27, 29, 21, 1), "winograd", threshold=3)
    assert k == 2 and np.array_equal(C.view(np.int64), ref.view(np.int64))


def test_balancer():
    from paper_1510_08642_b200.mgpu import balanced_slices, choose_depth
    assert balanced_slices(49, 8)[0] == (0, 7) and balanced_slices(49, 8)[-1] == (43, 49)
    assert choose_depth(5, 8) == 3 and choose_depth(5, 4) == 2 and choose_depth(5, 2) == 2
    assert choose_depth(5, 7) == 1 and choose_depth(0, 8) == 0



# ---- distributed LU (row f4) ------------------------------------------------------------------
def _lu_worker(rank, world, port, cfg, q):
    # one OpenMP thread per rank: several ranks spinning on all cores crawl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1510_08642_b200.mgpu import DistributedLU
        W, n, K, algo, T, pivot, seed = cfg
        if rank == 0:
            A0 = _lu_input(W, n, seed)
            A = torch.from_numpy(A0.copy())
            b = torch.from_numpy(oracle.gemm(A0, _ones(W, n), "block")[:, :, 0].copy())
        else:
            A = torch.zeros((W, n, n), dtype=torch.float64)
            b = None
        x, ipiv, info = DistributedLU(W, n, K, algo, T, dist, pivot=pivot, backend=OracleBackend(W))(A, b)
        if rank == 0:
            q.put((x.numpy().copy(), A.numpy().copy(), ipiv.numpy().copy(), info))
    finally:
        dist.destroy_process_group()


def _ones(W, n):
    o = np.zeros((W, n, 1))
    o[0] = 1.0
    return o


def _lu_input(W, n, seed):
    if W == 2:
        return gen.lu_matrix(n, seed)
    return gen.matrix(4, n, n, seed, 0)   # QD, non-dominant: exercises the interchanges


def _run_lu(cfg, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lu_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("cfg,world", [
    ((2, 70, 16, "strassen", 8, True, 5), 2),    # Strassen updates (depth 1-2), ragged last panel
    ((2, 61, 20, "winograd", 4, True, 6), 3),    # three ranks, deeper Winograd updates
    ((2, 50, 12, "block", 8, True, 7), 2),       # Block update: C row slabs with beta = 1
    ((4, 40, 16, "winograd", 4, True, 8), 2),    # QD, pivoting with interchanges
    ((2, 45, 16, "strassen", 4, False, 9), 2),   # the paper's pivot-free LU
])
def test_distributed_lu_matches_single_process(orc, cfg, world):
    """DistributedLU (row f4): the trailing updates run over the ranks; factors, pivots, info
    and the solution are bitwise those of the single-process oracle LU."""
    W, n, K, algo, T, pivot, seed = cfg
    x, LU, ipiv, info = _run_lu(cfg, world)
    A0 = _lu_input(W, n, seed)
    b = orc.gemm(A0, _ones(W, n), "block")[:, :, 0].copy()
    xr, LUr, pr, ir = orc.solve(A0, b, panel=K, algo=algo, threshold=T, pivot=pivot)
    assert info == ir
    assert np.array_equal(ipiv, pr)
    assert np.array_equal(LU.view(np.int64), LUr.view(np.int64))
    assert np.array_equal(x.view(np.int64), xr.view(np.int64))



@pytest.mark.parametrize("cfg,world", [
    ((2, "winograd", 4, 37, 29, 33, 1), 2),     # one level over peer memory
    ((2, "strassen", 3, 40, 41, 42, 2), 3),     # two levels: parents split over 3 ranks
    ((4, "winograd", 2, 19, 23, 17, 2), 2),     # QD
])
def test_p2p_combine_matches_single_process(orc, cfg, world):
    """The fused p2p combine: products stay on their ranks, every level's
    post-additions read them through (here: file-backed) shared mappings, split over the
    ranks, and the ranks write their rows of C into rank 0's buffer -- bit-identical to the
    single-process recursion."""
    W, algo, T, m, l, n, _ = cfg
    k, C = _run(cfg, world=world, combine="p2p")
    ref = orc.gemm(gen.matrix(W, m, l, 21, 0), gen.matrix(W, l, n, 21, 1), algo, threshold=T)
    assert k >= 1 and np.array_equal(C.view(np.int64), ref.view(np.int64))



def _auto_worker(rank, world, port, cfg, q):
    # one OpenMP thread per rank: several ranks spinning on all cores crawl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08642_b200.mgpu import AutoDistributedGemm, DistributedGemm
        W, algo, T, m, l, n = cfg
        A = torch.from_numpy(gen.matrix(W, m, l, 23, 0)) if rank == 0 else torch.zeros((W, m, l), dtype=torch.float64)
        B = torch.from_numpy(gen.matrix(W, l, n, 23, 1)) if rank == 0 else torch.zeros((W, l, n), dtype=torch.float64)
        C = torch.zeros((W, m, n), dtype=torch.float64)
        C2 = torch.zeros((W, m, n), dtype=torch.float64)
        C3 = torch.zeros((W, m, n), dtype=torch.float64)
        DistributedGemm(W, algo, T, m, l, n, dist, k=0, backend=OracleBackend(W))(A, B, C2)   # C tiles
        ag = AutoDistributedGemm(W, algo, T, m, l, n, dist, backend=OracleBackend(W))          # bitwise ones
        ag(A, B, C)
        choice1, t1 = ag.choice, dict(ag.timings)
        ag(A, B, C)
        ag.release()
        # every schedule incl. the C row slabs
        ag3 = AutoDistributedGemm(W, algo, T, m, l, n, dist, backend=OracleBackend(W),
                                  candidates=("ctiles", "bands", "products"))
        ag3(A, B, C3)
        # beta = 1 (C := C - A B): C restored before every trial, exactly one update in the end
        C4 = torch.from_numpy(gen.matrix(W, m, n, 23, 2)) if rank == 0 else None
        ag4 = AutoDistributedGemm(W, algo, T, m, l, n, dist, backend=OracleBackend(W), beta=1)
        ag4(A, B, C4)
        if rank == 0:
            q.put((choice1, ag.choice, sorted(t1), C.numpy().copy(), C2.numpy().copy(), ag3.choice,
                   C3.numpy().copy(), C4.numpy().copy(), sorted(ag4.timings)))
    finally:
        dist.destroy_process_group()


def test_c_tiles_and_auto_schedule(orc):
    """BJ:5 (4): the C-tile schedule (each rank recurses on its row slab of C) is bit-exact
    against the oracle run slab by slab; AutoDistributedGemm times its candidates, makes the same
    choice on every rank and returns the chosen schedule's exact result -- by default only the
    schedules bit-identical to one GPU compete, so the bits never depend on the timing; with
    beta = 1 (the LU update) C is restored before every trial and updated exactly once."""
    from paper_1510_08642_b200.mgpu import balanced_slices
    cfg = (2, "winograd", 4, 37, 29, 33)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_auto_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    choice1, choice2, names, C, C2, choice3, C3, C4, names4 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W, algo, T, m, l, n = cfg
    A, B = gen.matrix(W, m, l, 23, 0), gen.matrix(W, l, n, 23, 1)
    whole = orc.gemm(A, B, algo, threshold=T)
    tiles = np.concatenate([orc.gemm(np.ascontiguousarray(A[:, a:b]), B, algo, threshold=T)
                            for a, b in balanced_slices(m, 2)], axis=1)
    assert np.array_equal(C2.view(np.int64), tiles.view(np.int64))
    assert names == ["bands", "products", "products_p2p", "products_rows"] and choice1 == choice2 and choice1 in names
    assert np.array_equal(C.view(np.int64), whole.view(np.int64))
    assert choice3 in ("ctiles", "bands", "products")
    assert np.array_equal(C3.view(np.int64), (tiles if choice3 == "ctiles" else whole).view(np.int64))
    assert names4 == ["bands", "products", "products_rows"]
    ref4 = orc.dd_op("sub", gen.matrix(W, m, n, 23, 2).reshape(W, -1), whole.reshape(W, -1)).reshape(W, m, n)
    assert np.array_equal(C4.view(np.int64), ref4.view(np.int64))
    assert not np.array_equal(tiles, whole)   # the two schedules round differently
class _NoPeerBackend(OracleBackend):
    """Rank `bad` cannot map peer memory (a box without CUDA IPC between its GPUs)."""

    def __init__(self, W, bad):
        super().__init__(W)
        self.bad = bad

    def ipc_open(self, handle, shape, like):
        if dist.get_rank() == self.bad:
            raise RuntimeError("cudaIpcOpenMemHandle: peer access unsupported")
        return super().ipc_open(handle, shape, like)


def _unavail_worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08642_b200.mgpu import AutoDistributedGemm, DistributedGemm, ScheduleUnavailable
        W, algo, T, m, l, n = cfg
        A = torch.from_numpy(gen.matrix(W, m, l, 29, 0)) if rank == 0 else torch.zeros((W, m, l), dtype=torch.float64)
        B = torch.from_numpy(gen.matrix(W, l, n, 29, 1)) if rank == 0 else torch.zeros((W, l, n), dtype=torch.float64)
        C = torch.zeros((W, m, n), dtype=torch.float64)
        raised = None
        try:   # the p2p schedule alone: every rank raises, none is left in a collective
            DistributedGemm(W, algo, T, m, l, n, dist, backend=_NoPeerBackend(W, 1), combine="p2p")(A, B, C)
        except ScheduleUnavailable as e:
            raised = str(e)
        ag = AutoDistributedGemm(W, algo, T, m, l, n, dist, backend=_NoPeerBackend(W, 1))
        ag(A, B, C)
        dist.barrier()
        q.put((rank, raised, ag.choice, sorted(ag.unavailable), C.numpy().copy() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_p2p_unavailable_is_dropped_on_every_rank(orc):
    """A rank that cannot open its peers' memory makes the p2p combine raise ScheduleUnavailable
    on EVERY rank at the same point (the failure is agreed on before anyone leaves the setup),
    and the automatic choice (BJ:5 (4)) drops it and returns another bit-identical schedule's
    result -- the driver's multi-GPU run must not hang or crash on a box without CUDA IPC."""
    cfg = (2, "strassen", 4, 21, 19, 23)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unavail_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W, algo, T, m, l, n = cfg
    whole = orc.gemm(gen.matrix(W, m, l, 29, 0), gen.matrix(W, l, n, 29, 1), algo, threshold=T)
    for rank, raised, choice, unavailable, _ in res:
        assert raised and "rank 1" in raised and "peer access unsupported" in raised
        assert unavailable == ["products_p2p"] and choice in ("bands", "products", "products_rows")
    assert res[0][2] == res[1][2]
    assert np.array_equal(res[0][4].view(np.int64), whole.view(np.int64))


# ---- band schedule (BandGemm: each rank one tile of C, the whole problem's tree) ---------------
def _band_worker(rank, world, port, cfg, q):
    # one OpenMP thread per rank: several ranks spinning on all cores crawl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08642_b200.mgpu import BandGemm
        W, algo, T, m, l, n, beta = cfg
        A = torch.from_numpy(gen.matrix(W, m, l, 31, 0)) if rank == 0 else torch.zeros((W, m, l), dtype=torch.float64)
        B = torch.from_numpy(gen.matrix(W, l, n, 31, 1)) if rank == 0 else torch.zeros((W, l, n), dtype=torch.float64)
        C = torch.from_numpy(gen.matrix(W, m, n, 31, 2)) if rank == 0 else None
        bg = BandGemm(W, algo, T, m, l, n, dist, backend=OracleBackend(W), beta=beta)
        C0 = C.clone() if rank == 0 else None
        bg(A, B, C)
        if rank == 0 and beta:
            C.copy_(C0)
        bg(A, B, C)    # buffers are reused across steps
        if rank == 0:
            q.put(((bg.gr, bg.gc, bg.d), C.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [
    ((2, "winograd", 4, 37, 29, 33, 0), 2),     # 1 x 2 grid, odd shapes (virtual padding), d = 3
    ((2, "strassen", 3, 40, 41, 42, 0), 3),     # 1 x 3 grid
    ((2, "winograd", 3, 45, 30, 38, 0), 4),     # 2 x 2 grid, d = 4
    ((4, "winograd", 2, 19, 23, 17, 0), 2),     # QD
    ((2, "strassen", 4, 36, 16, 36, 1), 2),     # C := C - A B (the LU update form)
    ((2, "block", 8, 31, 20, 25, 0), 4),        # Block: plain 2 x 2 C tiles
])
def test_band_schedule_matches_single_process(orc, cfg, world):
    """BandGemm: every rank multiplies its packed (row band x column band) operands with the
    whole problem's depth (DDQD_DEPTH); rank 0 unpacks the tiles -- bit-identical to the
    single-process recursion for every grid."""
    W, algo, T, m, l, n, beta = cfg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    (gr, gc, d), C = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B = gen.matrix(W, m, l, 31, 0), gen.matrix(W, l, n, 31, 1)
    ref = orc.gemm(A, B, algo, threshold=T)
    if beta:
        ref = (orc.dd_op if W == 2 else orc.qd_op)("sub", gen.matrix(W, m, n, 31, 2).reshape(W, -1),
                                                   ref.reshape(W, -1)).reshape(W, m, n)
    assert gr * gc == world and (algo == "block" or d >= 1)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("cfg,world", [
    ((2, "winograd", 4, 37, 29, 33, None), 2),     # k chosen by the balancer (k = 2)
    ((2, "strassen", 3, 40, 41, 42, 2), 3),        # three ranks, odd band heights
    ((4, "winograd", 2, 19, 23, 17, 2), 2),        # QD
    ((2, "winograd", 3, 30, 27, 29, 2), 4),        # four ranks
])
def test_rows_combine_matches_single_process(orc, cfg, world):
    """combine='rows': products exchanged by row bands, every rank combines its band of C
    through the k levels, rank 0 gathers -- bit-identical to the single-process recursion."""
    W, algo, T, m, l, n, _ = cfg
    k, C = _run(cfg, world=world, combine="rows")
    ref = orc.gemm(gen.matrix(W, m, l, 21, 0), gen.matrix(W, l, n, 21, 1), algo, threshold=T)
    assert k >= 1 and np.array_equal(C.view(np.int64), ref.view(np.int64))
