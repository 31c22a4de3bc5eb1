"""Multi-GPU schedule for one large DD/QD GEMM (north_star subsystem (4)).

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing:

  Strassen / Winograd (depth d >= 1): "depth-k product distribution"
    1. broadcast A and B from rank 0 (NCCL over NVLink);
    2. every rank forms the top-k levels of pre-additions locally (fused library kernels),
       giving the 7^k operand pairs of depth k (the paper's 7 "sections" of P:33, k levels
       deep);
       -- pruned to the ancestors of the rank's own products;
    3. rank r multiplies a contiguous, balanced slice of those 7^k products with batched
       library calls (the recursion continues below depth k on the GPU), in ~6 chunks;
    4. each finished chunk is sent to rank 0 (NCCL point-to-point on its own stream) while
       the next chunk computes; rank 0 receives straight into its level-k product buffer and
       runs the top-k post-additions into C. DD/QD sums cannot use NCCL reductions (adding hi
       and lo planes separately is not DD addition), so the combine is the library's post-add.
  Block (or d = 0): C row-slab tiling -- rank r computes rows [r0, r1) of C from the same
    A row slab and all of B, and the slabs are gathered to rank 0.

Both schedules are numerically identical to the single-GPU call (same tree, same order),
so results are bit-identical to the oracle for any world size. With beta = 1 the result is
subtracted from C (C := C - A B), the form of the LU's Schur update.

  Bands (BandGemm): C is partitioned into a G_r x G_c grid of tiles, each a row band x column
    band of the depth-d LEAVES lifted to level 0, so every rank runs the whole problem's
    recursion tree restricted to its tile (DDQD_DEPTH) -- no products cross the network and
    nothing is combined on rank 0; bit-identical to one GPU.

AutoDistributedGemm (BJ:5 (4) "the top-level 7 products are distributed over GPUs, or C is
partitioned into tiles that each GPU recurses on, choosing whichever measures faster"): times
the candidate schedules once (max over ranks) and keeps the fastest; by default only the
bit-identical ones compete. The C-row-slab schedule (k = 0) recurses on each slab as its own
Strassen/Winograd tree, so it rounds differently from the one-GPU call; it is bit-exact against
the oracle run slab by slab and competes only when asked for.

DistributedLU: the blocked LU with its trailing update
A22 := A22 - L21 U12 run by DistributedGemm over all ranks; rank 0 keeps the matrix
and does the sequential panel steps (4096 dependent pivot steps at c4 do not shard) and the
solve. Every panel's update is the same recursion tree as on one GPU, so the factors and the
solution are bit-identical to the single-GPU LU (and the oracle) for any world size.

The compute steps go through a `backend` (default: the CUDA library); tests substitute a
CPU backend built from the oracle to check this host logic with gloo on CPU.
"""
from __future__ import annotations

import math


class ScheduleUnavailable(RuntimeError):
    """A schedule cannot run on this machine; raised on every rank at the same point."""


def rec_shapes(m, l, n, T):
    shapes = [(m, l, n)]
    while min(m, l, n) > T:
        m, l, n = (m + 1) // 2, (l + 1) // 2, (n + 1) // 2
        shapes.append((m, l, n))
    return shapes


def band_index_map(dims, a, b):
    """Level-0 indices of the band [a, b) of the depth-d index range, ascending.

    dims = [n_0, n_1, ..., n_d] with n_{j+1} = ceil(n_j / 2) (one dimension of the recursion's
    level shapes). Index r of a level-(j+1) child is index r of the parent's top/left quadrant
    and index n_{j+1} + r of its bottom/right quadrant (absent -- the virtual padding -- when
    that is >= n_j). Going up from [a, b) at level d gives the set the band touches at every
    level; taken in this order (top part, then bottom part) the compact sizes satisfy
    H_{j+1} = ceil(H_j / 2), so the compact band recursed with the same depth reproduces, entry
    for entry, the recursion of the whole problem (reading R21)."""
    idx = list(range(a, b))
    for j in range(len(dims) - 2, -1, -1):
        h = dims[j + 1]
        idx = idx + [h + r for r in idx if h + r < dims[j]]
    return idx


def band_grid(world: int):
    """(G_r, G_c) with G_r * G_c = world and G_r <= G_c as close as possible: rows of C split
    G_r ways, columns G_c ways (8 GPUs: 2 x 4)."""
    gr = int(math.isqrt(world))
    while world % gr:
        gr -= 1
    return gr, world // gr


def balanced_slices(count: int, world: int):
    """Contiguous LPT split of `count` equal-cost units over `world` ranks."""
    base, extra = divmod(count, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def choose_depth(d: int, world: int) -> int:
    """Smallest k <= d whose 7^k products balance within 10% over `world` ranks (k >= 1)."""
    if world <= 1 or d == 0:
        return 0
    for k in range(1, d + 1):
        units = 7 ** k
        if math.ceil(units / world) * world <= 1.10 * units:
            return k
    return d


class CudaBackend:
    """Library calls on torch CUDA tensors (all kernels are libddqd.so's)."""

    def __init__(self):
        import paper_1510_08642_b200 as ddqd
        self.ddqd = ddqd

    def empty(self, shape, like):
        import torch
        return torch.empty(shape, dtype=torch.float64, device=like.device)

    def empty_i64(self, n, like):
        import torch
        return torch.empty(n, dtype=torch.int64, device=like.device)

    def pre_add(self, algo, side, X, Y, keep=None):
        self.ddqd.pre_add(algo, side, X, Y, keep=keep)

    def post_add(self, algo, M, C, beta=0):
        self.ddqd.post_add(algo, M, C, beta)

    def sync(self):
        import torch
        torch.cuda.synchronize()

    def ipc_alloc(self, shape, like):
        t, ptr = self.ddqd.ipc_alloc(shape, like.device)
        return t, self.ddqd.ipc_handle(ptr), ptr

    def ipc_open(self, handle, shape, like):
        return self.ddqd.ipc_open(handle, shape, like.device)

    def ipc_close(self, ptr):
        self.ddqd.ipc_close(ptr)

    def ipc_free(self, ptr):
        self.ddqd.ipc_free(ptr)

    def post_add_ptrs(self, algo, children, C, r0, r1):
        return self.ddqd.post_add_ptrs(algo, children, C, r0, r1)

    # interprocess events: stream-ordered dependencies on other ranks' kernels (no host sync)
    def ipc_event(self, like):
        import torch
        with torch.cuda.device(like.device):
            e = torch.cuda.Event(enable_timing=False, interprocess=True)
            e.record()   # an event needs a record before its handle can be taken
            return e, e.ipc_handle()

    def open_event(self, handle, like):
        import torch
        return torch.cuda.Event.from_ipc_handle(like.device, handle)

    def record(self, e):
        e.record()

    def wait(self, e):
        import torch
        torch.cuda.current_stream().wait_event(e)

    def lu_panel(self, A, ipiv, p, kb, pivot):
        return self.ddqd.lu_panel(A, ipiv, p, kb, pivot)

    def lu_trsv(self, A, ipiv, b):
        return self.ddqd.lu_trsv(A, ipiv, b)

    def gemm_batched(self, A, B, C, algo, T):
        if A.shape[0]:
            self.ddqd.gemm_batched(A, B, C, algo, T)

    def index(self, values, like):
        import torch
        return torch.tensor(values, dtype=torch.int64, device=like.device)

    def band_copy(self, direction, full, compact, rmap, cmap):
        self.ddqd.band_copy(direction, full, compact, rmap, cmap)

    def gemm_depth(self, A, B, C, algo, depth, beta=0):
        """C := (C -) A B with exactly `depth` recursion levels on contiguous [W, r, c] tensors."""
        W, m, l = A.shape
        n = B.shape[2]
        self.ddqd._set_stream(A)
        self.ddqd.gemm_ex(W, algo, 1, m, l, n, 1, A.data_ptr(), l, m * l, 0, B.data_ptr(), n, l * n, 0,
                          C.data_ptr(), n, m * n, 0, beta, depth=depth if algo not in ("block", 0) else None)

    def gemm_rows(self, A, B, r0, r1, out, algo, T, beta=0):
        """out[:, :r1-r0, :] := (out -) A[:, r0:r1, :] B via strided views (no copies)."""
        W, m, l = A.shape
        n = B.shape[2]
        per = out.shape[1]
        self.ddqd._set_stream(A)
        self.ddqd.gemm_ex(W, algo, T, r1 - r0, l, n, 1,
                          A.data_ptr() + 8 * r0 * l, l, m * l, 0,
                          B.data_ptr(), n, l * n, 0,
                          out.data_ptr(), n, per * n, 0, beta)


class DistributedGemm:
    """C := A B (beta = 0) or C := C - A B (beta = 1) across the process group `dist` (rank 0
    holds the operands and C; C may be a strided view with unit-stride rows)."""

    def __init__(self, W, algo, T, m, l, n, dist, device=None, k=None, backend=None, chunk=None, beta=0,
                 combine="nccl", replicated_inputs=False, world=None, rank=0):
        self.W, self.algo, self.T, self.beta = W, algo, T, beta
        # combine = "nccl": products stream to rank 0 over NCCL point-to-point, rank 0 post-adds;
        # "p2p": products stay resident, the post-adds read peers' buffers through CUDA IPC
        # mappings (fused gather + combine kernels, levels split over the ranks, each rank writes
        # its rows of C straight into rank 0's C buffer). beta = 1 needs combine = "nccl".
        # "rows": products exchanged by row bands (all-to-all), every rank combines its band of C
        # through all k levels, rank 0 gathers the bands -- no combine tail on rank 0
        if combine not in ("nccl", "p2p", "rows"):
            raise ValueError("combine must be 'nccl', 'p2p' or 'rows'")
        if combine == "p2p" and beta:
            raise ValueError("the p2p combine computes C := A B (beta = 0)")
        self.combine = combine
        self.replicated_inputs = replicated_inputs   # every rank already holds A and B
        self.m, self.l, self.n = m, l, n
        self.dist = dist             # None: compute_share() only, as `rank` of `world` on one device
        self.rank = dist.get_rank() if dist is not None else int(rank)
        self.world = dist.get_world_size() if dist is not None else int(world)
        self.backend = backend or CudaBackend()
        self.shapes = rec_shapes(m, l, n, T) if algo not in ("block", 0) else [(m, l, n)]
        d = len(self.shapes) - 1
        self.k = min(d, k) if k is not None else choose_depth(d, self.world)
        if self.k > 0:
            units = 7 ** self.k
            self.slices = balanced_slices(units, self.world)
            self.per = max(hi - lo for lo, hi in self.slices)
            # products per send: ~6 chunks per rank so communication overlaps compute
            self.chunk = chunk or max(1, -(-self.per // 6))
        else:
            self.slices = balanced_slices(m, self.world)          # C row slabs
            self.per = max(hi - lo for lo, hi in self.slices)
        self._bufs = None
        self._p2p = None
        if self.k > 0:
            # p2p combine: parents of level j (1 <= j < k) split over the ranks; level 0 (C)
            # split by position rows of the level-1 products
            self.pslices = {j: balanced_slices(7 ** j, self.world) for j in range(1, self.k)}
            self.rslices = balanced_slices(self.shapes[1][0], self.world)

    # buffers are allocated lazily on the operands' device
    def _alloc(self, like):
        if self._bufs is not None:
            return self._bufs
        W, bk = self.W, self.backend
        bufs = {"A": [], "B": [], "M": []}
        for j in range(1, self.k + 1):
            mj, lj, nj = self.shapes[j]
            bufs["A"].append(bk.empty((7 ** j, W, mj, lj), like))
            bufs["B"].append(bk.empty((7 ** j, W, lj, nj), like))
            if self.rank == 0:
                bufs["M"].append(bk.empty((7 ** j, W, mj, nj), like))
        if self.k > 0:
            mk, _, nk = self.shapes[self.k]
            if self.rank != 0:
                bufs["local"] = bk.empty((self.per, W, mk, nk), like)
        else:
            bufs["local"] = bk.empty((W, self.per, self.n), like)
            if self.rank == 0:
                bufs["gather"] = [bk.empty((W, self.per, self.n), like) for _ in range(self.world)]
                if self.beta:
                    bufs["scatter"] = [bk.empty((W, self.per, self.n), like) for _ in range(self.world)]
        self._bufs = bufs
        return bufs

    def _pruned_pre_adds(self, A, B, bufs):
        """The top-k pre-additions, breadth-first, pruned to the ancestors of this rank's products:
        at level j only the parents above them, and of their children only those that are
        ancestors (or the products) themselves. Returns the level-k operand buffers."""
        bk, k = self.backend, self.k
        X, Y = A, B
        for j in range(k):
            a, b = self._ancestor_range(j)
            if b > a:
                Xs = X if j == 0 else X[a:b]
                Ys = Y if j == 0 else Y[a:b]
                c0, c1 = self._ancestor_range(j + 1) if j + 1 < k else self.slices[self.rank]
                keep = (c0 - 7 * a, c1 - 7 * a)
                bk.pre_add(self.algo, 0, Xs, bufs["A"][j][7 * a:7 * b], keep=keep)
                bk.pre_add(self.algo, 1, Ys, bufs["B"][j][7 * a:7 * b], keep=keep)
            X, Y = bufs["A"][j], bufs["B"][j]
        return X, Y

    def _ancestor_range(self, j):
        """Parents at level j (0 <= j < k) whose subtrees contain this rank's products."""
        lo, hi = self.slices[self.rank]
        if hi <= lo:
            return 0, 0
        span = 7 ** (self.k - j)
        return lo // span, (hi - 1) // span + 1

    def __call__(self, A, B, C):
        dist, W = self.dist, self.W
        if not self.replicated_inputs:
            dist.broadcast(A, 0)
            dist.broadcast(B, 0)
        if self.k > 0 and self.combine == "p2p":
            return self._p2p_call(A, B, C)
        if self.k > 0 and self.combine == "rows":
            return self._rows_call(A, B, C)
        bufs = self._alloc(A)
        if self.k == 0:
            return self._row_slabs(A, B, C, bufs)
        bk = self.backend
        # top-k pre-additions, breadth-first, pruned to the ancestors of this rank's products
        X, Y = self._pruned_pre_adds(A, B, bufs)
        lo, hi = self.slices[self.rank]
        # this rank's products, in chunks; each finished chunk streams to rank 0 while the next
        # one computes (point-to-point sends on the NCCL stream overlap the library's stream)
        if self.rank == 0:
            Mk = bufs["M"][self.k - 1]
            # receives are posted round by round (chunk c of every peer in one NCCL group), so
            # the transfers of all peers proceed together as their chunks finish
            chunks = {r: [(c0, min(self.slices[r][1], c0 + self.chunk))
                          for c0 in range(self.slices[r][0], self.slices[r][1], self.chunk)]
                      for r in range(1, self.world)}
            reqs = []
            for c in range(max((len(v) for v in chunks.values()), default=0)):
                ops = [dist.P2POp(dist.irecv, Mk[v[c][0]:v[c][1]], r)
                       for r, v in chunks.items() if c < len(v)]
                reqs += dist.batch_isend_irecv(ops)
            for c0 in range(lo, hi, self.chunk):
                c1 = min(hi, c0 + self.chunk)
                bk.gemm_batched(X[c0:c1], Y[c0:c1], Mk[c0:c1], self.algo, self.T)
            for q in reqs:
                q.wait()
            for j in range(self.k - 1, -1, -1):
                target = C if j == 0 else bufs["M"][j - 1]
                bk.post_add(self.algo, bufs["M"][j], target, self.beta if j == 0 else 0)
        else:
            local = bufs["local"]
            sends = []
            for c0 in range(lo, hi, self.chunk):
                c1 = min(hi, c0 + self.chunk)
                part = local[c0 - lo:c1 - lo]
                bk.gemm_batched(X[c0:c1], Y[c0:c1], part, self.algo, self.T)
                sends += dist.batch_isend_irecv([dist.P2POp(dist.isend, part, 0)])
            for q in sends:
                q.wait()
        return C

    def compute_share(self, A, B):
        """This rank's compute of the product schedule on the current device, no communication:
        the pruned top-k pre-additions and its slice of the depth-k products, then (combine =
        'rows') the k post-addition levels on its row band (over whatever the band buffer holds:
        timing only). For the one-GPU model of the multi-GPU step (bench.py)."""
        bk, k = self.backend, self.k
        bufs = self._alloc_operands(A)
        X, Y = self._pruned_pre_adds(A, B, bufs)
        lo, hi = self.slices[self.rank]
        st = self._rows_setup(A)
        for c0 in range(lo, hi, self.chunk):
            c1 = min(hi, c0 + self.chunk)
            bk.gemm_batched(X[c0:c1], Y[c0:c1], st["local"][c0 - lo:c1 - lo], self.algo, self.T)
        if self.combine == "rows" and st["H"][0]:
            for j in range(k - 1, -1, -1):
                bk.post_add(self.algo, st["lev"][j + 1], st["lev"][j], 0)

    # ---- row-band combine ------------------------------------------------------------------------
    def _rows_setup(self, like):
        if getattr(self, "_rows", None) is not None:
            return self._rows
        W, bk, G = self.W, self.backend, self.world
        mdims = [s[0] for s in self.shapes[: self.k + 1]]
        bands = balanced_slices(mdims[self.k], G)           # level-k product rows per rank
        maps = [band_index_map(mdims, a, b) for a, b in bands]
        # compact heights of this rank's band at every level 0..k
        a, b = bands[self.rank]
        H = [len(band_index_map(mdims[j:], a, b)) for j in range(self.k + 1)]
        lo, hi = self.slices[self.rank]
        mk, _, nk = self.shapes[self.k]
        st = {
            "bands": bands, "H": H,
            "local": bk.empty((max(hi - lo, 1), W, mk, nk), like),          # this rank's products
            "lev": [bk.empty((7 ** j, W, H[j], self.shapes[j][2]), like) for j in range(self.k + 1)],
            "rmap": bk.index(maps[self.rank], like) if H[0] else None,
        }
        if self.rank == 0:
            st["gather"] = [bk.empty((W, len(maps[g]), self.n), like) for g in range(G)]
            st["gmaps"] = [bk.index(maps[g], like) if maps[g] else None for g in range(G)]
        self._rows = st
        return st

    def _rows_call(self, A, B, C):
        """Products by depth-k units (as the NCCL combine), then (1) an all-to-all of product ROW
        BANDS: rank r receives rows [a_r, b_r) of every level-k product (each sender packs its
        products' band rows in product order, so a receive lands contiguously); (2) every rank
        runs the k levels of post-additions on its compact band (the band rows lifted level by
        level as in the band schedule: the same formulas on 1/G of the positions); (3) rank 0
        gathers the compact bands of C and unpacks their rows. Same operations per element as one
        GPU, so the same bits; rank 0 receives (G-1)/G of C instead of (G-1)/G of every product."""
        dist, bk, W, k = self.dist, self.backend, self.W, self.k
        st = self._rows_setup(A)
        bufs = self._alloc_operands(A)
        X, Y = self._pruned_pre_adds(A, B, bufs)
        # (1) products chunk by chunk; each finished chunk's row bands go to their ranks (and the
        # peers' chunks of the same round come in) while the next chunk computes -- the
        # exchanges run on NCCL's stream, ordered after the chunk that produced them
        lev_k = st["lev"][k]
        a_me, b_me = st["bands"][self.rank]
        Mk = st["local"]
        chunks = [[(c0, min(phi, c0 + self.chunk)) for c0 in range(plo, phi, self.chunk)]
                  for plo, phi in self.slices]
        lo = self.slices[self.rank][0]
        reqs, keep = [], []
        for rnd in range(max(len(c) for c in chunks)):
            ops = []
            if rnd < len(chunks[self.rank]):
                c0, c1 = chunks[self.rank][rnd]
                bk.gemm_batched(X[c0:c1], Y[c0:c1], Mk[c0 - lo:c1 - lo], self.algo, self.T)
                for r, (a, b) in enumerate(st["bands"]):
                    if b <= a:
                        continue
                    part = Mk[c0 - lo:c1 - lo, :, a:b, :]
                    if r == self.rank:
                        lev_k[c0:c1].copy_(part)
                    else:
                        packed = part.contiguous()     # [chunk][W][band rows][n_k], product order
                        keep.append(packed)
                        ops.append((dist.isend, packed, r))
            if b_me > a_me:
                for o in range(self.world):
                    if o != self.rank and rnd < len(chunks[o]):
                        pc0, pc1 = chunks[o][rnd]
                        ops.append((dist.irecv, lev_k[pc0:pc1], o))
            if ops:
                reqs += dist.batch_isend_irecv([dist.P2POp(op, t, peer) for op, t, peer in ops])
        for q in reqs:
            q.wait()
        del keep
        # beta = 1: this rank's rows of C arrive first (rank 0 holds C)
        Cb = st["lev"][0][0]
        if self.beta:
            if self.rank == 0:
                sends = []
                for g in range(self.world):
                    if st["gmaps"][g] is None:
                        continue
                    bk.band_copy("pack", C, st["gather"][g], st["gmaps"][g], None)
                    if g == 0:
                        Cb.copy_(st["gather"][0])
                    else:
                        sends.append((dist.isend, st["gather"][g], g))
                _p2p(dist, sends)
            elif st["H"][0]:
                _p2p(dist, [(dist.irecv, Cb, 0)])
        # (2) the k levels of post-additions on the compact band
        if st["H"][0]:
            for j in range(k - 1, -1, -1):
                bk.post_add(self.algo, st["lev"][j + 1], st["lev"][j], self.beta if j == 0 else 0)
        # (3) gather the compact bands of C on rank 0 and unpack their rows
        if self.rank == 0:
            _p2p(dist, [(dist.irecv, st["gather"][g], g) for g in range(1, self.world) if st["gmaps"][g] is not None])
            for g in range(self.world):
                if st["gmaps"][g] is None:
                    continue
                bk.band_copy("unpack", C, Cb if g == 0 else st["gather"][g], st["gmaps"][g], None)
        elif st["H"][0]:
            _p2p(dist, [(dist.isend, Cb, 0)])
        return C

    # ---- p2p combine ----------------------------------------------------------------------------
    def _owner(self, level, p):
        """(rank, offset) holding product/parent p of `level` (k: products; 1..k-1: parents)."""
        sl = self.slices if level == self.k else self.pslices[level]
        for r, (lo, hi) in enumerate(sl):
            if lo <= p < hi:
                return r, p - lo
        raise IndexError(p)

    def _p2p_setup(self, like):
        if self._p2p is not None:
            return self._p2p
        W, bk, dist = self.W, self.backend, self.dist
        local, handles, frees = {}, {}, []
        # Every local failure (allocation, exporting or opening a peer's handle) is agreed on by
        # all ranks before anyone leaves the setup, so a machine without CUDA IPC between its
        # GPUs makes every rank raise ScheduleUnavailable at the same point (and the automatic
        # choice drops the schedule) instead of leaving the other ranks waiting in a collective.
        err = None
        events = []
        try:
            # one interprocess event per level (k: the products, k-1 .. 0: the combine levels)
            events = [bk.ipc_event(like) for _ in range(self.k + 1)]
            handles["events"] = [h for _, h in events]
            for level in range(1, self.k + 1):
                mj, _, nj = self.shapes[level]
                sl = self.slices if level == self.k else self.pslices[level]
                cnt = max(1, max(hi - lo for lo, hi in sl))
                t, h, f = bk.ipc_alloc((cnt, W, mj, nj), like)
                local[level], handles[level] = t, h
                frees.append(f)
            if self.rank == 0:
                t, h, f = bk.ipc_alloc((W, self.m, self.n), like)
                local["C"], handles["C"] = t, h
                frees.append(f)
        except Exception as e:   # noqa: BLE001  (reported collectively below)
            err = f"rank {self.rank}: {type(e).__name__}: {e}"
        handles["error"] = err
        allh = [None] * self.world
        dist.all_gather_object(allh, handles)
        errs = [h["error"] for h in allh if h.get("error")]
        views, closes, ev = {}, [], None
        if not errs:
            try:
                for level in range(1, self.k + 1):
                    mj, _, nj = self.shapes[level]
                    sl = self.slices if level == self.k else self.pslices[level]
                    for r in range(self.world):
                        if r == self.rank:
                            views[(level, r)] = local[level]
                        else:
                            cnt = max(1, max(hi - lo for lo, hi in sl))
                            v, c = bk.ipc_open(allh[r][level], (cnt, W, mj, nj), like)
                            views[(level, r)] = v
                            closes.append(c)
                if self.rank == 0:
                    views["C"] = local["C"]
                else:
                    v, c = bk.ipc_open(allh[0]["C"], (W, self.m, self.n), like)
                    views["C"] = v
                    closes.append(c)
                ev = {"own": [e for e, _ in events],
                      "peers": {r: [bk.open_event(h, like) for h in allh[r]["events"]]
                                for r in range(self.world) if r != self.rank}}
            except Exception as e:   # noqa: BLE001
                err = f"rank {self.rank}: {type(e).__name__}: {e}"
            allerr = [None] * self.world
            dist.all_gather_object(allerr, err)
            errs = [x for x in allerr if x]
        if errs:
            for c in closes:
                bk.ipc_close(c)
            for f in frees:
                bk.ipc_free(f)
            raise ScheduleUnavailable("p2p combine unavailable: " + "; ".join(errs))
        # host-only rendezvous for the per-level barriers: an NCCL barrier is a device collective
        # that waits for this rank's queued kernels, which is what the events are there to avoid
        hb = dist.barrier
        try:
            if hasattr(dist, "new_group") and dist.get_backend() == "nccl":
                grp = dist.new_group(backend="gloo")
                hb = lambda: dist.barrier(group=grp)   # noqa: E731
        except Exception:   # noqa: BLE001  (no gloo: the NCCL barrier is still correct)
            hb = dist.barrier
        self._p2p = {"local": local, "views": views, "frees": frees, "closes": closes, "events": ev,
                     "host_barrier": hb}
        return self._p2p

    def _p2p_call(self, A, B, C):
        """Products stay where they are computed; the k levels of post-additions read them (and
        each other's level results) over peer memory, each level split over the ranks; the last
        level writes every rank's rows of C into rank 0's buffer."""
        dist, bk, W, k = self.dist, self.backend, self.W, self.k
        st = self._p2p_setup(A)
        bufs = self._alloc_operands(A)
        X, Y = self._pruned_pre_adds(A, B, bufs)
        lo, hi = self.slices[self.rank]
        Mk = st["local"][k]
        for c0 in range(lo, hi, self.chunk):
            c1 = min(hi, c0 + self.chunk)
            bk.gemm_batched(X[c0:c1], Y[c0:c1], Mk[c0 - lo:c1 - lo], self.algo, self.T)
        ev = st["events"]
        bk.record(ev["own"][k])
        keep = []
        for j in range(k - 1, -1, -1):
            # level j reads every rank's level-(j+1) results: each rank recorded an interprocess
            # event after that level; the host barrier only guarantees the records are enqueued,
            # the wait itself is stream-ordered (no device synchronisation per level)
            st["host_barrier"]()
            for r, evs in ev["peers"].items():
                bk.wait(evs[j + 1])
            if j > 0:
                a, b = self.pslices[j][self.rank]
                if b > a:
                    children = []
                    for q in range(a, b):
                        for c in range(7):
                            o, off = self._owner(j + 1, 7 * q + c)
                            children.append(st["views"][(j + 1, o)][off])
                    keep.append(bk.post_add_ptrs(self.algo, children, st["local"][j][:b - a], 0, None))
            else:
                r0, r1 = self.rslices[self.rank]
                if r1 > r0:
                    children = []
                    for c in range(7):
                        o, off = self._owner(1, c)
                        children.append(st["views"][(1, o)][off])
                    keep.append(bk.post_add_ptrs(self.algo, children, st["views"]["C"], r0, r1))
            bk.record(ev["own"][j])
        # every rank's rows of C are in rank 0's buffer, and no peer still reads this rank's
        # buffers when the next call overwrites them
        bk.sync()
        dist.barrier()
        if self.rank == 0:
            C.copy_(st["local"]["C"])
        return C

    def _alloc_operands(self, like):
        """Operand buffers of the top-k pre-additions (no product buffers: p2p keeps those)."""
        if getattr(self, "_opbufs", None) is None:
            W, bk = self.W, self.backend
            ob = {"A": [], "B": []}
            for j in range(1, self.k + 1):
                mj, lj, nj = self.shapes[j]
                ob["A"].append(bk.empty((7 ** j, W, mj, lj), like))
                ob["B"].append(bk.empty((7 ** j, W, lj, nj), like))
            self._opbufs = ob
        return self._opbufs

    def release(self):
        """Unmap peers' buffers and free this rank's exported buffers (p2p combine)."""
        if self._p2p is not None:
            self.backend.sync()
            self.dist.barrier()       # nobody reads a buffer that is about to go away
            for c in self._p2p["closes"]:
                self.backend.ipc_close(c)
            self._p2p["views"].clear()
            self._p2p["local"].clear()
            self.dist.barrier()
            for f in self._p2p["frees"]:
                self.backend.ipc_free(f)
            self._p2p = None

    def _row_slabs(self, A, B, C, bufs):
        r0, r1 = self.slices[self.rank]
        local = bufs["local"]
        if self.beta:
            # C := C - A B: each rank receives its C row slab and updates it in place
            if self.rank == 0:
                for r, (a, b) in enumerate(self.slices):
                    bufs["scatter"][r][:, : b - a, :].copy_(C[:, a:b, :])
            self.dist.scatter(local, bufs.get("scatter") if self.rank == 0 else None, src=0)
        if r1 > r0:
            self.backend.gemm_rows(A, B, r0, r1, local, self.algo, self.T, self.beta)
        self.dist.gather(local, bufs.get("gather") if self.rank == 0 else None, dst=0)
        if self.rank == 0:
            for r, (a, b) in enumerate(self.slices):
                C[:, a:b, :].copy_(bufs["gather"][r][:, : b - a, :])
        return C


def host_broadcast(hX, X, dist, chunks=8):
    """X (device, every rank) := hX (pinned host tensor on rank 0), the host-to-device copy of
    each chunk overlapping the NCCL broadcast of the previous one (the copy runs on the current
    stream, the broadcast on NCCL's, which waits only for its own chunk's copy)."""
    flat = X.view(-1)
    src = hX.view(-1) if hX is not None else None
    n = flat.numel()
    step = max(1, -(-n // chunks))
    for a in range(0, n, step):
        b = min(n, a + step)
        if dist.get_rank() == 0:
            flat[a:b].copy_(src[a:b], non_blocking=True)
        dist.broadcast(flat[a:b], 0)
    return X


def _p2p(dist, ops):
    """One group of point-to-point transfers (op, tensor, peer), waited for (empty: no-op)."""
    if ops:
        for q in dist.batch_isend_irecv([dist.P2POp(op, t, peer) for op, t, peer in ops]):
            q.wait()


class BandGemm:
    """The band schedule: C := A B (beta = 0) or C := C - A B (beta = 1)
    over the process group, each rank computing one (row band x column band) tile of C with the
    WHOLE problem's recursion tree restricted to it -- bitwise the single-GPU result.

    The ranks form a G_r x G_c grid (band_grid). The depth-d leaf rows [0, m_d) are cut into G_r
    contiguous bands and the leaf columns [0, n_d) into G_c; band_index_map lifts a band to the
    level-0 rows (columns) it touches. Rank (g_r, g_c) packs those rows of A and columns of B
    (ddqd_band_copy), multiplies the compact operands with DDQD_DEPTH(d) (the same d levels of
    pre-additions, leaves and post-additions, on 1/G of every level's positions) and sends its
    compact C tile to rank 0, which unpacks every tile into C. No products or partial sums cross
    the network and there is no combine tail on rank 0: the only traffic is the operand
    broadcast and the tiles of C (with beta = 1, the tiles of C also go out first). Every
    element follows the one-GPU operation sequence, so any world size gives the same bits."""

    def __init__(self, W, algo, T, m, l, n, dist, device=None, backend=None, beta=0, replicated_inputs=False,
                 grid=None, world=None):
        self.W, self.algo, self.T, self.beta = W, algo, T, beta
        self.m, self.l, self.n = m, l, n
        self.dist = dist             # None: emulate() only, for a `world` of ranks on one device
        self.rank = dist.get_rank() if dist is not None else 0
        self.world = dist.get_world_size() if dist is not None else int(world)
        self.backend = backend or CudaBackend()
        self.replicated_inputs = replicated_inputs
        block = algo in ("block", 0)
        self.shapes = [(m, l, n)] if block else rec_shapes(m, l, n, T)
        self.d = len(self.shapes) - 1
        self.gr, self.gc = grid or band_grid(self.world)
        if self.gr * self.gc != self.world:
            raise ValueError("grid must multiply to the world size")
        mdims = [s[0] for s in self.shapes]
        ndims = [s[2] for s in self.shapes]
        rb = balanced_slices(mdims[-1], self.gr)
        cb = balanced_slices(ndims[-1], self.gc)
        # rank g = g_r * G_c + g_c owns row band g_r and column band g_c
        self.rows = [band_index_map(mdims, a, b) for a, b in rb]
        self.cols = [band_index_map(ndims, a, b) for a, b in cb]
        self._maps = None
        self._bufs = None

    def tile(self, g):
        return self.rows[g // self.gc], self.cols[g % self.gc]

    def run_tile(self, g, A, B, C, timer=None):
        """Rank g's whole share on the current device: pack its operand bands out of the full
        A and B, multiply them with the problem's depth, unpack the tile into C (beta = 1: C's
        tile is packed first and updated). `timer(fn)` may wrap the compute call."""
        bk, W = self.backend, self.W
        rows, cols = self.tile(g)
        if not rows or not cols:
            return
        rm, cm = bk.index(rows, A), bk.index(cols, A)
        Ab = bk.empty((W, len(rows), self.l), A)
        Bb = bk.empty((W, self.l, len(cols)), A)
        Ct = bk.empty((W, len(rows), len(cols)), A)
        bk.band_copy("pack", A, Ab, rm, None)
        bk.band_copy("pack", B, Bb, None, cm)
        if self.beta:
            bk.band_copy("pack", C, Ct, rm, cm)
        step = lambda: bk.gemm_depth(Ab, Bb, Ct, self.algo, self.d, self.beta)   # noqa: E731
        timer(step) if timer else step()
        bk.band_copy("unpack", C, Ct, rm, cm)

    def emulate(self, A, B, C):
        """Every rank's tile in turn on one device (no communication): the schedule's result,
        for tests and for timing one rank's share on a single GPU."""
        for g in range(self.world):
            self.run_tile(g, A, B, C)
        return C

    def _setup(self, like):
        if self._bufs is not None:
            return self._bufs
        bk, W = self.backend, self.W
        rows, cols = self.tile(self.rank)
        maps = {"r": bk.index(rows, like) if self.gr > 1 else None,
                "c": bk.index(cols, like) if self.gc > 1 else None}
        bufs = {"A": bk.empty((W, len(rows), self.l), like) if self.gr > 1 else None,
                "B": bk.empty((W, self.l, len(cols)), like) if self.gc > 1 else None,
                "C": bk.empty((W, len(rows), len(cols)), like)}
        if self.rank == 0:
            bufs["tiles"], maps["tiles"] = [], []
            for g in range(self.world):
                r, c = self.tile(g)
                bufs["tiles"].append(bufs["C"] if g == 0 else bk.empty((W, len(r), len(c)), like))
                maps["tiles"].append((bk.index(r, like), bk.index(c, like)))
        self._maps, self._bufs = maps, bufs
        return bufs

    def __call__(self, A, B, C):
        dist, bk = self.dist, self.backend
        if not self.replicated_inputs:
            dist.broadcast(A, 0)
            dist.broadcast(B, 0)
        bufs = self._setup(A)
        maps = self._maps
        Ct = bufs["C"]
        if self.beta:
            # C := C - A B: every rank's tile of C goes out first (rank 0 holds C)
            # (the collectives are ordered after the pack kernels on the current stream)
            if self.rank == 0:
                for g in range(self.world):
                    rm, cm = maps["tiles"][g]
                    bk.band_copy("pack", C, bufs["tiles"][g], rm, cm)
                _p2p(dist, [(dist.isend, bufs["tiles"][g], g) for g in range(1, self.world)])
            else:
                _p2p(dist, [(dist.irecv, Ct, 0)])
        Ab, Bb = A, B
        if bufs["A"] is not None:
            bk.band_copy("pack", A, bufs["A"], maps["r"], None)
            Ab = bufs["A"]
        if bufs["B"] is not None:
            bk.band_copy("pack", B, bufs["B"], None, maps["c"])
            Bb = bufs["B"]
        if Ct.shape[1] and Ct.shape[2]:
            bk.gemm_depth(Ab, Bb, Ct, self.algo, self.d, self.beta)
        if self.rank == 0:
            _p2p(dist, [(dist.irecv, bufs["tiles"][g], g) for g in range(1, self.world)])
            for g in range(self.world):
                rm, cm = maps["tiles"][g]
                bk.band_copy("unpack", C, bufs["tiles"][g], rm, cm)
        else:
            _p2p(dist, [(dist.isend, Ct, 0)])
        return C


class DistributedLU:
    """Blocked right-looking DD/QD LU + solve (numerics.md s.5) whose Schur updates run on all
    ranks (row f4). Rank 0 holds A ([W,n,n], overwritten with the factors) and b ([W,n]); the
    call returns (x, ipiv, info) on rank 0 and (None, None, None) elsewhere."""

    def __init__(self, W, n, K, algo, T, dist, pivot=True, backend=None, k=None):
        self.W, self.n, self.K, self.algo, self.T = W, n, K, algo, T
        self.dist, self.pivot, self.k = dist, pivot, k
        self.rank = dist.get_rank()
        self.backend = backend or CudaBackend()

    def __call__(self, A, b):
        W, n, K, bk = self.W, self.n, self.K, self.backend
        root = self.rank == 0
        ipiv = bk.empty_i64(n, A) if root else None
        info = 0
        for p in range(0, n, K):
            kb = min(K, n - p)
            if root:
                pi = bk.lu_panel(A, ipiv, p, kb, self.pivot)
                info = info or pi
            n2 = n - p - kb
            if n2 <= 0:
                continue
            if root:
                L21 = A[:, p + kb:, p:p + kb].contiguous()
                U12 = A[:, p:p + kb, p + kb:].contiguous()
                C = A[:, p + kb:, p + kb:]
            else:
                L21 = bk.empty((W, n2, kb), A)
                U12 = bk.empty((W, kb, n2), A)
                C = None
            DistributedGemm(W, self.algo, self.T, n2, kb, n2, self.dist, k=self.k, backend=bk,
                            beta=1, combine="rows")(L21, U12, C)
        if not root:
            return None, None, None
        return bk.lu_trsv(A, ipiv, b), ipiv, info


class AutoDistributedGemm:
    """C := A B (or C := C - A B) with whichever multi-GPU schedule measures fastest on this
    machine (BJ:5 (4) "... choosing whichever measures faster"). Candidates (default: the three
    that are bit-identical to one GPU, so the result never depends on which one won):
      "bands"        BandGemm: one tile of C per rank, the whole problem's tree (no combine);
      "products"     DistributedGemm: depth-k products over the ranks, NCCL to rank 0, combine there;
      "products_p2p" the same products, combined over CUDA IPC peer memory split over the ranks
                     (beta = 0 only);
      "ctiles"       C row slabs each recursing on its own (rounds differently: opt-in only).
    The first call runs every candidate once, timed with device syncs and a barrier on either
    side and the max over ranks (so every rank makes the same choice), then leaves C holding the
    chosen schedule's result (with beta = 1, C is restored before each trial and the winner is
    run once more on the original C); later calls run only the winner. `timings` (s) and
    `choice` record the measurement."""

    BITWISE = ("bands", "products_rows", "products", "products_p2p")

    def __init__(self, W, algo, T, m, l, n, dist, device=None, backend=None, beta=0, candidates=None, **kw):
        self.dist = dist
        self.beta = beta
        self.backend = backend or CudaBackend()
        self.rank = dist.get_rank()
        names = list(candidates or self.BITWISE)
        if beta:
            names = [c for c in names if c != "products_p2p"]   # the p2p combine stores C
        kw = {k: v for k, v in kw.items() if k != "combine"}
        make = {
            "bands": lambda: BandGemm(W, algo, T, m, l, n, dist, device, backend=self.backend, beta=beta,
                                      replicated_inputs=kw.get("replicated_inputs", False)),
            "products": lambda: DistributedGemm(W, algo, T, m, l, n, dist, device, backend=self.backend,
                                                beta=beta, combine="nccl", **kw),
            "products_rows": lambda: DistributedGemm(W, algo, T, m, l, n, dist, device, backend=self.backend,
                                                     beta=beta, combine="rows", **kw),
            "products_p2p": lambda: DistributedGemm(W, algo, T, m, l, n, dist, device, backend=self.backend,
                                                    combine="p2p", **kw),
            "ctiles": lambda: DistributedGemm(W, algo, T, m, l, n, dist, device, k=0, backend=self.backend,
                                              beta=beta, **kw),
        }
        unknown = [c for c in names if c not in make]
        if unknown:
            raise ValueError(f"unknown schedules {unknown}")
        self.cands = {c: make[c]() for c in names}
        self.choice = None
        self.timings = {}
        self.unavailable = {}

    def _timed(self, name, A, B, C):
        import time
        self.backend.sync()
        self.dist.barrier()
        t0 = time.perf_counter()
        self.cands[name](A, B, C)
        self.backend.sync()
        dt = time.perf_counter() - t0
        allt = [None] * self.dist.get_world_size()
        self.dist.all_gather_object(allt, dt)
        return max(allt)

    def __call__(self, A, B, C):
        if self.choice is None:
            keep = C.clone() if (self.beta and C is not None) else None
            last = None
            for name in self.cands:
                if keep is not None:
                    C.copy_(keep)
                try:
                    self.timings[name] = self._timed(name, A, B, C)
                except ScheduleUnavailable as e:   # raised on every rank alike: drop it
                    self.timings[name] = float("inf")
                    self.unavailable[name] = str(e)
                    continue
                last = name
            self.choice = min(self.timings, key=self.timings.get)
            if keep is not None:
                C.copy_(keep)
            # (a collective decision: with beta = 1 only rank 0 holds C, but every rank reruns)
            if self.beta or (self.choice != last and not
                             (self.choice in self.BITWISE and last in self.BITWISE)):
                self.cands[self.choice](A, B, C)
            return C
        return self.cands[self.choice](A, B, C)

    def release(self):
        for c in self.cands.values():
            if hasattr(c, "release"):
                c.release()


class HostStagedGroup:
    """A torch.distributed-like group over gloo that stages CUDA tensors through host memory:
    the N-GPU code paths (schedules, bench.py's N > 1 line) run as N processes sharing ONE GPU
    with no kernel ever waiting on another process (every exchange is a host-side gloo
    transfer), which is how they are exercised where only one GPU exists. A functional test
    transport, not a performance one: NCCL over NVLink is the real one."""

    class _Done:
        def wait(self):
            return True

    def __init__(self, dist):
        self.d = dist
        self.ReduceOp = dist.ReduceOp

    # markers for P2POp
    @staticmethod
    def isend(*a, **k):
        raise RuntimeError("use batch_isend_irecv")

    @staticmethod
    def irecv(*a, **k):
        raise RuntimeError("use batch_isend_irecv")

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    def get_rank(self):
        return self.d.get_rank()

    def get_world_size(self):
        return self.d.get_world_size()

    def barrier(self):
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.d.barrier()

    def all_gather_object(self, out, obj):
        self.d.all_gather_object(out, obj)

    def _stage(self, t):
        return t.detach().cpu().contiguous() if t.is_cuda else t

    def broadcast(self, t, src):
        c = self._stage(t)
        self.d.broadcast(c, src)
        if c is not t:
            t.copy_(c)

    def all_reduce(self, t, op=None):
        c = self._stage(t)
        self.d.all_reduce(c, op=op if op is not None else self.d.ReduceOp.SUM)
        if c is not t:
            t.copy_(c)

    def batch_isend_irecv(self, ops):
        sends, recvs = [], []
        for o in ops:
            if o.op is HostStagedGroup.isend:
                c = self._stage(o.tensor)
                sends.append((self.d.isend(c, o.peer), c))
            else:
                c = o.tensor.new_empty(o.tensor.shape, device="cpu") if o.tensor.is_cuda else o.tensor
                recvs.append((self.d.irecv(c, o.peer), c, o.tensor))
        for w, _ in sends:
            w.wait()
        for w, c, t in recvs:
            w.wait()
            if c is not t:
                t.copy_(c)
        return [HostStagedGroup._Done()]

    def scatter(self, t, lst=None, src=0):
        c = self._stage(t)
        cl = [self._stage(x) for x in lst] if lst is not None else None
        self.d.scatter(c, cl, src=src)
        if c is not t:
            t.copy_(c)

    def gather(self, t, lst=None, dst=0):
        c = self._stage(t)
        cl = [x.new_empty(x.shape, device="cpu") if x.is_cuda else x for x in lst] if lst is not None else None
        self.d.gather(c, cl, dst=dst)
        if lst is not None:
            for x, y in zip(lst, cl):
                if x is not y:
                    x.copy_(y)

    def destroy_process_group(self):
        self.d.destroy_process_group()
