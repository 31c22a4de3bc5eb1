// recursion.cu -- Strassen/Winograd recursion planner + device-side schedule
// (north_star subsystem (3)).
//
// Planner: depth d from the stop rule min(m,l,n) <= T ("n_min"); per-level shapes
// halve with ceil (virtual zero padding). Schedule: level j holds a batch of
// problems of one shape. A batch is processed in chunks of parents: one fused pre-add
// launch per side writes the 7 children of every parent in the chunk, the children recurse
// as ONE batch (so the 7^d leaves run as a single batched leaf-GEMM launch instead of the
// paper's 7 OpenMP sections), and one fused post-add launch combines them. Chunk
// size = whole batch (breadth-first) below a split level s and 1 parent (depth-first)
// above it; s is the smallest level whose breadth-first workspace fits the limit. The
// chunking changes only the launch grouping, never the arithmetic: results are bitwise
// those of the oracle's recursion. Where level j+1 is breadth-first, the additions of two
// levels run as one pass (pre_add2 / post_add2, DD). Optionally (DDQD_LANES=2) the chunks of
// the last depth-first level alternate between two streams with separate workspace.
// Arithmetic variants ride in Plan::mv: bits 0-3 the madd/add variant, bits 4-5 log2 of the
// split-k factor of the leaves.
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <vector>

#include "common.cuh"

namespace ddqd {

void *workspace_get(size_t bytes, int *status);   // abi.cu
size_t workspace_limit();                          // abi.cu

struct Plan {
    int W = 2, algo = 0, d = 0, s = 0, mv = 0;
    int fd = -1;                        // DDQD_DEPTH(fd): recurse exactly fd levels (T unused)
    bool fuse_last = false;             // level d-1 runs fused with its leaves (fused_last_kernel)
    int64_t T = 1;
    std::vector<int64_t> m, l, n;       // level shapes, 0..d
    std::vector<int64_t> chunk;         // parents per chunk at level j (j < d)
    std::vector<size_t> offA, offB, offM;   // byte offsets of level j+1 buffers (index j+1)
    size_t bytes = 0;
    // Two-lane schedule of the last depth-first level (j = s-1): its chunks alternate between
    // the caller's stream and an auxiliary one, each lane with its own copy of the level >= s
    // buffers, so one branch's bandwidth-bound additions overlap the other's FP64-bound leaves.
    int lanes = 1;
    size_t lane_bytes = 0;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
// workspace leading dimension. DDQD_WS_PAD=1 pads every level's to even so every row is 16-byte
// aligned and odd-width leaves qualify for the TMA leaf; measured on c3 in round 1 (one-level
// additions) this cost more in the pre-additions (23.6 vs 20.3 ms/step) than TMA gained in the
// leaf. =2 pads only the LEAF level (the operands the leaf kernel reads, written once by the
// last pre-addition pass), so c3's 256 x 257 A leaves get ld 258 and take the TMA path. 0 = tight.
static int ws_pad_mode() {
    static int pad = -1;
    if (pad < 0) {
        const char *e = getenv("DDQD_WS_PAD");
        pad = (e && (e[0] == '0' || e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
    }
    return pad;
}
static int64_t ws_ld(int64_t cols) {
    return ws_pad_mode() == 1 ? ((cols + 1) & ~int64_t(1)) : cols;
}

// leading dimension of the level-`level` workspace operands
static int64_t ws_ld_at(const Plan &p, int level, int64_t cols) {
    const int mode = ws_pad_mode();
    return (mode == 1 || (mode == 2 && level == p.d)) ? ((cols + 1) & ~int64_t(1)) : cols;
}

static void plan_shapes(Plan &p, int64_t m, int64_t l, int64_t n) {
    p.m = {m}; p.l = {l}; p.n = {n};
    if (p.algo == 0) { p.d = 0; return; }
    int d = 0;
    while (p.fd >= 0 ? d < p.fd : std::min(std::min(m, l), n) > p.T) {
        m = (m + 1) / 2; l = (l + 1) / 2; n = (n + 1) / 2;
        p.m.push_back(m); p.l.push_back(l); p.n.push_back(n);
        d++;
    }
    p.d = d;
}

// memory of split level s (levels j < s depth-first, j >= s breadth-first); with two lanes the
// buffers of levels >= s exist twice
static size_t plan_layout(Plan &p, int64_t batch, int s, int lanes, bool fill) {
    const int d = p.d;
    std::vector<int64_t> chunk(d), cnt(d + 1);
    cnt[0] = batch;
    for (int j = 0; j < d; j++) {
        chunk[j] = (j < s) ? 1 : cnt[j];
        cnt[j + 1] = 7 * chunk[j];
    }
    size_t off = 0, lane0 = 0;
    std::vector<size_t> oa(d + 1, 0), ob(d + 1, 0), om(d + 1, 0);
    for (int j = 0; j < d; j++) {
        if (j + 1 == s) { off = align256(off); lane0 = off; }   // start of the per-lane region
        const int64_t k = cnt[j + 1];
        const size_t W = (size_t)p.W;
        const size_t a = (size_t)k * W * p.m[j + 1] * ws_ld_at(p, j + 1, p.l[j + 1]) * sizeof(double);
        const size_t b = (size_t)k * W * p.l[j + 1] * ws_ld_at(p, j + 1, p.n[j + 1]) * sizeof(double);
        const size_t c = (size_t)k * W * p.m[j + 1] * ws_ld_at(p, j + 1, p.n[j + 1]) * sizeof(double);
        oa[j + 1] = off; off = align256(off + a);
        ob[j + 1] = off; off = align256(off + b);
        om[j + 1] = off; off = align256(off + c);
    }
    const bool laned = lanes > 1 && s >= 1 && s <= d;
    const size_t lane_bytes = laned ? off - lane0 : 0;
    const size_t total = off + (laned ? (size_t)(lanes - 1) * lane_bytes : 0);
    if (fill) {
        p.s = s; p.chunk = chunk; p.offA = oa; p.offB = ob; p.offM = om; p.bytes = total;
        p.lanes = laned ? lanes : 1;
        p.lane_bytes = lane_bytes;
    }
    return total;
}

// DDQD_LANES=2 enables the two-lane schedule (opt-in). Measured on c3: 351.6 vs 352.9 ms per
// step (+0.4%) for twice the workspace of levels >= s -- the leaf grid fills every SM for its
// whole duration, so the other lane's additions only run in its tail waves -- and it blurs the
// per-kernel event timing the bench's roofline uses; the single-stream schedule is the default.
static int lanes_wanted() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LANES");
        v = (e && e[0] == '2') ? 2 : 1;
    }
    return v;
}

// DDQD_DEPTH(d) rides in algo bits 16-23 as d + 1 (0 = the threshold stop rule)
static int forced_depth(int algo) { return ((algo >> 16) & 0xff) - 1; }

static int make_plan(Plan &p, int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n,
                     int64_t batch, size_t limit) {
    p.fd = forced_depth(algo);
    algo &= 0xff;
    p.W = W; p.algo = algo; p.T = T;
    plan_shapes(p, m, l, n);
    if (p.d == 0) { p.bytes = 0; p.s = 0; return DDQD_OK; }
    for (int s = 0; s <= p.d; s++) {
        if (plan_layout(p, batch, s, 1, false) <= limit || s == p.d) {
            // a second lane when the depth-first level has several chunks and the copy fits
            const int lanes = (s >= 1 && lanes_wanted() == 2 && plan_layout(p, batch, s, 2, false) <= limit) ? 2 : 1;
            plan_layout(p, batch, s, lanes, true);
            return DDQD_OK;
        }
    }
    return DDQD_OK;
}

size_t gemm_workspace_bytes(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n,
                            int64_t batch, size_t limit, int *dfs_levels) {
    algo &= 0xff00ff;
    Plan p;
    make_plan(p, W, algo, T, m, l, n, batch, limit);
    if (dfs_levels) *dfs_levels = p.s;
    return p.bytes;
}

static MatDesc child(const Plan &p, char *ws, const std::vector<size_t> &off, int level,
                     int64_t rows, int64_t cols, int lane) {
    MatDesc d;
    d.p = reinterpret_cast<double *>(ws + off[level] + (level >= p.s ? (size_t)lane * p.lane_bytes : 0));
    d.rows = rows; d.cols = cols; d.ld = ws_ld_at(p, level, cols); d.ps = rows * d.ld; d.bs = (int64_t)p.W * d.ps;
    return d;
}

static MatDesc shift(MatDesc d, int64_t p0) { d.p += p0 * d.bs; return d; }

// Two-level fusion (launch_pre_add2 / launch_post_add2) replaces the level j -> j+1 -> j+2
// additions when level j+1 runs breadth-first over this chunk's 7*pc children (its operands
// and products are then only ever needed inside the fused passes). Pairs are taken from the
// leaves upward ((d - j) even), where the skipped level is largest. DD only: the QD kernels
// would need 4x the registers for the 28 intermediate values, and QD additions are < 4% of
// a QD step. DDQD_FUSE2=0 disables it.
static bool fuse2_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("DDQD_FUSE2");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// auxiliary stream and events of the two-lane schedule, per host thread and device (a shared
// stream or event pair would let concurrent callers' fork/join points cross)
struct LaneRes {
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static int lane_res(LaneRes **out) {
    static thread_local LaneRes res[64];
    LaneRes &r = res[current_device()];
    if (!r.aux) {
        DDQD_CUDA_CHECK(cudaStreamCreateWithFlags(&r.aux, cudaStreamNonBlocking));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming));
    }
    *out = &r;
    return DDQD_OK;
}

static int exec_level(const Plan &p, char *ws, int j, int64_t cnt, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s, int lane);

// one chunk of parents [p0, p0 + pc) at level j: pre-additions, the children's recursion,
// post-additions (one level, or two fused levels)
static int exec_chunk(const Plan &p, char *ws, int j, int64_t p0, int64_t pc, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s, int lane) {
    const int var = p.mv & 0xf;
    // two-level passes are paired from the last materialised level up (d, or d-1 when the last
    // level is fused with the leaves)
    const int de = p.fuse_last ? p.d - 1 : p.d;
    const bool two = fuse2_enabled() && p.W == 2 && var != 2 && j + 2 <= de && ((de - j) % 2 == 0);
    const int add_algo = p.algo | (var == 2 ? DDQD_ADD_ACCURATE : 0);   // the additions' variant
    int rc;
    if (two && p.chunk[j + 1] >= 7 * pc) {
        const int k = j + 2;
        const MatDesc gA = child(p, ws, p.offA, k, p.m[k], p.l[k], lane);
        const MatDesc gB = child(p, ws, p.offB, k, p.l[k], p.n[k], lane);
        const MatDesc gM = child(p, ws, p.offM, k, p.m[k], p.n[k], lane);
        if ((rc = launch_pre_add2(p.W, add_algo, 0, pc, shift(A, p0), p.m[j + 1], p.l[j + 1], gA, s))) return rc;
        if ((rc = launch_pre_add2(p.W, add_algo, 1, pc, shift(B, p0), p.l[j + 1], p.n[j + 1], gB, s))) return rc;
        if ((rc = exec_level(p, ws, k, 49 * pc, gA, gB, gM, 0, s, lane))) return rc;
        return launch_post_add2(p.W, add_algo, pc, gM, p.m[j + 1], p.n[j + 1], shift(C, p0), beta, s);
    }
    const MatDesc cA = child(p, ws, p.offA, j + 1, p.m[j + 1], p.l[j + 1], lane);
    const MatDesc cB = child(p, ws, p.offB, j + 1, p.l[j + 1], p.n[j + 1], lane);
    const MatDesc cM = child(p, ws, p.offM, j + 1, p.m[j + 1], p.n[j + 1], lane);
    if ((rc = launch_pre_add(p.W, add_algo, 0, pc, shift(A, p0), cA, s))) return rc;
    if ((rc = launch_pre_add(p.W, add_algo, 1, pc, shift(B, p0), cB, s))) return rc;
    if ((rc = exec_level(p, ws, j + 1, 7 * pc, cA, cB, cM, 0, s, lane))) return rc;
    return launch_post_add(p.W, add_algo, pc, cM, shift(C, p0), beta, s);
}

static bool fuse_last_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("DDQD_FUSE_LAST");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

static const char *kLevelNames[] = {"level 0", "level 1", "level 2", "level 3", "level 4", "level 5",
                                     "level 6", "level 7", "level 8+"};

static int exec_level(const Plan &p, char *ws, int j, int64_t cnt, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s, int lane) {
    if (j == p.d) {
        NvtxRange nv("leaf GEMM");
        return launch_leaf_gemm(p.W, p.m[j], p.l[j], p.n[j], cnt, A, B, C, beta, p.mv, s);
    }
    if (p.fuse_last && j == p.d - 1) {
        NvtxRange nv("last level fused with its leaves");
        const int add_algo = p.algo | ((p.mv & 0xf) == 2 ? DDQD_ADD_ACCURATE : 0);
        return launch_fused_last(p.W, add_algo, p.mv & 0xf, cnt, A, B, C, beta, p.m[p.d], p.l[p.d], p.n[p.d], s);
    }
    NvtxRange nv(kLevelNames[j < 8 ? j : 8]);
    const int64_t nch = (cnt + p.chunk[j] - 1) / p.chunk[j];
    int rc;
    if (p.lanes == 2 && j == p.s - 1 && nch >= 2) {
        // the last depth-first level: chunks alternate between s (lane 0) and the auxiliary
        // stream (lane 1); the lanes write disjoint parts of C and own separate workspace
        LaneRes *lr;
        if ((rc = lane_res(&lr))) return rc;
        DDQD_CUDA_CHECK(cudaEventRecord(lr->fork, s));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(lr->aux, lr->fork, 0));
        for (int64_t c = 0; c < nch; c++) {
            const int64_t p0 = c * p.chunk[j], pc = std::min<int64_t>(p.chunk[j], cnt - p0);
            const int ln = (int)(c & 1);
            if ((rc = exec_chunk(p, ws, j, p0, pc, A, B, C, beta, ln ? lr->aux : s, ln))) return rc;
        }
        DDQD_CUDA_CHECK(cudaEventRecord(lr->join, lr->aux));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, lr->join, 0));
        return DDQD_OK;
    }
    for (int64_t c = 0; c < nch; c++) {
        const int64_t p0 = c * p.chunk[j], pc = std::min<int64_t>(p.chunk[j], cnt - p0);
        if ((rc = exec_chunk(p, ws, j, p0, pc, A, B, C, beta, s, lane))) return rc;
    }
    return DDQD_OK;
}

int run_gemm(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n, int64_t batch,
             const MatDesc &A, const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s) {
    if (m == 0 || n == 0 || batch == 0) return DDQD_OK;
    const int mv = ((algo & DDQD_MADD_FUSED) ? 1 : (algo & DDQD_ADD_ACCURATE) ? 2 : 0) |
                   (((algo >> 12) & 3) << 4);   // split-k (DDQD_SPLITK) rides in bits 4-5
    algo &= 0xff00ff;                                // algorithm + forced depth
    Plan p;
    int rc = make_plan(p, W, algo, T, m, l, n, batch, workspace_limit());
    if (rc) return rc;
    p.mv = mv;
    if (p.d == 0) return launch_leaf_gemm(W, m, l, n, batch, A, B, C, beta, mv, s);
    // tiny leaves (<= 32 per side, e.g. Strassen(32) at n = 1025): the last level and its leaves
    // as one kernel, when its shared-memory footprint fits (DD leaves up to ~31^3, QD up to
    // 18^3); DDQD_FUSE_LAST=0 disables it. n = 1025, threshold 32: DD 1.69 -> 1.28 ms, QD
    // 11.07 -> 9.78 ms per product (profiles/r02/fused_last_level.md)
    p.fuse_last = fuse_last_enabled() && ((mv >> 4) & 3) == 0 &&
                  fused_last_smem(W, p.m[p.d], p.l[p.d], p.n[p.d]) > 0;
    int st = DDQD_OK;
    char *ws = static_cast<char *>(workspace_get(p.bytes, &st));
    if (st) return st;
    return exec_level(p, ws, 0, batch, A, B, C, beta, s, 0);
}

}  // namespace ddqd

namespace ddqd {

// ---- host-streamed top level (the host-pointer entry, Winograd) -----------------------------
// Winograd's first product M1 = A11 B11 reads only the leading quadrants, so the host
// path copies A11 and B11 first and runs M1 while the copy engine brings in the rest of A and
// B (`front` levels deep: M1's own M1 first, on the leading quadrants of A11 and B11, ...);
// then the top level's pre-additions and the other products in an order that completes C
// quadrant by quadrant -- C11 = U1 after M2; C22 = U7 after M6, M7, M5; C12 = U5 after M3;
// C21 = U6 after M4 (itself split `tail` levels deep, so C21 completes block by block) --
// each block formed by its own post-addition pass (the same chain of DD/QD operations per
// element) and handed to on_block, which starts its device-to-host copy while the next
// products run (for a small C -- on_block null -- M2..M7 run as one batch and one
// post-addition forms C: there the batch's fuller waves are worth more than the overlapped
// copy). Each product is the same recursion as in run_gemm (the planner's chunking never
// changes the arithmetic), so the result is bitwise that of the device-pointer call.
#define return_if_err(expr)        \
    do {                           \
        const int rc__ = (expr);   \
        if (rc__) return rc__;     \
    } while (0)

static void top_shapes(int64_t m, int64_t l, int64_t n, int64_t *hm, int64_t *hl, int64_t *hn) {
    *hm = (m + 1) / 2; *hl = (l + 1) / 2; *hn = (n + 1) / 2;
}

// the 7 children (r x c, planar, workspace leading dimension) of one streamed level at base
static MatDesc kid_desc(int W, char *base, int64_t r, int64_t c) {
    MatDesc d;
    d.p = reinterpret_cast<double *>(base);
    d.rows = r; d.cols = c; d.ld = ws_ld(c); d.ps = r * d.ld; d.bs = (int64_t)W * d.ps;
    return d;
}

size_t streamed_top_bytes(int W, int64_t m, int64_t l, int64_t n) {
    int64_t hm, hl, hn;
    top_shapes(m, l, n, &hm, &hl, &hn);
    const size_t w = (size_t)7 * W * sizeof(double);
    return align256(w * hm * ws_ld(hl)) + align256(w * hl * ws_ld(hn)) + align256(w * hm * ws_ld(hn));
}

// The last product one level deeper per level of `levels` (Winograd): Aop Bop -> Mout
// (hm x hl x hn) formed as the subproblem's recursion -- pre-additions into tws[0], the
// children in the order {M1, M2} {M5, M6, M7} {M3} {M4}, each group followed by the
// post-addition of the Mout block it completes (C11 = U1, C22 = U7, C12 = U5, C21 = U6) and
// done(block) -- with the last child (M4) itself split the same way while levels remain. The
// same operations per element as run_gemm on the subproblem, so the same bits.
using BlockDone = std::function<int(int64_t r0, int64_t nr, int64_t c0, int64_t nc)>;
static int tail_rec(int W, int algo, int add_algo, int64_t T, int64_t hm, int64_t hl, int64_t hn, const MatDesc &Aop,
                    const MatDesc &Bop, const MatDesc &Mout, char *const *tws, int levels, cudaStream_t s,
                    const BlockDone &done) {
    if (levels <= 0 || std::min(std::min(hm, hl), hn) <= T) {
        return_if_err(run_gemm(W, algo, T, hm, hl, hn, 1, Aop, Bop, Mout, 0, s));
        return done(0, hm, 0, hn);
    }
    int64_t h2m, h2l, h2n;
    top_shapes(hm, hl, hn, &h2m, &h2l, &h2n);
    const size_t w = (size_t)7 * W * sizeof(double);
    const MatDesc sA = kid_desc(W, tws[0], h2m, h2l);
    const MatDesc sB = kid_desc(W, tws[0] + align256(w * h2m * ws_ld(h2l)), h2l, h2n);
    const MatDesc sM = kid_desc(W, tws[0] + align256(w * h2m * ws_ld(h2l)) + align256(w * h2l * ws_ld(h2n)), h2m, h2n);
    return_if_err(launch_pre_add(W, add_algo, 0, 1, Aop, sA, s));
    return_if_err(launch_pre_add(W, add_algo, 1, 1, Bop, sB, s));
    // Mout's block of child-grid positions [r0, r0 + nr) x [c0, c0 + nc) in quadrant q is final
    auto sub_done = [&](int q, int64_t r0, int64_t nr, int64_t c0, int64_t nc) -> int {
        return_if_err(launch_post_quad(W, add_algo, q, sM, Mout, s, r0, nr, c0, nc));
        const int64_t mr = r0 + (q >= 2 ? h2m : 0), mc = c0 + ((q & 1) ? h2n : 0);
        nr = std::min(nr, hm - mr);
        nc = std::min(nc, hn - mc);
        return nr > 0 && nc > 0 ? done(mr, nr, mc, nc) : DDQD_OK;
    };
    static const int sub[3][3] = {{0, 2, 0}, {4, 3, 3}, {2, 1, 1}};
    for (const auto &ss : sub) {
        return_if_err(run_gemm(W, algo, T, h2m, h2l, h2n, ss[1], shift(sA, ss[0]), shift(sB, ss[0]),
                               shift(sM, ss[0]), 0, s));
        return_if_err(sub_done(ss[2], 0, h2m, 0, h2n));
    }
    MatDesc m4 = shift(sM, 3);
    m4.bs = 0;
    return tail_rec(W, algo, add_algo, T, h2m, h2l, h2n, shift(sA, 3), shift(sB, 3), m4, tws + 1, levels - 1, s,
                    [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc) { return sub_done(2, r0, nr, c0, nc); });
}

int run_gemm_streamed(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, char *const *tws, const cudaEvent_t *ready, int front,
                      int tail, cudaStream_t s, int (*on_block)(int64_t r0, int64_t nr, int64_t c0, int64_t nc, void *ctx),
                      void *ctx) {
    int64_t hm, hl, hn;
    top_shapes(m, l, n, &hm, &hl, &hn);
    const size_t w = (size_t)7 * W * sizeof(double);
    const MatDesc cA = kid_desc(W, tws[0], hm, hl);
    const MatDesc cB = kid_desc(W, tws[0] + align256(w * hm * ws_ld(hl)), hl, hn);
    const MatDesc cM = kid_desc(W, tws[0] + align256(w * hm * ws_ld(hl)) + align256(w * hl * ws_ld(hn)), hm, hn);
    const int add_algo = (algo & 0xff) | (algo & DDQD_ADD_ACCURATE);
    {
        NvtxRange nv("M1 = A11 B11 (overlaps the H2D copy)");
        MatDesc a11 = A, b11 = B;
        a11.rows = hm; a11.cols = hl; b11.rows = hl; b11.cols = hn;
        if (front > 0 && std::min(std::min(hm, hl), hn) > T) {
            // M1 streamed one level deeper: its own first product (A11's and B11's leading
            // quadrants, copied first) runs while the rest of A11 and B11 arrives (ready[1]),
            // then its other six products as one batch and one post-addition -- the
            // subproblem's recursion, so the same bits as run_gemm on it
            return_if_err(run_gemm_streamed(W, algo, T, hm, hl, hn, a11, b11, cM, tws + 1, ready + 1, front - 1, 0, s,
                                            nullptr, nullptr));
        } else {
            return_if_err(run_gemm(W, algo, T, hm, hl, hn, 1, a11, b11, cM, 0, s));
        }
    }
    DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, ready[0], 0));
    NvtxRange nv("level 0 (streamed)");
    return_if_err(launch_pre_add(W, add_algo, 0, 1, A, cA, s));
    return_if_err(launch_pre_add(W, add_algo, 1, 1, B, cB, s));
    if (!on_block) {   // small C: M2..M7 as one batch (better filled waves), one post-addition
        return_if_err(run_gemm(W, algo, T, hm, hl, hn, 6, shift(cA, 1), shift(cB, 1), shift(cM, 1), 0, s));
        return launch_post_add(W, add_algo, 1, cM, C, 0, s);
    }
    // C's quadrant-q block of product-grid positions [r0, r0 + nr) x [c0, c0 + nc) is final:
    // form it and hand it over (its device-to-host copy starts while the next products run)
    auto quad_done = [&](int q, int64_t r0, int64_t nr, int64_t c0, int64_t nc) -> int {
        return_if_err(launch_post_quad(W, add_algo, q, cM, C, s, r0, nr, c0, nc));
        const int64_t cr = r0 + (q >= 2 ? hm : 0), cc = c0 + ((q & 1) ? hn : 0);
        nr = std::min(nr, m - cr);
        nc = std::min(nc, n - cc);
        return nr > 0 && nc > 0 ? on_block(cr, nr, cc, nc, ctx) : DDQD_OK;
    };
    // (first product index, count) of each step, then the quadrant it completes
    static const int steps[3][3] = {{1, 1, 0}, {4, 3, 3}, {2, 1, 1}};
    for (const auto &st : steps) {
        return_if_err(run_gemm(W, algo, T, hm, hl, hn, st[1], shift(cA, st[0]), shift(cB, st[0]),
                               shift(cM, st[0]), 0, s));
        return_if_err(quad_done(st[2], 0, hm, 0, hn));
    }
    // the last product M4 (which only C21 = U3 - M4 waits for), `tail` levels deeper: C21 is
    // formed and copied back block by block, only its last block after the compute
    NvtxRange nv4("M4 (C21 block by block)");
    MatDesc m4 = shift(cM, 3);
    m4.bs = 0;
    return tail_rec(W, algo, add_algo, T, hm, hl, hn, shift(cA, 3), shift(cB, 3), m4, tws + 1, tail, s,
                    [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc) { return quad_done(2, r0, nr, c0, nc); });
}

}  // namespace ddqd
