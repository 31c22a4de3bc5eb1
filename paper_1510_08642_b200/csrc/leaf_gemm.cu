// leaf_gemm.cu -- the Block leaf GEMM for DD and QD on sm_100a (SURVEY.md N4/N5,
// north_star subsystem (2); "Block", Eq. (1)).
//
// C[b] := A[b] B[b] (beta = 0) or C[b] := C[b] - A[b] B[b] (beta = 1) for a batch of
// problems of identical shape (grid.z = problem index: the BFS-batched 7^d Strassen /
// Winograd leaves run as ONE launch).
//
// Per CTA: a BM x BN tile of C; per thread: a TM x TN register micro-tile of DD/QD
// accumulators. Each element is accumulated from +0 over k ascending (numerics.md s.4),
// so the result is bit-identical to the oracle's Simple/Block. The k loop streams
// BK-deep slabs of A (stored k-major, i.e. transposed, so a thread's TM rows are one
// 16-byte shared load per pair) and B through a STAGES-deep cp.async ring with zero-fill
// for the ragged edges; the FP64 pipe does DADD/DMUL/DFMA only (20 per DD madd, ~200 per
// QD madd). Shared-memory traffic per madd is 1/TM + 1/TN words per operand (tiny next to
// the 20-200 FP64 instructions), so the kernel is FP64-pipe bound by design.
#include <cstdlib>

#include "common.cuh"
#include "cp_async.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

// k-step unroll of the inner loop: 4 lets the compiler issue the next steps' shared-memory
// fragment loads under the current step's FP64 chains. Measured (c3 cp.async leaf / c2 QD):
// 1: 0.9162 / 0.8795, 2: 0.9194, 4: 0.9218 / 0.8799, 8: 0.9233 / 0.7997 of the FP64 peak.
// QD keeps 1: on ragged leaves (2000x1500x1800 Winograd(256): 500x375x450 leaves, whose edge
// tiles mix real and zero-padded lanes that take different renormalisation branches) the
// unrolled QD loop measured 0.633 vs 0.751 of the peak.
// (The TMA leaf takes 2: see leaf_tma.cu.)
#ifndef LEAF_KK_UNROLL
#define LEAF_KK_UNROLL 4
#endif
constexpr int kLeafKkUnroll = LEAF_KK_UNROLL;

template <int W, int BM, int BN, int BK, int TM, int TN, int STAGES>
struct LeafCfg {
    static constexpr int TX = BN / TN;          // threads along n
    static constexpr int TY = BM / TM;          // threads along m
    static constexpr int NT = TX * TY;
    static constexpr int LDA_S = BM + 2;        // k-major A slab row (even: 16B-aligned pairs)
    static constexpr int LDB_S = BN;            // k-major B slab row (natural layout)
    static constexpr int A_STAGE = W * BK * LDA_S;
    static constexpr int B_STAGE = W * BK * LDB_S;
    static constexpr size_t SMEM = sizeof(double) * (size_t)STAGES * (A_STAGE + B_STAGE);
    static_assert(TM % 2 == 0 && TN % 2 == 0, "micro-tile pairs");
};

// row of micro-tile entry i for thread coordinate t: pairs spread over BM/(TM/2) bands
template <int BM, int TM>
__device__ __forceinline__ int micro_idx(int t, int i) {
    return (i >> 1) * (BM / (TM / 2)) + t * 2 + (i & 1);
}

template <int W, int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int MV>
__global__ void __launch_bounds__(LeafCfg<W, BM, BN, BK, TM, TN, STAGES>::NT, MINB)
leaf_gemm_kernel(int64_t m, int64_t l, int64_t n, MatDesc A, MatDesc B, MatDesc C, int beta,
                 int64_t batch0) {
    using Cfg = LeafCfg<W, BM, BN, BK, TM, TN, STAGES>;
    using E = arith<W, MV>;   // MV: 0 canonical, 1 fused DD madd, 2 accurate adds
    constexpr int kUnroll = W == 2 ? kLeafKkUnroll : 1;   // QD: see kLeafKkUnroll
    using T = typename E::T;
    constexpr int NT = Cfg::NT;
    extern __shared__ __align__(16) double smem[];
    double *As = smem;
    double *Bs = smem + STAGES * Cfg::A_STAGE;

    const int tid = threadIdx.x;
    const int tx = tid % Cfg::TX, ty = tid / Cfg::TX;
    const int64_t b = batch0 + blockIdx.z;
    const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
    const double *Ab = A.p + b * A.bs;
    const double *Bb = B.p + b * B.bs;
    double *Cb = C.p + b * C.bs;

    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = E::zero();

    const int64_t KT = (l + BK - 1) / BK;
    // QD: micro-tile entries outside C (zero-padded rows/columns of edge tiles) are skipped.
    // Their lanes would otherwise take the zero branches of the renormalisation while their
    // neighbours take the data branches, and the warp would run both; skipping leaves one path.
    // (Never stored either way, so the results are unchanged; DD has no data branches.)
    bool live[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++)
            live[i][j] = W == 2 || (row0 + micro_idx<BM, TM>(ty, i) < m && col0 + micro_idx<BN, TN>(tx, j) < n);

    auto load_stage = [&](int stage, int64_t kt) {
        const int64_t k0 = kt * BK;
        double *as = As + stage * Cfg::A_STAGE;
        double *bs = Bs + stage * Cfg::B_STAGE;
#pragma unroll 4
        for (int e = tid; e < W * BM * BK; e += NT) {
            const int w = e / (BM * BK), rem = e % (BM * BK), r = rem / BK, kk = rem % BK;
            const int64_t gi = row0 + r, gk = k0 + kk;
            const bool ok = gi < m && gk < l;
            const double *src = ok ? Ab + w * A.ps + gi * A.ld + gk : Ab;
            cp_async8(as + (w * BK + kk) * Cfg::LDA_S + r, src, ok);
        }
#pragma unroll 4
        for (int e = tid; e < W * BK * BN; e += NT) {
            const int w = e / (BK * BN), rem = e % (BK * BN), kk = rem / BN, c = rem % BN;
            const int64_t gk = k0 + kk, gj = col0 + c;
            const bool ok = gk < l && gj < n;
            const double *src = ok ? Bb + w * B.ps + gk * B.ld + gj : Bb;
            cp_async8(bs + (w * BK + kk) * Cfg::LDB_S + c, src, ok);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (s < KT) load_stage(s, s);
        cp_async_commit();
    }

    for (int64_t kt = 0; kt < KT; kt++) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < KT) load_stage((int)(nk % STAGES), nk);
            cp_async_commit();
        }
        const int st = (int)(kt % STAGES);
        const double *as = As + st * Cfg::A_STAGE;
        const double *bs = Bs + st * Cfg::B_STAGE;
        const int64_t krem = l - kt * BK;
        const int kmax = krem < BK ? (int)krem : BK;   // uniform: no madds past l
#pragma unroll kUnroll
        for (int kk = 0; kk < kmax; kk++) {
            double av[W][TM], bv[W][TN];
#pragma unroll
            for (int w = 0; w < W; w++) {
                const double *arow = as + (w * BK + kk) * Cfg::LDA_S;
                const double *brow = bs + (w * BK + kk) * Cfg::LDB_S;
#pragma unroll
                for (int i = 0; i < TM; i += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(arow + micro_idx<BM, TM>(ty, i));
                    av[w][i] = v.x; av[w][i + 1] = v.y;
                }
#pragma unroll
                for (int j = 0; j < TN; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(brow + micro_idx<BN, TN>(tx, j));
                    bv[w][j] = v.x; bv[w][j + 1] = v.y;
                }
            }
#pragma unroll
            for (int i = 0; i < TM; i++) {
                T a;
                if constexpr (W == 2) { a.hi = av[0][i]; a.lo = av[1][i]; }
                else {
#pragma unroll
                    for (int w = 0; w < W; w++) a.w[w] = av[w][i];
                }
#pragma unroll
                for (int j = 0; j < TN; j++) {
                    T bb;
                    if constexpr (W == 2) { bb.hi = bv[0][j]; bb.lo = bv[1][j]; }
                    else {
#pragma unroll
                        for (int w = 0; w < W; w++) bb.w[w] = bv[w][j];
                    }
                    if (W == 2 || live[i][j]) acc[i][j] = E::madd(acc[i][j], a, bb);
                }
            }
        }
    }
    cp_async_wait<0>();

    // epilogue: masked stores (crop of ragged tiles), optional C := C - AB
#pragma unroll
    for (int i = 0; i < TM; i++) {
        const int64_t gi = row0 + micro_idx<BM, TM>(ty, i);
        if (gi >= m) continue;
#pragma unroll
        for (int j = 0; j < TN; j++) {
            const int64_t gj = col0 + micro_idx<BN, TN>(tx, j);
            if (gj >= n) continue;
            double *cp = Cb + gi * C.ld + gj;
            if (beta) {
                T old = E::load(cp, C.ps);
                E::store(cp, C.ps, E::sub(old, acc[i][j]));
            } else {
                E::store(cp, C.ps, acc[i][j]);
            }
        }
    }
}

template <int W, int BM, int BN, int BK, int TM, int TN, int STAGES, int MINB, int MV = 0>
static int launch_cfg(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s) {
    using Cfg = LeafCfg<W, BM, BN, BK, TM, TN, STAGES>;
    auto kern = leaf_gemm_kernel<W, BM, BN, BK, TM, TN, STAGES, MINB, MV>;
    static bool attr_set[64] = {};   // per template instance and device
    const int dev = current_device();
    if (!attr_set[dev]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)Cfg::SMEM));
        attr_set[dev] = true;
    }
    const int64_t gx = (n + BN - 1) / BN, gy = (m + BM - 1) / BM;
    if (gx > 0x7fffffff || gy > 65535) {
        set_error("leaf GEMM: matrix too large for the tile grid");
        return DDQD_EINVAL;
    }
    prof_begin(0, s);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t bz = (batch - b0) < 65535 ? (batch - b0) : 65535;
        dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)bz);
        kern<<<grid, Cfg::NT, Cfg::SMEM, s>>>(m, l, n, A, B, C, beta, b0);
        DDQD_LAUNCH_CHECK();
    }
    static const std::string nm = "leaf_gemm_kernel<" + std::to_string(W) + "," + std::to_string(BM) + "," +
                                  std::to_string(BN) + "," + std::to_string(BK) + "," + std::to_string(TM) + "," +
                                  std::to_string(TN) + "," + std::to_string(STAGES) + "," + std::to_string(MINB) + "," +
                                  std::to_string(MV) + "> (cp.async)";
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s, nm.c_str());
    return DDQD_OK;
}

// DDQD_LEAF_CFG selects an alternative tile configuration (tuning experiments only;
// tools/tune_leaf.py). Every configuration computes the same bits.
// DDQD_TAIL_CFG (experiments): the DD tail tile -- 0 32x32 (2x2 micro-tile, 256 threads),
// 1 32x32 (4x4, 64 threads), 2 32x64 (4x4, 128 threads). Measured on c1's tail (fraction of the
// FP64 peak): 0.699 / 0.648 / 0.669, step 0.969 / 0.982 / 0.976 ms -- the default stays.
static int tail_cfg() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_TAIL_CFG");
        v = e ? atoi(e) : 0;
    }
    return v;
}

static int leaf_cfg_override() {
    static int v = -2;
    if (v == -2) {
        const char *e = getenv("DDQD_LEAF_CFG");
        v = e ? atoi(e) : -1;
    }
    return v;
}

int try_leaf_tma(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                 const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc);   // leaf_tma.cu
int try_leaf_tma_qd(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                    const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc);   // leaf_tma.cu
int try_leaf_tma32_dd(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                      const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc);   // leaf_tma.cu

// DDQD_LEAF_TMA=0 disables the TMA + mbarrier DD leaf (A/B comparisons); default on
static bool tma_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_TMA");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

int launch_leaf_splitk(int W, int split, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                       const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);   // leaf_splitk.cu

// DDQD_LEAF_TAIL=0 disables the tail split below (A/B measurements)
static bool tail_split_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_TAIL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static MatDesc shift_batch(MatDesc d, int64_t b0) { d.p += b0 * d.bs; return d; }

int launch_leaf_small(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);   // leaf_small.cu
static bool small_enabled();

static int launch_leaf_one(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                           const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);

int launch_leaf_flat(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);   // leaf_small.cu
bool leaf_pack_fits(int W, int64_t m, int64_t l, int64_t n);                                       // leaf_small.cu
int launch_leaf_pack(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);   // leaf_small.cu

// DDQD_LEAF_RAGGED=0 disables the interior / strip split and the flat leaf (A/B measurements)
static bool ragged_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_RAGGED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// DDQD_LEAF_PACK=1 routes tiny leaves to the shared-memory packed kernel (A/B experiments)
static bool pack_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_PACK");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

static MatDesc rows_from(MatDesc d, int64_t r0, int64_t rows) { d.p += r0 * d.ld; d.rows = rows; return d; }
static MatDesc cols_from(MatDesc d, int64_t c0, int64_t cols) { d.p += c0; d.cols = cols; return d; }

int launch_leaf_gemm(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    if (m == 0 || n == 0 || batch == 0) return DDQD_OK;
    // mv: arithmetic variant (low 4 bits) | log2(split-k) << 4
    const int split = 1 << ((mv >> 4) & 3);
    if (split > 1) return launch_leaf_splitk(W, split, m, l, n, batch, A, B, C, beta, mv & 0xf, s);
    mv &= 0xf;
    // Ragged leaves (n = 1025 at threshold 128: 65 x 65; at 32: 17 x 17). The tile kernels pad
    // every leaf to whole CTA tiles: a 65 x 65 leaf is 4 tiles of 64 of which 3 are slivers
    // running the full k loop, a 17 x 17 leaf uses 28% of a 32 x 32 tile. Instead the tile-
    // aligned interior of ALL leaves runs as one batched tile launch (strided views of the same
    // leaves) and the remaining row / column strips -- or, for leaves below one tile, the whole
    // leaves -- go to the flat 2x2-per-thread kernel. Each element keeps its operation order.
    if (ragged_enabled() && leaf_cfg_override() < 0) {
        const int64_t TL = (W == 2 && m > 32 && n > 32) ? 64 : 32;
        const int64_t mt = m / TL * TL, nt = n / TL * TL;
        const double used = (double)m * (double)n /
                            (double)(((m + TL - 1) / TL * TL) * ((n + TL - 1) / TL * TL));
        if (used < 0.8) {
            if (mt == 0 || nt == 0) {   // below one tile: the flat kernel takes the whole leaves
                // (staging 3 such leaves per CTA through shared memory, leaf_pack_kernel, measured
                // slower: DD Strassen(32) n = 1025 2.07 vs 1.64 ms, QD 12.6 vs 11.0 ms)
                if (pack_enabled() && leaf_pack_fits(W, m, l, n))
                    return launch_leaf_pack(W, m, l, n, batch, A, B, C, beta, mv, s);
                return launch_leaf_flat(W, m, l, n, batch, A, B, C, beta, mv, s);
            }
            int rc = launch_leaf_gemm(W, mt, l, nt, batch, rows_from(A, 0, mt), cols_from(B, 0, nt),
                                      cols_from(rows_from(C, 0, mt), 0, nt), beta, mv, s);
            if (rc) return rc;
            // right strip: rows [0, mt) x cols [nt, n); bottom strip: rows [mt, m) x all columns
            auto strip = [&](int64_t sm, int64_t sn, const MatDesc &a, const MatDesc &b, const MatDesc &c) {
                if (sm == 0 || sn == 0) return (int)DDQD_OK;
                if (sm < 32 || sn < 32) return launch_leaf_flat(W, sm, l, sn, batch, a, b, c, beta, mv, s);
                return launch_leaf_gemm(W, sm, l, sn, batch, a, b, c, beta, mv, s);
            };
            if ((rc = strip(mt, n - nt, rows_from(A, 0, mt), cols_from(B, nt, n - nt),
                            cols_from(rows_from(C, 0, mt), nt, n - nt)))) return rc;
            return strip(m - mt, n, rows_from(A, mt, m - mt), B, rows_from(C, mt, m - mt));
        }
    }
    // Tail split (DD): a batch of 64x64-tile leaves whose last wave would leave most of the
    // GPU idle runs its whole waves with 64x64 tiles and the remaining leaves with 32x32 tiles
    // (4x the CTAs for the same work) -- same per-element order, so the same bits.
    // E.g. c1: 343 leaves x 4 tiles = 1372 CTAs = 4.64 waves of 296 (1.071 -> 1.047 ms).
    // Only for batches of >= 32 leaves: on the 7-leaf Strassen updates of the c4 LU the
    // model below also predicts a gain, but the measured step was not faster (58.25 vs 58.5 ms).
    if (W == 2 && tail_split_enabled() && leaf_cfg_override() < 0 && m > 32 && n > 32 && batch >= 32) {
        const int64_t t = ((m + 63) / 64) * ((n + 63) / 64), slots = 2 * (int64_t)sm_count();
        const int64_t total = t * batch, waves = total / slots, rem = total % slots;
        if (waves >= 2 && rem > 0 && rem * 4 < slots * 3) {   // last wave under 75% full
            const int64_t b1 = waves * slots / t;              // leaves filling the whole waves
            // cost model in big-tile wave times: a 32x32 tile is 1/4 of the work at ~0.8 of
            // the efficiency, 4 fit per SM; split only when it saves >= 5%
            const int64_t small = (batch - b1) * t * 4, slots_small = 4 * (int64_t)sm_count();
            const double t_split = (double)((b1 * t + slots - 1) / slots) +
                                   0.3125 * (double)((small + slots_small - 1) / slots_small);
            if (b1 > 0 && b1 < batch && t_split < 0.95 * (double)(waves + 1)) {
                int rc = launch_leaf_one(W, m, l, n, b1, A, B, C, beta, mv, s);
                if (rc) return rc;
                const MatDesc A2 = shift_batch(A, b1), B2 = shift_batch(B, b1), C2 = shift_batch(C, b1);
                if (tma_enabled() && try_leaf_tma32_dd(m, l, n, batch - b1, A2, B2, C2, beta, mv, s, &rc)) return rc;
                if (mv == 1) return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2, 1>(m, l, n, batch - b1, A2, B2, C2, beta, s);
                if (mv == 2) return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2, 2>(m, l, n, batch - b1, A2, B2, C2, beta, s);
                if (tail_cfg() == 1)   // 64-thread CTAs with 4x4 micro-tiles (16 chains per thread)
                    return launch_cfg<2, 32, 32, 8, 4, 4, 4, 8>(m, l, n, batch - b1, A2, B2, C2, beta, s);
                if (tail_cfg() == 2)
                    return launch_cfg<2, 32, 64, 8, 4, 4, 4, 4>(m, l, n, batch - b1, A2, B2, C2, beta, s);
                return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2>(m, l, n, batch - b1, A2, B2, C2, beta, s);
            }
        }
    }
    // QD: the same idea with the one-element-per-thread leaf for the remaining leaves (its four
    // shared loads per madd are small next to ~200 FP64 ops; a 128-thread CTA holds 1/4 of a
    // 32x32 2x2-micro-tile CTA's work). c2: 343 leaves x 16 tiles = 5488 CTAs = 18.5 waves:
    // 333 leaves on 32x32 tiles + 10 on the small leaf, 9.137 -> 9.004 ms (leaf 0.879 -> 0.892).
    if (W == 4 && mv != 1 && tail_split_enabled() && leaf_cfg_override() < 0 && small_enabled() && batch >= 32) {
        const int64_t t = ((m + 31) / 32) * ((n + 31) / 32), slots = 2 * (int64_t)sm_count();
        const int64_t total = t * batch, waves = total / slots, rem = total % slots;
        if (waves >= 2 && rem > 0 && rem * 4 < slots * 3) {
            const int64_t b1 = waves * slots / t;
            // small CTAs: 8x16 outputs, ~3 per SM at ~150 registers; one small wave ~0.19 of a
            // big one (per-SM FP64 work 9.8M vs 52M lane-ops)
            const int64_t small = (batch - b1) * ((m + 7) / 8) * ((n + 15) / 16), slots_small = 3 * (int64_t)sm_count();
            const double t_split = (double)((b1 * t + slots - 1) / slots) +
                                   0.19 * (double)((small + slots_small - 1) / slots_small);
            if (b1 > 0 && b1 < batch && t_split < 0.99 * (double)(waves + 1)) {
                int rc = launch_leaf_one(W, m, l, n, b1, A, B, C, beta, mv, s);
                if (rc) return rc;
                return launch_leaf_small(W, m, l, n, batch - b1, shift_batch(A, b1), shift_batch(B, b1),
                                         shift_batch(C, b1), beta, mv, s);
            }
        }
    }
    return launch_leaf_one(W, m, l, n, batch, A, B, C, beta, mv, s);
}

int launch_leaf_small(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);   // leaf_small.cu

// DDQD_LEAF_SMALL=0 disables the small-output leaf (A/B measurements)
static bool small_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_SMALL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static int launch_leaf_one(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                           const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    // few outputs (the 32x32 grid would leave SMs without a CTA, and one element per thread
    // gives <= 2 CTAs of 128 per SM): latency-bound, one element per thread (leaf_small.cu).
    // With more outputs its 4 shared loads per madd make it slower than the 2x2 micro-tiles
    // (c4's last Strassen update, 7 x 128^3: 30.7 us small vs ~21 us 32x32).
    if (small_enabled() && leaf_cfg_override() < 0 && ((m + 31) / 32) * ((n + 31) / 32) * batch < sm_count() &&
        m * n * batch <= (int64_t)sm_count() * 256)
        return launch_leaf_small(W, m, l, n, batch, A, B, C, beta, mv, s);
    if (W == 2 && mv != 2 && tma_enabled() && leaf_cfg_override() < 0) {
        const int64_t big_tiles = ((m + 63) / 64) * ((n + 63) / 64) * batch;
        if (big_tiles >= 2 * sm_count() && m > 32 && n > 32) {
            int rc = DDQD_OK;
            if (try_leaf_tma(m, l, n, batch, A, B, C, beta, mv, s, &rc)) return rc;
        }
    }
    if (mv == 1) {   // fused DD / QD madd (numerics.md s.2-3, row f3)
        if (W == 4) {
            int rc = DDQD_OK;
            if (try_leaf_tma_qd(m, l, n, batch, A, B, C, beta, mv, s, &rc)) return rc;
            return launch_cfg<4, 32, 32, 16, 2, 2, 3, 2, 1>(m, l, n, batch, A, B, C, beta, s);
        }
        const int64_t big_tiles = ((m + 63) / 64) * ((n + 63) / 64) * batch;
        if (big_tiles >= 2 * sm_count() && m > 32 && n > 32)
            return launch_cfg<2, 64, 64, 8, 4, 4, 4, 2, 1>(m, l, n, batch, A, B, C, beta, s);
        return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2, 1>(m, l, n, batch, A, B, C, beta, s);
    }
    if (mv == 2) {   // accurate adds (numerics.md s.2-3, row f3)
        if (W == 4) {
            int rc = DDQD_OK;
            if (try_leaf_tma_qd(m, l, n, batch, A, B, C, beta, mv, s, &rc)) return rc;
            return launch_cfg<4, 32, 32, 16, 2, 2, 3, 2, 2>(m, l, n, batch, A, B, C, beta, s);
        }
        const int64_t big_tiles = ((m + 63) / 64) * ((n + 63) / 64) * batch;
        if (big_tiles >= 2 * sm_count() && m > 32 && n > 32)
            return launch_cfg<2, 64, 64, 8, 4, 4, 4, 2, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2, 2>(m, l, n, batch, A, B, C, beta, s);
    }
    switch (leaf_cfg_override()) {
    case 0: return launch_cfg<2, 64, 64, 16, 4, 4, 3, 2>(m, l, n, batch, A, B, C, beta, s);
    case 1: return launch_cfg<2, 64, 64, 8, 4, 4, 4, 2>(m, l, n, batch, A, B, C, beta, s);
    case 2: return launch_cfg<2, 32, 64, 16, 2, 4, 3, 3>(m, l, n, batch, A, B, C, beta, s);
    case 3: return launch_cfg<2, 64, 32, 16, 4, 2, 3, 3>(m, l, n, batch, A, B, C, beta, s);
    case 4: return launch_cfg<2, 64, 64, 16, 4, 4, 2, 2>(m, l, n, batch, A, B, C, beta, s);
    case 5: return launch_cfg<2, 32, 32, 16, 2, 2, 3, 4>(m, l, n, batch, A, B, C, beta, s);
    case 6: return launch_cfg<2, 64, 64, 32, 4, 4, 2, 1>(m, l, n, batch, A, B, C, beta, s);
    case 10: return launch_cfg<4, 32, 32, 16, 2, 2, 3, 2>(m, l, n, batch, A, B, C, beta, s);
    case 11: return launch_cfg<4, 32, 32, 8, 2, 2, 4, 2>(m, l, n, batch, A, B, C, beta, s);
    case 12: return launch_cfg<4, 16, 32, 16, 2, 2, 3, 4>(m, l, n, batch, A, B, C, beta, s);
    case 13: return launch_cfg<4, 32, 64, 8, 2, 4, 3, 1>(m, l, n, batch, A, B, C, beta, s);
    default: break;
    }
    if (W == 2) {
        // 64x64 tiles when the grid fills the GPU and the leaf is not smaller than a tile
        const int64_t big_tiles = ((m + 63) / 64) * ((n + 63) / 64) * batch;
        if (big_tiles >= 2 * sm_count() && m > 32 && n > 32)   // tools/tune_leaf.py: BK = 8 x 4 stages is the fastest DD tile
            return launch_cfg<2, 64, 64, 8, 4, 4, 4, 2>(m, l, n, batch, A, B, C, beta, s);
        {
            int rc = DDQD_OK;
            if (tma_enabled() && try_leaf_tma32_dd(m, l, n, batch, A, B, C, beta, mv, s, &rc)) return rc;
        }
        return launch_cfg<2, 32, 32, 16, 2, 2, 3, 2>(m, l, n, batch, A, B, C, beta, s);
    }
    if (W == 4) {
        int rc = DDQD_OK;
        if (try_leaf_tma_qd(m, l, n, batch, A, B, C, beta, mv, s, &rc)) return rc;
        return launch_cfg<4, 32, 32, 16, 2, 2, 3, 2>(m, l, n, batch, A, B, C, beta, s);
    }
    set_error("leaf GEMM: precision must be 2 (DD) or 4 (QD)");
    return DDQD_EINVAL;
}

}  // namespace ddqd
