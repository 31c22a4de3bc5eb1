// leaf_tma.cu -- TMA + mbarrier variant of the DD leaf Block GEMM (sm_100a), used whenever
// the operands' strides are 16-byte aligned (all recursion workspace leaves: the planner pads
// their leading dimensions to even; aligned user matrices too). Same arithmetic and k order
// as leaf_gemm.cu -- bit-identical results.
//
// Per stage one elected thread arms a full-barrier with the stage's byte count and issues two
// 4-D tensor loads (A box [W][64 rows][8 k], B box [W][8 k][64 cols]; out-of-range rows/cols
// arrive zero-filled), so there is no per-element address arithmetic and no CTA-wide barrier
// in the k loop: each warp waits only for the stage it needs (full barrier) and releases it
// with one arrive (empty barrier, 8 warps). The producer refills a stage at the end of the
// following iteration, when every warp has normally finished with it.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

// k-step unroll of the inner loop. Measured (c1 / c4 leaf fraction of the FP64 peak):
// 1: 0.833 / 0.873, 2: 0.837 / 0.878, 4: 0.815 / -, 8: 0.768 / -; the cp.async leaf with its
// unroll of 4 measures 0.841 / 0.880 on the same shapes.
#ifndef LEAF_TMA_KK_UNROLL
#define LEAF_TMA_KK_UNROLL 2
#endif
constexpr int kLeafTmaKkUnroll = LEAF_TMA_KK_UNROLL;

namespace tma {
constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4, S = 4, W = 2;
constexpr int NT = (BM / TM) * (BN / TN);          // 256
constexpr int A_STAGE = W * BM * BK;                // doubles
constexpr int B_STAGE = W * BK * BN;
constexpr unsigned STAGE_BYTES = (unsigned)(sizeof(double) * (A_STAGE + B_STAGE));
constexpr size_t SMEM = sizeof(double) * (size_t)S * (A_STAGE + B_STAGE) + 2 * S * sizeof(uint64_t) + 1024;
// row-pair A stage: even rows [W][BM/2][BK + 2] from column k0, odd rows [W][BM/2][BK + 2] from
// column ld + k0 - 1 (one early, so that the box starts 16-byte aligned: TMA faults on an
// unaligned start); one box shape for both, so every thread reads its rows with one stride
constexpr int BKO = BK + 2;
constexpr int A_EVEN = W * (BM / 2) * BKO, A_ODD = W * (BM / 2) * BKO, A_STAGE_P = A_EVEN + A_ODD;
constexpr unsigned STAGE_BYTES_P = (unsigned)(sizeof(double) * (A_STAGE_P + B_STAGE));
constexpr size_t SMEM_P = sizeof(double) * (size_t)S * (A_STAGE_P + B_STAGE) + 2 * S * sizeof(uint64_t) + 1024;
}  // namespace tma

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// bounded wait: a pipeline bug traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    long long spins = 0;
    while (!mbar_try_wait(bar, parity))
        if (++spins > (1ll << 31)) __trap();
}
__device__ __forceinline__ void tma_load_4d(void *smem_dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// APAIR: A is addressed as a tensor of ROW PAIRS -- pair p = rows 2p and 2p+1 back to back, so
// its stride is 2 ld doubles = 16 ld bytes, a multiple of 16 whatever ld is. This puts odd
// leading dimensions (c3's 256 x 257 A leaves, ld 257) on TMA without padding the workspace:
// each stage loads the even rows (pair columns k0 .. k0+7, map tmA) and the odd rows (pair
// columns ld + k0 - 1 .. ld + k0 + 8, map tmA2: one column early, because a box must start on a
// 16-byte boundary -- tools/tma_align_probe showed an odd float64 start faulting) as two boxes.
// Entries past l in the even box are the odd row's first columns, not zeros -- the k loop
// never reads past l (kmax), so they are never used.
template <int MV, int APAIR>
__global__ void __launch_bounds__(tma::NT, 2)
leaf_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA2,
                const __grid_constant__ CUtensorMap tmB, int64_t m, int64_t l, int64_t n, int64_t lda, MatDesc C,
                int beta, int64_t batch0) {
    using namespace tma;
    using E = elem<2>;
    using T = dd;
    extern __shared__ unsigned char smraw[];
    constexpr int AST = APAIR ? A_STAGE_P : A_STAGE;
    // 1024-byte aligned start, by an offset from the shared array itself (a cast through an integer
    // would drop the shared address space and turn every fragment read into a generic LD)
    double *As = reinterpret_cast<double *>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
    double *Bs = As + S * AST;
    uint64_t *full = reinterpret_cast<uint64_t *>(Bs + S * B_STAGE);
    uint64_t *empty = full + S;

    const int tid = threadIdx.x, lane = tid & 31;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const int64_t b = batch0 + blockIdx.z;
    const int row0 = (int)blockIdx.y * BM, col0 = (int)blockIdx.x * BN;
    const int KT = (int)((l + BK - 1) / BK);

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        if (APAIR) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA2)) : "memory");
        for (int s = 0; s < S; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto produce = [&](int t) {   // thread 0 only: tile t into stage t % S
        const int st = t % S;
        mbar_arrive_expect_tx(full + st, APAIR ? STAGE_BYTES_P : STAGE_BYTES);
        if (APAIR) {
            tma_load_4d(As + st * AST, &tmA2, t * BK, row0 / 2, 0, (int)b, full + st);
            tma_load_4d(As + st * AST + A_EVEN, &tmA2, (int)lda + t * BK - 1, row0 / 2, 0, (int)b, full + st);
        } else {
            tma_load_4d(As + st * AST, &tmA, t * BK, row0, 0, (int)b, full + st);
        }
        tma_load_4d(Bs + st * B_STAGE, &tmB, col0, t * BK, 0, (int)b, full + st);
    };
    if (tid == 0)
        for (int t = 0; t < S - 1 && t < KT; t++) produce(t);

    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = E::zero();

    for (int kt = 0; kt < KT; kt++) {
        const int st = kt % S;
        mbar_wait(full + st, (unsigned)((kt / S) & 1));
        // [W][BM][BK]; row pairs: even [W][BM/2][BK], odd [W][BM/2][BK+2] from column 1; a
        // thread's rows all share ty's parity
        const double *as = As + st * AST + (APAIR ? (ty & 1) * (A_EVEN + 1) : 0);
        const double *bs = Bs + st * B_STAGE;   // [W][BK][BN]
        const int krem = (int)(l - (int64_t)kt * BK);
        const int kmax = krem < BK ? krem : BK;   // uniform: no madds past l
#pragma unroll (MV ? 1 : kLeafTmaKkUnroll)
        for (int kk = 0; kk < kmax; kk++) {
            double av[W][TM], bv[W][TN];
#pragma unroll
            for (int w = 0; w < W; w++) {
#pragma unroll
                for (int i = 0; i < TM; i++)
                    av[w][i] = APAIR ? as[(w * (BM / 2) + ((ty + 16 * i) >> 1)) * BKO + kk]
                                     : as[(w * BM + ty + 16 * i) * BK + kk];
                const double *brow = bs + (w * BK + kk) * BN;
#pragma unroll
                for (int j = 0; j < TN; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(brow + (j >> 1) * (BN / 2) + tx * 2);
                    bv[w][j] = v.x; bv[w][j + 1] = v.y;
                }
            }
#pragma unroll
            for (int i = 0; i < TM; i++) {
                const T a{av[0][i], av[1][i]};
#pragma unroll
                for (int j = 0; j < TN; j++) {
                    const T bb{bv[0][j], bv[1][j]};
                    acc[i][j] = MV ? dd_madd_fused(acc[i][j], a, bb) : dd_madd(acc[i][j], a, bb);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        // refill the stage of tile kt-1 with tile kt+S-1 once all warps released it
        if (tid == 0 && kt + S - 1 < KT) {
            const int t = kt + S - 1;
            if (t >= S) mbar_wait(empty + t % S, (unsigned)(((t - S) / S) & 1));
            produce(t);
        }
    }

#pragma unroll
    for (int i = 0; i < TM; i++) {
        const int64_t gi = row0 + ty + 16 * i;
        if (gi >= m) continue;
#pragma unroll
        for (int j = 0; j < TN; j++) {
            const int64_t gj = col0 + (j >> 1) * (BN / 2) + tx * 2 + (j & 1);
            if (gj >= n) continue;
            double *cp = C.p + b * C.bs + gi * C.ld + gj;
            if (beta) E::store(cp, C.ps, E::sub(E::load(cp, C.ps), acc[i][j]));
            else E::store(cp, C.ps, acc[i][j]);
        }
    }
}

// ---- 32x32 tiles: QD (4-plane boxes) and the DD tail --------------------------------------------
// 32x32 CTA tile, 2x2 micro-tile per thread (256 threads), 16-deep k slabs in 3 stages -- the
// cp.async 32x32 leaf's configuration (QD: 2 CTAs per SM; DD, the tail of a 64x64 batch and small
// grids: 4). A arrives as [W][32 rows][18 k] (two columns beyond the slab, zero or unused, so that
// the 144-byte row stride spreads a warp's four rows over distinct banks), B as [W][16 k][32
// cols]. Edge-tile entries outside C skip their madds, as in the cp.async leaf (QD: one
// renormalisation path per warp); same per-element order, same bits.
template <int W_> struct Tq {
    static constexpr int BM = 32, BN = 32, BK = 16, BKA = 18, TM = 2, TN = 2, S = 3, W = W_;
    static constexpr int NT = (BM / TM) * (BN / TN);   // 256
    static constexpr int A_STAGE = W * BM * BKA, B_STAGE = W * BK * BN;
    static constexpr unsigned STAGE_BYTES = (unsigned)(sizeof(double) * (A_STAGE + B_STAGE));
    static constexpr size_t SMEM = sizeof(double) * (size_t)S * (A_STAGE + B_STAGE) + 2 * S * sizeof(uint64_t) + 1024;
};

template <int W, int MV>
__global__ void __launch_bounds__(256, W == 2 ? 4 : 2)
leaf_tma_qd_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t m,
                   int64_t l, int64_t n, MatDesc C, int beta, int64_t batch0) {
    using Q = Tq<W>;
    constexpr int BM = Q::BM, BN = Q::BN, BK = Q::BK, BKA = Q::BKA, TM = Q::TM, TN = Q::TN, S = Q::S, NT = Q::NT;
    constexpr int A_STAGE = Q::A_STAGE, B_STAGE = Q::B_STAGE;
    constexpr unsigned STAGE_BYTES = Q::STAGE_BYTES;
    using E = arith<W, MV>;
    using T = typename E::T;
    extern __shared__ unsigned char smraw[];
    // 1024-byte aligned start, by an offset from the shared array itself (a cast through an integer
    // would drop the shared address space and turn every fragment read into a generic LD)
    double *As = reinterpret_cast<double *>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
    double *Bs = As + S * A_STAGE;
    uint64_t *full = reinterpret_cast<uint64_t *>(Bs + S * B_STAGE);
    uint64_t *empty = full + S;

    const int tid = threadIdx.x, lane = tid & 31;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const int64_t b = batch0 + blockIdx.z;
    const int row0 = (int)blockIdx.y * BM, col0 = (int)blockIdx.x * BN;
    const int KT = (int)((l + BK - 1) / BK);

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        for (int st = 0; st < S; st++) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto produce = [&](int t) {
        const int st = t % S;
        mbar_arrive_expect_tx(full + st, STAGE_BYTES);
        tma_load_4d(As + st * A_STAGE, &tmA, t * BK, row0, 0, (int)b, full + st);
        tma_load_4d(Bs + st * B_STAGE, &tmB, col0, t * BK, 0, (int)b, full + st);
    };
    if (tid == 0)
        for (int t = 0; t < S - 1 && t < KT; t++) produce(t);

    T acc[TM][TN];
    bool live[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) {
            acc[i][j] = E::zero();
            live[i][j] = row0 + 2 * ty + i < m && col0 + 2 * tx + j < n;
        }

    for (int kt = 0; kt < KT; kt++) {
        const int st = kt % S;
        mbar_wait(full + st, (unsigned)((kt / S) & 1));
        const double *as = As + st * A_STAGE;   // [W][BM][BKA]
        const double *bs = Bs + st * B_STAGE;   // [W][BK][BN]
        const int krem = (int)(l - (int64_t)kt * BK);
        const int kmax = krem < BK ? krem : BK;
        for (int kk = 0; kk < kmax; kk++) {
            T a[TM], bb[TN];
#pragma unroll
            for (int w = 0; w < W; w++) {
#pragma unroll
                for (int i = 0; i < TM; i++) E::set_word(a[i], w, as[(w * BM + 2 * ty + i) * BKA + kk]);
                const double2 v = *reinterpret_cast<const double2 *>(bs + (w * BK + kk) * BN + 2 * tx);
                E::set_word(bb[0], w, v.x);
                E::set_word(bb[1], w, v.y);
            }
#pragma unroll
            for (int i = 0; i < TM; i++)
#pragma unroll
                for (int j = 0; j < TN; j++)
                    if (live[i][j]) acc[i][j] = E::madd(acc[i][j], a[i], bb[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (tid == 0 && kt + S - 1 < KT) {
            const int t = kt + S - 1;
            if (t >= S) mbar_wait(empty + t % S, (unsigned)(((t - S) / S) & 1));
            produce(t);
        }
    }
#pragma unroll
    for (int i = 0; i < TM; i++) {
        const int64_t gi = row0 + 2 * ty + i;
        if (gi >= m) continue;
#pragma unroll
        for (int j = 0; j < TN; j++) {
            const int64_t gj = col0 + 2 * tx + j;
            if (gj >= n) continue;
            double *cp = C.p + b * C.bs + gi * C.ld + gj;
            if (beta) E::store(cp, C.ps, E::sub(E::load(cp, C.ps), acc[i][j]));
            else E::store(cp, C.ps, acc[i][j]);
        }
    }
}

// ---- host side --------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool encoder() {
    static int tried = 0;
    if (!tried) {
        tried = 1;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        else
            cudaGetLastError();
    }
    return g_encode != nullptr;
}

// 4-D map over a batch of planar matrices: dims {cols, rows, W, batch}; box {bc, br, W, 1}.
// pair = true: the row-pair view {ld + cols, rows / 2, W, batch} (rows must be even).
static bool make_map(CUtensorMap *map, const MatDesc &d, int64_t batch, unsigned bc, unsigned br, bool pair = false,
                     int W = 2) {
    const uint64_t al = 16;
    const int64_t rs = pair ? 2 * d.ld : d.ld;   // row (pair) stride in doubles
    if (reinterpret_cast<uintptr_t>(d.p) % al || (rs * 8) % al || (d.ps * 8) % al) return false;
    if (pair && (d.rows % 2)) return false;
    const int64_t bs = batch > 1 ? d.bs : W * d.ps;
    if ((bs * 8) % al || d.ld < d.cols || d.cols <= 0 || d.rows <= 0) return false;
    cuuint64_t dims[4] = {(cuuint64_t)(pair ? d.ld + d.cols : d.cols), (cuuint64_t)(pair ? d.rows / 2 : d.rows),
                          (cuuint64_t)W, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)rs * 8, (cuuint64_t)d.ps * 8, (cuuint64_t)bs * 8};
    cuuint32_t box[4] = {bc, br, (cuuint32_t)W, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d.p, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Odd-ld A operands (c3's 256 x 257 leaves) take TMA through the row-pair view; DDQD_LEAF_APAIR=0
// keeps them on the cp.async leaf. Measured on c3 (profiles/r02/c3_leaf_load_paths.md): 0.939 of
// the FP64 peak with row-pair TMA vs 0.923 cp.async (343.2 vs 349.8 ms per step).
static bool apair_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_APAIR");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// Returns 1 if launched (rc = status), 0 if the shape/strides do not qualify (caller falls back).
int try_leaf_tma(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                 const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc) {
    using namespace tma;
    *rc = DDQD_OK;
    if (l == 0 || batch > 0x7fffffffLL || m > 0x7fffffffLL || l > 0x7fffffffLL || !encoder()) return 0;
    CUtensorMap ma, mb;
    if (!make_map(&mb, B, batch, BN, BK)) return 0;
    // A: the plain view when its rows are 16-byte aligned, else the row-pair view
    CUtensorMap ma2;
    int pair = 0;
    if (!make_map(&ma, A, batch, BK, BM)) {
        // row pairs: the odd rows' boxes start at ld + k0 - 1, 16-byte aligned only for odd ld
        if (!apair_enabled() || A.ld % 2 == 0 || !make_map(&ma, A, batch, BK, BM / 2, true) ||
            !make_map(&ma2, A, batch, BKO, BM / 2, true))
            return 0;
        pair = 1;
    } else {
        ma2 = ma;
    }
    auto kern = mv ? (pair ? leaf_tma_kernel<1, 1> : leaf_tma_kernel<1, 0>)
                   : (pair ? leaf_tma_kernel<0, 1> : leaf_tma_kernel<0, 0>);
    static bool attr_set[4][64] = {};   // per variant and device
    bool &attr = attr_set[2 * mv + pair][current_device()];
    const size_t smem = pair ? SMEM_P : SMEM;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        attr = true;
    }
    const int64_t gx = (n + BN - 1) / BN, gy = (m + BM - 1) / BM;
    if (gx > 0x7fffffff || gy > 65535) return 0;
    prof_begin(0, s);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t bz = (batch - b0) < 65535 ? (batch - b0) : 65535;
        // the maps index the batch absolutely: shift the problem index by b0 inside the kernel
        kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)bz), NT, smem, s>>>(ma, ma2, mb, m, l, n, A.ld, C, beta, b0);
        count_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("TMA leaf launch: ") + cudaGetErrorString(e));
            *rc = DDQD_ECUDA;
            return 1;
        }
    }
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s,
             pair ? "leaf_tma_kernel (TMA, row-pair A)" : "leaf_tma_kernel (TMA)");
    return 1;
}

}  // namespace ddqd

namespace ddqd {

// DDQD_LEAF_TMA_QD=0 keeps QD on the cp.async leaf (A/B measurements)
static bool tma_qd_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_TMA_QD");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// 32x32-tile TMA leaf (QD, and the DD tail / small grids); returns 1 if launched (rc = status),
// 0 if the shape/strides do not qualify.
template <int W>
static int try_tma32(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                     const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc) {
    using Q = Tq<W>;
    constexpr int BM = Q::BM, BN = Q::BN, BK = Q::BK, BKA = Q::BKA, NT = Q::NT;
    constexpr size_t SMEM = Q::SMEM;
    *rc = DDQD_OK;
    if (l == 0 || batch > 0x7fffffffLL || m > 0x7fffffffLL || l > 0x7fffffffLL || !encoder()) return 0;
    CUtensorMap ma, mb;
    if (!make_map(&ma, A, batch, BKA, BM, false, W) || !make_map(&mb, B, batch, BN, BK, false, W)) return 0;
    auto kern = mv == 1 ? leaf_tma_qd_kernel<W, 1> : mv == 2 ? leaf_tma_qd_kernel<W, 2> : leaf_tma_qd_kernel<W, 0>;
    static bool attr_set[3][64] = {};
    bool &attr = attr_set[mv][current_device()];
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        attr = true;
    }
    const int64_t gx = (n + BN - 1) / BN, gy = (m + BM - 1) / BM;
    if (gx > 0x7fffffff || gy > 65535) return 0;
    prof_begin(0, s);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t bz = (batch - b0) < 65535 ? (batch - b0) : 65535;
        kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)bz), NT, SMEM, s>>>(ma, mb, m, l, n, C, beta, b0);
        count_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("32x32 TMA leaf launch: ") + cudaGetErrorString(e));
            *rc = DDQD_ECUDA;
            return 1;
        }
    }
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s,
             W == 4 ? "leaf_tma_qd_kernel (TMA)" : "leaf_tma32_kernel (TMA, DD 32x32)");
    return 1;
}

int try_leaf_tma_qd(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                    const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc) {
    *rc = DDQD_OK;
    if (!tma_qd_enabled()) return 0;
    return try_tma32<4>(m, l, n, batch, A, B, C, beta, mv, s, rc);
}

// DDQD_LEAF_TMA32=1 puts DD 32x32 tiles (the tail of a 64x64 batch, small grids) on this TMA leaf.
// Off by default: on c1's tail it measured 0.656 of the FP64 peak against 0.698 for the cp.async
// 32x32 leaf (both are bound by the 2x2 micro-tile's four dependent DD chains per thread).
static bool tma32_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LEAF_TMA32");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

int try_leaf_tma32_dd(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                      const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc) {
    *rc = DDQD_OK;
    if (!tma32_enabled()) return 0;
    return try_tma32<2>(m, l, n, batch, A, B, C, beta, mv, s, rc);
}

}  // namespace ddqd
