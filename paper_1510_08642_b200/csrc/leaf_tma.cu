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

template <int MV>
__global__ void __launch_bounds__(tma::NT, 2)
leaf_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t m,
                int64_t l, int64_t n, MatDesc C, int beta, int64_t batch0) {
    using namespace tma;
    using E = elem<2>;
    using T = dd;
    extern __shared__ unsigned char smraw[];
    double *As = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
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
        for (int s = 0; s < S; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto produce = [&](int t) {   // thread 0 only: tile t into stage t % S
        const int st = t % S;
        mbar_arrive_expect_tx(full + st, STAGE_BYTES);
        tma_load_4d(As + st * A_STAGE, &tmA, t * BK, row0, 0, (int)b, full + st);
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
        const double *as = As + st * A_STAGE;   // [W][BM][BK]
        const double *bs = Bs + st * B_STAGE;   // [W][BK][BN]
        const int krem = (int)(l - (int64_t)kt * BK);
        const int kmax = krem < BK ? krem : BK;   // uniform: no madds past l
#pragma unroll kLeafTmaKkUnroll
        for (int kk = 0; kk < kmax; kk++) {
            double av[W][TM], bv[W][TN];
#pragma unroll
            for (int w = 0; w < W; w++) {
#pragma unroll
                for (int i = 0; i < TM; i++) av[w][i] = as[(w * BM + ty + 16 * i) * BK + kk];
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

// 4-D map over a batch of planar matrices: dims {cols, rows, W, batch}; box {bc, br, W, 1}
static bool make_map(CUtensorMap *map, const MatDesc &d, int64_t batch, unsigned bc, unsigned br) {
    const uint64_t al = 16;
    if (reinterpret_cast<uintptr_t>(d.p) % al || (d.ld * 8) % al || (d.ps * 8) % al) return false;
    const int64_t bs = batch > 1 ? d.bs : 2 * d.ps;
    if ((bs * 8) % al || d.ld < d.cols || d.cols <= 0 || d.rows <= 0) return false;
    cuuint64_t dims[4] = {(cuuint64_t)d.cols, (cuuint64_t)d.rows, 2, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)d.ld * 8, (cuuint64_t)d.ps * 8, (cuuint64_t)bs * 8};
    cuuint32_t box[4] = {bc, br, 2, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d.p, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Returns 1 if launched (rc = status), 0 if the shape/strides do not qualify (caller falls back).
int try_leaf_tma(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                 const MatDesc &C, int beta, int mv, cudaStream_t s, int *rc) {
    using namespace tma;
    *rc = DDQD_OK;
    if (l == 0 || batch > 0x7fffffffLL || m > 0x7fffffffLL || l > 0x7fffffffLL || !encoder()) return 0;
    CUtensorMap ma, mb;
    if (!make_map(&ma, A, batch, BK, BM) || !make_map(&mb, B, batch, BN, BK)) return 0;
    auto kern = mv ? leaf_tma_kernel<1> : leaf_tma_kernel<0>;
    static bool attr_set[2][64] = {};   // per variant and device
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
        // the maps index the batch absolutely: shift the problem index by b0 inside the kernel
        kern<<<dim3((unsigned)gx, (unsigned)gy, (unsigned)bz), NT, SMEM, s>>>(ma, mb, m, l, n, C, beta, b0);
        count_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("TMA leaf launch: ") + cudaGetErrorString(e));
            *rc = DDQD_ECUDA;
            return 1;
        }
    }
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s);
    return 1;
}

}  // namespace ddqd
