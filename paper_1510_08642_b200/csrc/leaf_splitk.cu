// leaf_splitk.cu -- split-k leaf GEMM for small shapes (reading R10;
// numerics.md s.4 "Split-k leaf"), the Blackwell way: one thread-block CLUSTER of S CTAs per
// 32x32 tile of C. CTA rank q of the cluster forms the partial product over k-slice q
// (contiguous slices of ceil(l/S), k ascending from +0) in registers and parks it in its
// shared memory; after a cluster barrier the partials are combined through distributed shared
// memory (DSMEM) by the fixed pairwise tree ((p0+p1)+(p2+p3))+..., CTA q reducing rows
// [q*32/S, (q+1)*32/S) of the tile, and a second cluster barrier keeps every CTA's partial
// alive until its peers have read it. S x more CTAs than the 32x32 leaf, so a 128^3 problem
// (config 0: 16 tiles) occupies 128 SMs instead of 16.
#include <cooperative_groups.h>

#include "common.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

constexpr int SK_T = 32;    // C tile edge
constexpr int SK_KC = 16;   // k chunk staged in shared memory

template <int W, int S, int V>
__global__ void __launch_bounds__(256) leaf_splitk_kernel(int64_t m, int64_t l, int64_t n, MatDesc A,
                                                          MatDesc B, MatDesc C, int beta, int64_t batch0) {
    using E = arith<W, V>;
    using T = typename E::T;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    // the k-chunk staging buffers and, after the k loop, the partial share one array
    constexpr int A_SZ = W * SK_T * (SK_KC + 1), B_SZ = W * SK_KC * (SK_T + 1), P_SZ = W * SK_T * SK_T;
    constexpr int SM_SZ = (A_SZ + B_SZ) > P_SZ ? (A_SZ + B_SZ) : P_SZ;
    __shared__ double smem[SM_SZ];
    auto As = reinterpret_cast<double (*)[SK_T][SK_KC + 1]>(smem);            // [W][SK_T][SK_KC+1]
    auto Bs = reinterpret_cast<double (*)[SK_KC][SK_T + 1]>(smem + A_SZ);     // [W][SK_KC][SK_T+1]
    auto part = reinterpret_cast<double (*)[SK_T * SK_T]>(smem);              // [W][SK_T*SK_T]
    const int q = (int)cl.block_rank();
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int64_t b = batch0 + blockIdx.z;
    const int64_t row0 = (int64_t)blockIdx.y * SK_T, col0 = (int64_t)(blockIdx.x / S) * SK_T;
    const double *Ab = A.p + b * A.bs;
    const double *Bb = B.p + b * B.bs;
    const int64_t L = (l + S - 1) / S;
    const int64_t k0 = q * L < l ? q * L : l, k1 = (q + 1) * L < l ? (q + 1) * L : l;

    T acc[2][2];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) acc[i][j] = E::zero();
    for (int64_t kb = k0; kb < k1; kb += SK_KC) {
        const int kc_n = (int)((k1 - kb) < SK_KC ? (k1 - kb) : SK_KC);
        for (int e = tid; e < SK_T * SK_KC; e += 256) {
            const int r = e / SK_KC, kc = e % SK_KC;
            const int64_t gi = row0 + r, gk = kb + kc;
            const bool ok = gi < m && kc < kc_n;
#pragma unroll
            for (int w = 0; w < W; w++) As[w][r][kc] = ok ? Ab[w * A.ps + gi * A.ld + gk] : 0.0;
        }
        for (int e = tid; e < SK_KC * SK_T; e += 256) {
            const int kc = e / SK_T, c = e % SK_T;
            const int64_t gk = kb + kc, gj = col0 + c;
            const bool ok = gj < n && kc < kc_n;
#pragma unroll
            for (int w = 0; w < W; w++) Bs[w][kc][c] = ok ? Bb[w * B.ps + gk * B.ld + gj] : 0.0;
        }
        __syncthreads();
        for (int kc = 0; kc < kc_n; kc++) {
            T a[2], bb[2];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int w = 0; w < W; w++) {
                    E::set_word(a[i], w, As[w][ty + 16 * i][kc]);
                    E::set_word(bb[i], w, Bs[w][kc][tx + 16 * i]);
                }
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 2; j++) acc[i][j] = E::madd(acc[i][j], a[i], bb[j]);
        }
        __syncthreads();
    }
    __syncthreads();   // staging buffers dead: the partial takes their place
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
            for (int w = 0; w < W; w++) part[w][(ty + 16 * i) * SK_T + tx + 16 * j] = E::word(acc[i][j], w);
    cl.sync();   // every partial of the cluster is in its CTA's shared memory
    constexpr int RPC = SK_T / S;   // tile rows reduced by this CTA
    for (int e = tid; e < RPC * SK_T; e += 256) {
        const int r = q * RPC + e / SK_T, c = e % SK_T;
        T p[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            const double *peer = cl.map_shared_rank(&part[0][0], s);
#pragma unroll
            for (int w = 0; w < W; w++) E::set_word(p[s], w, peer[w * SK_T * SK_T + r * SK_T + c]);
        }
#pragma unroll
        for (int stride = 1; stride < S; stride *= 2)
#pragma unroll
            for (int s = 0; s + stride < S; s += 2 * stride) p[s] = E::add(p[s], p[s + stride]);
        const int64_t gi = row0 + r, gj = col0 + c;
        if (gi < m && gj < n) {
            double *cp = C.p + b * C.bs + gi * C.ld + gj;
            if (beta) E::store(cp, C.ps, E::sub(E::load(cp, C.ps), p[0]));
            else E::store(cp, C.ps, p[0]);
        }
    }
    cl.sync();   // peers may still be reading this CTA's partial
}

template <int W, int S, int V>
static int launch_splitk_t(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                           const MatDesc &C, int beta, cudaStream_t s) {
    const int64_t gx = (n + SK_T - 1) / SK_T * S, gy = (m + SK_T - 1) / SK_T;
    if (gx > 0x7fffffff || gy > 65535) {
        set_error("split-k leaf: matrix too large for the tile grid");
        return DDQD_EINVAL;
    }
    prof_begin(0, s);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t bz = (batch - b0) < 65535 ? (batch - b0) : 65535;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)bz);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, leaf_splitk_kernel<W, S, V>, m, l, n, A, B, C, beta, b0);
        count_launch();
        if (e != cudaSuccess) {
            set_error(std::string("split-k leaf launch: ") + cudaGetErrorString(e));
            return DDQD_ECUDA;
        }
    }
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s, "leaf_splitk_kernel (cluster DSMEM tree)");
    return DDQD_OK;
}

template <int W, int V>
static int launch_splitk_w(int split, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                           const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s) {
    if (split == 2) return launch_splitk_t<W, 2, V>(m, l, n, batch, A, B, C, beta, s);
    if (split == 4) return launch_splitk_t<W, 4, V>(m, l, n, batch, A, B, C, beta, s);
    return launch_splitk_t<W, 8, V>(m, l, n, batch, A, B, C, beta, s);
}

int launch_leaf_splitk(int W, int split, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                       const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    if (m == 0 || n == 0 || batch == 0) return DDQD_OK;
    if (W == 2) {
        if (mv == 1) return launch_splitk_w<2, 1>(split, m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_splitk_w<2, 2>(split, m, l, n, batch, A, B, C, beta, s);
        return launch_splitk_w<2, 0>(split, m, l, n, batch, A, B, C, beta, s);
    }
    if (mv == 1) return launch_splitk_w<4, 1>(split, m, l, n, batch, A, B, C, beta, s);
    if (mv == 2) return launch_splitk_w<4, 2>(split, m, l, n, batch, A, B, C, beta, s);
    return launch_splitk_w<4, 0>(split, m, l, n, batch, A, B, C, beta, s);
}

}  // namespace ddqd
