// leaf_small.cu -- the latency-bound leaf GEMM for small outputs (SURVEY.md s.8 row a4,
// BJ:7 config c0: DD Block 128^3; Eq. (1)).
//
// When a leaf call has few outputs (the 32x32-tile grid would not give every SM a CTA), the
// time is set by the dependent chain of each element's k-ascending accumulation, not by the
// FP64 pipe: one DD madd adds ~56 cycles of latency through the accumulator (TwoSum +
// FastTwoSum on acc.hi, numerics.md s.2), so a 128-deep k loop costs >= 7.2k cycles however
// many FP64 lanes are idle. The throughput leaf's 2x2 micro-tiles and 32x32 CTAs put c0's
// 16384 chains on 16 SMs (1024 chains per SM: the FP64 pipe, 320 cycles per k step, becomes
// the bound). Here every thread owns ONE element and a CTA an 8x16 tile (128 threads), so c0
// runs 128 CTAs -- ~28 chains per SM sub-partition, under the latency bound. Same per-element
// operation order as leaf_gemm_kernel (acc from +0, k ascending, E::madd), so the same bits.
#include "common.cuh"
#include "cp_async.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

namespace {

constexpr int kSmBM = 8, kSmBN = 16, kSmStages = 3, kSmNT = kSmBM * kSmBN;
// k depth per stage: 32 (DD) / 16 (QD) keeps the 3-stage ring at 36 KB of static shared memory
template <int W> struct SmBK { static constexpr int v = W == 2 ? 32 : 16; };

template <int W, int MV>
__global__ void __launch_bounds__(kSmNT) leaf_small_kernel(int64_t m, int64_t l, int64_t n, MatDesc A,
                                                           MatDesc B, MatDesc C, int beta, int64_t batch0) {
    using E = arith<W, MV>;
    using T = typename E::T;
    constexpr int kSmBK = SmBK<W>::v;
    constexpr int AST = W * kSmBM * kSmBK, BST = W * kSmBK * kSmBN;
    __shared__ __align__(16) double As[kSmStages * AST];   // [stage][w][r][kk]
    __shared__ __align__(16) double Bs[kSmStages * BST];   // [stage][w][kk][c]
    const int tid = threadIdx.x, tx = tid % kSmBN, ty = tid / kSmBN;
    const int64_t b = batch0 + blockIdx.z;
    const int64_t row0 = (int64_t)blockIdx.y * kSmBM, col0 = (int64_t)blockIdx.x * kSmBN;
    const double *Ab = A.p + b * A.bs;
    const double *Bb = B.p + b * B.bs;
    const int64_t gi = row0 + ty, gj = col0 + tx;
    const bool live = gi < m && gj < n;

    auto load_stage = [&](int st, int64_t kt) {
        const int64_t k0 = kt * kSmBK;
        double *as = As + st * AST;
        double *bs = Bs + st * BST;
#pragma unroll
        for (int e = tid; e < AST; e += kSmNT) {
            const int w = e / (kSmBM * kSmBK), rem = e % (kSmBM * kSmBK), r = rem / kSmBK, kk = rem % kSmBK;
            const int64_t ri = row0 + r, gk = k0 + kk;
            const bool ok = ri < m && gk < l;
            cp_async8(as + e, ok ? Ab + w * A.ps + ri * A.ld + gk : Ab, ok);
        }
#pragma unroll
        for (int e = tid; e < BST; e += kSmNT) {
            const int w = e / (kSmBK * kSmBN), rem = e % (kSmBK * kSmBN), kk = rem / kSmBN, c = rem % kSmBN;
            const int64_t gk = k0 + kk, cj = col0 + c;
            const bool ok = gk < l && cj < n;
            cp_async8(bs + e, ok ? Bb + w * B.ps + gk * B.ld + cj : Bb, ok);
        }
    };

    T acc = E::zero();
    const int64_t KT = (l + kSmBK - 1) / kSmBK;
#pragma unroll
    for (int st = 0; st < kSmStages - 1; st++) {
        if (st < KT) load_stage(st, st);
        cp_async_commit();
    }
    for (int64_t kt = 0; kt < KT; kt++) {
        cp_async_wait<kSmStages - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + kSmStages - 1;
            if (nk < KT) load_stage((int)(nk % kSmStages), nk);
            cp_async_commit();
        }
        const int st = (int)(kt % kSmStages);
        const double *as = As + st * AST + ty * kSmBK;
        const double *bs = Bs + st * BST + tx;
        const int64_t krem = l - kt * kSmBK;
        const int kmax = krem < kSmBK ? (int)krem : kSmBK;
        auto lda = [&](int kk) {
            T a;
            if constexpr (W == 2) { a.hi = as[kk]; a.lo = as[kSmBM * kSmBK + kk]; }
            else {
#pragma unroll
                for (int w = 0; w < W; w++) a.w[w] = as[w * kSmBM * kSmBK + kk];
            }
            return a;
        };
        auto ldb = [&](int kk) {
            T bb;
            if constexpr (W == 2) { bb.hi = bs[kk * kSmBN]; bb.lo = bs[kSmBK * kSmBN + kk * kSmBN]; }
            else {
#pragma unroll
                for (int w = 0; w < W; w++) bb.w[w] = bs[w * kSmBK * kSmBN + kk * kSmBN];
            }
            return bb;
        };
        if (live) {
            int kk = 0;
            if constexpr (MV != 1) {
                // madd = add(acc, mul(a, b)) (V 0 / 2): the 8 products of a group do not depend
                // on acc, so they are formed first and only the adds stay on the chain
                for (; kk + 8 <= kmax; kk += 8) {
                    T p[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) p[u] = E::mul(lda(kk + u), ldb(kk + u));
#pragma unroll
                    for (int u = 0; u < 8; u++) acc = E::add(acc, p[u]);
                }
            }
            for (; kk < kmax; kk++) acc = E::madd(acc, lda(kk), ldb(kk));
        }
    }
    cp_async_wait<0>();
    if (!live) return;
    double *cp = C.p + b * C.bs + gi * C.ld + gj;
    if (beta) E::store(cp, C.ps, E::sub(E::load(cp, C.ps), acc));
    else E::store(cp, C.ps, acc);
}

template <int W, int MV>
int launch_small(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                 const MatDesc &C, int beta, cudaStream_t s) {
    const int64_t gx = (n + kSmBN - 1) / kSmBN, gy = (m + kSmBM - 1) / kSmBM;
    if (gx > 0x7fffffff || gy > 65535) {
        set_error("small leaf GEMM: matrix too large for the tile grid");
        return DDQD_EINVAL;
    }
    prof_begin(0, s);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t bz = (batch - b0) < 65535 ? (batch - b0) : 65535;
        leaf_small_kernel<W, MV><<<dim3((unsigned)gx, (unsigned)gy, (unsigned)bz), kSmNT, 0, s>>>(
            m, l, n, A, B, C, beta, b0);
        DDQD_LAUNCH_CHECK();
    }
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s);
    return DDQD_OK;
}

}  // namespace

// the small-output leaf (mv = arithmetic variant 0 / 1 / 2)
int launch_leaf_small(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    if (W == 2) {
        if (mv == 1) return launch_small<2, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_small<2, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_small<2, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    if (W == 4) {
        if (mv == 1) return launch_small<4, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_small<4, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_small<4, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    set_error("leaf GEMM: precision must be 2 (DD) or 4 (QD)");
    return DDQD_EINVAL;
}

}  // namespace ddqd
