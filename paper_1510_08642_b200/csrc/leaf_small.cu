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
#include <cstdlib>

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
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s, "leaf_small_kernel");
    return DDQD_OK;
}

// ---- flat leaf for tiny leaves and the ragged strips of larger ones -------------------------
// One thread per RM x RN block of outputs of ONE leaf (DD 2 x 2, QD 1 x 1: its madd is ~200
// FP64 instructions, so loads are cheap and more, lighter threads hide its long chains better),
// threads numbered flat over (leaf, block row, block column), so leaves of 17 x 17
// (Strassen(32) at n = 1025) or the one-row / one-column strips of 65 x 65 leaves do not strand
// most of a 32x32 or 64x64 CTA tile. Operands come straight from global memory through L1 (a
// leaf's A and B rows are shared by its threads), software-pipelined one k step ahead (ncu:
// long-scoreboard stalls dominated without it). Each output is acc := +0, k ascending, E::madd
// -- the same per-element sequence as every other leaf, so the same bits.
template <int W, int MV, int RM, int RN>
__global__ void __launch_bounds__(256, W == 2 ? 3 : 2) leaf_flat_kernel(int64_t m, int64_t l, int64_t n, int64_t total,
                                                                     MatDesc A, MatDesc B, MatDesc C, int beta) {
    using E = arith<W, MV>;
    using T = typename E::T;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int64_t hn = (n + RN - 1) / RN, per = ((m + RM - 1) / RM) * hn;
    const int64_t b = t / per, r = t % per;
    const int64_t i = RM * (r / hn), j = RN * (r % hn);
    const double *ap[RM];
#pragma unroll
    for (int u = 0; u < RM; u++) ap[u] = A.p + b * A.bs + (i + u < m ? i + u : i) * A.ld;
    int64_t bo[RN];
#pragma unroll
    for (int v = 0; v < RN; v++) bo[v] = j + v < n ? v : 0;
    const double *b0 = B.p + b * B.bs + j;
    auto ld = [&](const double *q, int64_t ps) {
        T x;
#pragma unroll
        for (int w = 0; w < W; w++) E::set_word(x, w, __ldg(q + w * ps));
        return x;
    };
    T c[RM][RN];
#pragma unroll
    for (int u = 0; u < RM; u++)
#pragma unroll
        for (int v = 0; v < RN; v++) c[u][v] = E::zero();
    if (l > 0) {
        T x[RM], y[RN];
#pragma unroll
        for (int u = 0; u < RM; u++) x[u] = ld(ap[u], A.ps);
#pragma unroll
        for (int v = 0; v < RN; v++) y[v] = ld(b0 + bo[v], B.ps);
        for (int64_t k = 0; k < l; k++) {
            const int64_t kn = k + 1 < l ? k + 1 : k;
            T nx[RM], ny[RN];
#pragma unroll
            for (int u = 0; u < RM; u++) nx[u] = ld(ap[u] + kn, A.ps);
#pragma unroll
            for (int v = 0; v < RN; v++) ny[v] = ld(b0 + kn * B.ld + bo[v], B.ps);
#pragma unroll
            for (int u = 0; u < RM; u++)
#pragma unroll
                for (int v = 0; v < RN; v++) c[u][v] = E::madd(c[u][v], x[u], y[v]);
#pragma unroll
            for (int u = 0; u < RM; u++) x[u] = nx[u];
#pragma unroll
            for (int v = 0; v < RN; v++) y[v] = ny[v];
        }
    }
#pragma unroll
    for (int u = 0; u < RM; u++)
#pragma unroll
        for (int v = 0; v < RN; v++) {
            if (i + u >= m || j + v >= n) continue;
            double *q = C.p + b * C.bs + (i + u) * C.ld + j + v;
            if (beta) E::store(q, C.ps, E::sub(E::load(q, C.ps), c[u][v]));
            else E::store(q, C.ps, c[u][v]);
        }
}

template <int W, int MV, int RM = (W == 2 ? 2 : 1), int RN = (W == 2 ? 2 : 1)>
int launch_flat(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                const MatDesc &C, int beta, cudaStream_t s) {
    const int64_t total = batch * ((m + RM - 1) / RM) * ((n + RN - 1) / RN);
    if (total == 0) return DDQD_OK;
    if ((total + 255) / 256 > 0x7fffffff) {
        set_error("flat leaf GEMM: too many outputs for one grid");
        return DDQD_EINVAL;
    }
    prof_begin(0, s);
    leaf_flat_kernel<W, MV, RM, RN><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(m, l, n, total, A, B, C, beta);
    DDQD_LAUNCH_CHECK();
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s, "leaf_flat_kernel");
    return DDQD_OK;
}

// ---- packed leaf: several tiny leaves per CTA, operands staged whole in shared memory --------
// For leaves with m, n <= 32 and l <= 64 (Strassen(32) at n = 1025: 17 x 17 x 17). A CTA of
// 256 threads takes NL = 256 / (ceil(m/2) ceil(n/2)) leaves (3 for 17 x 17), copies their A and
// B planes into shared memory with coalesced loads, and each thread forms a 2x2 block of one
// leaf's outputs from shared memory. Same per-element sequence as every leaf kernel.
template <int W, int MV>
__global__ void __launch_bounds__(256, W == 2 ? 3 : 1) leaf_pack_kernel(int64_t m, int64_t l, int64_t n, int64_t batch, int NL,
                                                           MatDesc A, MatDesc B, MatDesc C, int beta) {
    using E = arith<W, MV>;
    using T = typename E::T;
    extern __shared__ double smp[];
    const int tid = threadIdx.x;
    const int64_t leaf0 = (int64_t)blockIdx.x * NL;
    const int nl = (int)((batch - leaf0) < NL ? (batch - leaf0) : NL);
    const int ml = (int)(m * l), ln = (int)(l * n);
    double *As = smp;                                   // [NL][W][m][l]
    double *Bs = smp + (size_t)NL * W * ml;             // [NL][W][l][n]
    for (int e = tid; e < nl * W * ml; e += blockDim.x) {
        const int q = e / (W * ml), rem = e % (W * ml), w = rem / ml, r2 = rem % ml;
        const int i = r2 / (int)l, k = r2 % (int)l;
        As[e] = __ldg(A.p + (leaf0 + q) * A.bs + w * A.ps + i * A.ld + k);
    }
    for (int e = tid; e < nl * W * ln; e += blockDim.x) {
        const int q = e / (W * ln), rem = e % (W * ln), w = rem / ln, r2 = rem % ln;
        const int k = r2 / (int)n, j = r2 % (int)n;
        Bs[e] = __ldg(B.p + (leaf0 + q) * B.bs + w * B.ps + k * B.ld + j);
    }
    __syncthreads();
    const int hn = (int)((n + 1) / 2), P = (int)((m + 1) / 2) * hn;
    const int q = tid / P, r = tid % P;
    if (q >= nl) return;
    const int i = 2 * (r / hn), j = 2 * (r % hn);
    const bool i1 = i + 1 < m, j1 = j + 1 < n;
    const double *a0 = As + (size_t)q * W * ml + i * l;
    const double *a1 = i1 ? a0 + l : a0;
    const double *b0 = Bs + (size_t)q * W * ln + j;
    const int bo = j1 ? 1 : 0;
    auto ld = [&](const double *p0, int ps) {
        T v;
#pragma unroll
        for (int w = 0; w < W; w++) E::set_word(v, w, p0[w * ps]);
        return v;
    };
    T c00 = E::zero(), c01 = E::zero(), c10 = E::zero(), c11 = E::zero();
    for (int k = 0; k < (int)l; k++) {
        const T x0 = ld(a0 + k, ml), x1 = ld(a1 + k, ml);
        const double *bk = b0 + k * n;
        const T y0 = ld(bk, ln), y1 = ld(bk + bo, ln);
        c00 = E::madd(c00, x0, y0);
        c01 = E::madd(c01, x0, y1);
        c10 = E::madd(c10, x1, y0);
        c11 = E::madd(c11, x1, y1);
    }
    double *cp = C.p + (leaf0 + q) * C.bs + i * C.ld + j;
    auto put = [&](double *p0, const T &v) {
        if (beta) E::store(p0, C.ps, E::sub(E::load(p0, C.ps), v));
        else E::store(p0, C.ps, v);
    };
    put(cp, c00);
    if (j1) put(cp + 1, c01);
    if (i1) {
        put(cp + C.ld, c10);
        if (j1) put(cp + C.ld + 1, c11);
    }
}

template <int W, int MV>
int launch_pack(int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A, const MatDesc &B,
                const MatDesc &C, int beta, cudaStream_t s) {
    const int P = (int)(((m + 1) / 2) * ((n + 1) / 2));
    const int NL = 256 / P;
    const size_t smem = sizeof(double) * (size_t)NL * W * (size_t)l * (size_t)(m + n);
    static bool attr[64] = {};
    if (!attr[current_device()]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(leaf_pack_kernel<W, MV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024));
        attr[current_device()] = true;
    }
    const int64_t blocks = (batch + NL - 1) / NL;
    prof_begin(0, s);
    leaf_pack_kernel<W, MV><<<(unsigned)blocks, 256, smem, s>>>(m, l, n, batch, NL, A, B, C, beta);
    DDQD_LAUNCH_CHECK();
    prof_end(0, (double)m * (double)l * (double)n * (double)batch, s, "leaf_pack_kernel");
    return DDQD_OK;
}

}  // namespace

// leaves with m, n <= 32 and l <= 64 whose staged operands fit in shared memory
bool leaf_pack_fits(int W, int64_t m, int64_t l, int64_t n) {
    if (m < 1 || n < 1 || m > 32 || n > 32 || l < 1 || l > 64) return false;
    const int NL = (int)(256 / (((m + 1) / 2) * ((n + 1) / 2)));
    return sizeof(double) * (size_t)NL * W * (size_t)l * (size_t)(m + n) <= 200 * 1024;
}

int launch_leaf_pack(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    if (W == 2) {
        if (mv == 1) return launch_pack<2, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_pack<2, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_pack<2, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    if (W == 4) {
        if (mv == 1) return launch_pack<4, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_pack<4, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_pack<4, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    set_error("leaf GEMM: precision must be 2 (DD) or 4 (QD)");
    return DDQD_EINVAL;
}

// the flat 2x2-per-thread leaf (mv = arithmetic variant 0 / 1 / 2)
int launch_leaf_flat(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s) {
    if (W == 2) {
        if (mv == 1) return launch_flat<2, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_flat<2, 2>(m, l, n, batch, A, B, C, beta, s);
        static int tile = -1;   // DDQD_FLAT_DD=11|12|21: per-thread output block (experiments)
        if (tile < 0) { const char *e = getenv("DDQD_FLAT_DD"); tile = e ? atoi(e) : 22; }
        if (tile == 11) return launch_flat<2, 0, 1, 1>(m, l, n, batch, A, B, C, beta, s);
        if (tile == 12) return launch_flat<2, 0, 1, 2>(m, l, n, batch, A, B, C, beta, s);
        if (tile == 21) return launch_flat<2, 0, 2, 1>(m, l, n, batch, A, B, C, beta, s);
        return launch_flat<2, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    if (W == 4) {
        if (mv == 1) return launch_flat<4, 1>(m, l, n, batch, A, B, C, beta, s);
        if (mv == 2) return launch_flat<4, 2>(m, l, n, batch, A, B, C, beta, s);
        return launch_flat<4, 0>(m, l, n, batch, A, B, C, beta, s);
    }
    set_error("leaf GEMM: precision must be 2 (DD) or 4 (QD)");
    return DDQD_EINVAL;
}

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
