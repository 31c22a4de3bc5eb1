// lu.cu -- blocked right-looking DD/QD LU (partial pivoting, or the paper's pivot-free
// variant) and the triangular solves (north_star subsystem (5), NEXT row f1;
// PAPER.md P:121-133 steps 1-3, Eq. (2); pivoting per BJ:11).
// Op sequences: docs/numerics.md s.5. Templated on W = 2 (DD) / 4 (QD) words.
//
// Per panel of width K: a persistent cooperative kernel factors the panel (rows held in
// shared memory across all SMs, one grid barrier per column: DD/QD argmax with ties to the
// lowest row, interchange, reciprocal, column scaling, rank-1 update); when the panel does not
// fit in shared memory a per-column pair of kernels does the same steps. Interchanges of the
// columns outside the panel are applied afterwards (they commute with the panel's column
// operations). U12 is formed by a shared-memory forward substitution (one CTA per column
// strip), and the Schur update A22 := A22 - L21 U12 (the underlined term of P:131) is the
// library GEMM (Block/Strassen/Winograd) with beta = 1. Nothing returns to the host until
// the end.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "cp_async.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

#ifndef LU_CREP
#define LU_CREP 16
#endif
// replicas of the panel's per-column candidate arrays: all CTAs read all candidates right after
// the grid barrier, and one copy puts every reader on the same few L2 lines. c4 (2 runs each):
// 1 replica 56.87 / 56.88 ms, 4: 56.57 / 56.91, 8: 56.20 / 56.78, 16: 56.22 / 56.22.
// (Every warp merging all candidates itself instead of one pass per CTA made the hot spot 8x
// worse: 82.5 ms.)
constexpr int kLuCrep = LU_CREP;
// replicas of the published pivot row in the speculated-pivot panel (CTA b reads replica b % R).
// Measured on c4 (ms per solve): R = 1 41.98, 4 42.22, 8 42.99, 16 44.70 -- the owner's extra
// stores cost more than the spread reads gain, so one copy.
#ifndef LU_RREP
#define LU_RREP 1
#endif
constexpr int kLuRrep = LU_RREP;

void *aux_get(size_t bytes, int *status);   // abi.cu (separate from the GEMM workspace)

template <int W>
__device__ __forceinline__ typename elem<W>::T ldA(const double *A, int64_t n, int64_t i, int64_t j) {
    return elem<W>::load(A + i * n + j, n * n);
}
template <int W>
__device__ __forceinline__ void stA(double *A, int64_t n, int64_t i, int64_t j, const typename elem<W>::T &v) {
    elem<W>::store(A + i * n + j, n * n, v);
}
// planar shared-memory arrays: word w of entry e at s[w * stride + e]
template <int W>
__device__ __forceinline__ typename elem<W>::T lds(const double *s, int stride, int e) {
    typename elem<W>::T v;
#pragma unroll
    for (int w = 0; w < W; w++) elem<W>::set_word(v, w, s[w * stride + e]);
    return v;
}
template <int W>
__device__ __forceinline__ void sts(double *s, int stride, int e, const typename elem<W>::T &v) {
#pragma unroll
    for (int w = 0; w < W; w++) s[w * stride + e] = elem<W>::word(v, w);
}

struct LuAux {
    int info;
    int skip;
    double rinv[4];
    int miss;   // split panel: some row outranked the speculated pivot, or a zero pivot
    int pad;
};

// is candidate (a, ia) preferred over (b, ib)? larger magnitude; ties -> lower row; -1 = none
template <int W>
__device__ __forceinline__ bool cand_better(const typename elem<W>::T &a, long long ia,
                                            const typename elem<W>::T &b, long long ib) {
    if (ia < 0) return false;
    if (ib < 0) return true;
    if (elem<W>::abs_gt(a, b)) return true;
    if (elem<W>::abs_gt(b, a)) return false;
    return ia < ib;
}

template <int W>
__device__ __forceinline__ typename elem<W>::T shfl_down(const typename elem<W>::T &v, int off) {
    typename elem<W>::T r;
#pragma unroll
    for (int w = 0; w < W; w++) elem<W>::set_word(r, w, __shfl_down_sync(0xffffffffu, elem<W>::word(v, w), off));
    return r;
}

// block-wide argmax (ties -> lower row); result in slot 0 of (rv [W][32], ri); all threads call
template <int W>
__device__ __forceinline__ void block_argmax(typename elem<W>::T v, long long i, double *rv, long long *ri) {
    using T = typename elem<W>::T;
    for (int off = 16; off > 0; off >>= 1) {
        const T ov = shfl_down<W>(v, off);
        const long long oi = __shfl_down_sync(0xffffffffu, i, off);
        if (cand_better<W>(ov, oi, v, i)) { v = ov; i = oi; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();   // slots may still be read from the previous use
    if (lane == 0) { sts<W>(rv, 32, warp, v); ri[warp] = i; }
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? lds<W>(rv, 32, lane) : elem<W>::zero();
        i = lane < nw ? ri[lane] : -1;
        for (int off = 16; off > 0; off >>= 1) {
            const T ov = shfl_down<W>(v, off);
            const long long oi = __shfl_down_sync(0xffffffffu, i, off);
            if (cand_better<W>(ov, oi, v, i)) { v = ov; i = oi; }
        }
        if (lane == 0) { sts<W>(rv, 32, 0, v); ri[0] = i; }
    }
    __syncthreads();
}

// warp-wide argmax (ties -> lower row): every lane ends with the warp's winner
template <int W>
__device__ __forceinline__ void warp_argmax(typename elem<W>::T &v, long long &i) {
    using T = typename elem<W>::T;
    for (int off = 16; off > 0; off >>= 1) {
        const T ov = shfl_down<W>(v, off);
        const long long oi = __shfl_down_sync(0xffffffffu, i, off);
        if (cand_better<W>(ov, oi, v, i)) { v = ov; i = oi; }
    }
    i = __shfl_sync(0xffffffffu, i, 0);
#pragma unroll
    for (int w = 0; w < W; w++) elem<W>::set_word(v, w, __shfl_sync(0xffffffffu, elem<W>::word(v, w), 0));
}

// ---- per-column path ---------------------------------------------------------------------
// pivot row r (argmax over i >= k, or r = k without pivoting), swap rows k <-> r over all n
// columns, rinv = 1 / a_kk, a_ik := a_ik * rinv for i > k.
template <int W>
__global__ void __launch_bounds__(1024) lu_pivot_kernel(double *A, int64_t n, int64_t k, int pivot,
                                                        int64_t *ipiv, LuAux *aux) {
    using E = elem<W>;
    using T = typename E::T;
    __shared__ double rv[W * 32];
    __shared__ long long ri[32];
    __shared__ int sh_skip;
    __shared__ double sh_r[4];
    const int tid = threadIdx.x;
    int64_t r = k;
    if (pivot) {
        T best = E::zero();
        long long bidx = -1;
        for (int64_t i = k + tid; i < n; i += blockDim.x) {
            const T v = ldA<W>(A, n, i, k);
            if (cand_better<W>(v, i, best, bidx)) { best = v; bidx = i; }
        }
        block_argmax<W>(best, bidx, rv, ri);
        r = ri[0];
    }
    if (r != k) {
        for (int64_t j = tid; j < n; j += blockDim.x) {
            const T a = ldA<W>(A, n, k, j), c = ldA<W>(A, n, r, j);
            stA<W>(A, n, k, j, c);
            stA<W>(A, n, r, j, a);
        }
    }
    __syncthreads();
    if (tid == 0) {
        ipiv[k] = r;
        const T piv = ldA<W>(A, n, k, k);
        if (E::word(piv, 0) == 0.0) {
            if (aux->info == 0) aux->info = (int)(k + 1);
            sh_skip = 1;
        } else {
            const T rvv = E::div(E::one(), piv);
            for (int w = 0; w < W; w++) sh_r[w] = E::word(rvv, w);
            sh_skip = 0;
        }
        aux->skip = sh_skip;
    }
    __syncthreads();
    if (sh_skip) return;
    const T rinv = lds<W>(sh_r, 1, 0);
    for (int64_t i = k + 1 + tid; i < n; i += blockDim.x) stA<W>(A, n, i, k, E::mul(ldA<W>(A, n, i, k), rinv));
}

// a_ij := a_ij - l_ik * a_kj for i in (k, n), j in (k, jend)
template <int W>
__global__ void lu_rank1_kernel(double *A, int64_t n, int64_t k, int64_t jend, const LuAux *aux) {
    using E = elem<W>;
    if (aux->skip) return;
    const int64_t j = k + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = k + 1 + (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    if (j >= jend || i >= n) return;
    stA<W>(A, n, i, j, E::sub(ldA<W>(A, n, i, j), E::mul(ldA<W>(A, n, i, k), ldA<W>(A, n, k, j))));
}

// ---- persistent cooperative panel factorisation --------------------------------------------
// One launch per panel. CTA b owns rows [p + b*rows_per, ...) of the panel (n-p rows x kb
// columns) in shared memory. Per column: local argmax -> candidate (value, row, the row's kb
// entries) published to a double-buffered global scratch -> ONE grid barrier -> every CTA
// reduces the G candidates identically, interchanges the rows it owns, forms rinv = 1/u_kk,
// scales its column entries and does its part of the rank-1 update.
//
// Diagonal fast path (spec = 1). The pivot-free LU always takes row k; under partial
// pivoting the diagonal is SPECULATED: row k's owner publishes it, ONE grid barrier, every CTA
// takes it as the pivot row and, while scaling its rows, checks that none of them is larger in
// the DD/QD magnitude order (|a_ik| > |a_kk| for an i > k, exactly the test that makes the
// argmax -- ties to the lowest row -- pick r = k). No candidates are published or merged. A CTA
// that sees a larger entry raises the step's flag; every CTA reads step kk-1's flag after
// barrier kk (so all break at the same step), nothing is written back, the slab is reloaded
// from A and the column loop below (the full pivot search) factors the panel from the start.
// When the speculation holds, every step is the one the search would have taken (r = k, the
// pivot row = row k's values), so the factors are bit-identical either way. For BJ:11's
// c4 matrix (column diagonally dominant) it always holds.
template <int W>
__global__ void __launch_bounds__(512) lu_panel_coop_kernel(double *A, int64_t n, int64_t p, int kb,
                                                            int rows_per, int pivot, int64_t *ipiv,
                                                            LuAux *aux, double *scr, int probe, int spec,
                                                            double *fscr, const int *gate) {
    using E = elem<W>;
    using T = typename E::T;
    namespace cg = cooperative_groups;
    // gate: the split panel's miss flag -- the fallback launch runs only when the split path's
    // speculation failed (every CTA reads the same value, so all return together)
    if (gate && __ldcg(gate) == 0) return;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int G = gridDim.x;
    const int tid = threadIdx.x;
    const int SS = rows_per * kb;                 // plane stride of the slab
    double *S = sm;                               // [W][rows_per][kb]
    double *U = S + (size_t)W * SS;               // [W][kb] new row k (pivot row)
    double *L = U + (size_t)W * kb;               // [W][rows_per] multipliers of owned rows
    __shared__ double rv[W * 32];
    __shared__ long long ri[32];
    __shared__ double s_rinv[4];
    __shared__ int s_skip;

    const int64_t r0 = p + (int64_t)blockIdx.x * rows_per;
    const int64_t left = n - r0;
    const int nrows = left <= 0 ? 0 : (int)(left < rows_per ? left : rows_per);
    // scratch per buffer parity: cand value [W][G], cand idx [G], cand rows [G][W][kb], krow [W][kb]
    const size_t per_buf = (size_t)G * (W + 1) * kLuCrep + (size_t)G * W * kb + (size_t)W * kb;

    if (spec != 2) {   // (the split-barrier fast path loads its own, cyclic, layout)
        for (int e = tid; e < nrows * kb; e += blockDim.x) {
            const int li = e / kb, j = e % kb;
            sts<W>(S, SS, e, ldA<W>(A, n, r0 + li, p + j));
        }
        __syncthreads();
    }

    if (spec == 2) {
        // Split-barrier form of the fast path, rows dealt CYCLICALLY (CTA b owns panel rows
        // p + b + G*li), so successive pivot rows belong to successive CTAs: the owner of row
        // k+1 scales and updates that row FIRST in step k, publishes it with its reciprocal and
        // arrives at barrier k+1; every other CTA arrives as soon as it has read row k, and then
        // scales and rank-1-updates its rows while the barrier completes. Step k's verification
        // flags are read after barrier k+2 (raised before the detector arrives there), so every
        // CTA breaks at the same step. The fallback reloads the slab in the block layout below.
        // fscr: [2][R][W][kb + 1] pivot rows (+ reciprocal in slot kb) | flags [kb] | counter
        const int RS = kb + 1;
        int *flag = reinterpret_cast<int *>(fscr + (size_t)2 * kLuRrep * W * RS);
        unsigned *ctr = reinterpret_cast<unsigned *>(flag + kb);
        const int64_t R = n - p;
        const int b = blockIdx.x;
        const int cr = b < R ? (int)((R - b + G - 1) / G) : 0;      // rows of this CTA (<= rows_per)
        auto grow = [&](int li) { return p + b + (int64_t)G * li; };
        for (int e = tid; e < cr * kb; e += blockDim.x) {
            const int li = e / kb, j = e % kb;
            sts<W>(S, SS, e, ldA<W>(A, n, grow(li), p + j));
        }
        auto publish = [&](int kk1, int li) {
            // (warp 0) row p+kk1, local row li, and its reciprocal -> every replica of the
            // pivot-row buffer (columns < kk1 are never read)
            double *kr = fscr + (size_t)(kk1 & 1) * kLuRrep * W * RS;
            for (int j = kk1 + tid; j < kb; j += 32)
                for (int w = 0; w < W; w++) {
                    const double v = S[w * SS + li * kb + j];
                    for (int q = 0; q < kLuRrep; q++) kr[((size_t)q * W + w) * RS + j] = v;
                }
            if (tid == 0) {
                const T d = lds<W>(S, SS, li * kb + kk1);
                const T rv2 = (E::word(d, 0) == 0.0) ? E::zero() : E::div(E::one(), d);
                for (int q = 0; q < kLuRrep; q++)
                    for (int w = 0; w < W; w++) kr[((size_t)q * W + w) * RS + kb] = E::word(rv2, w);
            }
        };
        if (blockIdx.x == 0) {
            for (int j = tid; j < kb; j += blockDim.x) flag[j] = 0;
            if (tid == 0) *ctr = 0u;
        }
        __syncthreads();
        if (tid < 32 && b == 0 && cr > 0) publish(0, 0);     // row p: CTA 0, local row 0
        grid.sync();   // flags and counter reset, row p published
        long long zero_k = -1;
        bool failed = false;
        long long q[6] = {0, 0, 0, 0, 0, 0};
        long long qt = clock64();
        auto qmark = [&](int ph) {   // DDQD_LU_PROBE: per-phase cycles of this path
            if (probe) { __syncthreads(); const long long t = clock64(); q[ph] += t - qt; qt = t; }
        };
        for (int kk = 0; kk < kb; kk++) {
            const int64_t k = p + kk;
            qmark(5);
            if (kk > 0 && tid == 0) {
                const unsigned target = (unsigned)G * (unsigned)kk;
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                } while (v < target);
            }
            __syncthreads();
            qmark(0);
            if (pivot && kk >= 2 && __ldcg(flag + kk - 2)) { failed = true; break; }
            const double *kr = fscr + ((size_t)(kk & 1) * kLuRrep + (b % kLuRrep)) * W * RS;
            for (int j = kk + tid; j < kb; j += blockDim.x)   // columns < kk are never read
                for (int w = 0; w < W; w++) U[w * kb + j] = __ldcg(kr + (size_t)w * RS + j);
            if (tid < W) s_rinv[tid] = __ldcg(kr + (size_t)tid * RS + kb);
            __syncthreads();
            qmark(1);
            const T akk = lds<W>(U, kb, kk);
            const bool skip = E::word(akk, 0) == 0.0;
            if (tid == 0) {
                if (blockIdx.x == 0) ipiv[k] = k;
                if (skip && zero_k < 0) zero_k = k;
            }
            const T rinv = lds<W>(s_rinv, 1, 0);
            // first owned row below k, and the owner of row k+1 (local li1)
            const int64_t dk = k - p - b;
            const int li0 = dk < 0 ? 0 : (int)(dk / G) + 1;
            const int li1 = (kk + 1 < kb && (kk + 1) % G == b) ? (kk + 1) / G : -1;
            // warp 0 arrives at barrier kk+1 as soon as the CTA has read row k (the barrier after
            // the fetch) -- after publishing row k+1 when this CTA owns it; the other warps go
            // straight on to the scaling and the update. The release fence orders this CTA's
            // reads of row k, its flags of step kk-1 and the published row before the arrival.
            // Only the owner's arrival publishes data (row k+1), so only it needs the release
            // fence; the others signal "row k has been read" (their loads have returned), and a
            // raised flag carries its own fence where it is raised (the rare miss path).
            auto arrive = [&](bool release) {
                __syncwarp();
                if (tid == 0) {
                    if (release) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    atomicAdd(ctr, 1u);
                }
            };
            if (tid < 32 && li1 < 0) arrive(false);
            if (li1 >= 0 && tid < 32) {
                const T a = lds<W>(S, SS, li1 * kb + kk);
                if (!skip) {
                    if (pivot && tid == 0 && E::abs_gt(a, akk)) { flag[kk] = 1; __threadfence(); }
                    const T lv = E::mul(a, rinv);
                    for (int j = kk + 1 + tid; j < kb; j += 32)
                        sts<W>(S, SS, li1 * kb + j, E::sub(lds<W>(S, SS, li1 * kb + j), E::mul(lv, lds<W>(U, kb, j))));
                    __syncwarp();
                    if (tid == 0) { sts<W>(S, SS, li1 * kb + kk, lv); sts<W>(L, rows_per, li1, lv); }
                    __syncwarp();
                } else if (pivot && tid == 0 && E::abs_gt(a, akk)) {
                    flag[kk] = 1;
                }
                publish(kk + 1, li1);
                arrive(true);
            }
            qmark(2);
            bool bigger = false;
            // the scaling starts at warp 1, so warp 0's arrival / owner work runs beside it
            const int ts = (tid + (int)blockDim.x - 32) % (int)blockDim.x;
            if (skip) {
                if (pivot)
                    for (int li = li0 + ts; li < cr; li += blockDim.x)
                        if (li != li1 && E::abs_gt(lds<W>(S, SS, li * kb + kk), akk)) bigger = true;
                if (bigger) { flag[kk] = 1; __threadfence(); }
                continue;
            }
            for (int li = li0 + ts; li < cr; li += blockDim.x) {
                if (li == li1) continue;
                const T a = lds<W>(S, SS, li * kb + kk);
                if (pivot && E::abs_gt(a, akk)) bigger = true;
                const T lv = E::mul(a, rinv);
                sts<W>(S, SS, li * kb + kk, lv);
                sts<W>(L, rows_per, li, lv);
            }
            if (bigger) { flag[kk] = 1; __threadfence(); }
            __syncthreads();
            qmark(3);
            {
                // rows in pairs, both loaded before either is stored: two independent DD chains
                // per thread (the loop is latency-bound at one CTA per SM)
                const int nwarp = blockDim.x >> 5, lane = tid & 31, wrp = tid >> 5;
                for (int j = kk + 1 + lane; j < kb; j += 32) {
                    const T u = lds<W>(U, kb, j);
                    int li = li0 + wrp;
                    for (; li + nwarp < cr; li += 2 * nwarp) {
                        const int lb = li + nwarp;
                        const T a0 = lds<W>(S, SS, li * kb + j), a1 = lds<W>(S, SS, lb * kb + j);
                        const T l0 = lds<W>(L, rows_per, li), l1 = lds<W>(L, rows_per, lb);
                        const T r0v = E::sub(a0, E::mul(l0, u)), r1v = E::sub(a1, E::mul(l1, u));
                        if (li != li1) sts<W>(S, SS, li * kb + j, r0v);
                        if (lb != li1) sts<W>(S, SS, lb * kb + j, r1v);
                    }
                    if (li < cr && li != li1)
                        sts<W>(S, SS, li * kb + j, E::sub(lds<W>(S, SS, li * kb + j), E::mul(lds<W>(L, rows_per, li), u)));
                }
            }
            __syncthreads();
        }
        if (probe && tid == 0 && (blockIdx.x == 0 || blockIdx.x == 1 || blockIdx.x == G / 2))
            printf("LUPROBE2 p=%lld G=%d cta=%d wait %lld fetch %lld owner+arrive %lld scale %lld update %lld\n",
                   (long long)p, G, blockIdx.x, q[0], q[1], q[2], q[3], q[5]);
        grid.sync();
        if (pivot && !failed && (__ldcg(flag + kb - 1) || (kb >= 2 && __ldcg(flag + kb - 2)))) failed = true;
        if (!failed) {
            if (blockIdx.x == 0 && tid == 0 && zero_k >= 0 && aux->info == 0) aux->info = (int)(zero_k + 1);
            for (int e = tid; e < cr * kb; e += blockDim.x) {
                const int li = e / kb, j = e % kb;
                stA<W>(A, n, grow(li), p + j, lds<W>(S, SS, e));
            }
            return;
        }
        for (int e = tid; e < nrows * kb; e += blockDim.x) {
            const int li = e / kb, j = e % kb;
            sts<W>(S, SS, e, ldA<W>(A, n, r0 + li, p + j));
        }
        __syncthreads();
    } else if (spec == 1) {
        // fscr: pivot rows [2][W][kb] (double-buffered by step parity) | per-step flags [kb]
        int *flag = reinterpret_cast<int *>(fscr + (size_t)2 * W * kb);
        if (blockIdx.x == 0)
            for (int j = tid; j < kb; j += blockDim.x) flag[j] = 0;
        long long zero_k = -1;               // first exactly-zero pivot (CTA-uniform)
        bool failed = false;
        for (int kk = 0; kk < kb; kk++) {
            const int64_t k = p + kk;
            double *krow = fscr + (size_t)(kk & 1) * W * kb;
            const bool own_k = k >= r0 && k < r0 + nrows;
            if (own_k) {
                const int li = (int)(k - r0);
                for (int j = tid; j < kb; j += blockDim.x)
                    for (int w = 0; w < W; w++) krow[(size_t)w * kb + j] = S[w * SS + li * kb + j];
            }
            grid.sync();
            if (pivot && kk > 0 && *reinterpret_cast<volatile int *>(flag + kk - 1)) { failed = true; break; }
            for (int j = tid; j < kb; j += blockDim.x)
                for (int w = 0; w < W; w++) U[w * kb + j] = __ldcg(krow + (size_t)w * kb + j);
            __syncthreads();
            if (tid == 0) {
                const T piv = lds<W>(U, kb, kk);
                if (blockIdx.x == 0) ipiv[k] = k;
                if (E::word(piv, 0) == 0.0) {
                    s_skip = 1;
                    if (zero_k < 0) zero_k = k;
                } else {
                    const T rvv = E::div(E::one(), piv);
                    for (int w = 0; w < W; w++) s_rinv[w] = E::word(rvv, w);
                    s_skip = 0;
                }
            }
            __syncthreads();
            const T akk = lds<W>(U, kb, kk);
            bool bigger = false;             // an owned row below k outranks the diagonal
            if (s_skip) {
                if (pivot)
                    for (int li = tid; li < nrows; li += blockDim.x)
                        if (r0 + li > k && E::abs_gt(lds<W>(S, SS, li * kb + kk), akk)) bigger = true;
                if (bigger) flag[kk] = 1;
                continue;
            }
            const T rinv = lds<W>(s_rinv, 1, 0);
            for (int li = tid; li < nrows; li += blockDim.x) {
                if (r0 + li <= k) continue;
                const T a = lds<W>(S, SS, li * kb + kk);
                if (pivot && E::abs_gt(a, akk)) bigger = true;
                const T lv = E::mul(a, rinv);
                sts<W>(S, SS, li * kb + kk, lv);
                sts<W>(L, rows_per, li, lv);
            }
            if (bigger) flag[kk] = 1;
            __syncthreads();
            {
                const int64_t first = k + 1 - r0;
                const int li0 = first <= 0 ? 0 : (first >= nrows ? nrows : (int)first);
                const int nwarp = blockDim.x >> 5, lane = tid & 31, wrp = tid >> 5;
                for (int j = kk + 1 + lane; j < kb; j += 32) {
                    const T u = lds<W>(U, kb, j);
                    for (int li = li0 + wrp; li < nrows; li += nwarp) {
                        const T a = lds<W>(S, SS, li * kb + j);
                        sts<W>(S, SS, li * kb + j, E::sub(a, E::mul(lds<W>(L, rows_per, li), u)));
                    }
                }
            }
            __syncthreads();
        }
        grid.sync();
        if (pivot && !failed && *reinterpret_cast<volatile int *>(flag + kb - 1)) failed = true;
        if (!failed) {
            if (blockIdx.x == 0 && tid == 0 && zero_k >= 0 && aux->info == 0) aux->info = (int)(zero_k + 1);
            for (int e = tid; e < nrows * kb; e += blockDim.x) {
                const int li = e / kb, j = e % kb;
                stA<W>(A, n, r0 + li, p + j, lds<W>(S, SS, e));
            }
            return;
        }
        // the speculation failed: A still holds the panel; factor it with the pivot search
        for (int e = tid; e < nrows * kb; e += blockDim.x) {
            const int li = e / kb, j = e % kb;
            sts<W>(S, SS, e, ldA<W>(A, n, r0 + li, p + j));
        }
        __syncthreads();
    }

    long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
    auto mark = [&](int ph) {   // DDQD_LU_PROBE timing (CTA 0 and G-1 report per-phase cycles)
        if (probe) {
            __syncthreads();
            const long long t = clock64();
            tph[ph] += t - tlast;
            tlast = t;
        }
    };
    for (int kk = 0; kk < kb; kk++) {
        const int64_t k = p + kk;
        mark(7);
        double *buf = scr + (size_t)(kk & 1) * per_buf;
        // kLuCrep replicas of the candidate arrays ([W][G] values, [G] rows each); CTA b reads
        // replica b % kLuCrep, so the 148 readers of a column spread over kLuCrep x the lines
        double *cand_v = buf + (size_t)(blockIdx.x % kLuCrep) * G * (W + 1);
        long long *cand_i = reinterpret_cast<long long *>(cand_v + (size_t)W * G);
        auto put_cand = [&](int q, const T &v, long long i) {
            double *cv = buf + (size_t)q * G * (W + 1);
            for (int w = 0; w < W; w++) cv[(size_t)w * G + blockIdx.x] = E::word(v, w);
            reinterpret_cast<long long *>(cv + (size_t)W * G)[blockIdx.x] = i;
        };
        double *cand_rows = buf + (size_t)(W + 1) * G * kLuCrep;         // [G][W][kb]
        double *krow = cand_rows + (size_t)G * W * kb;                   // [W][kb]

        // 1. local candidate of column kk over owned rows >= k (row k only without pivoting);
        // one warp suffices when the CTA owns <= 32 rows (one shared-memory barrier)
        long long lbi;
        if (nrows <= 32) {
            if (tid < 32) {
                T best = E::zero();
                long long bi = -1;
                if (tid < nrows) {
                    const int64_t gi = r0 + tid;
                    if (gi >= k && (pivot || gi == k)) { best = lds<W>(S, SS, tid * kb + kk); bi = gi; }
                }
                warp_argmax<W>(best, bi);
                if (tid < kLuCrep) put_cand(tid, best, bi);
                if (tid == 0) ri[0] = bi;
            }
            __syncthreads();
            lbi = ri[0];
        } else {
            T best = E::zero();
            long long bi = -1;
            for (int li = tid; li < nrows; li += blockDim.x) {
                const int64_t gi = r0 + li;
                if (gi < k || (!pivot && gi != k)) continue;
                const T v = lds<W>(S, SS, li * kb + kk);
                if (cand_better<W>(v, gi, best, bi)) { best = v; bi = gi; }
            }
            block_argmax<W>(best, bi, rv, ri);
            lbi = ri[0];
            if (tid < kLuCrep) put_cand(tid, lds<W>(rv, 32, 0), lbi);
        }
        if (lbi >= 0) {
            const int li = (int)(lbi - r0);
            for (int j = tid; j < kb; j += blockDim.x)
                for (int w = 0; w < W; w++) cand_rows[((size_t)blockIdx.x * W + w) * kb + j] = S[w * SS + li * kb + j];
        }
        const bool own_k = k >= r0 && k < r0 + nrows;
        if (own_k) {
            const int li = (int)(k - r0);
            for (int j = tid; j < kb; j += blockDim.x)
                for (int w = 0; w < W; w++) krow[(size_t)w * kb + j] = S[w * SS + li * kb + j];
        }
        mark(0);
        grid.sync();   // grid-wide barrier with memory ordering (bar.sync + fenced arrive)
        mark(1);

        // 2. global pivot, identical in every CTA; the winning CTA follows from the row index
        {
            T v = E::zero();
            long long i = -1;
            for (int g = tid; g < G; g += blockDim.x) {
                T cv;
                for (int w = 0; w < W; w++) E::set_word(cv, w, __ldcg(cand_v + (size_t)w * G + g));
                const long long ci = __ldcg(cand_i + g);
                if (cand_better<W>(cv, ci, v, i)) { v = cv; i = ci; }
            }
            warp_argmax<W>(v, i);
            const int warp = tid >> 5, nw = blockDim.x >> 5;
            if ((tid & 31) == 0) { sts<W>(rv, 32, warp, v); ri[warp] = i; }
            __syncthreads();
            // every warp merges the nw per-warp winners itself (no second barrier)
            v = (tid & 31) < nw ? lds<W>(rv, 32, tid & 31) : E::zero();
            i = (tid & 31) < nw ? ri[tid & 31] : -1;
            warp_argmax<W>(v, i);
            if (tid == 0) ri[0] = i;   // read below only after the next barrier
            __syncthreads();
        }
        mark(2);
        const int64_t r = ri[0];
        const int wc = (int)((r - p) / rows_per);
        const double *prow = cand_rows + (size_t)wc * W * kb;
        for (int j = tid; j < kb; j += blockDim.x)
            for (int w = 0; w < W; w++) U[w * kb + j] = __ldcg(prow + (size_t)w * kb + j);
        __syncthreads();
        mark(3);
        if (r != k) {
            if (own_k) {
                const int li = (int)(k - r0);
                for (int j = tid; j < kb; j += blockDim.x)
                    for (int w = 0; w < W; w++) S[w * SS + li * kb + j] = U[w * kb + j];
            }
            if (r >= r0 && r < r0 + nrows) {
                const int li = (int)(r - r0);
                for (int j = tid; j < kb; j += blockDim.x)
                    for (int w = 0; w < W; w++) S[w * SS + li * kb + j] = __ldcg(krow + (size_t)w * kb + j);
            }
        }
        if (tid == 0) {
            const T piv = lds<W>(U, kb, kk);
            if (blockIdx.x == 0) ipiv[k] = r;
            if (E::word(piv, 0) == 0.0) {
                s_skip = 1;
                if (blockIdx.x == 0 && aux->info == 0) aux->info = (int)(k + 1);
            } else {
                const T rvv = E::div(E::one(), piv);
                for (int w = 0; w < W; w++) s_rinv[w] = E::word(rvv, w);
                s_skip = 0;
            }
        }
        __syncthreads();
        mark(4);
        if (s_skip) continue;
        // 3. l_ik = a_ik * rinv for owned rows i > k
        const T rinv = lds<W>(s_rinv, 1, 0);
        for (int li = tid; li < nrows; li += blockDim.x) {
            if (r0 + li <= k) continue;
            const T lv = E::mul(lds<W>(S, SS, li * kb + kk), rinv);
            sts<W>(S, SS, li * kb + kk, lv);
            sts<W>(L, rows_per, li, lv);
        }
        __syncthreads();
        mark(5);
        // 4. rank-1 update a_ij -= l_ik u_kj, j in (kk, kb): thread per column, owned active rows
        {
            const int64_t first = k + 1 - r0;                 // first owned row below k
            const int li0 = first <= 0 ? 0 : (first >= nrows ? nrows : (int)first);
            // warps take row groups, lanes take columns: every warp stays busy, no division
            const int nwarp = blockDim.x >> 5, lane = tid & 31, wrp = tid >> 5;
            for (int j = kk + 1 + lane; j < kb; j += 32) {
                const T u = lds<W>(U, kb, j);
                for (int li = li0 + wrp; li < nrows; li += nwarp) {
                    const T a = lds<W>(S, SS, li * kb + j);
                    sts<W>(S, SS, li * kb + j, E::sub(a, E::mul(lds<W>(L, rows_per, li), u)));
                }
            }
        }
        __syncthreads();
        mark(6);
    }
    if (probe && tid == 0 && (p == 0 || blockIdx.x == 0 || blockIdx.x == G - 1))
        printf("LUPROBE p=%lld G=%d rows=%d cta=%d publish %lld sync %lld cand %lld prow %lld swap %lld scale %lld update %lld\n",
               (long long)p, G, rows_per, blockIdx.x, tph[0], tph[1], tph[2], tph[3], tph[4], tph[5], tph[6]);
    for (int e = tid; e < nrows * kb; e += blockDim.x) {
        const int li = e / kb, j = e % kb;
        stA<W>(A, n, r0 + li, p + j, lds<W>(S, SS, e));
    }
}

// ---- blocked speculated panel: 64-column sub-panels, no grid-wide barrier -----------------------
// The speculated-pivot panel (r = k at every step, verified) as a blocked LU of the panel itself.
// With the pivot rows known in advance, sub-panel q (columns [p0, p0 + w), w <= 64) splits into
//  D. its w x w diagonal block: the sequential part, ONE CTA with the block in shared memory
//     (two CTA barriers per column, no cross-SM traffic);
//  B. the rows below it, columns [p0, p0 + w): each row needs only D's U rows, so warps
//     eliminate their own rows column by column (lanes hold columns, the multiplier is
//     broadcast with shuffles);
//  T. the block's rows right of it: U12 := L11^-1 A12 (the warp TRSM kernel, column-parallel);
//  G. the rows below x the columns right: a_ij := a_ij - l_ik u_kj for k = p0 .. p0+w-1 in order.
// Every element receives exactly the operations of the right-looking column steps
// (l_ik = a_ik * (1 / u_kk), a_ij := a_ij - l_ik * u_kj, k ascending), so the factors are the
// bits of the cooperative kernel and the oracle when the speculation holds. At column k every
// row below checks that it does not outrank u_kk in the DD/QD magnitude order (the test that
// makes the argmax pick row k); a zero pivot also counts as a miss. The panel is snapshotted
// first; after a miss the later kernels return at once, the snapshot is restored and the gated
// cooperative kernel factors the panel with the full pivot search.
constexpr int kSubSB = 32;     // sub-panel width
constexpr int kSubDiagPad = 180 * 1024;   // D's SM to itself (see the launch)
constexpr int kSubDiagNT = 384; // 12 warps: the chain warp 0 alone on SM sub-partition 0, 9 bulk warps on 1-3

// D: the w x w (w <= 32) diagonal block of sub-panel [p0, p0 + w). Warp 0 (the chain warp) owns
// row kk+1 in step kk: it scales it, updates it and forms the next reciprocal 1/u_{kk+1,kk+1}
// (the dependent chain mul -> sub(mul) -> div of every column) while 9 bulk warps update rows
// kk+2.. (bulk warp b: rows kk+2+b+9t; lane: column kk+1+lane); one CTA barrier per column.
// Warps 4 and 8 idle: the chain warp has SM sub-partition 0 (warp % 4) to itself, so its
// dependent chain is not queued behind the bulk warps' FP64 instructions (measured: the chain
// took ~1.1k cycles per column sharing its sub-partition with two bulk warps).
template <int W>
__global__ void __launch_bounds__(kSubDiagNT, 1) lu_subdiag_kernel(double *A, int64_t n, int64_t p0, int w, int pivot,
                                                                   int *miss, double *rv_out, int probe) {
    using E = elem<W>;
    using T = typename E::T;
    if (__ldcg(miss)) return;
    constexpr int SB = kSubSB, SS = SB * SB, NT = kSubDiagNT;
    __shared__ double S[W * SS];        // [W][SB][SB]
    __shared__ double s_r[2 * 4];       // 1 / u_kk, by step parity
    const int tid = threadIdx.x, lane = tid & 31, wr = tid >> 5;
    {
        T v[(SS + NT - 1) / NT];
#pragma unroll
        for (int it = 0; it < (SS + NT - 1) / NT; it++) {
            const int e = tid + NT * it, i = e / SB, j = e % SB;
            v[it] = (e < SS && i < w && j < w) ? ldA<W>(A, n, p0 + i, p0 + j) : E::zero();
        }
#pragma unroll
        for (int it = 0; it < (SS + NT - 1) / NT; it++)
            if (tid + NT * it < SS) sts<W>(S, SS, tid + NT * it, v[it]);
    }
    __syncthreads();
    if (tid == 0) sts<W>(s_r, 1, 0, E::div(E::one(), lds<W>(S, SS, 0)));
    __syncthreads();
    bool bad = false;
    long long pc0 = 0, pc1 = 0, pc2 = 0, tst = clock64();
    const long long t_start = tst;
    for (int kk = 0; kk < w; kk++) {
        if (probe) { const long long t = clock64(); pc2 += t - tst; tst = t; }
        const T akk = lds<W>(S, SS, kk * SB + kk);
        const T rinv = lds<W>(s_r + (kk & 1) * W, 1, 0);
        if (tid == 0) {
            if (E::word(akk, 0) == 0.0) bad = true;
            for (int ww = 0; ww < W; ww++) rv_out[ww * SB + kk] = E::word(rinv, ww);   // for B
        }
        const int j = kk + 1 + lane;
        const int bw = (wr >> 2) * 3 + (wr & 3) - 1;   // bulk warp index 0..8 (wr % 4 != 0)
        if (wr == 0) {
            const int i = kk + 1;
            if (i < w) {
                const T a = lds<W>(S, SS, i * SB + kk);
                if (pivot && lane == 0 && E::abs_gt(a, akk)) bad = true;
                const T lv = E::mul(a, rinv);
                if (j < w) {
                    const T v = E::sub(lds<W>(S, SS, i * SB + j), E::mul(lv, lds<W>(S, SS, kk * SB + j)));
                    sts<W>(S, SS, i * SB + j, v);
                    if (lane == 0) sts<W>(s_r + ((kk + 1) & 1) * W, 1, 0, E::div(E::one(), v));
                }
                __syncwarp();
                if (lane == 0) sts<W>(S, SS, i * SB + kk, lv);
            }
            if (probe) { const long long t = clock64(); pc0 += t - tst; }
        } else if ((wr & 3) != 0 && kk + 2 + bw < w) {
            // this warp's rows kk+2+bw+9t (t < nr, warp-uniform count): the nr chains issued
            // together (no branch between them), so only valid rows cost FP64 issue slots
            const int nr = (w - (kk + 2 + bw) + 8) / 9;
            const int jc = j < w ? j : kk;
            const T u = lds<W>(S, SS, kk * SB + jc);
            auto rows_go = [&](auto NRc) {
                constexpr int NR = decltype(NRc)::value;
                T lv[NR], nv[NR];
#pragma unroll
                for (int t = 0; t < NR; t++) {
                    const int i = kk + 2 + bw + 9 * t;
                    const T a = lds<W>(S, SS, i * SB + kk);
                    if (pivot && lane == 0 && E::abs_gt(a, akk)) bad = true;
                    lv[t] = E::mul(a, rinv);
                    nv[t] = E::sub(lds<W>(S, SS, i * SB + jc), E::mul(lv[t], u));
                }
                if (j < w)
#pragma unroll
                    for (int t = 0; t < NR; t++) sts<W>(S, SS, (kk + 2 + bw + 9 * t) * SB + j, nv[t]);
                __syncwarp();
                if (lane == 0)
#pragma unroll
                    for (int t = 0; t < NR; t++) sts<W>(S, SS, (kk + 2 + bw + 9 * t) * SB + kk, lv[t]);
            };
            if (nr >= 4) rows_go(std::integral_constant<int, 4>{});
            else if (nr == 3) rows_go(std::integral_constant<int, 3>{});
            else if (nr == 2) rows_go(std::integral_constant<int, 2>{});
            else rows_go(std::integral_constant<int, 1>{});
            if (probe) { const long long t = clock64(); pc1 += t - tst; }
        }
        __syncthreads();
    }
    if (probe && (tid == 0 || tid == 32) && p0 < 64)
        printf("LUSUBPROBE p0=%lld tid=%d chain %lld bulk %lld step %lld total %lld\n", (long long)p0, tid, pc0, pc1, pc2,
               clock64() - t_start);
    for (int e = tid; e < w * w; e += NT) {
        const int i = e / w, jj = e % w;
        stA<W>(A, n, p0 + i, p0 + jj, lds<W>(S, SS, i * SB + jj));
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(miss, 1);
}

#ifndef LU_BELOW_TPR
#define LU_BELOW_TPR 8   // c4: 35.78 ms vs 35.92 with 4 threads per row (4 columns per thread)
#endif
template <int W> struct SubBelow {
    static constexpr int TPR = LU_BELOW_TPR;       // threads per row
    static constexpr int NT = 128;                 // 4 warps: one per SM sub-partition
    static constexpr int ROWS = NT / TPR;          // rows per CTA
};

// B: rows [r0, r0 + rows) x columns [p0, p0 + w): column elimination with the U rows and
// reciprocals of the sub-panel's diagonal block (U staged in shared memory, the reciprocals
// from D). TPR threads per row, thread t holding columns t + TPR c in registers: the
// column loop is unrolled, so at step k a thread only issues the slots that still have
// columns > k (no idle lanes beyond the partial slot), and the multiplier's source a_ik is one
// shuffle inside the row's TPR-lane group.
template <int W>
__global__ void __launch_bounds__(SubBelow<W>::NT) lu_subbelow_kernel(double *A, int64_t n, int64_t p0, int w,
                                                                      int pivot, int *miss, int64_t r0,
                                                                      int64_t rows, const double *rv_in, int probe) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int SB = kSubSB, SS = SB * SB, TPR = SubBelow<W>::TPR, NC = SB / TPR, NT = SubBelow<W>::NT;
    const long long tb0 = clock64();
    if (__ldcg(miss)) return;
    __shared__ double U[W * SS];        // [W][SB][SB]
    __shared__ double Rv[W * SB];       // [W][SB]
    const int tid = threadIdx.x, lane = tid & 31, t = tid % TPR;
    {
        T v[SS / NT];
#pragma unroll
        for (int it = 0; it < SS / NT; it++) {
            const int e = tid + NT * it, i = e / SB, j = e % SB;
            v[it] = (j >= i && i < w && j < w) ? ldA<W>(A, n, p0 + i, p0 + j) : E::zero();
        }
#pragma unroll
        for (int it = 0; it < SS / NT; it++) sts<W>(U, SS, tid + NT * it, v[it]);
    }
    if (tid < W * SB) Rv[tid] = rv_in[tid];   // D's reciprocals 1 / u_kk (the same bits)
    const int64_t i = r0 + (int64_t)blockIdx.x * SubBelow<W>::ROWS + tid / TPR;
    const bool valid = i < r0 + rows;
    T acc[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const int j = t + TPR * c;
        acc[c] = (valid && j < w) ? ldA<W>(A, n, i, p0 + j) : E::zero();
    }
    __syncthreads();
    const long long tb1 = clock64();
    bool bad = false;
    const int gl = lane & ~(TPR - 1);
#pragma unroll
    for (int k = 0; k < SB; k++) {
        if (k >= w) break;
        const int ck = k / TPR, tk = k % TPR;
        T a;
#pragma unroll
        for (int ww = 0; ww < W; ww++) E::set_word(a, ww, __shfl_sync(0xffffffffu, E::word(acc[ck], ww), gl | tk));
        const T ukk = lds<W>(U, SS, k * SB + k);
        if (pivot && valid && E::abs_gt(a, ukk)) bad = true;
        const T lv = E::mul(a, lds<W>(Rv, SB, k));
        // branch-free (selects, not branches), so the slots' chains interleave; U is zero past w
        {
            const int j = t + TPR * ck;
            const T nv = E::sub(acc[ck], E::mul(lv, lds<W>(U, SS, k * SB + j)));
            acc[ck] = t == tk ? lv : ((t > tk && j < w) ? nv : acc[ck]);
        }
#pragma unroll
        for (int c = ck + 1; c < NC; c++) {
            const int j = t + TPR * c;
            const T nv = E::sub(acc[c], E::mul(lv, lds<W>(U, SS, k * SB + j)));
            acc[c] = j < w ? nv : acc[c];
        }
    }
    const long long tb2 = clock64();
    if (valid)
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const int j = t + TPR * c;
            if (j < w) stA<W>(A, n, i, p0 + j, acc[c]);
        }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(miss, 1);
    if (probe && tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2) && p0 < 64)
        printf("LUBELOWPROBE p0=%lld cta=%d grid=%d prologue %lld steps %lld\n", (long long)p0, blockIdx.x, gridDim.x,
               tb1 - tb0, tb2 - tb1);
}

// G: rows [r0, r0 + rows) x columns [c0, c0 + cols): a_ij := a_ij - l_ik u_kj for
// k = p0 .. p0+w-1 ascending (w <= 32; l from columns [p0, p0 + w), u from rows [p0, p0 + w));
// 32 x 32 tiles, 128 threads with 2 x 4 outputs each
template <int W>
__global__ void __launch_bounds__(128) lu_subgemm_kernel(double *A, int64_t n, int64_t p0, int w, int64_t r0,
                                                         int64_t rows, int64_t c0, int64_t cols, const int *miss) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int BM = 32, BN = 32, BK = kSubSB, LDL = BK + 1;
    if (miss && __ldcg(miss)) return;
    extern __shared__ double sm[];
    double *Ls = sm;                      // [W][BM][LDL]
    double *Us = sm + W * BM * LDL;       // [W][BK][BN]
    const int tid = threadIdx.x, tx = tid % 8, ty = tid / 8;
    const int64_t i0 = r0 + (int64_t)blockIdx.y * BM, j0 = c0 + (int64_t)blockIdx.x * BN;
    // compile-time trip counts: every load of the two tiles is in flight at once (the small
    // grids of the next sub-panel's rows, Ga, sit on the critical path)
    {
        T lt[BM * BK / 128], ut[BK * BN / 128];
#pragma unroll
        for (int it = 0; it < BM * BK / 128; it++) {
            const int e = tid + 128 * it, r = e / BK, k = e % BK;
            const int64_t i = i0 + r;
            lt[it] = (i < r0 + rows && k < w) ? ldA<W>(A, n, i, p0 + k) : E::zero();
        }
#pragma unroll
        for (int it = 0; it < BK * BN / 128; it++) {
            const int e = tid + 128 * it, k = e / BN, c = e % BN;
            const int64_t j = j0 + c;
            ut[it] = (j < c0 + cols && k < w) ? ldA<W>(A, n, p0 + k, j) : E::zero();
        }
#pragma unroll
        for (int it = 0; it < BM * BK / 128; it++) {
            const int e = tid + 128 * it;
            sts<W>(Ls, BM * LDL, (e / BK) * LDL + e % BK, lt[it]);
        }
#pragma unroll
        for (int it = 0; it < BK * BN / 128; it++) sts<W>(Us, BK * BN, tid + 128 * it, ut[it]);
    }
    T acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int64_t i = i0 + ty + 16 * a, j = j0 + tx + 8 * b;
            acc[a][b] = (i < r0 + rows && j < c0 + cols) ? ldA<W>(A, n, i, j) : E::zero();
        }
    __syncthreads();
    for (int k = 0; k < w; k++) {
        T lv[2], uv[4];
#pragma unroll
        for (int a = 0; a < 2; a++) lv[a] = lds<W>(Ls, BM * LDL, (ty + 16 * a) * LDL + k);
#pragma unroll
        for (int b = 0; b < 4; b++) uv[b] = lds<W>(Us, BK * BN, k * BN + tx + 8 * b);
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) acc[a][b] = E::sub(acc[a][b], E::mul(lv[a], uv[b]));
    }
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int64_t i = i0 + ty + 16 * a, j = j0 + tx + 8 * b;
            if (i < r0 + rows && j < c0 + cols) stA<W>(A, n, i, j, acc[a][b]);
        }
}

// Ga (the next sub-panel's 32 rows: a short grid on the pivot chain): 8 x 8 tiles of 64 threads,
// ONE output per thread, so each thread's 32-step chain is latency- not issue-bound and the
// grid spreads over ~4x as many SMs as the 32 x 32 tiles (measured 13.5 us per Ga with those).
template <int W>
__global__ void __launch_bounds__(64) lu_subgemm_small_kernel(double *A, int64_t n, int64_t p0, int w, int64_t r0,
                                                              int64_t rows, int64_t c0, int64_t cols,
                                                              const int *miss) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int BK = kSubSB, LDL = BK + 1;
    if (miss && __ldcg(miss)) return;
    __shared__ double Ls[W * 8 * LDL];
    __shared__ double Us[W * BK * 8];
    const int tid = threadIdx.x, tx = tid % 8, ty = tid / 8;
    const int64_t i0 = r0 + (int64_t)blockIdx.y * 8, j0 = c0 + (int64_t)blockIdx.x * 8;
    T lt[4], ut[4];
#pragma unroll
    for (int it = 0; it < 4; it++) {
        const int e = tid + 64 * it;   // 256 = 8 rows x 32 k  /  32 k x 8 cols
        const int r = e / BK, k = e % BK, kk = e / 8, c = e % 8;
        lt[it] = (i0 + r < r0 + rows && k < w) ? ldA<W>(A, n, i0 + r, p0 + k) : E::zero();
        ut[it] = (j0 + c < c0 + cols && kk < w) ? ldA<W>(A, n, p0 + kk, j0 + c) : E::zero();
    }
    const int64_t i = i0 + ty, j = j0 + tx;
    const bool ok = i < r0 + rows && j < c0 + cols;
    T acc = ok ? ldA<W>(A, n, i, j) : E::zero();
#pragma unroll
    for (int it = 0; it < 4; it++) {
        const int e = tid + 64 * it;
        sts<W>(Ls, 8 * LDL, (e / BK) * LDL + e % BK, lt[it]);
        sts<W>(Us, BK * 8, e, ut[it]);
    }
    __syncthreads();
    for (int k = 0; k < w; k++) acc = E::sub(acc, E::mul(lds<W>(Ls, 8 * LDL, ty * LDL + k), lds<W>(Us, BK * 8, k * 8 + tx)));
    if (ok) stA<W>(A, n, i, j, acc);
}

template <int W> static size_t sub_gemm_smem() { return sizeof(double) * W * (32 * (kSubSB + 1) + kSubSB * 32); }

// dir 0: panel rows [p, n) x columns [p, p + kb) of A -> snapshot; dir 1: after the sub-panels,
// restore the snapshot if a row missed, else write ipiv = identity for the panel
__global__ void __launch_bounds__(256) lu_snap_kernel(double *A, int W, int64_t n, int64_t p, int kb, double *snap,
                                                      int64_t *ipiv, const int *miss, int dir) {
    if (dir == 1 && !__ldcg(miss)) {
        if (blockIdx.x == 0)
            for (int j = threadIdx.x; j < kb; j += blockDim.x) ipiv[p + j] = p + j;
        return;
    }
    const int64_t R = n - p, total = (int64_t)W * R * kb;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ww = e / (R * kb), rem = e % (R * kb), r = rem / kb, j = rem % kb;
        double *a = A + ww * n * n + (p + r) * n + p + j;
        if (dir == 0) snap[e] = *a;
        else *a = snap[e];
    }
}

// Apply the panel's interchanges (in order) to the columns outside the panel.
__global__ void __launch_bounds__(256) lu_laswp_kernel(double *A, int W, int64_t n, int64_t p, int64_t kb,
                                                       const int64_t *ipiv) {
    // the panel's pivots staged in shared memory (256 at a time): the per-column loop then
    // reads them without a global round trip per entry (the interchanges themselves stay in
    // order, one column-plane per thread)
    __shared__ long long ps[256];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ncols = n - kb;
    const bool act = t < (int64_t)W * ncols;
    const int plane = act ? (int)(t / ncols) : 0;
    int64_t j = act ? t % ncols : 0;
    if (j >= p) j += kb;
    double *Ap = A + (int64_t)plane * n * n;
    for (int64_t c0 = 0; c0 < kb; c0 += 256) {
        const int cn = (int)((kb - c0) < 256 ? (kb - c0) : 256);
        __syncthreads();
        for (int i = threadIdx.x; i < cn; i += blockDim.x) ps[i] = ipiv[p + c0 + i];
        __syncthreads();
        if (!act) continue;
        for (int i = 0; i < cn; i++) {
            const int64_t k = p + c0 + i, r = ps[i];
            if (r != k) {
                const double a = Ap[k * n + j];
                Ap[k * n + j] = Ap[r * n + j];
                Ap[r * n + j] = a;
            }
        }
    }
}

// ---- U12 := L11^{-1} A12 (unit lower, forward substitution in row order) ------------------
// One CTA per strip of cw columns held in shared memory; thread r owns panel row r and
// prefetches its next multiplier l_{r,i+1} during step i.
template <int W>
__global__ void __launch_bounds__(1024) lu_trsm_kernel(double *A, int64_t n, int64_t p, int64_t kb,
                                                       int64_t c0, int cw) {
    using E = elem<W>;
    using T = typename E::T;
    extern __shared__ double tile[];   // [W][kb][cw]
    const int TS = (int)(kb * cw);
    const int64_t col0 = c0 + (int64_t)blockIdx.x * cw;
    const int ncols = (int)((n - col0) < cw ? (n - col0) : cw);
    for (int64_t e = threadIdx.x; e < kb * cw; e += blockDim.x) {
        const int64_t r = e / cw, c = e % cw;
        if (c < ncols) sts<W>(tile, TS, (int)e, ldA<W>(A, n, p + r, col0 + c));
    }
    const int64_t r = threadIdx.x;   // blockDim.x >= kb (host guarantees)
    T lnext = E::zero();
    if (r > 0 && r < kb) lnext = ldA<W>(A, n, p + r, p);
    for (int64_t i = 0; i < kb; i++) {
        __syncthreads();
        const T l = lnext;
        if (i + 1 < r && r < kb) lnext = ldA<W>(A, n, p + r, p + i + 1);
        if (r > i && r < kb) {
            for (int c = 0; c < ncols; c++) {
                const T u = lds<W>(tile, TS, (int)(i * cw + c));
                const T a = lds<W>(tile, TS, (int)(r * cw + c));
                sts<W>(tile, TS, (int)(r * cw + c), E::sub(a, E::mul(l, u)));
            }
        }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < kb * cw; e += blockDim.x) {
        const int64_t rr = e / cw, c = e % cw;
        if (c < ncols) stA<W>(A, n, p + rr, col0 + c, lds<W>(tile, TS, (int)e));
    }
}

// Warp-per-column U12 := L11^{-1} A12 (default for kb <= 256). Every column of U12 is an
// independent forward substitution, so one warp owns one column: lane t holds rows
// r = t + 32q (q < RPL) in registers; at step i the owner of row i broadcasts it with
// shuffles and every lane updates its rows r > i -- a_ri := a_ri - l_ri * a_ii in i order,
// the same per-element sequence as lu_trsm_kernel and the oracle, with no CTA barrier per
// step. L11's columns stream through a double-buffered shared-memory ring (cp.async, 8-byte
// granules written transposed so the lanes' reads are conflict-free), CH columns per stage.
// warps (= columns) per CTA: 16 for DD; 8 for QD, whose 8 four-word rows per lane need
// more than the 128 registers a 512-thread CTA allows
template <int W> struct TrsmWpb { static constexpr int v = W == 2 ? 16 : 8; };
template <int W> struct TrsmCh { static constexpr int v = W == 2 ? 16 : 8; };   // 2 x 64 KB ring


template <int W, int RPL, int WPB = TrsmWpb<W>::v>
__global__ void __launch_bounds__(WPB * 32) lu_trsm_warp_kernel(double *A, int64_t n, int64_t p,
                                                               int kb, int64_t c0, int64_t ncols) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int CH = TrsmCh<W>::v;
    extern __shared__ double Ls[];   // [2][W][CH][kb]: word w of l_{p+r, p+i0+ii} at [b][w][ii][r]
    const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
    const int64_t col = c0 + (int64_t)blockIdx.x * WPB + wrp;
    const bool active = col < c0 + ncols;
    const int SS = CH * kb, BUF = W * SS;
    const int nst = (kb + CH - 1) / CH;
    auto issue = [&](int st) {   // stage st = L11 columns [st*CH, st*CH + ch) into buffer st & 1
        if (st < nst) {
            const int i0 = st * CH, ch = kb - i0 < CH ? kb - i0 : CH;
            double *buf = Ls + (st & 1) * BUF;
            for (int e = threadIdx.x; e < ch * kb; e += blockDim.x) {
                const int r = e / ch, ii = e % ch;   // consecutive threads walk a row of L11
                const double *src = A + (p + r) * n + (p + i0 + ii);
#pragma unroll
                for (int w = 0; w < W; w++) cp_async8(buf + w * SS + ii * kb + r, src + (int64_t)w * n * n);
            }
        }
        cp_async_commit();   // possibly empty: keeps the group count uniform
    };
    issue(0);
    issue(1);
    T v[RPL];
#pragma unroll
    for (int q = 0; q < RPL; q++) {
        const int r = lane + 32 * q;
        v[q] = (active && r < kb) ? ldA<W>(A, n, p + r, col) : E::zero();
    }
    // i = 32 qq + h: the owner slot qq of row i is a compile-time index (a runtime-indexed
    // pick would put v[] in local memory)
#pragma unroll
    for (int qq = 0; qq < RPL; qq++) {
        if (32 * qq >= kb) break;
        for (int h = 0; h < 32; h += CH) {
            const int i0 = 32 * qq + h;
            if (i0 >= kb) break;
            const int st = i0 / CH;
            const int ch = kb - i0 < CH ? kb - i0 : CH;
            cp_async_wait<1>();     // stage st has landed (only st + 1 may still be in flight)
            __syncthreads();
            const double *buf = Ls + (st & 1) * BUF;
            // every warp runs the steps (a warp past the last column works on zeros and stores
            // nothing), so the shuffles are never under a divergent branch
            for (int ii = 0; ii < ch; ii++) {
                const int i = i0 + ii;
                const double *lrow = buf + ii * kb;
                T x;
#pragma unroll
                for (int w = 0; w < W; w++) E::set_word(x, w, __shfl_sync(0xffffffffu, E::word(v[qq], w), h + ii));
                // rows of slots q > qq are all below row i: unmasked straight-line updates (the
                // chains interleave); only slot qq (rows <= i keep their value) and a ragged last
                // slot (rows >= kb) are masked
#pragma unroll
                for (int q = qq; q < RPL; q++) {
                    if (32 * q >= kb) break;
                    const bool full = 32 * q + 32 <= kb;
                    const int r = lane + 32 * q;
                    const int rc = full ? r : (r < kb ? r : kb - 1);
                    T l;
#pragma unroll
                    for (int w = 0; w < W; w++) E::set_word(l, w, lrow[w * SS + rc]);
                    const T nv = E::sub(v[q], E::mul(l, x));
                    if (q == qq) {
                        if (lane > h + ii && r < kb) v[q] = nv;
                    } else if (full || r < kb) {
                        v[q] = nv;
                    }
                }
            }
            __syncthreads();   // every warp is done with buffer st & 1
            issue(st + 2);
        }
    }
    if (!active) return;
#pragma unroll
    for (int q = 0; q < RPL; q++) {
        const int r = lane + 32 * q;
        if (r < kb) stA<W>(A, n, p + r, col, v[q]);
    }
}

// Blocked U12 := L11^{-1} A12 (default for kb <= 256). A CTA keeps a strip of TB_CW columns
// of U12 in shared memory and walks L11 in 32-row blocks b:
//   (a) the 32x32 diagonal block: one warp per column, lane = row, shuffles broadcast the
//       finished row (32 dependent steps);
//   (b) every row below the block takes the block's 32 updates, in i order, from registers:
//       a thread owns one column and up to TB_RPT rows, so each step is TB_RPT independent
//       DD chains fed by one broadcast x and TB_RPT multipliers from a staged L11 chunk.
// Element (r, c) still receives a_rc := a_rc - l_ri * u_ic for i = 0 .. r-1 ascending, the
// oracle's forward substitution, so the result is bit-identical to lu_trsm_kernel.
constexpr int TB_NT = 256;    // threads per CTA (8 warps: TB_CW / 8 columns each in phase (a))
constexpr int TB_LC = 8;      // L11 columns per off-diagonal stage
template <int W, int KB, int TB_CW>   // TB_CW columns per CTA: 16, or 8 to spread small panels
__global__ void __launch_bounds__(TB_NT) lu_trsm_blk_kernel(double *A, int64_t n, int64_t p,
                                                            int64_t c0, int64_t ncols) {
    constexpr int TB_G = TB_NT / TB_CW;          // row groups in phase (b)
    constexpr int TB_RPT = (KB - 32 + TB_G - 1) / TB_G;   // rows per thread in phase (b)
    constexpr int kb = KB;   // compile-time panel width: every block's row count below is static,
                             // so phase (b)'s TB_RPT chains are straight-line code
    using E = elem<W>;
    using T = typename E::T;
    extern __shared__ double sm[];
    // Ld and Lo rows are padded by one double (33, 225): the staging stores walk i / ii with r
    // fixed, and an unpadded 32- / 224-double stride put all of them in one bank
    double *Us = sm;                                  // [W][kb][TB_CW]
    double *Ld = Us + (size_t)W * kb * TB_CW;         // [W][32][33]: Ld[w][i][r]
    double *Lo = Ld + (size_t)W * 32 * 33;            // [W][TB_LC][225]: Lo[w][ii][r']
    const int US = kb * TB_CW, LDS_ = 32 * 33, LOS = TB_LC * 225;
    const int tid = threadIdx.x, lane = tid & 31, wrp = tid >> 5;
    const int64_t col0 = c0 + (int64_t)blockIdx.x * TB_CW;
    const int nc = (int)((c0 + ncols - col0) < TB_CW ? (c0 + ncols - col0) : TB_CW);

    for (int e = tid; e < kb * TB_CW; e += TB_NT) {
        const int r = e / TB_CW, c = e % TB_CW;
        const T v = c < nc ? ldA<W>(A, n, p + r, col0 + c) : E::zero();
#pragma unroll
        for (int w = 0; w < W; w++) Us[w * US + r * TB_CW + c] = E::word(v, w);
    }
#pragma unroll
    for (int b0 = 0; b0 < kb; b0 += 32) {
        constexpr int bs = 32;   // KB is a multiple of 32
        __syncthreads();   // Us rows of the previous block complete; Ld free
        for (int e = tid; e < bs * bs; e += TB_NT) {
            const int r = e / bs, i = e % bs;
            const T l = ldA<W>(A, n, p + b0 + r, p + b0 + i);
#pragma unroll
            for (int w = 0; w < W; w++) Ld[w * LDS_ + i * 33 + r] = E::word(l, w);
        }
        __syncthreads();
        // (a) diagonal block: warp wrp solves columns wrp (and wrp + 8), lane = row b0 + lane
        {
            const int ca = wrp, cb = TB_CW > 8 ? wrp + 8 : wrp;
            T va = E::zero(), vb = E::zero();
            if (lane < bs) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    E::set_word(va, w, Us[w * US + (b0 + lane) * TB_CW + ca]);
                    E::set_word(vb, w, Us[w * US + (b0 + lane) * TB_CW + cb]);
                }
            }
            for (int i = 0; i < bs; i++) {
                T xa, xb, l;
#pragma unroll
                for (int w = 0; w < W; w++) {
                    E::set_word(xa, w, __shfl_sync(0xffffffffu, E::word(va, w), i));
                    E::set_word(xb, w, __shfl_sync(0xffffffffu, E::word(vb, w), i));
                    E::set_word(l, w, Ld[w * LDS_ + i * 33 + lane]);
                }
                const T na = E::sub(va, E::mul(l, xa));
                const T nb = E::sub(vb, E::mul(l, xb));
                if (lane > i && lane < bs) { va = na; vb = nb; }
            }
            if (lane < bs) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    Us[w * US + (b0 + lane) * TB_CW + ca] = E::word(va, w);
                    if (TB_CW > 8) Us[w * US + (b0 + lane) * TB_CW + cb] = E::word(vb, w);
                }
            }
        }
        // (b) rows below the block: thread = (column c, row group g), rows rb + g + TB_G k
        const int rb = b0 + bs, R = kb - rb;   // compile-time after unrolling
        if (R <= 0) continue;
        const int c = tid % TB_CW, g = tid / TB_CW;
        T v[TB_RPT];
        __syncthreads();   // (a) results visible
#pragma unroll
        for (int k = 0; k < TB_RPT; k++) {
            const int r = g + TB_G * k;
            v[k] = E::zero();
            if (r < R) {
#pragma unroll
                for (int w = 0; w < W; w++) E::set_word(v[k], w, Us[w * US + (rb + r) * TB_CW + c]);
            }
        }
        for (int i0 = 0; i0 < bs; i0 += TB_LC) {
            const int lc = bs - i0 < TB_LC ? bs - i0 : TB_LC;
            __syncthreads();   // previous chunk consumed
            for (int e = tid; e < R * lc; e += TB_NT) {
                const int r = e / lc, ii = e % lc;
                const T l = ldA<W>(A, n, p + rb + r, p + b0 + i0 + ii);
#pragma unroll
                for (int w = 0; w < W; w++) Lo[w * LOS + ii * 225 + r] = E::word(l, w);
            }
            __syncthreads();
            for (int ii = 0; ii < lc; ii++) {
                const int i = b0 + i0 + ii;
                T x;
#pragma unroll
                for (int w = 0; w < W; w++) E::set_word(x, w, Us[w * US + i * TB_CW + c]);
#pragma unroll
                for (int k = 0; k < TB_RPT; k++) {
                    const int r = g + TB_G * k;
                    if (TB_G * k < R) {   // compile-time skip of whole empty row slots
                        const int rr = r < R ? r : R - 1;
                        T l;
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(l, w, Lo[w * LOS + ii * 225 + rr]);
                        const T nv = E::sub(v[k], E::mul(l, x));
                        if (r < R) v[k] = nv;
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < TB_RPT; k++) {
            const int r = g + TB_G * k;
            if (r < R) {
#pragma unroll
                for (int w = 0; w < W; w++) Us[w * US + (rb + r) * TB_CW + c] = E::word(v[k], w);
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < kb * TB_CW; e += TB_NT) {
        const int r = e / TB_CW, cc = e % TB_CW;
        if (cc < nc) {
            T v;
#pragma unroll
            for (int w = 0; w < W; w++) E::set_word(v, w, Us[w * US + r * TB_CW + cc]);
            stA<W>(A, n, p + r, col0 + cc, v);
        }
    }
}

// ---- solves ----------------------------------------------------------------------------------
// y := P b (ipiv swaps applied in order), in shared memory when it fits.
__global__ void __launch_bounds__(1024) lu_perm_kernel(const double *b, double *y, const int64_t *ipiv,
                                                       int W, int64_t n, int use_smem) {
    extern __shared__ double sy[];
    double *buf = use_smem ? sy : y;
    for (int64_t i = threadIdx.x; i < (int64_t)W * n; i += blockDim.x) buf[i] = b[i];
    // the swaps are applied in order by one thread; ipiv is staged through shared memory in
    // chunks first so that thread does not pay a global-memory round trip per entry
    __shared__ long long piv_s[2048];
    for (int64_t k0 = 0; k0 < n; k0 += 2048) {
        const int kc = (int)((n - k0) < 2048 ? (n - k0) : 2048);
        __syncthreads();
        for (int k = threadIdx.x; k < kc; k += blockDim.x) piv_s[k] = ipiv[k0 + k];
        __syncthreads();
        if (threadIdx.x < 32) {
            // warp 0 reads 32 pivots at a time and visits only the actual interchanges, in
            // order; lane w < W swaps plane w (the planes are independent, and each plane's
            // swaps stay in one thread, so their order is kept)
            const int lane = threadIdx.x;
            for (int k = 0; k < kc; k += 32) {
                const int64_t r_l = k + lane < kc ? piv_s[k + lane] : k0 + k + lane;
                unsigned mask = __ballot_sync(0xffffffffu, r_l != k0 + k + lane);
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const int64_t kk = k0 + k + j, r = __shfl_sync(0xffffffffu, r_l, j);
                    if (lane < W) {
                        const double t = buf[lane * n + kk];
                        buf[lane * n + kk] = buf[lane * n + r];
                        buf[lane * n + r] = t;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (use_smem)
        for (int64_t i = threadIdx.x; i < (int64_t)W * n; i += blockDim.x) y[i] = sy[i];
}

// The swaps of one panel, [p, p+kb), applied in order to y (the forward solve run panel by
// panel, alongside the factorisation): one warp, only the actual interchanges visited.
__global__ void __launch_bounds__(32) lu_yswap_kernel(double *y, const int64_t *ipiv, int W, int64_t n, int64_t p,
                                                      int64_t kb) {
    const int lane = threadIdx.x;
    for (int64_t k0 = p; k0 < p + kb; k0 += 32) {
        const int64_t k = k0 + lane;
        const int64_t r_l = k < p + kb ? ipiv[k] : k;
        unsigned mask = __ballot_sync(0xffffffffu, r_l != k);
        while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const int64_t kk = k0 + j, r = __shfl_sync(0xffffffffu, r_l, j);
            if (lane < W) {
                const double t = y[lane * n + kk];
                y[lane * n + kk] = y[lane * n + r];
                y[lane * n + r] = t;
            }
        }
    }
}

// y vectors: planar [W][n]
template <int W>
__device__ __forceinline__ typename elem<W>::T ldv(const double *y, int64_t n, int64_t i) {
    return elem<W>::load(y + i, n);
}
template <int W>
__device__ __forceinline__ void stv(double *y, int64_t n, int64_t i, const typename elem<W>::T &v) {
    elem<W>::store(y + i, n, v);
}

// Forward (unit L, j ascending) diagonal block [J, J+nb): one thread per row of the block.
template <int W>
__global__ void __launch_bounds__(1024) trsv_fwd_diag(const double *A, int64_t n, double *y, int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    __shared__ double ys[W * 256];
    const int s = threadIdx.x;
    if (s < nb) sts<W>(ys, 256, s, ldv<W>(y, n, J + s));
    T lnext = E::zero();
    if (s > 0 && s < nb) lnext = ldA<W>(A, n, J + s, J);
    for (int t = 0; t < nb; t++) {
        __syncthreads();
        const T l = lnext;
        if (t + 1 < s && s < nb) lnext = ldA<W>(A, n, J + s, J + t + 1);   // prefetch
        if (s > t && s < nb) sts<W>(ys, 256, s, E::sub(lds<W>(ys, 256, s), E::mul(l, lds<W>(ys, 256, t))));
    }
    __syncthreads();
    if (s < nb) stv<W>(y, n, J + s, lds<W>(ys, 256, s));
}

// rows i >= J+nb: y_i := y_i - l_ij y_j for j in [J, J+nb) ascending
template <int W>
__global__ void trsv_fwd_update(const double *A, int64_t n, double *y, int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    __shared__ double ys[W * 256];
    for (int t = threadIdx.x; t < nb; t += blockDim.x) sts<W>(ys, 256, t, ldv<W>(y, n, J + t));
    __syncthreads();
    const int64_t i = J + nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T v = ldv<W>(y, n, i);
    for (int t = 0; t < nb; t++) v = E::sub(v, E::mul(ldA<W>(A, n, i, J + t), lds<W>(ys, 256, t)));
    stv<W>(y, n, i, v);
}

// Backward diagonal block: for t descending, x_t = y_t / u_tt, then rows s < t update.
template <int W>
__global__ void __launch_bounds__(1024) trsv_bwd_diag(const double *A, int64_t n, double *y, double *x,
                                                      int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    __shared__ double ys[W * 256];
    const int s = threadIdx.x;
    if (s < nb) sts<W>(ys, 256, s, ldv<W>(y, n, J + s));
    // thread s < nb holds u_{s,t} for the current t (prefetched one step ahead; u_ss is the
    // divisor when t == s)
    T unext = E::zero();
    if (s < nb) unext = ldA<W>(A, n, J + s, J + nb - 1);
    for (int t = nb - 1; t >= 0; t--) {
        __syncthreads();
        const T u = unext;
        if (s < nb && t - 1 >= s) unext = ldA<W>(A, n, J + s, J + t - 1);
        if (s == t) sts<W>(ys, 256, t, E::div(lds<W>(ys, 256, t), u));   // slot t now holds x_t
        __syncthreads();
        if (s < t) sts<W>(ys, 256, s, E::sub(lds<W>(ys, 256, s), E::mul(u, lds<W>(ys, 256, t))));
    }
    __syncthreads();
    if (s < nb) stv<W>(x, n, J + s, lds<W>(ys, 256, s));
}

// rows i < J: y_i := y_i - u_ij x_j for j in [J, J+nb) descending
template <int W>
__global__ void trsv_bwd_update(const double *A, int64_t n, double *y, const double *x, int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    __shared__ double xs[W * 256];
    for (int t = threadIdx.x; t < nb; t += blockDim.x) sts<W>(xs, 256, t, ldv<W>(x, n, J + t));
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J) return;
    T v = ldv<W>(y, n, i);
    for (int t = nb - 1; t >= 0; t--) v = E::sub(v, E::mul(ldA<W>(A, n, i, J + t), lds<W>(xs, 256, t)));
    stv<W>(y, n, i, v);
}

// ---- blocked diagonal solves and coalesced updates (default when nb % 32 == 0) ---------------
// A diagonal block [J, J+nb) is walked in 32-row sub-blocks (forward: ascending, backward:
// descending). Warp 0 solves the sub-block's 32x32 triangle with shuffles (lane = row; forward
// broadcasts the finished row, backward forms x_t = div(y_t, u_tt) on the owner and broadcasts
// it); then every thread that owns a row outside the sub-block (below it going forward, above it
// going backward) folds the sub-block's 32 products into its row in the numerics.md s.5 order,
// with its 32 multipliers loaded up front (independent of the chain). Same per-element
// sequence as trsv_fwd_diag / trsv_bwd_diag and the oracle.
template <int W, bool FWD>
__global__ void __launch_bounds__(288) trsv_diag_blk(const double *A, int64_t n, double *y, double *x,
                                                     int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int PL = W == 2 ? 32 : 8;   // multipliers preloaded per chunk (registers)
    __shared__ double ys[W * 256];   // the block's y (forward) / x (backward) values
    extern __shared__ double dyn_smem[];   // DD: 8 warps x [W][32][33] multiplier tiles
    const int tid = threadIdx.x, lane = tid & 31, wrp = tid >> 5;
    if (tid < nb) sts<W>(ys, 256, tid, ldv<W>(y, n, J + tid));
    const int nsb = nb / 32;
    if constexpr (PL == 32) {
        // DD (launched with 288 threads): threads 0..255 own the block's rows, warp 8 solves the
        // 32x32 triangles. Every multiplier is loaded one phase AHEAD -- a row's 32 of sub-block
        // k while warp 8 solves triangle k, warp 8's next triangle's 32 while the rows fold --
        // so the uncoalesced row-segment loads (one row per lane) are never waited for on the
        // chain. Same operations in the same order as the generic path below.
        const bool solver = wrp == 8;
        T l[32];
        auto mine = [&](int b0) { return !solver && (FWD ? (tid >= b0 + 32 && tid < nb) : (tid < b0)); };
        auto tri_load = [&](int sb) {
#pragma unroll
            for (int i = 0; i < 32; i++) l[i] = ldA<W>(A, n, J + 32 * sb + lane, J + 32 * sb + i);
        };
        // A row-owning warp's 32 rows x 32 multipliers, read coalesced (lane = column: one
        // 256-byte row segment per load instead of 32 rows' sectors per load, which kept the
        // LSU busy ~16k cycles per sub-block) and transposed through a padded per-warp tile.
        // The warps are row-uniform (nb % 32 == 0), so whole warps own rows or none.
        double *tile = dyn_smem + wrp * (W * 32 * 33);
        auto rows_load = [&](int b0) {
#pragma unroll 8
            for (int q = 0; q < 32; q++) {
                const int64_t g = (J + 32 * wrp + q) * n + (J + b0 + lane);
#pragma unroll
                for (int w = 0; w < W; w++) tile[w * 32 * 33 + q * 33 + lane] = A[g + (int64_t)w * n * n];
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; i++) {
#pragma unroll
                for (int w = 0; w < W; w++) E::set_word(l[i], w, tile[w * 32 * 33 + lane * 33 + i]);
            }
            __syncwarp();
        };
        if (solver) tri_load(FWD ? 0 : nsb - 1);
        for (int k = 0; k < nsb; k++) {
            const int sb = FWD ? k : nsb - 1 - k;
            const int b0 = 32 * sb;
            __syncthreads();   // ys of the previous sub-block complete
            if (!solver && mine(b0)) rows_load(b0);   // alongside the triangle (a barrier-free phase)
            if (solver) {
                T v = lds<W>(ys, 256, b0 + lane);
#pragma unroll
                for (int ss = 0; ss < 32; ss++) {
                    const int t = FWD ? ss : 31 - ss;
                    T xt;
                    if (FWD) {
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(xt, w, __shfl_sync(0xffffffffu, E::word(v, w), t));
                    } else {
                        T u;
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(u, w, __shfl_sync(0xffffffffu, E::word(l[t], w), t));
                        const T d = E::div(v, u);
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(xt, w, __shfl_sync(0xffffffffu, E::word(d, w), t));
                        if (lane == t) v = xt;
                    }
                    const T nv = E::sub(v, E::mul(l[t], xt));
                    if (FWD ? (lane > t) : (lane < t)) v = nv;
                }
                sts<W>(ys, 256, b0 + lane, v);
            }
            __syncthreads();
            if (solver) {
                if (k + 1 < nsb) tri_load(FWD ? sb + 1 : sb - 1);
            } else if (mine(b0)) {
                T v = lds<W>(ys, 256, tid);
#pragma unroll
                for (int ss = 0; ss < 32; ss++) {
                    const int i = FWD ? ss : 31 - ss;
                    v = E::sub(v, E::mul(l[i], lds<W>(ys, 256, b0 + i)));
                }
                sts<W>(ys, 256, tid, v);
            }
        }
        __syncthreads();
        if (tid < nb) stv<W>(FWD ? y : x, n, J + tid, lds<W>(ys, 256, tid));
        return;
    }
    for (int k = 0; k < nsb; k++) {
        const int sb = FWD ? k : nsb - 1 - k;
        const int b0 = 32 * sb;
        __syncthreads();   // ys of the previous sub-block complete
        if (wrp == 0) {
            // the sub-block triangle: lane = row b0 + lane; multipliers PL columns at a time
            T v = lds<W>(ys, 256, b0 + lane);
#pragma unroll
            for (int c = 0; c < 32 / PL; c++) {
                const int s0 = FWD ? c * PL : 32 - (c + 1) * PL;
                T l[PL];
#pragma unroll
                for (int i = 0; i < PL; i++) l[i] = ldA<W>(A, n, J + b0 + lane, J + b0 + s0 + i);
#pragma unroll
                for (int ss = 0; ss < PL; ss++) {
                    const int i = FWD ? ss : PL - 1 - ss;
                    const int t = s0 + i;
                    T xt;
                    if (FWD) {
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(xt, w, __shfl_sync(0xffffffffu, E::word(v, w), t));
                    } else {
                        T u;   // u_tt, from lane t's multipliers
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(u, w, __shfl_sync(0xffffffffu, E::word(l[i], w), t));
                        const T d = E::div(v, u);
#pragma unroll
                        for (int w = 0; w < W; w++) E::set_word(xt, w, __shfl_sync(0xffffffffu, E::word(d, w), t));
                        if (lane == t) v = xt;   // this lane's row is finished: it now holds x_t
                    }
                    const T nv = E::sub(v, E::mul(l[i], xt));
                    if (FWD ? (lane > t) : (lane < t)) v = nv;
                }
            }
            sts<W>(ys, 256, b0 + lane, v);
        }
        __syncthreads();
        // rows outside the sub-block take its 32 products, in order
        const int r = tid;
        const bool mine = FWD ? (r >= b0 + 32 && r < nb) : (r < b0);
        if (mine) {
            T v = lds<W>(ys, 256, r);
#pragma unroll
            for (int c = 0; c < 32 / PL; c++) {
                const int s0 = FWD ? c * PL : 32 - (c + 1) * PL;
                T l[PL];
#pragma unroll
                for (int i = 0; i < PL; i++) l[i] = ldA<W>(A, n, J + r, J + b0 + s0 + i);
#pragma unroll
                for (int ss = 0; ss < PL; ss++) {
                    const int i = FWD ? ss : PL - 1 - ss;
                    v = E::sub(v, E::mul(l[i], lds<W>(ys, 256, b0 + s0 + i)));
                }
            }
            sts<W>(ys, 256, r, v);
        }
    }
    __syncthreads();
    if (tid < nb) stv<W>(FWD ? y : x, n, J + tid, lds<W>(ys, 256, tid));
}

// Coalesced off-diagonal update: 128 rows per CTA, the block's columns staged TU_CC at a time
// through a double-buffered cp.async ring (row segments read contiguously, stored transposed
// with padding), each thread folding its row in the numerics.md s.5 order (forward: j
// ascending into y; backward: j descending, with x).
constexpr int TU_ROWS = 128, TU_LD = TU_ROWS + 1;
template <int W> struct TuCc { static constexpr int v = W == 2 ? 32 : 16; };   // 2 x ~66 KB ring
template <int W, bool FWD>
__global__ void __launch_bounds__(TU_ROWS) trsv_update_co(const double *A, int64_t n, double *y,
                                                          const double *x, int64_t J, int nb) {
    using E = elem<W>;
    using T = typename E::T;
    constexpr int TU_CC = TuCc<W>::v;
    constexpr int LS = TU_CC * TU_LD, BUF = W * LS;
    extern __shared__ double sm[];
    double *vs = sm;                              // [W][256] the block's y (fwd) or x (bwd)
    double *Lt = sm + W * 256;                    // [2][W][TU_CC][TU_LD]
    const double *src = FWD ? y : x;
    for (int t = threadIdx.x; t < nb; t += blockDim.x) sts<W>(vs, 256, t, ldv<W>(src, n, J + t));
    const int64_t r0 = (FWD ? J + nb : 0) + (int64_t)blockIdx.x * TU_ROWS;
    const int64_t rend = FWD ? n : J;
    const int nr = (int)((rend - r0) < TU_ROWS ? (rend - r0) : TU_ROWS);
    const int me = threadIdx.x;
    const int nch = (nb + TU_CC - 1) / TU_CC;
    auto chunk_c0 = [&](int ch, int *cc_n) {
        const int cs = ch * TU_CC;
        *cc_n = nb - cs < TU_CC ? nb - cs : TU_CC;
        return FWD ? cs : nb - cs - *cc_n;   // backward: chunks from the right
    };
    auto issue = [&](int ch) {
        if (ch < nch) {
            int cc_n;
            const int c0 = chunk_c0(ch, &cc_n);
            double *buf = Lt + (ch & 1) * BUF;
            for (int e = threadIdx.x; e < nr * TU_CC; e += blockDim.x) {
                const int r = e / TU_CC, cc = e % TU_CC;
                if (cc < cc_n) {
                    const double *g = A + (r0 + r) * n + (J + c0 + cc);
#pragma unroll
                    for (int w = 0; w < W; w++) cp_async8(buf + w * LS + cc * TU_LD + r, g + (int64_t)w * n * n);
                }
            }
        }
        cp_async_commit();
    };
    issue(0);
    issue(1);
    T v = me < nr ? ldv<W>(y, n, r0 + me) : E::zero();
    __syncthreads();   // vs
    for (int ch = 0; ch < nch; ch++) {
        int cc_n;
        const int c0 = chunk_c0(ch, &cc_n);
        cp_async_wait<1>();
        __syncthreads();
        const double *buf = Lt + (ch & 1) * BUF;
        if (me < nr) {
            auto prod = [&](int cc) {
                T a;
#pragma unroll
                for (int w = 0; w < W; w++) E::set_word(a, w, buf[w * LS + cc * TU_LD + me]);
                return E::mul(a, lds<W>(vs, 256, c0 + cc));
            };
            if (cc_n == TU_CC) {
                // whole chunk: the products (independent of v) 8 at a time ahead of the subs, so
                // only the subtraction chain is serial (same operations, same order)
#pragma unroll
                for (int k0 = 0; k0 < TU_CC; k0 += 8) {
                    T pr[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) pr[u] = prod(FWD ? k0 + u : TU_CC - 1 - (k0 + u));
#pragma unroll
                    for (int u = 0; u < 8; u++) v = E::sub(v, pr[u]);
                }
            } else {
                for (int k = 0; k < cc_n; k++) v = E::sub(v, prod(FWD ? k : cc_n - 1 - k));
            }
        }
        __syncthreads();
        issue(ch + 2);
    }
    if (me < nr) stv<W>(y, n, r0 + me, v);
}

// ---- host driver -------------------------------------------------------------------------------
static int g_coop_sms[64];   // per device: SM count if cooperative launch is supported, else 0
static bool g_coop_init[64];

// DDQD_LU_PANEL=steps forces the per-column two-kernel path (kept as the reference schedule)
static bool use_coop_panel() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_PANEL");
        v = (e && std::string(e) == "steps") ? 0 : 1;
    }
    return v == 1;
}

// Diagonal fast path of the cooperative panel: DDQD_LU_SPEC=0 off (every column runs the full
// candidate exchange, as in round 1), =1 one grid barrier per column, default (2) the split
// arrive/wait barrier; the factors are the same bits in every mode
static int spec_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_SPEC");
        v = (e && (e[0] == '0' || e[0] == '1')) ? e[0] - '0' : 2;
    }
    return v;
}

// returns 1 if the cooperative path was launched, 0 if the caller should use the per-column path
template <int W>
static int try_panel_coop(double *A, int64_t n, int64_t p, int64_t kb, int pivot, int64_t *ipiv, LuAux *aux,
                          double *scr, size_t scr_bytes, cudaStream_t s, int *rc, cudaEvent_t pre_swap,
                          const int *gate = nullptr, bool probe_only = false) {
    *rc = DDQD_OK;
    const int64_t R = n - p;
    const int dv = current_device();
    if (!g_coop_init[dv]) {
        int dev = 0, coop = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_coop_sms[dv] = coop ? sms : 0;
        g_coop_init[dv] = true;
    }
    const int nsm = g_coop_sms[dv];
    if (nsm <= 0 || kb > 4096) return 0;
    int G = (int)std::min<int64_t>(nsm, R);
    const int rows_per = (int)((R + G - 1) / G);
    G = (int)((R + rows_per - 1) / rows_per);
    const size_t smem = sizeof(double) * W * ((size_t)rows_per * kb + (size_t)kb + (size_t)rows_per);
    if (smem > 200 * 1024) return 0;
    const size_t per_buf = (size_t)G * (W + 1) * kLuCrep + (size_t)G * W * kb + (size_t)W * kb;
    const size_t fast_bytes = sizeof(double) * (2 * (size_t)kLuRrep * W * (kb + 1) + (size_t)kb + 2);   // rows + flags + counter
    if (2 * per_buf * sizeof(double) + fast_bytes > scr_bytes) return 0;
    static size_t attr_dev[64];
    size_t &attr = attr_dev[dv];
    if (smem > 48 * 1024 && smem > attr) {
        if (cudaFuncSetAttribute(lu_panel_coop_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        attr = smem;
    }
    int occ = 0;
    static int nthr = -1;   // DDQD_LU_THREADS=256|512: threads of the panel CTA
    if (nthr < 0) {
        const char *e = getenv("DDQD_LU_THREADS");
        nthr = (e && std::string(e) == "256") ? 256 : 512;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lu_panel_coop_kernel<W>, nthr, smem);
    if (occ < 1 || G > occ * nsm) return 0;
    if (probe_only) return 1;   // (the split path asks whether its fallback can launch)
    int kbi = (int)kb;
    int piv = pivot;
    static int probe = -1;   // DDQD_LU_PROBE=1: per-phase clock64 report (timing experiments)
    if (probe < 0) {
        const char *e = getenv("DDQD_LU_PROBE");
        probe = (e && e[0] == '1') ? 1 : 0;
    }
    int spec = gate ? 0 : spec_mode();   // the split path's fallback: straight to the full search
    double *fscr = scr + 2 * per_buf;
    void *args[] = {&A, &n, &p, &kbi, (void *)&rows_per, &piv, &ipiv, &aux, &scr, &probe, &spec, &fscr,
                    (void *)&gate};
    cudaError_t e = cudaLaunchCooperativeKernel((void *)lu_panel_coop_kernel<W>, dim3(G), dim3(nthr), args, smem, s);
    count_launch();
    if (e != cudaSuccess) {
        set_error(std::string("cooperative panel launch: ") + cudaGetErrorString(e));
        *rc = DDQD_ECUDA;
        return 1;
    }
    if (pivot && n - kb > 0) {
        // the interchanges move rows of the earlier panels' L columns: a reader of those (the
        // panel-by-panel forward solve on another stream) must be done with them first
        if (pre_swap) DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, pre_swap, 0));
        const int64_t threads = (int64_t)W * (n - kb);
        lu_laswp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(A, W, n, p, kb, ipiv);
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("laswp launch: ") + cudaGetErrorString(e));
            *rc = DDQD_ECUDA;
        }
    }
    return 1;
}

// DDQD_LU_SPLIT=0 keeps the cooperative panel for the speculated path (A/B measurements)
static bool split_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_SPLIT");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static int sub_probe() {   // DDQD_LU_PROBE=1: per-phase clock64 of the sub-panel diagonal kernel
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_PROBE");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v;
}

// DDQD_LU_TIMELINE=p0,p1,...: for those panel starts (columns), record CUDA events around every
// blocked-panel kernel on its stream and print a start/end timeline (us from the panel's start;
// a diagnostic: it synchronises after the panel)
static bool timeline_panel(int64_t p) {
    static std::string v = [] { const char *e = getenv("DDQD_LU_TIMELINE"); return std::string(e ? e : ""); }();
    if (v.empty()) return false;
    size_t a = 0;
    while (a <= v.size()) {
        size_t b = v.find(',', a);
        if (b == std::string::npos) b = v.size();
        if (b > a && std::atoll(v.substr(a, b - a).c_str()) == (long long)p) return true;
        a = b + 1;
    }
    return false;
}

// DDQD_LU_SUB_OVERLAP=0 runs every sub-panel kernel on the one stream (A/B measurements)
static bool sub_overlap_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_SUB_OVERLAP");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// returns 1 if the blocked speculated panel (+ its gated cooperative fallback and the
// interchanges) was launched, 0 if the caller should use the cooperative/per-column path
template <int W>
static int try_panel_split(double *A, int64_t n, int64_t p, int64_t kb, int pivot, int64_t *ipiv, LuAux *aux,
                           double *scr, size_t scr_bytes, double *pout, cudaStream_t s, int *rc,
                           cudaEvent_t pre_swap) {
    *rc = DDQD_OK;
    // DD only. QD measured slower (n = 1024 / 2048, panel 256: 26.5 / 77.8 ms vs 19.7 / 62.8 ms
    // with the cooperative panel): QD arithmetic is ~10x DD's, so the one-CTA diagonal blocks
    // and the rank-32 updates become FP64-bound where the cooperative kernel spreads the panel
    // over every SM.
    if constexpr (W != 2) {
        return 0;
    } else {
    if (!pout || !split_enabled() || spec_mode() != 2 || kb > 256 || kb < 1) return 0;
    // the fallback must be able to run (cooperative launch with the slab in shared memory)
    int frc = DDQD_OK;
    if (!try_panel_coop<W>(A, n, p, kb, pivot, ipiv, aux, scr, scr_bytes, s, &frc, nullptr, nullptr, true)) return 0;
    constexpr int SB = kSubSB;
    const int dv = current_device();
    const size_t tsm = sizeof(double) * 2 * W * (size_t)TrsmCh<W>::v * SB;
    const size_t gsm = sub_gemm_smem<W>();
    static bool dattr[64];
    if (!dattr[dv]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_subdiag_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSubDiagPad));
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_subgemm_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
        dattr[dv] = true;
    }
    const int kbi = (int)kb;
    const int64_t R = n - p;
    int *miss = &aux->miss;
    const unsigned cgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(((int64_t)W * R * kb + 255) / 256,
                                                                             (int64_t)sm_count() * 8));
    DDQD_CUDA_CHECK(cudaMemsetAsync(miss, 0, sizeof(int), s));
    lu_snap_kernel<<<cgrid, 256, 0, s>>>(A, W, n, p, kbi, pout, ipiv, miss, 0);
    DDQD_LAUNCH_CHECK();
    // Two streams (not under graph capture): the latency-bound diagonal blocks D and the column
    // TRSMs T on a side stream, the row eliminations B and the updates G on s. G of sub-panel q
    // is split into Ga (the next sub-panel's rows, all columns right) and Gb (the rows below):
    // D_{q+1} and T_{q+1} need only Ga, so they run while Gb does. Dependencies (events):
    //   D_q, T_q  after Ga_{q-1} (side);  B_q after D_q and Gb_{q-1} (s);
    //   Ga_q, Gb_q after B_q (s) and T_q (side).
    cudaStream_t s2 = s;
    cudaEvent_t evA = nullptr, evD = nullptr, evT = nullptr;
    {
        cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cst) != cudaSuccess) { cudaGetLastError(); cst = cudaStreamCaptureStatusActive; }
        static thread_local cudaStream_t side[64];
        static thread_local cudaEvent_t evs[64][3];
        if (cst == cudaStreamCaptureStatusNone && sub_overlap_enabled()) {
            if (!side[dv]) {
                int lo = 0, hi = 0;
                DDQD_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                DDQD_CUDA_CHECK(cudaStreamCreateWithPriority(&side[dv], cudaStreamNonBlocking, hi));
                for (int e = 0; e < 3; e++) DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&evs[dv][e], cudaEventDisableTiming));
            }
            s2 = side[dv];
            evA = evs[dv][0]; evD = evs[dv][1]; evT = evs[dv][2];
        }
    }
    const bool two = s2 != s;
    struct TlRec { const char *nm; int q; bool side; cudaEvent_t e0, e1; };
    std::vector<TlRec> tlr;
    const bool tl = timeline_panel(p);
    cudaEvent_t tl_base = nullptr;
    if (tl) { cudaEventCreate(&tl_base); cudaEventRecord(tl_base, s); }
    auto tl0 = [&](cudaStream_t st) -> cudaEvent_t {
        cudaEvent_t e = nullptr;
        if (tl) { cudaEventCreate(&e); cudaEventRecord(e, st); }
        return e;
    };
    auto tl1 = [&](const char *nm, int q, cudaStream_t st, cudaEvent_t e0) {
        if (!tl) return;
        cudaEvent_t e1;
        cudaEventCreate(&e1);
        cudaEventRecord(e1, st);
        tlr.push_back({nm, q, two && st == s2, e0, e1});
    };
    if (two) {   // the side stream starts after the snapshot
        DDQD_CUDA_CHECK(cudaEventRecord(evA, s));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(s2, evA, 0));
    }
    constexpr int WPB = 4;   // TRSM: 4 columns per CTA (each column is a 32-step chain: spread them)
    // D -> B reciprocals, one [W][SB] slot per sub-panel (after the snapshot in pout)
    double *const rv_base = pout + (size_t)W * (size_t)n * 256;
    // The pivot chain D_q -> B_q -> Ga_q -> D_{q+1} stays on ONE stream (s2, high priority): a
    // same-stream hop costs ~2.6 us, a cross-stream one ~5.7 us (DDQD_LU_TIMELINE). The bulk
    // (T_q, then Gb_q) runs on s; the cross-stream waits are on work that normally finished
    // already: B_q waits for Gb_{q-1} (its rows), Ga_q for T_q (its U rows), T_q for D_q, Gb_q
    // for B_q.
    cudaEvent_t evB = evT;   // (the three events: evA = Gb done, evD = D done, evT = T done; evB below)
    static thread_local cudaEvent_t evBs[64];
    if (two) {
        if (!evBs[dv]) DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&evBs[dv], cudaEventDisableTiming));
        evB = evBs[dv];
    }
    bool gb_pending = false;   // evA holds a Gb of an earlier sub-panel
    for (int q0 = 0; q0 < kbi; q0 += SB) {
        const int w = std::min(SB, kbi - q0);
        const int64_t p0 = p + q0;
        const int64_t rows = n - (p0 + w);            // rows below the diagonal block
        const int64_t cols = p + kb - (p0 + w);       // columns right of it (inside the panel)
        double *const rvb = rv_base + (size_t)(q0 / SB) * W * SB;
        cudaEvent_t t0 = tl0(s2);
        lu_subdiag_kernel<W><<<1, kSubDiagNT, kSubDiagPad, s2>>>(A, n, p0, w, pivot, miss, rvb, sub_probe());
        DDQD_LAUNCH_CHECK();
        tl1("D", q0 / SB, s2, t0);
        if (cols > 0) {
            if (two) {
                DDQD_CUDA_CHECK(cudaEventRecord(evD, s2));
                DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, evD, 0));
            }
            t0 = tl0(s);
            lu_trsm_warp_kernel<W, 1, WPB><<<(unsigned)((cols + WPB - 1) / WPB), WPB * 32, tsm, s>>>(A, n, p0, w, p0 + w,
                                                                                                   cols);
            DDQD_LAUNCH_CHECK();
            tl1("T", q0 / SB, s, t0);
            if (two) DDQD_CUDA_CHECK(cudaEventRecord(evT, s));
        }
        if (rows > 0) {
            if (two && gb_pending) DDQD_CUDA_CHECK(cudaStreamWaitEvent(s2, evA, 0));
            t0 = tl0(s2);
            lu_subbelow_kernel<W><<<(unsigned)((rows + SubBelow<W>::ROWS - 1) / SubBelow<W>::ROWS), SubBelow<W>::NT, 0,
                                    s2>>>(A, n, p0, w, pivot, miss, p0 + w, rows, rvb, sub_probe());
            DDQD_LAUNCH_CHECK();
            tl1("B", q0 / SB, s2, t0);
        }
        if (cols > 0 && rows > 0) {
            if (two) {
                DDQD_CUDA_CHECK(cudaEventRecord(evB, s2));
                DDQD_CUDA_CHECK(cudaStreamWaitEvent(s2, evT, 0));
            }
            const int64_t ra = std::min<int64_t>(rows, SB);   // Ga: the next sub-panel's rows
            dim3 ga((unsigned)((cols + 7) / 8), (unsigned)((ra + 7) / 8));
            t0 = tl0(s2);
            lu_subgemm_small_kernel<W><<<ga, 64, 0, s2>>>(A, n, p0, w, p0 + w, ra, p0 + w, cols, miss);
            DDQD_LAUNCH_CHECK();
            tl1("Ga", q0 / SB, s2, t0);
            if (rows > ra) {
                if (two) DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, evB, 0));
                dim3 gb((unsigned)((cols + 31) / 32), (unsigned)((rows - ra + 31) / 32));
                t0 = tl0(s);
                lu_subgemm_kernel<W><<<gb, 128, gsm, s>>>(A, n, p0, w, p0 + w + ra, rows - ra, p0 + w, cols, miss);
                DDQD_LAUNCH_CHECK();
                tl1("Gb", q0 / SB, s, t0);
                if (two) DDQD_CUDA_CHECK(cudaEventRecord(evA, s));
                gb_pending = true;
            }
        }
    }
    if (two) {   // join: the last D / T
        DDQD_CUDA_CHECK(cudaEventRecord(evD, s2));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, evD, 0));
    }
    lu_snap_kernel<<<cgrid, 256, 0, s>>>(A, W, n, p, kbi, pout, ipiv, miss, 1);
    DDQD_LAUNCH_CHECK();
    if (tl) {
        cudaStreamSynchronize(s);
        for (const TlRec &r : tlr) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, tl_base, r.e0);
            cudaEventElapsedTime(&b, tl_base, r.e1);
            printf("LUTIMELINE p=%lld q=%d kernel=%s stream=%s start_us=%.2f end_us=%.2f\n", (long long)p, r.q, r.nm,
                   r.side ? "side" : "main", a * 1e3f, b * 1e3f);
            cudaEventDestroy(r.e0);
            cudaEventDestroy(r.e1);
        }
        cudaEventDestroy(tl_base);
    }
    // the fallback (full pivot search from the restored panel) runs only on a miss; then the
    // interchanges of the other columns, as after the cooperative kernel
    if (!try_panel_coop<W>(A, n, p, kb, pivot, ipiv, aux, scr, scr_bytes, s, rc, pre_swap, miss)) {
        set_error("split panel: the cooperative fallback could not be launched");
        *rc = DDQD_ECUDA;
    }
    return 1;
    }
}

// DDQD_LU_TRSM=strip selects the row-parallel strip kernel (one CTA barrier per step) for
// every panel width, =warp the warp-per-column kernel; default: the blocked kernel for
// 256-wide panels (c4's), the warp-per-column kernel for other widths <= 256.
static int trsm_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_TRSM");
        v = (e && std::string(e) == "strip") ? 0 : (e && std::string(e) == "warp") ? 1
          : (e && std::string(e) == "sub") ? 3 : 2;
    }
    return v;
}

// Steps 1-2 of numerics.md s.5 for the panel [p, p+kb): factorisation (cooperative kernel or
// the per-column pair), interchanges of the other columns, U12 := L11^{-1} A12.
template <int W>
static int lu_panel_w(int64_t n, int pivot, double *A, int64_t *ipiv, int64_t p, int64_t kb, LuAux *aux,
                      double *scr, size_t scr_bytes, cudaStream_t s, cudaEvent_t pre_swap = nullptr,
                      double *pout = nullptr) {
    NvtxRange nv("LU panel + TRSM");
    prof_begin(3, s);
    int crc = DDQD_OK;
    // the per-column kernels swap whole rows as they go: order them after the reader up front
    if (pre_swap && !use_coop_panel()) DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, pre_swap, 0));
    const bool split = use_coop_panel() && try_panel_split<W>(A, n, p, kb, pivot, ipiv, aux, scr, scr_bytes, pout, s,
                                                              &crc, pre_swap);
    if (crc) return crc;
    const bool coop = split || (use_coop_panel() && try_panel_coop<W>(A, n, p, kb, pivot, ipiv, aux, scr, scr_bytes,
                                                                      s, &crc, pre_swap));
    if (crc) return crc;
    if (!coop && pre_swap && use_coop_panel()) DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, pre_swap, 0));
    for (int64_t k = p; !coop && k < p + kb; k++) {
        lu_pivot_kernel<W><<<1, 1024, 0, s>>>(A, n, k, pivot, ipiv, aux);
        DDQD_LAUNCH_CHECK();
        const int64_t nc = p + kb - (k + 1), nr = n - (k + 1);
        if (nc > 0 && nr > 0) {
            dim3 blk(32, 8);
            dim3 grd((unsigned)((nc + 31) / 32), (unsigned)((nr + 7) / 8));
            lu_rank1_kernel<W><<<grd, blk, 0, s>>>(A, n, k, p + kb, aux);
            DDQD_LAUNCH_CHECK();
        }
    }
    prof_end(3, (double)kb * (double)(n - p) * (double)kb / 2.0, s,   // panel madds (approx.)
             split ? "lu split panel (lu_subdiag/subbelow/trsm_warp/subgemm kernels)"
                   : coop ? "lu_panel_coop_kernel (+ lu_laswp_kernel)" : "lu_pivot_kernel + lu_rank1_kernel");
    const int64_t n2 = n - p - kb;
    if (n2 <= 0) return DDQD_OK;
    // one CTA per SM when possible: cw = ceil(n2 / #SMs), capped by shared memory
    const int64_t cw_smem = std::max<int64_t>(1, (int64_t)(200 * 1024) / (8 * W * kb));
    int cw = (int)std::max<int64_t>(1, std::min<int64_t>(cw_smem, (n2 + sm_count() - 1) / sm_count()));
    const size_t smem = sizeof(double) * W * (size_t)kb * cw;
    if (smem > 48 * 1024)
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_trsm_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
    if (kb > 1024) { set_error("panel > 1024 not supported by the TRSM kernel"); return DDQD_ENOTSUP; }
    prof_begin(4, s);
    bool trsm_done = false;
    if constexpr (W == 2) {
    if (trsm_mode() == 3) {
        trsm_done = true;
        // DDQD_LU_TRSM=sub (DD): blocked by 32 rows of L11 -- the 32-row diagonal block's triangle solve
        // over all n2 columns (the warp TRSM, a 32-step chain per column), then the rows below
        // it inside the panel take that block's 32 updates (the k-ascending update kernel of
        // the blocked panel). Each U12 element still receives a_rj -= l_ri u_ij for i ascending
        // (numerics.md s.5 step 2), so the bits are those of the one-pass kernels. Measured on
        // c4: 36.8 ms vs 36.0 with the one-pass strip kernel (TRSM 10.1% vs 8.2% of the solve:
        // the 8 launches per panel re-read L11 and U12 from L2), so it stays opt-in.
        constexpr int SB = kSubSB, WPB = 4;
        const size_t tsm = sizeof(double) * 2 * W * (size_t)TrsmCh<W>::v * SB;
        for (int64_t b0 = 0; b0 < kb; b0 += SB) {
            const int w = (int)std::min<int64_t>(SB, kb - b0);
            lu_trsm_warp_kernel<W, 1, WPB><<<(unsigned)((n2 + WPB - 1) / WPB), WPB * 32, tsm, s>>>(A, n, p + b0, w,
                                                                                                  p + kb, n2);
            DDQD_LAUNCH_CHECK();
            const int64_t rows = kb - b0 - w;
            if (rows > 0) {
                dim3 g((unsigned)((n2 + 31) / 32), (unsigned)((rows + 31) / 32));
                lu_subgemm_kernel<W><<<g, 128, sub_gemm_smem<W>(), s>>>(A, n, p + b0, w, p + b0 + w, rows, p + kb, n2, nullptr);
                DDQD_LAUNCH_CHECK();
            }
        }
    }
    }
    if (trsm_done) {
    } else if (kb == 256 && trsm_mode() >= 2) {
        // 16-column strips while they fill ~1.5 waves of the SMs, else 8 (twice the CTAs, each
        // with half the chain): the per-CTA chain, not the FP64 rate, bounds small panels
        static bool battr[2][64] = {};
        const bool wide = (n2 + 15) / 16 >= 3 * sm_count() / 2;
        const size_t bsmem = sizeof(double) * W * ((size_t)256 * (wide ? 16 : 8) + 32 * 33 + (size_t)TB_LC * 225);
        auto kfn = wide ? lu_trsm_blk_kernel<W, 256, 16> : lu_trsm_blk_kernel<W, 256, 8>;
        if (!battr[wide][current_device()]) {
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
            battr[wide][current_device()] = true;
        }
        const int cw = wide ? 16 : 8;
        kfn<<<(unsigned)((n2 + cw - 1) / cw), TB_NT, bsmem, s>>>(A, n, p, p + kb, n2);
    } else if (kb <= 256 && trsm_mode() >= 1) {
        const size_t wsmem = sizeof(double) * 2 * W * (size_t)TrsmCh<W>::v * kb;
        static bool wattr[64] = {};   // set once per device to the largest ring (kb = 256)
        if (!wattr[current_device()]) {
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_trsm_warp_kernel<W, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(sizeof(double) * 2 * W * TrsmCh<W>::v * 256)));
            wattr[current_device()] = true;
        }
        constexpr int WPB = TrsmWpb<W>::v;
        lu_trsm_warp_kernel<W, 8><<<(unsigned)((n2 + WPB - 1) / WPB), WPB * 32, wsmem, s>>>(
            A, n, p, (int)kb, p + kb, n2);
    } else {
        const int tthreads = (int)(((kb + 31) / 32) * 32);
        lu_trsm_kernel<W><<<(unsigned)((n2 + cw - 1) / cw), tthreads, smem, s>>>(A, n, p, kb, p + kb, cw);
    }
    DDQD_LAUNCH_CHECK();
    prof_end(4, (double)kb * (double)kb / 2.0 * (double)n2, s, "lu_trsm_*_kernel (U12)");
    return DDQD_OK;
}

// DDQD_LU_TRSV=plain keeps the one-thread-per-row diagonal kernels and uncoalesced updates
// (the reference schedule); default: warp-level diagonal blocks + coalesced updates.
static bool trsv_fast_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_TRSV");
        v = (e && std::string(e) == "plain") ? 0 : 1;
    }
    return v == 1;
}

// shared-memory sizes / attributes of the solve kernels (set once per device)
template <int W>
static size_t trsv_diag_smem() { return W == 2 ? sizeof(double) * 8 * W * 32 * 33 : 0; }
template <int W>
static int trsv_setup(size_t *usm_out) {
    const size_t usm = sizeof(double) * W * (256 + 2 * (size_t)TuCc<W>::v * TU_LD);
    static bool tattr[64] = {};
    if (trsv_fast_enabled() && !tattr[current_device()]) {
        if (W == 2) {
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(trsv_diag_blk<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)trsv_diag_smem<W>()));
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(trsv_diag_blk<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)trsv_diag_smem<W>()));
        }
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(trsv_update_co<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(trsv_update_co<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
        tattr[current_device()] = true;
    }
    *usm_out = usm;
    return DDQD_OK;
}

// forward (unit L) for the diagonal block [J, J+nb) and the fold of its columns into rows >= J+nb
template <int W>
static int trsv_fwd_block(int64_t n, const double *A, double *y, int64_t J, int nb, size_t usm, cudaStream_t s) {
    const int64_t rows = n - J - nb;
    if (trsv_fast_enabled() && nb % 32 == 0) {
        trsv_diag_blk<W, true><<<1, W == 2 ? 288 : 256, trsv_diag_smem<W>(), s>>>(A, n, y, nullptr, J, nb);
        DDQD_LAUNCH_CHECK();
        if (rows > 0) {
            trsv_update_co<W, true><<<(unsigned)((rows + TU_ROWS - 1) / TU_ROWS), TU_ROWS, usm, s>>>(A, n, y, nullptr, J, nb);
            DDQD_LAUNCH_CHECK();
        }
        return DDQD_OK;
    }
    trsv_fwd_diag<W><<<1, 256, 0, s>>>(A, n, y, J, nb);
    DDQD_LAUNCH_CHECK();
    if (rows > 0) {
        trsv_fwd_update<W><<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(A, n, y, J, nb);
        DDQD_LAUNCH_CHECK();
    }
    return DDQD_OK;
}

// backward (upper, x_j = div(y_j, u_jj)), 256-row blocks from the bottom
template <int W>
static int trsv_bwd_all(int64_t n, const double *A, double *y, double *x, size_t usm, cudaStream_t s) {
    const int NB = 256;
    const bool fast = trsv_fast_enabled();
    const int64_t last = ((n - 1) / NB) * NB;
    for (int64_t J = last; J >= 0; J -= NB) {
        const int nb = (int)std::min<int64_t>(NB, n - J);
        if (fast && nb % 32 == 0) {
            trsv_diag_blk<W, false><<<1, W == 2 ? 288 : 256, trsv_diag_smem<W>(), s>>>(A, n, y, x, J, nb);
            DDQD_LAUNCH_CHECK();
            if (J > 0) {
                trsv_update_co<W, false><<<(unsigned)((J + TU_ROWS - 1) / TU_ROWS), TU_ROWS, usm, s>>>(A, n, y, x, J, nb);
                DDQD_LAUNCH_CHECK();
            }
            continue;
        }
        trsv_bwd_diag<W><<<1, 256, 0, s>>>(A, n, y, x, J, nb);
        DDQD_LAUNCH_CHECK();
        if (J > 0) {
            trsv_bwd_update<W><<<(unsigned)((J + 127) / 128), 128, 0, s>>>(A, n, y, x, J, nb);
            DDQD_LAUNCH_CHECK();
        }
    }
    return DDQD_OK;
}

// Eq. (2) with the factors: y := P b, forward (unit L), backward (numerics.md s.5).
template <int W>
static int lu_trsv_w(int64_t n, const double *A, const int64_t *ipiv, const double *b, double *x, double *y,
                     cudaStream_t s) {
    NvtxRange nv("LU solves");
    const int use_smem = ((int64_t)W * n * (int64_t)sizeof(double) <= 200 * 1024) ? 1 : 0;
    const size_t psmem = use_smem ? (size_t)W * n * sizeof(double) : 0;
    if (psmem > 48 * 1024)
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)psmem));
    size_t usm = 0;
    int rc = trsv_setup<W>(&usm);
    if (rc) return rc;
    prof_begin(5, s);
    lu_perm_kernel<<<1, 1024, psmem, s>>>(b, y, ipiv, W, n, use_smem);
    DDQD_LAUNCH_CHECK();
    const int NB = 256;
    for (int64_t J = 0; J < n; J += NB)
        if ((rc = trsv_fwd_block<W>(n, A, y, J, (int)std::min<int64_t>(NB, n - J), usm, s))) return rc;
    if ((rc = trsv_bwd_all<W>(n, A, y, x, usm, s))) return rc;
    prof_end(5, (double)n * (double)n, s, "lu solves (perm, trsv_diag_blk, trsv_update_co)");
    return DDQD_OK;
}

// aux layout: LuAux | y [W n] | cooperative-panel scratch (2 buffers)
struct LuMem {
    LuAux *aux;
    double *y, *scr;
    size_t scr_bytes;
    double *pout;   // split panel: [W][n - p][K] factors + [W][K] reciprocals
};
static int lu_mem(int W, int64_t n, int64_t K, LuMem *m) {
    int st = DDQD_OK;
    const size_t ybytes = (sizeof(double) * W * (size_t)n + 255) & ~size_t(255);
    // two candidate buffers for up to one CTA per SM, plus the fast path's pivot rows and flags
    const size_t G = (size_t)std::max(sm_count(), 1);
    m->scr_bytes = sizeof(double) * (2 * (G * ((W + 1) * kLuCrep + W * (size_t)K) + W * (size_t)K) +
                                     2 * (size_t)kLuRrep * W * (K + 1) + (size_t)K + 2);
    const size_t sb = (m->scr_bytes + 255) & ~size_t(255);
    const size_t pbytes = K <= 256 ? sizeof(double) * W * ((size_t)n * 256 + 256) : 0;   // snapshot + reciprocals
    char *mem = static_cast<char *>(aux_get(256 + ybytes + sb + pbytes, &st));
    if (st) return st;
    m->aux = reinterpret_cast<LuAux *>(mem);
    m->y = reinterpret_cast<double *>(mem + 256);
    m->scr = reinterpret_cast<double *>(mem + 256 + ybytes);
    m->pout = pbytes ? reinterpret_cast<double *>(mem + 256 + ybytes + sb) : nullptr;
    return DDQD_OK;
}

// side stream + events of the LU's panel-by-panel forward solve, per host thread and device
struct LuSide {
    cudaStream_t ss = nullptr;
    cudaEvent_t start = nullptr, panel = nullptr, done = nullptr;
};
static int lu_side(LuSide **out) {
    static thread_local LuSide res[64];
    LuSide &r = res[current_device()];
    if (!r.ss) {
        DDQD_CUDA_CHECK(cudaStreamCreateWithFlags(&r.ss, cudaStreamNonBlocking));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.start, cudaEventDisableTiming));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.panel, cudaEventDisableTiming));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    }
    *out = &r;
    return DDQD_OK;
}

// DDQD_LU_FWD_OVERLAP=0 keeps the forward solve after the factorisation (A/B measurements)
static bool fwd_overlap_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_FWD_OVERLAP");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

template <int W>
static int lu_solve_w(int64_t n, int pivot, double *A, const double *b, double *x, int64_t *ipiv, int64_t K,
                      int algo, int64_t T, cudaStream_t s, int *info_out) {
    *info_out = 0;
    if (n == 0) return DDQD_OK;
    LuMem mem;
    int rc = lu_mem(W, n, K, &mem);
    if (rc) return rc;
    DDQD_CUDA_CHECK(cudaMemsetAsync(mem.aux, 0, sizeof(LuAux), s));
    size_t usm = 0;
    if ((rc = trsv_setup<W>(&usm))) return rc;
    // The forward solve y := L^{-1} P b runs panel by panel on a side stream, each panel's part
    // (its interchanges applied to y, its diagonal block, the fold of its L21 columns into the rows
    // below) right after the panel is factored, alongside the Schur update -- b is the extra
    // column of a right-looking LU. Every y element still receives l_ij y_j for j ascending with
    // the same operands (its row and its L row move together under the later interchanges),
    // so the bits are those of the solve after the factorisation. The next panel's interchanges
    // wait for the side stream's reads of the L columns they move. Not under stream capture.
    LuSide *sd = nullptr;
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cst) != cudaSuccess) { cudaGetLastError(); cst = cudaStreamCaptureStatusActive; }
    const bool overlap = fwd_overlap_enabled() && cst == cudaStreamCaptureStatusNone && !lu_side(&sd);
    if (overlap) {
        DDQD_CUDA_CHECK(cudaMemcpyAsync(mem.y, b, sizeof(double) * W * (size_t)n, cudaMemcpyDeviceToDevice, s));
        DDQD_CUDA_CHECK(cudaEventRecord(sd->start, s));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(sd->ss, sd->start, 0));
    }
    bool side_pending = false;
    for (int64_t p = 0; p < n; p += K) {
        const int64_t kb = std::min(K, n - p);
        if ((rc = lu_panel_w<W>(n, pivot, A, ipiv, p, kb, mem.aux, mem.scr, mem.scr_bytes, s,
                                side_pending ? sd->done : nullptr, mem.pout))) return rc;
        if (overlap) {
            DDQD_CUDA_CHECK(cudaEventRecord(sd->panel, s));
            DDQD_CUDA_CHECK(cudaStreamWaitEvent(sd->ss, sd->panel, 0));
            if (pivot) {
                lu_yswap_kernel<<<1, 32, 0, sd->ss>>>(mem.y, ipiv, W, n, p, kb);
                DDQD_LAUNCH_CHECK();
            }
            if ((rc = trsv_fwd_block<W>(n, A, mem.y, p, (int)kb, usm, sd->ss))) return rc;
            DDQD_CUDA_CHECK(cudaEventRecord(sd->done, sd->ss));
            side_pending = true;
        }
        const int64_t n2 = n - p - kb;
        if (n2 <= 0) continue;
        MatDesc L21{A + (p + kb) * n + p, n2, kb, n, n * n, 0};
        MatDesc U12{A + p * n + (p + kb), kb, n2, n, n * n, 0};
        MatDesc A22{A + (p + kb) * n + (p + kb), n2, n2, n, n * n, 0};
        if ((rc = run_gemm(W, algo, T, n2, kb, n2, 1, L21, U12, A22, 1, s))) return rc;
    }
    if (overlap) {
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, sd->done, 0));
        prof_begin(5, s);
        if ((rc = trsv_bwd_all<W>(n, A, mem.y, x, usm, s))) return rc;
        prof_end(5, (double)n * (double)n / 2.0, s, "lu backward solve (trsv_diag_blk, trsv_update_co)");
    } else if ((rc = lu_trsv_w<W>(n, A, ipiv, b, x, mem.y, s))) {
        return rc;
    }
    int info_h = 0;
    DDQD_CUDA_CHECK(cudaMemcpyAsync(&info_h, &mem.aux->info, sizeof(int), cudaMemcpyDeviceToHost, s));
    DDQD_CUDA_CHECK(cudaStreamSynchronize(s));
    *info_out = info_h;
    return DDQD_OK;
}

// One panel step on its own (the multi-GPU LU drives the Schur update itself): returns this
// panel's info (first k+1 with an exactly zero pivot, else 0); synchronises.
int lu_panel_impl(int W, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t p, int64_t kb, cudaStream_t s,
                  int *info_out) {
    *info_out = 0;
    LuMem mem;
    int rc = lu_mem(W, n, kb, &mem);
    if (rc) return rc;
    DDQD_CUDA_CHECK(cudaMemsetAsync(mem.aux, 0, sizeof(LuAux), s));
    rc = W == 2 ? lu_panel_w<2>(n, pivot, A, ipiv, p, kb, mem.aux, mem.scr, mem.scr_bytes, s, nullptr, mem.pout)
                : lu_panel_w<4>(n, pivot, A, ipiv, p, kb, mem.aux, mem.scr, mem.scr_bytes, s, nullptr, mem.pout);
    if (rc) return rc;
    int info_h = 0;
    DDQD_CUDA_CHECK(cudaMemcpyAsync(&info_h, &mem.aux->info, sizeof(int), cudaMemcpyDeviceToHost, s));
    DDQD_CUDA_CHECK(cudaStreamSynchronize(s));
    *info_out = info_h;
    return DDQD_OK;
}

// The solve with given factors (asynchronous on s).
int lu_trsv_impl(int W, int64_t n, const double *A, const int64_t *ipiv, const double *b, double *x,
                 cudaStream_t s) {
    if (n == 0) return DDQD_OK;
    LuMem mem;
    int rc = lu_mem(W, n, 1, &mem);
    if (rc) return rc;
    return W == 2 ? lu_trsv_w<2>(n, A, ipiv, b, x, mem.y, s) : lu_trsv_w<4>(n, A, ipiv, b, x, mem.y, s);
}

int lu_solve_impl(int W, int pivot, int64_t n, double *A, const double *b, double *x, int64_t *ipiv, int64_t K,
                  int algo, int64_t T, cudaStream_t s, int *info_out) {
    if (W == 2) return lu_solve_w<2>(n, pivot, A, b, x, ipiv, K, algo, T, s, info_out);
    return lu_solve_w<4>(n, pivot, A, b, x, ipiv, K, algo, T, s, info_out);
}

}  // namespace ddqd
