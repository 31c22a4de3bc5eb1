// addsub.cu -- fused Strassen/Winograd pre- and post-addition kernels (SURVEY.md N7/N8,
// north_star subsystem (3); formulas S:239 / S:248 as fixed in docs/numerics.md s.4).
//
// Both are HBM-bound elementwise DD/QD kernels over a batch of P problems of one level:
//   pre-add : parent X[b] (rows x cols) -> 7 children Y[7b+c] (ceil(rows/2) x ceil(cols/2)),
//             reading the four quadrants once (virtual zero padding at odd edges) and
//             writing the 7 operands of one side (A or B) in one pass;
//   post-add: 7 children products M[7b+c] (hm x hn) -> parent C[b] quadrants, cropping,
//             optionally subtracting from C (beta = 1, the LU update).
// One thread per quadrant position; all additions are dd_add/dd_sub (qd_add/qd_sub) in the
// written left-to-right order, so results are bit-identical to the oracle's explicit-copy
// recursion. Per element: pre-add reads 4 and writes 7 W-word values; post-add reads 7 and
// writes 4 (8 with beta = 1).
#include <algorithm>

#include "common.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

template <int W>
__device__ __forceinline__ typename elem<W>::T ld_or_zero(const double *base, int64_t ps, bool ok) {
    return ok ? elem<W>::load(base, ps) : elem<W>::zero();
}

// One level of pre-additions on the four quadrant values of a position: the 7 operands of
// side 0 (A) or 1 (B); algo 1 = Strassen, 2 = Winograd (numerics.md s.4, S:239 / S:248).
template <class E, int ALGO, int SIDE>
__device__ __forceinline__ void pre_ops(const typename E::T &x11, const typename E::T &x12,
                                        const typename E::T &x21, const typename E::T &x22,
                                        typename E::T o[7]) {
    using T = typename E::T;
    if constexpr (ALGO == 1 && SIDE == 0) {        // Strassen, A side
        o[0] = E::add(x11, x22);                    // P1: A11+A22
        o[1] = E::add(x21, x22);                    // P2: A21+A22
        o[2] = x11;                                 // P3: A11
        o[3] = x22;                                 // P4: A22
        o[4] = E::add(x11, x12);                    // P5: A11+A12
        o[5] = E::sub(x21, x11);                    // P6: A21-A11
        o[6] = E::sub(x12, x22);                    // P7: A12-A22
    } else if constexpr (ALGO == 1 && SIDE == 1) { // Strassen, B side
        o[0] = E::add(x11, x22);                    // P1: B11+B22
        o[1] = x11;                                 // P2: B11
        o[2] = E::sub(x12, x22);                    // P3: B12-B22
        o[3] = E::sub(x21, x11);                    // P4: B21-B11
        o[4] = x22;                                 // P5: B22
        o[5] = E::add(x11, x12);                    // P6: B11+B12
        o[6] = E::add(x21, x22);                    // P7: B21+B22
    } else if constexpr (ALGO == 2 && SIDE == 0) { // Winograd, A side
        const T s1 = E::add(x21, x22);
        const T s2 = E::sub(s1, x11);
        const T s3 = E::sub(x11, x21);
        const T s4 = E::sub(x12, s2);
        o[0] = x11; o[1] = x12; o[2] = s4; o[3] = x22; o[4] = s1; o[5] = s2; o[6] = s3;
    } else {                                        // Winograd, B side
        const T t1 = E::sub(x12, x11);
        const T t2 = E::sub(x22, t1);
        const T t3 = E::sub(x22, x12);
        const T t4 = E::sub(t2, x21);
        o[0] = x11; o[1] = x21; o[2] = x22; o[3] = t4; o[4] = t1; o[5] = t2; o[6] = t3;
    }
}

// One level of post-additions: 7 products -> the 4 quadrant values of a position.
template <class E, int ALGO>
__device__ __forceinline__ void post_ops(const typename E::T p[7], typename E::T &c11,
                                         typename E::T &c12, typename E::T &c21,
                                         typename E::T &c22) {
    using T = typename E::T;
    if constexpr (ALGO == 1) {
        c11 = E::add(E::sub(E::add(p[0], p[3]), p[4]), p[6]);   // ((P1+P4)-P5)+P7
        c12 = E::add(p[2], p[4]);                                // P3+P5
        c21 = E::add(p[1], p[3]);                                // P2+P4
        c22 = E::add(E::add(E::sub(p[0], p[1]), p[2]), p[5]);   // ((P1-P2)+P3)+P6
    } else {
        const T u2 = E::add(p[0], p[5]);      // U2 = M1+M6
        const T u3 = E::add(u2, p[6]);        // U3 = U2+M7
        const T u4 = E::add(u2, p[4]);        // U4 = U2+M5
        c11 = E::add(p[0], p[1]);             // U1 = M1+M2
        c12 = E::add(u4, p[2]);               // U5 = U4+M3
        c21 = E::sub(u3, p[3]);               // U6 = U3-M4
        c22 = E::add(u3, p[4]);               // U7 = U3+M5
    }
}

// side 0 = A operands, side 1 = B operands; algo 1 = Strassen, 2 = Winograd
template <int W, int ALGO, int SIDE, int V>
__global__ void __launch_bounds__(256) pre_add_kernel(int64_t P, MatDesc X, MatDesc Y, int64_t keep_lo,
                                                      int64_t keep_hi) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t hr = Y.rows, hc = Y.cols;
    const int64_t per = hr * hc;
    const int64_t total = P * per;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, rem = t % per, i = rem / hc, j = rem % hc;
        const double *xb = X.p + b * X.bs;
        const bool r2 = i + hr < X.rows, c2 = j + hc < X.cols;
        const T x11 = E::load(xb + i * X.ld + j, X.ps);
        const T x12 = ld_or_zero<W>(xb + i * X.ld + (j + hc), X.ps, c2);
        const T x21 = ld_or_zero<W>(xb + (i + hr) * X.ld + j, X.ps, r2);
        const T x22 = ld_or_zero<W>(xb + (i + hr) * X.ld + (j + hc), X.ps, r2 && c2);
        T o[7];
        pre_ops<E, ALGO, SIDE>(x11, x12, x21, x22, o);
        // children outside [keep_lo, keep_hi) are not stored (the multi-GPU schedules form only
        // the ancestors of a rank's own products)
#pragma unroll
        for (int c = 0; c < 7; c++)
            if (7 * b + c >= keep_lo && 7 * b + c < keep_hi)
                E::store(Y.p + (7 * b + c) * Y.bs + i * Y.ld + j, Y.ps, o[c]);
        if (j == hc - 1 && Y.ld > hc)   // padded leading dimension: fill the gap so no sector is partial
#pragma unroll
            for (int c = 0; c < 7; c++)
                if (7 * b + c >= keep_lo && 7 * b + c < keep_hi)
                    E::store(Y.p + (7 * b + c) * Y.bs + i * Y.ld + hc, Y.ps, E::zero());
    }
}

// The two-level kernels hold 28 DD intermediates per thread (~170 registers unbounded);
// 128-thread CTAs at <= 170 registers (3 per SM-slot group) keep 12 warps per SM in flight
// without spilling: measured best of 128x3 / 128x4 (spills) / 256x1 / 64x6 on c3 (pre-adds
// 11.9 vs 12.0 / 13.9 / 12.7 ms per step).
#ifndef ADD2_THREADS
#define ADD2_THREADS 128
#endif
#ifndef ADD2_MINB
#define ADD2_MINB 3
#endif

// Two recursion levels in one pass (parent X at level j -> 49 grandchildren Y at level
// j+2, child 49b + 7c1 + c2). A thread owns one level-(j+2) position (i, c): it reads the 16
// level-j values the position depends on, forms the 7 level-(j+1) operands at each of the 4
// level-(j+1) positions (i + a*Y.rows, c + e*Y.cols) -- exact zeros where that position is
// the level-(j+1) padding, as the one-level kernel's zero-filled loads would read them --
// and then the 7 grandchildren of each. Same operations in the same order as two launches
// of pre_add_kernel, so bit-identical; the level-(j+1) operands never touch HBM.
template <int W, int ALGO, int SIDE, int V>
__global__ void __launch_bounds__(ADD2_THREADS, ADD2_MINB) pre_add2_kernel(int64_t P, MatDesc X, int64_t h1r,
                                                       int64_t h1c, MatDesc Y) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t hr = Y.rows, hc = Y.cols;
    const int64_t per = hr * hc;
    const int64_t total = P * per;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, rem = t % per, i = rem / hc, j = rem % hc;
        const double *xb = X.p + b * X.bs;
        // all 16 loads first (predicated, zero-filled), so they are in flight together
        T x[4][4];
        bool live[4];
#pragma unroll
        for (int sp = 0; sp < 4; sp++) {
            const int64_t r = i + (sp >> 1) * hr, c = j + (sp & 1) * hc;
            live[sp] = r < h1r && c < h1c;
            const bool r2 = r + h1r < X.rows, c2 = c + h1c < X.cols;
            x[sp][0] = ld_or_zero<W>(xb + r * X.ld + c, X.ps, live[sp]);
            x[sp][1] = ld_or_zero<W>(xb + r * X.ld + (c + h1c), X.ps, live[sp] && c2);
            x[sp][2] = ld_or_zero<W>(xb + (r + h1r) * X.ld + c, X.ps, live[sp] && r2);
            x[sp][3] = ld_or_zero<W>(xb + (r + h1r) * X.ld + (c + h1c), X.ps, live[sp] && r2 && c2);
        }
        T y[4][7];
#pragma unroll
        for (int sp = 0; sp < 4; sp++) {
            if (live[sp]) {
                pre_ops<E, ALGO, SIDE>(x[sp][0], x[sp][1], x[sp][2], x[sp][3], y[sp]);
            } else {
#pragma unroll
                for (int k = 0; k < 7; k++) y[sp][k] = E::zero();
            }
        }
#pragma unroll
        for (int c1 = 0; c1 < 7; c1++) {
            T o[7];
            pre_ops<E, ALGO, SIDE>(y[0][c1], y[1][c1], y[2][c1], y[3][c1], o);
#pragma unroll
            for (int c2 = 0; c2 < 7; c2++)
                E::store(Y.p + (49 * b + 7 * c1 + c2) * Y.bs + i * Y.ld + j, Y.ps, o[c2]);
        }
        // padded leading dimension (the TMA-aligned leaf level): fill the gap as well, so no
        // sector is left partially written (partial sectors cost DRAM read-fills on eviction)
        if (j == hc - 1 && Y.ld > hc)
            for (int g = 0; g < 49; g++) E::store(Y.p + (49 * b + g) * Y.bs + i * Y.ld + hc, Y.ps, E::zero());
    }
}

// Q >= 0 forms only C quadrant Q (0 = C11, 1 = C12, 2 = C21, 3 = C22; the other values and the
// products they alone read are dead code): the host-streamed top level writes C quadrant by
// quadrant so each one's device-to-host copy overlaps the remaining products.
template <int W, int ALGO, int V>
__global__ void __launch_bounds__(256) post_add_kernel(int64_t P, MatDesc M, MatDesc C, int beta) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t hm = M.rows, hn = M.cols;
    const int64_t per = hm * hn;
    const int64_t total = P * per;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, rem = t % per, i = rem / hn, j = rem % hn;
        T p[7];
#pragma unroll
        for (int c = 0; c < 7; c++) p[c] = E::load(M.p + (7 * b + c) * M.bs + i * M.ld + j, M.ps);
        T c11, c12, c21, c22;
        post_ops<E, ALGO>(p, c11, c12, c21, c22);
        double *cb = C.p + b * C.bs;
        const bool r2 = i + hm < C.rows, cc2 = j + hn < C.cols;
        auto put = [&](int64_t r, int64_t c, const T &v) {
            double *q = cb + r * C.ld + c;
            if (beta) E::store(q, C.ps, E::sub(E::load(q, C.ps), v));
            else E::store(q, C.ps, v);
        };
        if (i < C.rows && j < C.cols) put(i, j, c11);
        if (i < C.rows && cc2) put(i, j + hn, c12);
        if (r2 && j < C.cols) put(i + hm, j, c21);
        if (r2 && cc2) put(i + hm, j + hn, c22);
    }
}

// Two recursion levels in one pass (49 level-(j+2) products M, child 49b + 7c1 + c2 -> the
// level-j parent C[b]). A thread owns one level-(j+2) position: it combines the 7 products of
// each level-(j+1) child c1 into that child's 4 quadrant values (positions
// (i + a*M.rows, c + e*M.cols) of the level-(j+1) product), then, at every such position
// inside the level-(j+1) extent h1m x h1n (the one-level kernel crops the rest away), the
// 7 children into C's 4 quadrants. Bit-identical to two launches of post_add_kernel; the
// level-(j+1) products never touch HBM.
template <int W, int ALGO, int V>
__global__ void __launch_bounds__(ADD2_THREADS, ADD2_MINB) post_add2_kernel(int64_t P, MatDesc M, int64_t h1m,
                                                        int64_t h1n, MatDesc C, int beta) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t hm = M.rows, hn = M.cols;
    const int64_t per = hm * hn;
    const int64_t total = P * per;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, rem = t % per, i = rem / hn, j = rem % hn;
        T y[4][7];
#pragma unroll
        for (int c1 = 0; c1 < 7; c1++) {
            T p[7];
#pragma unroll
            for (int c2 = 0; c2 < 7; c2++)
                p[c2] = E::load(M.p + (49 * b + 7 * c1 + c2) * M.bs + i * M.ld + j, M.ps);
            post_ops<E, ALGO>(p, y[0][c1], y[1][c1], y[2][c1], y[3][c1]);
        }
        double *cb = C.p + b * C.bs;
        auto put = [&](int64_t r, int64_t c, const T &v) {
            double *q = cb + r * C.ld + c;
            if (beta) E::store(q, C.ps, E::sub(E::load(q, C.ps), v));
            else E::store(q, C.ps, v);
        };
#pragma unroll
        for (int sp = 0; sp < 4; sp++) {
            const int64_t r = i + (sp >> 1) * hm, c = j + (sp & 1) * hn;
            if (r < h1m && c < h1n) {
                T c11, c12, c21, c22;
                post_ops<E, ALGO>(y[sp], c11, c12, c21, c22);
                const bool r2 = r + h1m < C.rows, cc2 = c + h1n < C.cols;
                if (r < C.rows && c < C.cols) put(r, c, c11);
                if (r < C.rows && cc2) put(r, c + h1n, c12);
                if (r2 && c < C.cols) put(r + h1m, c, c21);
                if (r2 && cc2) put(r + h1m, c + h1n, c22);
            }
        }
    }
}

static unsigned grid_for(int64_t total, int threads = 256) {
    int64_t blocks = (total + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * 16 * 256 / threads;   // grid-stride beyond 16 CTAs (of 256) per SM
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

// Dispatch. `algo` is 1 (Strassen) or 2 (Winograd), optionally | DDQD_ADD_ACCURATE (every
// addition the accurate one, numerics.md s.2-3).
template <int W, int V>
static int pre_dispatch(int algo, int side, int64_t P, const MatDesc &X, const MatDesc &Y, cudaStream_t s,
                        int64_t klo, int64_t khi) {
    const int64_t total = P * Y.rows * Y.cols;
    if (total == 0) return DDQD_OK;
    const unsigned g = grid_for(total);
    prof_begin(1, s);
    if (algo == 1 && side == 0) pre_add_kernel<W, 1, 0, V><<<g, 256, 0, s>>>(P, X, Y, klo, khi);
    else if (algo == 1) pre_add_kernel<W, 1, 1, V><<<g, 256, 0, s>>>(P, X, Y, klo, khi);
    else if (side == 0) pre_add_kernel<W, 2, 0, V><<<g, 256, 0, s>>>(P, X, Y, klo, khi);
    else pre_add_kernel<W, 2, 1, V><<<g, 256, 0, s>>>(P, X, Y, klo, khi);
    DDQD_LAUNCH_CHECK();
    prof_end(1, (double)total * W * 8.0 * 11.0, s, "pre_add_kernel");   // 4 quadrant reads + 7 operand writes
    return DDQD_OK;
}

int launch_pre_add(int W, int algo, int side, int64_t P, const MatDesc &X, const MatDesc &Y,
                   cudaStream_t s, int64_t keep_lo, int64_t keep_hi) {
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    if (keep_hi < 0) keep_hi = 7 * P;
    if (W == 2)
        return acc ? pre_dispatch<2, 2>(algo, side, P, X, Y, s, keep_lo, keep_hi)
                   : pre_dispatch<2, 0>(algo, side, P, X, Y, s, keep_lo, keep_hi);
    return acc ? pre_dispatch<4, 2>(algo, side, P, X, Y, s, keep_lo, keep_hi)
               : pre_dispatch<4, 0>(algo, side, P, X, Y, s, keep_lo, keep_hi);
}

template <int W, int V>
static int pre2_dispatch(int algo, int side, int64_t P, const MatDesc &X, int64_t h1r, int64_t h1c,
                         const MatDesc &Y, cudaStream_t s) {
    const int64_t total = P * Y.rows * Y.cols;
    if (total == 0) return DDQD_OK;
    const unsigned g = grid_for(total, ADD2_THREADS);
    constexpr int TB = ADD2_THREADS;
    prof_begin(1, s);
    if (algo == 1 && side == 0) pre_add2_kernel<W, 1, 0, V><<<g, TB, 0, s>>>(P, X, h1r, h1c, Y);
    else if (algo == 1) pre_add2_kernel<W, 1, 1, V><<<g, TB, 0, s>>>(P, X, h1r, h1c, Y);
    else if (side == 0) pre_add2_kernel<W, 2, 0, V><<<g, TB, 0, s>>>(P, X, h1r, h1c, Y);
    else pre_add2_kernel<W, 2, 1, V><<<g, TB, 0, s>>>(P, X, h1r, h1c, Y);
    DDQD_LAUNCH_CHECK();
    prof_end(1, (double)total * W * 8.0 * 65.0, s, "pre_add2_kernel (two levels)");   // 16 level-j reads + 49 level-(j+2) writes
    return DDQD_OK;
}

int launch_pre_add2(int W, int algo, int side, int64_t P, const MatDesc &X, int64_t h1r,
                    int64_t h1c, const MatDesc &Y, cudaStream_t s) {
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    if (W == 2 && !acc) return pre2_dispatch<2, 0>(algo, side, P, X, h1r, h1c, Y, s);
    // QD: 28 live QD values would spill; the accurate variant keeps the one-level kernels
    set_error("two-level pre-add: canonical DD only");
    return DDQD_ENOTSUP;
}

template <int W, int V>
static int post2_dispatch(int algo, int64_t P, const MatDesc &M, int64_t h1m, int64_t h1n,
                          const MatDesc &C, int beta, cudaStream_t s) {
    const int64_t total = P * M.rows * M.cols;
    if (total == 0) return DDQD_OK;
    const unsigned g = grid_for(total, ADD2_THREADS);
    constexpr int TB = ADD2_THREADS;
    prof_begin(2, s);
    if (algo == 1) post_add2_kernel<W, 1, V><<<g, TB, 0, s>>>(P, M, h1m, h1n, C, beta);
    else post_add2_kernel<W, 2, V><<<g, TB, 0, s>>>(P, M, h1m, h1n, C, beta);
    DDQD_LAUNCH_CHECK();
    prof_end(2, (double)total * W * 8.0 * (beta ? 81.0 : 65.0), s, "post_add2_kernel (two levels)");   // 49 reads + 16 (32) C
    return DDQD_OK;
}

int launch_post_add2(int W, int algo, int64_t P, const MatDesc &M, int64_t h1m, int64_t h1n,
                     const MatDesc &C, int beta, cudaStream_t s) {
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    if (W == 2 && !acc) return post2_dispatch<2, 0>(algo, P, M, h1m, h1n, C, beta, s);
    set_error("two-level post-add: canonical DD only");
    return DDQD_ENOTSUP;
}

template <int W, int V>
static int post_dispatch(int algo, int64_t P, const MatDesc &M, const MatDesc &C, int beta, cudaStream_t s) {
    const int64_t total = P * M.rows * M.cols;
    if (total == 0) return DDQD_OK;
    const unsigned g = grid_for(total);
    prof_begin(2, s);
    if (algo == 1) post_add_kernel<W, 1, V><<<g, 256, 0, s>>>(P, M, C, beta);
    else post_add_kernel<W, 2, V><<<g, 256, 0, s>>>(P, M, C, beta);
    DDQD_LAUNCH_CHECK();
    prof_end(2, (double)total * W * 8.0 * (beta ? 15.0 : 11.0), s, "post_add_kernel");   // 7 product reads + 4 (8) C
    return DDQD_OK;
}

int launch_post_add(int W, int algo, int64_t P, const MatDesc &M, const MatDesc &C, int beta,
                    cudaStream_t s) {
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    if (W == 2) return acc ? post_dispatch<2, 2>(algo, P, M, C, beta, s) : post_dispatch<2, 0>(algo, P, M, C, beta, s);
    return acc ? post_dispatch<4, 2>(algo, P, M, C, beta, s) : post_dispatch<4, 0>(algo, P, M, C, beta, s);
}

// One C quadrant Q of a single parent's post-addition, restricted to the positions
// [r0, r0 + nr) x [c0, c0 + nc) of the hm x hn product grid (hm, hn = M.rows, M.cols): the
// host-streamed top level forms a quadrant block by block as its products complete.
template <int W, int ALGO, int V, int Q>
__global__ void __launch_bounds__(256) post_region_kernel(MatDesc M, MatDesc C, int64_t r0, int64_t nr, int64_t c0,
                                                          int64_t nc) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t hm = M.rows, hn = M.cols;
    const int64_t total = nr * nc;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = r0 + t / nc, j = c0 + t % nc;
        T p[7];
#pragma unroll
        for (int c = 0; c < 7; c++) p[c] = E::load(M.p + c * M.bs + i * M.ld + j, M.ps);
        T c11, c12, c21, c22;
        post_ops<E, ALGO>(p, c11, c12, c21, c22);
        const int64_t r = i + (Q >= 2 ? hm : 0), cc = j + ((Q & 1) ? hn : 0);
        if (r < C.rows && cc < C.cols)
            E::store(C.p + r * C.ld + cc, C.ps, Q == 0 ? c11 : Q == 1 ? c12 : Q == 2 ? c21 : c22);
    }
}

template <int W, int V, int ALGO>
static int post_region_dispatch(int q, const MatDesc &M, const MatDesc &C, int64_t r0, int64_t nr, int64_t c0,
                                int64_t nc, cudaStream_t s) {
    const int64_t total = nr * nc;
    if (total <= 0) return DDQD_OK;
    const unsigned g = grid_for(total);
    static const double reads[2][4] = {{4, 2, 2, 4}, {2, 4, 4, 4}};   // products read: Strassen, Winograd
    prof_begin(2, s);
    if (q == 0) post_region_kernel<W, ALGO, V, 0><<<g, 256, 0, s>>>(M, C, r0, nr, c0, nc);
    else if (q == 1) post_region_kernel<W, ALGO, V, 1><<<g, 256, 0, s>>>(M, C, r0, nr, c0, nc);
    else if (q == 2) post_region_kernel<W, ALGO, V, 2><<<g, 256, 0, s>>>(M, C, r0, nr, c0, nc);
    else post_region_kernel<W, ALGO, V, 3><<<g, 256, 0, s>>>(M, C, r0, nr, c0, nc);
    DDQD_LAUNCH_CHECK();
    prof_end(2, (double)total * W * 8.0 * (reads[ALGO == 2][q] + 1.0), s, "post_region_kernel (one C quadrant)");
    return DDQD_OK;
}

// one C quadrant of a single parent's post-addition (the host-streamed top level), over the
// position block [r0, r0 + nr) x [c0, c0 + nc) (nr < 0: the whole M.rows x M.cols grid)
int launch_post_quad(int W, int algo, int q, const MatDesc &M, const MatDesc &C, cudaStream_t s, int64_t r0,
                     int64_t nr, int64_t c0, int64_t nc) {
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    if (q < 0 || q > 3 || (algo != 1 && algo != 2)) { set_error("launch_post_quad: bad quadrant/algo"); return DDQD_EINVAL; }
    if (nr < 0) { r0 = 0; nr = M.rows; c0 = 0; nc = M.cols; }
#define PQ(WW, VV) return algo == 1 ? post_region_dispatch<WW, VV, 1>(q, M, C, r0, nr, c0, nc, s) \
                                    : post_region_dispatch<WW, VV, 2>(q, M, C, r0, nr, c0, nc, s)
    if (W == 2) { if (acc) PQ(2, 2); PQ(2, 0); }
    if (acc) PQ(4, 2);
    PQ(4, 0);
#undef PQ
}

// ---- post-addition over peer memory (the multi-GPU fused combine) --------
// Same combination as post_add_kernel, but the 7P children are addressed through a device
// array of pointers (each a W-plane hm x hn matrix with row stride ld and plane stride ps) --
// on a multi-GPU node they live on other GPUs and are read over NVLink (CUDA IPC mappings), so
// the gather and the DD/QD combine are one kernel -- and only the position rows [r0, r1) are
// formed (each rank assembles its share of C). Parent b's C quadrant rows sit at i and i + hm.
template <int W, int ALGO, int V>
__global__ void __launch_bounds__(256) post_add_ptr_kernel(int64_t P, const double *const *ch, int64_t hm,
                                                           int64_t hn, int64_t ld, int64_t ps, int64_t r0,
                                                           int64_t r1, MatDesc C, int beta) {
    using E = arith<W, V>;
    using T = typename E::T;
    const int64_t rows = r1 - r0;
    const int64_t per = rows * hn;
    const int64_t total = P * per;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / per, rem = t % per, i = r0 + rem / hn, j = rem % hn;
        T p[7];
#pragma unroll
        for (int c = 0; c < 7; c++) {
            // the children may live in peer GPUs' memory (CUDA IPC mappings): global loads,
            // cached in L2 only (a generic load through the pointer table would also work, slower)
            const double *q = ch[7 * b + c] + i * ld + j;
#pragma unroll
            for (int w = 0; w < W; w++) E::set_word(p[c], w, __ldcg(q + w * ps));
        }
        T c11, c12, c21, c22;
        post_ops<E, ALGO>(p, c11, c12, c21, c22);
        double *cb = C.p + b * C.bs;
        const bool r2 = i + hm < C.rows, cc2 = j + hn < C.cols;
        auto put = [&](int64_t r, int64_t c, const T &v) {
            double *q = cb + r * C.ld + c;
            if (beta) E::store(q, C.ps, E::sub(E::load(q, C.ps), v));
            else E::store(q, C.ps, v);
        };
        if (i < C.rows && j < C.cols) put(i, j, c11);
        if (i < C.rows && cc2) put(i, j + hn, c12);
        if (r2 && j < C.cols) put(i + hm, j, c21);
        if (r2 && cc2) put(i + hm, j + hn, c22);
    }
}

int launch_post_add_ptrs(int W, int algo, int64_t P, const double *const *ch, int64_t hm, int64_t hn,
                         int64_t ld, int64_t ps, int64_t r0, int64_t r1, const MatDesc &C, int beta,
                         cudaStream_t s) {
    const int64_t total = P * (r1 - r0) * hn;
    if (total <= 0) return DDQD_OK;
    const bool acc = (algo & DDQD_ADD_ACCURATE) != 0;
    algo &= 0xff;
    const unsigned g = grid_for(total);
    prof_begin(2, s);
#define DDQD_PP(WW, AA, VV) post_add_ptr_kernel<WW, AA, VV><<<g, 256, 0, s>>>(P, ch, hm, hn, ld, ps, r0, r1, C, beta)
    if (W == 2) {
        if (algo == 1) { if (acc) DDQD_PP(2, 1, 2); else DDQD_PP(2, 1, 0); }
        else { if (acc) DDQD_PP(2, 2, 2); else DDQD_PP(2, 2, 0); }
    } else {
        if (algo == 1) { if (acc) DDQD_PP(4, 1, 2); else DDQD_PP(4, 1, 0); }
        else { if (acc) DDQD_PP(4, 2, 2); else DDQD_PP(4, 2, 0); }
    }
#undef DDQD_PP
    DDQD_LAUNCH_CHECK();
    prof_end(2, (double)total * W * 8.0 * (beta ? 15.0 : 11.0), s, "post_add_ptrs_kernel (peer pointers)");
    return DDQD_OK;
}

// ---- elementwise arithmetic layer (parity tests of ddqd_arith.cuh) ---------------------
template <int W>
__global__ void elementwise_kernel(int op, int64_t count, const double *x, const double *y,
                                   const double *w, double *z) {
    using E = elem<W>;
    using T = typename E::T;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const T a = E::load(x + i, count), b = E::load(y + i, count);
        T r;
        if (op == 0) r = E::add(a, b);
        else if (op == 1) r = E::sub(a, b);
        else if (op == 4) r = E::madd(a, b, E::load(w + i, count));
        else if (op == 5) r = E::madd_fused(a, b, E::load(w + i, count));
        else if (op == 6) r = E::add_acc(a, b);
        else if (op == 7) r = E::sub_acc(a, b);
        else if (op == 8) r = E::madd_acc(a, b, E::load(w + i, count));
        else if constexpr (W == 2) {
            r = (op == 2) ? dd_mul(a, b) : dd_div(a, b);
        } else {
            r = (op == 2) ? qd_mul(a, b) : qd_div(a, b);
        }
        E::store(z + i, count, r);
    }
}

int launch_elementwise(int W, int op, int64_t count, const double *x, const double *y,
                       const double *w, double *z, cudaStream_t s) {
    if (count == 0) return DDQD_OK;
    const unsigned g = grid_for(count);
    if (W == 2) elementwise_kernel<2><<<g, 256, 0, s>>>(op, count, x, y, w, z);
    else elementwise_kernel<4><<<g, 256, 0, s>>>(op, count, x, y, w, z);
    DDQD_LAUNCH_CHECK();
    return DDQD_OK;
}

// ---- the last recursion level fused with its leaves (tiny leaves) ------------------------------
// For leaves of at most 32 x 32 x 32 (Strassen/Winograd(32) at n = 1025: 33^3 parents, 17^3
// leaves) one CTA takes one level-(d-1) parent: its threads form the 7 A and 7 B children in
// shared memory straight from the parent in global memory (pre_add_kernel's formulas, reads
// outside the parent are exact zeros -- the virtual padding), then each thread owns output
// positions (i, j) of the children: it forms the 7 products at (i, j) (7 independent chains,
// acc from +0, k ascending, E::madd) and combines them with the post-addition formulas straight
// into the parent's C (crop, beta). Every element sees the operation sequence of
// pre_add_kernel -> leaf -> post_add_kernel, so the bits are those of the unfused schedule; the
// children and the products never touch HBM.
constexpr int kFusedNT = 160;   // a 17 x 17 leaf: 17 rows x 9 position pairs = 153 DD tasks

struct FusedLastDims {
    int hm, hl, hn;   // child (leaf) dims
};

__host__ __device__ inline size_t fused_last_smem_doubles(int W, int hm, int hl, int hn) {
    return (size_t)7 * W * hm * hl + (size_t)7 * W * hl * hn;
}

template <int W, int ALGO, int VA, int MV>
__global__ void __launch_bounds__(kFusedNT) fused_last_kernel(int64_t P, MatDesc X, MatDesc Y, MatDesc C, int beta,
                                                              FusedLastDims dd) {
    using EA = arith<W, VA>;   // additions (canonical or accurate)
    using EM = arith<W, MV>;   // the leaf's multiply-add
    using T = typename EA::T;
    extern __shared__ double fs[];
    const int hm = dd.hm, hl = dd.hl, hn = dd.hn;
    const size_t psa = (size_t)hm * hl, psb = (size_t)hl * hn;
    double *CA = fs;                              // [7][W][hm][hl]
    double *CB = fs + (size_t)7 * W * psa;        // [7][W][hl][hn]
    const int tid = threadIdx.x;
    auto sld = [&](const double *base, size_t ps, int e) {
        T v;
#pragma unroll
        for (int w = 0; w < W; w++) EA::set_word(v, w, base[w * ps + e]);
        return v;
    };
    auto sst = [&](double *base, size_t ps, int e, const T &v) {
#pragma unroll
        for (int w = 0; w < W; w++) base[w * ps + e] = EA::word(v, w);
    };
    const int per = hm * hn;
    for (int64_t b = blockIdx.x; b < P; b += gridDim.x) {
        const double *xb = X.p + b * X.bs, *yb = Y.p + b * Y.bs;
        // 1. the 7 children of each side, read from the parent (4 quadrant values, zero outside)
        for (int e = tid; e < hm * hl; e += kFusedNT) {
            const int i = e / hl, k = e % hl;
            const bool r2 = i + hm < X.rows, c2 = k + hl < X.cols;
            const T x11 = ld_or_zero<W>(xb + i * X.ld + k, X.ps, true);
            const T x12 = ld_or_zero<W>(xb + i * X.ld + k + hl, X.ps, c2);
            const T x21 = ld_or_zero<W>(xb + (i + hm) * X.ld + k, X.ps, r2);
            const T x22 = ld_or_zero<W>(xb + (i + hm) * X.ld + k + hl, X.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 0>(x11, x12, x21, x22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) sst(CA + (size_t)c * W * psa, psa, e, o[c]);
        }
        for (int e = tid; e < hl * hn; e += kFusedNT) {
            const int k = e / hn, j = e % hn;
            const bool r2 = k + hl < Y.rows, c2 = j + hn < Y.cols;
            const T y11 = ld_or_zero<W>(yb + k * Y.ld + j, Y.ps, true);
            const T y12 = ld_or_zero<W>(yb + k * Y.ld + j + hn, Y.ps, c2);
            const T y21 = ld_or_zero<W>(yb + (k + hl) * Y.ld + j, Y.ps, r2);
            const T y22 = ld_or_zero<W>(yb + (k + hl) * Y.ld + j + hn, Y.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 1>(y11, y12, y21, y22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) sst(CB + (size_t)c * W * psb, psb, e, o[c]);
        }
        __syncthreads();
        // 2. per position: the 7 products (independent chains), then the post-additions. A
        // thread owns RP positions of one row (i, j .. j+RP-1), so each A value it loads feeds RP
        // chains (shared-memory loads per madd: (1 + RP) / RP words instead of 2)
        double *cb = C.p + b * C.bs;
        constexpr int RP = W == 2 ? 2 : 1;
        const int hnb = (hn + RP - 1) / RP;
        auto post_put = [&](int i, int j, const T pv[7]) {
            T c11, c12, c21, c22;
            post_ops<EA, ALGO>(pv, c11, c12, c21, c22);
            const bool r2 = i + hm < C.rows, cc2 = j + hn < C.cols;
            auto put = [&](int64_t r, int64_t c, const T &v) {
                double *q = cb + r * C.ld + c;
                if (beta) EA::store(q, C.ps, EA::sub(EA::load(q, C.ps), v));
                else EA::store(q, C.ps, v);
            };
            if (i < C.rows && j < C.cols) put(i, j, c11);
            if (i < C.rows && cc2) put(i, j + hn, c12);
            if (r2 && j < C.cols) put(i + hm, j, c21);
            if (r2 && cc2) put(i + hm, j + hn, c22);
        };
        for (int e = tid; e < hm * hnb; e += kFusedNT) {
            const int i = e / hnb, j0 = (e % hnb) * RP;
            T pv[RP][7];
#pragma unroll
            for (int r = 0; r < RP; r++)
#pragma unroll
                for (int c = 0; c < 7; c++) pv[r][c] = EM::zero();
            for (int k = 0; k < hl; k++) {
#pragma unroll
                for (int c = 0; c < 7; c++) {
                    const T a = sld(CA + (size_t)c * W * psa, psa, i * hl + k);
#pragma unroll
                    for (int r = 0; r < RP; r++) {
                        const int jj = j0 + r < hn ? j0 + r : j0;   // (a duplicate, never stored)
                        pv[r][c] = EM::madd(pv[r][c], a, sld(CB + (size_t)c * W * psb, psb, k * hn + jj));
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < RP; r++)
                if (j0 + r < hn) post_put(i, j0 + r, pv[r]);
        }
        __syncthreads();   // the children buffers are reused by the next parent
    }
}

// The fused last level, DD, second form (the default; DDQD_FUSED_S=0 selects the first): the
// children sit in shared memory with their two words side by side (one 16-byte load per
// value) and a thread owns RP positions (i, j0 + r * ceil(hn / RP)) of one row (RP = 1 in
// use: one thread per position, so a CTA has as many warps as a 17 x 17 leaf has positions /
// 32 and three CTAs share an SM). S > 0 fixes the S^3 leaf at compile time (S = 17: the
// paper's n = 1025 with n_min = 32) and unrolls the k loop; NT = 0 takes the block size at
// run time. Same per-element operation sequence as fused_last_kernel.
template <int ALGO, int VA, int MV, int S, int NT, int RP>
__global__ void __launch_bounds__(NT ? NT : 1024, NT ? 3 : 1) fused_last_s_kernel(int64_t P, MatDesc X, MatDesc Y, MatDesc C, int beta,
                                                                   FusedLastDims dd) {
    using EA = arith<2, VA>;
    using EM = arith<2, MV>;
    using T = typename EA::T;
    extern __shared__ double2 fs2[];
    // S = 0: the dims at run time (any leaf shape that fits)
    const int hm = S ? S : dd.hm, hl = S ? S : dd.hl, hn = S ? S : dd.hn;
    const int psa = hm * hl, psb = hl * hn, HNB = (hn + RP - 1) / RP;
    double2 *CA = fs2;              // [7][hm][hl] (hi, lo)
    double2 *CB = fs2 + 7 * psa;    // [7][hl][hn]
    const int tid = threadIdx.x, nt = NT ? NT : blockDim.x;
    auto l2 = [](const double2 &v) { T t; t.hi = v.x; t.lo = v.y; return t; };
    for (int64_t b = blockIdx.x; b < P; b += gridDim.x) {
        const double *xb = X.p + b * X.bs, *yb = Y.p + b * Y.bs;
        for (int e = tid; e < psa; e += nt) {
            const int i = e / hl, k = e % hl;
            const bool r2 = i + hm < X.rows, c2 = k + hl < X.cols;
            const T x11 = ld_or_zero<2>(xb + i * X.ld + k, X.ps, true);
            const T x12 = ld_or_zero<2>(xb + i * X.ld + k + hl, X.ps, c2);
            const T x21 = ld_or_zero<2>(xb + (i + hm) * X.ld + k, X.ps, r2);
            const T x22 = ld_or_zero<2>(xb + (i + hm) * X.ld + k + hl, X.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 0>(x11, x12, x21, x22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) CA[c * psa + e] = make_double2(o[c].hi, o[c].lo);
        }
        for (int e = tid; e < psb; e += nt) {
            const int k = e / hn, j = e % hn;
            const bool r2 = k + hl < Y.rows, c2 = j + hn < Y.cols;
            const T y11 = ld_or_zero<2>(yb + k * Y.ld + j, Y.ps, true);
            const T y12 = ld_or_zero<2>(yb + k * Y.ld + j + hn, Y.ps, c2);
            const T y21 = ld_or_zero<2>(yb + (k + hl) * Y.ld + j, Y.ps, r2);
            const T y22 = ld_or_zero<2>(yb + (k + hl) * Y.ld + j + hn, Y.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 1>(y11, y12, y21, y22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) CB[c * psb + e] = make_double2(o[c].hi, o[c].lo);
        }
        __syncthreads();
        double *cb = C.p + b * C.bs;
        for (int e = tid; e < hm * HNB; e += nt) {
            const int i = e / HNB, j0 = e % HNB;
            int jj[RP];
#pragma unroll
            for (int r = 0; r < RP; r++) jj[r] = j0 + r * HNB < hn ? j0 + r * HNB : j0;   // (a duplicate, never stored)
            T pv[RP][7];
#pragma unroll
            for (int r = 0; r < RP; r++)
#pragma unroll
                for (int c = 0; c < 7; c++) pv[r][c] = EM::zero();
#pragma unroll
            for (int k = 0; k < hl; k++) {
#pragma unroll
                for (int c = 0; c < 7; c++) {
                    const T a = l2(CA[c * psa + i * hl + k]);
#pragma unroll
                    for (int r = 0; r < RP; r++) pv[r][c] = EM::madd(pv[r][c], a, l2(CB[c * psb + k * hn + jj[r]]));
                }
            }
#pragma unroll
            for (int r = 0; r < RP; r++) {
                const int j = j0 + r * HNB;
                if (j >= hn) continue;
                T c11, c12, c21, c22;
                post_ops<EA, ALGO>(pv[r], c11, c12, c21, c22);
                const bool r2 = i + hm < C.rows, cc2 = j + hn < C.cols;
                auto put = [&](int64_t rr, int64_t cc, const T &v) {
                    double *q = cb + rr * C.ld + cc;
                    if (beta) EA::store(q, C.ps, EA::sub(EA::load(q, C.ps), v));
                    else EA::store(q, C.ps, v);
                };
                if (i < C.rows && j < C.cols) put(i, j, c11);
                if (i < C.rows && cc2) put(i, j + hn, c12);
                if (r2 && j < C.cols) put(i + hm, j, c21);
                if (r2 && cc2) put(i + hm, j + hn, c22);
            }
        }
        __syncthreads();   // the children buffers are reused by the next parent
    }
}

// QD: the same fused last level with one product chain per thread. A QD value is two 16-byte
// halves (w0, w1) and (w2, w3) in separate shared-memory planes; the 7 * hm * hn products
// (thread t: child c = t / (hm hn), position t % (hm hn), acc from +0, k ascending) go to
// their own shared buffer, then one thread per position forms the post-additions. 1024
// threads per CTA (one CTA per SM: the QD children of a 17^3 level take 129 KB).
template <int ALGO, int VA, int MV, int NQ>
__global__ void __launch_bounds__(NQ, 1) fused_last_q_kernel(int64_t P, MatDesc X, MatDesc Y, MatDesc C, int beta,
                                                               FusedLastDims dd) {
    using EA = arith<4, VA>;
    using EM = arith<4, MV>;
    using T = typename EA::T;
    extern __shared__ double2 fq[];
    const int hm = dd.hm, hl = dd.hl, hn = dd.hn;
    const int psa = hm * hl, psb = hl * hn, per = hm * hn;
    double2 *CA = fq;                    // [7][2][hm*hl]
    double2 *CB = CA + 14 * psa;         // [7][2][hl*hn]
    double2 *PR = CB + 14 * psb;         // [7][2][hm*hn] products
    const int tid = threadIdx.x, nt = blockDim.x;
    auto ldq = [](const double2 *base, int ps, int e) {
        const double2 u = base[e], v = base[ps + e];
        T t; t.w[0] = u.x; t.w[1] = u.y; t.w[2] = v.x; t.w[3] = v.y; return t;
    };
    auto stq = [](double2 *base, int ps, int e, const T &t) {
        base[e] = make_double2(t.w[0], t.w[1]);
        base[ps + e] = make_double2(t.w[2], t.w[3]);
    };
    for (int64_t b = blockIdx.x; b < P; b += gridDim.x) {
        const double *xb = X.p + b * X.bs, *yb = Y.p + b * Y.bs;
        for (int e = tid; e < psa; e += nt) {
            const int i = e / hl, k = e % hl;
            const bool r2 = i + hm < X.rows, c2 = k + hl < X.cols;
            const T x11 = ld_or_zero<4>(xb + i * X.ld + k, X.ps, true);
            const T x12 = ld_or_zero<4>(xb + i * X.ld + k + hl, X.ps, c2);
            const T x21 = ld_or_zero<4>(xb + (i + hm) * X.ld + k, X.ps, r2);
            const T x22 = ld_or_zero<4>(xb + (i + hm) * X.ld + k + hl, X.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 0>(x11, x12, x21, x22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) stq(CA + 2 * c * psa, psa, e, o[c]);
        }
        for (int e = tid; e < psb; e += nt) {
            const int k = e / hn, j = e % hn;
            const bool r2 = k + hl < Y.rows, c2 = j + hn < Y.cols;
            const T y11 = ld_or_zero<4>(yb + k * Y.ld + j, Y.ps, true);
            const T y12 = ld_or_zero<4>(yb + k * Y.ld + j + hn, Y.ps, c2);
            const T y21 = ld_or_zero<4>(yb + (k + hl) * Y.ld + j, Y.ps, r2);
            const T y22 = ld_or_zero<4>(yb + (k + hl) * Y.ld + j + hn, Y.ps, r2 && c2);
            T o[7];
            pre_ops<EA, ALGO, 1>(y11, y12, y21, y22, o);
#pragma unroll
            for (int c = 0; c < 7; c++) stq(CB + 2 * c * psb, psb, e, o[c]);
        }
        __syncthreads();
        for (int t = tid; t < 7 * per; t += nt) {
            const int c = t / per, pos = t % per, i = pos / hn, j = pos % hn;
            const double2 *ca = CA + 2 * c * psa + i * hl, *cbp = CB + 2 * c * psb + j;
            T acc = EM::zero();
            for (int k = 0; k < hl; k++) acc = EM::madd(acc, ldq(ca, psa, k), ldq(cbp, psb, k * hn));
            stq(PR + 2 * c * per, per, pos, acc);
        }
        __syncthreads();
        double *cb = C.p + b * C.bs;
        for (int pos = tid; pos < per; pos += nt) {
            const int i = pos / hn, j = pos % hn;
            T pv[7];
#pragma unroll
            for (int c = 0; c < 7; c++) pv[c] = ldq(PR + 2 * c * per, per, pos);
            T c11, c12, c21, c22;
            post_ops<EA, ALGO>(pv, c11, c12, c21, c22);
            const bool r2 = i + hm < C.rows, cc2 = j + hn < C.cols;
            auto put = [&](int64_t rr, int64_t cc, const T &v) {
                double *q = cb + rr * C.ld + cc;
                if (beta) EA::store(q, C.ps, EA::sub(EA::load(q, C.ps), v));
                else EA::store(q, C.ps, v);
            };
            if (i < C.rows && j < C.cols) put(i, j, c11);
            if (i < C.rows && cc2) put(i, j + hn, c12);
            if (r2 && j < C.cols) put(i + hm, j, c21);
            if (r2 && cc2) put(i + hm, j + hn, c22);
        }
        __syncthreads();   // the buffers are reused by the next parent
    }
}

size_t fused_last_q_smem(int64_t hm, int64_t hl, int64_t hn) {
    if (hm < 1 || hl < 1 || hn < 1 || hm > 32 || hl > 32 || hn > 32) return 0;
    const size_t b = sizeof(double) * 4 * 7 * (size_t)(hm * hl + hl * hn + hm * hn);
    return b <= 220 * 1024 ? b : 0;
}

template <int ALGO, int VA, int MV, int NQ>
static int fused_last_q_go2(int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C, int beta,
                            FusedLastDims dd, cudaStream_t s) {
    auto kern = fused_last_q_kernel<ALGO, VA, MV, NQ>;
    const size_t smem = fused_last_q_smem(dd.hm, dd.hl, dd.hn);
    static bool attr[64] = {};
    if (!attr[current_device()]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr[current_device()] = true;
    }
    const int64_t blocks = P < 8 * sm_count() ? P : 8 * sm_count();
    const int nt = (int)std::min<int64_t>(NQ, (7 * dd.hm * (int64_t)dd.hn + 31) / 32 * 32);
    prof_begin(0, s);
    kern<<<(unsigned)blocks, nt, smem, s>>>(P, X, Y, C, beta, dd);
    DDQD_LAUNCH_CHECK();
    prof_end(0, 7.0 * dd.hm * (double)dd.hl * dd.hn * (double)P, s, "fused_last_q_kernel (pre-add + leaves + post-add)");
    return DDQD_OK;
}

// 768 threads: QD Strassen(32) at n = 1025, ms of the fused level: 512 / 768 / 1024 threads
// 8.59 / 8.55 / 8.76 (1024 spills at 64 registers); unfused leaf 8.88 plus the additions
template <int ALGO, int VA, int MV>
static int fused_last_q_go(int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C, int beta,
                           FusedLastDims dd, cudaStream_t s) {
    return fused_last_q_go2<ALGO, VA, MV, 768>(P, X, Y, C, beta, dd, s);
}

static int fused_s_mode() {
    static int m = -1;
    if (m < 0) {
        const char *e = getenv("DDQD_FUSED_S");   // 0: the first fused kernel (A/B)
        m = e ? atoi(e) : 1;
    }
    return m;
}

template <int ALGO, int VA, int MV, int S, int NT, int RP>
static int fused_last_s_go(int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C, int beta,
                           FusedLastDims dd, cudaStream_t s) {
    auto kern = fused_last_s_kernel<ALGO, VA, MV, S, NT, RP>;
    const size_t smem = sizeof(double2) * 7 * ((size_t)dd.hm * dd.hl + (size_t)dd.hl * dd.hn);
    static bool attr[64] = {};
    if (!attr[current_device()]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr[current_device()] = true;
    }
    const int64_t per_sm = (int64_t)((228 * 1024) / (smem + 1024));
    const int64_t cap = (per_sm < 1 ? 1 : per_sm) * 8 * sm_count();
    const int64_t blocks = P < cap ? P : cap;
    prof_begin(0, s);
    // NT = 0: one thread per output position of a leaf (a multiple of 32, at most 1024)
    const int nt = NT ? NT : (int)std::min<int64_t>(1024, (dd.hm * (int64_t)dd.hn + 31) / 32 * 32);
    kern<<<(unsigned)blocks, nt, smem, s>>>(P, X, Y, C, beta, dd);
    DDQD_LAUNCH_CHECK();
    prof_end(0, 7.0 * dd.hm * (double)dd.hl * dd.hn * (double)P, s, "fused_last_s_kernel (pre-add + leaves + post-add)");
    return DDQD_OK;
}

template <int ALGO, int VA, int MV>
static int fused_last_s_pick(FusedLastDims dd, int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C,
                             int beta, cudaStream_t s) {
    // measured on DD Strassen(32), n = 1025 (17^3 leaves), ms of the fused level: 160 threads x
    // 2 positions (fused_last_kernel) 1.14; unrolled 17^3 with 160 x 2 / 128 x 3 positions
    // 1.27 / 1.26; one position per thread, 320 threads: run-time dims 0.96, unrolled 0.89
    if (dd.hm == 17 && dd.hl == 17 && dd.hn == 17) return fused_last_s_go<ALGO, VA, MV, 17, 320, 1>(P, X, Y, C, beta, dd, s);
    return fused_last_s_go<ALGO, VA, MV, 0, 0, 1>(P, X, Y, C, beta, dd, s);
}

// shared memory a fused last level needs (bytes), or 0 when the leaves are too large for it
size_t fused_last_q_smem(int64_t hm, int64_t hl, int64_t hn);
size_t fused_last_smem(int W, int64_t hm, int64_t hl, int64_t hn) {
    if (W == 4) return fused_last_q_smem(hm, hl, hn);
    if (hm < 1 || hl < 1 || hn < 1 || hm > 32 || hl > 32 || hn > 32) return 0;
    const size_t b = sizeof(double) * fused_last_smem_doubles(W, (int)hm, (int)hl, (int)hn);
    return b <= 220 * 1024 ? b : 0;
}

template <int W, int ALGO, int VA, int MV>
static int fused_last_go(int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C, int beta, FusedLastDims dd,
                         size_t smem, cudaStream_t s) {
    auto kern = fused_last_kernel<W, ALGO, VA, MV>;
    static bool attr[64] = {};
    if (!attr[current_device()]) {
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr[current_device()] = true;
    }
    const int64_t per_sm = (int64_t)((228 * 1024) / (smem + 1024));
    const int64_t cap = (per_sm < 1 ? 1 : per_sm) * 8 * sm_count();
    const int64_t blocks = P < cap ? P : cap;
    prof_begin(0, s);
    kern<<<(unsigned)blocks, kFusedNT, smem, s>>>(P, X, Y, C, beta, dd);
    DDQD_LAUNCH_CHECK();
    prof_end(0, 7.0 * dd.hm * (double)dd.hl * dd.hn * (double)P, s, "fused_last_kernel (pre-add + leaves + post-add)");
    return DDQD_OK;
}

// P parents X (A side), Y (B side) -> parents C, one recursion level + its leaves in one kernel.
// mv: the leaf's arithmetic variant (0 canonical, 1 fused madd, 2 accurate adds everywhere).
int launch_fused_last(int W, int algo, int mv, int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C,
                      int beta, int64_t hm, int64_t hl, int64_t hn, cudaStream_t s) {
    const size_t smem = fused_last_smem(W, hm, hl, hn);
    if (!smem) { set_error("fused last level: leaves too large"); return DDQD_EINVAL; }
    if (P == 0) return DDQD_OK;
    const FusedLastDims dd{(int)hm, (int)hl, (int)hn};
    algo &= 0xff;
    if (W == 2 && fused_s_mode() > 0) {
        int rc = 1;
        if (algo == 1) rc = mv == 1 ? fused_last_s_pick<1, 0, 1>(dd, P, X, Y, C, beta, s)
                          : mv == 2 ? fused_last_s_pick<1, 2, 2>(dd, P, X, Y, C, beta, s)
                                    : fused_last_s_pick<1, 0, 0>(dd, P, X, Y, C, beta, s);
        else rc = mv == 1 ? fused_last_s_pick<2, 0, 1>(dd, P, X, Y, C, beta, s)
                  : mv == 2 ? fused_last_s_pick<2, 2, 2>(dd, P, X, Y, C, beta, s)
                            : fused_last_s_pick<2, 0, 0>(dd, P, X, Y, C, beta, s);
        if (rc != 1) return rc;
    }
    if (W == 4 && fused_s_mode() > 0) {
        if (algo == 1) return mv == 1 ? fused_last_q_go<1, 0, 1>(P, X, Y, C, beta, dd, s)
                            : mv == 2 ? fused_last_q_go<1, 2, 2>(P, X, Y, C, beta, dd, s)
                                      : fused_last_q_go<1, 0, 0>(P, X, Y, C, beta, dd, s);
        return mv == 1 ? fused_last_q_go<2, 0, 1>(P, X, Y, C, beta, dd, s)
             : mv == 2 ? fused_last_q_go<2, 2, 2>(P, X, Y, C, beta, dd, s)
                       : fused_last_q_go<2, 0, 0>(P, X, Y, C, beta, dd, s);
    }
#define FL_GO(WW, AL, VA, MV) return fused_last_go<WW, AL, VA, MV>(P, X, Y, C, beta, dd, smem, s)
    if (W == 2) {
        if (algo == 1) { if (mv == 1) FL_GO(2, 1, 0, 1); if (mv == 2) FL_GO(2, 1, 2, 2); FL_GO(2, 1, 0, 0); }
        if (mv == 1) FL_GO(2, 2, 0, 1);
        if (mv == 2) FL_GO(2, 2, 2, 2);
        FL_GO(2, 2, 0, 0);
    }
    if (algo == 1) { if (mv == 1) FL_GO(4, 1, 0, 1); if (mv == 2) FL_GO(4, 1, 2, 2); FL_GO(4, 1, 0, 0); }
    if (mv == 1) FL_GO(4, 2, 0, 1);
    if (mv == 2) FL_GO(4, 2, 2, 2);
    FL_GO(4, 2, 0, 0);
#undef FL_GO
}

}  // namespace ddqd
