// lu.cu -- blocked right-looking DD LU with partial pivoting and the triangular solves
// (north_star subsystem (5); PAPER.md P:121-133 steps 1-3, Eq. (2)
// P:124-126; pivoting per BJ:11). Op sequences: docs/numerics.md s.5.
//
// Per panel of width K: for each column k a single-CTA kernel does the DD argmax (ties to
// the lowest row), the full-row interchange, the reciprocal of the pivot and the scaling
// of the column; a 2-D kernel does the rank-1 update of the rest of the panel. U12 is
// formed by a shared-memory forward substitution (one CTA per column strip), and the
// Schur update A22 := A22 - L21 U12 (the underlined term of P:131) is the library GEMM
// (Block/Strassen/Winograd) with beta = 1. Nothing returns to the host until the end.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "ddqd_arith.cuh"

namespace ddqd {

void *aux_get(size_t bytes, int *status);   // abi.cu (separate from the GEMM workspace)

__device__ __forceinline__ dd ldA(const double *A, int64_t n, int64_t i, int64_t j) {
    return dd{A[i * n + j], A[n * n + i * n + j]};
}
__device__ __forceinline__ void stA(double *A, int64_t n, int64_t i, int64_t j, dd v) {
    A[i * n + j] = v.hi;
    A[n * n + i * n + j] = v.lo;
}

struct LuAux {
    int info;
    int skip;
    double rinv_hi, rinv_lo;
};

// argmax |a_ik| over i >= k (first index on ties), swap rows k <-> r over all n columns,
// rinv = 1 / a_kk (dd_div), a_ik := a_ik * rinv for i > k.
__global__ void __launch_bounds__(1024) lu_pivot_kernel(double *A, int64_t n, int64_t k,
                                                        int64_t *ipiv, LuAux *aux) {
    __shared__ double sh_hi[1024], sh_lo[1024];
    __shared__ int64_t sh_idx[1024];
    __shared__ int sh_skip;
    __shared__ double sh_r[2];
    const int tid = threadIdx.x;
    dd best{0.0, 0.0};
    int64_t bidx = -1;
    for (int64_t i = k + tid; i < n; i += blockDim.x) {
        dd v = ldA(A, n, i, k);
        if (bidx < 0 || dd_abs_gt(v, best)) { best = v; bidx = i; }
    }
    sh_hi[tid] = best.hi; sh_lo[tid] = best.lo; sh_idx[tid] = bidx;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
        if (tid < off) {
            const int64_t oi = sh_idx[tid + off];
            if (oi >= 0) {
                const dd o{sh_hi[tid + off], sh_lo[tid + off]};
                const dd me{sh_hi[tid], sh_lo[tid]};
                const int64_t mi = sh_idx[tid];
                bool take;
                if (mi < 0) take = true;
                else if (dd_abs_gt(o, me)) take = true;
                else if (dd_abs_gt(me, o)) take = false;
                else take = oi < mi;
                if (take) { sh_hi[tid] = o.hi; sh_lo[tid] = o.lo; sh_idx[tid] = oi; }
            }
        }
        __syncthreads();
    }
    const int64_t r = sh_idx[0];
    if (r != k) {
        for (int64_t j = tid; j < n; j += blockDim.x) {
            const dd a = ldA(A, n, k, j), c = ldA(A, n, r, j);
            stA(A, n, k, j, c);
            stA(A, n, r, j, a);
        }
    }
    __syncthreads();
    if (tid == 0) {
        ipiv[k] = r;
        const dd piv = ldA(A, n, k, k);
        if (piv.hi == 0.0) {
            if (aux->info == 0) aux->info = (int)(k + 1);
            sh_skip = 1;
        } else {
            const dd rv = dd_div(dd{1.0, 0.0}, piv);
            sh_r[0] = rv.hi; sh_r[1] = rv.lo;
            sh_skip = 0;
        }
        aux->skip = sh_skip;
        aux->rinv_hi = sh_r[0]; aux->rinv_lo = sh_r[1];
    }
    __syncthreads();
    if (sh_skip) return;
    const dd rinv{sh_r[0], sh_r[1]};
    for (int64_t i = k + 1 + tid; i < n; i += blockDim.x) stA(A, n, i, k, dd_mul(ldA(A, n, i, k), rinv));
}

// a_ij := a_ij - l_ik * a_kj for i in (k, n), j in (k, jend)
__global__ void lu_rank1_kernel(double *A, int64_t n, int64_t k, int64_t jend, const LuAux *aux) {
    if (aux->skip) return;
    const int64_t j = k + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = k + 1 + (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    if (j >= jend || i >= n) return;
    stA(A, n, i, j, dd_sub(ldA(A, n, i, j), dd_mul(ldA(A, n, i, k), ldA(A, n, k, j))));
}

// U12 := L11^{-1} A12 (unit lower, forward substitution in row order), one CTA per strip
// of cw columns held in shared memory; thread r owns panel row r and prefetches its next
// multiplier l_{r,i+1} during step i (row-major, so consecutive i are contiguous).
__global__ void __launch_bounds__(1024) lu_trsm_kernel(double *A, int64_t n, int64_t p, int64_t kb,
                                                       int64_t c0, int cw) {
    extern __shared__ double tile[];   // [2][kb][cw]
    const int64_t col0 = c0 + (int64_t)blockIdx.x * cw;
    const int ncols = (int)((n - col0) < cw ? (n - col0) : cw);
    for (int64_t e = threadIdx.x; e < kb * cw; e += blockDim.x) {
        const int64_t r = e / cw, c = e % cw;
        if (c < ncols) {
            const dd v = ldA(A, n, p + r, col0 + c);
            tile[r * cw + c] = v.hi;
            tile[kb * cw + r * cw + c] = v.lo;
        }
    }
    const int64_t r = threadIdx.x;   // blockDim.x >= kb (host guarantees)
    dd lnext{0.0, 0.0};
    if (r > 0 && r < kb) lnext = ldA(A, n, p + r, p);
    for (int64_t i = 0; i < kb; i++) {
        __syncthreads();
        const dd l = lnext;
        if (i + 1 < r && r < kb) lnext = ldA(A, n, p + r, p + i + 1);
        if (r > i && r < kb) {
            for (int c = 0; c < ncols; c++) {
                const dd u{tile[i * cw + c], tile[kb * cw + i * cw + c]};
                dd a{tile[r * cw + c], tile[kb * cw + r * cw + c]};
                a = dd_sub(a, dd_mul(l, u));
                tile[r * cw + c] = a.hi;
                tile[kb * cw + r * cw + c] = a.lo;
            }
        }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < kb * cw; e += blockDim.x) {
        const int64_t rr = e / cw, c = e % cw;
        if (c < ncols) stA(A, n, p + rr, col0 + c, dd{tile[rr * cw + c], tile[kb * cw + rr * cw + c]});
    }
}

// y := P b (ipiv swaps applied in order), in shared memory when it fits.
__global__ void __launch_bounds__(1024) lu_perm_kernel(const double *b, double *y, const int64_t *ipiv,
                                                       int64_t n, int use_smem) {
    extern __shared__ double sy[];
    double *buf = use_smem ? sy : y;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) { buf[i] = b[i]; buf[n + i] = b[n + i]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int64_t k = 0; k < n; k++) {
            const int64_t r = ipiv[k];
            if (r != k) {
                double t0 = buf[k], t1 = buf[n + k];
                buf[k] = buf[r]; buf[n + k] = buf[n + r];
                buf[r] = t0; buf[n + r] = t1;
            }
        }
    }
    __syncthreads();
    if (use_smem)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) { y[i] = sy[i]; y[n + i] = sy[n + i]; }
}

// Forward (unit L, j ascending) diagonal block [J, J+nb): one thread per row of the block.
__global__ void __launch_bounds__(1024) trsv_fwd_diag(const double *A, int64_t n, double *y, int64_t J, int nb) {
    __shared__ double yh[1024], yl[1024];
    const int s = threadIdx.x;
    if (s < nb) { yh[s] = y[J + s]; yl[s] = y[n + J + s]; }
    dd lnext{0.0, 0.0};
    if (s > 0 && s < nb) lnext = ldA(A, n, J + s, J);
    for (int t = 0; t < nb; t++) {
        __syncthreads();
        const dd l = lnext;
        if (t + 1 < s && s < nb) lnext = ldA(A, n, J + s, J + t + 1);   // prefetch
        if (s > t && s < nb) {
            dd v{yh[s], yl[s]};
            v = dd_sub(v, dd_mul(l, dd{yh[t], yl[t]}));
            yh[s] = v.hi; yl[s] = v.lo;
        }
    }
    __syncthreads();
    if (s < nb) { y[J + s] = yh[s]; y[n + J + s] = yl[s]; }
}

// rows i >= J+nb: y_i := y_i - l_ij y_j for j in [J, J+nb) ascending
__global__ void trsv_fwd_update(const double *A, int64_t n, double *y, int64_t J, int nb) {
    __shared__ double yh[1024], yl[1024];
    for (int t = threadIdx.x; t < nb; t += blockDim.x) { yh[t] = y[J + t]; yl[t] = y[n + J + t]; }
    __syncthreads();
    const int64_t i = J + nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dd v{y[i], y[n + i]};
    for (int t = 0; t < nb; t++) v = dd_sub(v, dd_mul(ldA(A, n, i, J + t), dd{yh[t], yl[t]}));
    y[i] = v.hi; y[n + i] = v.lo;
}

// Backward diagonal block: for t descending, x_t = y_t / u_tt, then rows s < t update.
__global__ void __launch_bounds__(1024) trsv_bwd_diag(const double *A, int64_t n, double *y, double *x,
                                                      int64_t J, int nb) {
    __shared__ double yh[1024], yl[1024];
    const int s = threadIdx.x;
    if (s < nb) { yh[s] = y[J + s]; yl[s] = y[n + J + s]; }
    // thread s < nb holds u_{s,t} for the current t (prefetched one step ahead; u_ss is the
    // divisor when t == s)
    dd unext{0.0, 0.0};
    if (s < nb) unext = ldA(A, n, J + s, J + nb - 1);
    for (int t = nb - 1; t >= 0; t--) {
        __syncthreads();
        const dd u = unext;
        if (s < nb && t - 1 >= s) unext = ldA(A, n, J + s, J + t - 1);
        if (s == t) {
            const dd xv = dd_div(dd{yh[t], yl[t]}, u);
            yh[t] = xv.hi; yl[t] = xv.lo;   // slot t now holds x_t
        }
        __syncthreads();
        if (s < t) {
            dd v{yh[s], yl[s]};
            v = dd_sub(v, dd_mul(u, dd{yh[t], yl[t]}));
            yh[s] = v.hi; yl[s] = v.lo;
        }
    }
    __syncthreads();
    if (s < nb) { x[J + s] = yh[s]; x[n + J + s] = yl[s]; }
}

// rows i < J: y_i := y_i - u_ij x_j for j in [J, J+nb) descending
__global__ void trsv_bwd_update(const double *A, int64_t n, double *y, const double *x, int64_t J, int nb) {
    __shared__ double xh[1024], xl[1024];
    for (int t = threadIdx.x; t < nb; t += blockDim.x) { xh[t] = x[J + t]; xl[t] = x[n + J + t]; }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J) return;
    dd v{y[i], y[n + i]};
    for (int t = nb - 1; t >= 0; t--) v = dd_sub(v, dd_mul(ldA(A, n, i, J + t), dd{xh[t], xl[t]}));
    y[i] = v.hi; y[n + i] = v.lo;
}

// ---- persistent cooperative panel factorisation ------------------------------------------
// One launch per panel. CTA b owns rows [p + b*rows_per, ...) of the panel (n-p rows x kb
// columns) in shared memory. Per column: local DD argmax -> candidate (value, row, the row's
// kb words) published to a double-buffered global scratch -> ONE grid-wide barrier -> every
// CTA reduces the G candidates identically (ties -> lowest row), applies the row interchange
// to the rows it owns, forms rinv = 1/u_kk, scales its column entries and does its part of the
// rank-1 update. Rows outside the panel are interchanged afterwards by lu_laswp_kernel (the
// swaps commute with the panel's column operations), so results equal the per-step
// full-row-swap order of numerics.md s.5 bit for bit.
__device__ __forceinline__ bool cand_better(double h1, double l1, long long i1, double h2, double l2,
                                            long long i2) {
    // is candidate 1 preferred over candidate 2? (larger DD magnitude; ties -> lower row; -1 = none)
    if (i1 < 0) return false;
    if (i2 < 0) return true;
    const dd a{h1, l1}, b{h2, l2};
    if (dd_abs_gt(a, b)) return true;
    if (dd_abs_gt(b, a)) return false;
    return i1 < i2;
}

// block-wide DD argmax (ties -> lower row); result in slot 0 of (rh, rl, ri); all threads call
__device__ __forceinline__ void block_argmax(double h, double l, long long i, double *rh, double *rl,
                                             long long *ri) {
    for (int off = 16; off > 0; off >>= 1) {
        const double oh = __shfl_down_sync(0xffffffffu, h, off);
        const double ol = __shfl_down_sync(0xffffffffu, l, off);
        const long long oi = __shfl_down_sync(0xffffffffu, i, off);
        if (cand_better(oh, ol, oi, h, l, i)) { h = oh; l = ol; i = oi; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();   // slots may still be read from the previous use
    if (lane == 0) { rh[warp] = h; rl[warp] = l; ri[warp] = i; }
    __syncthreads();
    if (warp == 0) {
        h = lane < nw ? rh[lane] : 0.0;
        l = lane < nw ? rl[lane] : 0.0;
        i = lane < nw ? ri[lane] : -1;
        for (int off = 16; off > 0; off >>= 1) {
            const double oh = __shfl_down_sync(0xffffffffu, h, off);
            const double ol = __shfl_down_sync(0xffffffffu, l, off);
            const long long oi = __shfl_down_sync(0xffffffffu, i, off);
            if (cand_better(oh, ol, oi, h, l, i)) { h = oh; l = ol; i = oi; }
        }
        if (lane == 0) { rh[0] = h; rl[0] = l; ri[0] = i; }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) lu_panel_coop_kernel(double *A, int64_t n, int64_t p, int kb,
                                                            int rows_per, int64_t *ipiv, LuAux *aux,
                                                            double *scr) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int G = gridDim.x;
    const int tid = threadIdx.x;
    double *Sh = sm;                              // [rows_per][kb]
    double *Sl = Sh + (size_t)rows_per * kb;
    double *Uh = Sl + (size_t)rows_per * kb;      // new row k (pivot row)
    double *Ul = Uh + kb;
    double *Lh = Ul + kb;                          // l_ik of owned rows
    double *Ll = Lh + rows_per;
    __shared__ double rh[256], rl[256];
    __shared__ long long ri[256];
    __shared__ double s_rinv[2];
    __shared__ long long s_r;
    __shared__ int s_w, s_skip;

    const int64_t r0 = p + (int64_t)blockIdx.x * rows_per;
    const int64_t left = n - r0;
    const int nrows = left <= 0 ? 0 : (int)(left < rows_per ? left : rows_per);
    // scratch layout per buffer parity: cand (h, l, idx) [G] x 3, cand rows [G][2][kb], krow [2][kb]
    const size_t per_buf = (size_t)G * 3 + (size_t)G * 2 * kb + 2 * (size_t)kb;

    for (int e = tid; e < nrows * kb; e += blockDim.x) {
        const int li = e / kb, j = e % kb;
        const dd v = ldA(A, n, r0 + li, p + j);
        Sh[e] = v.hi; Sl[e] = v.lo;
    }
    __syncthreads();

    for (int kk = 0; kk < kb; kk++) {
        const int64_t k = p + kk;
        double *buf = scr + (size_t)(kk & 1) * per_buf;
        double *cand_h = buf, *cand_l = buf + G;
        long long *cand_i = reinterpret_cast<long long *>(buf + 2 * G);
        double *cand_rows = buf + 3 * G;                 // [G][2][kb]
        double *krow = cand_rows + (size_t)G * 2 * kb;   // [2][kb]

        // 1. local argmax of column kk over owned rows >= k
        double bh = 0.0, bl = 0.0;
        long long bi = -1;
        for (int li = tid; li < nrows; li += blockDim.x) {
            const int64_t gi = r0 + li;
            if (gi < k) continue;
            const double h = Sh[li * kb + kk], l = Sl[li * kb + kk];
            if (cand_better(h, l, gi, bh, bl, bi)) { bh = h; bl = l; bi = gi; }
        }
        block_argmax(bh, bl, bi, rh, rl, ri);
        const long long lbi = ri[0];
        if (tid == 0) { cand_h[blockIdx.x] = rh[0]; cand_l[blockIdx.x] = rl[0]; cand_i[blockIdx.x] = lbi; }
        if (lbi >= 0) {
            const int li = (int)(lbi - r0);
            for (int j = tid; j < kb; j += blockDim.x) {
                cand_rows[((size_t)blockIdx.x * 2 + 0) * kb + j] = Sh[li * kb + j];
                cand_rows[((size_t)blockIdx.x * 2 + 1) * kb + j] = Sl[li * kb + j];
            }
        }
        const bool own_k = k >= r0 && k < r0 + nrows;
        if (own_k) {
            const int li = (int)(k - r0);
            for (int j = tid; j < kb; j += blockDim.x) { krow[j] = Sh[li * kb + j]; krow[kb + j] = Sl[li * kb + j]; }
        }
        __threadfence();
        grid.sync();

        // 2. global pivot (identical reduction in every CTA): candidates are rows, so the
        // winning CTA is recovered from the winning row index
        {
            double h = 0.0, l = 0.0;
            long long i = -1;
            for (int g = tid; g < G; g += blockDim.x) {
                const double ch = cand_h[g], cl = cand_l[g];
                const long long ci = cand_i[g];
                if (cand_better(ch, cl, ci, h, l, i)) { h = ch; l = cl; i = ci; }
            }
            block_argmax(h, l, i, rh, rl, ri);
            if (tid == 0) { s_r = ri[0]; s_w = (int)((ri[0] - p) / rows_per); }
        }
        __syncthreads();
        const int64_t r = s_r;
        const double *prow = cand_rows + (size_t)s_w * 2 * kb;
        for (int j = tid; j < kb; j += blockDim.x) { Uh[j] = prow[j]; Ul[j] = prow[kb + j]; }
        __syncthreads();
        if (r != k) {
            if (own_k) {
                const int li = (int)(k - r0);
                for (int j = tid; j < kb; j += blockDim.x) { Sh[li * kb + j] = Uh[j]; Sl[li * kb + j] = Ul[j]; }
            }
            if (r >= r0 && r < r0 + nrows) {
                const int li = (int)(r - r0);
                for (int j = tid; j < kb; j += blockDim.x) { Sh[li * kb + j] = krow[j]; Sl[li * kb + j] = krow[kb + j]; }
            }
        }
        if (tid == 0) {
            const dd piv{Uh[kk], Ul[kk]};
            if (blockIdx.x == 0) ipiv[k] = r;
            if (piv.hi == 0.0) {
                s_skip = 1;
                if (blockIdx.x == 0 && aux->info == 0) aux->info = (int)(k + 1);
            } else {
                const dd rv = dd_div(dd{1.0, 0.0}, piv);
                s_rinv[0] = rv.hi; s_rinv[1] = rv.lo;
                s_skip = 0;
            }
        }
        __syncthreads();
        if (s_skip) continue;
        // 3. l_ik = a_ik * rinv for owned rows i > k
        const dd rinv{s_rinv[0], s_rinv[1]};
        for (int li = tid; li < nrows; li += blockDim.x) {
            if (r0 + li <= k) continue;
            const dd lv = dd_mul(dd{Sh[li * kb + kk], Sl[li * kb + kk]}, rinv);
            Sh[li * kb + kk] = lv.hi; Sl[li * kb + kk] = lv.lo;
            Lh[li] = lv.hi; Ll[li] = lv.lo;
        }
        __syncthreads();
        // 4. rank-1 update a_ij -= l_ik u_kj, j in (kk, kb)
        const int ncol = kb - kk - 1;
        if (ncol > 0) {
            for (int e = tid; e < nrows * ncol; e += blockDim.x) {
                const int li = e / ncol, j = kk + 1 + e % ncol;
                if (r0 + li <= k) continue;
                const dd a{Sh[li * kb + j], Sl[li * kb + j]};
                const dd v = dd_sub(a, dd_mul(dd{Lh[li], Ll[li]}, dd{Uh[j], Ul[j]}));
                Sh[li * kb + j] = v.hi; Sl[li * kb + j] = v.lo;
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < nrows * kb; e += blockDim.x) {
        const int li = e / kb, j = e % kb;
        stA(A, n, r0 + li, p + j, dd{Sh[e], Sl[e]});
    }
}

// Apply the panel's interchanges (in order) to the columns outside the panel.
__global__ void lu_laswp_kernel(double *A, int64_t n, int64_t p, int64_t kb, const int64_t *ipiv) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ncols = n - kb;
    if (t >= 2 * ncols) return;
    const int plane = (int)(t / ncols);
    int64_t j = t % ncols;
    if (j >= p) j += kb;
    double *Ap = A + (int64_t)plane * n * n;
    for (int64_t kk = 0; kk < kb; kk++) {
        const int64_t k = p + kk, r = ipiv[k];
        if (r != k) {
            const double a = Ap[k * n + j];
            Ap[k * n + j] = Ap[r * n + j];
            Ap[r * n + j] = a;
        }
    }
}

static int g_coop_sms = -1;

// DDQD_LU_PANEL=steps forces the per-column two-kernel path (kept as the reference schedule)
static bool use_coop_panel() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_LU_PANEL");
        v = (e && std::string(e) == "steps") ? 0 : 1;
    }
    return v == 1;
}

// returns 1 if the cooperative path was launched, 0 if the caller should use the per-column path
static int try_panel_coop(double *A, int64_t n, int64_t p, int64_t kb, int64_t *ipiv, LuAux *aux,
                          double *scr, size_t scr_bytes, cudaStream_t s, int *rc) {
    *rc = DDQD_OK;
    const int64_t R = n - p;
    if (g_coop_sms < 0) {
        int dev = 0, coop = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_coop_sms = coop ? sms : 0;
    }
    if (g_coop_sms <= 0 || kb > 4096) return 0;
    int G = (int)std::min<int64_t>(g_coop_sms, R);
    const int rows_per = (int)((R + G - 1) / G);
    G = (int)((R + rows_per - 1) / rows_per);
    const size_t smem = sizeof(double) * (2 * (size_t)rows_per * kb + 2 * (size_t)kb + 2 * (size_t)rows_per);
    if (smem > 200 * 1024) return 0;
    const size_t per_buf = (size_t)G * 3 + (size_t)G * 2 * kb + 2 * (size_t)kb;
    if (2 * per_buf * sizeof(double) > scr_bytes) return 0;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        if (cudaFuncSetAttribute(lu_panel_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        attr = smem;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lu_panel_coop_kernel, 256, smem);
    if (occ < 1 || G > occ * g_coop_sms) return 0;
    int kbi = (int)kb;
    void *args[] = {&A, &n, &p, &kbi, (void *)&rows_per, &ipiv, &aux, &scr};
    cudaError_t e = cudaLaunchCooperativeKernel((void *)lu_panel_coop_kernel, dim3(G), dim3(256), args, smem, s);
    count_launch();
    if (e != cudaSuccess) {
        set_error(std::string("cooperative panel launch: ") + cudaGetErrorString(e));
        *rc = DDQD_ECUDA;
        return 1;
    }
    if (n - kb > 0) {
        const int64_t threads = 2 * (n - kb);
        lu_laswp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(A, n, p, kb, ipiv);
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("laswp launch: ") + cudaGetErrorString(e));
            *rc = DDQD_ECUDA;
        }
    }
    return 1;
}

int lu_solve_impl(int64_t n, double *A, const double *b, double *x, int64_t *ipiv, int64_t K,
                  int algo, int64_t T, cudaStream_t s, int *info_out) {
    *info_out = 0;
    if (n == 0) return DDQD_OK;
    int st = DDQD_OK;
    // aux: LuAux | y [2n] | cooperative-panel scratch (2 buffers of G*(3 + 2K) + 2K doubles)
    const size_t ybytes = (sizeof(double) * 2 * (size_t)n + 255) & ~size_t(255);
    const size_t scr_bytes = sizeof(double) * 2 * ((size_t)160 * (3 + 2 * (size_t)K) + 2 * (size_t)K);
    const size_t aux_bytes = 256 + ybytes + scr_bytes;
    char *aux_mem = static_cast<char *>(aux_get(aux_bytes, &st));
    if (st) return st;
    LuAux *aux = reinterpret_cast<LuAux *>(aux_mem);
    double *y = reinterpret_cast<double *>(aux_mem + 256);
    double *scr = reinterpret_cast<double *>(aux_mem + 256 + ybytes);
    DDQD_CUDA_CHECK(cudaMemsetAsync(aux, 0, sizeof(LuAux), s));

    for (int64_t p = 0; p < n; p += K) {
        const int64_t kb = std::min(K, n - p);
        prof_begin(3, s);
        int crc = DDQD_OK;
        const bool coop = use_coop_panel() && try_panel_coop(A, n, p, kb, ipiv, aux, scr, scr_bytes, s, &crc);
        if (crc) return crc;
        for (int64_t k = p; !coop && k < p + kb; k++) {
            lu_pivot_kernel<<<1, 1024, 0, s>>>(A, n, k, ipiv, aux);
            DDQD_LAUNCH_CHECK();
            const int64_t nc = p + kb - (k + 1), nr = n - (k + 1);
            if (nc > 0 && nr > 0) {
                dim3 blk(32, 8);
                dim3 grd((unsigned)((nc + 31) / 32), (unsigned)((nr + 7) / 8));
                lu_rank1_kernel<<<grd, blk, 0, s>>>(A, n, k, p + kb, aux);
                DDQD_LAUNCH_CHECK();
            }
        }
        prof_end(3, (double)kb * (double)(n - p) * (double)kb / 2.0, s);   // panel madds (approx.)
        const int64_t n2 = n - p - kb;
        if (n2 <= 0) continue;
        // one CTA per SM when possible: cw = ceil(n2 / 148), capped by shared memory
        const int64_t cw_smem = std::max<int64_t>(1, (int64_t)(200 * 1024) / (16 * kb));
        int cw = (int)std::max<int64_t>(1, std::min<int64_t>(cw_smem, (n2 + 147) / 148));
        const size_t smem = sizeof(double) * 2 * (size_t)kb * cw;
        if (smem > 48 * 1024)
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
        prof_begin(4, s);
        if (kb > 1024) { set_error("panel > 1024 not supported by the TRSM kernel"); return DDQD_ENOTSUP; }
        const int tthreads = (int)(((kb + 31) / 32) * 32);
        lu_trsm_kernel<<<(unsigned)((n2 + cw - 1) / cw), tthreads, smem, s>>>(A, n, p, kb, p + kb, cw);
        DDQD_LAUNCH_CHECK();
        prof_end(4, (double)kb * (double)kb / 2.0 * (double)n2, s);
        MatDesc L21{A + (p + kb) * n + p, n2, kb, n, n * n, 0};
        MatDesc U12{A + p * n + (p + kb), kb, n2, n, n * n, 0};
        MatDesc A22{A + (p + kb) * n + (p + kb), n2, n2, n, n * n, 0};
        const int rc = run_gemm(2, algo, T, n2, kb, n2, 1, L21, U12, A22, 1, s);
        if (rc) return rc;
    }

    // solve: y = P b; L y' = y (j ascending); U x = y' (j descending)
    const int use_smem = (2 * n * (int64_t)sizeof(double) <= 200 * 1024) ? 1 : 0;
    const size_t psmem = use_smem ? 2 * n * sizeof(double) : 0;
    if (psmem > 48 * 1024)
        DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)psmem));
    prof_begin(5, s);
    lu_perm_kernel<<<1, 1024, psmem, s>>>(b, y, ipiv, n, use_smem);
    DDQD_LAUNCH_CHECK();
    const int NB = 256;
    for (int64_t J = 0; J < n; J += NB) {
        const int nb = (int)std::min<int64_t>(NB, n - J);
        trsv_fwd_diag<<<1, 1024, 0, s>>>(A, n, y, J, nb);
        DDQD_LAUNCH_CHECK();
        const int64_t rows = n - J - nb;
        if (rows > 0) {
            trsv_fwd_update<<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(A, n, y, J, nb);
            DDQD_LAUNCH_CHECK();
        }
    }
    const int64_t last = ((n - 1) / NB) * NB;
    for (int64_t J = last; J >= 0; J -= NB) {
        const int nb = (int)std::min<int64_t>(NB, n - J);
        trsv_bwd_diag<<<1, 1024, 0, s>>>(A, n, y, x, J, nb);
        DDQD_LAUNCH_CHECK();
        if (J > 0) {
            trsv_bwd_update<<<(unsigned)((J + 127) / 128), 128, 0, s>>>(A, n, y, x, J, nb);
            DDQD_LAUNCH_CHECK();
        }
    }
    prof_end(5, (double)n * (double)n, s);
    int info_h = 0;
    DDQD_CUDA_CHECK(cudaMemcpyAsync(&info_h, &aux->info, sizeof(int), cudaMemcpyDeviceToHost, s));
    DDQD_CUDA_CHECK(cudaStreamSynchronize(s));
    *info_out = info_h;
    return DDQD_OK;
}

}  // namespace ddqd
