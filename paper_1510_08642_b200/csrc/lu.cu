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
#include <algorithm>

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
// of CW columns held in shared memory.
__global__ void __launch_bounds__(256) lu_trsm_kernel(double *A, int64_t n, int64_t p, int64_t kb,
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
    for (int64_t i = 0; i < kb; i++) {
        __syncthreads();
        for (int64_t r = i + 1 + threadIdx.x; r < kb; r += blockDim.x) {
            const dd l = ldA(A, n, p + r, p + i);
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
        const int64_t r = e / cw, c = e % cw;
        if (c < ncols) stA(A, n, p + r, col0 + c, dd{tile[r * cw + c], tile[kb * cw + r * cw + c]});
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
    for (int t = 0; t < nb; t++) {
        __syncthreads();
        if (s > t && s < nb) {
            dd v{yh[s], yl[s]};
            v = dd_sub(v, dd_mul(ldA(A, n, J + s, J + t), dd{yh[t], yl[t]}));
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
    for (int t = nb - 1; t >= 0; t--) {
        __syncthreads();
        if (s == t) {
            const dd xv = dd_div(dd{yh[t], yl[t]}, ldA(A, n, J + t, J + t));
            yh[t] = xv.hi; yl[t] = xv.lo;   // slot t now holds x_t
        }
        __syncthreads();
        if (s < t) {
            dd v{yh[s], yl[s]};
            v = dd_sub(v, dd_mul(ldA(A, n, J + s, J + t), dd{yh[t], yl[t]}));
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

int lu_solve_impl(int64_t n, double *A, const double *b, double *x, int64_t *ipiv, int64_t K,
                  int algo, int64_t T, cudaStream_t s, int *info_out) {
    *info_out = 0;
    if (n == 0) return DDQD_OK;
    int st = DDQD_OK;
    const size_t aux_bytes = 256 + sizeof(double) * 2 * (size_t)n;
    char *aux_mem = static_cast<char *>(aux_get(aux_bytes, &st));
    if (st) return st;
    LuAux *aux = reinterpret_cast<LuAux *>(aux_mem);
    double *y = reinterpret_cast<double *>(aux_mem + 256);
    DDQD_CUDA_CHECK(cudaMemsetAsync(aux, 0, sizeof(LuAux), s));

    for (int64_t p = 0; p < n; p += K) {
        const int64_t kb = std::min(K, n - p);
        prof_begin(3, s);
        for (int64_t k = p; k < p + kb; k++) {
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
        int cw = (int)std::max<int64_t>(1, std::min<int64_t>(32, 6144 / kb));
        const size_t smem = sizeof(double) * 2 * (size_t)kb * cw;
        if (smem > 48 * 1024)
            DDQD_CUDA_CHECK(cudaFuncSetAttribute(lu_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
        prof_begin(4, s);
        lu_trsm_kernel<<<(unsigned)((n2 + cw - 1) / cw), 256, smem, s>>>(A, n, p, kb, p + kb, cw);
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
