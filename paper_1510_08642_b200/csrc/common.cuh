// common.cuh -- shared host/device plumbing of libddqd (descriptors, status, launch count).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/ddqd.h"

namespace ddqd {

// A batch of planar row-major W-word matrices: element (b,i,j) word w at
// p[b*bs + w*ps + i*ld + j]. rows/cols are the LOGICAL extent; reads outside it are
// exact zeros (virtual padding of numerics.md s.4), writes outside it are dropped.
struct MatDesc {
    double *p;
    int64_t rows, cols, ld, ps, bs;
};


// thread-local error message + stream + launch counter (abi.cu)
void set_error(const std::string &msg);
cudaStream_t cur_stream();
void count_launch(int64_t n = 1);
int current_device();   // cudaGetDevice, masked to [0, 64) for per-device caches
int sm_count();         // multiprocessors of the current device (cached)

// NVTX ranges (header-only NVTX3; free when no profiler is attached): the recursion levels,
// the LU phases and the ABI entry points show up by name in Nsight Systems / Compute.
struct NvtxRange {
    explicit NvtxRange(const char *name);
    ~NvtxRange();
};

// Live per-class kernel timing for bench.py (CUDA events on the launching stream), active
// only between ddqd_profile_start/stop. Classes: 0 leaf GEMM (work = madds), 1 pre-add
// (work = algorithmic bytes), 2 post-add (bytes), 3 LU kernels.
void prof_begin(int cls, cudaStream_t s);
// name: a string literal (or other static storage) naming the kernel, for the per-kernel
// breakdown of ddqd_profile_kernels; null = the class name
void prof_end(int cls, double work, cudaStream_t s, const char *name = nullptr);
int fp64_peak(int op, double *lane_ops_per_s, double *ms, cudaStream_t s);

#define DDQD_CUDA_CHECK(expr)                                                            \
    do {                                                                                 \
        cudaError_t e__ = (expr);                                                        \
        if (e__ != cudaSuccess) {                                                        \
            ::ddqd::set_error(std::string(#expr) + ": " + cudaGetErrorString(e__));      \
            return DDQD_ECUDA;                                                        \
        }                                                                                \
    } while (0)

#define DDQD_LAUNCH_CHECK()                                                              \
    do {                                                                                 \
        ::ddqd::count_launch();                                                          \
        cudaError_t e__ = cudaGetLastError();                                            \
        if (e__ != cudaSuccess) {                                                        \
            ::ddqd::set_error(std::string("kernel launch: ") + cudaGetErrorString(e__)); \
            return DDQD_ECUDA;                                                        \
        }                                                                                \
    } while (0)

// Leaf GEMM (leaf_gemm.cu): C[b] (=|-=) A[b] B[b] for b < batch; beta 0: store, 1: C := C - AB.
int launch_leaf_gemm(int W, int64_t m, int64_t l, int64_t n, int64_t batch, const MatDesc &A,
                     const MatDesc &B, const MatDesc &C, int beta, int mv, cudaStream_t s);

// Strassen/Winograd pre/post additions (addsub.cu).
// keep_lo/keep_hi: only children with index (7b + c) in [keep_lo, keep_hi) are stored (-1: all)
int launch_pre_add(int W, int algo, int side, int64_t P, const MatDesc &X, const MatDesc &Y,
                   cudaStream_t s, int64_t keep_lo = 0, int64_t keep_hi = -1);
int launch_post_add(int W, int algo, int64_t P, const MatDesc &M, const MatDesc &C, int beta,
                    cudaStream_t s);
// Two levels at once (j -> j+2; h1r x h1c / h1m x h1n = the skipped level-(j+1) extent).
int launch_pre_add2(int W, int algo, int side, int64_t P, const MatDesc &X, int64_t h1r,
                    int64_t h1c, const MatDesc &Y, cudaStream_t s);
int launch_post_add2(int W, int algo, int64_t P, const MatDesc &M, int64_t h1m, int64_t h1n,
                     const MatDesc &C, int beta, cudaStream_t s);
// One C quadrant q (0 C11, 1 C12, 2 C21, 3 C22) of a single parent's post-addition, over the
// product-grid positions [r0, r0 + nr) x [c0, c0 + nc) (nr < 0: all of them).
int launch_post_quad(int W, int algo, int q, const MatDesc &M, const MatDesc &C, cudaStream_t s, int64_t r0 = 0,
                     int64_t nr = -1, int64_t c0 = 0, int64_t nc = 0);
// Post-addition with the 7P children addressed through a device pointer array (peer memory).
int launch_post_add_ptrs(int W, int algo, int64_t P, const double *const *ch, int64_t hm, int64_t hn,
                         int64_t ld, int64_t ps, int64_t r0, int64_t r1, const MatDesc &C, int beta,
                         cudaStream_t s);
// The last recursion level fused with its (tiny) leaves (addsub.cu): P parents -> parents C.
size_t fused_last_smem(int W, int64_t hm, int64_t hl, int64_t hn);   // 0: leaves too large
int launch_fused_last(int W, int algo, int mv, int64_t P, const MatDesc &X, const MatDesc &Y, const MatDesc &C,
                      int beta, int64_t hm, int64_t hl, int64_t hn, cudaStream_t s);
// Band pack (dir 0) / unpack (dir 1) through row / column index maps (band.cu).
int launch_band_copy(int W, int dir, int64_t rows, int64_t cols, const int64_t *rmap, const int64_t *cmap,
                     const MatDesc &full, const MatDesc &compact, cudaStream_t s);
int launch_elementwise(int W, int op, int64_t count, const double *x, const double *y,
                       const double *w, double *z, cudaStream_t s);

// Recursion planner + executor (recursion.cu).
size_t gemm_workspace_bytes(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n,
                            int64_t batch, size_t limit, int *dfs_levels);
// algo may carry DDQD_MADD_FUSED (bit 8): the leaf then uses the fused DD madd
int run_gemm(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n, int64_t batch,
             const MatDesc &A, const MatDesc &B, const MatDesc &C, int beta, cudaStream_t s);

}  // namespace ddqd
