// Latency probe of one LU-panel column exchange on a B200 (cooperative launch, 1 CTA per SM):
// every CTA publishes a candidate (value, index) and a 512-double row, crosses a grid
// barrier, merges the G candidates and fetches the winning row into shared memory.
// Variants: barrier = cg grid.sync | split atomic counter; merge = one candidate per thread
// (smem combine) | warp 0 loads all candidates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pxp tools/panel_exchange_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int ROW = 512;

__device__ __forceinline__ void bar_ctr(unsigned *ctr, unsigned target, int fence_kind) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (fence_kind == 0) __threadfence();
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(ctr, 1u);
        while ((int)(*(volatile unsigned *)ctr - target) < 0) {}
        if (fence_kind == 0) __threadfence();
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// "bulk" stands in for the LU's rank-1 update between columns: a long straight-line FP64
// block that evicts the exchange code from the instruction cache.
template <int BULK>
__device__ __forceinline__ double bulk_work(double x) {
#pragma unroll
    for (int i = 0; i < BULK; i++) x = __dadd_rn(__dmul_rn(x, 1.0000001 + i * 1e-9), 1e-7 * (i & 7));
    return x;
}

template <int BULK>
__global__ void k_probe(int iters, int barrier, int merge, int fence_kind, double *scr, unsigned *ctr,
                        long long *out) {
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, tid = threadIdx.x;
    __shared__ double U[ROW];
    __shared__ double wv[8];
    __shared__ int wi[8];
    __shared__ int s_win;
    const size_t per_buf = (size_t)G * 2 + (size_t)G * ROW;
    long long t_pub = 0, t_bar = 0, t_merge = 0, t_row = 0;
    for (int it = 0; it < iters; it++) {
        long long t0 = clock64();
        double *buf = scr + (size_t)(it & 1) * per_buf;
        double *cv = buf;
        long long *ci = reinterpret_cast<long long *>(buf + G);
        double *rows = buf + 2 * G;
        const double myv = (double)((blockIdx.x * 7919 + it * 104729) % 1000);
        if (tid == 0) { cv[blockIdx.x] = myv; ci[blockIdx.x] = blockIdx.x; }
        for (int j = tid; j < ROW; j += blockDim.x) rows[(size_t)blockIdx.x * ROW + j] = myv + j;
        long long t1 = clock64();
        if (barrier == 0) grid.sync();
        else bar_ctr(ctr, (unsigned)G * (unsigned)(it + 1), fence_kind);
        long long t2 = clock64();
        if (merge == 0) {
            double v = -1.0;
            int i = -1;
            if (tid < G) { v = __ldcg(cv + tid); i = (int)__ldcg(ci + tid); }
            for (int off = 16; off; off >>= 1) {
                const double ov = __shfl_down_sync(~0u, v, off);
                const int oi = __shfl_down_sync(~0u, i, off);
                if (ov > v || (ov == v && oi >= 0 && oi < i)) { v = ov; i = oi; }
            }
            if ((tid & 31) == 0) { wv[tid >> 5] = v; wi[tid >> 5] = i; }
            __syncthreads();
            if (tid < 32) {
                v = tid < 8 ? wv[tid] : -1.0;
                i = tid < 8 ? wi[tid] : -1;
                for (int off = 16; off; off >>= 1) {
                    const double ov = __shfl_down_sync(~0u, v, off);
                    const int oi = __shfl_down_sync(~0u, i, off);
                    if (ov > v || (ov == v && oi >= 0 && oi < i)) { v = ov; i = oi; }
                }
                if (tid == 0) s_win = i;
            }
            __syncthreads();
        } else {
            if (tid < 32) {
                double v = -1.0;
                int i = -1;
                double vv[8];
                long long ii[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int g = tid + 32 * q;
                    ii[q] = -1;
                    if (g < G) { vv[q] = __ldcg(cv + g); ii[q] = __ldcg(ci + g); }
                }
#pragma unroll
                for (int q = 0; q < 8; q++)
                    if (ii[q] >= 0 && (vv[q] > v || (vv[q] == v && ii[q] < i))) { v = vv[q]; i = (int)ii[q]; }
                for (int off = 16; off; off >>= 1) {
                    const double ov = __shfl_down_sync(~0u, v, off);
                    const int oi = __shfl_down_sync(~0u, i, off);
                    if (ov > v || (ov == v && oi >= 0 && oi < i)) { v = ov; i = oi; }
                }
                if (tid == 0) s_win = i;
            }
            __syncthreads();
        }
        long long t3 = clock64();
        const int w = s_win;
        for (int j = tid; j < ROW; j += blockDim.x) U[j] = __ldcg(rows + (size_t)w * ROW + j);
        __syncthreads();
        long long t4 = clock64();
        t_pub += t1 - t0; t_bar += t2 - t1; t_merge += t3 - t2; t_row += t4 - t3;
        if (BULK) {
            const double x = bulk_work<BULK>(U[tid & 255]);
            if (x == 12345.0) out[6] = 1;
        }
        if (U[3] < -1.0) out[7] = 1;   // keep U live
    }
    if (blockIdx.x == 0 && tid == 0) {
        out[0] = t_pub / iters; out[1] = t_bar / iters; out[2] = t_merge / iters; out[3] = t_row / iters;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *scr; unsigned *ctr; long long *out;
    cudaMalloc(&scr, sizeof(double) * 2 * (256 * 2 + 256 * ROW));
    cudaMalloc(&ctr, 64); cudaMalloc(&out, 64);
    int iters = 2000;
    int G = sms;
    const char *bn[] = {"cg grid.sync", "atomic ctr"};
    const char *mn[] = {"thread/cand + smem", "warp0 loads all"};
    const char *fn[] = {"threadfence", "fence.acq_rel"};
    for (int bulk = 0; bulk < 2; bulk++)
    for (int barrier = 0; barrier < 2; barrier++)
        for (int merge = 0; merge < 2; merge++)
            for (int fk = 0; fk < (barrier ? 2 : 1); fk++) {
                cudaMemset(ctr, 0, 64);
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                void *args[] = {&iters, &barrier, &merge, &fk, &scr, &ctr, &out};
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel(bulk ? (void *)k_probe<4096> : (void *)k_probe<0>, G, 256, args, 0, 0);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                long long h[4]; cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
                printf("bulk=%d G=%d %-13s %-19s %-13s: %.3f us/column | cycles publish %lld barrier %lld merge %lld row %lld  (%s)\n",
                       bulk, G, bn[barrier], mn[merge], barrier ? fn[fk] : "-", ms * 1000 / iters, h[0], h[1], h[2], h[3],
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
