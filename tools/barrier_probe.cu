// Grid-barrier latency probe on one B200 (cooperative launch, 1 CTA per SM).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long *out) {
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void k_ctr(int iters, unsigned *ctr, unsigned long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            unsigned target = (unsigned)(i + 1) * gridDim.x;
            while (*(volatile unsigned *)ctr < target) {}
            __threadfence();
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void k_flags(int iters, unsigned long long *flags, unsigned long long *out, int relaxed) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + blockIdx.x * 16), "l"((unsigned long long)(i + 1)) : "memory");
        }
        for (int g = threadIdx.x; g < gridDim.x; g += blockDim.x) {
            unsigned long long v;
            if (relaxed) {
                do { v = *(volatile unsigned long long *)(flags + g * 16); } while (v < (unsigned long long)(i + 1));
            } else {
                do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + g * 16) : "memory"); } while (v < (unsigned long long)(i + 1));
            }
        }
        if (relaxed) __threadfence();
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *out, *flags; unsigned *ctr;
    cudaMalloc(&out, 64); cudaMalloc(&flags, 256 * 16 * 8); cudaMalloc(&ctr, 64);
    int iters = 2000;
    for (int G : {sms, sms / 2, 32, 8}) {
        for (int variant = 0; variant < 4; variant++) {
            cudaMemset(flags, 0, 256 * 16 * 8); cudaMemset(ctr, 0, 64);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (variant == 0) { void *args[] = {&iters, &out}; cudaLaunchCooperativeKernel((void *)k_cg, G, 256, args, 0, 0); }
            if (variant == 1) { void *args[] = {&iters, &ctr, &out}; cudaLaunchCooperativeKernel((void *)k_ctr, G, 256, args, 0, 0); }
            if (variant >= 2) { int rel = variant == 3; void *args[] = {&iters, &flags, &out, &rel}; cudaLaunchCooperativeKernel((void *)k_flags, G, 256, args, 0, 0); }
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
            printf("G=%d variant=%d (%s): %.3f us/barrier, %.0f cycles/barrier  err=%s\n", G, variant,
                   variant == 0 ? "cg grid.sync" : variant == 1 ? "atomic ctr" : variant == 2 ? "flags acquire" : "flags relaxed+fence",
                   ms * 1000 / iters, (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
