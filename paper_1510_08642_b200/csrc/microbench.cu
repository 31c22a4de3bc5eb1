// microbench.cu -- FP64-pipe throughput probe (the roofline denominator for the DD/QD
// leaf GEMM: "P64 must be measured"). MEASURED_PEAKS.json carries no FP64
// figure, so bench.py measures the pipe live, right before its timed region, with this
// kernel: 16 independent dependent-chains of DFMA (or DADD) per thread, 8 CTAs x 256 threads
// per SM, timed with CUDA events on the caller's stream.
#include "common.cuh"

namespace ddqd {

template <int OP>
__global__ void __launch_bounds__(256) fp64_peak_kernel(double *out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            if (OP == 0) x[j] = __fma_rn(x[j], a, b);
            else x[j] = __dadd_rn(x[j], b);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; j++) s += x[j];
    if (s == 12345.678) out[blockIdx.x] = s;   // keep the work alive
}

int fp64_peak(int op, double *lane_ops_per_s, double *ms_out, cudaStream_t s) {
    int dev = 0, sms = 0;
    DDQD_CUDA_CHECK(cudaGetDevice(&dev));
    DDQD_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double *out = nullptr;
    DDQD_CUDA_CHECK(cudaMalloc(&out, sizeof(double) * sms * 8));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&]() {
        if (op == 0) fp64_peak_kernel<0><<<blocks, threads, 0, s>>>(out, iters, 0.9999999, 1e-9);
        else fp64_peak_kernel<1><<<blocks, threads, 0, s>>>(out, iters, 0.9999999, 1e-9);
    };
    for (int w = 0; w < 3; w++) launch();
    cudaEventRecord(e0, s);
    const int reps = 10;
    for (int r = 0; r < reps; r++) launch();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    DDQD_CUDA_CHECK(cudaGetLastError());
    const double ops = (double)blocks * threads * iters * 16.0 * reps;
    *lane_ops_per_s = ops / (ms * 1e-3);
    if (ms_out) *ms_out = ms / reps;
    return DDQD_OK;
}

}  // namespace ddqd
