// Register-only throughput of the canonical DD multiply-add (20 FP64 instructions) on one
// B200: how close can ANY kernel with this instruction mix get to the FP64-pipe peak?
// Compares against the plain DADD stream (the roofline denominator bench.py uses).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I include \
//        -o tools/madd_ceiling tools/madd_ceiling.cu
#include <cstdio>

#include "../paper_1510_08642_b200/csrc/ddqd_arith.cuh"

using namespace ddqd;

// CH independent DD accumulators per thread; per step the operands come from shared memory
// (as in the leaf GEMM: one a per step, CH/4 b values reused), so nothing can be hoisted
template <int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_madd(double *out, int iters, double s0) {
    __shared__ double sa[2][64], sb[2][64];
    if (threadIdx.x < 64) {
        sa[0][threadIdx.x] = s0 + 0.001 * threadIdx.x;
        sa[1][threadIdx.x] = 1e-20 * threadIdx.x;
        sb[0][threadIdx.x] = 0.5 - 0.0001 * threadIdx.x;
        sb[1][threadIdx.x] = -3e-21 * threadIdx.x;
    }
    __syncthreads();
    dd acc[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) acc[j] = dd{0.0, 0.0};
    for (int i = 0; i < iters; i++) {
        const int r = (i + threadIdx.x) & 63;
        dd a[CH / 4 > 0 ? CH / 4 : 1], b[4];
#pragma unroll
        for (int q = 0; q < (CH / 4 > 0 ? CH / 4 : 1); q++) a[q] = dd{sa[0][(r + q) & 63], sa[1][(r + q) & 63]};
#pragma unroll
        for (int q = 0; q < 4; q++) b[q] = dd{sb[0][(r + 7 * q) & 63], sb[1][(r + 7 * q) & 63]};
#pragma unroll
        for (int j = 0; j < CH; j++) acc[j] = dd_madd(acc[j], a[j / 4], b[j & 3]);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CH; j++) s += acc[j].hi + acc[j].lo;
    if (s == 12345.678) out[blockIdx.x] = s;
}

// QD: CH accumulators, operands from shared memory (4 words each)
template <int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_qmadd(double *out, int iters, double s0) {
    __shared__ double sa[4][64], sb[4][64];
    if (threadIdx.x < 64) {
        for (int w = 0; w < 4; w++) {
            sa[w][threadIdx.x] = (s0 + 0.001 * threadIdx.x) * (w ? 1e-17 * w : 1.0);
            sb[w][threadIdx.x] = (0.5 - 0.0001 * threadIdx.x) * (w ? -3e-18 * w : 1.0);
        }
    }
    __syncthreads();
    qd acc[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) acc[j] = qd{{0.0, 0.0, 0.0, 0.0}};
    for (int i = 0; i < iters; i++) {
        const int r = (i + threadIdx.x) & 63;
        qd a[2], b[2];
#pragma unroll
        for (int q = 0; q < 2; q++)
#pragma unroll
            for (int w = 0; w < 4; w++) { a[q].w[w] = sa[w][(r + q) & 63]; b[q].w[w] = sb[w][(r + 7 * q) & 63]; }
#pragma unroll
        for (int j = 0; j < CH; j++) acc[j] = qd_madd(acc[j], a[j / 2 % 2], b[j % 2]);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CH; j++) s += acc[j].w[0] + acc[j].w[3];
    if (s == 12345.678) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dadd(double *out, int iters, double b) {
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = 1.0 + 1e-3 * (threadIdx.x + j);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = __dadd_rn(x[j], b);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; j++) s += x[j];
    if (s == 12345.678) out[blockIdx.x] = s;
}

template <class F>
static double time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; w++) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out; cudaMalloc(&out, 1 << 20);
    const int iters = 2048;
    const double dadd_ms = time_ms([&] { k_dadd<<<sms * 8, 256>>>(out, iters * 4, 1e-9); });
    const double dadd_rate = (double)sms * 8 * 256 * iters * 4 * 16 / (dadd_ms * 1e-3);
    printf("DADD stream: %.3f T lane-ops/s\n", dadd_rate / 1e12);
    auto run = [&](const char *name, auto kern, int ch, int ctas_per_sm) {
        const int blocks = sms * ctas_per_sm * 4;
        const double ms = time_ms([&] { kern<<<blocks, 256>>>(out, iters, 1.0); });
        const double rate = (double)blocks * 256 * iters * ch * 20 / (ms * 1e-3);
        printf("%-28s %.3f T lane-ops/s = %.3f of the DADD stream  (%s)\n", name, rate / 1e12,
               rate / dadd_rate, cudaGetErrorString(cudaGetLastError()));
    };
    run("madd CH=4  MINB=2", k_madd<4, 2>, 4, 2);
    run("madd CH=8  MINB=2", k_madd<8, 2>, 8, 2);
    run("madd CH=16 MINB=2", k_madd<16, 2>, 16, 2);
    run("madd CH=16 MINB=1", k_madd<16, 1>, 16, 1);
    run("madd CH=8  MINB=4", k_madd<8, 4>, 8, 4);
    run("madd CH=4  MINB=4", k_madd<4, 4>, 4, 4);
    run("madd CH=32 MINB=1", k_madd<32, 1>, 32, 1);
    // QD: count 200 FP64 lane-ops per madd (the common-path count ncu confirmed in the leaf)
    auto runq = [&](const char *name, auto kern, int ch, int ctas_per_sm) {
        const int blocks = sms * ctas_per_sm * 4;
        const double ms = time_ms([&] { kern<<<blocks, 256>>>(out, iters / 4, 1.0); });
        const double rate = (double)blocks * 256 * (iters / 4) * ch * 200 / (ms * 1e-3);
        printf("%-28s %.3f T lane-ops/s = %.3f of the DADD stream  (%s)\n", name, rate / 1e12,
               rate / dadd_rate, cudaGetErrorString(cudaGetLastError()));
    };
    runq("qd madd CH=4 MINB=2", k_qmadd<4, 2>, 4, 2);
    runq("qd madd CH=2 MINB=2", k_qmadd<2, 2>, 2, 2);
    runq("qd madd CH=4 MINB=1", k_qmadd<4, 1>, 4, 1);
    runq("qd madd CH=8 MINB=1", k_qmadd<8, 1>, 8, 1);
    return 0;
}
