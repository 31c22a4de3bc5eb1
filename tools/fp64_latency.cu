// Dependent-chain latency of FP64 DADD / DMUL / DFMA, SHFL and a DD sub(mul) on one B200 SM
// (one warp, clock64): the step latency that bounds the LU's sequential chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I include -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>

#include "../paper_1510_08642_b200/csrc/ddqd_arith.cuh"
using namespace ddqd;

__global__ void k_lat(double *out, long long *cyc, double a, double b, int iters) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) x = __dadd_rn(x, b);
    long long t1 = clock64();
    for (int i = 0; i < iters; i++) x = __dmul_rn(x, b);
    long long t2 = clock64();
    for (int i = 0; i < iters; i++) x = __fma_rn(x, b, a);
    long long t3 = clock64();
    for (int i = 0; i < iters; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    long long t4 = clock64();
    dd v{x, 0.0}, l{b, 1e-20}, y{a, -1e-21};
    for (int i = 0; i < iters; i++) { v = dd_sub(v, dd_mul(l, y)); y.hi = v.hi; }
    long long t5 = clock64();
    double z = a;
    for (int i = 0; i < iters; i++) z = 1.0 / (z + 1.0);                  // IEEE division (+ DADD)
    long long t6 = clock64();
    for (int i = 0; i < iters; i++) z = __drcp_rn(z + 1.0);              // correctly rounded reciprocal (+ DADD)
    long long t7 = clock64();
    dd u{a, 1e-20};
    for (int i = 0; i < iters; i++) { u = dd_div(dd{1.0, 0.0}, u); u.hi += 1.0; }   // DD reciprocal (+ DADD)
    long long t8 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
        cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
        out[0] = x + v.hi + v.lo + z + u.hi;
    }
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
    const int iters = 4096;
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, iters);
    k_lat<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, iters);
    long long h[8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *nm[] = {"DADD", "DMUL", "DFMA", "SHFL (64-bit)", "DD sub(v, mul(l, y)) with y <- v.hi",
                        "IEEE 1/(z+1) (div + DADD)", "__drcp_rn(z+1) (+ DADD)", "DD 1/u = dd_div(1, u) (+ DADD)"};
    for (int i = 0; i < 8; i++) printf("%-40s %.1f cycles per dependent step\n", nm[i], (double)h[i] / iters);
    return 0;
}
