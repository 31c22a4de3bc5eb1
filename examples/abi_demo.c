/* abi_demo.c -- the library used from plain C through include/ddqd.h (no Python, no torch):
 * C := A B in DD with Winograd (threshold 32) on the device, checked against a naive host DD
 * reference written here with the same op sequence (docs/numerics.md s.2), then a DD LU solve.
 *
 *   gcc -std=c11 -O2 -ffp-contract=off examples/abi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1510_08642_b200 -lddqd -L/usr/local/cuda/lib64 -lcudart -lm -o abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ddqd.h"

static void two_sum(double a, double b, double *s, double *e) {
    double ss = a + b, bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}
static void madd(double *ch, double *cl, double ah, double al, double bh, double bl) {
    double p = ah * bh, e = fma(ah, bh, -p), t = (ah * bl) + (al * bh), s, f, ph, pl, hs, he;
    e = e + t;
    ph = p + e; pl = e - (ph - p);                     /* dd_mul */
    two_sum(*ch, ph, &s, &f);
    t = *cl + pl; f = f + t;
    hs = s + f; he = f - (hs - s);                      /* dd_add */
    *ch = hs; *cl = he;
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("cuda: %s\n", cudaGetErrorString(e_)); return 1; } } while (0)

int main(void) {
    const int64_t m = 150, l = 97, n = 131;
    size_t sa = 2 * m * l, sb = 2 * l * n, sc = 2 * m * n;
    double *A = malloc(sa * 8), *B = malloc(sb * 8), *C = malloc(sc * 8);
    srand(7);
    for (size_t i = 0; i < sa / 2; i++) { A[i] = rand() / (double)RAND_MAX - 0.5; A[sa / 2 + i] = A[i] * 0x1p-60; }
    for (size_t i = 0; i < sb / 2; i++) { B[i] = rand() / (double)RAND_MAX - 0.5; B[sb / 2 + i] = -B[i] * 0x1p-61; }
    double *dA, *dB, *dC;
    CK(cudaMalloc((void **)&dA, sa * 8)); CK(cudaMalloc((void **)&dB, sb * 8)); CK(cudaMalloc((void **)&dC, sc * 8));
    CK(cudaMemcpy(dA, A, sa * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B, sb * 8, cudaMemcpyHostToDevice));
    /* Block: bit-identical to the naive k-ascending loop */
    int rc = dd_gemm(m, l, n, dA, dB, dC, DDQD_BLOCK, 0);
    if (rc) { printf("dd_gemm: %d %s\n", rc, ddqd_last_error()); return 1; }
    CK(cudaMemcpy(C, dC, sc * 8, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int64_t i = 0; i < m; i++)
        for (int64_t j = 0; j < n; j++) {
            double ch = 0.0, cl = 0.0;
            for (int64_t k = 0; k < l; k++)
                madd(&ch, &cl, A[i * l + k], A[m * l + i * l + k], B[k * n + j], B[l * n + k * n + j]);
            if (ch != C[i * n + j] || cl != C[m * n + i * n + j]) bad++;
        }
    printf("dd_gemm Block %ldx%ldx%ld: %ld mismatching entries\n", (long)m, (long)l, (long)n, bad);
    /* Winograd(32) through the host-pointer path (staged copies inside the call) */
    rc = dd_gemm(m, l, n, A, B, C, DDQD_WINOGRAD, 32);
    printf("dd_gemm Winograd(32) host pointers: rc=%d, C[0]=%.17g%+.3g\n", rc, C[0], C[m * n]);
    /* error path */
    rc = dd_gemm(-1, l, n, dA, dB, dC, DDQD_BLOCK, 0);
    printf("negative size -> %d (%s)\n", rc, ddqd_last_error());
    /* DD LU solve of a diagonally dominant system with x = 1 */
    const int64_t N = 64;
    double *M = calloc(2 * N * N, 8), *b = calloc(2 * N, 8), *x = calloc(2 * N, 8);
    for (int64_t i = 0; i < N; i++)
        for (int64_t j = 0; j < N; j++) M[i * N + j] = (i == j) ? N : 1.0 / (1 + i + j);
    for (int64_t i = 0; i < N; i++)
        for (int64_t j = 0; j < N; j++) b[i] += M[i * N + j];   /* exact: small dyadics not needed */
    double *dM, *db, *dx; int64_t *dp;
    CK(cudaMalloc((void **)&dM, 2 * N * N * 8)); CK(cudaMalloc((void **)&db, 2 * N * 8));
    CK(cudaMalloc((void **)&dx, 2 * N * 8)); CK(cudaMalloc((void **)&dp, N * 8));
    CK(cudaMemcpy(dM, M, 2 * N * N * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b, 2 * N * 8, cudaMemcpyHostToDevice));
    rc = dd_lu_solve(N, dM, db, dx, dp, 16, DDQD_STRASSEN, 8);
    CK(cudaMemcpy(x, dx, 2 * N * 8, cudaMemcpyDeviceToHost));
    double worst = 0;
    for (int64_t i = 0; i < N; i++) worst = fmax(worst, fabs(x[i] - 1.0));
    printf("dd_lu_solve n=%ld: info=%d, max|x-1| (hi words) = %.3g\n", (long)N, rc, worst);
    printf("kernels launched by this thread: %lld\n", (long long)ddqd_launch_count());
    ddqd_release();
    return (bad == 0 && rc == 0 && worst < 1e-12) ? 0 : 1;
}
