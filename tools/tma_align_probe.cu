// tma_align_probe.cu -- does a tiled TMA load accept a box whose start is NOT 16-byte aligned
// in the innermost dimension (float64, start column odd)? Prints the loaded values or reports
// a timeout (bounded mbarrier wait). Used to decide how the row-pair A view may be addressed.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int c0, double *out, int *ok) {
    __shared__ __align__(1024) double buf[8 * 4];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(8 * 4 * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sa(buf)), "l"((uint64_t)&tm), "r"(c0), "r"(0), "r"(sa(&bar)) : "memory");
        uint32_t done = 0;
        for (long long i = 0; i < (1ll << 26) && !done; i++)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(sa(&bar)) : "memory");
        *ok = done;
        for (int i = 0; i < 32; i++) out[i] = buf[i];
    }
}

int main() {
    const int cols = 602, rows = 8;
    double *h = new double[cols * rows], *d, *o;
    int *ok;
    for (int i = 0; i < cols * rows; i++) h[i] = i;
    cudaMalloc(&d, sizeof(double) * cols * rows);
    cudaMalloc(&o, sizeof(double) * 32);
    cudaMalloc(&ok, sizeof(int));
    cudaMemcpy(d, h, sizeof(double) * cols * rows, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
    cuuint32_t box[2] = {8, 4}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int c0 : {0, 8, 1, 301, 297}) {
        probe<<<1, 32>>>(tm, c0, o, ok);
        cudaError_t e = cudaDeviceSynchronize();
        int okh = 0;
        double oh[32];
        cudaMemcpy(&okh, ok, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMemcpy(oh, o, sizeof(oh), cudaMemcpyDeviceToHost);
        printf("c0=%d err=%s done=%d first=%g %g %g row1=%g expect=%d\n", c0, cudaGetErrorString(e), okh, oh[0], oh[1],
               oh[7], oh[8], c0);
        if (e != cudaSuccess) break;
    }
    return 0;
}
