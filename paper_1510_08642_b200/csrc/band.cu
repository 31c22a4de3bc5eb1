// band.cu -- pack / unpack of a band sub-matrix through row and column index maps, the data
// movement of the multi-GPU band schedule (mgpu.py BandGemm). A band is a
// union of contiguous runs of rows (columns), so consecutive threads of a row touch mostly
// consecutive addresses on both sides. No arithmetic: an HBM-bound copy of W words per element.
#include <algorithm>

#include "common.cuh"

namespace ddqd {

// one CTA row-group per compact row (grid-stride over rows), threads over columns
template <int DIR>
__global__ void __launch_bounds__(256) band_copy_kernel(int W, int64_t rows, int64_t cols, const int64_t *rmap,
                                                        const int64_t *cmap, MatDesc F, MatDesc Cm) {
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
        const int64_t fi = rmap ? rmap[i] : i;
        for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
            const int64_t fj = cmap ? cmap[j] : j;
            double *f = F.p + fi * F.ld + fj;
            double *c = Cm.p + i * Cm.ld + j;
            for (int w = 0; w < W; w++) {
                if (DIR == 0) c[w * Cm.ps] = f[w * F.ps];
                else f[w * F.ps] = c[w * Cm.ps];
            }
        }
    }
}

int launch_band_copy(int W, int dir, int64_t rows, int64_t cols, const int64_t *rmap, const int64_t *cmap,
                     const MatDesc &full, const MatDesc &compact, cudaStream_t s) {
    const int threads = cols >= 256 ? 256 : cols >= 128 ? 128 : 64;
    const int64_t blocks = std::min<int64_t>(rows, (int64_t)sm_count() * 16);
    if (dir == 0)
        band_copy_kernel<0><<<(unsigned)blocks, threads, 0, s>>>(W, rows, cols, rmap, cmap, full, compact);
    else
        band_copy_kernel<1><<<(unsigned)blocks, threads, 0, s>>>(W, rows, cols, rmap, cmap, full, compact);
    DDQD_LAUNCH_CHECK();
    return DDQD_OK;
}

}  // namespace ddqd
