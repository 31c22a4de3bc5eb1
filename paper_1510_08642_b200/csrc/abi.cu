// abi.cu -- the extern "C" boundary of libddqd.so (include/ddqd.h).
// Argument checking, per-thread stream / error / workspace state, the library-owned
// workspace cache, and the host-pointer staging path used for end-to-end timing.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ddqd.h"
#include "common.cuh"

#include <nvtx3/nvToolsExt.h>

namespace ddqd {

NvtxRange::NvtxRange(const char *name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }


static thread_local std::string t_err;
static thread_local cudaStream_t t_stream = nullptr;
static thread_local int64_t t_launches = 0;
static thread_local void *t_user_ws = nullptr;
static thread_local size_t t_user_ws_bytes = 0;

void set_error(const std::string &msg) { t_err = msg; }

struct ProfRec {
    int cls;
    double work;
    cudaEvent_t e0, e1;
    const char *name;
};
struct ProfAgg {
    int cls;
    double ms, launches, work;
};
static thread_local std::vector<std::pair<std::string, ProfAgg>> t_kern;   // per-kernel totals of the last stop
static thread_local bool t_prof = false;
static thread_local std::vector<ProfRec> t_recs;
static thread_local cudaEvent_t t_open = nullptr;

void prof_begin(int cls, cudaStream_t s) {
    (void)cls;
    if (!t_prof) return;
    cudaEventCreate(&t_open);
    cudaEventRecord(t_open, s);
}
void prof_end(int cls, double work, cudaStream_t s, const char *name) {
    if (!t_prof || !t_open) return;
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, s);
    t_recs.push_back(ProfRec{cls, work, t_open, e1, name});
    t_open = nullptr;
}
cudaStream_t cur_stream() { return t_stream; }
void count_launch(int64_t n) { t_launches += n; }
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
}

// SM count of the current device (148 on a B200), cached per device: grid sizing and the leaf
// configuration choices count waves in units of it
int sm_count() {
    static int cache[64];
    const int d = current_device();
    if (!cache[d]) {
        int v = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        cache[d] = v;
    }
    return cache[d];
}

// Library-owned per-device buffers (GEMM workspace, LU auxiliary, host-path staging), shared by
// every host thread and stream of the device. Ordering between users:
//  * the first use of a library buffer inside an entry point takes the device's CALL LOCK (held
//    until the entry point has enqueued everything, LibCall below), so two threads never
//    enqueue work on the same buffers at once;
//  * if the previous user enqueued on a different stream, the new stream first waits for that
//    user's last kernels (an event recorded at the end of every call that touched the buffers);
//  * calls that touch no library buffer (Block GEMMs on device pointers, caller workspace via
//    ddqd_set_workspace) take neither and stay fully concurrent.
// Growth frees the old buffer (cudaFree synchronises the device) -- unless a CUDA graph has
// captured a call that used library buffers: from then on old buffers are retired and freed
// only by ddqd_release, so a captured graph never points at freed memory; growing a buffer
// DURING capture is refused (allocation is not capturable), see ddqd.h.
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};
struct DevSync {
    std::mutex call;
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    bool have = false;
};
static std::mutex g_mu;
static DevBuf g_ws[64], g_aux[64], g_stage[64];
static DevSync g_sync[64];
static std::vector<void *> g_retired[64];
static bool g_captured = false;
static size_t g_limit = 0;
static thread_local int t_lock_dev = -1;   // device whose call lock this thread holds (-1: none)

static int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st != cudaStreamCaptureStatusNone;
}

// first library-buffer use of this entry point: take the call lock, order after the last user
static void lib_acquire() {
    const int d = cur_dev() & 63;
    if (t_lock_dev == d) return;
    g_sync[d].call.lock();
    t_lock_dev = d;
    DevSync &y = g_sync[d];
    if (capturing(t_stream)) {
        g_captured = true;   // (a captured graph must not wait on work outside the capture)
        return;
    }
    if (y.have && y.last != t_stream) cudaStreamWaitEvent(t_stream, y.done, 0);
}

// RAII guard of every entry point that may use library buffers
struct LibCall {
    ~LibCall() {
        if (t_lock_dev < 0) return;
        DevSync &y = g_sync[t_lock_dev];
        if (!capturing(t_stream)) {
            if (!y.done) cudaEventCreateWithFlags(&y.done, cudaEventDisableTiming);
            if (y.done && cudaEventRecord(y.done, t_stream) == cudaSuccess) {
                y.last = t_stream;
                y.have = true;
            } else {
                cudaGetLastError();
            }
        }
        t_lock_dev = -1;
        y.call.unlock();
    }
};

static void *buf_get(DevBuf *arr, size_t bytes, int *status, const char *what) {
    lib_acquire();
    std::lock_guard<std::mutex> lk(g_mu);
    const int dv = cur_dev() & 63;
    DevBuf &b = arr[dv];
    if (b.bytes < bytes) {
        if (capturing(t_stream)) {
            set_error(std::string("the library's ") + what + " must grow to " + std::to_string(bytes) +
                      " bytes, which cannot happen during stream capture: make the same call once before "
                      "capturing, or install a caller workspace (ddqd_set_workspace)");
            *status = DDQD_ENOTSUP;
            return nullptr;
        }
        if (b.p) {
            if (g_captured) g_retired[dv].push_back(b.p);   // a captured graph may still use it
            else cudaFree(b.p);
        }
        b.p = nullptr;
        b.bytes = 0;
        if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
            cudaGetLastError();
            b.p = nullptr;
            set_error(std::string("cannot allocate ") + std::to_string(bytes) + " bytes of " + what);
            *status = DDQD_ENOMEM;
            return nullptr;
        }
        b.bytes = bytes;
    }
    *status = DDQD_OK;
    return b.p;
}

void *workspace_get(size_t bytes, int *status) {
    if (bytes == 0) { *status = DDQD_OK; return nullptr; }
    if (t_user_ws) {
        if (bytes > t_user_ws_bytes) {
            set_error("caller workspace too small: need " + std::to_string(bytes) + " bytes");
            *status = DDQD_ENOMEM;
            return nullptr;
        }
        *status = DDQD_OK;
        return t_user_ws;
    }
    return buf_get(g_ws, bytes, status, "GEMM workspace");
}

void *aux_get(size_t bytes, int *status) { return buf_get(g_aux, bytes, status, "LU auxiliary"); }

size_t workspace_limit() {
    if (t_user_ws) return t_user_ws_bytes;
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_limit == 0) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            cudaGetLastError();
            fr = size_t(8) << 30;
        }
        g_limit = (size_t)(0.4 * (double)(fr + g_ws[cur_dev() & 63].bytes));
    }
    return g_limit;
}

int lu_panel_impl(int W, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t p, int64_t kb, cudaStream_t s,
                  int *info_out);
int lu_trsv_impl(int W, int64_t n, const double *A, const int64_t *ipiv, const double *b, double *x,
                 cudaStream_t s);
int lu_solve_impl(int W, int pivot, int64_t n, double *A, const double *b, double *x, int64_t *ipiv,
                  int64_t K, int algo, int64_t T, cudaStream_t s, int *info_out);

static bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
    const char *pa = static_cast<const char *>(a), *pb = static_cast<const char *>(b);
    return na && nb && pa < pb + nb && pb < pa + na;
}

// 0 = device, 1 = host, -1 = error/mixed
static int where(const void *p) {
    if (!p) return 0;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return 0;
    return 1;
}

static int check_gemm_args(int64_t m, int64_t l, int64_t n, int algo, int64_t T) {
    if (m < 0 || l < 0 || n < 0) { set_error("negative dimension"); return DDQD_EINVAL; }
    if (algo & ~(0xff | DDQD_MADD_FUSED | DDQD_ADD_ACCURATE | 0x3000 | 0xff0000)) { set_error("unknown algo flag"); return DDQD_EINVAL; }
    const bool depth_forced = (algo & 0xff0000) != 0;   // DDQD_DEPTH(d): the threshold is unused
    if ((algo & DDQD_MADD_FUSED) && (algo & DDQD_ADD_ACCURATE)) {
        set_error("DDQD_MADD_FUSED and DDQD_ADD_ACCURATE are exclusive");
        return DDQD_EINVAL;
    }
    algo &= 0xff;
    if (algo < 0 || algo > 2) { set_error("algo must be DDQD_BLOCK, DDQD_STRASSEN or DDQD_WINOGRAD"); return DDQD_EINVAL; }
    if (algo != 0 && T < 1 && !depth_forced) { set_error("threshold must be >= 1"); return DDQD_EINVAL; }
    const double elems = (double)m * (double)l + (double)l * (double)n + (double)m * (double)n;
    if (elems * 4.0 > 9.0e18) { set_error("size overflow"); return DDQD_EINVAL; }
    return DDQD_OK;
}

size_t streamed_top_bytes(int W, int64_t m, int64_t l, int64_t n);   // recursion.cu
int run_gemm_streamed(int W, int algo, int64_t T, int64_t m, int64_t l, int64_t n, const MatDesc &A,
                      const MatDesc &B, const MatDesc &C, char *const *tws, const cudaEvent_t *ready, int front,
                      int tail, cudaStream_t s, int (*on_block)(int64_t r0, int64_t nr, int64_t c0, int64_t nc, void *ctx),
                      void *ctx);

// DDQD_HOST_DEEP=0 keeps M1's inputs as one copy stage (A/B measurements), =2 nests as deep as
// the recursion allows (up to 3, tests); default: one level deeper while that level's leading
// blocks of A and B are >= 64 MB. DDQD_HOST_TAIL: the same for the last product's split
// (0 off, 2 as deep as possible; default while the blocks it completes are >= 16 MB).
static int host_mode(const char *name) {
    const char *e = getenv(name);
    return (e && (e[0] == '0' || e[0] == '2')) ? e[0] - '0' : 1;
}
static int host_deep_mode() {
    static int v = -1;
    if (v < 0) v = host_mode("DDQD_HOST_DEEP");
    return v;
}
static int host_tail_mode() {
    static int v = -1;
    if (v < 0) v = host_mode("DDQD_HOST_TAIL");
    return v;
}

// DDQD_HOST_STREAM=0 disables the overlapped host path (A/B measurements)
static bool host_stream_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DDQD_HOST_STREAM");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// copy stream + events of the overlapped host path, per host thread and device
constexpr int kHostLevels = 4;   // nested streamed levels (M1 front, M4 tail) + the top level
struct CopyRes {
    cudaStream_t cs = nullptr;
    cudaEvent_t start = nullptr, first = nullptr, quad = nullptr;
    cudaEvent_t ready[kHostLevels] = {};   // ready[j]: the level-j leading blocks of A and B resident
};

// device-to-host copy of one finished block of C on the copy stream (run_gemm_streamed's hook)
struct QuadCopy {
    CopyRes *cr;
    cudaStream_t s;
    int W;
    int64_t m, n;
    const double *dC;
    double *hC;
};
static int copy_block(int64_t r0, int64_t nr, int64_t c0, int64_t nc, void *ctx) {
    const QuadCopy &c = *static_cast<QuadCopy *>(ctx);
    if (nr <= 0 || nc <= 0) return DDQD_OK;
    DDQD_CUDA_CHECK(cudaEventRecord(c.cr->quad, c.s));
    DDQD_CUDA_CHECK(cudaStreamWaitEvent(c.cr->cs, c.cr->quad, 0));
    const size_t d8 = sizeof(double);
    for (int w = 0; w < c.W; w++) {
        const int64_t off = w * c.m * c.n + r0 * c.n + c0;
        DDQD_CUDA_CHECK(cudaMemcpy2DAsync(c.hC + off, c.n * d8, c.dC + off, c.n * d8, nc * d8, nr,
                                          cudaMemcpyDeviceToHost, c.cr->cs));
    }
    return DDQD_OK;
}
static int copy_res(CopyRes **out) {
    static thread_local CopyRes res[64];
    CopyRes &r = res[current_device()];
    if (!r.cs) {
        DDQD_CUDA_CHECK(cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.start, cudaEventDisableTiming));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.first, cudaEventDisableTiming));
        DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&r.quad, cudaEventDisableTiming));
        for (auto &e : r.ready) DDQD_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    *out = &r;
    return DDQD_OK;
}

static int gemm_entry(int W, int64_t m, int64_t l, int64_t n, const double *A, const double *B,
                       double *C, int algo, int64_t T) {
    NvtxRange nv(W == 2 ? "dd_gemm" : "qd_gemm");
    LibCall guard;
    t_err.clear();
    int rc = check_gemm_args(m, l, n, algo, T);
    if (rc) return rc;
    const size_t bA = sizeof(double) * W * (size_t)m * l, bB = sizeof(double) * W * (size_t)l * n,
                 bC = sizeof(double) * W * (size_t)m * n;
    if (overlaps(A, bA, C, bC) || overlaps(B, bB, C, bC)) { set_error("C overlaps A or B"); return DDQD_EALIAS; }
    if (m == 0 || n == 0) return DDQD_OK;
    if ((l > 0 && (!A || !B)) || !C) { set_error("null pointer"); return DDQD_EINVAL; }
    const int wa = where(A), wb = where(B), wc = where(C);
    cudaStream_t s = t_stream;
    if (wa == 0 && wb == 0 && wc == 0) {
        MatDesc dA{const_cast<double *>(A), m, l, l, m * l, 0};
        MatDesc dB{const_cast<double *>(B), l, n, n, l * n, 0};
        MatDesc dC{C, m, n, n, m * n, 0};
        return run_gemm(W, algo, T, m, l, n, 1, dA, dB, dC, 0, s);
    }
    if (!(wa == 1 && wb == 1 && wc == 1)) { set_error("A, B, C must be all device or all host pointers"); return DDQD_EINVAL; }
    // host path: stage through library-owned device memory, copy back, synchronise
    const bool streamed = (algo & 0xff) == DDQD_WINOGRAD && !(algo & 0xff0000) &&
                          std::min(std::min(m, l), n) > T && host_stream_enabled();
    // the nested levels' shapes (ceil halving) and children workspaces
    int64_t dm[kHostLevels + 1], dl[kHostLevels + 1], dn[kHostLevels + 1];
    dm[0] = m; dl[0] = l; dn[0] = n;
    for (int j = 0; j < kHostLevels; j++) { dm[j + 1] = (dm[j] + 1) / 2; dl[j + 1] = (dl[j] + 1) / 2; dn[j + 1] = (dn[j] + 1) / 2; }
    auto recurses = [&](int j) { return std::min(std::min(dm[j], dl[j]), dn[j]) > T; };
    const size_t d8 = sizeof(double);
    // front: M1 streamed this many levels deeper (its own leading blocks first)
    int front = 0;
    if (streamed && host_deep_mode())
        while (front + 1 < kHostLevels && recurses(front + 1) &&
               (host_deep_mode() == 2 || (size_t)W * (dm[front + 1] * dl[front + 1] + dl[front + 1] * dn[front + 1]) * d8 >= (size_t(64) << 20)))
            front++;
    // C copied back block by block (each block while the next products run) when a quadrant is
    // >= 32 MB; measured on c2 (8 MB quadrants) the split products cost more than the
    // overlapped copy gains (10.5 vs 10.2 ms), on c3 (268 MB) it saves 14 ms per call
    const bool quads = streamed && (size_t)W * dm[1] * dn[1] * d8 >= (size_t(32) << 20);
    // tail: the last product split this many levels deep (only its last block waits)
    int tail = 0;
    if (quads && host_tail_mode())
        while (tail + 1 < kHostLevels && recurses(tail + 1) &&
               (host_tail_mode() == 2 || (size_t)W * dm[tail + 2] * dn[tail + 2] * d8 >= (size_t(16) << 20)))
            tail++;
    const size_t oB = (bA + 255) & ~size_t(255), oC = oB + ((bB + 255) & ~size_t(255)),
                 oT = oC + ((bC + 255) & ~size_t(255));
    size_t ot[kHostLevels + 1];
    ot[0] = oT;
    const int nlev = streamed ? 1 + std::max(front, tail) : 0;
    for (int j = 0; j < kHostLevels; j++) ot[j + 1] = ot[j] + (j < nlev ? streamed_top_bytes(W, dm[j], dl[j], dn[j]) : 0);
    int st = DDQD_OK;
    char *dev = static_cast<char *>(buf_get(g_stage, ot[kHostLevels] + 256, &st, "staging buffers"));
    if (st) return st;
    double *dA = reinterpret_cast<double *>(dev);
    double *dB = reinterpret_cast<double *>(dev + oB);
    double *dC = reinterpret_cast<double *>(dev + oC);
    MatDesc mA{dA, m, l, l, m * l, 0}, mB{dB, l, n, n, l * n, 0}, mC{dC, m, n, n, m * n, 0};
    if (streamed) {
        // Winograd: the innermost leading blocks of A and B first on the copy stream; M1 (its
        // own M1 first, `front` levels deep) runs while the rest of A and B is copied
        // (run_gemm_streamed); bitwise the same result as the plain path
        CopyRes *cr;
        if ((rc = copy_res(&cr))) return rc;
        cudaStream_t cs = cr->cs;
        DDQD_CUDA_CHECK(cudaEventRecord(cr->start, s));
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(cs, cr->start, 0));
        // a rows x cols block at (r0, c0) of every plane of X (ld = cols of X) to the device copy
        auto blk = [&](double *dX, const double *hX, int64_t xr, int64_t xc, int64_t r0, int64_t c0, int64_t rows,
                       int64_t cols) -> int {
            if (rows <= 0 || cols <= 0) return DDQD_OK;
            for (int w = 0; w < W; w++) {
                const int64_t off = w * xr * xc + r0 * xc + c0;
                DDQD_CUDA_CHECK(cudaMemcpy2DAsync(dX + off, xc * d8, hX + off, xc * d8, cols * d8, rows,
                                                  cudaMemcpyHostToDevice, cs));
            }
            return DDQD_OK;
        };
        // stage 1: the level-(front + 1) leading blocks; then, level by level outwards, the rest
        // of the level-j leading blocks (ready[j]); ready[0]: all of A and B
        const int f1 = front + 1;
        if ((rc = blk(dA, A, m, l, 0, 0, dm[f1], dl[f1])) || (rc = blk(dB, B, l, n, 0, 0, dl[f1], dn[f1]))) return rc;
        DDQD_CUDA_CHECK(cudaEventRecord(cr->first, cs));
        for (int j = front; j >= 0; j--) {
            // level j's leading blocks (all of A and B at j = 0) minus level j + 1's
            const int64_t am = j ? dm[j] : m, al = j ? dl[j] : l, bn = j ? dn[j] : n;
            if ((rc = blk(dA, A, m, l, 0, dl[j + 1], dm[j + 1], al - dl[j + 1])) ||
                (rc = blk(dA, A, m, l, dm[j + 1], 0, am - dm[j + 1], al)) ||
                (rc = blk(dB, B, l, n, 0, dn[j + 1], dl[j + 1], bn - dn[j + 1])) ||
                (rc = blk(dB, B, l, n, dl[j + 1], 0, al - dl[j + 1], bn)))
                return rc;
            DDQD_CUDA_CHECK(cudaEventRecord(cr->ready[j], cs));
        }
        DDQD_CUDA_CHECK(cudaStreamWaitEvent(s, cr->first, 0));
        QuadCopy qc{cr, s, W, m, n, dC, C};
        char *tws[kHostLevels];
        for (int j = 0; j < kHostLevels; j++) tws[j] = dev + ot[j];
        rc = run_gemm_streamed(W, algo, T, m, l, n, mA, mB, mC, tws, cr->ready, front, tail, s,
                               quads ? copy_block : nullptr, &qc);
        // the copy stream must not outlive the call into the caller's buffers
        cudaError_t e = cudaStreamSynchronize(cs);
        if (rc) return rc;
        if (e != cudaSuccess) { set_error(std::string("copy stream: ") + cudaGetErrorString(e)); return DDQD_ECUDA; }
        if (quads) {
            DDQD_CUDA_CHECK(cudaStreamSynchronize(s));
            return DDQD_OK;
        }
    } else {
        if (bA) DDQD_CUDA_CHECK(cudaMemcpyAsync(dA, A, bA, cudaMemcpyHostToDevice, s));
        if (bB) DDQD_CUDA_CHECK(cudaMemcpyAsync(dB, B, bB, cudaMemcpyHostToDevice, s));
        rc = run_gemm(W, algo, T, m, l, n, 1, mA, mB, mC, 0, s);
        if (rc) return rc;
    }
    DDQD_CUDA_CHECK(cudaMemcpyAsync(C, dC, bC, cudaMemcpyDeviceToHost, s));
    DDQD_CUDA_CHECK(cudaStreamSynchronize(s));
    return DDQD_OK;
}

}  // namespace ddqd

using namespace ddqd;

extern "C" {

int dd_gemm(int64_t m, int64_t l, int64_t n, const double *A, const double *B, double *C, int algo,
            int64_t threshold) {
    return gemm_entry(2, m, l, n, A, B, C, algo, threshold);
}

int qd_gemm(int64_t m, int64_t l, int64_t n, const double *A, const double *B, double *C, int algo,
            int64_t threshold) {
    return gemm_entry(4, m, l, n, A, B, C, algo, threshold);
}

// Do two strided planar views share an element? Exact for two single (batch 1) views with the
// same ld and plane stride -- the LU's and the multi-GPU schedule's sub-blocks of one matrix;
// otherwise conservative (overlapping address extents count as aliasing).
struct View {
    const double *p;
    int64_t rows, cols, ld, ps, bs, batch;
};
static const double *view_end(const View &v, int W) {   // one past the last element
    return v.p + (v.batch - 1) * v.bs + (int64_t)(W - 1) * v.ps + (v.rows - 1) * v.ld + v.cols;
}
static bool views_alias(const View &a, const View &c, int W) {
    if (a.rows == 0 || a.cols == 0 || c.rows == 0 || c.cols == 0 || a.batch == 0 || c.batch == 0) return false;
    if (!(a.p < view_end(c, W) && c.p < view_end(a, W))) return false;   // disjoint extents
    if (a.batch != 1 || c.batch != 1 || a.ld != c.ld || a.ps != c.ps || a.ld <= 0 || a.ps <= 0) return true;
    const View &lo = a.p <= c.p ? a : c, &hi = a.p <= c.p ? c : a;
    const int64_t delta = hi.p - lo.p;
    const int64_t q = delta / lo.ps, r = delta % lo.ps;           // plane, then row / column offsets
    const int64_t row = r / lo.ld, col = r % lo.ld;
    if (q >= W) return false;                                     // all planes disjoint
    if (col + hi.cols > lo.ld) return true;                       // wraps a row: be conservative
    const bool rows_meet = row < lo.rows && 0 < row + hi.rows;
    const bool cols_meet = col < lo.cols && 0 < col + hi.cols;
    // plane k of the higher view sits at plane q + k of the lower one (q < W: some planes meet),
    // at the same (row, col) offset in every plane
    return rows_meet && cols_meet;
}

int ddqd_gemm_ex(const ddqd_gemm_desc *d) {
    NvtxRange nv("ddqd_gemm_ex");
    LibCall guard;
    t_err.clear();
    if (!d) { set_error("null descriptor"); return DDQD_EINVAL; }
    if (d->prec != 2 && d->prec != 4) { set_error("prec must be DDQD_DD or DDQD_QD"); return DDQD_EINVAL; }
    int rc = check_gemm_args(d->m, d->l, d->n, d->algo, d->threshold);
    if (rc) return rc;
    if (d->batch < 0 || (d->beta != 0 && d->beta != 1)) { set_error("bad batch or beta"); return DDQD_EINVAL; }
    if (d->lda < d->l || d->ldb < d->n || d->ldc < d->n) { set_error("leading dimension too small"); return DDQD_EINVAL; }
    if (d->m == 0 || d->n == 0 || d->batch == 0) return DDQD_OK;
    const int W = d->prec;
    // plane strides must clear a plane, batch strides a whole W-word matrix
    if ((d->l && d->psA < d->m * d->lda) || d->psB < d->l * d->ldb || d->psC < d->m * d->ldc ||
        (d->batch > 1 && ((d->l && d->bsA < W * d->psA) || d->bsB < W * d->psB || d->bsC < W * d->psC))) {
        set_error("plane stride < rows * ld, or batch stride < words * plane stride");
        return DDQD_EINVAL;
    }
    {
        const View va{d->A, d->m, d->l, d->lda, d->psA, d->bsA, d->batch};
        const View vb{d->B, d->l, d->n, d->ldb, d->psB, d->bsB, d->batch};
        const View vc{d->C, d->m, d->n, d->ldc, d->psC, d->bsC, d->batch};
        if (views_alias(va, vc, W) || views_alias(vb, vc, W)) { set_error("C overlaps A or B"); return DDQD_EALIAS; }
    }
    if (where(d->A) || where(d->B) || where(d->C)) { set_error("ddqd_gemm_ex takes device pointers only"); return DDQD_ENOTSUP; }
    MatDesc A{const_cast<double *>(d->A), d->m, d->l, d->lda, d->psA, d->bsA};
    MatDesc B{const_cast<double *>(d->B), d->l, d->n, d->ldb, d->psB, d->bsB};
    MatDesc C{d->C, d->m, d->n, d->ldc, d->psC, d->bsC};
    return run_gemm(d->prec, d->algo, d->threshold, d->m, d->l, d->n, d->batch, A, B, C, d->beta, t_stream);
}

int ddqd_lu_solve(int prec, int pivot, int64_t n, double *A, const double *b, double *x, int64_t *ipiv,
                  int64_t panel, int algo, int64_t threshold) {
    NvtxRange nv("ddqd_lu_solve");
    LibCall guard;
    t_err.clear();
    if (prec != 2 && prec != 4) { set_error("prec must be DDQD_DD or DDQD_QD"); return DDQD_EINVAL; }
    if (pivot != 0 && pivot != 1) { set_error("pivot must be 0 or 1"); return DDQD_EINVAL; }
    if (n < 0 || panel < 1) { set_error("n must be >= 0 and panel >= 1"); return DDQD_EINVAL; }
    if (panel > 1024 && n > panel) { set_error("panel > 1024 is not supported by the TRSM kernels (n > panel)"); return DDQD_ENOTSUP; }
    int rc = check_gemm_args(n, panel, n, algo, threshold);
    if (rc) return rc;
    if (algo & DDQD_ADD_ACCURATE) { set_error("the accurate-add variant is a GEMM variant (LU: canonical)"); return DDQD_ENOTSUP; }
    if (n == 0) return DDQD_OK;
    if (!A || !b || !x || !ipiv) { set_error("null pointer"); return DDQD_EINVAL; }
    if (where(A) || where(b) || where(x) || where(ipiv)) { set_error("LU takes device pointers only"); return DDQD_ENOTSUP; }
    int info = 0;
    rc = lu_solve_impl(prec, pivot, n, A, b, x, ipiv, panel, algo, threshold, t_stream, &info);
    if (rc) return rc;
    return info;
}

int ddqd_lu_panel(int prec, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t p, int64_t kb) {
    LibCall guard;
    t_err.clear();
    if (prec != 2 && prec != 4) { set_error("prec must be DDQD_DD or DDQD_QD"); return DDQD_EINVAL; }
    if (pivot != 0 && pivot != 1) { set_error("pivot must be 0 or 1"); return DDQD_EINVAL; }
    if (n < 0 || p < 0 || kb < 1 || p + kb > n) { set_error("need 0 <= p, 1 <= kb, p + kb <= n"); return DDQD_EINVAL; }
    if (kb > 1024 && p + kb < n) { set_error("panel > 1024 is not supported by the TRSM kernels"); return DDQD_ENOTSUP; }
    if (!A || !ipiv) { set_error("null pointer"); return DDQD_EINVAL; }
    if (where(A) || where(ipiv)) { set_error("LU takes device pointers only"); return DDQD_ENOTSUP; }
    int info = 0;
    const int rc = lu_panel_impl(prec, pivot, n, A, ipiv, p, kb, t_stream, &info);
    if (rc) return rc;
    return info;
}

int ddqd_lu_trsv(int prec, int64_t n, const double *LU, const int64_t *ipiv, const double *b, double *x) {
    LibCall guard;
    t_err.clear();
    if (prec != 2 && prec != 4) { set_error("prec must be DDQD_DD or DDQD_QD"); return DDQD_EINVAL; }
    if (n < 0) { set_error("n must be >= 0"); return DDQD_EINVAL; }
    if (n == 0) return DDQD_OK;
    if (!LU || !ipiv || !b || !x) { set_error("null pointer"); return DDQD_EINVAL; }
    if (where(LU) || where(ipiv) || where(b) || where(x)) { set_error("LU takes device pointers only"); return DDQD_ENOTSUP; }
    return lu_trsv_impl(prec, n, LU, ipiv, b, x, t_stream);
}

int dd_lu_solve(int64_t n, double *A, const double *b, double *x, int64_t *ipiv, int64_t panel, int algo,
                int64_t threshold) {
    return ddqd_lu_solve(2, 1, n, A, b, x, ipiv, panel, algo, threshold);
}

int qd_lu_solve(int64_t n, double *A, const double *b, double *x, int64_t *ipiv, int64_t panel, int algo,
                int64_t threshold) {
    return ddqd_lu_solve(4, 1, n, A, b, x, ipiv, panel, algo, threshold);
}

static MatDesc to_desc(const ddqd_mat *x) { return MatDesc{x->p, x->rows, x->cols, x->ld, x->ps, x->bs}; }

int ddqd_pre_add(int prec, int algo, int side, int64_t P, const ddqd_mat *X, const ddqd_mat *Y) {
    return ddqd_pre_add_range(prec, algo, side, P, X, Y, 0, 7 * P);
}

int ddqd_pre_add_range(int prec, int algo, int side, int64_t P, const ddqd_mat *X, const ddqd_mat *Y,
                       int64_t keep_lo, int64_t keep_hi) {
    t_err.clear();
    if (keep_lo < 0 || keep_hi < keep_lo || keep_hi > 7 * P) {
        set_error("pre_add: keep range must satisfy 0 <= lo <= hi <= 7P");
        return DDQD_EINVAL;
    }
    const int a = algo & ~DDQD_ADD_ACCURATE;   // the accurate-add variant may be OR-ed in
    if ((prec != 2 && prec != 4) || (a != 1 && a != 2) || (side != 0 && side != 1) || P < 0 || !X || !Y) {
        set_error("bad pre_add arguments");
        return DDQD_EINVAL;
    }
    if (Y->rows != (X->rows + 1) / 2 || Y->cols != (X->cols + 1) / 2) {
        set_error("pre_add: child shape must be ceil(parent/2)");
        return DDQD_EINVAL;
    }
    return launch_pre_add(prec, algo, side, P, to_desc(X), to_desc(Y), t_stream, keep_lo, keep_hi);
}

int ddqd_post_add(int prec, int algo, int64_t P, const ddqd_mat *M, const ddqd_mat *C, int beta) {
    t_err.clear();
    const int a = algo & ~DDQD_ADD_ACCURATE;
    if ((prec != 2 && prec != 4) || (a != 1 && a != 2) || P < 0 || !M || !C || (beta != 0 && beta != 1)) {
        set_error("bad post_add arguments");
        return DDQD_EINVAL;
    }
    if (M->rows != (C->rows + 1) / 2 || M->cols != (C->cols + 1) / 2) {
        set_error("post_add: product shape must be ceil(parent/2)");
        return DDQD_EINVAL;
    }
    return launch_post_add(prec, algo, P, to_desc(M), to_desc(C), beta, t_stream);
}

int ddqd_elementwise(int prec, int op, int64_t count, const double *x, const double *y, const double *w,
                     double *z) {
    t_err.clear();
    if ((prec != 2 && prec != 4) || op < 0 || op > 8 || count < 0) {
        set_error("bad elementwise arguments");
        return DDQD_EINVAL;
    }
    return launch_elementwise(prec, op, count, x, y, w, z, t_stream);
}

int ddqd_set_stream(void *s) {
    t_stream = static_cast<cudaStream_t>(s);
    return DDQD_OK;
}

size_t ddqd_workspace_bytes(int prec, int64_t m, int64_t l, int64_t n, int algo, int64_t threshold) {
    if ((prec != 2 && prec != 4) || check_gemm_args(m, l, n, algo, threshold)) return 0;
    return gemm_workspace_bytes(prec, algo, threshold, m, l, n, 1, workspace_limit(), nullptr);
}

int ddqd_set_workspace(void *dptr, size_t bytes) {
    t_user_ws = bytes ? dptr : nullptr;
    t_user_ws_bytes = dptr ? bytes : 0;
    return DDQD_OK;
}

int ddqd_set_workspace_limit(size_t bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_limit = bytes;
    return DDQD_OK;
}

int64_t ddqd_launch_count(void) { return t_launches; }

int ddqd_profile_start(void) {
    t_prof = true;
    t_recs.clear();
    return DDQD_OK;
}

int ddqd_profile_stop(double *out, int cap) {
    static const char *kClassNames[] = {"leaf", "pre_add", "post_add", "lu_panel", "lu_trsm", "lu_solve"};
    t_prof = false;
    t_kern.clear();
    for (int i = 0; i < cap; i++) out[i] = 0.0;
    for (auto &r : t_recs) {
        cudaEventSynchronize(r.e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.e0, r.e1);
        if (3 * r.cls + 2 < cap) {
            out[3 * r.cls + 0] += ms;
            out[3 * r.cls + 1] += 1.0;
            out[3 * r.cls + 2] += r.work;
        }
        const std::string nm = r.name ? r.name : (r.cls >= 0 && r.cls < 6 ? kClassNames[r.cls] : "?");
        auto it = t_kern.begin();
        for (; it != t_kern.end() && it->first != nm; ++it) {}
        if (it == t_kern.end()) { t_kern.push_back({nm, ProfAgg{r.cls, 0.0, 0.0, 0.0}}); it = t_kern.end() - 1; }
        it->second.ms += ms;
        it->second.launches += 1.0;
        it->second.work += r.work;
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    t_recs.clear();
    DDQD_CUDA_CHECK(cudaGetLastError());
    return DDQD_OK;
}

int ddqd_profile_kernels(char *out, size_t cap) {
    std::string s;
    for (auto &kv : t_kern) {
        char line[512];
        snprintf(line, sizeof(line), "%s\t%d\t%.6f\t%.0f\t%.6e\n", kv.first.c_str(), kv.second.cls, kv.second.ms,
                 kv.second.launches, kv.second.work);
        s += line;
    }
    if (!out || cap == 0) return (int)s.size() + 1;
    const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    memcpy(out, s.data(), k);
    out[k] = 0;
    return (int)s.size() + 1;
}

int ddqd_fp64_peak(int op, double *lane_ops_per_s, double *ms) {
    t_err.clear();
    return fp64_peak(op, lane_ops_per_s, ms, t_stream);
}

int ddqd_release(void) {
    const int d = cur_dev() & 63;
    std::lock_guard<std::mutex> cl(g_sync[d].call);   // no call of another thread is enqueuing
    std::lock_guard<std::mutex> lk(g_mu);
    for (DevBuf *arr : {g_ws, g_aux, g_stage}) {
        if (arr[d].p) cudaFree(arr[d].p);
        arr[d].p = nullptr;
        arr[d].bytes = 0;
    }
    for (void *p : g_retired[d]) cudaFree(p);
    g_retired[d].clear();
    g_sync[d].have = false;
    return DDQD_OK;
}

const char *ddqd_last_error(void) { return t_err.c_str(); }

int ddqd_post_add_ptrs(int prec, int algo, int64_t P, const double *const *children, int64_t hm, int64_t hn,
                       int64_t ld, int64_t ps, int64_t r0, int64_t r1, const ddqd_mat *C, int beta) {
    t_err.clear();
    const int a = algo & ~DDQD_ADD_ACCURATE;
    if ((prec != 2 && prec != 4) || (a != 1 && a != 2) || P < 0 || !children || !C || (beta != 0 && beta != 1) ||
        hm < 0 || hn < 0 || ld < hn || r0 < 0 || r1 < r0 || r1 > hm) {
        set_error("bad post_add_ptrs arguments");
        return DDQD_EINVAL;
    }
    if (hm != (C->rows + 1) / 2 || hn != (C->cols + 1) / 2) {
        set_error("post_add_ptrs: product shape must be ceil(parent/2)");
        return DDQD_EINVAL;
    }
    return launch_post_add_ptrs(prec, algo, P, children, hm, hn, ld, ps, r0, r1, to_desc(C), beta, t_stream);
}

int ddqd_band_copy(int prec, int dir, int64_t rows, int64_t cols, const int64_t *rmap, const int64_t *cmap,
                   const ddqd_mat *full, const ddqd_mat *compact) {
    t_err.clear();
    if ((prec != 2 && prec != 4) || (dir != 0 && dir != 1) || rows < 0 || cols < 0 || !full || !compact ||
        !full->p || !compact->p) {
        set_error("bad band_copy arguments");
        return DDQD_EINVAL;
    }
    if (compact->rows < rows || compact->cols < cols || compact->ld < cols || full->ld < full->cols ||
        (!rmap && rows > full->rows) || (!cmap && cols > full->cols)) {
        set_error("band_copy: shapes do not fit");
        return DDQD_EINVAL;
    }
    if (rows == 0 || cols == 0) return DDQD_OK;
    return launch_band_copy(prec, dir, rows, cols, rmap, cmap, to_desc(full), to_desc(compact), t_stream);
}

// CUDA IPC plumbing for the multi-GPU combine (buffers other processes map and read/write)
int ddqd_ipc_alloc(size_t bytes, void **ptr) {
    t_err.clear();
    if (!ptr) { set_error("null pointer"); return DDQD_EINVAL; }
    *ptr = nullptr;
    const cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 256);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return DDQD_ENOMEM;
    }
    return DDQD_OK;
}
int ddqd_ipc_free(void *ptr) {
    DDQD_CUDA_CHECK(cudaFree(ptr));
    return DDQD_OK;
}
int ddqd_ipc_handle(const void *ptr, void *handle64) {
    t_err.clear();
    if (!ptr || !handle64) { set_error("null pointer"); return DDQD_EINVAL; }
    cudaIpcMemHandle_t h;
    DDQD_CUDA_CHECK(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, sizeof(h));
    return DDQD_OK;
}
int ddqd_ipc_open(const void *handle64, void **ptr) {
    t_err.clear();
    if (!ptr || !handle64) { set_error("null pointer"); return DDQD_EINVAL; }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    DDQD_CUDA_CHECK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return DDQD_OK;
}
int ddqd_ipc_close(void *ptr) {
    DDQD_CUDA_CHECK(cudaIpcCloseMemHandle(ptr));
    return DDQD_OK;
}

int ddqd_version(void) { return 100; }

}  // extern "C"
