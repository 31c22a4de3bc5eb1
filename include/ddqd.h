/*
 * ddqd.h -- C ABI of the B200-native DD/QD GEMM + LU library (libddqd.so).
 *
 * Method: arXiv 1510.08642 (Kouya 2015). Citation key: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, BJ:n = BASELINE.json line n. Numerics: docs/numerics.md.
 *
 * Data layout (all matrices): PLANAR row-major float64. A DD r x c matrix is
 * double[2][r][c] (plane 0 = hi words, plane 1 = lo words); a QD matrix is
 * double[4][r][c] (words of decreasing magnitude). Plane stride = r*c doubles for
 * the simple entry points; the *_ex entry points take explicit strides.
 *
 * Pointers: DEVICE pointers on the current CUDA device (cudaMalloc / torch CUDA
 * tensors). The simple GEMM entry points also accept HOST pointers for A, B and C
 * together (detected with cudaPointerGetAttributes): the library then stages them
 * through its own device buffers, copies the result back and synchronises the stream
 * before returning (the end-to-end path bench.py times as "e2e"). For Winograd the
 * copies overlap the products (A11, B11 first; M1 = A11 B11 runs while the rest
 * arrives; large C is copied back quadrant by quadrant from a library copy stream);
 * the result is bitwise that of the device-pointer call. Pinned host memory is needed
 * for the overlap; pageable memory works, with the copies serialised.
 *
 * Ownership: the caller owns every buffer passed in; the library never frees caller
 * memory. The library owns a per-device workspace, LU auxiliary and host-path staging
 * buffers (grown on demand, freed by ddqd_release) unless the calling thread installed
 * a workspace with ddqd_set_workspace.
 *
 * Synchronisation: device-pointer GEMM calls are asynchronous on the calling
 * thread's stream (ddqd_set_stream; default = legacy default stream), like cuBLAS;
 * kernel faults surface at the next synchronisation. dd_lu_solve synchronises once
 * at the end to read `info`.
 *
 * Concurrency: calls from several host threads and on several streams are safe. A call
 * that uses the library-owned buffers (Strassen/Winograd recursion workspace, LU, host
 * pointers) holds the device's call lock while it enqueues, and when the previous such
 * call was on another stream its stream first waits for that call's kernels (an event),
 * so those calls serialise on the device; calls that use no library buffer (Block on
 * device pointers, or with a per-thread caller workspace) run fully concurrently.
 *
 * CUDA graphs: calls may be captured. The library buffers a captured call uses must
 * already be large enough (make the same call once before capturing, or install a
 * caller workspace); growing one during capture fails with DDQD_ENOTSUP. Once a call
 * has been captured, buffers the library outgrows are kept (not freed) until
 * ddqd_release, so a captured graph never points at freed memory; do not call
 * ddqd_release while captured graphs that use library buffers may still be replayed.
 * A captured call does not wait for library calls on other streams outside the graph.
 *
 * Errors: every entry point returns an int status. 0 = success; negative values are
 * the DDQD_E* codes below (no C++ exception crosses the ABI); a human-readable
 * message for the last failure of the calling thread is ddqd_last_error().
 * Zero sizes are valid no-ops (l = 0 gives C := 0). A threshold >= min(m,l,n)
 * degenerates to Block.
 */
#ifndef DDQD_H
#define DDQD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Algorithms. */
enum { DDQD_BLOCK = 0, DDQD_STRASSEN = 1, DDQD_WINOGRAD = 2 };

/* Flag OR-ed into `algo`: the leaf uses the fused multiply-add of docs/numerics.md s.2-3
 * (DD: 15 FP64 instructions instead of the QD-library dd_add(c, dd_mul(a,b)) = 20; QD: the
 * product's expansion enters qd_add's network unrenormalised, one renormalisation fewer;
 * SURVEY.md s.8(f) row f3). Results are then bit-identical to the oracle's fused variant,
 * not (in general) to the canonical one. */
enum { DDQD_MADD_FUSED = 0x100 };

/* Flag OR-ed into `algo` (DD and QD): every addition of the GEMM -- the multiply-add's and
 * every Strassen/Winograd pre/post addition -- is the accurate ("IEEE-style") add of
 * docs/numerics.md s.2-3 (DD 20 FP64 instructions instead of 11; QD the merge-and-accumulate
 * addition), which meets a relative error bound even when leading words cancel (SPEC's
 * add contract S:74). Bit-identical to the oracle's accurate
 * variant. Combined with DDQD_MADD_FUSED -> DDQD_EINVAL; the LU entry points return
 * DDQD_ENOTSUP (their panel/TRSM/solve arithmetic is the canonical one). */
enum { DDQD_ADD_ACCURATE = 0x200 };

/* Split-k leaf (docs/numerics.md s.4): OR DDQD_SPLITK(s), s = 2, 4 or
 * 8, into `algo` and every leaf product (the whole product for DDQD_BLOCK) cuts k into s
 * contiguous slices of ceil(l/s), forms each slice's partial from +0 with k ascending, and
 * combines the partials by the fixed pairwise tree ((p0+p1)+(p2+p3))+... . On the device one
 * thread-block cluster of s CTAs owns a 32x32 tile and the partials meet in distributed shared
 * memory, so small products (config 0: 128^3) fill s times more SMs. A different, documented
 * rounding from the canonical k-ascending sum: bit-identical to the oracle's split-k. */
#define DDQD_SPLITK(s) ((s) == 2 ? 0x1000 : (s) == 4 ? 0x2000 : (s) == 8 ? 0x3000 : 0)

/* Forced recursion depth (reading R21): OR DDQD_DEPTH(d), 0 <= d <= 254, into `algo`
 * (Strassen / Winograd) and the recursion halves (m, l, n) with ceil exactly d times instead of
 * applying the threshold stop rule (`threshold` is then ignored). Used by the multi-GPU band
 * schedule: a row band of A and a column band of B, each the union of one contiguous band of
 * the depth-d leaves' rows (columns) mapped up through the d levels, multiplied with the depth
 * of the whole problem, gives exactly (bitwise) those rows and columns of the whole product --
 * the same recursion tree restricted to the band. Bit-identical to the oracle's forced depth. */
#define DDQD_DEPTH(d) ((int)(((d) + 1) & 0xff) << 16)

/* Precisions: number of float64 words per element. */
enum { DDQD_DD = 2, DDQD_QD = 4 };

/* Status codes. */
enum {
    DDQD_OK = 0,
    DDQD_EINVAL = -1,  /* negative size, bad algo/precision, threshold < 1, bad stride   */
    DDQD_EALIAS = -2,  /* C overlaps A or B                                              */
    DDQD_ENOMEM = -3,  /* workspace / staging allocation failed                          */
    DDQD_ECUDA = -4,   /* a CUDA runtime error (message in ddqd_last_error)              */
    DDQD_ENOTSUP = -5  /* not supported (host pointers to *_ex / LU, accurate-add LU)    */
};

/*
 * dd_gemm / qd_gemm -- C := A B (Eq. (1)) in DD (~106-bit) / QD (~212-bit).
 *   m, l, n   : A is m x l, B is l x n, C is m x n (>= 0).
 *   A, B, C   : planar contiguous [W][rows][cols] (W = 2 for dd_gemm, 4 for qd_gemm).
 *   algo      : DDQD_BLOCK, DDQD_STRASSEN or DDQD_WINOGRAD (the 7-product
 *               recursions whose leaves are Block), optionally OR-ed with DDQD_MADD_FUSED or
 *               DDQD_ADD_ACCURATE, and with DDQD_SPLITK(s) (arithmetic variants above).
 *   threshold : n_min of P:52 -- a (sub)problem recurses while min(m,l,n) > threshold
 *               (>= 1; ignored for DDQD_BLOCK). Odd halves are zero padded virtually.
 * Results are bit-identical to the oracle under docs/numerics.md (k ascending per leaf
 * element, additions in the written order).
 */
int dd_gemm(int64_t m, int64_t l, int64_t n, const double *A, const double *B, double *C,
            int algo, int64_t threshold);
int qd_gemm(int64_t m, int64_t l, int64_t n, const double *A, const double *B, double *C,
            int algo, int64_t threshold);

/* Strided / batched / accumulate form used by the LU and the multi-GPU driver.
 * Element (b, i, j) word w of X lives at X[b*bs + w*ps + i*ld + j] (device pointers only).
 * DDQD_EINVAL if ld < cols, ps < rows*ld, or (batch > 1) bs < words*ps; DDQD_EALIAS if C shares
 * an element with A or B (exact for single views with equal ld and ps -- e.g. disjoint
 * sub-blocks of one matrix are accepted; conservative, by address extent, otherwise).
 * beta = 0: C := A B.  beta = 1: C := C - A B, where A B is first formed from +0 and then
 * subtracted elementwise (dd_sub / qd_sub) -- the LU Schur update of P:131.
 * batch >= 1 independent problems of identical shape share one schedule. */
typedef struct {
    int prec;             /* DDQD_DD or DDQD_QD */
    int algo;             /* DDQD_BLOCK / DDQD_STRASSEN / DDQD_WINOGRAD */
    int64_t threshold;
    int64_t m, l, n;
    int64_t batch;
    const double *A; int64_t lda, psA, bsA;
    const double *B; int64_t ldb, psB, bsB;
    double *C;       int64_t ldc, psC, bsC;
    int beta;             /* 0 or 1 (see above) */
} ddqd_gemm_desc;

int ddqd_gemm_ex(const ddqd_gemm_desc *desc);

/* One recursion level's fused additions, exported for the multi-GPU schedule (which runs
 * the top k levels itself and distributes the 7^k products). A batch of matrices: element
 * (b, i, j) word w at p[b*bs + w*ps + i*ld + j]; rows/cols are the logical extent.
 *   ddqd_pre_add : P parents X (rows x cols) -> 7P children Y (ceil(rows/2) x ceil(cols/2)),
 *                  child c of parent b at batch index 7b + c, for side 0 (A operands) or
 *                  side 1 (B operands) of Strassen / Winograd in the child
 *                  order of docs/numerics.md s.4; missing quadrant rows/cols read as zero.
 *   ddqd_post_add: 7P products M -> P parents C (cropped to C's rows x cols); beta = 1
 *                  subtracts from C instead of storing.
 * algo = DDQD_STRASSEN or DDQD_WINOGRAD, optionally | DDQD_ADD_ACCURATE (accurate adds).
 * Device pointers only; asynchronous on the thread's stream. */
typedef struct {
    double *p;
    int64_t rows, cols, ld, ps, bs;
} ddqd_mat;

int ddqd_pre_add(int prec, int algo, int side, int64_t P, const ddqd_mat *X, const ddqd_mat *Y);
/* ddqd_pre_add storing only the children with index 7b + c in [keep_lo, keep_hi) (the others are
 * left untouched): the multi-GPU schedules form only the ancestors of a rank's own products. */
int ddqd_pre_add_range(int prec, int algo, int side, int64_t P, const ddqd_mat *X, const ddqd_mat *Y,
                       int64_t keep_lo, int64_t keep_hi);
int ddqd_post_add(int prec, int algo, int64_t P, const ddqd_mat *M, const ddqd_mat *C, int beta);

/* The multi-GPU fused combine: one recursion level's post-additions with the
 * 7P children given as a DEVICE array of 7P pointers (child c of parent b at children[7b + c];
 * each a planar W-word hm x hn matrix: word w of (i, j) at child[w*ps + i*ld + j]). The
 * pointers may be CUDA IPC mappings of other GPUs' buffers, so the gather over NVLink and the
 * DD/QD combination run in one kernel. Only position rows [r0, r1) are formed: C quadrant rows
 * i and i + hm of every parent (cropped to C; C = P parents as in ddqd_post_add; beta = 1
 * subtracts). hm, hn must be ceil(C rows / 2), ceil(C cols / 2). Asynchronous. */
int ddqd_post_add_ptrs(int prec, int algo, int64_t P, const double *const *children, int64_t hm, int64_t hn,
                       int64_t ld, int64_t ps, int64_t r0, int64_t r1, const ddqd_mat *C, int beta);

/* Band packing for the multi-GPU band schedule (paper_1510_08642_b200/mgpu.py): a gather /
 * scatter of a rows x cols sub-matrix given by index maps.
 *   dir 0 (pack)  : compact[w][i][j] := full[w][rmap[i]][cmap[j]]
 *   dir 1 (unpack): full[w][rmap[i]][cmap[j]] := compact[w][i][j]
 * rmap: DEVICE int64[rows], cmap: DEVICE int64[cols] (NULL = identity); indices must lie inside
 * full's rows / cols (not checked on the device: the maps come from the caller's own band
 * plan); full and compact are single matrices (bs ignored) with their own ld / ps. Pure data
 * movement (no arithmetic), asynchronous on the thread's stream; DDQD_EINVAL on bad shapes. */
int ddqd_band_copy(int prec, int dir, int64_t rows, int64_t cols, const int64_t *rmap, const int64_t *cmap,
                   const ddqd_mat *full, const ddqd_mat *compact);

/* CUDA IPC plumbing for that combine: ddqd_ipc_alloc allocates a device buffer (cudaMalloc,
 * so it is exportable as a whole); ddqd_ipc_handle writes its 64-byte cudaIpcMemHandle_t;
 * another process maps it with ddqd_ipc_open (peer access enabled lazily) and unmaps it with
 * ddqd_ipc_close; ddqd_ipc_free releases the owner's allocation. DDQD_ENOMEM / DDQD_ECUDA on
 * failure (message in ddqd_last_error). */
int ddqd_ipc_alloc(size_t bytes, void **ptr);
int ddqd_ipc_free(void *ptr);
int ddqd_ipc_handle(const void *ptr, void *handle64);
int ddqd_ipc_open(const void *handle64, void **ptr);
int ddqd_ipc_close(void *ptr);

/*
 * dd_lu_solve -- blocked right-looking LU with partial pivoting (P:121-133 steps 1-3,
 * pivoting per BJ:11) and the solve of Eq. (2), DD only.
 *   n         : order (>= 0).
 *   A         : device [2][n][n], overwritten by P A = L U (unit L below the diagonal, U on
 *               and above it).
 *   b         : device [2][n], untouched.       x: device [2][n], the solution.
 *   ipiv      : device int64[n], ipiv[k] = row swapped with row k at step k (0-based).
 *   panel     : K of P:127 (>= 1); the last panel is ragged.
 *   algo, threshold : GEMM used for the trailing update T := L21 U12.
 * Returns 0, a negative DDQD_E* code, or info > 0: U(info-1, info-1) is exactly zero
 * (LAPACK convention; x is then not a solution). Synchronises the stream once.
 */
int dd_lu_solve(int64_t n, double *A, const double *b, double *x, int64_t *ipiv,
                int64_t panel, int algo, int64_t threshold);

/* QD (4-word) LU with partial pivoting + solve; arguments as dd_lu_solve with [4][n][n] /
 * [4][n] planes (divisions are qd_div of docs/numerics.md s.3). */
int qd_lu_solve(int64_t n, double *A, const double *b, double *x, int64_t *ipiv,
                int64_t panel, int algo, int64_t threshold);

/* General form: prec = DDQD_DD / DDQD_QD; pivot = 1 partial pivoting (BJ:11), 0 = the paper's
 * pivot-free LU ("none of the LU decomposition involves pivoting"; ipiv[k] = k, a zero
 * pivot returns info = k+1). Other arguments and return values as dd_lu_solve. */
int ddqd_lu_solve(int prec, int pivot, int64_t n, double *A, const double *b, double *x,
                  int64_t *ipiv, int64_t panel, int algo, int64_t threshold);

/* The LU's steps as separate calls, for a caller that runs the Schur update itself (the
 * multi-GPU LU of paper_1510_08642_b200/mgpu.py distributes it).
 *   ddqd_lu_panel: steps 1-2 of docs/numerics.md s.5 for the panel of columns [p, p+kb) of the
 *     planar row-major [prec][n][n] matrix A (rows p..n-1): pivot search (pivot = 1) or the
 *     pivot-free rule (pivot = 0), interchanges over all n columns (ipiv[k] for k in the panel),
 *     reciprocal and scaling, the panel's rank-1 updates, then U12 := L11^{-1} A12 by forward
 *     substitution. The caller then forms A22 := A22 - L21 U12 (e.g. ddqd_gemm_ex with beta = 1).
 *     Returns 0, k+1 for the first exactly zero pivot in this panel (LAPACK-style, the rest of
 *     that column's step skipped), or a negative DDQD_E* code. Synchronises.
 *   ddqd_lu_trsv: the solve of Eq. (2) with the factors (y := P b, unit-lower forward,
 *     upper backward with dd_div / qd_div); b, x: [prec][n]; b untouched. Asynchronous.
 * Device pointers only; 0 <= p, 1 <= kb, p + kb <= n (kb <= 1024 when p + kb < n). */
int ddqd_lu_panel(int prec, int pivot, int64_t n, double *A, int64_t *ipiv, int64_t p, int64_t kb);
int ddqd_lu_trsv(int prec, int64_t n, const double *LU, const int64_t *ipiv, const double *b, double *x);

/* Elementwise arithmetic layer, for parity tests of the device DD/QD ops (device
 * pointers, planar [W][count]): op 0 add, 1 sub, 2 mul, 3 div, 4 madd z = x + y*w,
 * 5 fused madd (DDQD_MADD_FUSED's operation), 6 accurate add, 7 accurate sub,
 * 8 accurate madd z = x + y*w (DDQD_ADD_ACCURATE's operations, DD and QD). */
int ddqd_elementwise(int prec, int op, int64_t count, const double *x, const double *y,
                     const double *w, double *z);

/* Stream used by the calling thread (a cudaStream_t; NULL = legacy default stream). */
int ddqd_set_stream(void *cuda_stream);

/* Bytes of device workspace a GEMM of this shape uses (0 for Block). */
size_t ddqd_workspace_bytes(int prec, int64_t m, int64_t l, int64_t n, int algo, int64_t threshold);

/* Caller-owned workspace for the calling thread (NULL/0 to revert to the library's own).
 * Calls that need more than `bytes` fail with DDQD_ENOMEM. */
int ddqd_set_workspace(void *dptr, size_t bytes);

/* Upper bound on the library-owned workspace (bytes); the recursion schedule runs its top
 * levels depth-first when breadth-first batching would exceed it. 0 = default (40% of free
 * device memory at first use). Numerics do not depend on it. */
int ddqd_set_workspace_limit(size_t bytes);

/* Number of kernels this thread's library calls have launched so far (evidence counter). */
int64_t ddqd_launch_count(void);

/* Live kernel timing (CUDA events on the launching stream) for bench.py's roofline:
 * between start and stop every leaf-GEMM / pre-add / post-add launch is bracketed by
 * events. stop() synchronises and writes, for class c = 0 leaf GEMM, 1 pre-add, 2 post-add,
 * 3 LU panel factorisation, 4 LU TRSM, 5 LU solve: out[3c+0] = total ms, out[3c+1] =
 * bracketed regions, out[3c+2] = work (madds for c = 0, 3, 4; algorithmic bytes for c = 1, 2;
 * n^2 for c = 5); cap = number of doubles in out (18 for all classes). */
int ddqd_profile_start(void);
int ddqd_profile_stop(double *out, int cap);
/* Per-kernel breakdown of the last ddqd_profile_stop: one line per kernel (leaf variants are
 * named separately, e.g. "leaf_tma_kernel (TMA, row-pair A)" / "leaf_gemm_kernel<...> (cp.async)"),
 * "name \t class \t total ms \t launches \t work \n", NUL-terminated, truncated to cap bytes.
 * Returns the bytes needed (including the NUL); out = NULL / cap = 0 only measures. */
int ddqd_profile_kernels(char *out, size_t cap);

/* FP64-pipe throughput probe: op 0 = DFMA, 1 = DADD stream; returns lane-operations per
 * second on the current device (and the per-launch ms). Roofline denominator of the leaf. */
int ddqd_fp64_peak(int op, double *lane_ops_per_s, double *ms);

/* Free library-owned device memory (workspace, staging buffers) of the current device. */
int ddqd_release(void);

/* Message of the last failure on the calling thread ("" if none). */
const char *ddqd_last_error(void);

/* ABI version (major*100 + minor). */
int ddqd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DDQD_H */
