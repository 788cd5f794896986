/*
 * my_dgemm.h -- C ABI of the B200-native (sm_100a) FP64 GEMM.
 *
 * Drop-in for the reference's `my_dgemm` path: C := A*B + C on column-major
 * float64 matrices with explicit leading dimensions.  Element (i, j) of a
 * matrix with leading dimension ld is at offset j*ld + i
 * (reference PAPER.md:273, pkg/src/gemmforge/matrix.py:34-36).
 *
 * Every entry point below replaces a reference interface; the citation is on
 * each declaration (paths relative to /root/reference).  Plain pointers and
 * sizes only; no torch or CUDA types appear in the signatures (streams are
 * passed as void*, a cudaStream_t).
 *
 * Status codes (int-returning calls):
 *      0                    success
 *     -1 .. -9              argument i (1-based: m, n, k, A, lda, B, ldb, C, ldc)
 *                           is invalid; nothing was read or written.  This is
 *                           the ValueError of pkg/src/gemmforge/kernels.py:41-49
 *                           and matrix.py:50-53 (dims < 1, ld < rows, NULL).
 *    -10                    flags invalid
 *    -11                    argument out of range for a non-GEMM entry point
 *     1000 + cudaError_t    CUDA runtime failure (C may be partially written)
 *     2000 + ncclResult_t   reserved for the collective layer
 * my_dgemm_last_error() returns a message for the last non-zero status on the
 * calling thread, in the reference's ValueError wording where one exists.
 */
#ifndef MY_DGEMM_B200_H
#define MY_DGEMM_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define MY_DGEMM_API __attribute__((visibility("default")))
#else
#define MY_DGEMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Flags for my_dgemm_ex. */
#define MY_DGEMM_DEVICE_PTRS 0x1u /* A, B, C are device pointers; async on `stream` */
#define MY_DGEMM_EXACT 0x2u       /* bitwise twin of the reference oracle (verification) */
#define MY_DGEMM_FORCE_TILED 0x4u /* bypass the m==1 / n==1 bandwidth kernels */
#define MY_DGEMM_FORCE_VEC1 0x8u  /* force 8-byte operand staging (odd-ld path) */
#define MY_DGEMM_FORCE_STRIPS2 0x10u /* run every tile as two 128x64 strips (tests) */
#define MY_DGEMM_FORCE_STRIPS4 0x20u /* run every tile as four 128x32 strips (tests) */
#define MY_DGEMM_FORCE_UNITS8 0x40u  /* run every tile as eight 64x32 units (tests) */
#define MY_DGEMM_FORCE_ROWS16 0x80u  /* run every tile as eight 16x128 units (tests) */
#define MY_DGEMM_FORCE_STREAMK 0x800u /* stream-K schedule (tests): of full tiles, or with STRIPS2 / STRIPS4 /
                                          UNITS8 of those units, when there is at least one per SM */
#define MY_DGEMM_BLAS_EPILOGUE 0x1000u /* my_dgemm_blas (tests): apply alpha / beta in the kernel epilogue
                                          instead of the reference-BLAS order (C := beta C, alpha folded
                                          into an operand, then the contract) that large tiled calls use */
#define MY_DGEMM_FORCE_SMALL 0x2000u /* tiled path on the small-block kernel (tests, tuner); variant below */
/* Small-block kernel variant v (1..10, block / slab / ring shapes listed in
 * csrc/dgemm_small.cu; 0: the cheapest by the planner's model), with
 * MY_DGEMM_FORCE_SMALL. */
#define MY_DGEMM_SMALL_VARIANT(v) ((unsigned)(v) << 14)
#define MY_DGEMM_SMALL_MASK 0x3C000u
#define MY_DGEMM_FORCE_TILES 0x40000u /* every tile as a full 128x128 tile (tests, tuner: plan 1) */
/* Every launch plan of the tiled path but one gives each element of C the same
 * ascending chain of k-steps, so C is bitwise independent of the plan, of
 * k-chunking at multiples of 16 and of the shard count.  The exception is the
 * opt-in K-split plan (plan 48) for problems with fewer 128x128 tiles than
 * SMs: a tile's K range is cut into pieces that run on several SMs at once
 * and whose partial sums the tile's owner adds in a fixed order -- still
 * deterministic (a function of m, n, k and the SM count) and within the
 * stated tolerance, but not that chain.  It runs only when asked for:
 * MY_DGEMM_FORCE_KSPLIT on the call (when the shape allows it; otherwise the
 * heuristic's plan-invariant choice), or MY_DGEMM_KSPLIT=1 in the environment,
 * which lets the planner cost it against the other plans (off by default: it
 * measured no faster).  MY_DGEMM_PLAN_INVARIANT keeps a call to
 * the plan-invariant plans even then; MY_DGEMM_FORCE_PATH (sharded drivers),
 * an SM cap, a pinned plan and the host path's panel pipeline imply it. */
#define MY_DGEMM_PLAN_INVARIANT 0x80000u
#define MY_DGEMM_FORCE_KSPLIT 0x100000u
/* Run this call on kernel family p (MY_DGEMM_PATH_*, see my_dgemm_path) whatever
 * the shape's own choice would be: sharded drivers pass the whole problem's
 * path to every shard so C is bitwise independent of the shard count.  The
 * path must suit the shape (n == 1 / m == 1 / n <= 16 / m <= 16), else -10. */
#define MY_DGEMM_FORCE_PATH(p) ((unsigned)((p) + 1) << 8)
#define MY_DGEMM_PATH_MASK 0x700u

/*
 * The BASELINE.json north_star signature.  Replaces the reference's
 * `my_dgemm(m, n, k, A, lda, B, ldb, C, ldc)` whose
 * Python realisation is gemm_goto / gemm_goto_parallel
 * (pkg/src/gemmforge/goto.py:187-239, parallel.py:108-243).  Host pointers,
 * synchronous.  On invalid arguments C is untouched and the status is kept
 * for my_dgemm_last_error() / my_dgemm_last_status().
 */
MY_DGEMM_API void my_dgemm(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc);

/* Same-signature alias named after the paper's test driver. */
MY_DGEMM_API void bl_dgemm(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc);

/*
 * Status-returning form with flags and a CUDA stream (NULL = default stream).
 * With MY_DGEMM_DEVICE_PTRS the call is asynchronous on `stream`; otherwise
 * it stages through device memory and returns when C is written back.
 * Replaces the engine call of the registry variant factory
 * (pkg/src/gemmforge/registry.py:185-198, `_goto_factory.run`).
 */
MY_DGEMM_API int my_dgemm_ex(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
                unsigned flags, void *stream);

/*
 * Full BLAS dgemm surface: C := alpha * op(A) * op(B) + beta * C with
 * op(X) = X ('N') or X^T ('T'/'C'); the interface of PAPER.md:542-556, which
 * the reference leaves out of scope.  Reference-BLAS argument
 * rules: status -i names the first invalid parameter i (1 transa, 2 transb,
 * 3 m, 4 n, 5 k, 7 A, 8 lda, 9 B, 10 ldb, 12 C, 13 ldc, 14 flags); m, n or
 * k = 0 and alpha = 0 are legal (quick return / C := beta C, C not read when
 * beta = 0).  With alpha = beta = 1 the result is bitwise my_dgemm_ex on
 * op(A), op(B).  Flags as for my_dgemm_ex (MY_DGEMM_EXACT only with
 * alpha = beta = 1).
 */
MY_DGEMM_API int my_dgemm_blas(char transa, char transb, int m, int n, int k, double alpha, const double *A, int lda,
                  const double *B, int ldb, double beta, double *C, int ldc, unsigned flags, void *stream);

/*
 * GEMM-based level-3 BLAS ("poorman's BLAS",
 * PAPER.md:1-15): blocked algorithms whose O(n^3) work is my_dgemm_blas
 * calls on the DMMA kernels, plus small diagonal-block kernels.  Reference-
 * BLAS argument order, checks (negative status = 1-based index of the bad
 * argument; the flags argument is the last index) and quick returns.
 * Device pointers only (flags must hold MY_DGEMM_DEVICE_PTRS; optional
 * MY_DGEMM_FORCE_TILED), asynchronous on `stream`.
 *   my_dsyrk: C := alpha op(A) op(A)^T + beta C on the uplo triangle of the
 *             n x n C (op(A) n x k); the other triangle is never touched.
 *   my_dtrmm: B := alpha op(A) B (side 'L') or alpha B op(A) (side 'R').
 *   my_dtrsm: solves op(A) X = alpha B (side 'L') or X op(A) = alpha B
 *             (side 'R'); X overwrites B.  A triangular (uplo), diag 'U'
 *             takes its diagonal as 1 without reading it.
 */
MY_DGEMM_API int my_dsyrk(char uplo, char trans, int n, int k, double alpha, const double *A, int lda, double beta,
                          double *C, int ldc, unsigned flags, void *stream);
MY_DGEMM_API int my_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha, const double *A,
                          int lda, double *B, int ldb, unsigned flags, void *stream);
MY_DGEMM_API int my_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha, const double *A,
                          int lda, double *B, int ldb, unsigned flags, void *stream);

/*
 * jc-sharded piece of a multi-GPU GEMM: the caller's rank computes
 * C[:, j0:j0+nloc] += A[:, p0:p0+kc] * B[p0:p0+kc, j0:j0+nloc] with device
 * pointers already offset by the caller.  Identical to my_dgemm_ex with
 * MY_DGEMM_DEVICE_PTRS; kept as a separate symbol so the collective layer's
 * calls are visible in traces.  Replaces the per-worker block call of
 * pkg/src/gemmforge/parallel.py:156-164 (`block_call`).
 */
MY_DGEMM_API int my_dgemm_shard(int m, int nloc, int kc, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
                   void *stream);

/*
 * Host-pointer my_dgemm spread over the GPUs 0..ngpu-1 of this process
 * (SURVEY.md 8b `my_dgemm_multi(int ngpu, ...)`; the reference's threaded
 * driver pkg/src/gemmforge/parallel.py:108-243 split over devices instead of
 * cores).  Device g owns the balanced column panel g of B and C
 * (128-column units); A's k-chunks are uploaded round-robin over the
 * devices' PCIe links and copied peer to peer.  C is bitwise the
 * single-device my_dgemm result for every ngpu.  Status: -1 bad ngpu (< 1
 * or more than the visible devices), -2..-10 as my_dgemm_ex's -1..-9.
 */
MY_DGEMM_API int my_dgemm_multi(int ngpu, int m, int n, int k, const double *A, int lda, const double *B, int ldb,
                                double *C, int ldc);

/*
 * my_dgemm_multi on an explicit device list (shard s on devices[s]; an entry
 * may repeat -- each entry is an independent shard with its own buffers,
 * which is how the multi-device logic is exercised on one GPU).  flags: 0 or
 * MY_DGEMM_EXACT.  Status: -1 devices NULL, -2 bad ndev / device id,
 * -3..-11 as my_dgemm_ex's -1..-9, -12 unknown flags.
 */
MY_DGEMM_API int my_dgemm_multi_ex(const int *devices, int ndev, int m, int n, int k, const double *A, int lda,
                                   const double *B, int ldb, double *C, int ldc, unsigned flags);

/*
 * Device-side splitmix64-v1 operand fill: element (i, j) of the m x n matrix
 * at `dev` (leading dimension ld) takes stream position t = (col0 + j)*m + i,
 * i.e. exactly pkg/src/gemmforge/matrix.py:184-207 (`random_values`,
 * `fill_random`) when col0 = 0.  A non-zero col0 lets a rank fill the column
 * panel [col0, col0+n) of a larger m x N matrix with the values the full fill
 * would give it.  Padding rows are never written.  Asynchronous on `stream`.
 */
MY_DGEMM_API int my_dgemm_fill_random(double *dev, int64_t m, int64_t n, int64_t ld, uint64_t seed, int64_t col0, void *stream);

/* pkg/src/gemmforge/bench.py:89-98 (`_operand_seed`). Pure host integer hash. */
MY_DGEMM_API uint64_t my_dgemm_operand_seed(uint64_t seed, uint64_t role, int64_t m, int64_t n, int64_t k);

/*
 * Device-side parity metric (pkg/src/gemmforge/matrix.py:210-232,
 * `max_abs_diff`): max |X - Y| over the valid m x n region, and the first
 * element (column-major scan) with |X - Y| > tol, or -1.  Device pointers;
 * synchronous.  out_first_bad receives the flat index j*m + i.
 */
MY_DGEMM_API int my_dgemm_max_abs_diff(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy,
                          double tol, double *out_max, int64_t *out_first_bad, void *stream);

/*
 * The same scan plus the offender's pair (X and Y at the first bad element),
 * i.e. the reference's DiffReport (matrix.py:90-107: max_abs_diff,
 * first_bad_i/j, value_got, value_expected) from which its
 * "C[ i ][ j ] != C_ref, %E, %E" line is formed (bench.py:84-86,150-156).
 * out_got / out_want are left untouched when there is no offender.
 * Offender rule as the reference: strict |X - Y| > tol, so a NaN difference
 * is not an offender but makes out_max NaN.
 */
MY_DGEMM_API int my_dgemm_diff_report(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y,
                                      int64_t ldy, double tol, double *out_max, int64_t *out_first_bad,
                                      double *out_got, double *out_want, void *stream);

/*
 * CTA-plan autotuner (the GPU analogue of the reference's grid tuner,
 * pkg/src/gemmforge/bench.py:238-311): times every launch plan of the fast
 * kernel for this shape (heuristic, full tiles only, all 128x64 / 128x32 /
 * 64x32 units) on scratch device operands and remembers the fastest for
 * later calls of the same shape and operand alignment in this process.
 * These plans are bitwise-equivalent: tuning changes speed, never results
 * (the opt-in K-split plan, 48, is not among them).
 * out_plan: 0 heuristic, 1 full tiles, 2/4/8 units per tile (128x64 / 128x32 /
 * 64x32), 16 for 16x128 units, 32 / 34 / 36 / 40 stream-K over full tiles /
 * 128x64 / 128x32 / 64x32 units.
 */
MY_DGEMM_API int my_dgemm_tune(int m, int n, int k, int lda, int ldb, int ldc, int reps, int *out_plan, double *out_ms);
/*
 * Tile parameters of launch plan `plan` (my_dgemm_tune's plan ids, plus
 * 65..74 = the small-block kernel's variants 1..10) at depth k: the CTA block
 * bm x bn, the K-slab depth bk and the shared-memory ring depth stages, as
 * compiled (vec2 != 0: 16-byte operand staging).  These are the GPU's blocking
 * parameters (the reference's mc / nc / kc, Config.goto, config.py:24-40);
 * engine.tune_grid searches them like the reference's tune()
 * (pkg/src/gemmforge/bench.py:238-311).  Returns 0, or -1 for an unknown plan.
 */
MY_DGEMM_API int my_dgemm_plan_geometry(int plan, int k, int vec2, int *bm, int *bn, int *bk, int *stages);
/*
 * The tiled path's launch plan for a shape, as one line of text ("... units |
 * stream-K | K-split | small split=.. sk_split=.. sk_dp_rounds=.. q=.. edge=..
 * small=.. model_us=.."), without launching anything: the planner is host code
 * (csrc/dgemm_fast.cu:launch_dgemm_fast), so this works without a GPU (it then
 * plans for 148 SMs).  plan: 0 = the heuristic, what a default call of this
 * shape runs (pins of my_dgemm_tune_set aside); -1 = the heuristic kept to the
 * plan-invariant plans; otherwise a plan id as my_dgemm_tune reports them.
 * The analogue of the reference's make_plan (pkg/src/gemmforge/parallel.py:60-105):
 * the work decomposition as data, testable on its own.  Returns 0, -1 for bad
 * arguments, -2 if the shape cannot be planned.
 */
MY_DGEMM_API int my_dgemm_plan_describe(int m, int n, int k, int lda, int ldb, int ldc, int plan, char *buf, int len);
/* Pin `plan` for later calls of this shape and operand alignment (what
 * my_dgemm_tune records; engine.tune_grid's winner).  Negative status for a
 * bad argument or an unknown plan. */
MY_DGEMM_API int my_dgemm_tune_set(int m, int n, int k, int lda, int ldb, int plan);
MY_DGEMM_API void my_dgemm_tune_clear(void);

/*
 * Cap the persistent tiled kernel's grid at n CTAs (one per SM) for this
 * process, leaving the other SMs to concurrent work -- e.g. the NCCL kernels
 * of a broadcast overlapped with the GEMM (the reference's analogue is the
 * thread count of gemm_goto_parallel, pkg/src/gemmforge/parallel.py:108-243).
 * 0 = every SM (default).  Returns the previous cap, or -1 for n < 0.
 * Results are bitwise independent of the cap.
 */
MY_DGEMM_API int my_dgemm_set_max_ctas(int n);

/*
 * The kernel family a call of this shape and these flags runs on: the tiled
 * DMMA kernel, or one of the bandwidth kernels for a short dimension.  Tiled
 * calls of one problem are bitwise invariant to column sharding, k-chunking
 * (multiples of 16) and launch plan; sharded drivers therefore pass
 * MY_DGEMM_FORCE_TILED to every shard exactly when the whole problem's path
 * is MY_DGEMM_PATH_TILED.  Negative status for m or n < 1.
 */
#define MY_DGEMM_PATH_TILED 0
#define MY_DGEMM_PATH_GEMV_N1 1  /* n == 1 */
#define MY_DGEMM_PATH_GEMV_M1 2  /* m == 1 */
#define MY_DGEMM_PATH_FEW_COLS 3 /* 2 <= n <= 16, m >= 4096 */
#define MY_DGEMM_PATH_FEW_ROWS 4 /* 2 <= m <= 4, n <= 65536 (FMA kernel; forced: m <= 16) */
#define MY_DGEMM_PATH_EXACT 5    /* MY_DGEMM_EXACT */
#define MY_DGEMM_PATH_ROWS_DMMA 6 /* 5 <= m <= 16 (forced: m <= 32): B streamed into DMMA fragments */
MY_DGEMM_API int my_dgemm_path(int m, int n, unsigned flags);

/*
 * NVLink peer-memory plumbing of the multi-GPU driver's exchange step (the A
 * broadcast of SURVEY 8e; the reference's threads share A in one address
 * space, pkg/src/gemmforge/parallel.py:108-243, so it has no counterpart
 * call).  paper_1609_00076_b200/peer.py builds a copy-engine chain from them:
 * each rank pulls k-chunks of A from its predecessor's HBM and signals its
 * successor, all stream-ordered, no SM involved.
 *
 * my_dgemm_ipc_export: CUDA IPC handle (MY_DGEMM_IPC_HANDLE_BYTES bytes) of the
 *   allocation holding dev_ptr, and dev_ptr's offset in it.
 * my_dgemm_ipc_open / _close: map another process's buffer (lazy peer access);
 *   returns base + offset.  Not within the exporting process.
 * my_dgemm_signal_write: stream-ordered 32-bit store to a (local or peer-mapped)
 *   device flag, after the stream's earlier work is complete and visible.
 * my_dgemm_signal_wait_geq: the stream waits until (int32_t)(*flag - value) >= 0.
 * my_dgemm_copy_async: stream-ordered copy between device (or peer) addresses
 *   by the copy engines.
 */
#define MY_DGEMM_IPC_HANDLE_BYTES 64
MY_DGEMM_API int my_dgemm_ipc_export(const void *dev_ptr, unsigned char *handle_out, uint64_t *offset_out);
MY_DGEMM_API int my_dgemm_ipc_open(const unsigned char *handle, uint64_t offset, void **dev_ptr_out);
MY_DGEMM_API int my_dgemm_ipc_close(void *dev_ptr, uint64_t offset);
MY_DGEMM_API int my_dgemm_signal_write(void *stream, uint32_t *dev_flag, uint32_t value);
MY_DGEMM_API int my_dgemm_signal_wait_geq(void *stream, const uint32_t *dev_flag, uint32_t value);
MY_DGEMM_API int my_dgemm_copy_async(void *dst, const void *src, uint64_t bytes, void *stream);

/* Diagnostics. */
MY_DGEMM_API const char *my_dgemm_last_error(void);
MY_DGEMM_API int my_dgemm_last_status(void);
MY_DGEMM_API const char *my_dgemm_version(void);
/* Number of kernels this library has launched since load (all threads). */
MY_DGEMM_API uint64_t my_dgemm_kernel_launches(void);
/* Release cached device/pinned workspace of the host-pointer path. */
MY_DGEMM_API void my_dgemm_release_workspace(void);

#ifdef __cplusplus
}
#endif

#endif /* MY_DGEMM_B200_H */
