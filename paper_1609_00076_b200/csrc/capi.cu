// capi.cu -- the drop-in C ABI (include/my_dgemm.h) over the sm_100a kernels.
//
// Validation mirrors the reference's ValueError checks, always before any
// memory is touched (pkg/src/gemmforge/goto.py:196-204, kernels.py:41-49,
// matrix.py:50-53).  The host-pointer path stages operands through cached
// device workspace with pitched copies (width m*8, pitch ld*8), so padding
// rows are never read or written and nothing past (n-1)*ld+m is touched
// (matrix.py:5-6,42-45,58-61).  The host path lives in host_path.cu.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/my_dgemm.h"
#include "common.cuh"

namespace myd {

cudaError_t launch_dgemm_fast(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                              double *C, int64_t ldc, cudaStream_t stream, bool force_vec1, int force_split,
                              const Epilogue &ep);
cudaError_t launch_dgemm_exact(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream);
cudaError_t launch_gemv_n1(int M, int K, const double *A, int64_t lda, const double *b, double *C,
                           cudaStream_t stream, const Epilogue &ep);
cudaError_t launch_gemv_m1(int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                           int64_t ldc, cudaStream_t stream, const Epilogue &ep);
cudaError_t launch_gemm_nsmall(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep);
cudaError_t launch_gemm_msmall(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep);
cudaError_t launch_gemm_rows_dmma(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                                  double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep);
cudaError_t launch_fill_random(double *out, int64_t m, int64_t n, int64_t ld, uint64_t seed, int64_t col0,
                               cudaStream_t stream);
cudaError_t launch_copy2d(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd,
                          cudaStream_t stream);
cudaError_t launch_max_abs_diff(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy,
                                double tol, unsigned long long *d_out2, cudaStream_t stream);

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int tuned_plan(int m, int n, int k, int64_t lda, int64_t ldb);

// Stream-ordered scratch (odd-ld copies, BLAS transposes) comes from the
// device's default memory pool; keep its memory instead of returning it to
// the OS at every synchronisation, so repeated calls do not re-map pages.
void keep_pool_memory() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done.fetch_or(bit, std::memory_order_release);
}

// Which kernel a call uses (my_dgemm_path): the bandwidth kernels take the
// shapes with one short dimension -- m == 1; few rows: m <= 4 with
// n <= 65536 on the FMA kernel, 5 <= m <= 16 on the DMMA row kernel (1.1-2x
// the tiled kernel's 16x128 units, which use only n/128 SMs;
// profiles/rows_dmma_r01.log); n == 1; few columns (n <= 16 with m >= 4096)
// -- every other shape is tiled.  Sharded drivers pass the whole problem's
// path to every shard (MY_DGEMM_FORCE_PATH), so a narrow shard never changes
// kernel.  Measurements: tools/nsmall_probe.py, tools/msmall_probe.py,
// tools/rows_dmma_probe.py.
int path_kind(int m, int n, unsigned flags) {
  if (flags & MY_DGEMM_EXACT) return MY_DGEMM_PATH_EXACT;
  if (flags & MY_DGEMM_PATH_MASK) return (int)((flags & MY_DGEMM_PATH_MASK) >> 8) - 1;
  if (flags & MY_DGEMM_FORCE_TILED) return MY_DGEMM_PATH_TILED;
  if (m == 1) return MY_DGEMM_PATH_GEMV_M1;
  if (m <= 4 && n <= 65536) return MY_DGEMM_PATH_FEW_ROWS;
  if (n == 1) return MY_DGEMM_PATH_GEMV_N1;
  if (m >= 5 && m <= 16) return MY_DGEMM_PATH_ROWS_DMMA;
  if (n <= 16 && m >= 4096) return MY_DGEMM_PATH_FEW_COLS;
  return MY_DGEMM_PATH_TILED;
}

// A forced path must suit the shape.
bool path_fits(int m, int n, unsigned flags) {
  if (!(flags & MY_DGEMM_PATH_MASK)) return true;
  switch ((int)((flags & MY_DGEMM_PATH_MASK) >> 8) - 1) {
    case MY_DGEMM_PATH_TILED: return true;
    case MY_DGEMM_PATH_GEMV_N1: return n == 1;
    case MY_DGEMM_PATH_GEMV_M1: return m == 1;
    case MY_DGEMM_PATH_FEW_COLS: return n <= 16;
    case MY_DGEMM_PATH_FEW_ROWS: return m <= 16;
    case MY_DGEMM_PATH_ROWS_DMMA: return m <= 32;
    default: return false;
  }
}

// Device-pointer dispatch: picks the kernel for the shape.
cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags, const Epilogue &ep) {
  switch (path_kind(m, n, flags)) {
    case MY_DGEMM_PATH_EXACT: return launch_dgemm_exact(m, n, k, A, lda, B, ldb, C, ldc, st);
    case MY_DGEMM_PATH_GEMV_M1: return launch_gemv_m1(n, k, A, lda, B, ldb, C, ldc, st, ep);
    case MY_DGEMM_PATH_FEW_ROWS: return launch_gemm_msmall(m, n, k, A, lda, B, ldb, C, ldc, st, ep);
    case MY_DGEMM_PATH_ROWS_DMMA: return launch_gemm_rows_dmma(m, n, k, A, lda, B, ldb, C, ldc, st, ep);
    case MY_DGEMM_PATH_GEMV_N1: return launch_gemv_n1(m, k, A, lda, B, C, st, ep);
    case MY_DGEMM_PATH_FEW_COLS: return launch_gemm_nsmall(m, n, k, A, lda, B, ldb, C, ldc, st, ep);
    default: break;
  }
  int split = (flags & MY_DGEMM_FORCE_ROWS16)    ? 16
              : (flags & MY_DGEMM_FORCE_UNITS8)  ? 8
              : (flags & MY_DGEMM_FORCE_STRIPS4) ? 4
              : (flags & MY_DGEMM_FORCE_STRIPS2) ? 2
                                                 : 0;
  if (flags & MY_DGEMM_FORCE_STREAMK) split = 32 + (split == 16 ? 0 : split);  // stream-K over those units
  if (flags & MY_DGEMM_FORCE_SMALL) split = 64 + (int)((flags & MY_DGEMM_SMALL_MASK) >> 14);  // small-block kernel
  if (flags & MY_DGEMM_FORCE_TILES) split = 1;  // full tiles only
  if (flags & MY_DGEMM_FORCE_KSPLIT) split = 48;  // K-split plan (when the shape allows it)
  if (split == 0) split = tuned_plan(m, n, k, lda, ldb);  // 0 unless my_dgemm_tune chose one
  // sharded drivers (forced path) and callers asking for it: heuristic over the plan-invariant plans only
  if (split == 0 && (flags & (MY_DGEMM_PATH_MASK | MY_DGEMM_PLAN_INVARIANT))) split = -1;
  const bool force_vec1 = (flags & MY_DGEMM_FORCE_VEC1) != 0;
  const bool a_ok = lda % 2 == 0 && (uintptr_t)A % 16 == 0, b_ok = ldb % 2 == 0 && (uintptr_t)B % 16 == 0;
  // Worth a scratch copy when the GEMM is big, or when its K chain is long:
  // a small m x n problem runs K in order on few SMs, and 8-byte staging
  // costs it ~2x (17 x 64 x 4096: 194 us vs 83 us at m = 64, profiles/shape_scan_r01.log).
  if (!force_vec1 && (!a_ok || !b_ok) && ((double)m * n * k >= (double)(1 << 24) || k >= 512)) {
    keep_pool_memory();
    // Odd leading dimension (or 8-byte aligned view) of A or B: copy the
    // operand once into an even-ld scratch copy so the bulk-copy staging
    // applies.  Each copy costs 16 bytes per element of the operand against
    // 2mnk flops; the arithmetic, hence C, is bitwise unchanged.  C itself is
    // never copied: the kernel stages an unaligned C with 8-byte copies and
    // stores it with scalar stores, which is cheaper than a round trip
    // through scratch (tools/oddc_probe.py: 16384^2 x 256, ldc odd: 4.41 ms
    // in place vs 5.71 ms with a C copy; 8192^3: 30.28 vs 30.65 ms).
    double *wa = nullptr, *wb = nullptr;
    const double *a2 = A, *b2 = B;
    int64_t lda2 = lda, ldb2 = ldb;
    bool ok = true;
    if (!a_ok) {
      lda2 = ((int64_t)m + 1) & ~1LL;
      ok = cudaMallocAsync((void **)&wa, (size_t)lda2 * k * 8, st) == cudaSuccess &&
           launch_copy2d(m, k, A, lda, wa, lda2, st) == cudaSuccess;
      a2 = wa;
    }
    if (ok && !b_ok) {
      ldb2 = ((int64_t)k + 1) & ~1LL;
      ok = cudaMallocAsync((void **)&wb, (size_t)ldb2 * n * 8, st) == cudaSuccess &&
           launch_copy2d(k, n, B, ldb, wb, ldb2, st) == cudaSuccess;
      b2 = wb;
    }
    cudaError_t e = cudaSuccess;
    if (ok) e = launch_dgemm_fast(m, n, k, a2, lda2, b2, ldb2, C, ldc, st, false, split, ep);
    if (wa) cudaFreeAsync(wa, st);
    if (wb) cudaFreeAsync(wb, st);
    if (ok) return e;
    cudaGetLastError();  // scratch unavailable: fall through to 8-byte staging
  }
  return launch_dgemm_fast(m, n, k, A, lda, B, ldb, C, ldc, st, force_vec1, split, ep);
}

}  // namespace myd

using namespace myd;

namespace {

thread_local int t_status = 0;
thread_local std::string t_error;

int fail(int status, const std::string &msg) {
  t_status = status;
  t_error = msg;
  return status;
}

int ok() {
  t_status = 0;
  t_error.clear();
  return 0;
}

int cuda_fail(cudaError_t e, const char *where) {
  return fail(1000 + (int)e, std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
}

// Reference messages: kernels.py:41-49 (conformal), matrix.py:50-53 (dims, ld).
int validate(int m, int n, int k, const void *A, int lda, const void *B, int ldb, const void *C, int ldc) {
  char buf[256];
  if (m < 1 || n < 1 || k < 1) {
    const int which = m < 1 ? -1 : (n < 1 ? -2 : -3);
    snprintf(buf, sizeof buf, "matrix dims must be positive, got m=%d n=%d k=%d", m, n, k);
    return fail(which, buf);
  }
  if (!A) return fail(-4, "A is NULL");
  if (lda < m) {
    snprintf(buf, sizeof buf, "leading dimension ld=%d smaller than row count m=%d", lda, m);
    return fail(-5, buf);
  }
  if (!B) return fail(-6, "B is NULL");
  if (ldb < k) {
    snprintf(buf, sizeof buf, "leading dimension ld=%d smaller than row count m=%d", ldb, k);
    return fail(-7, buf);
  }
  if (!C) return fail(-8, "C is NULL");
  if (ldc < m) {
    snprintf(buf, sizeof buf, "leading dimension ld=%d smaller than row count m=%d", ldc, m);
    return fail(-9, buf);
  }
  return 0;
}

int visible_devices() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    count = 0;
  }
  return count;
}

cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags) {
  return myd::dispatch(m, n, k, A, lda, B, ldb, C, ldc, st, flags, Epilogue{});
}

}  // namespace

namespace myd {
int host_path(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
              unsigned flags);
void release_host_workspace();
void release_multi_workspace();
int set_max_ctas(int n);
int multi_host_path(const int *devices, int G, int m, int n, int k, const double *A, int lda, const double *B,
                    int ldb, double *C, int ldc, unsigned flags);
int capi_fail(int status, const std::string &msg) { return fail(status, msg); }
int capi_ok() { return ok(); }
int capi_cuda_fail(cudaError_t e, const char *where) { return cuda_fail(e, where); }
}  // namespace myd

extern "C" {

int my_dgemm_ex(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
                unsigned flags, void *stream) {
  int v = validate(m, n, k, A, lda, B, ldb, C, ldc);
  if (v) return v;
  const unsigned known = MY_DGEMM_DEVICE_PTRS | MY_DGEMM_EXACT | MY_DGEMM_FORCE_TILED | MY_DGEMM_FORCE_VEC1 |
                         MY_DGEMM_FORCE_STRIPS2 | MY_DGEMM_FORCE_STRIPS4 | MY_DGEMM_FORCE_UNITS8 |
                         MY_DGEMM_FORCE_ROWS16 | MY_DGEMM_FORCE_STREAMK | MY_DGEMM_PATH_MASK | MY_DGEMM_FORCE_SMALL |
                         MY_DGEMM_SMALL_MASK | MY_DGEMM_FORCE_TILES | MY_DGEMM_PLAN_INVARIANT |
                         MY_DGEMM_FORCE_KSPLIT;
  if (flags & ~known) return fail(-10, "unknown flag bits");
  if (!path_fits(m, n, flags)) return fail(-10, "MY_DGEMM_FORCE_PATH does not suit the shape");
  if (flags & MY_DGEMM_DEVICE_PTRS) {
    // A host pointer here would fault the GPU; reject it as an argument error.
    const void *ptrs[3] = {A, B, C};
    for (int i = 0; i < 3; ++i) {
      cudaPointerAttributes at;
      const bool dev_ok = cudaPointerGetAttributes(&at, ptrs[i]) == cudaSuccess &&
                          (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
      if (!dev_ok) {
        cudaGetLastError();
        const int which[3] = {-4, -6, -8};
        return fail(which[i], std::string(i == 0 ? "A" : (i == 1 ? "B" : "C")) +
                                  " is not a device pointer (MY_DGEMM_DEVICE_PTRS)");
      }
    }
    cudaError_t e = dispatch(m, n, k, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, flags);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return ok();
  }
  return myd::host_path(m, n, k, A, lda, B, ldb, C, ldc, flags);
}

void my_dgemm(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc) {
  const int s = my_dgemm_ex(m, n, k, A, lda, B, ldb, C, ldc, 0u, nullptr);
  if (s != 0 && getenv("MY_DGEMM_VERBOSE")) fprintf(stderr, "my_dgemm: %s\n", t_error.c_str());
}

void bl_dgemm(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc) {
  my_dgemm(m, n, k, A, lda, B, ldb, C, ldc);
}

int my_dgemm_shard(int m, int nloc, int kc, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
                   void *stream) {
  return my_dgemm_ex(m, nloc, kc, A, lda, B, ldb, C, ldc, MY_DGEMM_DEVICE_PTRS, stream);
}

int my_dgemm_fill_random(double *dev, int64_t m, int64_t n, int64_t ld, uint64_t seed, int64_t col0, void *stream) {
  if (m < 1) return fail(-1, "matrix dims must be positive");
  if (n < 1) return fail(-2, "matrix dims must be positive");
  if (ld < m) return fail(-3, "leading dimension smaller than row count");
  if (!dev) return fail(-4, "buffer is NULL");
  if (col0 < 0) return fail(-11, "col0 must be non-negative");
  cudaError_t e = launch_fill_random(dev, m, n, ld, seed, col0, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill_random");
  return ok();
}

uint64_t my_dgemm_operand_seed(uint64_t seed, uint64_t role, int64_t m, int64_t n, int64_t k) {
  const uint64_t G = 0x9E3779B97F4A7C15ULL;
  uint64_t h = seed ^ (role * G);
  const int64_t dims[3] = {m, n, k};
  for (int d = 0; d < 3; ++d) {
    h = h + G + (uint64_t)dims[d];
    h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ULL;
    h = (h ^ (h >> 27)) * 0x94D049BB133111EBULL;
    h ^= h >> 31;
  }
  return h;
}

int my_dgemm_diff_report(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy, double tol,
                         double *out_max, int64_t *out_first_bad, double *out_got, double *out_want, void *stream) {
  if (m < 1) return fail(-1, "matrix dims must be positive");
  if (n < 1) return fail(-2, "matrix dims must be positive");
  if (!X) return fail(-3, "X is NULL");
  if (ldx < m) return fail(-4, "leading dimension smaller than row count");
  if (!Y) return fail(-5, "Y is NULL");
  if (ldy < m) return fail(-6, "leading dimension smaller than row count");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *d = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&d, 16, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  unsigned long long init[2] = {0ULL, ~0ULL};
  e = cudaMemcpyAsync(d, init, 16, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = launch_max_abs_diff(m, n, X, ldx, Y, ldy, tol, d, st);
  unsigned long long h[2] = {0ULL, ~0ULL};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "max_abs_diff");
  double mx;
  memcpy(&mx, &h[0], 8);
  const int64_t first = (h[1] == ~0ULL) ? -1 : (int64_t)h[1];
  if (out_max) *out_max = mx;
  if (out_first_bad) *out_first_bad = first;
  if (first >= 0 && (out_got || out_want)) {  // the offender's pair, for the reference's failure line
    const int64_t j = first / m, i = first % m;
    double g = 0.0, w = 0.0;
    e = cudaMemcpyAsync(&g, X + j * ldx + i, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&w, Y + j * ldy + i, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "max_abs_diff offender");
    if (out_got) *out_got = g;
    if (out_want) *out_want = w;
  }
  return ok();
}

int my_dgemm_max_abs_diff(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy,
                          double tol, double *out_max, int64_t *out_first_bad, void *stream) {
  return my_dgemm_diff_report(m, n, X, ldx, Y, ldy, tol, out_max, out_first_bad, nullptr, nullptr, stream);
}

const char *my_dgemm_last_error(void) { return t_error.c_str(); }
int my_dgemm_last_status(void) { return t_status; }
const char *my_dgemm_version(void) { return "paper_1609_00076_b200 0.1.0 sm_100a dmma"; }
uint64_t my_dgemm_kernel_launches(void) { return g_launches.load(); }

int my_dgemm_path(int m, int n, unsigned flags) {
  if (m < 1) return fail(-1, "matrix dims must be positive");
  if (n < 1) return fail(-2, "matrix dims must be positive");
  if (!path_fits(m, n, flags)) return fail(-3, "MY_DGEMM_FORCE_PATH does not suit the shape");
  return myd::path_kind(m, n, flags);
}

int my_dgemm_set_max_ctas(int n) {
  if (n < 0) return fail(-1, "max_ctas must be >= 0 (0 = every SM), got " + std::to_string(n));
  return myd::set_max_ctas(n);
}

void my_dgemm_release_workspace(void) {
  myd::release_host_workspace();
  myd::release_multi_workspace();
}

int my_dgemm_multi_ex(const int *devices, int ndev, int m, int n, int k, const double *A, int lda, const double *B,
                      int ldb, double *C, int ldc, unsigned flags) {
  if (!devices) return fail(-1, "devices is NULL");
  if (ndev < 1 || ndev > 64) return fail(-2, "ndev must be in 1..64, got " + std::to_string(ndev));
  int v = validate(m, n, k, A, lda, B, ldb, C, ldc);
  if (v) return fail(v - 2, t_error);
  if (flags & ~MY_DGEMM_EXACT) return fail(-12, "unknown flag bits (my_dgemm_multi_ex takes 0 or MY_DGEMM_EXACT)");
  const int count = visible_devices();
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count)
      return fail(-2, "device id " + std::to_string(devices[i]) + " not visible (" + std::to_string(count) +
                          " devices)");
  return myd::multi_host_path(devices, ndev, m, n, k, A, lda, B, ldb, C, ldc, flags);
}

int my_dgemm_multi(int ngpu, int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C,
                   int ldc) {
  if (ngpu < 1 || ngpu > 64) return fail(-1, "ngpu must be in 1..64, got " + std::to_string(ngpu));
  int v = validate(m, n, k, A, lda, B, ldb, C, ldc);
  if (v) return fail(v - 1, t_error);
  const int count = visible_devices();
  if (ngpu > count)
    return fail(-1, "ngpu=" + std::to_string(ngpu) + " but " + std::to_string(count) + " devices are visible");
  int devs[64];
  for (int i = 0; i < ngpu; ++i) devs[i] = i;
  return myd::multi_host_path(devs, ngpu, m, n, k, A, lda, B, ldb, C, ldc, 0u);
}

}  // extern "C"
