// capi.cu -- the drop-in C ABI (include/my_dgemm.h) over the sm_100a kernels.
//
// Validation mirrors the reference's ValueError checks, always before any
// memory is touched (pkg/src/gemmforge/goto.py:196-204, kernels.py:41-49,
// matrix.py:50-53).  The host-pointer path stages operands through cached
// device workspace with pitched copies (width m*8, pitch ld*8), so padding
// rows are never read or written and nothing past (n-1)*ld+m is touched
// (matrix.py:5-6,42-45,58-61).  Large problems are pipelined (host_path).
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
cudaError_t launch_fill_random(double *out, int64_t m, int64_t n, int64_t ld, uint64_t seed, int64_t col0,
                               cudaStream_t stream);
cudaError_t launch_max_abs_diff(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy,
                                double tol, unsigned long long *d_out2, cudaStream_t stream);

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

// Device-pointer dispatch: picks the kernel for the shape.
cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags, const Epilogue &ep) {
  if (flags & MY_DGEMM_EXACT) return launch_dgemm_exact(m, n, k, A, lda, B, ldb, C, ldc, st);
  if (!(flags & MY_DGEMM_FORCE_TILED)) {
    if (n == 1) return launch_gemv_n1(m, k, A, lda, B, C, st, ep);
    if (m == 1) return launch_gemv_m1(n, k, A, lda, B, ldb, C, ldc, st, ep);
  }
  const int split = (flags & MY_DGEMM_FORCE_UNITS8)    ? 8
                    : (flags & MY_DGEMM_FORCE_STRIPS4) ? 4
                    : (flags & MY_DGEMM_FORCE_STRIPS2) ? 2
                                                       : 0;
  return launch_dgemm_fast(m, n, k, A, lda, B, ldb, C, ldc, st, (flags & MY_DGEMM_FORCE_VEC1) != 0, split, ep);
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

cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags) {
  return myd::dispatch(m, n, k, A, lda, B, ldb, C, ldc, st, flags, Epilogue{});
}

// ---- host-pointer path: cached per-device workspace, panel pipeline ----
struct Workspace {
  int device = -1;
  double *dA = nullptr, *dB = nullptr, *dC = nullptr;
  size_t capA = 0, capB = 0, capC = 0;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done, ev_out;
};

std::mutex g_ws_mutex;
Workspace g_ws[64];

cudaError_t grow(double **p, size_t *cap, size_t need) {
  if (*cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void **)p, need);
  if (e == cudaSuccess) *cap = need;
  return e;
}

cudaError_t ensure_streams(Workspace &w, size_t panels) {
  cudaError_t e;
  if (!w.s_h2d) {
    if ((e = cudaStreamCreateWithFlags(&w.s_h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&w.s_comp, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&w.s_d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
  }
  while (w.ev_in.size() < panels) {
    cudaEvent_t a, b, c;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&c, cudaEventDisableTiming)) != cudaSuccess) return e;
    w.ev_in.push_back(a);
    w.ev_done.push_back(b);
    w.ev_out.push_back(c);
  }
  return cudaSuccess;
}

int host_path(int m, int n, int k, const double *A, int lda, const double *B, int ldb, double *C, int ldc,
              unsigned flags) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(-11, "device index out of range");
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  Workspace &w = g_ws[dev];
  w.device = dev;
  // Device copies use even leading dimensions so every column starts 16-byte
  // aligned and the 16-byte staging path applies whatever the host ld was.
  const int64_t dlda = (m + 1) & ~1LL, dldb = (k + 1) & ~1LL, dldc = (m + 1) & ~1LL;
  // Schedule (host path, large problems).  Measured on the B200 box: 55 GB/s
  // H2D and 57 GB/s D2H over PCIe 5, but only ~34 GB/s in total when both
  // directions run at once, so uploads go first and downloads are deferred
  // until every upload is queued; the GEMM overlaps both.  A first column
  // group (half of C) is computed in k-chunks as A arrives, so the GEMM runs
  // at full width while A is still uploading (chunks are multiples of 16:
  // bitwise the unchunked result); the remaining panels run whole as their
  // B and C land.  (tools/e2e_schedule_sim.py models the alternatives.)
  const double flops = 2.0 * m * (double)n * k;
  const bool pipelined = flops > 4e9 && n >= 1024 && m > 1 && n > 1;
  int64_t nc0 = n, panel = n;
  if (pipelined) {
    nc0 = std::max<int64_t>(128, (n / 2) / 128 * 128);
    panel = std::max<int64_t>(512, ((n / 8 + 127) / 128) * 128);
  }
  const size_t panels = 1 + (size_t)((n - nc0 + panel - 1) / panel);  // group 0 + whole panels
  auto panel_j0 = [&](size_t p) -> int64_t { return p == 0 ? 0 : nc0 + (int64_t)(p - 1) * panel; };
  auto panel_nc = [&](size_t p) -> int64_t { return p == 0 ? nc0 : std::min<int64_t>(panel, n - panel_j0(p)); };
  int64_t kchunk = k;
  if (pipelined && k >= 256) kchunk = (((k + 7) / 8) + 15) / 16 * 16;
  const size_t kchunks = (size_t)((k + kchunk - 1) / kchunk);
  if ((e = ensure_streams(w, std::max(panels, kchunks) + 1)) != cudaSuccess) return cuda_fail(e, "stream setup");
  if ((e = grow(&w.dA, &w.capA, (size_t)dlda * k * 8)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(A)");
  if ((e = grow(&w.dB, &w.capB, (size_t)dldb * n * 8)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(B)");
  if ((e = grow(&w.dC, &w.capC, (size_t)dldc * n * 8)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(C)");

  auto h2d = [&](double *dst, int64_t dpitch, const double *src, int64_t spitch, int64_t rows, int64_t cols) {
    return cudaMemcpy2DAsync(dst, dpitch * 8, src, (size_t)spitch * 8, (size_t)rows * 8, cols,
                             cudaMemcpyHostToDevice, w.s_h2d);
  };
  // uploads: C of group 0, then (A chunk, B chunk of group 0) pairs, then (B_p, C_p)
  if ((e = h2d(w.dC, dldc, C, ldc, m, nc0)) != cudaSuccess) return cuda_fail(e, "H2D C");
  for (size_t c = 0; c < kchunks; ++c) {
    const int64_t p0 = (int64_t)c * kchunk, kl = std::min<int64_t>(kchunk, k - p0);
    if ((e = h2d(w.dA + p0 * dlda, dlda, A + p0 * lda, lda, m, kl)) != cudaSuccess) return cuda_fail(e, "H2D A");
    if ((e = h2d(w.dB + p0, dldb, B + p0, ldb, kl, nc0)) != cudaSuccess) return cuda_fail(e, "H2D B");
    cudaEventRecord(w.ev_in[c], w.s_h2d);
  }
  for (size_t p = 1; p < panels; ++p) {
    const int64_t j0 = panel_j0(p), nc = panel_nc(p);
    if ((e = h2d(w.dB + j0 * dldb, dldb, B + j0 * ldb, ldb, k, nc)) != cudaSuccess) return cuda_fail(e, "H2D B");
    if ((e = h2d(w.dC + j0 * dldc, dldc, C + j0 * ldc, ldc, m, nc)) != cudaSuccess) return cuda_fail(e, "H2D C");
    cudaEventRecord(w.ev_done[p], w.s_h2d);  // reused below as the panel's "inputs landed" event
  }
  cudaEvent_t all_in = w.ev_in[kchunks];  // every upload done: downloads may start
  cudaEventRecord(all_in, w.s_h2d);

  // compute: group 0 by k-chunks, then whole panels
  for (size_t c = 0; c < kchunks; ++c) {
    const int64_t p0 = (int64_t)c * kchunk, kl = std::min<int64_t>(kchunk, k - p0);
    cudaStreamWaitEvent(w.s_comp, w.ev_in[c], 0);
    e = dispatch(m, (int)nc0, (int)kl, w.dA + p0 * dlda, dlda, w.dB + p0, dldb, w.dC, dldc, w.s_comp, flags);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  }
  auto d2h = [&](int64_t j0, int64_t nc) {
    return cudaMemcpy2DAsync(C + j0 * ldc, (size_t)ldc * 8, w.dC + j0 * dldc, dldc * 8, (size_t)m * 8, nc,
                             cudaMemcpyDeviceToHost, w.s_d2h);
  };
  std::vector<cudaEvent_t> &done = w.ev_out;
  cudaEventRecord(done[0], w.s_comp);
  for (size_t p = 1; p < panels; ++p) {
    const int64_t j0 = panel_j0(p), nc = panel_nc(p);
    cudaStreamWaitEvent(w.s_comp, w.ev_done[p], 0);
    e = dispatch(m, (int)nc, k, w.dA, dlda, w.dB + j0 * dldb, dldb, w.dC + j0 * dldc, dldc, w.s_comp, flags);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    cudaEventRecord(done[p], w.s_comp);
  }
  cudaStreamWaitEvent(w.s_d2h, all_in, 0);
  for (size_t p = 0; p < panels; ++p) {
    const int64_t j0 = panel_j0(p), nc = panel_nc(p);
    cudaStreamWaitEvent(w.s_d2h, done[p], 0);
    if ((e = d2h(j0, nc)) != cudaSuccess) return cuda_fail(e, "D2H C");
  }
  e = cudaStreamSynchronize(w.s_d2h);
  if (e != cudaSuccess) return cuda_fail(e, "synchronize");
  e = cudaStreamSynchronize(w.s_comp);
  if (e != cudaSuccess) return cuda_fail(e, "synchronize");
  return ok();
}

}  // namespace

namespace myd {
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
                         MY_DGEMM_FORCE_STRIPS2 | MY_DGEMM_FORCE_STRIPS4 | MY_DGEMM_FORCE_UNITS8;
  if (flags & ~known) return fail(-10, "unknown flag bits");
  if (flags & MY_DGEMM_DEVICE_PTRS) {
    cudaError_t e = dispatch(m, n, k, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, flags);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return ok();
  }
  return host_path(m, n, k, A, lda, B, ldb, C, ldc, flags);
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

int my_dgemm_max_abs_diff(int64_t m, int64_t n, const double *X, int64_t ldx, const double *Y, int64_t ldy,
                          double tol, double *out_max, int64_t *out_first_bad, void *stream) {
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
  if (out_max) *out_max = mx;
  if (out_first_bad) *out_first_bad = (h[1] == ~0ULL) ? -1 : (int64_t)h[1];
  return ok();
}

const char *my_dgemm_last_error(void) { return t_error.c_str(); }
int my_dgemm_last_status(void) { return t_status; }
const char *my_dgemm_version(void) { return "paper_1609_00076_b200 0.1.0 sm_100a dmma"; }
uint64_t my_dgemm_kernel_launches(void) { return g_launches.load(); }

void my_dgemm_release_workspace(void) {
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  for (auto &w : g_ws) {
    if (w.device < 0) continue;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(w.device);
    if (w.dA) cudaFree(w.dA);
    if (w.dB) cudaFree(w.dB);
    if (w.dC) cudaFree(w.dC);
    w.dA = w.dB = w.dC = nullptr;
    w.capA = w.capB = w.capC = 0;
    cudaSetDevice(prev);
  }
}

}  // extern "C"
