// blas.cu -- the full BLAS dgemm surface on top of the my_dgemm kernels
// (SURVEY.md 8f "next" rank 3):  C := alpha * op(A) * op(B) + beta * C,
// op(X) = X or X^T.  The reference describes this interface
// and keeps only the simplified C := A B + C; this entry point is
// the natural next caller-facing step for LAPACK-style code.
//
// * op(A) / op(B) = transpose: an HBM-bound tiled transpose into stream-
//   ordered workspace, then the NN kernels (so the per-element arithmetic is
//   exactly the NN kernels' on the explicitly transposed operand);
// * alpha == 1 && beta == 1: the my_dgemm contract (accumulator starts at C);
//   beta == 0: the BLAS epilogue alpha * (A B accumulated from 0), C never
//   read; any other beta on the tiled kernel: the reference BLAS order --
//   C := beta C first (skipped for beta == 1), the smaller of op(A), op(B)
//   scaled by alpha into workspace (netlib's temp = alpha * B(l, j)), then
//   the contract (the epilogue's read of C after the K loop cost ~370 us
//   per 8192^2 C, tools/blas_epilogue_probe.py); the bandwidth kernels keep
//   the epilogue alpha * (A B) + beta * C;
// * quick returns and alpha == 0 / k == 0 follow the reference BLAS rules.
#include <algorithm>
#include <cstdio>
#include <string>

#include "../../include/my_dgemm.h"
#include "common.cuh"

namespace myd {

cudaError_t dispatch(int m, int n, int k, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                     int64_t ldc, cudaStream_t st, unsigned flags, const Epilogue &ep);
int capi_fail(int status, const std::string &msg);
bool path_fits(int m, int n, unsigned flags);
int capi_ok();
int capi_cuda_fail(cudaError_t e, const char *where);
void keep_pool_memory();

// dst (cols x rows, ld ldd) = src^T (src: rows x cols, ld lds); 32x32 tiles.
__global__ void transpose_kernel(int64_t rows, int64_t cols, const double *__restrict__ src, int64_t lds,
                                 double *__restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int dj = threadIdx.y; dj < 32; dj += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + dj;
    if (i < rows && j < cols) tile[dj][threadIdx.x] = src[j * lds + i];
  }
  __syncthreads();
  for (int di = threadIdx.y; di < 32; di += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + di;  // dst(j, i)
    if (i < rows && j < cols) dst[i * ldd + j] = tile[threadIdx.x][di];
  }
}

// dst (rows x cols) := alpha * src
__global__ void scale_copy_kernel(int64_t rows, int64_t cols, const double *__restrict__ src, int64_t lds,
                                  double *__restrict__ dst, int64_t ldd, double alpha) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
      dst[j * ldd + i] = alpha * src[j * lds + i];
}

// C := beta * C over the valid region (beta == 0 writes zeros without reading).
__global__ void scale_kernel(int64_t m, int64_t n, double *__restrict__ C, int64_t ldc, double beta) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      C[j * ldc + i] = beta == 0.0 ? 0.0 : beta * C[j * ldc + i];
}

static cudaError_t launch_transpose(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst,
                                    int64_t ldd, cudaStream_t st) {
  const int64_t gy = (cols + 31) / 32;
  for (int64_t y0 = 0; y0 < gy; y0 += 65535) {  // gridDim.y limit
    const int64_t gyy = std::min<int64_t>(65535, gy - y0);
    transpose_kernel<<<dim3((unsigned)((rows + 31) / 32), (unsigned)gyy), dim3(32, 8), 0, st>>>(
        rows, cols - y0 * 32, src + y0 * 32 * lds, lds, dst + y0 * 32, ldd);
    count_launch();
  }
  return cudaGetLastError();
}

static cudaError_t launch_scale(int64_t m, int64_t n, double *C, int64_t ldc, double beta, cudaStream_t st) {
  const int64_t gx = std::min<int64_t>((m + 255) / 256, 64), gy = std::min<int64_t>(n, 65535);
  scale_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(m, n, C, ldc, beta);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_scale_copy(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst,
                                     int64_t ldd, double alpha, cudaStream_t st) {
  const int64_t gx = std::min<int64_t>((rows + 255) / 256, 64), gy = std::min<int64_t>(cols, 65535);
  scale_copy_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(rows, cols, src, lds, dst, ldd, alpha);
  count_launch();
  return cudaGetLastError();
}

int path_kind(int m, int n, unsigned flags);

static bool is_trans(char t) { return t == 'T' || t == 't' || t == 'C' || t == 'c'; }
static bool valid_trans(char t) { return t == 'N' || t == 'n' || is_trans(t); }

// Device-resident BLAS dgemm (asynchronous on st).  Arguments validated.
// fold: allow the reference-BLAS order (scale C, scale an operand, then the
// contract) on the tiled kernel; callers issuing many small updates from one
// operand (level3.cu) keep the epilogue, which needs no extra pass.
int blas_device(char ta, char tb, int m, int n, int k, double alpha, const double *A, int lda,
                       const double *B, int ldb, double beta, double *C, int ldc, unsigned flags, cudaStream_t st,
                       bool fold) {
  cudaError_t e;
  if (alpha == 0.0 || k == 0) {
    if (beta == 1.0) return capi_ok();
    e = launch_scale(m, n, C, ldc, beta, st);
    return e == cudaSuccess ? capi_ok() : capi_cuda_fail(e, "scale");
  }
  const bool tA = is_trans(ta), tB = is_trans(tb);
  if (tA || tB) keep_pool_memory();
  const int64_t ldA = ((int64_t)m + 1) & ~1LL, ldB = ((int64_t)k + 1) & ~1LL;
  // workspace freed (stream-ordered) on every return path
  struct Scratch {
    double *p[2] = {nullptr, nullptr};
    cudaStream_t st;
    ~Scratch() {
      for (double *q : p)
        if (q) cudaFreeAsync(q, st);
    }
  } scratch{{nullptr, nullptr}, st};
  double *&wa = scratch.p[0], *&wb = scratch.p[1];
  const double *opA = A, *opB = B;
  int64_t lda_op = lda, ldb_op = ldb;
  if (tA) {  // A stored k x m; op(A) = A^T (m x k)
    if ((e = cudaMallocAsync((void **)&wa, (size_t)ldA * k * 8, st)) != cudaSuccess)
      return capi_cuda_fail(e, "cudaMallocAsync(op(A))");
    if ((e = launch_transpose(k, m, A, lda, wa, ldA, st)) != cudaSuccess) return capi_cuda_fail(e, "transpose A");
    opA = wa;
    lda_op = ldA;
  }
  if (tB) {  // B stored n x k; op(B) = B^T (k x n)
    if ((e = cudaMallocAsync((void **)&wb, (size_t)ldB * n * 8, st)) != cudaSuccess)
      return capi_cuda_fail(e, "cudaMallocAsync(op(B))");
    if ((e = launch_transpose(n, k, B, ldb, wb, ldB, st)) != cudaSuccess) return capi_cuda_fail(e, "transpose B");
    opB = wb;
    ldb_op = ldB;
  }
  Epilogue ep;
  ep.alpha = alpha;
  ep.beta = beta;
  ep.blas = !(alpha == 1.0 && beta == 1.0);
  if (fold && ep.blas && beta != 0.0 && path_kind(m, n, flags & ~MY_DGEMM_DEVICE_PTRS) == MY_DGEMM_PATH_TILED) {
    if (beta != 1.0 && (e = launch_scale(m, n, C, ldc, beta, st)) != cudaSuccess) return capi_cuda_fail(e, "scale C");
    if (alpha != 1.0) {
      keep_pool_memory();
      const bool on_a = (int64_t)m * k <= (int64_t)k * n;  // scale the smaller operand
      double *&w = on_a ? wa : wb;
      const double *&op = on_a ? opA : opB;
      int64_t &ldo = on_a ? lda_op : ldb_op;
      const int64_t rows = on_a ? m : k, cols = on_a ? k : n;
      if (!w) {
        const int64_t ldw = (rows + 1) & ~1LL;
        if ((e = cudaMallocAsync((void **)&w, (size_t)ldw * cols * 8, st)) != cudaSuccess)
          return capi_cuda_fail(e, "cudaMallocAsync(alpha op)");
        if ((e = launch_scale_copy(rows, cols, op, ldo, w, ldw, alpha, st)) != cudaSuccess)
          return capi_cuda_fail(e, "alpha op");
        op = w;
        ldo = ldw;
      } else if ((e = launch_scale(rows, cols, w, ldo, alpha, st)) != cudaSuccess) {  // transposed copy: in place
        return capi_cuda_fail(e, "alpha op");
      }
    }
    ep = Epilogue{};  // the my_dgemm contract
  }
  e = dispatch(m, n, k, opA, lda_op, opB, ldb_op, C, ldc, st, flags & ~MY_DGEMM_DEVICE_PTRS, ep);
  return e == cudaSuccess ? capi_ok() : capi_cuda_fail(e, "kernel launch");
}

}  // namespace myd

using namespace myd;

extern "C" int my_dgemm_blas(char transa, char transb, int m, int n, int k, double alpha, const double *A, int lda,
                             const double *B, int ldb, double beta, double *C, int ldc, unsigned flags,
                             void *stream) {
  // Reference-BLAS argument checks, in its order (1-based parameter index).
  char buf[160];
  if (!valid_trans(transa)) return capi_fail(-1, "transa must be 'N', 'T' or 'C'");
  if (!valid_trans(transb)) return capi_fail(-2, "transb must be 'N', 'T' or 'C'");
  if (m < 0) return capi_fail(-3, "m must be non-negative");
  if (n < 0) return capi_fail(-4, "n must be non-negative");
  if (k < 0) return capi_fail(-5, "k must be non-negative");
  const int nrowa = is_trans(transa) ? k : m, nrowb = is_trans(transb) ? n : k;
  if (lda < std::max(1, nrowa)) {
    snprintf(buf, sizeof buf, "lda=%d smaller than max(1, %d)", lda, nrowa);
    return capi_fail(-8, buf);
  }
  if (ldb < std::max(1, nrowb)) {
    snprintf(buf, sizeof buf, "ldb=%d smaller than max(1, %d)", ldb, nrowb);
    return capi_fail(-10, buf);
  }
  if (ldc < std::max(1, m)) {
    snprintf(buf, sizeof buf, "ldc=%d smaller than max(1, %d)", ldc, m);
    return capi_fail(-13, buf);
  }
  const unsigned known = MY_DGEMM_DEVICE_PTRS | MY_DGEMM_EXACT | MY_DGEMM_FORCE_TILED | MY_DGEMM_FORCE_VEC1 |
                         MY_DGEMM_FORCE_STRIPS2 | MY_DGEMM_FORCE_STRIPS4 | MY_DGEMM_FORCE_UNITS8 |
                         MY_DGEMM_FORCE_ROWS16 | MY_DGEMM_FORCE_STREAMK | MY_DGEMM_PATH_MASK |
                         MY_DGEMM_BLAS_EPILOGUE | MY_DGEMM_PLAN_INVARIANT | MY_DGEMM_FORCE_KSPLIT;
  if (flags & ~known) return capi_fail(-14, "unknown flag bits");
  const bool fold = !(flags & MY_DGEMM_BLAS_EPILOGUE);
  flags &= ~MY_DGEMM_BLAS_EPILOGUE;
  if (m > 0 && n > 0 && !path_fits(m, n, flags))
    return capi_fail(-14, "MY_DGEMM_FORCE_PATH does not suit the shape");
  if ((flags & MY_DGEMM_EXACT) && !(alpha == 1.0 && beta == 1.0))
    return capi_fail(-14, "MY_DGEMM_EXACT needs alpha == 1 and beta == 1 (the reference oracle's operation)");
  // quick return (reference BLAS)
  if (m == 0 || n == 0 || ((alpha == 0.0 || k == 0) && beta == 1.0)) return capi_ok();
  const bool need_ab = alpha != 0.0 && k > 0;
  if (need_ab && !A) return capi_fail(-7, "A is NULL");
  if (need_ab && !B) return capi_fail(-9, "B is NULL");
  if (!C) return capi_fail(-12, "C is NULL");

  if (flags & MY_DGEMM_DEVICE_PTRS)
    return blas_device(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, flags, (cudaStream_t)stream,
                       fold);

  // Host operands: stage through stream-ordered device buffers (pitched
  // copies never touch padding rows), run on the device, copy C back.
  keep_pool_memory();
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return capi_cuda_fail(e, "cudaStreamCreate");
  const int ncola = is_trans(transa) ? m : k, ncolb = is_trans(transb) ? k : n;
  double *dA = nullptr, *dB = nullptr, *dC = nullptr;
  const int64_t dlda = ((int64_t)std::max(1, nrowa) + 1) & ~1LL, dldb = ((int64_t)std::max(1, nrowb) + 1) & ~1LL,
                dldc = ((int64_t)m + 1) & ~1LL;
  int status = 0;
  do {
    if (need_ab) {
      if ((e = cudaMallocAsync((void **)&dA, (size_t)dlda * ncola * 8, st)) != cudaSuccess) break;
      if ((e = cudaMallocAsync((void **)&dB, (size_t)dldb * ncolb * 8, st)) != cudaSuccess) break;
      if ((e = cudaMemcpy2DAsync(dA, dlda * 8, A, (size_t)lda * 8, (size_t)nrowa * 8, ncola, cudaMemcpyHostToDevice,
                                 st)) != cudaSuccess)
        break;
      if ((e = cudaMemcpy2DAsync(dB, dldb * 8, B, (size_t)ldb * 8, (size_t)nrowb * 8, ncolb, cudaMemcpyHostToDevice,
                                 st)) != cudaSuccess)
        break;
    }
    if ((e = cudaMallocAsync((void **)&dC, (size_t)dldc * n * 8, st)) != cudaSuccess) break;
    if (beta != 0.0 && (e = cudaMemcpy2DAsync(dC, dldc * 8, C, (size_t)ldc * 8, (size_t)m * 8, n,
                                              cudaMemcpyHostToDevice, st)) != cudaSuccess)
      break;
    status = blas_device(transa, transb, m, n, k, alpha, dA, (int)dlda, dB, (int)dldb, beta, dC, (int)dldc,
                         flags | MY_DGEMM_DEVICE_PTRS, st, fold);
    if (status != 0) break;
    if ((e = cudaMemcpy2DAsync(C, (size_t)ldc * 8, dC, dldc * 8, (size_t)m * 8, n, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      break;
    e = cudaStreamSynchronize(st);
  } while (false);
  if (dA) cudaFreeAsync(dA, st);
  if (dB) cudaFreeAsync(dB, st);
  if (dC) cudaFreeAsync(dC, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (status != 0) return status;
  if (e != cudaSuccess) return capi_cuda_fail(e, "host-path BLAS dgemm");
  return capi_ok();
}
