// level3.cu -- GEMM-based level-3 BLAS on the my_dgemm kernels (SURVEY.md 8f
// "next" rank 4: "poorman's BLAS", PAPER.md:1-15 after Kagstrom, Ling and
// Van Loan, TOMS 24(3) 1998): DSYRK, DTRMM and DTRSM, each a blocked
// algorithm whose O(n^3) part is BLAS dgemm calls (blas.cu, i.e. the tiled /
// few-row DMMA kernels) and whose remainder is a small diagonal-block kernel:
//
// * DSYRK: C := alpha op(A) op(A)^T + beta C on one triangle.  Off-diagonal
//   panels of each 512-column block are plain dgemm calls on C; the 512x512
//   diagonal block is computed whole into workspace (alpha = 1, beta = 0:
//   the product from zero) and merged into the triangle with the dgemm
//   epilogue's own arithmetic (beta == 0 ? alpha s : fma(alpha, s, beta c)),
//   so the other triangle is never read or written.
// * DTRMM / DTRSM: B := alpha op(A) B, B := alpha B op(A) and their solves.
//   The four side x effective-triangle cases are ordered so that each block
//   row / column is finished from operands not yet overwritten; blocks of 512
//   recurse into blocks of 128 and 32 (trmm: one dgemm on a dense copy of
//   each 512 diagonal block instead), whose diagonal part runs in
//   tri_diag_kernel (one thread per vector, the 32x32 triangle staged in
//   shared memory, the vector in registers) and the rest in dgemm calls (beta = 1, alpha = +-1).
//
// Device pointers only (MY_DGEMM_DEVICE_PTRS), asynchronous on the stream;
// argument checks and quick returns follow the reference BLAS, with the
// 1-based parameter index as the negative status.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/my_dgemm.h"
#include "common.cuh"

namespace myd {

int blas_device(char ta, char tb, int m, int n, int k, double alpha, const double *A, int lda, const double *B,
                int ldb, double beta, double *C, int ldc, unsigned flags, cudaStream_t st, bool fold);
int capi_fail(int status, const std::string &msg);
int capi_ok();
int capi_cuda_fail(cudaError_t e, const char *where);
void keep_pool_memory();

namespace {

constexpr int TB = 32;    // diagonal-block kernel size (the vector stays in registers)
constexpr int OB = 512;   // outer block: dgemm updates are rank-512

// Block sizes (MY_DGEMM_L3_BLOCKS="outer,middle" overrides, for A/B only):
// outer blocks recurse into middle blocks (0: straight to TB), then TB.
struct Blocks {
  int outer = OB, middle = 128;
};
const Blocks &blocks() {
  static const Blocks b = [] {
    Blocks v;
    if (const char *e = getenv("MY_DGEMM_L3_BLOCKS")) {
      int o = 0, mdl = 0;
      if (sscanf(e, "%d,%d", &o, &mdl) == 2 && o >= TB && o % TB == 0 && mdl >= 0 && mdl < o && mdl % TB == 0) {
        v.outer = o;
        v.middle = mdl;
      }
    }
    return v;
  }();
  return b;
}
int inner_bs(int bs) {
  const Blocks &b = blocks();
  return bs > b.middle && b.middle > TB ? b.middle : TB;
}

bool up(char c) { return c == 'U' || c == 'u'; }
bool lo(char c) { return c == 'L' || c == 'l'; }
bool tr(char c) { return c == 'T' || c == 't' || c == 'C' || c == 'c'; }
bool nt(char c) { return c == 'N' || c == 'n'; }

// C(triangle) := beta == 0 ? alpha W : fma(alpha, W, beta C) on an nb x nb
// diagonal block; the other triangle is untouched.
__global__ void syrk_merge_kernel(int nb, const double *__restrict__ W, int64_t ldw, double *__restrict__ C,
                                  int64_t ldc, double alpha, double beta, bool lower) {
  const int64_t c = blockIdx.y;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nb; r += (int64_t)gridDim.x * blockDim.x) {
    if (lower ? r < c : r > c) continue;
    const double s = W[c * ldw + r];
    double *cp = C + c * ldc + r;
    *cp = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *cp);
  }
}

// One diagonal block of a triangular multiply / solve on nv vectors of
// length nb <= TB.  T(r, c) = op(A)(r, c) (left side) or op(A)(c, r) (right
// side, where the vector is a row of B and y op(A) = (op(A)^T y^T)^T), zero
// outside the `lower` / upper triangle, 1 on the diagonal when unit.
// Vector v of thread t: element r at x + t * xs_v + r * xs_e.
//   multiply, lower: x_r = sum_{c<=r} T(r,c) x_c  (r descending, in place)
//   multiply, upper: x_r = sum_{c>=r} T(r,c) x_c  (r ascending)
//   solve,   lower: x_r = (x_r - sum_{c<r} T(r,c) x_c) / T(r,r)  (forward)
//   solve,   upper: x_r = (x_r - sum_{c>r} T(r,c) x_c) / T(r,r)  (backward)
template <bool SOLVE, bool LOWER>
__global__ void __launch_bounds__(128) tri_diag_kernel(int nb, int64_t nv, const double *__restrict__ A, int64_t lda,
                                                       bool opt, bool unit, double *__restrict__ x, int64_t xs_v,
                                                       int64_t xs_e) {
  __shared__ double T[TB][TB + 1];
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    const int r = e % TB, c = e / TB;
    double v = 0.0;
    if (r < nb && c < nb) {
      if (r == c)
        v = unit ? 1.0 : A[(int64_t)c * lda + r];
      else if (LOWER ? r > c : r < c)
        v = opt ? A[(int64_t)r * lda + c] : A[(int64_t)c * lda + r];
    } else if (r == c) {
      v = 1.0;  // identity padding past nb
    }
    T[r][c] = v;
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nv) return;
  double *xv = x + t * xs_v;
  double v[TB];
#pragma unroll
  for (int r = 0; r < TB; ++r) v[r] = r < nb ? xv[r * xs_e] : 0.0;
  if constexpr (SOLVE) {
    if constexpr (LOWER) {
#pragma unroll
      for (int r = 0; r < TB; ++r) {
        double s = v[r];
#pragma unroll
        for (int c = 0; c < r; ++c) s -= T[r][c] * v[c];
        v[r] = unit ? s : s / T[r][r];
      }
    } else {
#pragma unroll
      for (int r = TB - 1; r >= 0; --r) {
        double s = v[r];
#pragma unroll
        for (int c = r + 1; c < TB; ++c) s -= T[r][c] * v[c];
        v[r] = unit ? s : s / T[r][r];
      }
    }
  } else {
    if constexpr (LOWER) {
#pragma unroll
      for (int r = TB - 1; r >= 0; --r) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c <= r; ++c) s += T[r][c] * v[c];
        v[r] = s;
      }
    } else {
#pragma unroll
      for (int r = 0; r < TB; ++r) {
        double s = 0.0;
#pragma unroll
        for (int c = r; c < TB; ++c) s += T[r][c] * v[c];
        v[r] = s;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < TB; ++r)
    if (r < nb) xv[r * xs_e] = v[r];
}

// T (nb x nb, ld nb) := the dense op(A) diagonal block: the effective
// triangle of op(A)(i0.., i0..), zeros elsewhere, ones on the diagonal when unit.
__global__ void dense_tri_kernel(int nb, const double *__restrict__ A, int64_t lda, bool opt, bool elow, bool unit,
                                 double *__restrict__ T) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)nb * nb;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % nb), c = (int)(e / nb);
    double v = 0.0;
    if (r == c)
      v = unit ? 1.0 : A[(int64_t)c * lda + r];
    else if (elow ? r > c : r < c)
      v = opt ? A[(int64_t)r * lda + c] : A[(int64_t)c * lda + r];
    T[e] = v;
  }
}

// After dense_block's W := T B_i (left) or B_i T (right): every vector of B_i
// holding an Inf or NaN has its W vector recomputed from the triangle only,
// so the zeros dense_tri_kernel wrote outside the triangle never meet a
// non-finite B value (0 * Inf would turn a finite or infinite result into
// NaN; reference BLAS reads the triangle only).  One warp per column (left:
// columns of B_i are the vectors) or one thread per row (right: rows are the
// vectors, read across threads so the scan is coalesced).  For finite B the
// kernel is a read-only scan of B_i.
__global__ void trmm_nonfinite_fix_kernel(bool left, bool elow, int nb, int64_t nv, const double *__restrict__ T,
                                          const double *__restrict__ bi, int64_t ldb, double *__restrict__ W,
                                          int64_t ldw) {
  if (left) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nv;
         j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
      const double *b = bi + j * ldb;
      bool bad = false;
      for (int c = lane; c < nb; c += 32) bad |= !isfinite(b[c]);
      if (!__any_sync(0xffffffffu, bad)) continue;
      for (int r = lane; r < nb; r += 32) {
        double s = 0.0;
        const int c0 = elow ? 0 : r, c1 = elow ? r + 1 : nb;
        for (int c = c0; c < c1; ++c) s += T[(int64_t)c * nb + r] * b[c];
        W[j * ldw + r] = s;
      }
    }
  } else {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nv; r += (int64_t)gridDim.x * blockDim.x) {
      bool bad = false;
      for (int c = 0; c < nb; ++c) bad |= !isfinite(bi[(int64_t)c * ldb + r]);
      if (!bad) continue;
      for (int cc = 0; cc < nb; ++cc) {  // W(r, cc) = sum over the triangle's column cc of B_i(r, c) T(c, cc)
        double s = 0.0;
        const int c0 = elow ? cc : 0, c1 = elow ? nb : cc + 1;
        for (int c = c0; c < c1; ++c) s += bi[(int64_t)c * ldb + r] * T[(int64_t)cc * nb + c];
        W[cc * ldw + r] = s;
      }
    }
  }
}

// dst (rows x cols) := src
__global__ void copy_kernel(int64_t rows, int64_t cols, const double *__restrict__ src, int64_t lds,
                            double *__restrict__ dst, int64_t ldd) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
      dst[j * ldd + i] = src[j * lds + i];
}

// The triangular operation in canonical form: op(A) is effectively lower
// (`elow`) or upper; `opt`: op(A)(r, c) = A(c, r).  B is m x n.
struct Tri {
  bool left, elow, opt, unit, solve;
  const double *A;
  int64_t lda;
  double *B;
  int64_t ldb;
  unsigned flags;
  cudaStream_t st;
  double *T = nullptr, *W = nullptr;  // multiply: dense diagonal block and its product (dense_block)
  // pointer to op(A)(r0.., c0..) and the transa to use for that block in dgemm
  const double *blk(int64_t r0, int64_t c0) const { return opt ? A + r0 * lda + c0 : A + c0 * lda + r0; }
  char ta() const { return opt ? 'T' : 'N'; }
};

int diag(const Tri &t, int64_t i0, int nb, int64_t m, int64_t n) {
  // left: vectors are the n columns of B rows [i0, i0+nb); right: the m rows of B columns [i0, i0+nb)
  const double *a = t.blk(i0, i0);
  double *x = t.left ? t.B + i0 : t.B + i0 * t.ldb;
  const int64_t nv = t.left ? n : m, xs_v = t.left ? t.ldb : 1, xs_e = t.left ? 1 : t.ldb;
  // right side: the vector operation uses op(A)^T, whose triangle is the other one
  const bool low = t.left ? t.elow : !t.elow, opt = t.left ? t.opt : !t.opt;
  const unsigned grid = (unsigned)((nv + 127) / 128);
  if (grid == 0) return capi_ok();
  if (t.solve) {
    if (low) tri_diag_kernel<true, true><<<grid, 128, 0, t.st>>>(nb, nv, a, t.lda, opt, t.unit, x, xs_v, xs_e);
    else tri_diag_kernel<true, false><<<grid, 128, 0, t.st>>>(nb, nv, a, t.lda, opt, t.unit, x, xs_v, xs_e);
  } else {
    if (low) tri_diag_kernel<false, true><<<grid, 128, 0, t.st>>>(nb, nv, a, t.lda, opt, t.unit, x, xs_v, xs_e);
    else tri_diag_kernel<false, false><<<grid, 128, 0, t.st>>>(nb, nv, a, t.lda, opt, t.unit, x, xs_v, xs_e);
  }
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? capi_ok() : capi_cuda_fail(e, "triangular diagonal block");
}

// Update of the range [i0, i0+nb) of B (rows for left, columns for right)
// from its range [p0, p1): left  B_i += s op(A)(i, p) B_p
//                          right B_i += s B_p op(A)(p, i)
int update(const Tri &t, int64_t i0, int nb, int64_t p0, int64_t p1, int64_t m, int64_t n, double s) {
  const int kk = (int)(p1 - p0);
  if (kk <= 0 || nb <= 0) return capi_ok();
  if (t.left)
    return blas_device(t.ta(), 'N', nb, (int)n, kk, s, t.blk(i0, p0), (int)t.lda, t.B + p0, (int)t.ldb, 1.0,
                       t.B + i0, (int)t.ldb, t.flags, t.st, false);
  return blas_device('N', t.ta(), (int)m, nb, kk, s, t.B + p0 * t.ldb, (int)t.ldb, t.blk(p0, i0), (int)t.lda, 1.0,
                     t.B + i0 * t.ldb, (int)t.ldb, t.flags, t.st, false);
}

// Multiply of an outer diagonal block as one dgemm: T := dense op(A)(i, i),
// W := T B_i (left) or B_i T (right) from zero, B_i := W.  Twice the block's
// triangle flops, but one full-width dgemm instead of the 128 / 32 recursion
// (whose small launches dominated: profiles/level3_r01.log).
int dense_block(const Tri &t, int64_t i0, int nb, int64_t m, int64_t n) {
  cudaError_t e;
  const int64_t cnt = (int64_t)nb * nb;
  dense_tri_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 1024), 256, 0, t.st>>>(
      nb, t.blk(i0, i0), t.lda, t.opt, t.elow, t.unit, t.T);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return capi_cuda_fail(e, "dense triangle");
  const int64_t rows = t.left ? nb : m, cols = t.left ? n : nb, ldw = (rows + 1) & ~1LL;
  double *bi = t.left ? t.B + i0 : t.B + i0 * t.ldb;
  int s = t.left ? blas_device('N', 'N', nb, (int)n, nb, 1.0, t.T, nb, bi, (int)t.ldb, 0.0, t.W, (int)ldw, t.flags,
                               t.st, false)
                 : blas_device('N', 'N', (int)m, nb, nb, 1.0, bi, (int)t.ldb, t.T, nb, 0.0, t.W, (int)ldw, t.flags,
                               t.st, false);
  if (s != 0) return s;
  {
    const int64_t nv = t.left ? n : m;
    const int64_t threads = t.left ? nv * 32 : nv;
    trmm_nonfinite_fix_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256, 4096)), 256,
                                0, t.st>>>(t.left, t.elow, nb, nv, t.T, bi, t.ldb, t.W, ldw);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return capi_cuda_fail(e, "trmm non-finite fix");
  }
  copy_kernel<<<dim3((unsigned)std::min<int64_t>((rows + 255) / 256, 64), (unsigned)std::min<int64_t>(cols, 65535)),
                256, 0, t.st>>>(rows, cols, t.W, ldw, bi, t.ldb);
  count_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? capi_ok() : capi_cuda_fail(e, "copy back");
}

// Blocked triangular multiply / solve over [lo_, hi_) of the triangle's
// dimension with block size bs (outer blocks of 512, then 128, then TB
// inside each diagonal block), left-looking: block i is finished from all of
// its dependencies in one long-K dgemm.
//   left,  lower: B_i depends on B_{p<=i}   right, lower: B_j on B_{p>=j}
//   left,  upper: B_i depends on B_{p>=i}   right, upper: B_j on B_{p<=j}
// Multiply visits blocks so that the B_p it reads are still original
// (dependence on p > i: ascending; p < i: descending); solve the opposite.
// Measured against the right-looking order (each solved block pushed into
// all its dependents by one short-K dgemm): left-looking is 1.1-1.2x faster
// at 4096-8192 for every block-size choice (profiles/level3_r01.log).
int tri_range(const Tri &t, int64_t lo_, int64_t hi_, int bs, int64_t m, int64_t n) {
  const bool dep_after = t.left ? !t.elow : t.elow;  // B_i depends on blocks after i
  const bool ascending = t.solve ? !dep_after : dep_after;
  const int64_t nblk = (hi_ - lo_ + bs - 1) / bs;
  for (int64_t q = 0; q < nblk; ++q) {
    const int64_t b = ascending ? q : nblk - 1 - q;
    const int64_t i0 = lo_ + b * bs;
    const int nb = (int)std::min<int64_t>(bs, hi_ - i0);
    const int64_t p0 = dep_after ? i0 + nb : lo_, p1 = dep_after ? hi_ : i0;
    int s;
    if (t.solve) {  // B_i := solve(diag, B_i - sum_p ... X_p)
      if ((s = update(t, i0, nb, p0, p1, m, n, -1.0)) != 0) return s;
      s = bs > TB ? tri_range(t, i0, i0 + nb, inner_bs(bs), m, n) : diag(t, i0, nb, m, n);
      if (s != 0) return s;
    } else {  // B_i := diag B_i + sum_p ... B_p (B_p still original)
      s = t.T && bs >= 256 ? dense_block(t, i0, nb, m, n)
                           : (bs > TB ? tri_range(t, i0, i0 + nb, inner_bs(bs), m, n) : diag(t, i0, nb, m, n));
      if (s != 0) return s;
      if ((s = update(t, i0, nb, p0, p1, m, n, 1.0)) != 0) return s;
    }
  }
  return capi_ok();
}

__global__ void scale_region_kernel(int64_t m, int64_t n, double *__restrict__ B, int64_t ldb, double alpha) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      B[j * ldb + i] = alpha == 0.0 ? 0.0 : alpha * B[j * ldb + i];
}

int scale(int64_t m, int64_t n, double *B, int64_t ldb, double alpha, cudaStream_t st) {
  const int64_t gx = std::min<int64_t>((m + 255) / 256, 64), gy = std::min<int64_t>(n, 65535);
  scale_region_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(m, n, B, ldb, alpha);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? capi_ok() : capi_cuda_fail(e, "scale");
}

int tri(bool solve, char side, char uplo, char transa, char diagc, int m, int n, double alpha, const double *A,
        int lda, double *B, int ldb, unsigned flags, void *stream) {
  char buf[160];
  const bool left = lo(side);
  if (!left && !(side == 'R' || side == 'r')) return capi_fail(-1, "side must be 'L' or 'R'");
  if (!up(uplo) && !lo(uplo)) return capi_fail(-2, "uplo must be 'U' or 'L'");
  if (!nt(transa) && !tr(transa)) return capi_fail(-3, "transa must be 'N', 'T' or 'C'");
  if (!(diagc == 'U' || diagc == 'u' || diagc == 'N' || diagc == 'n')) return capi_fail(-4, "diag must be 'U' or 'N'");
  if (m < 0) return capi_fail(-5, "m must be non-negative");
  if (n < 0) return capi_fail(-6, "n must be non-negative");
  const int na = left ? m : n;
  if (lda < std::max(1, na)) {
    snprintf(buf, sizeof buf, "lda=%d smaller than max(1, %d)", lda, na);
    return capi_fail(-9, buf);
  }
  if (ldb < std::max(1, m)) {
    snprintf(buf, sizeof buf, "ldb=%d smaller than max(1, %d)", ldb, m);
    return capi_fail(-11, buf);
  }
  if (!(flags & MY_DGEMM_DEVICE_PTRS)) return capi_fail(-12, "level-3 routines take device pointers (MY_DGEMM_DEVICE_PTRS)");
  if (flags & ~(MY_DGEMM_DEVICE_PTRS | MY_DGEMM_FORCE_TILED)) return capi_fail(-12, "unsupported flag bits");
  if (m == 0 || n == 0) return capi_ok();
  if (!B) return capi_fail(-10, "B is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (alpha == 0.0) return scale(m, n, B, ldb, 0.0, st);
  if (!A) return capi_fail(-8, "A is NULL");
  keep_pool_memory();
  int s;
  if (alpha != 1.0 && (s = scale(m, n, B, ldb, alpha, st)) != 0) return s;
  Tri t{left, lo(uplo) != tr(transa), tr(transa), diagc == 'U' || diagc == 'u', solve, A, lda, B, ldb,
        flags & MY_DGEMM_FORCE_TILED, st, nullptr, nullptr};
  const int bs0 = na > TB ? std::min(blocks().outer, ((na + TB - 1) / TB) * TB) : TB;
  if (!solve && bs0 >= 256) {  // dense diagonal-block multiply: T and W workspace
    const int64_t rows = left ? bs0 : m, cols = left ? n : bs0;
    cudaError_t e = cudaMallocAsync((void **)&t.T, (size_t)bs0 * bs0 * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void **)&t.W, (size_t)((rows + 1) & ~1LL) * cols * 8, st);
    if (e != cudaSuccess) {
      if (t.T) cudaFreeAsync(t.T, st);
      return capi_cuda_fail(e, "cudaMallocAsync(trmm block)");
    }
  }
  s = tri_range(t, 0, na, bs0, m, n);
  if (t.T) cudaFreeAsync(t.T, st);
  if (t.W) cudaFreeAsync(t.W, st);
  return s;
}

}  // namespace
}  // namespace myd

using namespace myd;

extern "C" int my_dsyrk(char uplo, char trans, int n, int k, double alpha, const double *A, int lda, double beta,
                        double *C, int ldc, unsigned flags, void *stream) {
  char buf[160];
  if (!up(uplo) && !lo(uplo)) return capi_fail(-1, "uplo must be 'U' or 'L'");
  if (!nt(trans) && !tr(trans)) return capi_fail(-2, "trans must be 'N', 'T' or 'C'");
  if (n < 0) return capi_fail(-3, "n must be non-negative");
  if (k < 0) return capi_fail(-4, "k must be non-negative");
  const int nrowa = tr(trans) ? k : n;
  if (lda < std::max(1, nrowa)) {
    snprintf(buf, sizeof buf, "lda=%d smaller than max(1, %d)", lda, nrowa);
    return capi_fail(-7, buf);
  }
  if (ldc < std::max(1, n)) {
    snprintf(buf, sizeof buf, "ldc=%d smaller than max(1, %d)", ldc, n);
    return capi_fail(-10, buf);
  }
  if (!(flags & MY_DGEMM_DEVICE_PTRS)) return capi_fail(-11, "level-3 routines take device pointers (MY_DGEMM_DEVICE_PTRS)");
  if (flags & ~(MY_DGEMM_DEVICE_PTRS | MY_DGEMM_FORCE_TILED)) return capi_fail(-11, "unsupported flag bits");
  if (n == 0 || ((alpha == 0.0 || k == 0) && beta == 1.0)) return capi_ok();
  if (!C) return capi_fail(-9, "C is NULL");
  if (alpha != 0.0 && k > 0 && !A) return capi_fail(-6, "A is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned gf = flags & MY_DGEMM_FORCE_TILED;
  const bool lower = lo(uplo), at = tr(trans);
  // rows r0.. of op(A) as a dgemm operand, and the transa that reads them
  auto rows = [&](int64_t r0) { return at ? A + r0 * lda : A + r0; };
  const char ta = at ? 'T' : 'N', tb = at ? 'N' : 'T';
  double *W = nullptr;
  cudaError_t e;
  keep_pool_memory();
  const int wb = std::min(n, OB);
  if ((e = cudaMallocAsync((void **)&W, (size_t)wb * wb * 8, st)) != cudaSuccess)
    return capi_cuda_fail(e, "cudaMallocAsync(syrk block)");
  int s = 0;
  for (int64_t j0 = 0; j0 < n && s == 0; j0 += OB) {
    const int nb = (int)std::min<int64_t>(OB, n - j0);
    // off-diagonal panel of this column block: rows below (lower) or above (upper)
    const int64_t r0 = lower ? j0 + nb : 0, r1 = lower ? n : j0;
    if (r1 > r0)
      s = blas_device(ta, tb, (int)(r1 - r0), nb, k, alpha, rows(r0), lda, rows(j0), lda, beta, C + j0 * ldc + r0,
                      ldc, gf, st, true);  // one large panel: the BLAS order pays
    if (s != 0) break;
    // diagonal block: W = op(A)_j op(A)_j^T from zero, merged into the triangle
    if (alpha == 0.0 || k == 0) {
      if ((e = cudaMemsetAsync(W, 0, (size_t)nb * nb * 8, st)) != cudaSuccess) {
        s = capi_cuda_fail(e, "memset");
        break;
      }
    } else if ((s = blas_device(ta, tb, nb, nb, k, 1.0, rows(j0), lda, rows(j0), lda, 0.0, W, nb, gf, st, false)) != 0) {
      break;
    }
    syrk_merge_kernel<<<dim3((unsigned)((nb + 255) / 256), (unsigned)nb), 256, 0, st>>>(
        nb, W, nb, C + j0 * ldc + j0, ldc, alpha, beta, lower);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) s = capi_cuda_fail(e, "syrk merge");
  }
  cudaFreeAsync(W, st);
  return s == 0 ? capi_ok() : s;
}

extern "C" int my_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha, const double *A,
                        int lda, double *B, int ldb, unsigned flags, void *stream) {
  return tri(false, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, flags, stream);
}

extern "C" int my_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha, const double *A,
                        int lda, double *B, int ldb, unsigned flags, void *stream) {
  return tri(true, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, flags, stream);
}
