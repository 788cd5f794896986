// dgemm_small.cu -- the tiled path's kernel for problems below one wave of the
// persistent kernel's units (sm_100a): C := A*B + C, FP64, column-major, any ld.
//
// The persistent kernel (dgemm_fast.cu) keeps one 384-thread CTA per SM and
// cuts a small problem into 64x32 units at the finest, so 256^3 runs on 32
// SMs, each doing a 64x32x256 DMMA chain (profiles/timeline_r01.log: 5 us of
// an 8.7 us call in the K loop).  Here a CTA owns a 16x16 .. 64x32 block of C
// and 4 warps, several CTAs share an SM, and the grid is the block count, so
// every SM sub-partition runs a couple of short accumulator chains at once:
// the same loop nest as the reference's goto_block over one ic/jc block
// (pkg/src/gemmforge/goto.py:215-229, _ckernels.pyx:142-195), with the jr/ir
// micro-panels as 8x8 DMMA fragments.
//
// Per-element arithmetic is the persistent kernel's exactly: DMMA.8x8x4 on the
// C^T block (a = B^T fragment, b = A^T fragment, same lane layout), k grouped
// in fours from p = 0, one DMMA per group holding at least one k < K (the
// zero-filled tail of the last group included, all-zero groups skipped),
// groups in ascending order, the accumulator starting at C.  So this kernel
// is one more launch plan of the tiled path: C is bitwise the same as every
// other plan's (tests/test_gpu_parity.py::test_small_kernel_bitwise_equals_units),
// and the multi-GPU shards stay bitwise independent of the shard count.
//
// Staging: a STAGES-deep cp.async (LDGSTS) ring of BK-deep slabs, A slab
// [BK][BM+4] (m contiguous) and B slab [BN][BK+4] (k contiguous), the pitches
// 4 mod 16 doubles as in the persistent kernel so every fragment load is
// bank-conflict free; 16-byte copies when lda/ldb are even and the bases
// 16-byte aligned, 8-byte copies otherwise; zero fill outside A and B.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace myd {

namespace small {
constexpr int WARPS = 4;  // one per SM sub-partition when a CTA has the SM alone
constexpr int THREADS = WARPS * 32;

template <int BM, int BN, int BK, int STAGES>
struct Geo {
  static constexpr int AP = BM + 4, BP = BK + 4;
  static constexpr int A_ST = BK * AP, B_ST = BN * BP, SLOT = A_ST + B_ST;
  static constexpr int BYTES = STAGES * SLOT * 8;
  static_assert(AP % 16 == 4 && BP % 16 == 4, "pitches must be 4 mod 16 doubles (conflict-free fragments)");
};
}  // namespace small

// BM x BN block per CTA, warps 2 x 2 over it (WM = BM / 2, WN = BN / 2 rows /
// columns per warp: FM x FN 8x8 accumulator fragments).  Grid: one CTA per
// block, m fastest (neighbouring CTAs share B columns in L2).
template <int BM, int BN, int BK, int STAGES, int VEC>
__global__ void __launch_bounds__(small::THREADS)
    dgemm_small_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                       int64_t ldb, double *__restrict__ C, int64_t ldc, int tiles_m, Epilogue ep) {
  using namespace small;
  using G = Geo<BM, BN, BK, STAGES>;
  constexpr int AP = G::AP, BP = G::BP, A_ST = G::A_ST, SLOT = G::SLOT;
  constexpr int WM = BM / 2, WN = BN / 2, FM = WM / 8, FN = WN / 8;
  constexpr int KSTEPS = BK / 4;
  static_assert(FM >= 1 && FN >= 1 && BK % 4 == 0, "tile shape");
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = (int)(blockIdx.x % (unsigned)tiles_m) * BM, n0 = (int)(blockIdx.x / (unsigned)tiles_m) * BN;
  const int KT = (K + BK - 1) / BK;

  // Programmatic dependent launch: wait for the previous grid before the
  // first global access; let the next one start its prologue now.
  asm volatile("griddepcontrol.wait;\n" "griddepcontrol.launch_dependents;\n" ::: "memory");

  auto load_slab = [&](int slot, int kt) {
    double *as = smem + slot * SLOT;
    double *bs = as + A_ST;
    const int kbase = kt * BK;
    constexpr int A_CH = BK * BM / VEC, B_CH = BN * BK / VEC;
#pragma unroll
    for (int c = 0; c < (A_CH + THREADS - 1) / THREADS; ++c) {
      const int e = c * THREADS + tid;
      if (A_CH % THREADS == 0 || e < A_CH) {
        const int kk = e / (BM / VEC), mm = (e % (BM / VEC)) * VEC;
        const int gk = kbase + kk, gm = m0 + mm;
        int bytes = 0;
        const double *src = A;
        if (gk < K && gm < M) {
          bytes = min(VEC, M - gm) * 8;
          src = A + (int64_t)gk * lda + gm;
        }
        cp_async<VEC * 8>(as + kk * AP + mm, src, bytes);
      }
    }
#pragma unroll
    for (int c = 0; c < (B_CH + THREADS - 1) / THREADS; ++c) {
      const int e = c * THREADS + tid;
      if (B_CH % THREADS == 0 || e < B_CH) {
        const int nn = e / (BK / VEC), kk = (e % (BK / VEC)) * VEC;
        const int gk = kbase + kk, gn = n0 + nn;
        int bytes = 0;
        const double *src = B;
        if (gn < N && gk < K) {
          bytes = min(VEC, K - gk) * 8;
          src = B + (int64_t)gn * ldb + gk;
        }
        cp_async<VEC * 8>(bs + nn * BP + kk, src, bytes);
      }
    }
  };

  // Full slabs of an interior block (no bounds, whole 16 / 8-byte chunks):
  // each thread's chunks sit at fixed offsets that advance by a constant
  // per pass, so a slab costs a few instructions per cp.async instead of the
  // bounds arithmetic above -- with one warp per sub-partition those
  // instructions sit between the DMMAs of the K chain.
  constexpr int A_CPR = BM / VEC, B_CPC = BK / VEC;  // chunks per A k-row / per B column
  static_assert(THREADS % A_CPR == 0 && (THREADS % B_CPC == 0 || B_CPC % THREADS == 0), "chunk passes");
  constexpr int A_ROWS_PP = THREADS / A_CPR, A_PASSES = BK / A_ROWS_PP;
  constexpr int B_COLS_PP = THREADS >= B_CPC ? THREADS / B_CPC : 1, B_PASSES = BK * BN / VEC / THREADS;
  const bool interior = m0 + BM <= M && n0 + BN <= N;
  const int a_kk0 = tid / A_CPR, a_mm0 = (tid % A_CPR) * VEC;
  const int b_nn0 = tid / B_CPC, b_kk0 = (tid % B_CPC) * VEC;
  const double *const a_base = A + (int64_t)a_kk0 * lda + m0 + a_mm0;
  const double *const b_base = B + (int64_t)(n0 + b_nn0) * ldb + b_kk0;
  auto load_slab_fast = [&](int slot, int kt) {
    double *as = smem + slot * SLOT + a_kk0 * AP + a_mm0;
    double *bs = smem + slot * SLOT + A_ST + b_nn0 * BP + b_kk0;
    const double *pa = a_base + (int64_t)kt * BK * lda;
    const double *pb = b_base + kt * BK;
#pragma unroll
    for (int c = 0; c < A_PASSES; ++c) cp_async<VEC * 8>(as + c * A_ROWS_PP * AP, pa + (int64_t)c * A_ROWS_PP * lda, VEC * 8);
#pragma unroll
    for (int c = 0; c < B_PASSES; ++c) {
      if constexpr (THREADS >= B_CPC) {
        cp_async<VEC * 8>(bs + c * B_COLS_PP * BP, pb + (int64_t)c * B_COLS_PP * ldb, VEC * 8);
      } else {  // a column takes several passes
        constexpr int PPC = B_CPC / THREADS;  // passes per column
        cp_async<VEC * 8>(bs + (c / PPC) * BP + (c % PPC) * THREADS * VEC,
                          pb + (int64_t)(c / PPC) * ldb + (c % PPC) * THREADS * VEC, VEC * 8);
      }
    }
  };
  auto issue_slab = [&](int slot, int kt) {
    if (interior && (kt + 1) * BK <= K) load_slab_fast(slot, kt);
    else load_slab(slot, kt);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) issue_slab(s, s);
    cp_async_commit();
  }

  // accumulators start at C (_mk's tile load); BLAS epilogue: at 0
  const int wm = warp & 1, wn = warp >> 1;
  const int r = lane >> 2, q = lane & 3;
  const int row0 = m0 + wm * WM + 2 * q, col0 = n0 + wn * WN + r;
  const bool c_aligned = (ldc % 2 == 0) && ((uintptr_t)C % 16 == 0);
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int row = row0 + i * 8, col = col0 + j * 8;
      double v0 = 0.0, v1 = 0.0;
      if (!ep.blas && col < N && row < M) {
        const double *cp = C + (int64_t)col * ldc + row;
        if (c_aligned && row + 1 < M) {
          const double2 v = __ldcg(reinterpret_cast<const double2 *>(cp));
          v0 = v.x;
          v1 = v.y;
        } else {
          v0 = __ldcg(cp);
          if (row + 1 < M) v1 = __ldcg(cp + 1);
        }
      }
      acc[i][j][0] = v0;
      acc[i][j][1] = v1;
    }

  const int a_off = q * AP + wm * WM + r;    // + kk*4*AP + i*8
  const int b_off = (wn * WN + r) * BP + q;  // + j*8*BP + kk*4
  auto kstep = [&](const double *as, const double *bs, int kk) {
    double fa[FM], fb[FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[i] = as[a_off + kk * 4 * AP + i * 8];
#pragma unroll
    for (int j = 0; j < FN; ++j) fb[j] = bs[b_off + kk * 4 + j * 8 * BP];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], fb[j], fa[i]);
  };

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // slab kt landed for every thread; slot (kt - 1) % STAGES free
    const int nk = kt + STAGES - 1;
    const double *as = smem + (kt % STAGES) * SLOT;
    const double *bs = as + A_ST;
    if (kt + 1 < KT || K % BK == 0) {
      // the next slab's copies go out after the first k-step, so the chain
      // restarts at once after the barrier
      kstep(as, bs, 0);
      if (nk < KT) issue_slab(nk % STAGES, nk);
      cp_async_commit();
#pragma unroll
      for (int kk = 1; kk < KSTEPS; ++kk) kstep(as, bs, kk);
    } else {
      if (nk < KT) issue_slab(nk % STAGES, nk);
      cp_async_commit();
      // last slab of a ragged K: only the k-groups holding some k < K
      const int nsteps = (K - kt * BK + 3) / 4;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        if (kk >= nsteps) break;
        kstep(as, bs, kk);
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: valid region only (padding rows never touched)
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int row = row0 + i * 8, col = col0 + j * 8;
      if (col >= N || row >= M) continue;
      double *cp = C + (int64_t)col * ldc + row;
      double v0 = acc[i][j][0], v1 = acc[i][j][1];
      const bool pair = row + 1 < M;
      if (ep.blas) {  // alpha * (A B) + beta * C, C not read when beta == 0 (dgemm_fast_kernel's arithmetic)
        if (ep.beta == 0.0) {
          v0 *= ep.alpha;
          v1 *= ep.alpha;
        } else {
          v0 = fma(ep.alpha, v0, ep.beta * cp[0]);
          if (pair) v1 = fma(ep.alpha, v1, ep.beta * cp[1]);
        }
      }
      if (pair && c_aligned) {
        *reinterpret_cast<double2 *>(cp) = make_double2(v0, v1);
      } else {
        cp[0] = v0;
        if (pair) cp[1] = v1;
      }
    }
}

namespace {

bool small_pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("MY_DGEMM_NO_PDL");
    return !(v && *v && *v != '0');
  }();
  return on;
}

template <int BM, int BN, int BK, int STAGES, int VEC>
cudaError_t launch_small_t(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                           int64_t ldc, cudaStream_t st, const Epilogue &ep) {
  using G = small::Geo<BM, BN, BK, STAGES>;
  auto kern = dgemm_small_kernel<BM, BN, BK, STAGES, VEC>;
  if constexpr (G::BYTES > 48 * 1024) {
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::BYTES);
      if (e != cudaSuccess) return e;
      attr_done.fetch_or(bit, std::memory_order_release);
    }
  }
  const long long tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  if (tiles_m * tiles_n > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles_m * tiles_n));
  cfg.blockDim = dim3(small::THREADS);
  cfg.dynamicSmemBytes = G::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = small_pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, M, N, K, A, lda, B, ldb, C, ldc, (int)tiles_m, ep);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// The variant table: block shape, slab depth, ring depth (the tuner's grid,
// my_dgemm_tune plans 64 + v; the planner costs every entry).
#define MYD_SMALL_VARIANTS(X) \
  X(1, 16, 16, 32, 4)         \
  X(2, 32, 16, 32, 4)         \
  X(3, 32, 32, 32, 4)         \
  X(4, 64, 32, 32, 4)         \
  X(5, 64, 64, 16, 6)         \
  X(6, 16, 16, 64, 6)         \
  X(7, 32, 16, 64, 6)         \
  X(8, 32, 32, 64, 4)         \
  X(9, 16, 16, 128, 4)        \
  X(10, 64, 64, 32, 3)

template <int VEC>
cudaError_t launch_small_v(int variant, int M, int N, int K, const double *A, int64_t lda, const double *B,
                           int64_t ldb, double *C, int64_t ldc, cudaStream_t st, const Epilogue &ep) {
  switch (variant) {
#define MYD_SMALL_CASE(v, bm, bn, bk, stages) \
  case v: return launch_small_t<bm, bn, bk, stages, VEC>(M, N, K, A, lda, B, ldb, C, ldc, st, ep);
    MYD_SMALL_VARIANTS(MYD_SMALL_CASE)
#undef MYD_SMALL_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

struct SmallGeo {  // also declared in dgemm_fast.cu
  int bm = 0, bn = 0, bk = 0, stages = 0;
};
// Geometry of small-kernel variant v (bm == 0: no such variant).
SmallGeo small_geo(int v) {
  switch (v) {
#define MYD_SMALL_GEO(v_, bm, bn, bk, stages) \
  case v_: return SmallGeo{bm, bn, bk, stages};
    MYD_SMALL_VARIANTS(MYD_SMALL_GEO)
#undef MYD_SMALL_GEO
    default: return SmallGeo{};
  }
}
int small_variants() { return 10; }

// Estimated device time (us) of variant v on G SMs, a resource model fitted
// (log least squares over tools/small_kernel_probe.py timings,
// profiles/r02/small_kernel_r02b.log) on 18 shapes x 10 variants:
//  * a resident CTA's k-step (4 k) costs the SM max(DMMA issue: 4 warps x
//    FM x FN DMMAs at 4 cycles; shared memory: fragment loads 4 x (FM + FN)
//    x 256 B plus the slab fill (BM + BN) x 32 B at 128 B/cycle) x 1.51;
//  * one warp's k-step is never shorter than its dependent chain: 75 / 67 /
//    50 cycles of DMMA latency, fragment loads and the per-slab handshake
//    for 32 / 64 / 128-deep slabs, plus its own FM x FN DMMA issue;
//  * CTAs beyond the resident count (shared memory) run in further rounds;
//  * the operands' L2 -> SM traffic is capped at 5142 B/cycle chip-wide;
//  * plus 1.78 us of launch and first-slab latency.
double small_cost_us(int v, int M, int N, int K, int G) {
  const SmallGeo g = small_geo(v);
  if (g.bm == 0) return 1e300;
  const double ctas = (double)((M + g.bm - 1) / g.bm) * ((N + g.bn - 1) / g.bn);
  const double ksteps = (double)((K + 3) / 4);
  const double fm = g.bm / 16, fn = g.bn / 16;
  const double bytes = (double)g.stages * ((double)g.bk * (g.bm + 4) + (double)g.bn * (g.bk + 4)) * 8.0;
  const double occ = std::max(1.0, std::min(16.0, std::floor(232448.0 / bytes)));
  const double per_sm = std::ceil(ctas / G);
  const double res = std::min(per_sm, occ), rounds = std::ceil(per_sm / occ);
  const double ck = std::max(16.0 * fm * fn, 8.0 * (fm + fn) + (g.bm + g.bn) / 4.0) * 1.51;
  const double chain = (g.bk >= 128 ? 50.2 : (g.bk >= 64 ? 67.2 : 74.6)) + 16.0 * fm * fn;
  const double t_sm = rounds * ksteps * std::max(res * ck, chain);
  const double t_l2 = ctas * ksteps * (g.bm + g.bn) * 32.0 / 5142.0;
  return 1.78 + std::max(t_sm, t_l2) / 1965.0;
}

cudaError_t launch_dgemm_small(int variant, int M, int N, int K, const double *A, int64_t lda, const double *B,
                               int64_t ldb, double *C, int64_t ldc, cudaStream_t st, const Epilogue &ep, bool vec2) {
  return vec2 ? launch_small_v<2>(variant, M, N, K, A, lda, B, ldb, C, ldc, st, ep)
              : launch_small_v<1>(variant, M, N, K, A, lda, B, ldb, C, ldc, st, ep);
}

}  // namespace myd
