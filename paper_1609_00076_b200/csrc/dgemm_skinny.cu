// dgemm_skinny.cu -- the HBM-bound shapes of the my_dgemm path (sm_100a):
//   * n == 1 (cfg 3c): C(:,0) += A * B(:,0)          bytes 8(mk + k + 2m)
//   * m == 1 (cfg 3b): C(0,:) += A(0,:) * B          bytes 8(k + kn + 2n)
// Both stream one operand exactly once at full width, accumulate with FMA,
// and reduce in a fixed order (no atomics, no workspace), so results are
// deterministic and independent of the grid.  The reference computes these
// shapes with the same five-loop code as every other shape
// (goto.py:187-239); on the GPU they are bandwidth problems, not DMMA ones.
#include <algorithm>
#include <atomic>

#include "common.cuh"

#ifndef MYD_N1_WARPS
#define MYD_N1_WARPS 32
#endif
#ifndef MYD_N1_UNROLL
#define MYD_N1_UNROLL 8
#endif
#ifndef MYD_M1_TEAM
#define MYD_M1_TEAM 4
#endif
#ifndef MYD_M1_UNROLL
#define MYD_M1_UNROLL 8
#endif

namespace myd {

// ---------------------------------------------------------------------------
// n == 1.  A CTA owns 32 rows (one per lane); its WARPS warps take contiguous
// k-slices, so each warp load is one coalesced 256-byte column segment of A.
// Slice partials meet in shared memory and are added in warp order.
// ---------------------------------------------------------------------------
template <int WARPS, int UNROLL>
__global__ void __launch_bounds__(32 * WARPS)
    gemv_n1_kernel(int M, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ b,
                   double *__restrict__ C, Epilogue ep) {
  __shared__ double part[WARPS][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x * 32 + lane;
  const int per = (K + WARPS - 1) / WARPS;
  const int p0 = warp * per, p1 = min(K, p0 + per);
  double acc = 0.0;
  if (row < M) {
    const double *a = A + row;
    int p = p0;
    for (; p + UNROLL <= p1; p += UNROLL) {
      double av[UNROLL], bv[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        av[u] = __ldcs(a + (int64_t)(p + u) * lda);
        bv[u] = __ldg(b + p + u);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc = fma(av[u], bv[u], acc);
    }
    for (; p < p1; ++p) acc = fma(__ldcs(a + (int64_t)p * lda), __ldg(b + p), acc);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && row < M) {
    if (!ep.blas) {
      double s = C[row];
#pragma unroll
      for (int w = 0; w < WARPS; ++w) s += part[w][lane];
      C[row] = s;
    } else {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) s += part[w][lane];
      C[row] = ep.beta == 0.0 ? ep.alpha * s : fma(ep.alpha, s, ep.beta * C[row]);
    }
  }
}

// ---------------------------------------------------------------------------
// m == 1.  Teams of TEAM warps own columns (round-robin over all teams of the
// grid); warp t of a team reduces k-quarter t of the column with lane-strided
// coalesced loads, then the team combines its TEAM partials in order behind
// a named barrier.  The A row (stride lda) is staged once per CTA in shared
// memory when it fits, else read through L1.
// ---------------------------------------------------------------------------
constexpr int M1_TEAMS = 8;  // teams per CTA (8 x TEAM warps)

template <int TEAM, int UNROLL, bool STAGED>
__global__ void __launch_bounds__(32 * TEAM * M1_TEAMS, 1)
    gemv_m1_kernel(int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B, int64_t ldb,
                   double *__restrict__ C, int64_t ldc, Epilogue ep) {
  extern __shared__ double arow[];  // K doubles when STAGED
  __shared__ double part[2][M1_TEAMS][TEAM];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int team = warp / TEAM, t = warp % TEAM;
  if (STAGED) {
    for (int p = threadIdx.x; p < K; p += blockDim.x) arow[p] = A[(int64_t)p * lda];
    __syncthreads();
  }
  const int per = (K + TEAM - 1) / TEAM;
  const int p0 = t * per, p1 = min(K, p0 + per);
  const int64_t teams_total = (int64_t)gridDim.x * M1_TEAMS;
  int buf = 0;
  for (int64_t j = (int64_t)blockIdx.x * M1_TEAMS + team; j < N; j += teams_total, buf ^= 1) {
    const double *bc = B + j * ldb;
    double acc = 0.0;
    int p = p0 + lane;
    for (; p + 32 * (UNROLL - 1) < p1; p += 32 * UNROLL) {
      double bv[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) bv[u] = __ldcs(bc + p + 32 * u);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const double av = STAGED ? arow[p + 32 * u] : __ldg(A + (int64_t)(p + 32 * u) * lda);
        acc = fma(av, bv[u], acc);
      }
    }
    for (; p < p1; p += 32) acc = fma(STAGED ? arow[p] : __ldg(A + (int64_t)p * lda), __ldcs(bc + p), acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) part[buf][team][t] = acc;
    // team barrier (ids 1..M1_TEAMS; 0 is __syncthreads)
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(32 * TEAM) : "memory");
    if (t == 0 && lane == 0) {
      double s = ep.blas ? 0.0 : C[j * ldc];
#pragma unroll
      for (int w = 0; w < TEAM; ++w) s += part[buf][team][w];
      if (ep.blas) s = ep.beta == 0.0 ? ep.alpha * s : fma(ep.alpha, s, ep.beta * C[j * ldc]);
      C[j * ldc] = s;
    }
  }
}

namespace {
int sm_count_skinny() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}
}  // namespace

cudaError_t launch_gemv_n1(int M, int K, const double *A, int64_t lda, const double *b, double *C,
                           cudaStream_t stream, const Epilogue &ep) {
  gemv_n1_kernel<MYD_N1_WARPS, MYD_N1_UNROLL><<<(M + 31) / 32, 32 * MYD_N1_WARPS, 0, stream>>>(M, K, A, lda, b, C, ep);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_gemv_m1(int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                           int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  constexpr int TEAM = MYD_M1_TEAM;
  const int threads = 32 * TEAM * M1_TEAMS;
  const int64_t want = (N + M1_TEAMS - 1) / M1_TEAMS;
  const unsigned grid = (unsigned)std::min<int64_t>(want, sm_count_skinny());
  const size_t smem = (size_t)K * 8;
  if (smem <= 160 * 1024) {
    // per-device function attribute, set once per device (a race only repeats it)
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(gemv_m1_kernel<TEAM, MYD_M1_UNROLL, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      if (e != cudaSuccess) return e;
      attr_done.fetch_or(bit, std::memory_order_release);
    }
    gemv_m1_kernel<TEAM, MYD_M1_UNROLL, true><<<grid, threads, smem, stream>>>(N, K, A, lda, B, ldb, C, ldc, ep);
  } else {
    gemv_m1_kernel<TEAM, MYD_M1_UNROLL, false><<<grid, threads, 0, stream>>>(N, K, A, lda, B, ldb, C, ldc, ep);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace myd
