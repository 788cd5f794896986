// dgemm_fast.cu -- the hot path: C := A*B + C, FP64, column-major, any ld, on sm_100a.
//
// The reference's five BLIS loops (pkg/src/gemmforge/goto.py:187-239 and
// _ckernels.pyx:15-45,142-195) re-derived for Blackwell:
//   loop 5/3 (jc, ic)  -> the CTA grid over 128x128 tiles of C, rastered in
//                         bands of GROUP_M tile-rows so co-resident CTAs share
//                         A and B panels in the 126 MB L2;
//   loop 4 (pc)        -> the in-CTA K loop over BK=16 slabs;
//   pack_a / pack_b    -> cp.async (LDGSTS) staging of the A and B slabs into a
//                         STAGES-deep shared-memory ring; zero-fill of the
//                         out-of-range lanes replaces the zero-padded panels;
//                         no separate pack pass touches HBM;
//   loops 2/1 + _mk    -> 8 warps, each a 64x32 register tile of C built from
//                         8x4 DMMA.8x8x4 fragments (mma.sync f64).  FP64 has
//                         no tcgen05 kind on sm_100a; the DMMA pipe measured
//                         37.1 TFLOP/s (128 flop/clk/SM) vs 34.0 for DFMA
//                         (tools/microbench/fp64_peak.cu, profiles/).
// C is loaded into the accumulators first, like _mk's tile load
// (_ckernels.pyx:28-32), and only the valid region is stored back.
#include <type_traits>

#include "common.cuh"

namespace myd {

#ifdef MYD_FAST_PROFILE
// [0] consumer slow-wait cycles, [1] consumer slow waits, [2] producer empty-wait cycles,
// [3] producer waits, [4] consumer first-slab wait cycles, [5] consumer total loop cycles,
// [6] producer issue cycles
__device__ unsigned long long g_fast_prof[8];
#define PROF_T0() long long _pt0 = clock64()
#define PROF_ADD(i, v) atomicAdd(&g_fast_prof[i], (unsigned long long)(v))
#else
#define PROF_T0()
#define PROF_ADD(i, v)
#endif

namespace fast {
constexpr int BM = 128;          // CTA tile rows (m)
constexpr int BN = 128;          // CTA tile cols (n)
#ifndef MYD_FAST_BK
#define MYD_FAST_BK 16
#endif
#ifndef MYD_FAST_STAGES
#define MYD_FAST_STAGES 5
#endif
#ifndef MYD_FAST_GROUP_M
#define MYD_FAST_GROUP_M 8
#endif
constexpr int BK = MYD_FAST_BK;          // K slab per pipeline stage
constexpr int STAGES = MYD_FAST_STAGES;  // cp.async ring depth
constexpr int CONSUMER_WARPS = 8;  // 2 (m) x 4 (n) DMMA warps: 2 per SM sub-partition
constexpr int PRODUCER_WARPS = 4;  // one staging warp per sub-partition
constexpr int THREADS = (CONSUMER_WARPS + PRODUCER_WARPS) * 32;
// Register split per sub-partition (16K regs): 1 producer + 2 consumers.
// Launch at 168 (12 warps x 168 x 32 <= 64K), then setmaxnreg moves
// producers down to 40 and consumers up to 232: the CTA keeps the 168 x 384
// registers it launched with (40*128 + 232*256 = 168*384); asking for more
// would block setmaxnreg.inc forever.
constexpr int PRODUCER_REGS = 40;
constexpr int CONSUMER_REGS = 232;
constexpr int WM = 64, WN = 32;  // warp tile
constexpr int FM = WM / 8, FN = WN / 8;
// Padded pitches make every fragment load and every 16-byte staging store
// conflict-free: a half-warp's 4 k-rows of A (4 n-rows of B) land in 4
// distinct 32-byte bank groups (pitch = 4 mod 16 doubles).
constexpr int AP = BM + 4;  // A slab: [BK][AP]   (m contiguous, as in HBM)
constexpr int BP = BK + 4;  // B slab: [BN][BP]   (k contiguous, as in HBM)
constexpr int A_STAGE = BK * AP;
constexpr int B_STAGE = BN * BP;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
constexpr int GROUP_M = MYD_FAST_GROUP_M;
constexpr int KSTEPS = BK / 4;                  // DMMA k-steps per slab
constexpr int PROBE_STEP = KSTEPS > 2 ? 1 : 0;  // where the next slab's barrier is probed
constexpr int PROBE_STEP_ALT = KSTEPS - 1;      // ... by the second warp of each sub-partition
#ifndef MYD_FAST_STAGGER
#define MYD_FAST_STAGGER 0
#endif
constexpr bool STAGGER = MYD_FAST_STAGGER != 0;
}  // namespace fast

// VEC doubles per cp.async (2: 16-byte copies, needs even ld and 16-B aligned
// bases; 1: 8-byte copies for odd leading dimensions / 8-B aligned views).
//
// Warp roles: warps 0..7 are consumers (DMMA micro-tiles, 2 per SM
// sub-partition); warp 8 is the producer that stages every K slab with
// cp.async and signals slab arrival on full[s] (cp.async.mbarrier.arrive).
// Consumers release a slab on empty[s] when their fragments are in
// registers.  No CTA-wide barrier in the main loop: each consumer warp runs
// at its own pace, bounded only by the STAGES-deep ring.
template <int VEC>
__global__ void __launch_bounds__(fast::THREADS, 1)
    dgemm_fast_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                      int64_t ldb, double *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n) {
  using namespace fast;
  extern __shared__ __align__(128) double smem[];
  double *As = smem;
  double *Bs = smem + STAGES * A_STAGE;
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];

  // Grouped raster: GROUP_M tile-rows per band, column-major inside a band.
  const int bid = blockIdx.x;
  const int band = GROUP_M * tiles_n;
  const int first_m = (bid / band) * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (bid % band) % gm;
  const int tn = (bid % band) / gm;
  const int m0 = tm * BM, n0 = tn * BN;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int KT = (K + BK - 1) / BK;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], PRODUCER_WARPS);       // one arrival per producer warp
      mbar_init(&empty_bar[s], CONSUMER_WARPS);      // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= CONSUMER_WARPS) {
    // ================= producers: pack_a / pack_b equivalent =================
    // One producer warp per SM sub-partition; registers handed to consumers.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int pw = warp - CONSUMER_WARPS;
    // Interior tiles with 16-byte aligned operands use the bulk-copy (TMA)
    // engine: one cp.async.bulk per A k-row (BM*8 bytes) and per B column
    // segment (BK*8 bytes), straight into the padded slab layout, no LSU
    // traffic.  Edge tiles and a ragged last slab use zero-filling LDGSTS.
    const bool interior = (VEC == 2) && (m0 + BM <= M) && (n0 + BN <= N);
    for (int kt = 0; kt < KT; ++kt) {
      const int slot = kt % STAGES;
      if (kt >= STAGES) {
        PROF_T0();
        mbar_wait(&empty_bar[slot], ((kt / STAGES) - 1) & 1);
        if (lane == 0) { PROF_ADD(2, clock64() - _pt0); PROF_ADD(3, 1); }
      }
      const int kbase = kt * BK;
      double *as = As + slot * A_STAGE;
      double *bs = Bs + slot * B_STAGE;
      if (interior && kbase + BK <= K) {
        constexpr int A_ROWS = BK / PRODUCER_WARPS;  // k-rows of A per producer warp
        constexpr uint32_t BYTES = (A_ROWS * BM + 32 * BK) * 8;
        if (lane == 0) mbar_arrive_expect_tx(&full_bar[slot], BYTES);
        __syncwarp();
        if (lane < A_ROWS) {
          const int kk = pw * A_ROWS + lane;
          bulk_g2s(as + kk * AP, A + (int64_t)(kbase + kk) * lda + m0, BM * 8, &full_bar[slot]);
        }
        const int nn = pw * 32 + lane;
        bulk_g2s(bs + nn * BP, B + (int64_t)(n0 + nn) * ldb + kbase, BK * 8, &full_bar[slot]);
        continue;
      }
      // A slab [BK][BM], m contiguous: a warp instruction covers 32*VEC
      // consecutive m of one k-row (coalesced, conflict-free at pitch AP).
#pragma unroll
      for (int i = 0; i < BK * BM / (VEC * 32 * PRODUCER_WARPS); ++i) {
        const int e = ((pw * 32 + lane) + i * 32 * PRODUCER_WARPS) * VEC;
        const int kk = e / BM, mm = e % BM;
        const int gk = kbase + kk, gmr = m0 + mm;
        int bytes = 0;
        const double *src = A;
        if (gk < K && gmr < M) {
          bytes = min(VEC, M - gmr) * 8;
          src = A + (int64_t)gk * lda + gmr;
        }
        cp_async<VEC * 8>(as + kk * AP + mm, src, bytes);
      }
      // B slab [BN][BK], k contiguous: producer pw owns n-rows [32pw, 32pw+32);
      // a quarter-warp writes 4 rows x 2 chunks (conflict-free at pitch BP).
#pragma unroll
      for (int i = 0; i < BK * 32 / (VEC * 32); ++i) {
        int nn, kk;
        if constexpr (VEC == 2) {  // 16 rows x 2 chunks per instruction
          nn = pw * 32 + (lane >> 1) + 16 * (i / (BK / 4));
          kk = 2 * ((lane & 1) + 2 * (i % (BK / 4)));
        } else {  // 8 rows x 4 doubles per instruction
          nn = pw * 32 + (lane >> 2) + 8 * (i / (BK / 4));
          kk = (lane & 3) + 4 * (i % (BK / 4));
        }
        const int gk = kbase + kk, gn = n0 + nn;
        int bytes = 0;
        const double *src = B;
        if (gn < N && gk < K) {
          bytes = min(VEC, K - gk) * 8;
          src = B + (int64_t)gn * ldb + gk;
        }
        cp_async<VEC * 8>(bs + nn * BP + kk, src, bytes);
      }
      // full_bar counts one arrival per producer warp; each lane's copies are
      // tracked by its own pending +1/-1 (cp.async.mbarrier.arrive).
      cp_async_mbar_arrive_inc(&full_bar[slot]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[slot]);
    }
    cp_async_wait<0>();
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  // ================= consumers: loops 2/1 + micro-kernel =================
  const int wm = warp & 1, wn = warp >> 1;
  const int r = lane >> 2, q = lane & 3;
  double acc[FM][FN][2];
  const int row0 = m0 + wm * WM + r;
  const int col0 = n0 + wn * WN + 2 * q;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = row0 + i * 8, col = col0 + j * 8 + e;
        acc[i][j][e] = (row < M && col < N) ? C[(int64_t)col * ldc + row] : 0.0;
      }

  const int a_off = q * AP + wm * WM + r;    // + kk*4*AP + i*8
  const int b_off = (wn * WN + r) * BP + q;  // + j*8*BP + kk*4
  double fa[2][FM], fb[2][FN];
  auto load_frags = [&](int buf, int slot, int kk) {
    const double *as = As + slot * A_STAGE + a_off + kk * 4 * AP;
    const double *bs = Bs + slot * B_STAGE + b_off + kk * 4;
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[buf][i] = as[i * 8];
#pragma unroll
    for (int j = 0; j < FN; ++j) fb[buf][j] = bs[j * 8 * BP];
  };

#ifdef MYD_FAST_PROFILE
  long long loop_t0 = clock64();
#endif
  {
    PROF_T0();
    mbar_wait(&full_bar[0], 0);
    if (lane == 0) PROF_ADD(4, clock64() - _pt0);
  }
  load_frags(0, 0, 0);
  auto main_loop = [&](auto probe_c) {
  constexpr int PROBE = decltype(probe_c)::value;
  for (int kt = 0; kt < KT; ++kt) {
    const int slot = kt % STAGES;
    const int nslot = (kt + 1) % STAGES;
    const uint32_t nparity = ((kt + 1) / STAGES) & 1;
    bool next_ready = true;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int cur = kk & 1;
      // Probe the next slab's barrier early; its latency hides behind DMMAs.
      if (kk == PROBE && kt + 1 < KT) next_ready = mbar_try_wait(&full_bar[nslot], nparity);
      if (kk + 1 < KSTEPS) {
        load_frags(cur ^ 1, slot, kk + 1);
      } else if (kt + 1 < KT) {
        if (!next_ready) {
          PROF_T0();
          mbar_wait(&full_bar[nslot], nparity);
          if (lane == 0) { PROF_ADD(0, clock64() - _pt0); PROF_ADD(1, 1); }
        }
        load_frags(cur ^ 1, nslot, 0);
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], fa[cur][i], fb[cur][j]);
    }
    // every fragment of this slab has been consumed by an issued DMMA
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
  }
  };
  // The two consumer warps of a sub-partition (w, w+4) probe at different
  // k-steps so their probe latencies do not coincide.
  if (STAGGER && (warp & 4)) main_loop(std::integral_constant<int, PROBE_STEP_ALT>{});
  else main_loop(std::integral_constant<int, PROBE_STEP>{});

#ifdef MYD_FAST_PROFILE
  if (lane == 0) PROF_ADD(5, clock64() - loop_t0);
#endif
  // ---- epilogue: valid region only (padding rows never touched) ----
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = row0 + i * 8, col = col0 + j * 8 + e;
        if (row < M && col < N) C[(int64_t)col * ldc + row] = acc[i][j][e];
      }
}

cudaError_t launch_dgemm_fast(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                              double *C, int64_t ldc, cudaStream_t stream, bool force_vec1) {
  using namespace fast;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const long long tiles = (long long)tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const bool aligned16 = (lda % 2 == 0) && (ldb % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  // Set on every call: cheap, per-device, and thread-safe without a flag.
  if (aligned16 && !force_vec1) {
    cudaError_t e = cudaFuncSetAttribute(dgemm_fast_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    dgemm_fast_kernel<2><<<(unsigned)tiles, THREADS, SMEM_BYTES, stream>>>(M, N, K, A, lda, B, ldb, C, ldc, tiles_m,
                                                                           tiles_n);
  } else {
    cudaError_t e = cudaFuncSetAttribute(dgemm_fast_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    dgemm_fast_kernel<1><<<(unsigned)tiles, THREADS, SMEM_BYTES, stream>>>(M, N, K, A, lda, B, ldb, C, ldc, tiles_m,
                                                                           tiles_n);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace myd

#ifdef MYD_FAST_PROFILE
extern "C" __attribute__((visibility("default"))) void my_dgemm_fast_profile(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, myd::g_fast_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(myd::g_fast_prof, z, sizeof z);
  }
}
#endif
