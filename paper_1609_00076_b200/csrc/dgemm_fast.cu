// dgemm_fast.cu -- the hot path: C := A*B + C, FP64, column-major, any ld, on sm_100a.
//
// The reference's five BLIS loops (pkg/src/gemmforge/goto.py:187-239 and
// _ckernels.pyx:15-45,142-195) re-derived for Blackwell:
//   loop 5/3 (jc, ic)  -> persistent CTAs (one per SM) walking 128x128 units of
//                         C round-robin, rastered in bands of GROUP_M tile-rows
//                         so co-resident CTAs share A and B panels in the
//                         126 MB L2; the last partial wave, a ragged last
//                         tile column or a small problem is re-cut into
//                         128x64 / 128x32 / 64x32 units so every SM gets work,
//                         the plan chosen by a measured cost model
//                         (launch_dgemm_fast); a partial last wave can run
//                         as stream-K (slabs of cut tiles split between two
//                         CTAs, the exact accumulator state handed over, so C
//                         is unchanged; its workspace is owned by the stream,
//                         nothing is allocated or zeroed per call); launches
//                         overlap their neighbours by programmatic dependent
//                         launch;
//   loop 4 (pc)        -> the in-CTA K loop over BK-deep slabs;
//   pack_a / pack_b    -> producer warps stage each A and B slab (and, for
//                         narrow units, first the unit's C block; full tiles
//                         read C from global, prefetched to L2) into a
//                         multi-stage shared-memory ring: bulk copies by the
//                         TMA engine (cp.async.bulk) for aligned interior
//                         data (partial units of small or long-K ragged
//                         problems too: the valid part only, EDGE), else
//                         zero-filling cp.async (LDGSTS) -- a ragged last K
//                         slab, 16x128 units; no pack pass touches HBM;
//   loops 2/1 + _mk    -> 8 consumer warps, each a register tile of C built
//                         from DMMA.8x8x4 fragments (mma.sync f64).  FP64 has
//                         no tcgen05 kind on sm_100a; the DMMA pipe measured
//                         37.1 TFLOP/s (128 flop/clk/SM) vs 34.0 for DFMA
//                         (profiles/fp64_peak_r01.txt).
// The accumulators start from C, like _mk's tile load (_ckernels.pyx:28-32),
// and only the valid region is stored back.  The DMMA computes the C^T block
// (B^T A^T) so each thread's accumulator pair is 16 contiguous bytes of C.
//
// Per-element arithmetic (k grouped in fours from p = 0, one DMMA per group
// that holds at least one k < K, groups in ascending order, accumulator
// starting at C) does not depend on the unit shape, the tile position, the
// K-slab depth, the launch plan or which CTA runs which slabs, so every plan
// (stream-K included) and every k-chunking at multiples of 16 gives bitwise
// the same C, down to the sign of zeros.  (One exception, never chosen unless
// asked for: the K-split plan, which sums partial chains -- see the SUM
// instantiation and include/my_dgemm.h, MY_DGEMM_PLAN_INVARIANT.)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <string>
#include <type_traits>

#include "common.cuh"

namespace myd {

#ifdef MYD_TIMELINE
// globaltimer (ns), main launches only: [0] min CTA entry, [1] max CTA exit;
// CTA 0 / consumer warp 0, first unit: [2] after barrier init, [3] unit start
// (C in registers), [4] first slab ready, [5] main loop done, [6] stores issued
// and next C block loaded; [16 + 4o + 0..3] the same marks 3..6 for units
// 8..11; [7..12] producer warp 0 marks (tools/timeline_probe.py)
__device__ unsigned long long g_tl[32];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL_MARK(i)                                                     \
  do {                                                                 \
    if (blockIdx.x == 0 && tid == 0 && !after_main) {                  \
      const unsigned long long _t = gtimer();                          \
      if (unit_ord == 0) g_tl[i] = _t;                                 \
      if (i >= 3 && unit_ord >= 8 && unit_ord < 12)                    \
        g_tl[16 + (unit_ord - 8) * 4 + (i - 3)] = _t;                  \
    }                                                                  \
  } while (0)
#else
#define TL_MARK(i) do { } while (0)
#endif
#ifdef MYD_KS_TIMELINE
// Stream-K / K-split launches: globaltimer marks of every CTA's consumer warp 0
// (tools/ksplit_timeline.py): [15] entry, [14] exit; per segment s (5 s + ..):
// +0 accumulators ready, +1 K loop done, +2 partial stored / fix-up done,
// +3 C stored, +4 next accumulators ready
__device__ unsigned long long g_kst[160][16];
#define KST(i)                                                                       \
  do {                                                                               \
    if (SKM && warp == 0 && lane == 0 && (i) < 16) {                                 \
      unsigned long long _t;                                                         \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(_t));                          \
      g_kst[blockIdx.x % 160][i] = _t;                                               \
    }                                                                                \
  } while (0)
#else
#define KST(i) do { } while (0)
#endif
#ifdef MYD_FAST_PROFILE
// [0] consumer slow-wait cycles, [1] consumer slow waits, [2] producer empty-wait cycles,
// [3] producer waits, [4] consumer first-slab wait cycles, [5] consumer total loop cycles,
// [6] consumer C-load cycles, [7] consumer units
__device__ unsigned long long g_fast_prof[8];
#define PROF_T0() long long _pt0 = clock64()
#define PROF_ADD(i, v) atomicAdd(&g_fast_prof[i], (unsigned long long)(v))
#else
#define PROF_T0()
#define PROF_ADD(i, v)
#endif

#ifndef MYD_SKIP_ZERO_KSTEPS
#define MYD_SKIP_ZERO_KSTEPS 1  // ragged-K instantiation skips the all-zero k-steps of the last K slab (0: off)
#endif
#ifndef MYD_ROWS16_BK
#define MYD_ROWS16_BK 32  // K-slab depth of the 16x128 units
#endif
#ifndef MYD_BK32_MIN_K
#define MYD_BK32_MIN_K 1024  // full tiles use 32-deep K slabs from this K on (16 below)
#endif
#ifndef MYD_CGLOBAL_SK
#define MYD_CGLOBAL_SK 1  // the stream-K kernel's full tiles too (0: ring, for A/B timing)
#endif
#ifndef MYD_CGLOBAL
#define MYD_CGLOBAL 1  // full 128x128 tiles read C from global memory (0: through the ring, for A/B timing)
#endif
#ifndef MYD_L2_HINTS
#define MYD_L2_HINTS 0  // 1: A slabs evict_last, B slabs evict_first (full tiles); 2: the reverse;
                        // 3: A evict_last only; 4: B evict_first only (profiles/r02/l2_hints_r02*.log)
#endif
#ifndef MYD_L2_PERSIST_MB
#define MYD_L2_PERSIST_MB 0  // > 0 (with MYD_L2_HINTS): persisting-L2 carve-out for evict_last lines, MB
#endif
#ifndef MYD_SPLIT_BOUNDARY
#define MYD_SPLIT_BOUNDARY 1  // full tiles: half the write-back overlaps the next unit's first slab (0: off)
#endif
#ifndef MYD_SB_KSTEPS
#define MYD_SB_KSTEPS 4  // k-steps of first-half DMMA work the split boundary overlaps with the second half's write-back
#endif
#ifndef MYD_ROUND_SYNC
#define MYD_ROUND_SYNC 0  // default of MY_DGEMM_ROUND_SYNC (rounds between re-alignments of long-K calls; 0 = off):
                          // cfg5 DRAM reads 722 -> 417 GB but +0.3 % time (profiles/r02/round_sync_r02b.log)
#endif
#ifndef MYD_KSPLIT_FIXUP_US
#define MYD_KSPLIT_FIXUP_US 2.5  // K-split plan: owner's fix-up cost per piece of a tile (us, planner model)
#endif
#ifndef MYD_EDGE_BULK
#define MYD_EDGE_BULK 1  // ragged problems of up to MYD_EDGE_BULK_WAVES waves of tiles (any size for K >= 1024) run the EDGE instantiations:
                         // partial units staged by bulk copies of their valid part (0: zero-filling LDGSTS everywhere)
#endif
#ifndef MYD_EDGE_BULK_WAVES
#define MYD_EDGE_BULK_WAVES 4
#endif
#ifndef MYD_SKIP_FIRST_C_PREFETCH
#define MYD_SKIP_FIRST_C_PREFETCH 1  // 0: L2-prefetch the first unit's C block too (A/B timing)
#endif
#if MYD_SKIP_FIRST_C_PREFETCH
#define MYD_FIRST_C_PREFETCH_OK(first) (!(first))
#else
#define MYD_FIRST_C_PREFETCH_OK(first) true
#endif
#ifndef MYD_EP_SHFL
#define MYD_EP_SHFL 1  // 128-byte-per-column epilogue stores (lane-pair swap); 0 = plain fragment stores
#endif

namespace fast {
#ifndef MYD_FAST_SMEM_KB
#define MYD_FAST_SMEM_KB 224
#endif
#ifndef MYD_FAST_GROUP_M
#define MYD_FAST_GROUP_M 8
#endif
constexpr int TILE_M = 128;              // full CTA tile rows (m); small-problem units are 64 high
constexpr int TILE_N = 128;              // full CTA tile cols (n); strips are TILE_N / split wide
constexpr int MAX_STAGES = 16;                        // ring depth cap (mbarrier arrays)
constexpr int SMEM_BUDGET = MYD_FAST_SMEM_KB * 1024;  // ring bytes per CTA
constexpr int CONSUMER_WARPS = 8;        // 2 per SM sub-partition
constexpr int PRODUCER_WARPS = 4;        // one staging warp per sub-partition
constexpr int THREADS = (CONSUMER_WARPS + PRODUCER_WARPS) * 32;
// Register split per sub-partition (16K regs): 1 producer + 2 consumers.
// Launch at 168 (12 warps x 168 x 32 <= 64K), then setmaxnreg moves
// producers down to 40 and consumers up to 232: the CTA keeps the 168 x 384
// registers it launched with (40*128 + 232*256 = 168*384); asking for more
// would block setmaxnreg.inc forever.
constexpr int PRODUCER_REGS = 40;
constexpr int CONSUMER_REGS = 232;
constexpr int WN = 32;  // warp tile width (4 DMMA column fragments)
// Ring geometry per CTA shape.  The K slab grows as the unit shrinks so
// every consumer warp still issues >= 64 DMMAs per slab (the per-slab
// barrier probe and release cost ~200 cycles): 16 for 128x128 / 128x64,
// 32 for 128x32, 64 for 64x32; full tiles of long-K aligned problems use 32
// (3 stages: fewer probes, 97.4 % vs 96.4 % at 8192^3) while short-K ones
// keep 16 (6 stages: deeper prefetch across unit boundaries, cfg4 89 % vs
// 84 %).  As many stages as fit the budget.  Pitches are 4 mod 16 doubles,
// so a half-warp's 4 k-rows of A (4 n-rows of B) land in 4 distinct 32-byte
// bank groups and every fragment load and 16-byte staging store is
// conflict-free: A slab [BK][BM+4] (m contiguous, as in HBM), B slab
// [BN][BK+4] (k contiguous, as in HBM).
template <int BM, int BN>
constexpr int default_bk() {
  return (BM * BN) / (CONSUMER_WARPS * 64) >= 16 ? 16 : ((BM * BN) / (CONSUMER_WARPS * 64) >= 8 ? 32 : 64);
}

template <int BM, int BN, int BK_ = default_bk<BM, BN>()>
struct Ring {
  static constexpr int BK = BK_;
  static constexpr int AP = BM + 4;
  static constexpr int BP = BK + 4;
  static constexpr int A_ST = BK * AP;  // doubles per A slab
  static constexpr int B_ST = BN * BP;  // doubles per B slab
  static constexpr int SLOT = A_ST + B_ST;  // one ring slot: A slab then B slab
  // A unit's C block is staged through ring slots before its first slab:
  // CPS columns per slot at pitch CP = BM + 8 (column stride = 64 B mod 128:
  // a quarter-warp's 16-byte fragment loads of 2 columns x 64 B are
  // conflict-free), CS slots.
  static constexpr int CP = BM + 8;
  static constexpr int CPS = (64 <= BN && 64 * CP <= SLOT) ? 64
                             : (32 <= BN && 32 * CP <= SLOT) ? 32
                             : (16 * CP <= SLOT) ? 16 : 8;
  static constexpr int CS = BN / CPS;
  static constexpr int STAGES_FIT = SMEM_BUDGET / ((A_ST + B_ST) * 8);
  static constexpr int STAGES = STAGES_FIT < MAX_STAGES ? STAGES_FIT : MAX_STAGES;
  static constexpr int BYTES = STAGES * SLOT * 8;
  static_assert(STAGES >= 3, "ring too shallow");
  static_assert(CS < STAGES && BN % CPS == 0 && CPS * CP <= SLOT, "C staging must leave a slab slot");
};
constexpr int GROUP_M = MYD_FAST_GROUP_M;
constexpr int PROBE_STEP = 1;  // k-step at which the next slab's barrier is probed
}  // namespace fast

// VEC: doubles per LDGSTS (2: 16-byte copies and the bulk path, needs even
// ld and 16-B aligned bases; 1: 8-byte copies for odd ld / 8-B aligned views
// -- dispatch() normally copies such operands to even-ld scratch first).
// BM x BN: unit shape (128x128 full tiles; 128x64, 128x32, 64x32 units).
// Warps tile the unit as (8 / (BN/32)) x (BN/32) with 32-column warp tiles, so
// all 8 consumer warps work whatever the shape.  BKT: K-slab depth.
//
// Warp roles: warps 0..7 consume (DMMA), warps 8..11 produce (staging).
// full[s] completes when slab s has landed (bulk-copy transaction bytes or
// LDGSTS completions); empty[s] when all 8 consumers have their fragments of
// slab s in registers.  No CTA-wide barrier in the main loop.
template <int VEC, int BM, int BN, int BKT, bool SKM, bool CGT, bool RK, bool RS = false, bool SUM = false,
          bool EDGE = false>
__global__ void __launch_bounds__(fast::THREADS, 1)
    dgemm_fast_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                      int64_t ldb, double *__restrict__ C, int64_t ldc, int tiles_m, int tiles_n, int tile0, int edge,
                      int units, int after_main, StreamK sk, Epilogue ep) {
  using namespace fast;
  constexpr int SPLIT_M = TILE_M / BM, SPLIT_N = TILE_N / BN;
  constexpr int SPLIT = SPLIT_M * SPLIT_N;  // work units per full tile
  using R = Ring<BM, BN, BKT>;
  constexpr int BK = R::BK;          // K slab per stage
  constexpr int KSTEPS = BK / 4;     // DMMA k-steps per slab
  constexpr int AP = R::AP, BP = R::BP;
  constexpr int STAGES = R::STAGES;
  constexpr int SLOT = R::SLOT, A_STAGE = R::A_ST;
  constexpr int CP = R::CP, CPS = R::CPS, CS = R::CS;
  constexpr int WARPS_N = BN / WN;
  constexpr int WARPS_M = CONSUMER_WARPS / WARPS_N;
  constexpr int WM = BM / WARPS_M;
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int RW = BN / PRODUCER_WARPS;  // B rows staged by each producer warp
  static_assert(WARPS_M * WARPS_N == CONSUMER_WARPS && FM >= 1 && RW >= 8, "tile shape");
  // Full tiles of the unit-mode kernel read their C block straight from
  // global memory (the producers prefetch it to L2 when they start the
  // unit; the consumers read it into each fragment pair right after storing
  // that pair of the previous unit) instead of staging it through ring slots:
  // the C block no longer takes 2 of 3 (BK 32) or 4 of 6 (BK 16) slots at
  // every unit boundary, so slab prefetch keeps going across it.  cfg4
  // 91.4 -> 94.3 %, k = 128 85.5 -> 91.5 %, 8192^3 +0.2 %
  // (profiles/c_from_global_r01.log); the stream-K kernel's full tiles too
  // (2048^3, all stream-K, +0.6 %).  Narrower units keep the ring path
  // (measured slower this way).
  constexpr bool CG = CGT && MYD_CGLOBAL && VEC == 2 && BM == 128 && BN == 128 && (!SKM || MYD_CGLOBAL_SK);
  // The full-tile instantiation launched for an unaligned C (odd ldc, see
  // launch_one): its C columns alternate 16-byte alignment, so every other
  // column is still staged by bulk copy and stored with 16-byte stores.  Kept
  // out of the other instantiations, whose code this slows (2-5 %).
  constexpr bool ODD_C = VEC == 2 && BM == 128 && BN == 128 && !CGT;

  extern __shared__ __align__(128) double smem[];  // STAGES slots of [A slab | B slab]
  __shared__ __align__(8) uint64_t full_bar[MAX_STAGES];
  __shared__ __align__(8) uint64_t empty_bar[MAX_STAGES];

  // Work unit u (persistent CTA b takes u = b, b + gridDim.x, ...): full
  // 128x128 tile tile0 + u / SPLIT in the grouped raster (GROUP_M tile-rows
  // per band, column-major inside a band), sub-block u % SPLIT of it.  With
  // edge = ns > 0 the ragged last tile column is kept out of the raster and
  // its units follow the raster's: per tile row, the SPLIT_M x ns sub-blocks
  // that hold valid columns; with edge = -ms < 0 the same for a ragged last
  // tile row: per tile column, the ms x SPLIT_N sub-blocks holding valid rows
  // (launch_dgemm_fast's edge plans).  Units wholly outside C are skipped.
  const int raster_units = (tiles_m * tiles_n - tile0) * SPLIT;  // units of raster tiles in this launch
  const int edge_ns = edge > 0 ? edge : 0, edge_ms = edge < 0 ? -edge : 0;
  auto unit_origin = [&](int u, int &m0, int &n0) {
    if (edge_ns > 0 && u >= raster_units) {  // edge column: only its edge_ns valid strips per sub-row
      const int e = u - raster_units, per = SPLIT_M * edge_ns, idx = e % per;
      m0 = (e / per) * TILE_M + (idx / edge_ns) * BM;
      n0 = tiles_n * TILE_N + (idx % edge_ns) * BN;
      return;
    }
    if (edge_ms > 0 && u >= raster_units) {  // edge row: only its edge_ms valid sub-rows per tile column
      const int e = u - raster_units, per = edge_ms * SPLIT_N, idx = e % per;
      m0 = tiles_m * TILE_M + (idx / SPLIT_N) * BM;
      n0 = (e / per) * TILE_N + (idx % SPLIT_N) * BN;
      return;
    }
    const int tile = tile0 + u / SPLIT, sub = u % SPLIT;
    const int band = GROUP_M * tiles_n;
    const int first_m = (tile / band) * GROUP_M;
    const int gm = min(tiles_m - first_m, GROUP_M);
    m0 = (first_m + (tile % band) % gm) * TILE_M + (sub / SPLIT_N) * BM;
    n0 = ((tile % band) / gm) * TILE_N + (sub % SPLIT_N) * BN;
  };
  // this CTA's next non-empty unit at or after u (u itself on this CTA's stride)
  const bool ragged = (M % TILE_M) != 0 || (N % TILE_N) != 0;  // else no unit can be empty
  auto next_unit = [&](int u) {
    if (!ragged) return u;
    for (; u < units; u += gridDim.x) {
      int m0, n0;
      unit_origin(u, m0, n0);
      if (m0 < M && n0 < N) break;
    }
    return u;
  };

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
#ifdef MYD_TIMELINE
  int unit_ord = 0;  // units finished by this consumer warp (timeline marks)
  if (tid == 0 && !after_main) atomicMin(&g_tl[0], gtimer());
#endif
  const int KT = (K + BK - 1) / BK;

  // Work segments.  Unit mode (sk.iters == 0): unit u, all K slabs, from C to
  // C.  Stream-K mode (full tiles only): tiles [0, dp_tiles) run whole,
  // round-robin (data-parallel rounds: co-running tiles stay neighbours in
  // the raster, sharing A/B panels in L2); the remaining tiles' (tile, slab)
  // iterations are split evenly over the CTAs.  Within a tile the iterations
  // are numbered by DESCENDING slab, so a tile cut between CTA b (end of its
  // range) and b + 1 (start of its range) leaves CTA b + 1 -- which gets
  // there first -- the LOWER slabs, from C to a partial accumulator written
  // to workspace slot b, and CTA b the UPPER slabs, from that partial to C.
  // Each segment runs its slabs in ascending order, so every element sees
  // exactly the DMMA chain of one CTA doing the whole K: bitwise the same C,
  // without the last round's quantisation.  The stream-K phase spans at
  // least one tile per CTA, so a tile is cut at most once, and CTA b only
  // ever waits for CTA b + 1's first segment (which waits on nothing): no
  // deadlock.  Cursor: < SK0 a data-parallel tile, else SK0 + iteration.
  //
  // K-split mode (SUM, its own instantiation; fewer tiles than CTAs, so a
  // CTA's range is shorter than a tile and a tile is cut into several pieces):
  // the same even split, but the pieces of a tile are independent.  The piece
  // holding the top slab (the end of CTA b's range) is the owner: it starts
  // from C and, after its slabs, adds the partial sums of the tile's other
  // pieces -- each accumulated from zero by CTAs b + 1, b + 2, ... as the
  // first segment of their ranges (so they are done, or finish together with
  // the owner) -- in CTA order, then stores C.  No piece waits before its
  // slabs, so the K chain of a tile runs on several SMs at once; each element
  // is a fixed function of (m, n, k, CTA count), but no longer the single
  // ascending chain of the other plans (launch_dgemm_fast: only chosen when
  // the caller has not asked for plan-invariant results).
  struct Seg {
    int m0, n0, kb, ke, slot;
    bool from_c, to_c;
  };
  constexpr int SK0 = 1 << 30;  // stream-K cursors (the planner keeps iterations < 2^30)
  const int sk_iters = (int)sk.iters, sk_dp = (int)sk.dp_tiles;
  const int sk_per = sk_iters / (int)gridDim.x, sk_rem = sk_iters % (int)gridDim.x;
  const int sk_lo = sk_per * (int)blockIdx.x + min((int)blockIdx.x, sk_rem);
  const int sk_hi = sk_lo + sk_per + ((int)blockIdx.x < sk_rem ? 1 : 0);
  auto seg_at = [&](int cur, Seg &sg) -> bool {
    if constexpr (!SKM) {
      if (cur >= units) return false;
      unit_origin(cur, sg.m0, sg.n0);
      sg.kb = 0;
      sg.ke = KT;
      sg.from_c = sg.to_c = true;
      sg.slot = -1;
      return true;
    } else {
      if (cur < SK0) {  // data-parallel tile
        unit_origin(cur, sg.m0, sg.n0);
        sg.kb = 0;
        sg.ke = KT;
        sg.from_c = sg.to_c = true;
        sg.slot = -1;
        return true;
      }
      const int it = cur - SK0;
      if (it >= sk_hi) return false;
      const int t = it / KT, l0 = it - t * KT;
      const int l1 = min(KT, sk_hi - t * KT);
      unit_origin((int)sk.tile0 + t, sg.m0, sg.n0);
      sg.kb = KT - l1;
      sg.ke = KT - l0;
      sg.to_c = sg.ke == KT;
      if constexpr (SUM) {
        sg.from_c = sg.to_c;          // the owner starts from C, the other pieces from zero
        sg.slot = (int)blockIdx.x;    // a CTA's only non-owner piece is the first of its range
      } else {
        sg.from_c = sg.kb == 0;
        sg.slot = sg.to_c ? (int)blockIdx.x : (int)blockIdx.x - 1;  // upper part reads b; lower part writes b - 1
      }
      return true;
    }
  };
  auto seg_first = [&]() -> int {
    if constexpr (!SKM) {
      return next_unit(blockIdx.x);
    } else {
      return (int)blockIdx.x < sk_dp ? (int)blockIdx.x : SK0 + sk_lo;
    }
  };
  auto seg_next = [&](int cur, const Seg &sg) -> int {
    if constexpr (!SKM) {
      return next_unit(cur + gridDim.x);
    } else {
      if (cur < SK0) return cur + (int)gridDim.x < sk_dp ? cur + (int)gridDim.x : SK0 + sk_lo;
      const int it = cur - SK0;
      return SK0 + (it / KT) * KT + (KT - sg.kb);
    }
  };


  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], PRODUCER_WARPS);   // one arrival per producer warp
      mbar_init(&empty_bar[s], CONSUMER_WARPS);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  TL_MARK(2);
  // Programmatic dependent launch (PDL): a call's first launch may start
  // while the previous kernel in the stream drains, so it waits for that
  // grid's completion (and memory flush) before touching global memory --
  // the producers after working out their first unit, the consumers at once
  // (their first global access comes after the producers' data anyway).  A
  // call's tail launch works on tiles the main launch never touches and
  // reads only A and B, so it starts as soon as SMs free up and waits at the
  // very end instead (stream order of completion is kept).  Dependents are
  // released only once this grid has passed its own wait (the tail launch
  // reads A and B, which the grid before the main launch may have written).
  // Without the PDL launch attribute all of this is a no-op.
  if (after_main) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

  if (warp >= CONSUMER_WARPS) {
    // ================= producers: pack_a / pack_b equivalent =================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int pw = warp - CONSUMER_WARPS;
    const bool c_aligned = (ldc % 2 == 0) && ((uintptr_t)C % 16 == 0);
    const bool c16 = ODD_C && ((uintptr_t)C % 16 == 0);
#ifdef MYD_TIMELINE
    if (blockIdx.x == 0 && pw == 0 && lane == 0) g_tl[8] = gtimer();
#endif
    uint32_t g = 0;  // ring slots filled by this CTA so far (C blocks and slabs)
    [[maybe_unused]] uint64_t pol_a = 0, pol_b = 0;
    if constexpr (MYD_L2_HINTS == 1) {
      pol_a = l2_policy_evict_last();
      pol_b = l2_policy_evict_first();
    } else if constexpr (MYD_L2_HINTS == 2) {
      pol_a = l2_policy_evict_first();
      pol_b = l2_policy_evict_last();
    } else if constexpr (MYD_L2_HINTS == 3) {
      pol_a = l2_policy_evict_last();
      pol_b = l2_policy_evict_normal();
    } else if constexpr (MYD_L2_HINTS == 4) {
      pol_a = l2_policy_evict_normal();
      pol_b = l2_policy_evict_first();
    }
    int cur = seg_first();
    Seg sg;
    bool have = seg_at(cur, sg);  // integer work, overlapping the previous grid's drain
    if (!after_main) asm volatile("griddepcontrol.wait;\n" "griddepcontrol.launch_dependents;\n" ::: "memory");
    bool first_seg = true;
    for (; have; cur = seg_next(cur, sg), have = seg_at(cur, sg), first_seg = false) {
      const int m0 = sg.m0, n0 = sg.n0;
      if constexpr (RS && !SKM) {
        // Round re-alignment (its own instantiation, long-K whole-tile
        // launches only, co-resident grid): before the first slab of round w
        // (a multiple of R = sk.iters, below sk.dp_tiles whole rounds) the CTA
        // arrives on the zeroed counter sk.flags[0] and waits for all of
        // them; only producer warp 0 waits -- no slab of the round completes
        // without its arrival, so the whole CTA follows.  Over a 1.9 s cfg5
        // call the CTAs otherwise drift apart in K and read shared panel
        // slabs from HBM once per drifted sharer instead of once per round
        // (profiles/r02/dram_drift_r02a.log).
        if (pw == 0) {
          const int w = cur / (int)gridDim.x, R = (int)sk.iters;
          if (w > 0 && w < (int)sk.dp_tiles && w % R == 0) {
            if (lane == 0) {
              atomicAdd(sk.flags, 1ull);
              const unsigned long long target = (unsigned long long)(w / R) * gridDim.x;
              for (;;) {
                unsigned long long v;
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(sk.flags) : "memory");
                if (v >= target) break;
                __nanosleep(200);
              }
            }
            __syncwarp();
          }
        }
      }
#ifdef MYD_TIMELINE
      if (blockIdx.x == 0 && pw == 0 && lane == 0 && first_seg) g_tl[9] = gtimer();
#endif
      // C block of the unit through CS ring slots (my_dgemm contract only:
      // the BLAS epilogue reads C at the end instead).  The copies are issued
      // while the consumers finish the previous unit, so the C load is off the
      // critical path and spread in time instead of bursting at unit start.
      // (not for a launch's first unit: the consumers read that C block at the
      // same moment anyway, and the 128 prefetch operations queue in the
      // bulk-copy engine ahead of the first slabs -- the first slab went out
      // 2.8 us after the grid dependency cleared, profiles/r02/timeline_1536_r02a.log)
      if (CG && (!ep.blas || ep.beta != 0.0) && sg.from_c && MYD_FIRST_C_PREFETCH_OK(first_seg)) {  // BLAS: C is read by the epilogue
        const int rows = max(0, min(BM, M - m0));
        const int col = pw * (BN / PRODUCER_WARPS) + lane;
        if (c_aligned && rows > 0 && rows % 2 == 0 && lane < BN / PRODUCER_WARPS && n0 + col < N)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(C + (int64_t)(n0 + col) * ldc + m0),
                       "r"(rows * 8)
                       : "memory");
      }
      if (!CG && !ep.blas && sg.from_c) {
        const bool c_bulk = c_aligned && (m0 + BM <= M) && (n0 + BN <= N);
        for (int cs = 0; cs < CS; ++cs, ++g) {
          const int slot = g % STAGES;
          if (g >= STAGES) mbar_wait(&empty_bar[slot], ((g / STAGES) - 1) & 1);
          double *cb = smem + slot * SLOT;
          const int c_first = n0 + cs * CPS;
          // Producer warp pw stages columns [pw*CW, pw*CW+CW) of this slot.
          // Whole aligned columns go by bulk copy; otherwise only the valid
          // rows of valid columns are copied (8-byte cp.async); rows/columns
          // outside C stay stale -- their accumulators are never stored.
          constexpr int CW = CPS / PRODUCER_WARPS;
          const int rows = max(0, min(BM, M - m0));  // 0 for a unit wholly below C
          // a column goes by bulk copy when its first valid element is 16-byte
          // aligned and it holds an even number of rows (with an odd ldc,
          // every other column of a 16-byte aligned C)
          auto col_bulk = [&](int gcol) {
            return c_bulk || (c16 && rows % 2 == 0 && ((((int64_t)gcol * ldc + m0) & 1) == 0));
          };
          for (int c = 0; c < CW; ++c) {
            const int col = pw * CW + c;
            if (c_first + col >= N) break;
            if (col_bulk(c_first + col)) continue;
            for (int row = lane; row < rows; row += 32)
              cp_async<8>(cb + col * CP + row, C + (int64_t)(c_first + col) * ldc + m0 + row, 8);
          }
          cp_async_mbar_arrive_inc(&full_bar[slot]);
          __syncwarp();
          int valid_cols = min(CW, N - c_first - pw * CW);
          valid_cols = (valid_cols < 0 || rows == 0) ? 0 : valid_cols;
          const bool mine = lane < valid_cols && col_bulk(c_first + pw * CW + lane);
          const uint32_t bulk_bytes = (uint32_t)__popc(__ballot_sync(0xffffffffu, mine)) * rows * 8;
          if (lane == 0) mbar_arrive_expect_tx(&full_bar[slot], bulk_bytes);
          __syncwarp();
          if (mine) {
            const int col = pw * CW + lane;
            bulk_g2s(cb + col * CP, C + (int64_t)(c_first + col) * ldc + m0, rows * 8, &full_bar[slot]);
          }
#ifdef MYD_TIMELINE
          if (blockIdx.x == 0 && pw == 0 && lane == 0 && first_seg) g_tl[10 + cs] = gtimer();
#endif
        }
      }
      // Interior units with 16-byte aligned operands use the bulk-copy (TMA)
      // engine straight into the padded slab layout, with no LSU traffic.
      // Edge units and a ragged last slab use zero-filling LDGSTS.  So do the
      // 16x128 units: their slab is 160 small copies (32 A rows of 128 B, 128
      // B columns of 256 B) per 1024 DMMA cycles, more than the bulk-copy
      // engine issues -- LDGSTS staging runs them 1.8x faster, while every
      // other shape is 3-5 % faster with bulk copies
      // (profiles/rows16_staging_r01.log).
      constexpr bool BULK_UNIT = BM != 16;
      const bool interior = BULK_UNIT && (VEC == 2) && (m0 + BM <= M) && (n0 + BN <= N);
      for (int kt = sg.kb; kt < sg.ke; ++kt, ++g) {
        const int slot = g % STAGES;
        if (g >= STAGES) {
          PROF_T0();
          mbar_wait(&empty_bar[slot], ((g / STAGES) - 1) & 1);
          if (lane == 0) {
            PROF_ADD(2, clock64() - _pt0);
            PROF_ADD(3, 1);
          }
        }
        const int kbase = kt * BK;
        double *as = smem + slot * SLOT;
        double *bs = as + A_STAGE;
        if (interior && kbase + BK <= K) {
          constexpr int A_ROWS = BK / PRODUCER_WARPS;  // k-rows of A per producer warp
          constexpr uint32_t BYTES = (A_ROWS * BM + RW * BK) * 8;
          if (lane == 0) mbar_arrive_expect_tx(&full_bar[slot], BYTES);
          __syncwarp();
          if constexpr (MYD_L2_HINTS != 0 && BM == 128 && BN == 128) {
            // raster bands share A panels across waves (GROUP_M tile rows) and
            // B panels within a wave: keep the band's A (or B) in L2
            if (lane < A_ROWS) {
              const int kk = pw * A_ROWS + lane;
              bulk_g2s_hint(as + kk * AP, A + (int64_t)(kbase + kk) * lda + m0, BM * 8, &full_bar[slot], pol_a);
            }
            if (lane < RW) {
              const int nn = pw * RW + lane;
              bulk_g2s_hint(bs + nn * BP, B + (int64_t)(n0 + nn) * ldb + kbase, BK * 8, &full_bar[slot], pol_b);
            }
          } else {
            if (lane < A_ROWS) {
              const int kk = pw * A_ROWS + lane;
              bulk_g2s(as + kk * AP, A + (int64_t)(kbase + kk) * lda + m0, BM * 8, &full_bar[slot]);
            }
            if (lane < RW) {
              const int nn = pw * RW + lane;
              bulk_g2s(bs + nn * BP, B + (int64_t)(n0 + nn) * ldb + kbase, BK * 8, &full_bar[slot]);
            }
          }
#ifdef MYD_TIMELINE
          if (blockIdx.x == 0 && pw == 0 && lane == 0 && first_seg && kt == sg.kb) g_tl[7] = gtimer();
#endif
          continue;
        }
        if constexpr (BULK_UNIT && VEC == 2 && EDGE) {
          // Partial units (the ragged last tile row / column) on a full K slab:
          // bulk copies of the valid part only -- each k-row of A over the
          // unit's valid rows (an even count; the last row of an odd one by an
          // 8-byte cp.async), each valid column of B.  Rows and columns past
          // M and N keep whatever the slot held: they only ever reach
          // accumulators that are never stored (an element of C depends on
          // its own row of A and column of B alone), so they need no zero
          // fill -- unlike a ragged last K slab, which stays on the
          // zero-filling LDGSTS path below.  Bounds-checked LDGSTS made a
          // partial unit 1.3 - 1.7x as long as a whole one
          // (profiles/r02/planner_regret_r02b.log).  Its own instantiation
          // (EDGE, launch_one): with this code in every kernel the whole-tile
          // kernel lost 8 % at cfg4 and 0.3 % at 8192^3 on problems that have
          // no partial unit at all (profiles/r02/ab_libs_r02d.log).
          if (kbase + BK <= K) {
            constexpr int A_ROWS = BK / PRODUCER_WARPS;
            const int vcols = max(0, min(BN, N - n0));
            const int vrows = vcols > 0 ? max(0, min(BM, M - m0)) : 0;  // (an empty unit stages nothing)
            const int ev = vrows & ~1;
            const bool a_mine = lane < A_ROWS && ev > 0;
            const bool b_mine = vrows > 0 && lane < RW && pw * RW + lane < vcols;
            if (vrows & 1) {
              if (lane < A_ROWS) {
                const int kk = pw * A_ROWS + lane;
                cp_async<8>(as + kk * AP + ev, A + (int64_t)(kbase + kk) * lda + m0 + ev, 8);
              }
              cp_async_mbar_arrive_inc(&full_bar[slot]);
              __syncwarp();
            }
            const uint32_t bytes = (uint32_t)__popc(__ballot_sync(0xffffffffu, a_mine)) * ev * 8 +
                                   (uint32_t)__popc(__ballot_sync(0xffffffffu, b_mine)) * BK * 8;
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[slot], bytes);
            __syncwarp();
            if (a_mine) {
              const int kk = pw * A_ROWS + lane;
              bulk_g2s(as + kk * AP, A + (int64_t)(kbase + kk) * lda + m0, ev * 8, &full_bar[slot]);
            }
            if (b_mine) {
              const int nn = pw * RW + lane;
              bulk_g2s(bs + nn * BP, B + (int64_t)(n0 + nn) * ldb + kbase, BK * 8, &full_bar[slot]);
            }
            continue;
          }
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
        // B slab [BN][BK], k contiguous: producer pw owns rows [RW*pw, RW*pw+RW).
        // VEC=2: a quarter-warp writes 4 rows x 2 chunks (conflict-free at BP).
#pragma unroll
        for (int i = 0; i < RW * BK / (VEC * 32); ++i) {
          const int idx = i * 32 + lane;
          int nn, kk;
          if constexpr (VEC == 2) {
            nn = pw * RW + (idx >> 1) % RW;
            kk = 2 * (((idx >> 1) / RW) * 2 + (idx & 1));
          } else {
            nn = pw * RW + (idx >> 2) % RW;
            kk = ((idx >> 2) / RW) * 4 + (idx & 3);
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
    }
    cp_async_wait<0>();
    if (after_main) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  if (!after_main) asm volatile("griddepcontrol.wait;\n" "griddepcontrol.launch_dependents;\n" ::: "memory");
  // ================= consumers: loops 2/1 + micro-kernel =================
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int r = lane >> 2, q = lane & 3;
  const int a_off = q * AP + wm * WM + r;    // + kk*4*AP + i*8
  const int b_off = (wn * WN + r) * BP + q;  // + j*8*BP + kk*4
  double fa[2][FM], fb[2][FN];
  auto load_frags = [&](int buf, int slot, int kk) {
    const double *as = smem + slot * SLOT + a_off + kk * 4 * AP;
    const double *bs = smem + slot * SLOT + A_STAGE + b_off + kk * 4;
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[buf][i] = as[i * 8];
#pragma unroll
    for (int j = 0; j < FN; ++j) fb[buf][j] = bs[j * 8 * BP];
  };

  // smem index of fragment pair (i, j) inside a C block staged at ring
  // position gpos: column cl = wn*WN + 8j + r lives in slot gpos + cl / CPS at
  // column cl % CPS (r < 8 and CPS a multiple of 8, so the slot offset is
  // fixed per warp and j: one base register per slot, constant offsets).
  auto c_index = [&](uint32_t gpos, int i, int j) -> int {
    const int c8 = wn * WN + j * 8;
    int so, ci;
    if constexpr (CPS >= WN) {
      so = (wn * WN) / CPS;
      ci = (wn * WN) % CPS + j * 8 + r;
    } else {
      so = c8 / CPS;
      ci = c8 % CPS + r;
    }
    return (int)((gpos + so) % STAGES) * SLOT + ci * CP + wm * WM + i * 8 + 2 * q;
  };
  const bool c_aligned = (ldc % 2 == 0) && ((uintptr_t)C % 16 == 0);
  double acc[FM][FN][2];
  // The accumulator starts at C (_mk's tile load): the unit's C block is
  // staged in CS ring slots ahead of its slabs.  BLAS epilogue: starts at 0.
  auto load_c_block = [&](uint32_t gpos) {
#ifdef MYD_FAST_PROFILE
    long long c_t0 = clock64();
#endif
    if (ep.blas) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      return;
    }
    for (int cs = 0; cs < CS; ++cs) mbar_wait(&full_bar[(gpos + cs) % STAGES], ((gpos + cs) / STAGES) & 1);
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const double2 v = *reinterpret_cast<const double2 *>(&smem[c_index(gpos, i, j)]);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
    __syncwarp();
    if (lane == 0)
      for (int cs = 0; cs < CS; ++cs) mbar_arrive(&empty_bar[(gpos + cs) % STAGES]);
#ifdef MYD_FAST_PROFILE
    if (lane == 0) PROF_ADD(6, clock64() - c_t0);
#endif
  };
  // Stream-K partial accumulators: workspace slot s, warp w holds this
  // warp's FM x FN x 2 values as double2 [v][lane] (coalesced); the flag of
  // (s, w) carries the launch's epoch once they are written.
  constexpr int NV2 = FM * FN;  // double2 per lane
  auto part_base = [&](int slot) -> double2 * {
    return reinterpret_cast<double2 *>(sk.work) + ((int64_t)slot * CONSUMER_WARPS + warp) * NV2 * 32 + lane;
  };
  // (two steps: the stores are issued, the caller starts loading the next
  // segment's accumulators, and only then does the flag go out -- its release,
  // cumulative over the warp's stores through the warp barrier, waits for them
  // while the loads are already in flight)
  auto store_partial = [&](int slot) {
    double2 *p = part_base(slot);
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) __stcg(p + (i * FN + j) * 32, make_double2(acc[i][j][0], acc[i][j][1]));
  };
  auto publish_partial = [&](int slot) {
    __syncwarp();
    if (lane == 0)
      asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(sk.flags + slot * CONSUMER_WARPS + warp),
                   "l"(sk.epoch)
                   : "memory");
  };
  auto wait_partial = [&](int slot) {
    const unsigned long long *f = sk.flags + slot * CONSUMER_WARPS + warp;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(f) : "memory");
      if (v == sk.epoch) break;
      __nanosleep(64);
    }
  };
  // K-split: acc += the partial sums in workspace slot `slot`
  // (loads in batches of PB, all in flight before the first add: with the
  // compiler's 4 per batch a 128 KB partial took ~2.5 us of L2 round trips)
  [[maybe_unused]] auto add_partial = [&](int slot) {
    wait_partial(slot);
    const double2 *p = part_base(slot);
    constexpr int PB = NV2 < 16 ? NV2 : 16;
#pragma unroll
    for (int v0 = 0; v0 < NV2; v0 += PB) {
      double2 t[PB];
#pragma unroll
      for (int v = 0; v < PB; ++v)
        asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];\n" : "=d"(t[v].x), "=d"(t[v].y) : "l"(p + (v0 + v) * 32));
#pragma unroll
      for (int v = 0; v < PB; ++v) {
        acc[(v0 + v) / FN][(v0 + v) % FN][0] += t[v].x;
        acc[(v0 + v) / FN][(v0 + v) % FN][1] += t[v].y;
      }
    }
  };
  auto load_partial = [&](int slot) {
    wait_partial(slot);
    const double2 *p = part_base(slot);
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const double2 v = __ldcg(p + (i * FN + j) * 32);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      }
  };
  // CG: fragment pair (i, j) of a unit at (row0, col0) straight from C
  auto load_c_pair = [&](int i, int j, int row0, int col0, bool inside) {
    const int row = row0 + i * 8, col = col0 + j * 8;
    const double *cp = C + (int64_t)col * ldc + row;
    if (inside) {
      const double2 v = __ldcg(reinterpret_cast<const double2 *>(cp));
      acc[i][j][0] = v.x;
      acc[i][j][1] = v.y;
    } else {
      acc[i][j][0] = (row < M && col < N) ? __ldcg(cp) : 0.0;
      acc[i][j][1] = (row + 1 < M && col < N) ? __ldcg(cp + 1) : 0.0;
    }
  };
  auto c_inside = [&](const Seg &s) { return c_aligned && s.m0 + BM <= M && s.n0 + BN <= N; };
  constexpr int CSR = CG ? 0 : CS;  // ring slots a unit's C block occupies
  // accumulator initialisation of a segment whose C block (if any) sits at
  // ring position gpos; returns the ring position of its first slab
  auto init_acc = [&](const Seg &sg, uint32_t gpos) -> uint32_t {
    if (!sg.from_c) {
      if constexpr (SUM) {  // a K-split piece that does not own the tile: partial sums from zero
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      } else {
        load_partial(sg.slot);
      }
      return gpos;
    }
    if constexpr (CG) {
      if (!ep.blas) {
        const bool inside = c_inside(sg);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) load_c_pair(i, j, sg.m0 + wm * WM + 2 * q, sg.n0 + wn * WN + r, inside);
        return gpos;
      }
    }
    load_c_block(gpos);
    return ep.blas ? gpos : gpos + CSR;
  };
  uint32_t g = 0;  // ring position (C blocks and slabs consumed so far)
  int cur = seg_first();
  Seg sg;
  bool have = seg_at(cur, sg);
  KST(15);
  if (have) g = init_acc(sg, 0);
  [[maybe_unused]] int seg_ord = 0;
  int kt0 = 0;  // slabs of this segment already done (the split boundary runs the first one)
  while (have) {
    const int NS = sg.ke - sg.kb;
    TL_MARK(3);
    KST(seg_ord * 5);
#ifdef MYD_FAST_PROFILE
    long long loop_t0 = clock64();
#endif
    if (kt0 < NS) {
      PROF_T0();
      mbar_wait(&full_bar[(g + kt0) % STAGES], ((g + kt0) / STAGES) & 1);
      if (lane == 0) PROF_ADD(4, clock64() - _pt0);
      TL_MARK(4);
      load_frags(0, (g + kt0) % STAGES, 0);
    }
    for (int kt = kt0; kt < NS; ++kt) {
      const uint32_t gs = g + kt;
      const int slot = gs % STAGES;
      const int nslot = (gs + 1) % STAGES;
      const uint32_t nparity = ((gs + 1) / STAGES) & 1;
      bool next_ready = true;
      // RK (K not a multiple of BK, its own instantiation: a runtime exit in
      // the unrolled k-step loop costs the other shapes 0.3-4 %): the k-steps
      // of the last slab past K hold only the zero fill and are skipped.
      // Every unit shape, plan and k-chunking of a problem computes the same
      // k-steps (those holding at least one k < K; chunks are multiples of
      // 16), so C stays bitwise plan-invariant, the sign of zeros included.
      const int kvalid = (RK && sg.kb + kt == KT - 1) ? (K - (KT - 1) * BK + 3) / 4 : KSTEPS;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        if constexpr (RK) {
          if (kk > 0 && kk >= kvalid) break;
        }
        const int cur_buf = kk & 1;
        // Probe the next slab's barrier early; its latency hides behind DMMAs.
        if (kk == PROBE_STEP && kt + 1 < NS) next_ready = mbar_try_wait(&full_bar[nslot], nparity);
        if (kk + 1 < KSTEPS) {
          load_frags(cur_buf ^ 1, slot, kk + 1);
        } else if (kt + 1 < NS) {
          if (!next_ready) {
            PROF_T0();
            mbar_wait(&full_bar[nslot], nparity);
            if (lane == 0) {
              PROF_ADD(0, clock64() - _pt0);
              PROF_ADD(1, 1);
            }
          }
          load_frags(cur_buf ^ 1, nslot, 0);
        }
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], fb[cur_buf][j], fa[cur_buf][i]);
      }
      // every fragment of this slab has been consumed by an issued DMMA
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
    }

#ifdef MYD_FAST_PROFILE
    if (lane == 0) {
      PROF_ADD(5, clock64() - loop_t0);
      PROF_ADD(7, 1);
    }
#endif
    TL_MARK(5);
    KST(seg_ord * 5 + 1);
    // the next segment (worked out after the K loop: nothing extra stays live in it)
    const int ncur = seg_next(cur, sg);
    Seg nsg;
    const bool has_next = seg_at(ncur, nsg);
    bool c_loaded = false;  // the next unit's C block already in the accumulators
    kt0 = 0;
    if (!sg.to_c) {
      store_partial(sg.slot);  // the lower slabs of a tile another CTA finishes (published below)
      KST(seg_ord * 5 + 2);
    } else {
      if constexpr (SKM && SUM) {
        // K-split owner of a cut tile: the other pieces' partial sums, in CTA
        // order (CTAs b + 1, ... whose range starts inside this tile)
        if (cur >= SK0 && sg.kb > 0) {
          const int tile_end = ((cur - SK0) / KT + 1) * KT;
          for (int b2 = (int)blockIdx.x + 1; b2 < (int)gridDim.x; ++b2) {
            if (sk_per * b2 + min(b2, sk_rem) >= tile_end) break;
            add_partial(b2);
          }
        }
      }
      KST(seg_ord * 5 + 2);
      // Accumulator map (the DMMA computes the C^T block, B^T A^T, so each
      // thread's pair is two consecutive rows of one column: 16 contiguous
      // bytes in column-major C):  acc[i][j][e] = C(row0 + 8i + e, col0 + 8j).
      const int row0 = sg.m0 + wm * WM + 2 * q;
      const int col0 = sg.n0 + wn * WN + r;
      // ---- epilogue: valid region only (padding rows never touched) ----
      const bool vec_store = c_aligned;
      // odd ldc with a 16-byte aligned base: every other column still takes 16-byte stores
      const bool c16 = ODD_C && ((uintptr_t)C % 16 == 0);
      bool stored = false;
      if (ep.blas) {
        // BLAS epilogue, alpha * (A B) + beta * C (C not read when beta == 0),
        // applied to the accumulators before any store: with no store between
        // them the C reads (L2-prefetched at unit start) are all in flight at
        // once instead of one round trip per fragment behind each store.
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) {
            const int row = row0 + i * 8, col = col0 + j * 8;
            double &v0 = acc[i][j][0], &v1 = acc[i][j][1];
            if (ep.beta == 0.0 || col >= N || row >= M) {
              v0 *= ep.alpha;
              v1 *= ep.alpha;
              continue;
            }
            const double *cp = C + (int64_t)col * ldc + row;
            v0 = fma(ep.alpha, v0, ep.beta * cp[0]);
            if (row + 1 < M) v1 = fma(ep.alpha, v1, ep.beta * cp[1]);
          }
      }
#if MYD_EP_SHFL
      // Interior units: lanes r < 4 and r >= 4 (lane ^ 16) swap one pair of
      // every two row-fragments so each warp store writes 4 columns x 128
      // contiguous bytes instead of 8 columns x 64: half the cache lines per
      // store instruction, which is what bounds the write-back of a unit.
      if constexpr (FM % 2 == 0) {
        if (c_aligned && sg.m0 + BM <= M && sg.n0 + BN <= N) {
          const bool lo = r < 4;
          const int rowb = row0 + (lo ? 0 : 8), colb = col0 - (lo ? 0 : 4);
          // The next unit's C block (already staged in the ring) is read into
          // each fragment pair right after that pair is stored, so the
          // shared-memory reads overlap the global write-back.
          const uint32_t gn = g + NS;
          const bool pre = has_next && nsg.from_c && !ep.blas;  // the BLAS epilogue starts from 0
          const bool n_inside = CG && pre && c_inside(nsg);
          const int nrow0 = nsg.m0 + wm * WM + 2 * q, ncol0 = nsg.n0 + wn * WN + r;
          if (!CG && pre)
            for (int cs = 0; cs < CS; ++cs) mbar_wait(&full_bar[(gn + cs) % STAGES], ((gn + cs) / STAGES) & 1);
          // write back fragment pair (i, i+1) x j of this unit, then (pre) read
          // the next unit's C into it
          auto ep_pair = [&](int i, int j) {
            const double s0 = lo ? acc[i + 1][j][0] : acc[i][j][0];
            const double s1 = lo ? acc[i + 1][j][1] : acc[i][j][1];
            const double g0 = __shfl_xor_sync(0xffffffffu, s0, 16);
            const double g1 = __shfl_xor_sync(0xffffffffu, s1, 16);
            double *cp = C + (int64_t)(colb + j * 8) * ldc + rowb + i * 8;
            *reinterpret_cast<double2 *>(cp) = lo ? make_double2(acc[i][j][0], acc[i][j][1]) : make_double2(g0, g1);
            *reinterpret_cast<double2 *>(cp + 4 * ldc) =
                lo ? make_double2(g0, g1) : make_double2(acc[i + 1][j][0], acc[i + 1][j][1]);
            if (pre) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if constexpr (CG) {
                  load_c_pair(i + h, j, nrow0, ncol0, n_inside);
                } else {
                  const double2 v = *reinterpret_cast<const double2 *>(&smem[c_index(gn, i + h, j)]);
                  acc[i + h][j][0] = v.x;
                  acc[i + h][j][1] = v.y;
                }
              }
            }
          };
          // Split boundary (full tiles, C from global, the next unit a whole
          // interior tile of >= 2 slabs): write back / reload the first half
          // of the columns (j < FN/2), run the next unit's first slab on that
          // half while the second half is written back and reloaded, then
          // run the same slab on the second half.  Each element still sees
          // its k-steps in ascending order from C, so C is bitwise unchanged;
          // the DMMA pipe works through half of the write-back instead of
          // idling (the boundary is ~7 % of a unit at K = 256).
          // Phase 2 spans SBS slabs (~MYD_SB_KSTEPS k-steps of first-half DMMA
          // work); those slabs stay in the ring until the catch-up has used
          // them.  One slab measured best: 12000^2 x 100 78.0 -> 81.5 %,
          // 8192^2 x 512 93.2 -> 93.8 %, cfg4 93.3 -> 93.8 %, 8192^3
          // 98.27 -> 98.37 %; 2-5 slabs gain less (profiles/r02/split_boundary_r02a.log).
          // (Less than the write-back's share of the boundary: the rest of
          // it -- the reload's latency and the pipeline drain -- stays.)
          constexpr int SBS = MYD_SB_KSTEPS / KSTEPS > 1 ? MYD_SB_KSTEPS / KSTEPS : 1;
          constexpr bool SB_OK = MYD_SPLIT_BOUNDARY && CG && !SKM && FN == 4 && (FM / 2) * 2 == FM && STAGES >= SBS + 2;
          const bool sb = SB_OK && pre && n_inside && nsg.kb == 0 && nsg.ke - nsg.kb >= SBS + 1;
          if (sb) {
            if constexpr (SB_OK) {
              constexpr int FH = FN / 2;
#pragma unroll
              for (int i = 0; i < FM; i += 2)
#pragma unroll
                for (int j = 0; j < FH; ++j) ep_pair(i, j);
              const uint32_t g0 = g + NS;  // the next unit's first slab (CG: no C slots)
              constexpr int NPAIR = (FM / 2) * FH;  // second-half write-back pairs, spread over the k-steps
              constexpr int NK = SBS * KSTEPS;
#pragma unroll
              for (int sl = 0; sl < SBS; ++sl) {
                const uint32_t gs = g0 + sl;
                mbar_wait(&full_bar[gs % STAGES], (gs / STAGES) & 1);
                const double *as0 = smem + (gs % STAGES) * SLOT + a_off;
                const double *bs0 = smem + (gs % STAGES) * SLOT + A_STAGE + b_off;
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk) {
                  double xa[FM], xb[FH];
#pragma unroll
                  for (int i = 0; i < FM; ++i) xa[i] = as0[kk * 4 * AP + i * 8];
#pragma unroll
                  for (int j = 0; j < FH; ++j) xb[j] = bs0[kk * 4 + j * 8 * BP];
#pragma unroll
                  for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < FH; ++j) dmma_884(acc[i][j][0], acc[i][j][1], xb[j], xa[i]);
                  const int ks = sl * KSTEPS + kk;  // (compile-time after unrolling)
#pragma unroll
                  for (int t = ks * NPAIR / NK; t < (ks + 1) * NPAIR / NK; ++t) ep_pair(2 * (t / FH), FH + t % FH);
                }
              }
#pragma unroll
              for (int sl = 0; sl < SBS; ++sl) {
                const uint32_t gs = g0 + sl;
                const double *as0 = smem + (gs % STAGES) * SLOT + a_off;
                const double *bs0 = smem + (gs % STAGES) * SLOT + A_STAGE + b_off;
#pragma unroll
                for (int kk = 0; kk < KSTEPS; ++kk) {
                  double xa[FM], xb[FH];
#pragma unroll
                  for (int i = 0; i < FM; ++i) xa[i] = as0[kk * 4 * AP + i * 8];
#pragma unroll
                  for (int j = 0; j < FH; ++j) xb[j] = bs0[kk * 4 + (FH + j) * 8 * BP];
#pragma unroll
                  for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < FH; ++j) dmma_884(acc[i][FH + j][0], acc[i][FH + j][1], xb[j], xa[i]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[gs % STAGES]);
              }
              kt0 = SBS;
            }
          } else {
#pragma unroll
            for (int i = 0; i < FM; i += 2)
#pragma unroll
              for (int j = 0; j < FN; ++j) ep_pair(i, j);
          }
          if (pre) {
            if constexpr (!CG) {
              __syncwarp();
              if (lane == 0)
                for (int cs = 0; cs < CS; ++cs) mbar_arrive(&empty_bar[(gn + cs) % STAGES]);
            }
            c_loaded = true;
          }
          stored = true;
        }
      }
#endif
      if (!stored)
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          const int row = row0 + i * 8, col = col0 + j * 8;
          if (col >= N || row >= M) continue;
          double *cp = C + (int64_t)col * ldc + row;
          double v0 = acc[i][j][0], v1 = acc[i][j][1];
          const bool pair = row + 1 < M;
          if (pair && (vec_store || (c16 && ((((int64_t)col * ldc + row) & 1) == 0)))) {
            *reinterpret_cast<double2 *>(cp) = make_double2(v0, v1);
          } else {
            cp[0] = v0;
            if (pair) cp[1] = v1;
          }
        }
    }
    KST(seg_ord * 5 + 3);
    g += NS;
    // (a next segment that itself starts from another CTA's partial waits for
    // it: publish first, or the waits would chain from CTA to CTA)
    const bool publish_first = !sg.to_c && !SUM && has_next && !nsg.from_c;
    if (publish_first) publish_partial(sg.slot);
    if (has_next) g = c_loaded ? g + CSR : init_acc(nsg, g);
    if (!sg.to_c && !publish_first) publish_partial(sg.slot);
    KST(seg_ord * 5 + 4);
    ++seg_ord;
    TL_MARK(6);
#ifdef MYD_TIMELINE
    ++unit_ord;
#endif
    cur = ncur;
    sg = nsg;
    have = has_next;
  }
  KST(14);
  if (after_main) asm volatile("griddepcontrol.wait;\n" ::: "memory");
#ifdef MYD_TIMELINE
  if (tid == 0) atomicMax(&g_tl[1], gtimer());
#endif
}

void keep_pool_memory();  // capi.cu

namespace {

int sm_count();

// PDL between consecutive launches (MY_DGEMM_NO_PDL=1 turns it off, for A/B timing).
bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("MY_DGEMM_NO_PDL");
    return !(v && *v && *v != '0');
  }();
  return on;
}

template <int VEC, int BM, int BN, int BK, bool SKM, bool CGT, bool RK, bool RS = false, bool SUM = false,
          bool EDGE = false>
cudaError_t launch_kernel(const Epilogue &ep, unsigned units, int M, int N, int K, const double *A, int64_t lda,
                          const double *B, int64_t ldb, double *C, int64_t ldc, int tiles_m, int tiles_n, int tile0,
                          int edge, int after_main, cudaStream_t st, const StreamK &sk) {
  using namespace fast;
  // The opt-in shared-memory size is a per-device function attribute: set it
  // once per (device, instantiation); racing first calls just set it twice.
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_done.load(std::memory_order_acquire) & bit)) {
    if constexpr (MYD_L2_PERSIST_MB > 0) {  // experiment builds: bound the evict_last (persisting) lines
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)MYD_L2_PERSIST_MB << 20);
      cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(dgemm_fast_kernel<VEC, BM, BN, BK, SKM, CGT, RK, RS, SUM, EDGE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Ring<BM, BN, BK>::BYTES);
    if (e != cudaSuccess) return e;
    attr_done.fetch_or(bit, std::memory_order_release);
  }
  // persistent: at most one CTA per SM, each walking units b, b+grid, ...
  const unsigned grid = std::min<unsigned>(units, (unsigned)sm_count());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = Ring<BM, BN, BK>::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // RS: the round re-alignment needs every CTA resident
  attr[1].val.cooperative = 1;
  cfg.attrs = pdl_enabled() ? attr : attr + 1;
  cfg.numAttrs = (pdl_enabled() ? 1 : 0) + (RS ? 1 : 0);
  cudaError_t e = cudaLaunchKernelEx(&cfg, dgemm_fast_kernel<VEC, BM, BN, BK, SKM, CGT, RK, RS, SUM, EDGE>, M, N, K, A, lda, B, ldb,
                                     C, ldc, tiles_m, tiles_n, tile0, edge, (int)units, after_main, sk, ep);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Full tiles with a 16-byte aligned C run the instantiation that reads C from
// global memory (CGT); any other C (odd ldc, 8-byte aligned view) runs the
// ring-staged one, whose 8-byte staging copies hide the latency scalar global
// loads would expose (16384^2 x 256, ldc odd: 5.43 ms -> 4.45 ms).  A runtime
// switch inside one kernel cost the aligned case 2-10 %.
template <int VEC, int BM, int BN, int BK = fast::default_bk<BM, BN>(), bool SKM = false, bool SUM = false>
cudaError_t launch_one(const Epilogue &ep, unsigned units, int M, int N, int K, const double *A, int64_t lda,
                       const double *B, int64_t ldb, double *C, int64_t ldc, int tiles_m, int tiles_n, int tile0,
                       int edge, int after_main, cudaStream_t st, const StreamK &sk = StreamK{}) {
  const bool c_aligned = (ldc % 2 == 0) && ((uintptr_t)C % 16 == 0);
  // K with a ragged last slab holding at least one all-zero k-step: the RK
  // instantiation skips them -- for every unit shape, so the set of k-steps
  // each element sees (hence C, bitwise, even the sign of a zero) does not
  // depend on the plan or on which kernel a shard's tile lands in.
  const bool rk = MYD_SKIP_ZERO_KSTEPS && K % BK != 0 && BK - K % BK >= 4;
  // partial units worth their own instantiation (see the EDGE staging path)
  // (long-K problems of more waves too: +0.5 % at 4093 x 4099 x 2047 and 5000^2 x 1000, while
  // 6001^2 x 512 loses 0.3 % to the heavier producers, profiles/r02/ab_libs_r02f.log)
  [[maybe_unused]] const bool edge_bulk =
      (M % BM != 0 || N % BN != 0) &&
      (K >= 1024 ||
       (long long)((M + fast::TILE_M - 1) / fast::TILE_M) * ((N + fast::TILE_N - 1) / fast::TILE_N) <=
           (long long)MYD_EDGE_BULK_WAVES * sm_count());
#define MYD_LAUNCH(CGT_, RK_)                                                                                   \
  do {                                                                                                            \
    if constexpr (VEC == 2 && BM != 16 && MYD_EDGE_BULK && !SUM) {                                                \
      if (edge_bulk)                                                                                              \
        return launch_kernel<VEC, BM, BN, BK, SKM, CGT_, RK_, false, SUM, true>(                                  \
            ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st, sk);       \
    }                                                                                                             \
    return launch_kernel<VEC, BM, BN, BK, SKM, CGT_, RK_, false, SUM>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, \
                                                                      tiles_m, tiles_n, tile0, edge, after_main,  \
                                                                      st, sk);                                    \
  } while (0)
  if constexpr (VEC == 2 && BM == 128 && BN == 128) {
    if (c_aligned) {
      if constexpr (BK == 32 && !SKM) {
        if (sk.iters > 0 && sk.flags) {  // round re-alignment (RoundSync)
          cudaError_t e = rk ? launch_kernel<VEC, BM, BN, BK, SKM, true, true, true>(
                                   ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st, sk)
                             : launch_kernel<VEC, BM, BN, BK, SKM, true, false, true>(
                                   ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st, sk);
          if (e == cudaSuccess) return e;
          cudaGetLastError();  // no co-resident launch here: the plain instantiation, without re-alignment
        }
      }
      if (rk) MYD_LAUNCH(true, true);
      MYD_LAUNCH(true, false);
    }
  }
  if (rk) MYD_LAUNCH(false, true);
  MYD_LAUNCH(false, false);
#undef MYD_LAUNCH
}

template <int VEC>
cudaError_t launch_split(const Epilogue &ep, int split, unsigned units, int M, int N, int K, const double *A, int64_t lda,
                         const double *B, int64_t ldb, double *C, int64_t ldc, int tiles_m, int tiles_n, int tile0, int edge,
                         int after_main,
                         cudaStream_t st, const StreamK &rs = StreamK{}) {
  switch (split) {  // units per 128x128 tile
    case 1:
      if constexpr (VEC == 2) {
        if (K >= MYD_BK32_MIN_K)  // long K: deeper slabs, fewer ring handshakes (rs: round re-alignment)
          return launch_one<VEC, 128, 128, 32>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st, rs);
      }
      return launch_one<VEC, 128, 128, 16>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st);
    case 2: return launch_one<VEC, 128, 64>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st);
    case 4: return launch_one<VEC, 128, 32>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st);
    case 16:  // 16x128 units (8 per tile, stacked in m): few-row problems and ragged last tile rows
      return launch_one<VEC, 16, 128, MYD_ROWS16_BK>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st);
    default: return launch_one<VEC, 64, 32>(ep, units, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, tile0, edge, after_main, st);
  }
}

// Full-tile slab depth, as launch_split's case 1 picks it.
template <int VEC>
constexpr int full_bk(int K) {
  return (VEC == 2 && K >= MYD_BK32_MIN_K) ? 32 : 16;
}

inline void keep_pool_memory_fast() { keep_pool_memory(); }

// Stream-K launch over every SM (see the kernel's segment comment) of the
// BM x BN units from unit0 on (unit numbering of the unit-mode kernel with
// tile0 = 0): workspace of one partial unit per CTA plus per-warp flags from
// the stream-ordered pool; the epoch makes stale flags never match.
// One epoch counter for every stream-K launch of the process (all
// instantiations); the flags are also zeroed before every stream-K call, so
// neither an earlier launch's flags nor other data left in pool memory can
// match.
std::atomic<unsigned long long> g_sk_epochs{0};

// Workspace of one stream-K / K-split call: one partial unit per CTA plus
// per-warp flags.  Normally a block owned by the call's stream (up to
// SK_STREAMS streams per device, keyed by cudaStreamGetId, allocated from the
// stream-ordered pool and its flags zeroed on that stream once, never freed): calls on one stream run in order -- a PDL
// successor touches global memory only after its griddepcontrol.wait, i.e.
// after the previous grid has completed -- and every launch has its own epoch,
// so flags left by earlier calls never match and nothing has to be zeroed or
// allocated per call (the memset between two kernels also kept the launch from
// overlapping its predecessor: 896^3 stream-K 59.1 -> 53.6 us, 1280^3
// 138.8 -> 133.8 us, profiles/r02/ksplit_r02b.log).  During stream capture, with more streams
// than slots, or when the allocation fails: a block from the stream-ordered
// pool, flags zeroed by a memset node ahead of the launch, freed after it.
constexpr int SK_STREAMS = 8;
struct SkOwned {
  unsigned long long stream_id = 0;
  void *base = nullptr;
  size_t ctas = 0;
};
struct SkDevice {
  std::mutex mu;
  SkOwned own[SK_STREAMS];
  int n = 0;
};
SkDevice g_sk_dev[64];

struct SkWorkspace {
  void *base = nullptr;  // pooled block (freed by release), else nullptr
  StreamK sk;
  static constexpr size_t part_bytes(size_t G) { return G * fast::CONSUMER_WARPS * 32 * 64 * 8; }
  static constexpr size_t flag_bytes(size_t G) { return G * fast::CONSUMER_WARPS * 8; }
  void point(void *b, size_t G) {
    sk.work = static_cast<double *>(b);
    sk.flags = reinterpret_cast<unsigned long long *>(static_cast<char *>(b) + part_bytes(G));
    sk.epoch = 0x5DA7000000000000ull | (g_sk_epochs.fetch_add(1) + 1);
  }
  bool owned(int G, cudaStream_t st) {
    static const bool off = [] {  // MY_DGEMM_SK_POOLED=1: always the pooled block (A/B timing)
      const char *v = getenv("MY_DGEMM_SK_POOLED");
      return v && *v && *v != '0';
    }();
    if (off) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    unsigned long long id = 0;
    int dev = 0;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone ||
        cudaStreamGetId(st, &id) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
      cudaGetLastError();
      return false;
    }
    SkDevice &d = g_sk_dev[dev];
    std::lock_guard<std::mutex> lock(d.mu);
    for (int i = 0; i < d.n; ++i)
      if (d.own[i].stream_id == id) {
        if (d.own[i].ctas < (size_t)G) return false;
        point(d.own[i].base, d.own[i].ctas);
        return true;
      }
    if (d.n >= SK_STREAMS) return false;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t ctas = (size_t)std::max(G, sms);
    // (stream-ordered allocation and zeroing on the owning stream itself, once: unlike cudaMalloc /
    // cudaMemset they do not disturb a stream capture another thread may have open)
    void *b = nullptr;
    if (cudaMallocAsync(&b, part_bytes(ctas) + flag_bytes(ctas), st) != cudaSuccess ||
        cudaMemsetAsync(static_cast<char *>(b) + part_bytes(ctas), 0, flag_bytes(ctas), st) != cudaSuccess) {
      cudaGetLastError();
      if (b) cudaFreeAsync(b, st);
      return false;
    }
    d.own[d.n++] = SkOwned{id, b, ctas};
    point(b, ctas);
    return true;
  }
  cudaError_t alloc(int G, cudaStream_t st) {
    // (the pool's release threshold is set on a device's first call, here and
    // not only on the pooled branch: that branch is the one stream captures
    // take, and setting a pool attribute inside a capture invalidates it)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) keep_pool_memory_fast();
    cudaGetLastError();
    if (owned(G, st)) return cudaSuccess;
    cudaError_t e = cudaMallocAsync(&base, part_bytes(G) + flag_bytes(G), st);
    if (e != cudaSuccess) return e;
    point(base, G);
    return cudaMemsetAsync(sk.flags, 0, flag_bytes(G), st);
  }
  void release(cudaStream_t st) {
    if (base) cudaFreeAsync(base, st);
    base = nullptr;
  }
};

// Stream-K launch over every SM (see the kernel's segment comment) of the
// BM x BN units from unit0 on (unit numbering of the unit-mode kernel with
// tile0 = 0).
template <int VEC, int BM, int BN, int BK, bool SUM = false>
cudaError_t launch_streamk(const Epilogue &ep, int M, int N, int K, const double *A, int64_t lda, const double *B,
                           int64_t ldb, double *C, int64_t ldc, int tiles_m, int tiles_n, long long unit0,
                           int after_main, cudaStream_t st, StreamK sk) {
  constexpr int PER_TILE = (fast::TILE_M / BM) * (fast::TILE_N / BN);
  const int G = sm_count();
  const int KT = (K + BK - 1) / BK;
  sk.dp_tiles = 0;
  sk.tile0 = unit0;
  sk.iters = ((long long)tiles_m * tiles_n * PER_TILE - unit0) * KT;
  return launch_one<VEC, BM, BN, BK, true, SUM>(ep, (unsigned)G, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0,
                                                after_main, st, sk);
}

// stream-K over units of `split` per tile (1 = full tiles), from unit0 on
template <int VEC>
cudaError_t launch_streamk_split(const Epilogue &ep, int split, int M, int N, int K, const double *A, int64_t lda,
                                 const double *B, int64_t ldb, double *C, int64_t ldc, int tiles_m, int tiles_n,
                                 long long unit0, int after_main, cudaStream_t st, const StreamK &sk) {
  switch (split) {
    case 1:
      if (full_bk<VEC>(K) == 32)
        return launch_streamk<VEC, 128, 128, 32>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, unit0,
                                                 after_main, st, sk);
      return launch_streamk<VEC, 128, 128, 16>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, unit0,
                                               after_main, st, sk);
    case 2:
      return launch_streamk<VEC, 128, 64, fast::default_bk<128, 64>()>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m,
                                                                       tiles_n, unit0, after_main, st, sk);
    case 4:
      return launch_streamk<VEC, 128, 32, fast::default_bk<128, 32>()>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m,
                                                                       tiles_n, unit0, after_main, st, sk);
    default:
      return launch_streamk<VEC, 64, 32, fast::default_bk<64, 32>()>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m,
                                                                     tiles_n, unit0, after_main, st, sk);
  }
}

std::atomic<int> g_max_ctas{0};  // my_dgemm_set_max_ctas: 0 = every SM

// The K-split plan is opt-in: MY_DGEMM_FORCE_KSPLIT per call, or
// MY_DGEMM_KSPLIT=1 in the environment lets the heuristic cost it against the
// plan-invariant plans (off by default: measured, it does not beat them --
// 1024^3 77.7 vs 77.3 us, 1408^3 170.0 vs 172.4, 896^3 60.1 vs 52.4,
// profiles/r02/ksplit_r02c.log -- because writing, re-reading and adding a
// 128 KB accumulator block costs each CTA ~2 us per step, which eats what the
// even split gains, profiles/r02/ksplit_timeline_r02b.log).
bool ksplit_enabled() {
  static const bool on = [] {
    const char *v = getenv("MY_DGEMM_KSPLIT");
    return v && *v && *v != '0';
  }();
  return on;
}

// Round re-alignment of long-K whole-tile launches (MY_DGEMM_ROUND_SYNC=R,
// default MYD_ROUND_SYNC: every R rounds; 0 = off; only K >= 16384, where a
// call lasts long enough for the CTAs to drift): a zeroed counter from the
// stream-ordered pool, passed in the unit-mode launch's unused StreamK fields
// (flags = counter, iters = R, dp_tiles = whole rounds).
int round_sync_rounds() {
  static const int r = [] {
    const char *v = getenv("MY_DGEMM_ROUND_SYNC");
    return v && *v ? atoi(v) : MYD_ROUND_SYNC;
  }();
  return r;
}
struct RoundSync {
  unsigned long long *ctr = nullptr;
  StreamK sk;
  cudaError_t setup(long long units, long long G, bool ragged, int K, cudaStream_t st) {
    const int R = round_sync_rounds();
    if (R <= 0 || ragged || K < 16384 || units / G < 2LL * R) return cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;  // (no cooperative launch inside a capture)
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return cudaSuccess;
    }
    keep_pool_memory_fast();
    cudaError_t e = cudaMallocAsync((void **)&ctr, sizeof(*ctr), st);
    if (e != cudaSuccess) return e;
    sk.flags = ctr;
    sk.iters = R;
    sk.dp_tiles = units / G;
    return cudaMemsetAsync(ctr, 0, sizeof(*ctr), st);
  }
  void release(cudaStream_t st) {
    if (ctr) cudaFreeAsync(ctr, st);
    ctr = nullptr;
  }
};

// SMs the persistent grid may occupy: the device's count, or fewer when the
// caller reserves SMs for concurrent work (e.g. NCCL kernels of an
// overlapped broadcast).  Results do not depend on it.
int sm_count() {
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cached[dev & 63].load(std::memory_order_relaxed);
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cached[dev & 63].store(v, std::memory_order_relaxed);
  }
  const int lim = g_max_ctas.load(std::memory_order_relaxed);
  return (lim > 0 && lim < v) ? lim : v;
}

}  // namespace

int set_max_ctas(int n) { return g_max_ctas.exchange(n); }

// Launch plan.  With G SMs (one persistent CTA each) and T full 128x128
// tiles, T = q*G + r, the candidates are: every tile as a full tile;
// q*G full tiles plus the r leftovers cut into `split` units (128x64,
// 128x32 or 64x32; all 8 consumer warps busy) in a second launch; every tile
// as units.  Ragged last tile column (N mod 128 in 1..64, e.g. cfg3a's
// n = 4099): the column may be kept out of the full-tile raster and run in
// the tail launch as units, only those covering valid columns scheduled.
// Each candidate is costed with whole-call times measured on the B200
// (round 2: tools/unit_model_probe.py, profiles/r02/unit_model_r02a.log): a
// launch of r rounds of 1/s-tile units at depth K takes launch_us(s) +
// r * round_us(s) microseconds (round_us = ideal / e_s + c_s, ideal at
// 128 flop/clk, 1.965 GHz), a tail launch after whole-tile rounds ~16 us, the
// stream-K schedules their own fitted slab factors and fixed costs; the
// cheapest wins (mean regret against the best forced plan ~1.1 % over seeded
// random shapes, tools/planner_regret.py).  A ragged last tile row (M mod 128 in 1..64, and problems of <= 64
// rows) gets the same treatment as a ragged column, with 64x32 or 16x128
// units.  force_split pins the plan (tests and the tuner): 0 = heuristic,
// 1 = full tiles only, 2 / 4 / 8 / 16 = every tile as 128x64 / 128x32 /
// 64x32 / 16x128 units, 32 + s = stream-K over those, 64 + v = the small-block
// kernel.  Every one of these computes bitwise the same C; 48, the opt-in
// K-split plan, is the exception (deterministic, within the tolerance).
double small_cost_us(int v, int M, int N, int K, int G);  // dgemm_small.cu
int small_variants();
cudaError_t launch_dgemm_small(int variant, int M, int N, int K, const double *A, int64_t lda, const double *B,
                               int64_t ldb, double *C, int64_t ldc, cudaStream_t st, const Epilogue &ep, bool vec2);

thread_local std::string *t_plan_out = nullptr;  // my_dgemm_plan_describe's dry run
bool plan_trace_env() {  // MY_DGEMM_PLAN_TRACE=1: print each call's launch plan to stderr
  static const bool on = [] {
    const char *v = getenv("MY_DGEMM_PLAN_TRACE");
    return v && *v && *v != '0';
  }();
  return on;
}
inline bool trace_wanted() { return t_plan_out != nullptr || plan_trace_env(); }

cudaError_t launch_dgemm_fast(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                              double *C, int64_t ldc, cudaStream_t stream, bool force_vec1, int force_split,
                              const Epilogue &ep) {
  using namespace fast;
  // force_split < 0: the heuristic restricted to plan-invariant plans (no
  // K-split); 48: the K-split plan when the shape allows it (else as < 0)
  const bool force_ksplit = force_split == 48;
  const bool allow_ksplit = force_split == 0 && ksplit_enabled();
  if (force_split < 0 || force_ksplit) force_split = 0;
  const int tiles_m = (M + TILE_M - 1) / TILE_M, tiles_n = (N + TILE_N - 1) / TILE_N;
  const long long tiles = (long long)tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL / 8) return cudaErrorInvalidConfiguration;
  const bool vec2 =
      !force_vec1 && (lda % 2 == 0) && (ldb % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  const long long G = sm_count();
  int raster_m = tiles_m, raster_n = tiles_n;  // tile rows / columns in the grouped raster
  int edge = 0;  // edge plans: > 0 valid strips of a separate last tile column, < 0 sub-rows of a last row
  long long q = tiles / G;  // full-tile rounds of the main launch
  int split = 1;            // 1 full tiles; 2 / 4 / 8 units 128x64 / 128x32 / 64x32; 16 units 16x128
  auto per_tile = [](int s) { return s == 16 ? 8 : s; };
  int sk_split = force_split >= 32 ? (force_split == 32 ? 1 : force_split - 32) : 1;  // stream-K unit shape
  bool streamk = force_split >= 32 && force_split < 64 && tiles * sk_split >= G;
  // whole-tile rounds ahead of a full-tile stream-K phase (forced plan 32: all
  // but the last one to two waves; MY_DGEMM_SK_DP_ROUNDS overrides, for probes)
  long long sk_dp_rounds = std::max(0LL, tiles / G - 1);
  // K-split (sum) plan over full tiles, tiles < G (the kernel's segment
  // comment; opt-in, see ksplit_enabled): pieces of a tile's K range on
  // several SMs, partial sums added by the tile's owner.  Needs 16-byte
  // staging (so the slab depth, hence the cut points, depend on K alone) and
  // the whole device (the cut depends on the CTA count).  Cost: ceil(T KT / G)
  // slabs per CTA at the stream-K slab rate, the fixed ramp with the piece
  // boundary, and the owner's fix-up of G / T - 1 partials
  // (tools/ksplit_probe.py, profiles/r02/ksplit_r02c.log).
  const int ks_bk = full_bk<2>(K);
  const long long ks_KT = (K + ks_bk - 1) / ks_bk;
  const bool ks_ok = vec2 && tiles < G && tiles * ks_KT >= 2 * G && tiles * ks_KT < (1LL << 30) &&
                     g_max_ctas.load(std::memory_order_relaxed) == 0;
  bool ksplit = force_ksplit && ks_ok;
  double plan_best = 1e300;  // the heuristic's cost of its persistent-kernel plan (us)
  if (ksplit) {
    q = tiles;
  } else if (force_split >= 64) {
    q = tiles;  // small-block kernel, below
  } else if (force_split >= 32) {
    q = tiles;  // (fewer units than SMs: plain full tiles instead)
  } else if (force_split > 1) {
    split = force_split >= 16 ? 16 : (force_split >= 8 ? 8 : (force_split >= 4 ? 4 : 2));  // every tile as units
    q = 0;
  } else if (force_split == 0) {
    // A launch of r rounds of 1/s-tile units at depth K costs launch_us(s) +
    // r * round_us(s) microseconds: refitted in round 2 on whole calls of
    // exactly r * 148 units, r = 1..8, K = 64..4096 (tools/unit_model_probe.py,
    // profiles/r02/unit_model_r02a.log).  The round-1 model (ideal / e_s + b_s
    // per round, b = 2.8 / 7.2 / 4.4 / 4.0 us, no per-launch term) charged the
    // narrow units' launch ramp to every round -- several rounds of 128x64
    // units at K = 128 looked 40 % dearer than they are (5376 x 1536 x 128:
    // full tiles 93.8 us, the 128x64 units it rejected 78.3 us,
    // profiles/r02/planner_regret_r02a.log) -- and their DMMA rate at long K
    // 3 % better than it is.  16x128 units (LDGSTS-staged) keep the round-1
    // fit on tools/rows16_probe.py and short-K ragged rows: e 0.74, b 2.
    auto ideal_us = [&](int s) { return 2.0 * TILE_M * TILE_N / per_tile(s) * K / 251.5e3; };
    auto round_us = [&](int s) -> double {
      // a ragged last K slab is staged by zero-filling LDGSTS: ~1.7 us per unit
      // (2582 x 1906 x 144 as 128x32 units, 32-deep slabs: 73.7 us against 58.1 modelled)
      const int bk = s == 1 ? (vec2 ? full_bk<2>(K) : full_bk<1>(K))
                            : (s == 2 ? default_bk<128, 64>() : (s == 4 ? default_bk<128, 32>() : (s == 16 ? MYD_ROWS16_BK : default_bk<64, 32>())));
      const double ideal = ideal_us(s) + (K % bk != 0 ? 1.7 : 0.0);
      switch (s) {
        case 1: return ideal / 0.986 + 2.8 + (K < 128 ? 0.05 * (128 - K) : 0.0);
        case 2: return ideal / 0.953 + 1.26;
        case 4: return ideal / 0.957 + 0.86;
        case 16: return ideal / 0.740 + 2.0;
        // (+1 us per round over the fit on whole, balanced rounds: on real shapes 64x32 units
        // come out ~5 % behind it, 1000 x 1100 x 1200: 96.5 us against 91.4 modelled)
        default: return ideal / 0.945 + 1.48 + std::max(0.0, 1.7 - K / 300.0);
      }
    };
    auto launch_us = [&](int s, double r = 2.0) -> double {
      switch (s) {
        case 1: return 11.5;
        case 2: return 7.2;
        case 4: return 6.3;
        case 16: return 0.0;
        // (a single round of 64x32 units ends ~3 us sooner than the fit on 2..8 rounds says: 512^3 13.4 us)
        default: return std::min(r <= 1.0 ? 4.0 : 6.8, 1.0 + K / 40.0);
      }
    };
    // (the stream-K fits below are relative to the round-1 unit work, ideal / e_s)
    auto sk_work_us = [&](int s) {
      return ideal_us(s) / (s == 1 ? 0.990 : (s == 2 ? 0.984 : (s == 4 ? 0.983 : 0.977)));
    };
    auto rounds = [&](long long units) { return (double)((units + G - 1) / G); };
    constexpr double TAIL_LAUNCH_US = 16.0;  // a second (PDL tail) launch after whole-tile rounds
    // (Partial units of a ragged M or N cost what whole ones do since their
    // valid part is staged by bulk copies; with zero-filling LDGSTS they ran
    // 1.3 - 1.7x as long and a one- or two-round call could not hide the one
    // some CTA always got: 506 x 1188 x 1616 as 64x32 units 113 us against 92
    // modelled, profiles/r02/planner_regret_r02b.log.)
    const bool ragged_mn = M % TILE_M != 0 || N % TILE_N != 0;
    double best = launch_us(1) + rounds(tiles) * round_us(1);  // full tiles only
    q = tiles;  // (split == 1: one launch of every tile)
    for (int s : {2, 4, 8}) {
      const double all = launch_us(s, rounds(tiles * s)) + rounds(tiles * s) * round_us(s);
      if (all < best - 1e-9) {
        best = all;
        split = s;
        q = 0;
      }
      const long long q1 = tiles / G, r1 = tiles % G;
      if (q1 > 0 && r1 > 0) {
        const double tail = launch_us(1) + q1 * round_us(1) + rounds(r1 * s) * round_us(s) + TAIL_LAUNCH_US;
        if (tail < best - 1e-9) {
          best = tail;
          split = s;
          q = q1;
        }
      }
    }
    const int rem_n = N % TILE_N;
    // Ragged last tile column (any remainder, also N < 128): kept out of the
    // raster and run as only its valid strips -- round-robin over a raster
    // that includes empty units would pile the valid ones onto a quarter of
    // the CTAs when N < 128 (8192 x 32 x 8192: 573 -> ~150 us).
    if (rem_n >= 1 && tiles_n >= 1) {  // edge column out of the raster
      const long long te = (long long)tiles_m * (tiles_n - 1);
      const long long qe = te / G, re = te % G;
      for (int s : {2, 4, 8}) {
        const int bn = s == 2 ? 64 : 32;
        const int ns = (rem_n + bn - 1) / bn;  // valid strips of the 128x64 / 128x32 / 64x32 units
        const long long nonempty = re * s + (long long)tiles_m * (s == 8 ? 2 : 1) * ns;
        const double cost = (qe > 0 ? launch_us(1) + qe * round_us(1) + TAIL_LAUNCH_US : launch_us(s, rounds(nonempty))) +
                            rounds(nonempty) * round_us(s);
        if (cost < best - 1e-9) {
          best = cost;
          split = s;
          raster_m = tiles_m;
          raster_n = tiles_n - 1;
          edge = ns;
          q = qe;
        }
      }
    }
    // Stream-K: the T*KT (tile, slab) iterations evenly over the SMs, a tile
    // cut between two CTAs finished from the partial the first one leaves
    // (bitwise the uncut chain).  Needs T >= G (a tile is cut at most once).
    // Below one wave of tiles: stream-K over units (>= one unit per CTA, so a
    // unit is cut at most once), when the problem has no ragged edge (empty
    // units would be scheduled, not skipped).
    // Round 2 (workspace owned by the stream, no per-call memset): refitted on
    // 640..1536^3 (tools/midsize_plans.py, profiles/r02/midsize_plans_r02a.log;
    // residuals < 0.6 us): a stream-K slab of 128x64 / 128x32 / 64x32 units
    // costs 1.037 / 1.058 / 1.086 of the whole-unit slab, the call 12.0 / 10.3 /
    // 9.9 us on top.  The same schedule is also costed above one wave of tiles
    // and on ragged problems (every unit of the problem in the stream-K phase:
    // empty units are scheduled and cost their slabs, as modelled; m and n of
    // at least a tile, so most units are whole).
    for (int s : {2, 4, 8}) {
      const long long units_s = tiles * s;
      const int bk = s == 2 ? default_bk<128, 64>() : (s == 4 ? default_bk<128, 32>() : default_bk<64, 32>());
      const long long KT = (K + bk - 1) / bk;
      if (units_s < G || units_s * KT >= (1LL << 30)) continue;
      if (ragged_mn && (M < TILE_M || N < TILE_N)) continue;  // (narrower than a tile: the edge plans)
      const double f = s == 2 ? 1.037 : (s == 4 ? 1.058 : 1.086), fixed = s == 2 ? 12.0 : (s == 4 ? 10.3 : 9.9);
      const double slab_us = f * sk_work_us(s) / (double)KT;
      // (the fit covers 1.3 - 2.9 units per CTA; each further unit boundary ~2 us:
      // 2688 x 4096 x 512 as 128x64 units 345.8 us, 2304^3 709.5 us)
      const double cost = (double)((units_s * KT + G - 1) / G) * slab_us + fixed +
                          2.0 * std::max(0.0, (double)units_s / (double)G - 2.0);
      if (cost < best - 1e-9) {
        best = cost;
        streamk = true;
        sk_split = s;
      }
    }
    // Data-parallel rounds for all but the last (one to two waves of tiles).
    // Either every tile in the stream-K phase (no whole-tile rounds), or all
    // but the last one to two waves as whole tiles: the stream-K phase runs
    // ~2 % slower per slab than whole tiles, but following a whole-tile launch
    // costs it ~17 us (the whole-tile launch's own 11.5 us and ~5 us of
    // hand-over; refit on 1664..3072^3, profiles/r02/midsize_plans_r02a.log:
    // the round-1 model was 20 us under wherever there were whole-tile rounds
    // and 5.5 us under where there were none).  A tile
    // boundary inside the phase costs ~3.2 us (no split boundary there), which
    // is what keeps short-K problems on whole-tile rounds (cfg4 with every
    // tile in the phase: 4.05 ms vs 3.93 ms).
    if (tiles >= G && tiles % G != 0) {
      const int bk = vec2 ? full_bk<2>(K) : full_bk<1>(K);
      const long long KT = (K + bk - 1) / bk;
      const double slab_us = 1.02 * sk_work_us(1) / (double)KT;
      for (long long d : {0LL, tiles / G - 1}) {
        const long long sk_tiles = tiles - d * G;
        if (sk_tiles * KT >= (1LL << 30)) continue;
        // (every tile in the phase only on 32-deep slabs, where it was fitted: at K = 256 .. 512 the
        // model is 10 - 20 us under, 5888 x 2944 x 256: 293 us against 282 modelled)
        if (d == 0 && tiles / G - 1 > 0 && bk < 32) continue;
        const double cost = (d > 0 ? launch_us(1) + (double)d * round_us(1) + 5.0 : 0.0) +
                            (double)((sk_tiles * KT + G - 1) / G) * slab_us + 12.0 +
                            3.2 * (double)sk_tiles / (double)G;
        if (cost < best - 1e-9) {
          best = cost;
          streamk = true;
          sk_split = 1;
          sk_dp_rounds = d;
        }
      }
    }
    const int rem_m = M % TILE_M;
    if (rem_m >= 1) {  // ragged last tile row (or a problem < 128 rows) out of the raster
      const long long te = (long long)(tiles_m - 1) * tiles_n;
      const long long qe = te / G, re = te % G;
      for (int s : {8, 16}) {
        // valid sub-rows: 64x32 units (x 4 strips per tile column) or 16x128 units
        const int ms = s == 8 ? (rem_m + 63) / 64 : (rem_m + 15) / 16;
        const long long nonempty = re * per_tile(s) + (long long)tiles_n * ms * (s == 8 ? 4 : 1);
        const double cost = (qe > 0 ? launch_us(1) + qe * round_us(1) + TAIL_LAUNCH_US : launch_us(s, rounds(nonempty))) +
                            rounds(nonempty) * round_us(s);
        if (cost < best - 1e-9) {
          best = cost;
          split = s;
          raster_m = tiles_m - 1;
          raster_n = tiles_n;
          edge = -ms;
          q = qe;
          streamk = false;
        }
      }
    }
    if (allow_ksplit && ks_ok) {
      const double slab_us = 1.02 * sk_work_us(1) / (double)ks_KT;
      const double cost = (double)((tiles * ks_KT + G - 1) / G) * slab_us + 3 * 2.8 + 8.0 +
                          MYD_KSPLIT_FIXUP_US * ((double)G / (double)tiles);
      if (cost < best - 1e-9) {
        best = cost;
        ksplit = true;
        streamk = false;
      }
    }
    plan_best = best;
  }
  // Small-block kernel (dgemm_small.cu): below a few waves of units, CTAs
  // of 16x16 .. 64x64 blocks with several per SM beat the persistent grid's
  // few long unit chains; bitwise the same C.  force_split 64 + v pins
  // variant v (64: the cheapest variant by the model).
  int small_v = 0;
  double small_us = -1.0;  // the small-block kernel's cheapest variant by its model (trace / plan_describe)
  if (trace_wanted() && force_split == 0 && !force_ksplit) {
    for (int v = 1; v <= small_variants(); ++v) {
      const double c = small_cost_us(v, M, N, K, (int)G);
      if (small_us < 0 || c < small_us) small_us = c;
    }
  }
  if (force_split >= 64) {
    small_v = force_split - 64;
    if (small_v == 0) {
      double sbest = 1e300;
      for (int v = 1; v <= small_variants(); ++v) {
        const double c = small_cost_us(v, M, N, K, (int)G);
        if (c < sbest) sbest = c, small_v = v;
      }
    }
  } else if (force_split == 0 && !force_ksplit && tiles <= 2 * G && g_max_ctas.load(std::memory_order_relaxed) == 0) {
    // (not under an SM cap: its grid is the block count, not a persistent
    // grid the cap could bound; results do not depend on the choice)
    double sbest = plan_best;
    for (int v = 1; v <= small_variants(); ++v) {
      const double c = small_cost_us(v, M, N, K, (int)G);
      if (c < sbest - 1e-9) sbest = c, small_v = v;
    }
  }
  const bool trace = plan_trace_env();
  if (trace || t_plan_out) {
    // (a full-tile stream-K call: the whole-tile rounds it will actually run)
    const long long dp_shown = streamk && sk_split == 1 ? sk_dp_rounds : 0;
    char line[320];
    snprintf(line, sizeof line,
             "m=%d n=%d k=%d tiles=%lldx%d %s split=%d sk_split=%d sk_dp_rounds=%lld q=%lld raster=%dx%d edge=%d small=%d "
             "model_us=%.1f small_us=%.1f",
             M, N, K, (long long)tiles_m, tiles_n,
             small_v ? "small" : (ksplit ? "K-split" : (streamk ? "stream-K" : "units")), split, sk_split, dp_shown, q,
             raster_m, raster_n, edge, small_v, plan_best < 1e299 ? plan_best : -1.0, small_us);
    if (trace && !t_plan_out) fprintf(stderr, "my_dgemm plan: %s\n", line);
    if (t_plan_out) {  // my_dgemm_plan_describe: the plan only, nothing is launched
      *t_plan_out = line;
      return cudaSuccess;
    }
  }
  if (small_v > 0) return launch_dgemm_small(small_v, M, N, K, A, lda, B, ldb, C, ldc, stream, ep, vec2);
  if (ksplit) {
    SkWorkspace ws;
    cudaError_t e = ws.alloc((int)G, stream);
    if (e == cudaSuccess)
      e = ks_bk == 32 ? launch_streamk<2, 128, 128, 32, true>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0,
                                                              stream, ws.sk)
                      : launch_streamk<2, 128, 128, 16, true>(ep, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0,
                                                              stream, ws.sk);
    ws.release(stream);
    return e;
  }
  if (streamk) {
    SkWorkspace ws;
    cudaError_t e = ws.alloc((int)G, stream);
    if (e != cudaSuccess) {
      ws.release(stream);
      return e;
    }
    if (sk_split > 1) {
      e = vec2 ? launch_streamk_split<2>(ep, sk_split, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0, stream,
                                         ws.sk)
               : launch_streamk_split<1>(ep, sk_split, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0, stream,
                                         ws.sk);
      ws.release(stream);
      return e;
    }
    // whole-tile rounds for all but the last one-to-two waves in the unit-mode
    // kernel, then the stream-K phase as a tail launch (its own tiles only)
    static const long long dp_env = [] {
      const char *v = getenv("MY_DGEMM_SK_DP_ROUNDS");
      return v && *v ? atoll(v) : -1LL;
    }();
    if (dp_env >= 0) sk_dp_rounds = std::min(dp_env, std::max(0LL, tiles / G - 1));
    if ((tiles - sk_dp_rounds * G) * (long long)(K / 16 + 1) >= (1LL << 30)) sk_dp_rounds = std::max(0LL, tiles / G - 1);
    const long long dp_tiles = sk_dp_rounds * G;
    RoundSync rsync;
    if (dp_tiles > 0) {
      e = rsync.setup(dp_tiles, G, M % TILE_M != 0 || N % TILE_N != 0, K, stream);
      if (e == cudaSuccess)
        e = vec2 ? launch_split<2>(ep, 1, (unsigned)dp_tiles, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0, 0,
                                   stream, rsync.sk)
                 : launch_split<1>(ep, 1, (unsigned)dp_tiles, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, 0, 0, 0,
                                   stream, rsync.sk);
    }
    rsync.release(stream);
    if (e == cudaSuccess)
      e = vec2 ? launch_streamk_split<2>(ep, 1, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, dp_tiles,
                                         dp_tiles > 0, stream, ws.sk)
               : launch_streamk_split<1>(ep, 1, M, N, K, A, lda, B, ldb, C, ldc, tiles_m, tiles_n, dp_tiles,
                                         dp_tiles > 0, stream, ws.sk);
    ws.release(stream);
    return e;
  }
  const long long raster_tiles = (long long)raster_m * raster_n;
  const long long main_tiles = split == 1 ? tiles : q * G;
  cudaError_t e = cudaSuccess;
  if (main_tiles > 0)
    e = vec2 ? launch_split<2>(ep, 1, (unsigned)main_tiles, M, N, K, A, lda, B, ldb, C, ldc, raster_m, raster_n, 0, 0,
                               0, stream)
             : launch_split<1>(ep, 1, (unsigned)main_tiles, M, N, K, A, lda, B, ldb, C, ldc, raster_m, raster_n, 0, 0,
                               0, stream);
  if (e != cudaSuccess || split == 1) return e;
  long long edge_units = 0;
  if (edge > 0) edge_units = (long long)tiles_m * (split == 8 ? 2 : 1) * edge;
  if (edge < 0) edge_units = (long long)tiles_n * (-edge) * (split == 8 ? 4 : 1);
  const long long raster_left = edge == 0 ? tiles - main_tiles : raster_tiles - main_tiles;
  const unsigned units = (unsigned)(raster_left * per_tile(split) + edge_units);
  return vec2 ? launch_split<2>(ep, split, units, M, N, K, A, lda, B, ldb, C, ldc, raster_m, raster_n,
                                (int)main_tiles, edge, main_tiles > 0, stream)
              : launch_split<1>(ep, split, units, M, N, K, A, lda, B, ldb, C, ldc, raster_m, raster_n,
                                (int)main_tiles, edge, main_tiles > 0, stream);
}

struct SmallGeo {
  int bm = 0, bn = 0, bk = 0, stages = 0;
};
SmallGeo small_geo(int v);  // dgemm_small.cu

// Blocking parameters of a launch plan (my_dgemm_plan_geometry).
bool plan_geometry(int plan, int K, bool vec2, int &bm, int &bn, int &bk, int &stages) {
  using namespace fast;
  if (plan >= 65) {
    const SmallGeo g = small_geo(plan - 64);
    bm = g.bm, bn = g.bn, bk = g.bk, stages = g.stages;
    return g.bm != 0;
  }
  const int s = plan >= 32 ? (plan == 32 ? 1 : plan - 32) : (plan == 0 ? 1 : plan);
  switch (s) {
    case 1:
      if (vec2 && K >= MYD_BK32_MIN_K) {
        bm = 128, bn = 128, bk = 32, stages = Ring<128, 128, 32>::STAGES;
      } else {
        bm = 128, bn = 128, bk = 16, stages = Ring<128, 128, 16>::STAGES;
      }
      return true;
    case 2: bm = 128, bn = 64, bk = Ring<128, 64>::BK, stages = Ring<128, 64>::STAGES; return true;
    case 4: bm = 128, bn = 32, bk = Ring<128, 32>::BK, stages = Ring<128, 32>::STAGES; return true;
    case 8: bm = 64, bn = 32, bk = Ring<64, 32>::BK, stages = Ring<64, 32>::STAGES; return true;
    case 16:
      if (plan >= 32) return false;
      bm = 16, bn = 128, bk = MYD_ROWS16_BK, stages = Ring<16, 128, MYD_ROWS16_BK>::STAGES;
      return true;
    default: return false;
  }
}

}  // namespace myd

extern "C" __attribute__((visibility("default"))) int my_dgemm_plan_geometry(int plan, int k, int vec2, int *bm,
                                                                             int *bn, int *bk, int *stages) {
  int a = 0, b = 0, c = 0, d = 0;
  if (!myd::plan_geometry(plan, k, vec2 != 0, a, b, c, d)) return -1;
  if (bm) *bm = a;
  if (bn) *bn = b;
  if (bk) *bk = c;
  if (stages) *stages = d;
  return 0;
}

// The tiled path's launch plan for a shape, as text, without launching anything
// (no GPU needed: the planner is host code; without a device it plans for 148
// SMs).  plan: 0 the heuristic (what a default call runs, tuned plans aside),
// -1 the heuristic kept to plan-invariant plans, else a pinned plan id.
extern "C" __attribute__((visibility("default"))) int my_dgemm_plan_describe(int m, int n, int k, int lda, int ldb,
                                                                             int ldc, int plan, char *buf, int len) {
  if (m < 1 || n < 1 || k < 1 || lda < m || ldb < k || ldc < m || !buf || len < 1) return -1;
  std::string out;
  myd::t_plan_out = &out;
  const cudaError_t e = myd::launch_dgemm_fast(m, n, k, nullptr, lda, nullptr, ldb, nullptr, ldc, nullptr, false, plan,
                                               myd::Epilogue{});
  myd::t_plan_out = nullptr;
  cudaGetLastError();
  if (e != cudaSuccess) return -2;
  snprintf(buf, (size_t)len, "%s", out.c_str());
  return 0;
}

#ifdef MYD_TIMELINE
extern "C" __attribute__((visibility("default"))) void my_dgemm_timeline(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, myd::g_tl, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {~0ull};
    cudaMemcpyToSymbol(myd::g_tl, z, sizeof z);
  }
}
#endif
#ifdef MYD_KS_TIMELINE
extern "C" __attribute__((visibility("default"))) void my_dgemm_ks_timeline(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, myd::g_kst, sizeof(unsigned long long) * 160 * 16);
  if (reset) {
    static unsigned long long z[160 * 16];
    cudaMemcpyToSymbol(myd::g_kst, z, sizeof z);
  }
}
#endif
#ifdef MYD_FAST_PROFILE
extern "C" __attribute__((visibility("default"))) void my_dgemm_fast_profile(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, myd::g_fast_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(myd::g_fast_prof, z, sizeof z);
  }
}
#endif
