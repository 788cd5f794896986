// dgemm_skinny.cu -- the HBM-bound shapes of the my_dgemm path (sm_100a):
//   * n == 1 (cfg 3c): C(:,0) += A * B(:,0)          bytes 8(mk + k + 2m)
//   * 2 <= n <= 16:    C(:,0:n) += A * B(:,0:n)      bytes 8(mk + kn + 2mn)
//   * 2 <= m <= 16:    C(0:m,:) += A(0:m,:) * B      bytes 8(mk + kn + 2mn)
//   * m == 1 (cfg 3b): C(0,:) += A(0,:) * B          bytes 8(k + kn + 2n)
// Each streams the big operand exactly once at full width, accumulates with
// FMA and reduces partial sums in a fixed order (the few-column kernel's k
// split adds its per-CTA partials in chunk order in the last CTA of a row
// block), so results are deterministic run to run.  The reference computes these
// shapes with the same five-loop code as every other shape
// (goto.py:187-239); on the GPU they are bandwidth problems, not DMMA ones.
#include <algorithm>
#include <atomic>
#include <cstdlib>

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
// 2 <= n <= NC (a few right-hand sides: tall-skinny block updates).  The n == 1
// kernel widened: a thread owns ROWS rows (32 apart, so every warp load is a
// coalesced 256-byte column segment of A) and NC accumulators per row, so
// each warp-uniform B(p, j) load (an L1 broadcast) feeds ROWS FMAs; A is
// streamed once, 2n flop per 8 bytes.  Slice partials meet in shared memory
// and are added in warp order per element.  HBM-bound up to n = 16
// (4 flop/B); the tiled kernel would waste 1 - n/32 of every unit.
// ---------------------------------------------------------------------------
template <int NC, int ROWS, int WARPS, int KW>
__global__ void __launch_bounds__(32 * WARPS)
    gemm_nsmall_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                       int64_t ldb, double *__restrict__ C, int64_t ldc, Epilogue ep, int kchunk,
                       double *__restrict__ work, unsigned *__restrict__ counters) {
  constexpr int KS = WARPS * KW;               // k per staged sub-chunk (warp w: KW of them)
  extern __shared__ double part[];             // [WARPS][ROWS * NC][32]; first 2 x KS x NC: B stages
  double *bst = part;                          // B(p, 0..NC) rows of the current sub-chunk, 2 buffers
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row0 = blockIdx.x * 32 * ROWS + lane;  // rows row0 + 32 r
  const int ks = blockIdx.y, nks = gridDim.y;     // this CTA's k-chunk
  const int kb = ks * kchunk, ke = min(K, kb + kchunk);
  double acc[ROWS][NC];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[r][j] = 0.0;
  const double *a = A + row0;
  bool ok[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) ok[r] = row0 + 32 * r < M;
  // stage B(s .. s+KS, 0..N) into buffer `buf` (zeros past K / N)
  auto stage = [&](int s, int buf) {
    for (int t = threadIdx.x; t < KS * NC; t += 32 * WARPS) {
      const int pp = t % KS, j = t / KS, p = s + pp;
      bst[(buf * KS + pp) * NC + j] = (p < ke && j < N) ? __ldg(B + (int64_t)j * ldb + p) : 0.0;
    }
  };
  int buf = 0;
  stage(kb, 0);
  __syncthreads();
  // A values of the warp's KW k-steps: for NC >= 8 loaded one sub-chunk
  // ahead, so each warp keeps a sub-chunk of HBM loads in flight while it
  // computes (for fewer columns the extra registers cost more occupancy than
  // the prefetch gains; tools/nsmall_probe.py)
  constexpr bool PREFETCH = NC >= 8;
  double av[KW][ROWS], an[KW][ROWS];
  auto load_a = [&](int s, double (&dst)[KW][ROWS]) {
    const int pw = s + warp * KW;
#pragma unroll
    for (int u = 0; u < KW; ++u)
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
        dst[u][r] = (ok[r] && pw + u < ke) ? __ldcs(a + (int64_t)(pw + u) * lda + 32 * r) : 0.0;
  };
  load_a(kb, av);
  for (int s = kb; s < ke; s += KS, buf ^= 1) {
    if (s + KS < ke) {
      stage(s + KS, buf ^ 1);  // next sub-chunk's B, behind this one's FMAs
      if constexpr (PREFETCH) load_a(s + KS, an);
    }
#pragma unroll
    for (int u = 0; u < KW; ++u) {
      const double *bp = bst + (buf * KS + warp * KW + u) * NC;
#pragma unroll
      for (int j = 0; j < NC; j += 2) {
        const double2 bv = *reinterpret_cast<const double2 *>(bp + j);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          acc[r][j] = fma(av[u][r], bv.x, acc[r][j]);
          acc[r][j + 1] = fma(av[u][r], bv.y, acc[r][j + 1]);
        }
      }
    }
    __syncthreads();  // buffer `buf` free, `buf ^ 1` complete
    if constexpr (PREFETCH) {
#pragma unroll
      for (int u = 0; u < KW; ++u)
#pragma unroll
        for (int r = 0; r < ROWS; ++r) av[u][r] = an[u][r];
    } else if (s + KS < ke) {
      load_a(s + KS, av);
    }
  }
  // partials of the WARPS warps per element (the B stages are no longer needed)
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int j = 0; j < NC; ++j) part[((warp * ROWS + r) * NC + j) * 32 + lane] = acc[r][j];
  __syncthreads();
  // element e = (r, j) of this CTA's ROWS x n block: warps take elements round-robin
  if (nks == 1) {
    for (int e = warp; e < ROWS * N; e += WARPS) {
      const int r = e / N, j = e % N, row = row0 + 32 * r;
      if (row >= M) continue;
      double *cp = C + (int64_t)j * ldc + row;
      double s = ep.blas ? 0.0 : *cp;
      for (int w = 0; w < WARPS; ++w) s += part[((w * ROWS + r) * NC + j) * 32 + lane];
      if (ep.blas) s = ep.beta == 0.0 ? ep.alpha * s : fma(ep.alpha, s, ep.beta * *cp);
      *cp = s;
    }
    return;
  }
  // k split over nks CTAs: each writes its partial block to work[ks][j][row];
  // the last CTA of the row block (counter) adds C + partial_0 + ... in order.
  for (int e = warp; e < ROWS * N; e += WARPS) {
    const int r = e / N, j = e % N, row = row0 + 32 * r;
    if (row >= M) continue;
    double s = 0.0;
    for (int w = 0; w < WARPS; ++w) s += part[((w * ROWS + r) * NC + j) * 32 + lane];
    work[((int64_t)ks * N + j) * M + row] = s;
  }
  __threadfence();
  __syncthreads();
  __shared__ unsigned last;
  if (threadIdx.x == 0) last = atomicAdd(&counters[blockIdx.x], 1u) == (unsigned)(nks - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int e = warp; e < ROWS * N; e += WARPS) {
    const int r = e / N, j = e % N, row = row0 + 32 * r;
    if (row >= M) continue;
    double *cp = C + (int64_t)j * ldc + row;
    double s = ep.blas ? 0.0 : *cp;
    for (int q = 0; q < nks; ++q) s += __ldcg(&work[((int64_t)q * N + j) * M + row]);
    if (ep.blas) s = ep.beta == 0.0 ? ep.alpha * s : fma(ep.alpha, s, ep.beta * *cp);
    *cp = s;
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0;  // ready for the next call's reuse
}

// ---------------------------------------------------------------------------
// 2 <= m <= MC (a few rows: wide-short updates).  B is the big operand, k
// contiguous per column: each warp owns one column at a time and streams it
// with coalesced lane-strided loads (two k per lane per step); the m rows of
// A for the current k-chunk sit in shared memory ([i][p], conflict-free), so
// every B value feeds m FMAs.  Lane partials are reduced by shuffles in a
// fixed tree order, per row.  A chunk is re-read from L2 by every CTA
// (m * K * 8 bytes, small); B is read once.
// ---------------------------------------------------------------------------
template <int MC, int MAXC, int WARPS, int KC>
__global__ void __launch_bounds__(32 * WARPS)
    gemm_msmall_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                       int64_t ldb, double *__restrict__ C, int64_t ldc, Epilogue ep) {
  extern __shared__ double as[];  // [MC][KC]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this CTA's columns: j0 + warp, j0 + warp + WARPS, ... (COLS per warp)
  const int64_t cols_per_cta = (int64_t)WARPS * ((N + (int64_t)gridDim.x * WARPS - 1) / ((int64_t)gridDim.x * WARPS));
  const int64_t j_begin = (int64_t)blockIdx.x * cols_per_cta, j_end = min((int64_t)N, j_begin + cols_per_cta);
  const int ncols = (int)((cols_per_cta + WARPS - 1) / WARPS);
  for (int c0 = 0; c0 < ncols; c0 += MAXC) {
    double acc[MAXC][MC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
      for (int i = 0; i < MC; ++i) acc[c][i] = 0.0;
    for (int kb = 0; kb < K; kb += KC) {
      const int kc = min(KC, K - kb);
      __syncthreads();  // previous chunk consumed
      for (int t = threadIdx.x; t < MC * KC; t += 32 * WARPS) {
        const int i = t / KC, p = t % KC;
        as[t] = (i < M && p < kc) ? __ldg(A + (int64_t)(kb + p) * lda + i) : 0.0;
      }
      __syncthreads();
      // every A value read from shared memory feeds MAXC columns; UNROLL k
      // steps of B loads are issued before their FMAs
      const double *bc[MAXC];
      bool live[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int64_t j = j_begin + warp + (int64_t)(c0 + c) * WARPS;
        live[c] = j < j_end;
        bc[c] = B + (live[c] ? j : 0) * ldb + kb;
      }
      constexpr int UNROLL = MC <= 4 ? 8 : 4;  // B loads in flight per column (tools/msmall_variants.sh)
      int p = lane;
      for (; p + 32 * (UNROLL - 1) < kc; p += 32 * UNROLL) {
        double bv[UNROLL][MAXC];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
          for (int c = 0; c < MAXC; ++c) bv[u][c] = live[c] ? __ldcs(bc[c] + p + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
          for (int i = 0; i < MC; ++i) {
            const double av = as[i * KC + p + 32 * u];
#pragma unroll
            for (int c = 0; c < MAXC; ++c) acc[c][i] = fma(av, bv[u][c], acc[c][i]);
          }
      }
      for (; p < kc; p += 32) {
        double bv[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) bv[c] = live[c] ? __ldcs(bc[c] + p) : 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          const double av = as[i * KC + p];
#pragma unroll
          for (int c = 0; c < MAXC; ++c) acc[c][i] = fma(av, bv[c], acc[c][i]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int64_t j = j_begin + warp + (int64_t)(c0 + c) * WARPS;
#pragma unroll
      for (int i = 0; i < MC; ++i) {
        double v = acc[c][i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        acc[c][i] = v;
      }
      if (j < j_end && lane < M && lane < MC) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i)
          if (i == lane) v = acc[c][i];
        double *cp = C + j * ldc + lane;
        double s = ep.blas ? 0.0 : *cp;
        s += v;
        if (ep.blas) s = ep.beta == 0.0 ? ep.alpha * v : fma(ep.alpha, v, ep.beta * *cp);
        *cp = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 2 <= m <= 8*MT with a wide B (few rows on the FP64 tensor path).  B is the
// big operand and streams once from HBM straight into DMMA fragments: a CTA
// owns 8*CT columns, its WARPS warps split k into contiguous slices of k4
// groups, and per k4 group a warp loads CT B fragments (8 columns x 32
// contiguous bytes: full sectors, evict-first) and MT A fragments (8 rows x 4
// k; A is m*k*8 bytes and stays in L2) and issues CT*MT DMMA.8x8x4 computing
// the C^T block (B^T A^T).  The main loop touches no shared memory and keeps
// U k4 groups of loads in flight per warp, so the SM is bound by HBM, not by
// operand staging (the FMA kernel above is bound by its shared-memory A reads
// from m = 8 on).  Out-of-range columns / rows read a clamped (valid) address
// and are never stored; the partials of the WARPS slices meet in shared
// memory and are added in warp order, then onto C.  The per-element order
// depends only on K, so C is bitwise invariant to any split of the columns.
// ---------------------------------------------------------------------------
template <int MT, int CT, int WARPS, int U, bool VB>
__global__ void __launch_bounds__(32 * WARPS)
    gemm_rows_dmma_kernel(int M, int N, int K, const double *__restrict__ A, int64_t lda,
                          const double *__restrict__ B, int64_t ldb, double *__restrict__ C, int64_t ldc,
                          Epilogue ep) {
  static_assert(!VB || U % 2 == 0, "16-byte B loads take k in pairs");
  extern __shared__ double part[];  // [WARPS][8*CT columns][8*MT rows]
  constexpr int NB = 8 * CT, MB = 8 * MT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;  // fragment row (a column j of C, or a row i) and k in the group
  const int64_t j0 = (int64_t)blockIdx.x * NB;
  const int G = (K + 3) >> 2, per = (G + WARPS - 1) / WARPS;
  const int g0 = min(G, warp * per), g1 = min(G, g0 + per), gfull = min(g1, K >> 2);
  const double *bp[CT];
  const double *ap[MT];
#pragma unroll
  for (int ct = 0; ct < CT; ++ct) bp[ct] = B + min(j0 + 8 * ct + r, (int64_t)N - 1) * ldb;
#pragma unroll
  for (int rt = 0; rt < MT; ++rt) ap[rt] = A + min(8 * rt + r, M - 1);
  double acc[MT][CT][2];
#pragma unroll
  for (int rt = 0; rt < MT; ++rt)
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) acc[rt][ct][0] = acc[rt][ct][1] = -0.0;  // the additive identity: -0 sums stay -0
  // Main loop: batches of U full k4 groups (4U consecutive k).  Within a
  // batch, slot q of DMMA u holds k = k0 + U q + u, so a lane's U B values
  // of a column are contiguous (VB: U/2 16-byte loads) and a column's 4U
  // values are one contiguous 32U-byte run per warp batch.
  int g = g0;
  for (; g + U <= gfull; g += U) {
    const int64_t k0 = 4 * (int64_t)g + U * q;
    double fb[U][CT], fa[U][MT];
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) {
      if constexpr (VB) {
#pragma unroll
        for (int u = 0; u < U; u += 2) {
          const double2 v = __ldcs(reinterpret_cast<const double2 *>(bp[ct] + k0 + u));
          fb[u][ct] = v.x;
          fb[u + 1][ct] = v.y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) fb[u][ct] = __ldcs(bp[ct] + k0 + u);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int rt = 0; rt < MT; ++rt) fa[u][rt] = __ldg(ap[rt] + (k0 + u) * lda);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int ct = 0; ct < CT; ++ct)
#pragma unroll
        for (int rt = 0; rt < MT; ++rt) dmma_884(acc[rt][ct][0], acc[rt][ct][1], fb[u][ct], fa[u][rt]);
  }
  for (; g < g1; ++g) {
    const bool kv = 4 * g + q < K;  // only the last group of k can be partial
    double fb[CT], fa[MT];
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) fb[ct] = kv ? __ldcs(bp[ct] + 4 * g + q) : 0.0;
#pragma unroll
    for (int rt = 0; rt < MT; ++rt) fa[rt] = kv ? __ldg(ap[rt] + (int64_t)(4 * g + q) * lda) : -0.0;  // (+0)(-0) = -0
#pragma unroll
    for (int ct = 0; ct < CT; ++ct)
#pragma unroll
      for (int rt = 0; rt < MT; ++rt) dmma_884(acc[rt][ct][0], acc[rt][ct][1], fb[ct], fa[rt]);
  }
  // lane holds C[i = 8rt + 2q + {0,1}][j = j0 + 8ct + r]
  double *pw = part + (size_t)warp * NB * MB;
#pragma unroll
  for (int ct = 0; ct < CT; ++ct)
#pragma unroll
    for (int rt = 0; rt < MT; ++rt)
      *reinterpret_cast<double2 *>(pw + (8 * ct + r) * MB + 8 * rt + 2 * q) =
          make_double2(acc[rt][ct][0], acc[rt][ct][1]);
  __syncthreads();
  for (int e = threadIdx.x; e < NB * MB; e += 32 * WARPS) {
    const int i = e % MB;
    const int64_t j = j0 + e / MB;
    if (i >= M || j >= N) continue;
    double s = part[e];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) s += part[(size_t)w * NB * MB + e];
    double *cp = C + j * ldc + i;
    if (!ep.blas)
      *cp = *cp + s;
    else
      *cp = ep.beta == 0.0 ? ep.alpha * s : fma(ep.alpha, s, ep.beta * *cp);
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

int sm_count_skinny() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}

cudaError_t launch_gemv_n1(int M, int K, const double *A, int64_t lda, const double *b, double *C,
                           cudaStream_t stream, const Epilogue &ep) {
  gemv_n1_kernel<MYD_N1_WARPS, MYD_N1_UNROLL><<<(M + 31) / 32, 32 * MYD_N1_WARPS, 0, stream>>>(M, K, A, lda, b, C, ep);
  count_launch();
  return cudaGetLastError();
}

void keep_pool_memory();
int sm_count_skinny();

namespace {
template <int NC, int ROWS, int WARPS, int KW>
cudaError_t launch_nsmall_t(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                            double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  constexpr size_t part_bytes = (size_t)WARPS * ROWS * NC * 32 * 8, stage_bytes = (size_t)2 * WARPS * KW * NC * 8;
  constexpr size_t smem = part_bytes > stage_bytes ? part_bytes : stage_bytes;
  if constexpr (smem > 48 * 1024) {
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(gemm_nsmall_kernel<NC, ROWS, WARPS, KW>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_done.fetch_or(bit, std::memory_order_release);
    }
  }
  // Enough CTAs to keep every SM streaming: split k (chunks of >= 512) when
  // the row blocks alone do not cover 2 CTAs per SM.
  const int row_blocks = (M + 32 * ROWS - 1) / (32 * ROWS);
  const int want = (2 * sm_count_skinny() + row_blocks - 1) / row_blocks;
  const int nks = std::max(1, std::min({want, (K + 511) / 512, 64}));
  const int kchunk = (K + nks - 1) / nks;
  double *work = nullptr;
  unsigned *counters = nullptr;
  if (nks > 1) {
    keep_pool_memory();
    cudaError_t e = cudaMallocAsync((void **)&work, (size_t)nks * N * M * 8 + (size_t)row_blocks * 4 + 16, stream);
    if (e != cudaSuccess) return e;
    counters = reinterpret_cast<unsigned *>(work + (size_t)nks * N * M);
    if ((e = cudaMemsetAsync(counters, 0, (size_t)row_blocks * 4, stream)) != cudaSuccess) return e;
  }
  gemm_nsmall_kernel<NC, ROWS, WARPS, KW><<<dim3(row_blocks, nks), 32 * WARPS, smem, stream>>>(
      M, N, K, A, lda, B, ldb, C, ldc, ep, kchunk, work, counters);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (work) cudaFreeAsync(work, stream);
  return e;
}
}  // namespace

// 2 <= N <= 16 columns (dispatch checks).
cudaError_t launch_gemm_nsmall(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  if (N <= 2) return launch_nsmall_t<2, 4, 8, 8>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if (N <= 4) return launch_nsmall_t<4, 4, 8, 8>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
#ifndef MYD_NS16_ROWS
#define MYD_NS16_ROWS 2
#endif
#ifndef MYD_NS16_WARPS
#define MYD_NS16_WARPS 4
#endif
#ifndef MYD_NS16_KW
#define MYD_NS16_KW 8
#endif
  if (N <= 8) return launch_nsmall_t<8, 2, 8, 8>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  return launch_nsmall_t<16, MYD_NS16_ROWS, MYD_NS16_WARPS, MYD_NS16_KW>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
}

namespace {
template <int MC, int MAXC, int WARPS, int KC>
cudaError_t launch_msmall_t(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                            double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  constexpr size_t smem = (size_t)MC * KC * 8;
  if constexpr (smem > 48 * 1024) {
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(gemm_msmall_kernel<MC, MAXC, WARPS, KC>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_done.fetch_or(bit, std::memory_order_release);
    }
  }
  // each warp holds MAXC columns at a time; 8 (4-warp) or 2 (16-warp) CTAs per SM at most
  const int64_t want = std::min<int64_t>((N + (int64_t)WARPS * MAXC - 1) / ((int64_t)WARPS * MAXC),
                                         (long long)(WARPS <= 4 ? 8 : 2) * sm_count_skinny());
  gemm_msmall_kernel<MC, MAXC, WARPS, KC>
      <<<(unsigned)want, 32 * WARPS, smem, stream>>>(M, N, K, A, lda, B, ldb, C, ldc, ep);
  count_launch();
  return cudaGetLastError();
}

// columns per warp held in registers: enough columns per warp for ~2 CTAs
// per SM, at most 32 / MC (register budget)
template <int MC>
cudaError_t launch_msmall_cols(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  // measured (tools/msmall_variants.sh): 4-warp CTAs, 8 per SM, for <= 4 rows;
  // 16-warp CTAs, 2 per SM, for 5..8 rows
  constexpr int WARPS = MC <= 4 ? 4 : 16, KC = MC >= 16 ? 512 : 1024;
  const int64_t per_warp = N / ((int64_t)WARPS * 2 * sm_count_skinny());
  if constexpr (32 / MC >= 8)
    if (per_warp >= 8) return launch_msmall_t<MC, 8, WARPS, KC>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if constexpr (32 / MC >= 4)
    if (per_warp >= 4) return launch_msmall_t<MC, 4, WARPS, KC>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if (per_warp >= 2) return launch_msmall_t<MC, 2, WARPS, KC>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  return launch_msmall_t<MC, 1, WARPS, KC>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
}
}  // namespace

// 2 <= M <= 16 rows (dispatch checks).
cudaError_t launch_gemm_msmall(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  if (M <= 4) return launch_msmall_cols<4>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if (M <= 8) return launch_msmall_cols<8>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  return launch_msmall_cols<16>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
}

namespace {
#ifndef MYD_RD_WARPS
#define MYD_RD_WARPS 8
#endif
// k4 groups per load batch: 2 for m <= 8, 4 for m <= 16, 8 for m <= 32
// (tools/rows_dmma_probe.py, profiles/rows_dmma_r01.log); MYD_RD_U pins it
#ifdef MYD_RD_U
template <int MT> constexpr int rd_u() { return MYD_RD_U; }
#else
template <int MT> constexpr int rd_u() { return MT == 1 ? 2 : (MT == 2 ? 4 : 8); }
#endif
template <int MT, int CT, bool VB>
cudaError_t launch_rows_dmma_t(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                               double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  constexpr int WARPS = MYD_RD_WARPS, U = rd_u<MT>();
  constexpr size_t smem = (size_t)WARPS * 8 * CT * 8 * MT * 8;
  if constexpr (smem > 48 * 1024) {
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(gemm_rows_dmma_kernel<MT, CT, WARPS, U, VB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr_done.fetch_or(bit, std::memory_order_release);
    }
  }
  const int64_t grid = (N + 8 * CT - 1) / (8 * CT);
  gemm_rows_dmma_kernel<MT, CT, WARPS, U, VB><<<(unsigned)grid, 32 * WARPS, smem, stream>>>(M, N, K, A, lda, B, ldb,
                                                                                            C, ldc, ep);
  count_launch();
  return cudaGetLastError();
}

template <int MT>
cudaError_t launch_rows_dmma_ct(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                                double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  // Wider column blocks re-read A from L2 less often (N / (8 CT) times);
  // narrower ones give more CTAs: 32 columns per CTA for m > 8 once that
  // still covers every SM, else 16.  MY_DGEMM_RD_CT overrides (A/B only).
  static const int force_ct = [] {
    const char *v = getenv("MY_DGEMM_RD_CT");
    return v ? atoi(v) : 0;
  }();
  const int sms = sm_count_skinny();
  int ct = force_ct;
  if (ct != 1 && ct != 2 && ct != 4) ct = MT > 1 && N >= 32 * sms ? 4 : 2;
  // 16-byte B loads need an even ldb and a 16-byte aligned B
  if ((ldb & 1) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0) {
    if (ct == 4) return launch_rows_dmma_t<MT, 4, true>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
    if (ct == 2) return launch_rows_dmma_t<MT, 2, true>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
    return launch_rows_dmma_t<MT, 1, true>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  }
  if (ct == 4) return launch_rows_dmma_t<MT, 4, false>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if (ct == 2) return launch_rows_dmma_t<MT, 2, false>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  return launch_rows_dmma_t<MT, 1, false>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
}
}  // namespace

// 2 <= M <= 32 rows on DMMA (dispatch checks).
cudaError_t launch_gemm_rows_dmma(int M, int N, int K, const double *A, int64_t lda, const double *B, int64_t ldb,
                                  double *C, int64_t ldc, cudaStream_t stream, const Epilogue &ep) {
  if (M <= 8) return launch_rows_dmma_ct<1>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  if (M <= 16) return launch_rows_dmma_ct<2>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
  return launch_rows_dmma_ct<4>(M, N, K, A, lda, B, ldb, C, ldc, stream, ep);
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
