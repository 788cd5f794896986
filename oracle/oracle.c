/*
 * oracle.c -- CPU restatement of the reference's my_dgemm path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
 * `bench.py --impl reference`) may load it, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_1609_00076_b200) never links,
 * imports or executes this file.
 *
 * Parity is pinned: tests/golden/make_golden.py (which writes the fixtures)
 * and tests/test_oracle.py compare every function here with the reference
 * package (/root/reference/pkg, imported in the build
 * container) and with the reference tests' own golden values
 * (pkg/tests/test_matrix.py:42-52 GOLDEN_SEED42), and the resulting fixtures
 * are committed under tests/golden/.
 *
 * Arithmetic contract (pkg/setup.py:5-17, pkg/src/gemmforge/kernels.py:1-7):
 * IEEE binary64, one rounded multiply and one rounded add per product, no
 * contraction.  This file MUST be compiled with -ffp-contract=off.
 *
 * Citations are relative to /root/reference/pkg/src/gemmforge/.
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FP_FAST_FMA) && !defined(ORACLE_ALLOW_FMA)
/* Not an error by itself, but -ffp-contract=off is what keeps mul+add split. */
#endif

/* ------------------------------------------------------------------------ */
/* splitmix64-v1 operand generator  (matrix.py:167-207, bench.py:89-106)     */
/* ------------------------------------------------------------------------ */

#define SM_GAMMA 0x9E3779B97F4A7C15ULL
#define SM_MIX1 0xBF58476D1CE4E5B9ULL
#define SM_MIX2 0x94D049BB133111EBULL

/* matrix.py:178-181 `_mix64` */
uint64_t oracle_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * SM_MIX1;
  z = (z ^ (z >> 27)) * SM_MIX2;
  return z ^ (z >> 31);
}

/* matrix.py:184-194 `random_values`: element t -> ((mix64(seed+(t+1)*G)>>11) * 2^-52) - 1 */
static inline double value_at(uint64_t seed, uint64_t t) {
  uint64_t z = oracle_mix64(seed + (t + 1) * SM_GAMMA);
  return (double)(z >> 11) * 0x1p-52 - 1.0;
}

void oracle_random_values(uint64_t seed, int64_t count, int64_t start, double *out) {
  for (int64_t t = 0; t < count; ++t) out[t] = value_at(seed, (uint64_t)(start + t));
}

/* Stream values at arbitrary positions (for sampled-element oracles). */
void oracle_values_at(uint64_t seed, const int64_t *pos, int64_t count, double *out) {
  for (int64_t t = 0; t < count; ++t) out[t] = value_at(seed, (uint64_t)pos[t]);
}

/* matrix.py:197-207 `fill_random`: element (i,j) takes stream position j*m+i;
 * padding rows (i >= m) are never written. */
void oracle_fill(double *data, int64_t m, int64_t n, int64_t ld, uint64_t seed) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) data[j * ld + i] = value_at(seed, (uint64_t)(j * m + i));
}

/* bench.py:89-98 `_operand_seed` */
uint64_t oracle_operand_seed(uint64_t seed, uint64_t role, int64_t m, int64_t n, int64_t k) {
  uint64_t h = seed ^ (role * SM_GAMMA);
  const int64_t dims[3] = {m, n, k};
  for (int d = 0; d < 3; ++d) {
    h = h + SM_GAMMA + (uint64_t)dims[d];
    h = (h ^ (h >> 30)) * SM_MIX1;
    h = (h ^ (h >> 27)) * SM_MIX2;
    h ^= h >> 31;
  }
  return h;
}

/* ------------------------------------------------------------------------ */
/* The oracle: naive triple loop  (_ckernels.pyx:48-59, kernels.py:52-58)    */
/* ------------------------------------------------------------------------ */

/* C(i,j) := C(i,j) + sum_p A(i,p) B(p,j), p ascending, unfused. */
void oracle_naive(int64_t m, int64_t n, int64_t k, const double *a, int64_t lda, const double *b,
                  int64_t ldb, double *c, int64_t ldc) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = c[j * ldc + i];
      for (int64_t p = 0; p < k; ++p) acc = acc + a[p * lda + i] * b[j * ldb + p];
      c[j * ldc + i] = acc;
    }
}

/* Same per-element operation sequence as oracle_naive (acc starts at C(i,j),
 * then p = 0..k-1 each as round(acc + round(a*b))), so it is bitwise equal to
 * it; only the traversal is blocked (i-block x 4 columns, p innermost-outer)
 * and split over threads by column blocks.  This mirrors the reference's
 * claim that every order-preserving engine is bitwise naive
 * (kernels.py:1-7, blocking.py, parallel.py:1-12). */
typedef struct {
  int64_t m, n, k, lda, ldb, ldc;
  const double *a, *b;
  double *c;
  int64_t j_lo, j_hi;
} naive_job;

#define NB_I 128
static void naive_block_run(const naive_job *jb) {
  const int64_t m = jb->m, k = jb->k, lda = jb->lda, ldb = jb->ldb, ldc = jb->ldc;
  double acc[4][NB_I];
  for (int64_t j0 = jb->j_lo; j0 < jb->j_hi; j0 += 4) {
    const int64_t nj = (jb->j_hi - j0) < 4 ? (jb->j_hi - j0) : 4;
    for (int64_t i0 = 0; i0 < m; i0 += NB_I) {
      const int64_t ni = (m - i0) < NB_I ? (m - i0) : NB_I;
      for (int64_t jj = 0; jj < nj; ++jj) memcpy(acc[jj], jb->c + (j0 + jj) * ldc + i0, ni * sizeof(double));
      for (int64_t p = 0; p < k; ++p) {
        const double *ap = jb->a + p * lda + i0;
        for (int64_t jj = 0; jj < nj; ++jj) {
          const double bv = jb->b[(j0 + jj) * ldb + p];
          double *ac = acc[jj];
          for (int64_t ii = 0; ii < ni; ++ii) ac[ii] = ac[ii] + ap[ii] * bv;
        }
      }
      for (int64_t jj = 0; jj < nj; ++jj) memcpy(jb->c + (j0 + jj) * ldc + i0, acc[jj], ni * sizeof(double));
    }
  }
}

static void *naive_thread(void *arg) {
  naive_block_run((const naive_job *)arg);
  return NULL;
}

void oracle_naive_par(int64_t m, int64_t n, int64_t k, const double *a, int64_t lda, const double *b,
                      int64_t ldb, double *c, int64_t ldc, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  naive_job jobs[256];
  pthread_t tid[256];
  const int64_t groups = (n + 3) / 4;
  int64_t lo = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t share = groups / threads + (t < groups % threads ? 1 : 0);
    int64_t hi = lo + share * 4;
    if (hi > n) hi = n;
    jobs[t] = (naive_job){m, n, k, lda, ldb, ldc, a, b, c, lo, hi};
    lo = hi;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, naive_thread, &jobs[t]);
  naive_block_run(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* Five-loop packed algorithm  (goto.py:187-239, _ckernels.pyx:15-45,142-195)*/
/* Used as the CPU baseline ("port") and as an independent bitwise check.   */
/* ------------------------------------------------------------------------ */

/* _ckernels.pyx:142-158 `pack_a`: panel q, element (i,p) at q*mr*kc + p*mr + (i mod mr); pad lanes 0 */
void oracle_pack_a(const double *src, int64_t ld, int64_t mc, int64_t kc, int64_t mr, double *buf) {
  const int64_t npan = (mc + mr - 1) / mr;
  for (int64_t q = 0; q < npan; ++q) {
    const int64_t r0 = q * mr, rows = (mc - r0) < mr ? (mc - r0) : mr;
    for (int64_t p = 0; p < kc; ++p) {
      double *dst = buf + q * mr * kc + p * mr;
      const double *s = src + p * ld + r0;
      int64_t ii = 0;
      for (; ii < rows; ++ii) dst[ii] = s[ii];
      for (; ii < mr; ++ii) dst[ii] = 0.0;
    }
  }
}

/* _ckernels.pyx:161-176 `pack_b`: panel q, element (p,j) at q*nr*kc + p*nr + (j mod nr); pad lanes 0 */
void oracle_pack_b(const double *src, int64_t ld, int64_t kc, int64_t nc, int64_t nr, double *buf) {
  const int64_t npan = (nc + nr - 1) / nr;
  for (int64_t q = 0; q < npan; ++q) {
    const int64_t c0 = q * nr, cols = (nc - c0) < nr ? (nc - c0) : nr;
    for (int64_t p = 0; p < kc; ++p) {
      double *dst = buf + q * nr * kc + p * nr;
      int64_t jj = 0;
      for (; jj < cols; ++jj) dst[jj] = src[(c0 + jj) * ld + p];
      for (; jj < nr; ++jj) dst[jj] = 0.0;
    }
  }
}

/* _ckernels.pyx:15-45 `_mk`: zero tile, load valid C, kc rank-1 updates, store valid C */
static void mk(int64_t kc, const double *ap, const double *bp, double *c, int64_t ldc, int64_t mr, int64_t nr,
               int64_t mv, int64_t nv) {
  double tile[144];
  for (int64_t t = 0; t < mr * nr; ++t) tile[t] = 0.0;
  for (int64_t jj = 0; jj < nv; ++jj)
    for (int64_t ii = 0; ii < mv; ++ii) tile[jj * mr + ii] = c[jj * ldc + ii];
  for (int64_t p = 0; p < kc; ++p) {
    const double *a = ap + p * mr, *bb = bp + p * nr;
    for (int64_t jj = 0; jj < nr; ++jj) {
      const double bv = bb[jj];
      double *t = tile + jj * mr;
      for (int64_t ii = 0; ii < mr; ++ii) t[ii] = t[ii] + a[ii] * bv;
    }
  }
  for (int64_t jj = 0; jj < nv; ++jj)
    for (int64_t ii = 0; ii < mv; ++ii) c[jj * ldc + ii] = tile[jj * mr + ii];
}

/* _ckernels.pyx:179-195 `goto_block`: loop 2 (jr panels [jr_lo,jr_hi)) x loop 1 (ir) */
void oracle_goto_block(const double *apack, const double *bpack, double *c, int64_t ldc, int64_t mcp, int64_t ncp,
                       int64_t kcp, int64_t mr, int64_t nr, int64_t jr_lo, int64_t jr_hi) {
  const int64_t npan_a = (mcp + mr - 1) / mr;
  for (int64_t jrp = jr_lo; jrp < jr_hi; ++jrp) {
    const int64_t jr = jrp * nr, nv = (ncp - jr) < nr ? (ncp - jr) : nr;
    for (int64_t irp = 0; irp < npan_a; ++irp) {
      const int64_t ir = irp * mr, mv = (mcp - ir) < mr ? (mcp - ir) : mr;
      mk(kcp, apack + irp * mr * kcp, bpack + jrp * nr * kcp, c + jr * ldc + ir, ldc, mr, nr, mv, nv);
    }
  }
}

/* parallel.py:108-243 `gemm_goto_parallel`, loop "ic": static contiguous split
 * of the ic blocks (split_range, parallel.py:39-57), worker 0 packs B with a
 * barrier before use and one after compute; per-worker A packs. */
typedef struct {
  int64_t m, n, k, lda, ldb, ldc, mr, nr, mc, kc, nc;
  const double *a, *b;
  double *c;
  double *bpack;
  int threads;
  pthread_barrier_t *bar;
} goto_shared;

typedef struct {
  goto_shared *sh;
  int w;
  int64_t lo, hi;
  double *apack;
} goto_worker;

static void *goto_run_ic(void *arg) {
  goto_worker *wk = (goto_worker *)arg;
  goto_shared *s = wk->sh;
  for (int64_t jc = 0; jc < s->n; jc += s->nc) {
    const int64_t ncp = (s->n - jc) < s->nc ? (s->n - jc) : s->nc;
    const int64_t jr_panels = (ncp + s->nr - 1) / s->nr;
    for (int64_t pc = 0; pc < s->k; pc += s->kc) {
      const int64_t kcp = (s->k - pc) < s->kc ? (s->k - pc) : s->kc;
      if (wk->w == 0) oracle_pack_b(s->b + jc * s->ldb + pc, s->ldb, kcp, ncp, s->nr, s->bpack);
      if (s->threads > 1) pthread_barrier_wait(s->bar);
      for (int64_t t = wk->lo; t < wk->hi; ++t) {
        const int64_t ic = t * s->mc;
        const int64_t mcp = (s->m - ic) < s->mc ? (s->m - ic) : s->mc;
        oracle_pack_a(s->a + pc * s->lda + ic, s->lda, mcp, kcp, s->mr, wk->apack);
        oracle_goto_block(wk->apack, s->bpack, s->c + jc * s->ldc + ic, s->ldc, mcp, ncp, kcp, s->mr, s->nr, 0,
                          jr_panels);
      }
      if (s->threads > 1) pthread_barrier_wait(s->bar);
    }
  }
  return NULL;
}

static size_t round64(size_t x) { return ((x + 63) / 64) * 64 + 64; }

/* Returns 0 on success, -1 on invalid parameters (goto.py:65-80), -2 on OOM. */
int oracle_goto(int64_t m, int64_t n, int64_t k, const double *a, int64_t lda, const double *b, int64_t ldb,
                double *c, int64_t ldc, int64_t mr, int64_t nr, int64_t mc, int64_t kc, int64_t nc, int threads) {
  if (mr < 1 || mr > 12 || nr < 1 || nr > 12 || mc < 1 || kc < 1 || nc < 1 || mc % mr || nc % nr) return -1;
  if (threads < 1 || threads > 256) return -1;
  const int64_t kc_buf = kc < k ? kc : k;
  const int64_t mcb = mc < m ? mc : m, ncb = nc < n ? nc : n;
  const int64_t ic_count = (m + mc - 1) / mc;
  double *bpack = (double *)aligned_alloc(64, round64((size_t)(((ncb + nr - 1) / nr) * nr * kc_buf * 8)));
  if (!bpack) return -2;
  goto_shared sh = {m, n, k, lda, ldb, ldc, mr, nr, mc, kc, nc, a, b, c, bpack, threads, NULL};
  pthread_barrier_t bar;
  if (threads > 1) {
    pthread_barrier_init(&bar, NULL, (unsigned)threads);
    sh.bar = &bar;
  }
  goto_worker wk[256];
  pthread_t tid[256];
  const size_t apack_bytes = round64((size_t)(((mcb + mr - 1) / mr) * mr * kc_buf * 8));
  int64_t lo = 0;
  for (int w = 0; w < threads; ++w) {
    const int64_t share = ic_count / threads + (w < ic_count % threads ? 1 : 0);
    wk[w] = (goto_worker){&sh, w, lo, lo + share, (double *)aligned_alloc(64, apack_bytes)};
    lo += share;
  }
  for (int w = 1; w < threads; ++w) pthread_create(&tid[w], NULL, goto_run_ic, &wk[w]);
  goto_run_ic(&wk[0]);
  for (int w = 1; w < threads; ++w) pthread_join(tid[w], NULL);
  for (int w = 0; w < threads; ++w) free(wk[w].apack);
  free(bpack);
  if (threads > 1) pthread_barrier_destroy(&bar);
  return 0;
}
