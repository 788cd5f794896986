// common.cuh -- shared device helpers for the sm_100a FP64 GEMM kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define MYD_DEVICE __device__ __forceinline__

namespace myd {

// 64-bit flat index of (i, j) under leading dimension ld (matrix.py:34-36).
MYD_DEVICE int64_t at(int64_t i, int64_t j, int64_t ld) { return j * ld + i; }

// cp.async (LDGSTS): BYTES in {8, 16}; src_bytes < BYTES zero-fills the tail,
// src_bytes == 0 reads nothing and writes zeros.
template <int BYTES>
MYD_DEVICE void cp_async(void *smem_dst, const void *gmem_src, int src_bytes) {
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gmem_src), "r"(src_bytes)
                 : "memory");
  } else {
    static_assert(BYTES == 8, "cp.async size");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gmem_src), "r"(src_bytes)
                 : "memory");
  }
}

MYD_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
MYD_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- mbarrier (shared::cta) ----
MYD_DEVICE uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

MYD_DEVICE void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

MYD_DEVICE void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Single non-blocking probe; issue early, consume the result later so the
// probe latency overlaps independent work.
MYD_DEVICE bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Arrive on `bar` once every cp.async this thread issued so far has landed.
// .noinc: the arrival counts against the count given at init.
MYD_DEVICE void cp_async_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Tracks this thread's prior cp.async ops: +1 pending now, -1 when they land.
MYD_DEVICE void cp_async_mbar_arrive_inc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// One arrival plus `bytes` of expected async-proxy transactions.
MYD_DEVICE void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Bulk (TMA-engine) copy of `bytes` contiguous bytes global -> shared,
// completion counted on `bar` (complete_tx).  16-byte aligned src/dst,
// bytes a multiple of 16.
MYD_DEVICE void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same with an L2 eviction-priority hint (a createpolicy value).
MYD_DEVICE void bulk_g2s_hint(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
MYD_DEVICE uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
MYD_DEVICE uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
MYD_DEVICE uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// Bulk (TMA-engine) copy shared -> global, tracked in this thread's bulk
// group; same alignment rules.  Generic-proxy writes to the source must be
// made visible first (fence_proxy_async_smem by the writing threads).
MYD_DEVICE void bulk_s2g(void *gmem_dst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
MYD_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// Wait until this thread's bulk groups have finished READING shared memory.
MYD_DEVICE void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// Wait until this thread's bulk groups have completed (global writes done).
MYD_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
MYD_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

MYD_DEVICE void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// One DMMA.8x8x4: d(8x8) += a(8x4, row) * b(4x8, col).
// Fragment ownership (lane = threadIdx.x % 32):
//   a: A[lane/4][lane%4]     b: B[lane%4][lane/4]
//   c: C[lane/4][2*(lane%4) + {0,1}]
MYD_DEVICE void dmma_884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Epilogue mode of the GEMM kernels.  blas == 0: the my_dgemm contract,
// accumulate onto C (the accumulator starts at C, like _mk).  blas == 1:
// the BLAS dgemm contract, C := alpha * (A B) + beta * C with the product
// accumulated from zero and C not read when beta == 0.
struct Epilogue {
  double alpha = 1.0, beta = 1.0;
  int blas = 0;
};

// Stream-K schedule of the tiled kernel (iters == 0: unit mode): the first
// dp_tiles tiles run as whole tiles round-robin (data-parallel rounds), then
// the (tile, slab) iterations of the tiles from tile0 on -- `iters` of them --
// are split evenly over the grid; partial accumulators of cut tiles in `work`
// (one slot per CTA), per-(slot, warp) flags set to `epoch`.
struct StreamK {
  long long dp_tiles = 0;  // whole tiles [0, dp_tiles) first, round-robin
  long long tile0 = 0;     // first tile of the stream-K phase
  long long iters = 0;
  double *work = nullptr;
  unsigned long long *flags = nullptr;
  unsigned long long epoch = 0;
};

// Kernel launch counter shared by every launcher (my_dgemm_kernel_launches).
void count_launch(int n = 1);

}  // namespace myd
