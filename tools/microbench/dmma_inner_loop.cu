// Ceiling of the fast kernel's inner loop: the same fragment loads (LDS.64 at
// the padded pitches) and 8x4 DMMA micro-tiles per warp, 8 warps/SM, looping
// over one resident slab with no barriers -- and variants with a per-slab
// __syncthreads or mbarrier probe to price the synchronisation.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int BM = 128, BN = 128, BK = 16, AP = BM + 4, BP = BK + 4;
constexpr int FM = 8, FN = 4;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// SYNC: 0 none, 1 __syncthreads per slab, 2 mbarrier probe+arrive per slab.
// PROD: 4 extra warps stream cp.async copies (same bytes/slab as the real
// producers) from an L2-resident buffer into a separate smem ring.
template <int SYNC, int PROD>
__global__ void __launch_bounds__(384, 1) inner(double *out, int iters, const double *src) {
  __shared__ double As[BK * AP];
  __shared__ double Bs[BN * BP];
  __shared__ __align__(8) unsigned long long bar[2];
  extern __shared__ __align__(16) double ring[];
  for (int i = threadIdx.x; i < BK * AP; i += 256) As[i] = 1.0 + i * 1e-9;
  for (int i = threadIdx.x; i < BN * BP; i += 256) Bs[i] = 1.0 - i * 1e-9;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[1])), "r"((1u << 20) - 1));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar[0])));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (PROD) {
      // 16 x 16-byte copies per lane per "slab", ring of 4 x 32 KB
      for (int it = 0; it < iters * 3 / 2; ++it) {
        const int slot = it & 3;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int e = ((warp - 8) * 32 + lane + c * 128) * 2;
          unsigned dst = (unsigned)__cvta_generic_to_shared(ring + slot * 4096 + e);
          const double *g = src + ((size_t)(blockIdx.x * 16 + (it % 64)) * 4096 + e);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 16;" ::"r"(dst), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 2;" ::: "memory");
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
  const int wm = warp & 1, wn = warp >> 1, r = lane >> 2, q = lane & 3;
  const int a_off = q * AP + wm * 64 + r, b_off = (wn * 32 + r) * BP + q;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  double fa[2][FM], fb[2][FN];
  auto load = [&](int buf, int kk) {
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[buf][i] = As[a_off + kk * 4 * AP + i * 8];
#pragma unroll
    for (int j = 0; j < FN; ++j) fb[buf][j] = Bs[b_off + j * 8 * BP + kk * 4];
  };
  load(0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int cur = kk & 1;
      if (kk == 3 && SYNC == 1) asm volatile("bar.sync 1, 256;");
      if (kk == 1 && SYNC == 2) {
        unsigned ok;
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(&bar[0])) : "memory");
        if (!ok) out[0] = 1.0;
      }
      load(cur ^ 1, (kk + 1) & 3);
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[cur][i], fb[cur][j]);
    }
    if (SYNC == 2) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar[1])) : "memory");
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int SYNC, int PROD>
void run(double *out, int sms, int clk, const double *src) {
  const int iters = 2000;
  const int dyn = 4 * 4096 * 8;
  cudaFuncSetAttribute(inner<SYNC, PROD>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  inner<SYNC, PROD><<<sms, 384, dyn>>>(out, iters, src);
  cudaEventRecord(e0);
  inner<SYNC, PROD><<<sms, 384, dyn>>>(out, iters, src);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * BM * BN * BK * (double)iters * sms;
  printf("inner loop sync=%d prod=%d: %.2f TFLOP/s (%.1f%% of 128 flop/clk/SM)\n", SYNC, PROD, flop / ms / 1e9,
         100.0 * flop / (ms * 1e-3) / sms / (clk * 1e3) / 128.0);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *out; cudaMalloc(&out, 4096 * 8);
  double *src; cudaMalloc(&src, (size_t)148 * 16 * 64 * 4096 * 8 / 16);  // ~76 MB, L2-resident-ish
  cudaMemset(src, 0, (size_t)148 * 16 * 64 * 4096 * 8 / 16);
  run<0, 0>(out, p.multiProcessorCount, clk, src);
  run<1, 0>(out, p.multiProcessorCount, clk, src);
  run<2, 0>(out, p.multiProcessorCount, clk, src);
  run<0, 1>(out, p.multiProcessorCount, clk, src);
  run<2, 1>(out, p.multiProcessorCount, clk, src);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
