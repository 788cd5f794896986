// One warp's DMMA.8x8x4 accumulator chain with operands from shared memory:
// cycles per k-step for (a) fragments loaded by plain LDS just before use
// (the compiler's schedule), (b) fragments loaded PD k-steps ahead with the
// loads pinned in program order (volatile ld.shared), (c) constant operands.
// Question answered: is the small-block kernel's ~66 cycles per k-step the
// DMMA chain itself or the LDS -> DMMA dependency?  (profiles/r02/dmma_chain_r02a.txt)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_chain.cu -o dmma_chain
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds_v(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

constexpr int KS = 64;  // k-steps per pass (fragments resident in shared memory)

template <int MODE, int PD, int CH>
__global__ void chain(double *out, long long *clk, int passes) {
  __shared__ double sa[KS * 32], sb[KS * 32];
  for (int i = threadIdx.x; i < KS * 32; i += blockDim.x) {
    sa[i] = 1.0 + i * 1e-9;
    sb[i] = 1.0 - i * 1e-9;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double c0[CH], c1[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) c0[c] = c1[c] = 0.0;
  long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
    if constexpr (MODE == 0) {
#pragma unroll 16
      for (int k = 0; k < KS; ++k) {
        const double a = sa[k * 32 + lane], b = sb[k * 32 + lane];
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(c0[c], c1[c], a, b);
      }
    } else if constexpr (MODE == 1) {
      double fa[PD], fb[PD];
#pragma unroll
      for (int q = 0; q < PD - 1; ++q) {
        fa[q] = lds_v(&sa[q * 32 + lane]);
        fb[q] = lds_v(&sb[q * 32 + lane]);
      }
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        if (k + PD - 1 < KS) {
          fa[(k + PD - 1) % PD] = lds_v(&sa[(k + PD - 1) * 32 + lane]);
          fb[(k + PD - 1) % PD] = lds_v(&sb[(k + PD - 1) * 32 + lane]);
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(c0[c], c1[c], fa[k % PD], fb[k % PD]);
      }
    } else {
      const double a = sa[lane], b = sb[lane];
#pragma unroll 16
      for (int k = 0; k < KS; ++k)
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(c0[c], c1[c], a, b);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += c0[c] + c1[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *clk = t1 - t0;
}

template <int MODE, int PD, int CH>
void run(const char *name, double *out, long long *dclk) {
  const int passes = 20;
  chain<MODE, PD, CH><<<1, 32>>>(out, dclk, passes);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
  printf("%-34s chains=%d: %.1f cycles per k-step (%.1f per DMMA)\n", name, CH, (double)c / (passes * KS),
         (double)c / (passes * KS * CH));
}

int main() {
  double *out;
  long long *clk;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&clk, 8);
  run<0, 2, 1>("(a) LDS before use (compiler)", out, clk);
  run<1, 2, 1>("(b) pinned LDS, 1 k-step ahead", out, clk);
  run<1, 4, 1>("(b) pinned LDS, 3 k-steps ahead", out, clk);
  run<1, 8, 1>("(b) pinned LDS, 7 k-steps ahead", out, clk);
  run<2, 2, 1>("(c) constant operands", out, clk);
  run<0, 2, 2>("(a) LDS before use (compiler)", out, clk);
  run<1, 4, 2>("(b) pinned LDS, 3 k-steps ahead", out, clk);
  run<2, 2, 2>("(c) constant operands", out, clk);
  run<0, 2, 4>("(a) LDS before use (compiler)", out, clk);
  run<1, 4, 4>("(b) pinned LDS, 3 k-steps ahead", out, clk);
  run<2, 2, 4>("(c) constant operands", out, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
