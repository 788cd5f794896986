// DMMA.8x8x4 throughput vs warps per SM sub-partition and independent chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = c; c1[c] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
void run(double *out, int sms, int clk_khz, int warps_per_sm) {
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_loop<CHAINS><<<sms, 32 * warps_per_sm>>>(out, iters);
  cudaEventRecord(e0);
  dmma_loop<CHAINS><<<sms, 32 * warps_per_sm>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * 256 * CHAINS * (double)iters * sms * warps_per_sm;
  printf("chains=%2d warps/SM=%2d (%.1f/SMSP): %.2f TFLOP/s  %.1f flop/clk/SM\n", CHAINS, warps_per_sm,
         warps_per_sm / 4.0, flop / ms / 1e9, flop / (ms * 1e-3) / sms / (clk_khz * 1e3));
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *out; cudaMalloc(&out, 4096 * 8);
  for (int w : {4, 8, 12, 16}) {
    run<2>(out, p.multiProcessorCount, clk, w);
    run<4>(out, p.multiProcessorCount, clk, w);
    run<8>(out, p.multiProcessorCount, clk, w);
    run<32>(out, p.multiProcessorCount, clk, w);
  }
  return 0;
}
