// FP64 pipe microbenchmarks for sm_100a: DFMA and DMMA (mma.sync f64) issue rate per SM.
// Used once to pick the micro-tile instruction.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// m8n8k4: 256 FMA per warp instruction.
template <int CHAINS>
__global__ void dmma884_loop(double *out, int iters) {
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

// m16n8k16: 2048 FMA per warp instruction (A 8 regs/thread, B 4, C 4).
template <int CHAINS>
__global__ void dmma16816_loop(double *out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-12;
  double c[CHAINS][4];
#pragma unroll
  for (int q = 0; q < CHAINS; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[q][i] = q + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < CHAINS; ++q)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < CHAINS; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock_khz %d smem/block optin %zu regs/SM %d\n", p.name, p.multiProcessorCount, clk,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double *out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    int blocks = sms * (1024 / threads) ;
    float ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
    double flop = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA chains=8 threads=%d blocks=%d: %.3f ms  %.2f TFLOP/s  (%.1f flop/clk/SM at %d MHz)\n", threads, blocks, ms,
           flop / ms / 1e9, flop / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads);
    float ms = time_it([&] { dmma884_loop<8><<<blocks, threads>>>(out, iters); });
    double flop = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4 chains=8 threads=%d: %.3f ms  %.2f TFLOP/s (%.1f flop/clk/SM)\n", threads, ms, flop / ms / 1e9,
           flop / (ms * 1e-3) / sms / (clk * 1e3));
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads);
    float ms = time_it([&] { dmma16816_loop<4><<<blocks, threads>>>(out, iters / 4); });
    double flop = 2.0 * 2048 * 4 * (iters / 4) * (double)blocks * (threads / 32);
    printf("DMMA m16n8k16 chains=4 threads=%d: %.3f ms  %.2f TFLOP/s (%.1f flop/clk/SM)\n", threads, ms, flop / ms / 1e9,
           flop / (ms * 1e-3) / sms / (clk * 1e3));
  }
  // single-warp latency probes
  {
    float ms = time_it([&] { dfma_loop<1><<<1, 32>>>(out, iters * 10, 1.0000001, 1e-9); });
    printf("DFMA dependent latency ~ %.2f ns/iter\n", ms * 1e6 / (iters * 10));
    ms = time_it([&] { dmma884_loop<1><<<1, 32>>>(out, iters * 10); });
    printf("DMMA884 dependent latency ~ %.2f ns/iter\n", ms * 1e6 / (iters * 10));
    ms = time_it([&] { dmma16816_loop<1><<<1, 32>>>(out, iters * 10); });
    printf("DMMA16816 dependent latency ~ %.2f ns/iter\n", ms * 1e6 / (iters * 10));
  }
  CK(cudaGetLastError());
  return 0;
}
