// Host-side cost of one my_dgemm_ex(DEVICE_PTRS) call from C (no Python):
// wall time of N asynchronous calls on a tiny problem vs the device time of
// the same N calls replayed from a CUDA graph.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a host_overhead.cu -I../../include \
//        -L../../paper_1609_00076_b200 -lmy_dgemm_b200 -Xlinker -rpath=$PWD/../../paper_1609_00076_b200
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "my_dgemm.h"

__global__ void empty_kernel() {}

int main(int argc, char **argv) {
  const int mn = argc > 1 ? atoi(argv[1]) : 256, k = argc > 2 ? atoi(argv[2]) : 256, N = 2000;
  double *a, *b, *c;
  cudaMalloc(&a, sizeof(double) * mn * k);
  cudaMalloc(&b, sizeof(double) * mn * k);
  cudaMalloc(&c, sizeof(double) * mn * mn);
  my_dgemm_fill_random(a, mn, k, mn, 1, 0, nullptr);
  my_dgemm_fill_random(b, k, mn, k, 2, 0, nullptr);
  my_dgemm_fill_random(c, mn, mn, mn, 3, 0, nullptr);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < 10; ++i) my_dgemm_ex(mn, mn, k, a, mn, b, k, c, mn, MY_DGEMM_DEVICE_PTRS, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0, st);
  for (int i = 0; i < N; ++i) my_dgemm_ex(mn, mn, k, a, mn, b, k, c, mn, MY_DGEMM_DEVICE_PTRS, st);
  cudaEventRecord(e1, st);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / N;
  printf("%dx%dx%d stream loop: host %.2f us/call, device span %.2f us/call\n", mn, mn, k, host_us, ms * 1e3 / N);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 100; ++i) my_dgemm_ex(mn, mn, k, a, mn, b, k, c, mn, MY_DGEMM_DEVICE_PTRS, st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%dx%dx%d graph replay: %.2f us/call  (%.2f TF)\n", mn, mn, k, ms * 1e3 / 2000,
         2.0 * mn * mn * k / (ms * 1e-3 / 2000) / 1e12);
  if (argc > 3) {  // calibration: the same replay of an empty <<<148, 384>>> kernel
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 100; ++i) empty_kernel<<<148, 384, 0, st>>>();
    cudaStreamEndCapture(st, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    cudaGraphLaunch(ge2, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge2, st);
    cudaEventRecord(e1, st);
    cudaStreamSynchronize(st);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel graph replay: %.2f us/launch\n", ms * 1e3 / 2000);
  }
  return 0;
}
