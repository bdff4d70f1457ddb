// Per-launch GPU time vs K for a single 64x64 output tile (qtt_gemm), and an
// empty kernel for the launch floor.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/qtt_b200.h"
__global__ void empty_kernel() {}
int main() {
  double *A, *C;
  cudaMalloc(&A, sizeof(double) * 64 * 8192);
  cudaMalloc(&C, sizeof(double) * 8192 * 64);
  cudaMemset(A, 0, sizeof(double) * 64 * 8192);
  cudaMemset(C, 0, sizeof(double) * 8192 * 64);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto go) {
    for (int i = 0; i < 5; ++i) go();
    cudaEventRecord(e0, s);
    const int reps = 200;
    for (int i = 0; i < reps; ++i) go();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-32s %8.2f us/launch\n", name, ms * 1000.0 / reps);
  };
  timeit("empty kernel", [&] { empty_kernel<<<1, 128, 0, s>>>(); });
  char buf[64];
  for (int k : {4, 16, 64, 256, 1024}) {
    snprintf(buf, 64, "gemm 64x64 k=%d beta=1", k);
    timeit(buf, [&] { qtt_gemm(1, 0, 64, 64, k, -1.0, A, k, A, k, 1.0, C, 64, s); });
    snprintf(buf, 64, "gemm 64x64 k=%d beta=0", k);
    timeit(buf, [&] { qtt_gemm(1, 0, 64, 64, k, 1.0, A, k, A, k, 0.0, C, 64, s); });
  }
  // host-side cost of one call (no sync)
  cudaDeviceSynchronize();
  cudaEventRecord(e0, s);
  auto t0 = clock();
  for (int i = 0; i < 2000; ++i) qtt_gemm(1, 0, 64, 64, 16, 1.0, A, 16, A, 16, 0.0, C, 64, s);
  auto t1 = clock();
  printf("host cpu time per qtt_gemm call: %.2f us\n", (double)(t1 - t0) / CLOCKS_PER_SEC * 1e6 / 2000);
  cudaDeviceSynchronize();
  return 0;
}
