// GPU time per launch of small / skinny-K GEMMs through the C ABI (qtt_gemm),
// back-to-back launches timed with events (no Python in the loop).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/qtt_b200.h"

int main() {
  double *A, *C;
  cudaMalloc(&A, sizeof(double) * 64 * 8192);
  cudaMalloc(&C, sizeof(double) * 8192 * 8192);
  cudaMemset(A, 0, sizeof(double) * 64 * 8192);
  cudaMemset(C, 0, sizeof(double) * 8192 * 8192);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ta = 0; ta < 2; ++ta)
    for (int n : {64, 256, 512, 1024, 1984, 4096}) {
      const int k = 64;
      auto go = [&] {
        if (ta) qtt_gemm(1, 0, n, n, k, -1.0, A, k, A, k, 1.0, C, n, s);
        else qtt_gemm(0, 1, n, n, k, -1.0, A, n, A, n, 1.0, C, n, s);
      };
      for (int i = 0; i < 5; ++i) go();
      cudaEventRecord(e0, s);
      const int reps = 100;
      for (int i = 0; i < reps; ++i) go();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1000.0 / reps;
      printf("gemm ta=%d n=%5d k=%d: %8.2f us  %6.2f TF/s\n", ta, n, k, us, 2.0 * n * n * k / us / 1e6);
    }
  return 0;
}
