// Micro-benchmark of the register-resident 64x64 block routines (common.cuh):
// cycles per call inside one CTA, data already on chip.
#include <cstdio>
#include "../../paper_2501_07778_b200/csrc/common.cuh"
using namespace qtt;

template <int WHICH>
__global__ void __launch_bounds__(256) bench(const double* g, double* out, long long* cyc, int* bad) {
  __shared__ double S[kBlk][kBlk + 1];
  __shared__ double line[256];
  __shared__ double dinv[kBlk];
  double a[16], x[16], y[16];
  blk_load(a, g, 64, 64);
  blk_to_smem(a, S);
  __syncthreads();
  long long t0 = clock64();
  if (WHICH == 0) blk_factor<true>(a, line, bad);
  if (WHICH == 1) blk_factor<false>(a, line, bad);
  if (WHICH == 2) blk_tri_inverse<false>(S, x, y, line, dinv);
  if (WHICH == 3) blk_tri_inverse<true>(S, x, y, line, dinv);
  __syncthreads();
  long long t1 = clock64();
  if (WHICH >= 2) {
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = x[q] + (WHICH == 3 ? y[q] : 0.0);
  }
  blk_store(a, out, 64, 64);
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double h[4096];
  for (int c = 0; c < 64; ++c)
    for (int r = 0; r < 64; ++r) h[r + 64 * c] = (r == c ? 64.0 : 0.0) + 1.0 / (1 + r + c);
  double *g, *o;
  long long* cyc;
  int* bad;
  cudaMalloc(&g, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&cyc, 8); cudaMalloc(&bad, 4);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  const char* names[] = {"factor CHOL", "factor LU", "inverse upper", "inverse upper+lower"};
  auto run = [&](int w, auto launch) {
    launch(); launch(); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-22s %6lld cycles (%5.1f cyc/step)  kernel %.2f us\n", names[w], c, c / 64.0, ms * 10.0);
  };
  run(0, [&] { bench<0><<<1, 256>>>(g, o, cyc, bad); });
  run(1, [&] { bench<1><<<1, 256>>>(g, o, cyc, bad); });
  run(2, [&] { bench<2><<<1, 256>>>(g, o, cyc, bad); });
  run(3, [&] { bench<3><<<1, 256>>>(g, o, cyc, bad); });
  return 0;
}
