// Which part of the in-register 64x64 Cholesky step costs the cycles?
// Variants of the CHOL step with parts removed (results are garbage for the
// timing-only variants).
#include <cstdio>
#include "../../paper_2501_07778_b200/csrc/common.cuh"
using namespace qtt;

template <int V>
__device__ __forceinline__ void factor_v(double (&a)[16], double* line) {
  const int c = blk_col(), part = blk_part();
#pragma unroll
  for (int j = 0; j < kBlk; ++j) {
    const int qj = j >> 2, pj = j & 3;
    double* rb = line + (j & 1) * 128;
    if (part == pj) rb[c] = a[qj];
    __syncthreads();
    const double piv = rb[j];
    double inv;
    if (V == 1) inv = piv * 0.5;             // no rsqrt
    else if (V == 2) {                       // approx + 1 Newton step
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(piv));
      inv = y * (1.5 - 0.5 * piv * y * y);
    } else inv = rsqrt(piv);
    const double rc = rb[c] * inv;
    if (part == pj) a[qj] = (c >= j) ? rc : 0.0;
    if (V != 3 && c > j) {                   // V3: no trailing update
      const double t = -rc * inv;
      const double* r = rb + part;
      if (part > pj) a[qj] = fma(r[4 * qj], t, a[qj]);
#pragma unroll
      for (int q = qj + 1; q < 16; ++q) a[q] = fma(r[4 * q], t, a[q]);
    }
  }
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(256) bench(const double* g, double* out, long long* cyc) {
  __shared__ double line[256];
  double a[16];
  blk_load(a, g, 64, 64);
  __syncthreads();
  long long t0 = clock64();
  factor_v<V>(a, line);
  long long t1 = clock64();
  blk_store(a, out, 64, 64);
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double h[4096];
  for (int c = 0; c < 64; ++c)
    for (int r = 0; r < 64; ++r) h[r + 64 * c] = (r == c ? 64.0 : 0.0) + 1.0 / (1 + r + c);
  double *g, *o; long long* cyc;
  cudaMalloc(&g, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&cyc, 8);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  const char* names[] = {"full", "no rsqrt", "approx rsqrt + newton", "no trailing update"};
  auto run = [&](int w, auto launch) {
    launch(); launch(); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %6lld cycles (%5.1f /step)\n", names[w], c, c / 64.0);
  };
  run(0, [&] { bench<0><<<1, 256>>>(g, o, cyc); });
  run(1, [&] { bench<1><<<1, 256>>>(g, o, cyc); });
  run(2, [&] { bench<2><<<1, 256>>>(g, o, cyc); });
  run(3, [&] { bench<3><<<1, 256>>>(g, o, cyc); });
  return 0;
}
