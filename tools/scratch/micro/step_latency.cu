// Micro-benchmark: per-step latency of barrier-synchronised elimination steps
// on one SM (clock64 inside the kernel).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bar_only(long long* out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void sts_bar_lds(long long* out, int iters, double seed) {
  __shared__ double line[2][256];
  double v = seed + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    line[i & 1][threadIdx.x] = v;
    __syncthreads();
    v = fma(line[i & 1][(threadIdx.x + 1) & 255], 0.5, v);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

__global__ void dfma_chain(long long* out, int iters, double seed) {
  double v = seed + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = fma(v, 0.999, 0.001);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

__global__ void rsqrt_chain(long long* out, int iters, double seed) {
  double v = seed + threadIdx.x + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = rsqrt(v) + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

__global__ void div_chain(long long* out, int iters, double seed) {
  double v = seed + threadIdx.x + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = 1.0 / v + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

__global__ void shfl_chain(long long* out, int iters, double seed) {
  double v = seed + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) * 0.999;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

__global__ void lds_chain(long long* out, int iters) {
  __shared__ int idx[256];
  idx[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = idx[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (p == 12345) out[1] = 1;
}

__global__ void syncwarp_chain(long long* out, int iters, double seed) {
  __shared__ double line[2][256];
  double v = seed + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    line[i & 1][threadIdx.x] = v;
    __syncwarp();
    v = fma(line[i & 1][threadIdx.x ^ 1], 0.5, v);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == 12345.0) out[1] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  const int it = 4096;
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize(); launch(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s %lld cycles/iter\n", name, h[0]);
  };
  for (int nt : {32, 128, 256, 512, 1024}) {
    char buf[64];
    snprintf(buf, 64, "bar_only %d thr", nt);
    run(buf, [&] { bar_only<<<1, nt>>>(d, it); });
  }
  for (int nt : {32, 256}) {
    char buf[64];
    snprintf(buf, 64, "sts_bar_lds_fma %d thr", nt);
    run(buf, [&] { sts_bar_lds<<<1, nt>>>(d, it, 1.0); });
  }
  run("syncwarp sts/lds/fma 256", [&] { syncwarp_chain<<<1, 256>>>(d, it, 1.0); });
  run("dfma chain 32", [&] { dfma_chain<<<1, 32>>>(d, it, 1.0); });
  run("rsqrt chain 32", [&] { rsqrt_chain<<<1, 32>>>(d, it, 1.0); });
  run("div chain 32", [&] { div_chain<<<1, 32>>>(d, it, 1.0); });
  run("shfl chain 32", [&] { shfl_chain<<<1, 32>>>(d, it, 1.0); });
  run("lds chain 32", [&] { lds_chain<<<1, 256>>>(d, it); });
  return 0;
}
