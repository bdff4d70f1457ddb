// Cycle split of the 64x64 register-block LU kernel: load / factor / smem /
// triangular inverses / store (tools/micro, not part of the library).
#include <cstdio>
#include <vector>
#include "../../paper_2501_07778_b200/csrc/common.cuh"
using namespace qtt;
__global__ void __launch_bounds__(256) probe(double* A, double* linv, double* uinv, long long* t, int* bad) {
  extern __shared__ double sm[];
  double (*S)[kBlk + 1] = reinterpret_cast<double (*)[kBlk + 1]>(sm);
  double* line = sm + kBlk * (kBlk + 1);
  double* dinv = line + 256;
  double a[16], x[16], y[16];
  long long t0 = clock64();
  blk_load(a, A, 64, 64);
  __syncthreads();
  long long t1 = clock64();
  blk_factor<false>(a, line, bad);
  long long t2 = clock64();
  blk_to_smem(a, S);
  __syncthreads();
  long long t3 = clock64();
  blk_tri_inverse<true>(S, x, y, line, dinv);
  long long t4 = clock64();
  blk_store(x, uinv, 64, 64);
  blk_store(y, linv, 64, 64);
  __syncthreads();
  long long t5 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
}

__device__ __forceinline__ void tri_inv_rd(const double (*S)[kBlk + 1], double (*X)[kBlk + 1],
                                           double (*Y)[kBlk + 1], double* T) {
  for (int idx = threadIdx.x; idx < kBlk * kBlk; idx += blockDim.x) {
    X[idx >> 6][idx & 63] = 0.0;
    Y[idx >> 6][idx & 63] = 0.0;
  }
  __syncthreads();
  {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b0 = 8 * w, j = lane & 7, i4 = lane >> 3;
    for (int i = 7; i >= 0; --i) {
      if ((i & 3) == i4 && j >= i) {
        double acc = (i == j) ? 1.0 : 0.0;
        for (int k = i + 1; k <= j; ++k) acc = fma(-S[b0 + i][b0 + k], X[b0 + k][b0 + j], acc);
        X[b0 + i][b0 + j] = acc / S[b0 + i][b0 + i];
      }
      __syncwarp();
    }
    for (int i = 0; i < 8; ++i) {
      if ((i & 3) == i4 && j <= i) {
        double acc = (i == j) ? 1.0 : 0.0;
        for (int k = j; k < i; ++k) acc = fma(-S[b0 + i][b0 + k], Y[b0 + k][b0 + j], acc);
        Y[b0 + i][b0 + j] = acc;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int h = 8; h < kBlk; h *= 2) {
    const int npair = kBlk / (2 * h), per = h * h, tot = npair * per;
    for (int idx = threadIdx.x; idx < 2 * tot; idx += blockDim.x) {
      const bool up = idx < tot;
      const int e = up ? idx : idx - tot;
      const int p = e / per, i = (e % per) / h, jj = e % h;
      const int a0 = 2 * p * h, b0 = a0 + h;
      double acc = 0.0;
      if (up) { for (int k = 0; k <= jj; ++k) acc = fma(S[a0 + i][b0 + k], X[b0 + k][b0 + jj], acc); }
      else { for (int k = jj; k < h; ++k) acc = fma(S[b0 + i][a0 + k], Y[a0 + k][a0 + jj], acc); }
      T[idx] = acc;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * tot; idx += blockDim.x) {
      const bool up = idx < tot;
      const int e = up ? idx : idx - tot;
      const int p = e / per, i = (e % per) / h, jj = e % h;
      const int a0 = 2 * p * h, b0 = a0 + h;
      const double* t = T + (up ? 0 : tot) + p * per;
      double acc = 0.0;
      if (up) { for (int k = i; k < h; ++k) acc = fma(X[a0 + i][a0 + k], t[k * h + jj], acc); X[a0 + i][b0 + jj] = -acc; }
      else { for (int k = 0; k <= i; ++k) acc = fma(Y[b0 + i][b0 + k], t[k * h + jj], acc); Y[b0 + i][a0 + jj] = -acc; }
    }
    __syncthreads();
  }
}
__global__ void __launch_bounds__(256) probe_rd(double* A, double* linv, double* uinv, long long* t, int* bad) {
  extern __shared__ double sm[];
  double (*S)[kBlk + 1] = reinterpret_cast<double (*)[kBlk + 1]>(sm);
  double* line = sm + kBlk * (kBlk + 1);
  double (*X)[kBlk + 1] = reinterpret_cast<double (*)[kBlk + 1]>(line + 256);
  double (*Y)[kBlk + 1] = X + kBlk;
  double* T = reinterpret_cast<double*>(Y + kBlk);
  double a[16];
  blk_load(a, A, 64, 64);
  blk_factor<false>(a, line, bad);
  blk_to_smem(a, S);
  __syncthreads();
  long long t3 = clock64();
  tri_inv_rd(S, X, Y, T);
  long long t4 = clock64();
  if (threadIdx.x == 0) t[3] = t4 - t3;
}
int main() {
  std::vector<double> h(64 * 64);
  for (int j = 0; j < 64; ++j) for (int i = 0; i < 64; ++i) h[i + 64 * j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double *A, *L, *U; long long* t; int* bad;
  cudaMalloc(&A, 8 * 4096); cudaMalloc(&L, 8 * 4096); cudaMalloc(&U, 8 * 4096); cudaMalloc(&t, 64); cudaMalloc(&bad, 4);
  const int smem = (64 * 65 + 256 + 64) * 8;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<1, 256, smem>>>(A, L, U, t, bad);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long ht[5]; cudaMemcpy(ht, t, 40, cudaMemcpyDeviceToHost);
    printf("rep %d: %.1f us  cycles load %lld factor %lld smem %lld inverse %lld store %lld  (%s)\n", rep, ms * 1e3,
           ht[0], ht[1], ht[2], ht[3], ht[4], cudaGetErrorString(cudaGetLastError()));
  }
  const int smem2 = (3 * 64 * 65 + 256 + 4096) * 8;
  cudaFuncSetAttribute(probe_rd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), 8 * 4096, cudaMemcpyHostToDevice);
    probe_rd<<<1, 256, smem2>>>(A, L, U, t, bad);
    cudaDeviceSynchronize();
    long long ht[5]; cudaMemcpy(ht, t, 40, cudaMemcpyDeviceToHost);
    printf("rd inverse cycles %lld (%s)\n", ht[3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
