// Shared helpers for the B200 QTT kernels (sm_100a, FP64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <utility>
#include <vector>

namespace qtt {

// Status codes returned by every C-ABI entry point (include/qtt_b200.h).
enum Status : int {
  kOk = 0,
  kInvalid = 1,
  kCuda = 2,
  kWorkspace = 3,
  kUnsupported = 4,
};

constexpr int kMaxCores = 96;  // QTT depth supported by by-value descriptors

#define QTT_CUDA(expr)                                                     \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      fprintf(stderr, "[qtt_b200] CUDA error %s at %s:%d: %s\n",           \
              cudaGetErrorName(_e), __FILE__, __LINE__,                    \
              cudaGetErrorString(_e));                                     \
      return ::qtt::kCuda;                                                 \
    }                                                                      \
  } while (0)

// Every kernel launch of the library is followed by QTT_CHECK_LAUNCH(), which
// also counts it (qtt_launch_count() in the C ABI).
void note_launch();
#define QTT_CHECK_LAUNCH()  \
  do {                      \
    ::qtt::note_launch();   \
    QTT_CUDA(cudaGetLastError()); \
  } while (0)

#define QTT_TRY(expr)                    \
  do {                                   \
    int _s = (expr);                     \
    if (_s != ::qtt::kOk) return _s;     \
  } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// X = S^{-1} for an upper-triangular B x B block in shared memory (B = 64,
// 256 threads): rows bottom-up, all columns of a row in one step, 4 lanes per
// column splitting the dot product.  Replaces column-per-thread substitution
// (B^2/2 dependent shared-memory FMAs per thread).
template <int B>
__device__ __forceinline__ void upper_inverse_smem(double (*S)[B + 1], double (*X)[B + 1], int tid) {
  static_assert(B * 4 == 256, "256 threads per block");
  const int c = tid >> 2, part = tid & 3;
  for (int r = part; r < B; r += 4) X[r][c] = 0.0;
  __syncthreads();
  for (int i = B - 1; i >= 0; --i) {
    double acc = 0.0, acc2 = 0.0;
    if (c > i) {
      int l = i + 1 + part;
#pragma unroll 2
      for (; l + 4 <= c; l += 8) {
        acc = fma(S[i][l], X[l][c], acc);
        acc2 = fma(S[i][l + 4], X[l + 4][c], acc2);
      }
      if (l <= c) acc = fma(S[i][l], X[l][c], acc);
    }
    acc += acc2;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (part == 0 && c >= i) X[i][c] = (c == i) ? 1.0 / S[i][i] : -acc / S[i][i];
    __syncthreads();
  }
}

// X = L^{-1} for the unit lower-triangular part of S (diagonal taken as 1).
template <int B>
__device__ __forceinline__ void unit_lower_inverse_smem(double (*S)[B + 1], double (*X)[B + 1],
                                                        int tid) {
  static_assert(B * 4 == 256, "256 threads per block");
  const int c = tid >> 2, part = tid & 3;
  for (int r = part; r < B; r += 4) X[r][c] = 0.0;
  __syncthreads();
  for (int i = 0; i < B; ++i) {
    double acc = 0.0;
    if (c < i)
      for (int l = c + part; l < i; l += 4) acc = fma(S[i][l], X[l][c], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (part == 0 && c <= i) X[i][c] = (c == i) ? 1.0 : -acc;
    __syncthreads();
  }
}

// Left-looking (Crout) factorisation of the leading kb x kb part of a 64 x 64
// shared-memory block, 256 threads, two barriers per step.  Step j computes
// every entry of row j (and, for LU, column j) as ONE dot product of length j
// against the already finished rows/columns, two lanes per entry:
//   CHOL: R[j][c] = (G[j][c] - sum_l R[l][j] R[l][c]) / R[j][j],  c >= j
//   LU  : U[j][c] =  A[j][c] - sum_l L[j][l] U[l][c],            c >= j
//         L[r][j] = (A[r][j] - sum_l L[r][l] U[l][j]) / U[j][j], r >  j
// `tmp` needs 128 doubles of shared memory.  *bad is set on a non-positive
// (CHOL) or zero (LU) pivot.  For CHOL the strictly lower part is zeroed.
template <bool CHOL>
__device__ __forceinline__ void crout_factor64(double (*S)[65], double* tmp, int kb, int* bad) {
  const int tid = threadIdx.x, item = tid >> 1, half = tid & 1;
  for (int j = 0; j < kb; ++j) {
    const int nrow = kb - j;                 // row items c = j .. kb-1
    const int ncol = CHOL ? 0 : kb - j - 1;  // column items r = j+1 .. kb-1
    double acc = 0.0, acc2 = 0.0;
    if (item < nrow) {
      const int c = j + item;
      int l = half;
#pragma unroll 2
      for (; l + 2 < j; l += 4) {
        acc = fma(CHOL ? S[l][j] : S[j][l], S[l][c], acc);
        acc2 = fma(CHOL ? S[l + 2][j] : S[j][l + 2], S[l + 2][c], acc2);
      }
      if (l < j) acc = fma(CHOL ? S[l][j] : S[j][l], S[l][c], acc);
    } else if (item < nrow + ncol) {
      const int r = j + 1 + (item - nrow);
      int l = half;
#pragma unroll 2
      for (; l + 2 < j; l += 4) {
        acc = fma(S[r][l], S[l][j], acc);
        acc2 = fma(S[r][l + 2], S[l + 2][j], acc2);
      }
      if (l < j) acc = fma(S[r][l], S[l][j], acc);
    }
    acc += acc2;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (half == 0 && item < nrow + ncol) {
      const double base = item < nrow ? S[j][j + item] : S[j + 1 + (item - nrow)][j];
      tmp[item] = base - acc;
    }
    __syncthreads();
    const double piv = tmp[0];
    if (tid == 0 && (CHOL ? !(piv > 0.0) : !(fabs(piv) > 0.0))) atomicExch(bad, 1);
    if (half == 0 && item < nrow + ncol) {
      if (item < nrow) S[j][j + item] = CHOL ? tmp[item] / sqrt(piv) : tmp[item];
      else S[j + 1 + (item - nrow)][j] = tmp[item] / piv;
    }
    __syncthreads();
  }
  if (CHOL) {
    for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
      const int r = idx % kb, c = idx / kb;
      if (r > c) S[r][c] = 0.0;
    }
    __syncthreads();
  }
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ------------------------------------------------------------------ GEMM
// Column-major FP64 GEMM on the DMMA (mma.sync m8n8k4 f64) tensor pipe:
//   C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b]
// op(X) = X or X^T.  Batched through strides (0 stride = shared operand).
struct GemmArgs {
  int m, n, k;
  int trans_a, trans_b;
  double alpha, beta;
  const double* a;
  int64_t lda, stride_a;
  const double* b;
  int64_t ldb, stride_b;
  double* c;
  int64_t ldc, stride_c;
  int batch;
};

int gemm(const GemmArgs& g, cudaStream_t stream);

// Keep freed stream-ordered allocations cached in the device's default pool
// (release threshold = max): the TT sweeps allocate and free workspaces on
// every step, and trimming the pool at each synchronisation would re-map
// memory every time.  Called by every C-ABI entry point.
void pool_init();

// Optional per-launch GEMM timing (CUDA events on the launching stream) used
// by bench.py to report the DMMA kernel's achieved FLOP rate.
struct GemmProfile {
  bool on = false;
  double flops = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  std::vector<double> launch_flops;
};
GemmProfile& gemm_profile();

// Convenience: single column-major GEMM.
inline int dgemm(cudaStream_t s, int ta, int tb, int m, int n, int k, double alpha,
                 const double* a, int64_t lda, const double* b, int64_t ldb,
                 double beta, double* c, int64_t ldc) {
  GemmArgs g{m, n, k, ta, tb, alpha, beta, a, lda, 0, b, ldb, 0, c, ldc, 0, 1};
  return gemm(g, s);
}

// Out-of-place transpose of a column-major (rows x cols) matrix into
// a column-major (cols x rows) matrix.
int transpose(cudaStream_t s, int rows, int cols, const double* src, int64_t lds,
              double* dst, int64_t ldd);

int fill(cudaStream_t s, double* p, int64_t n, double v);
int copy_matrix(cudaStream_t s, int rows, int cols, const double* src, int64_t lds,
                double* dst, int64_t ldd);

}  // namespace qtt
