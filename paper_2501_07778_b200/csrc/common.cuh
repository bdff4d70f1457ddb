// Shared helpers for the B200 QTT kernels (sm_100a, FP64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <utility>
#include <array>
#include <vector>
#include <atomic>
#include <mutex>

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

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

// SM count of the current device (cached per device; thread-safe).
inline int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Per-device "done" flag for one-time setup such as cudaFuncSetAttribute
// (a per-device property).  Atomic, so concurrent first calls from several
// host threads are well defined (at worst the idempotent setup runs twice).
struct DeviceFlag {
  std::atomic<uint64_t> bits{0};
  static int cur() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool test() const { return (bits.load(std::memory_order_acquire) >> cur()) & 1ull; }
  void set() { bits.fetch_or(1ull << cur(), std::memory_order_release); }
};

// ------------------------------------------------- 64 x 64 register blocks
// The diagonal-block kernels of the blocked Cholesky / LU / triangular
// inverse keep a 64 x 64 block in the registers of 256 threads: thread t
// holds column c = t >> 2, rows part + 4q (part = t & 3, q = 0..15).  Each
// elimination step is right-looking (one rank-1 update of at most 16 entries
// per thread) and exchanges the pivot row / column through a double-buffered
// shared-memory line, so a step costs ONE block barrier and its critical
// path is store -> barrier -> load -> fma.  The 64 steps are fully unrolled
// so every register index is a compile-time constant.
constexpr int kBlk = 64;
__device__ __forceinline__ int blk_col() { return threadIdx.x >> 2; }
__device__ __forceinline__ int blk_part() { return threadIdx.x & 3; }

// Load rows/cols [0, kb) of a column-major block, identity padding outside.
__device__ __forceinline__ void blk_load(double (&a)[16], const double* __restrict__ g,
                                         int64_t ld, int kb) {
  const int c = blk_col(), part = blk_part();
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int i = part + 4 * q;
    a[q] = (i < kb && c < kb) ? g[i + (int64_t)c * ld] : (i == c ? 1.0 : 0.0);
  }
}
__device__ __forceinline__ void blk_store(const double (&a)[16], double* __restrict__ g, int64_t ld,
                                          int kb) {
  const int c = blk_col(), part = blk_part();
  if (c >= kb) return;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int i = part + 4 * q;
    if (i < kb) g[i + (int64_t)c * ld] = a[q];
  }
}
__device__ __forceinline__ void blk_to_smem(const double (&a)[16], double (*S)[kBlk + 1]) {
  const int c = blk_col(), part = blk_part();
#pragma unroll
  for (int q = 0; q < 16; ++q) S[part + 4 * q][c] = a[q];
}

// In-register factorisation of the 64 x 64 block (identity-padded beyond the
// active size, so always 64 steps).  `line` needs 256 doubles of shared
// memory.  *bad is set on a non-positive (CHOL) / zero (LU) pivot.
//   CHOL: G = R^T R, a <- R (upper, strictly lower part zeroed)
//   LU  : A = L U without pivoting, a <- L (unit, strictly lower) + U
// Full-precision 1/sqrt(x) and 1/x from the hardware approximations plus
// two Newton steps (off the slow-path call of rsqrt()/division; x > 0 finite
// resp. x != 0 normal, which the callers guarantee or flag).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

template <bool CHOL>
__device__ __forceinline__ void blk_factor(double (&a)[16], double* line, int* bad) {
  const int c = blk_col(), part = blk_part();
#pragma unroll
  for (int j = 0; j < kBlk; ++j) {
    const int qj = j >> 2, pj = j & 3;
    double* rb = line + (j & 1) * 128;  // pivot row
    double* cb = rb + 64;               // pivot column (LU)
    if (part == pj) rb[c] = a[qj];
    if (!CHOL && c == j) {
#pragma unroll
      for (int q = qj; q < 16; ++q) cb[part + 4 * q] = a[q];
    }
    __syncthreads();
    const double piv = rb[j];
    // Row i = part + 4q lies below the pivot iff q > qj, or q == qj and
    // part > pj: only the q == qj entry needs a predicate.
    if (CHOL) {
      if (threadIdx.x == 0 && !(piv > 0.0)) *bad = 1;
      const double inv = rsqrt_nr(piv);
      const double rc = rb[c] * inv;
      if (part == pj) a[qj] = (c >= j) ? rc : 0.0;
      if (c > j) {
        const double t = -rc * inv;  // G[i][c] -= (G[j][i] / sqrt(piv)) * R[j][c]
        const double* r = rb + part;
        if (part > pj) a[qj] = fma(r[4 * qj], t, a[qj]);
#pragma unroll
        for (int q = qj + 1; q < 16; ++q) a[q] = fma(r[4 * q], t, a[q]);
      }
    } else {
      if (threadIdx.x == 0 && !(fabs(piv) > 0.0)) *bad = 1;
      const double inv = rcp_nr(piv);
      if (c == j) {
        if (part > pj) a[qj] *= inv;
#pragma unroll
        for (int q = qj + 1; q < 16; ++q) a[q] *= inv;
      } else if (c > j) {
        const double t = -rb[c] * inv;  // A[i][c] -= (A[i][j] / piv) * U[j][c]
        const double* l = cb + part;
        if (part > pj) a[qj] = fma(l[4 * qj], t, a[qj]);
#pragma unroll
        for (int q = qj + 1; q < 16; ++q) a[q] = fma(l[4 * q], t, a[q]);
      }
    }
  }
  __syncthreads();
}

// Inverses of the triangles of a factor held in shared memory S (64 x 64):
// x <- U^{-1} (upper triangle incl. diagonal of S), and, if LOWER,
// y <- L^{-1} (unit lower triangle of S).  Back / forward substitution on the
// identity, right-looking, both sweeps sharing one barrier per step.
// `line` needs 256 doubles, `dinv` 64 doubles of shared memory, both
// scratch; S must be complete (barrier) on entry.
template <bool LOWER>
__device__ __forceinline__ void blk_tri_inverse(double (*S)[kBlk + 1], double (&x)[16],
                                                double (&y)[16], double* line, double* dinv) {
  const int c = blk_col(), part = blk_part();
  if (threadIdx.x < kBlk) dinv[threadIdx.x] = 1.0 / S[threadIdx.x][threadIdx.x];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    x[q] = (part + 4 * q == c) ? 1.0 : 0.0;
    if (LOWER) y[q] = x[q];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kBlk; ++s) {
    const int j = kBlk - 1 - s, qj = j >> 2, pj = j & 3;  // upper: rows bottom-up
    const int k = s, qk = k >> 2, pk = k & 3;             // lower: rows top-down
    double* ub = line + (s & 1) * 128;
    double* lb = ub + 64;
    if (part == pj) {
      x[qj] *= dinv[j];
      ub[c] = x[qj];
    }
    if (LOWER && part == pk) lb[c] = y[qk];
    __syncthreads();
    const double xj = -ub[c];
#pragma unroll
    for (int q = 0; q < qj; ++q) x[q] = fma(S[part + 4 * q][j], xj, x[q]);
    if (part < pj) x[qj] = fma(S[part + 4 * qj][j], xj, x[qj]);
    if (LOWER) {
      const double yk = -lb[c];
      if (part > pk) y[qk] = fma(S[part + 4 * qk][k], yk, y[qk]);
#pragma unroll
      for (int q = qk + 1; q < 16; ++q) y[q] = fma(S[part + 4 * q][k], yk, y[q]);
    }
  }
  __syncthreads();
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
  int flags = 0;  // kGemm* structure flags below
};
// Structure flags (tiles of 64): only the upper-triangular tiles of C are
// computed (the strictly lower tiles of C are left unspecified); op(A) / op(B)
// are upper triangular (kGemmLowA / kGemmLowB: lower triangular), so each
// tile's K range is clipped to the nonzeros.
constexpr int kGemmUpperC = 1, kGemmTriA = 2, kGemmTriB = 4, kGemmLowA = 8, kGemmLowB = 16;

int gemm(const GemmArgs& g, cudaStream_t stream);

// Stream-ordered allocation of library temporaries.  Two kinds of host
// thread use the library: the chain workers of run_concurrent (one thread +
// stream per independent TT problem, all alive at once) and everything else
// (the caller's thread: serial roundings, the AMEn sweep).  Measured on the
// config-2 step (tools/scratch/serial_state_probe.py, QTT_SHARED_POOL A/B):
// * the chain workers are fastest on the device's SHARED default pool with
//   its opportunistic cross-stream reuse (44.7 ms per concurrent step; 46-47
//   ms on private pools or without opportunistic reuse: blocks just freed by
//   a neighbour chain are still in L2);
// * but once those chains have populated the shared pool, every allocation
//   made on another thread polls the completion of their frees: the ~15
//   workspace allocations of each CholeskyQR2 cost ~0.25 ms more (serial
//   step 89 -> 115 ms, constant-E solve 2.9 -> 3.3 s).
// So worker threads opt in to the shared pool (qtt_thread_shared_pool) and
// every other thread allocates from a pool PRIVATE to it (one per device,
// created on first use, release threshold = max).  cudaFreeAsync returns a
// block to the pool it came from, whichever thread frees it.
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s);
template <typename T>
inline cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t s) {
  return malloc_async(reinterpret_cast<void**>(p), bytes, s);
}
// Trim every pool created by malloc_async (qtt_release_cached).
void trim_thread_pools();
// The calling thread allocates from the device's shared default pool from now on.
void set_thread_shared_pool(bool shared);

// Keep freed stream-ordered allocations cached in the device's default pool
// (release threshold = max): the TT sweeps allocate and free workspaces on
// every step, and trimming the pool at each synchronisation would re-map
// memory every time.  Called by every C-ABI entry point.
void pool_init();

// Optional per-launch GEMM timing (CUDA events on the launching stream) used
// by bench.py to report the DMMA kernel's achieved FLOP rate.
struct GemmProfile {
  std::mutex mu;  // chains on several host threads may record concurrently
  std::atomic<bool> on{false};
  double flops = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  std::vector<double> launch_flops;
  std::vector<std::array<int64_t, 7>> shapes;  // m, n, k, batch, flags, splits, tile BM
};
GemmProfile& gemm_profile();

// Convenience: single column-major GEMM.
inline int dgemm(cudaStream_t s, int ta, int tb, int m, int n, int k, double alpha,
                 const double* a, int64_t lda, const double* b, int64_t ldb,
                 double beta, double* c, int64_t ldc, int flags = 0) {
  GemmArgs g{m, n, k, ta, tb, alpha, beta, a, lda, 0, b, ldb, 0, c, ldc, 0, 1, flags};
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
