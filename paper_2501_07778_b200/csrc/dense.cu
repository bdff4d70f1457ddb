// Dense realisation (a8), dense operator application for the residual
// (a14) and the bit-exact Z-order index maps (a9).
#include <vector>

#include "../../include/qtt_b200.h"
#include "common.cuh"

namespace qtt {
namespace {

// Dense matrix from the merged-mode contraction: K = sum_l (i_l*m_l + j_l) *
// prod_{t<l} n_t m_t  ->  (I, J) with I = sum i_l prod n_t, J = sum j_l prod m_t.
struct MatPerm {
  int d;
  int n[QTT_MAX_CORES], m[QTT_MAX_CORES];
};

__global__ void merged_to_dense_kernel(const __grid_constant__ MatPerm mp, int64_t rows, int64_t total,
                                       const double* __restrict__ merged, double* __restrict__ out) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t I = g % rows, J = g / rows;
    int64_t K = 0, stride = 1;
    for (int l = 0; l < mp.d; ++l) {
      const int i = (int)(I % mp.n[l]);
      const int j = (int)(J % mp.m[l]);
      I /= mp.n[l];
      J /= mp.m[l];
      K += (int64_t)(i * mp.m[l] + j) * stride;
      stride *= (int64_t)mp.n[l] * mp.m[l];
    }
    out[g] = merged[K];
  }
}

__device__ __forceinline__ int64_t spread(int64_t x, int d) {
  int64_t z = 0;
  for (int b = 0; b < d; ++b) z |= ((x >> b) & 1LL) << (2 * b);
  return z;
}
__device__ __forceinline__ int64_t squeeze(int64_t z, int d) {
  int64_t x = 0;
  for (int b = 0; b < d; ++b) x |= ((z >> (2 * b)) & 1LL) << b;
  return x;
}

__global__ void zorder_kernel(int d, int dof, int64_t nodes, int64_t* __restrict__ perm) {
  for (int64_t z = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; z < nodes;
       z += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = squeeze(z, d), j = squeeze(z >> 1, d);
    const int64_t L = i + (j << d);
    if (dof) {
      perm[2 * z] = 2 * L;
      perm[2 * z + 1] = 2 * L + 1;
    } else {
      perm[z] = L;
    }
  }
}

__global__ void z_index_kernel(int d, int64_t count, const int64_t* __restrict__ i,
                               const int64_t* __restrict__ j, int64_t* __restrict__ z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x)
    z[t] = spread(i[t], d) | (spread(j[t], d) << 1);
}

inline int grid1d(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 16 * num_sms()));
}

// Vector contraction of merged order-3 cores: acc (r_k x P_k) column-major.
int contract_merged(const qtt_layout* L, const double* a, double* out, cudaStream_t s) {
  const int d = L->d;
  int64_t total = 1, maxbuf = 1;
  for (int l = 0; l < d; ++l) {
    total *= L->rows[l] * L->cols[l];
    maxbuf = std::max(maxbuf, total * L->ranks[l + 1]);
  }
  double *b0, *b1;
  QTT_CUDA(malloc_async(&b0, sizeof(double) * maxbuf, s));
  QTT_CUDA(malloc_async(&b1, sizeof(double) * maxbuf, s));
  QTT_TRY(fill(s, b0, 1, 1.0));
  double* cur = b0;
  double* nxt = b1;
  int64_t P = 1;
  for (int l = 0; l < d; ++l) {
    const int r0 = (int)L->ranks[l], r1 = (int)L->ranks[l + 1];
    const int n = (int)(L->rows[l] * L->cols[l]);
    const double* core = a + L->offsets[l];
    for (int i = 0; i < n; ++i)
      QTT_TRY(dgemm(s, 0, 0, r1, (int)P, r0, 1.0, core + (int64_t)i * r1, (int64_t)n * r1, cur, r0,
                    0.0, nxt + (int64_t)r1 * P * i, r1));
    P *= n;
    std::swap(cur, nxt);
  }
  QTT_CUDA(cudaMemcpyAsync(out, cur, sizeof(double) * P, cudaMemcpyDeviceToDevice, s));
  QTT_CUDA(cudaFreeAsync(b0, s));
  QTT_CUDA(cudaFreeAsync(b1, s));
  return kOk;
}

}  // namespace

int contract(const qtt_layout* L, const double* a, double* dense, cudaStream_t s) {
  const int d = L->d;
  int bits = 0;
  int64_t rows = 1, cols = 1;
  for (int l = 0; l < d; ++l) {
    rows *= L->rows[l];
    cols *= L->cols[l];
  }
  for (int64_t t = rows * cols; t > 1; t >>= 1) ++bits;
  if (bits > 26) return kUnsupported;
  if (!L->is_matrix) return contract_merged(L, a, dense, s);
  double* merged;
  QTT_CUDA(malloc_async(&merged, sizeof(double) * rows * cols, s));
  QTT_TRY(contract_merged(L, a, merged, s));
  MatPerm mp;
  mp.d = d;
  for (int l = 0; l < d; ++l) {
    mp.n[l] = (int)L->rows[l];
    mp.m[l] = (int)L->cols[l];
  }
  merged_to_dense_kernel<<<grid1d(rows * cols), 256, 0, s>>>(mp, rows, rows * cols, merged, dense);
  QTT_CHECK_LAUNCH();
  QTT_CUDA(cudaFreeAsync(merged, s));
  return kOk;
}

// core (r0, n, m, r1) C-order -> out[i][(j*r0 + q) * r1 + p] = core[q, i, j, p]
__global__ void repack_core_kernel(int r0, int n, int m, int r1, const double* __restrict__ core,
                                   double* __restrict__ out) {
  const int64_t total = (int64_t)r0 * n * m * r1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(t % r1);
    int64_t rest = t / r1;
    const int q = (int)(rest % r0);
    rest /= r0;
    const int j = (int)(rest % m);
    const int i = (int)(rest / m);
    out[t] = core[(((int64_t)q * n + i) * m + j) * r1 + p];
  }
}

// y = A v for a dense v (solver.apply_tt_matrix, solver.py:57-73).  The
// running tensor T_k is column-major (r_k*m_k x L_k) with rows (bond, col
// bit) and the finished row bits appended as the slowest axes.
int dense_apply(const qtt_layout* LA, const double* a, const double* v, double* out,
                cudaStream_t s) {
  const int d = LA->d;
  int64_t cols = 1, rows = 1;
  for (int l = 0; l < d; ++l) {
    cols *= LA->cols[l];
    rows *= LA->rows[l];
  }
  int64_t maxbuf = std::max(cols, rows);
  {
    int64_t rem_cols = cols, done_rows = 1;
    for (int l = 0; l < d; ++l) {
      rem_cols /= LA->cols[l];
      done_rows *= LA->rows[l];
      maxbuf = std::max(maxbuf, LA->ranks[l + 1] * rem_cols * done_rows);
    }
  }
  int64_t maxcore = 1;
  for (int l = 0; l < d; ++l)
    maxcore = std::max(maxcore, LA->ranks[l] * LA->rows[l] * LA->cols[l] * LA->ranks[l + 1]);
  double *b0, *b1, *apk;
  QTT_CUDA(malloc_async(&b0, sizeof(double) * maxbuf, s));
  QTT_CUDA(malloc_async(&b1, sizeof(double) * maxbuf, s));
  QTT_CUDA(malloc_async(&apk, sizeof(double) * maxcore, s));
  QTT_CUDA(cudaMemcpyAsync(b0, v, sizeof(double) * cols, cudaMemcpyDeviceToDevice, s));
  double* cur = b0;
  double* nxt = b1;
  int64_t rem_cols = cols, done_rows = 1;
  for (int l = 0; l < d; ++l) {
    const int r0 = (int)LA->ranks[l], r1 = (int)LA->ranks[l + 1];
    const int n = (int)LA->rows[l], m = (int)LA->cols[l];
    rem_cols /= m;
    const int64_t Lc = rem_cols * done_rows;  // columns of T_k viewed (r0*m x Lc)
    if (Lc > 0x7fffffff) return kUnsupported;
    const double* core = a + LA->offsets[l];
    // Repack the core so that, per row bit i, A_i (r1 x m*r0) has column
    // index j*r0 + q matching T_k's row order: one K = m*r0 GEMM per i
    // instead of m accumulating K = r0 GEMMs (T_{k+1} written once).
    repack_core_kernel<<<grid1d((int64_t)r0 * n * m * r1), 256, 0, s>>>(r0, n, m, r1, core, apk);
    QTT_CHECK_LAUNCH();
    for (int i = 0; i < n; ++i)
      QTT_TRY(dgemm(s, 0, 0, r1, (int)Lc, m * r0, 1.0, apk + (int64_t)i * r1 * m * r0, r1, cur,
                    (int64_t)r0 * m, 0.0, nxt + (int64_t)r1 * Lc * i, r1));
    done_rows *= n;
    std::swap(cur, nxt);
  }
  QTT_CUDA(cudaMemcpyAsync(out, cur, sizeof(double) * rows, cudaMemcpyDeviceToDevice, s));
  QTT_CUDA(cudaFreeAsync(b0, s));
  QTT_CUDA(cudaFreeAsync(b1, s));
  QTT_CUDA(cudaFreeAsync(apk, s));
  return kOk;
}

int zorder_perm(int d, int64_t* perm, int dof, cudaStream_t s) {
  const int64_t nodes = 1LL << (2 * d);
  zorder_kernel<<<grid1d(nodes), 256, 0, s>>>(d, dof, nodes, perm);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int z_index(int d, int64_t count, const int64_t* i, const int64_t* j, int64_t* z, cudaStream_t s) {
  if (count == 0) return kOk;
  z_index_kernel<<<grid1d(count), 256, 0, s>>>(d, count, i, j, z);
  QTT_CHECK_LAUNCH();
  return kOk;
}

}  // namespace qtt
