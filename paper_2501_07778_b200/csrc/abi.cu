// extern "C" boundary of libqttb200.so (declared in include/qtt_b200.h).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/qtt_b200.h"
#include "linalg.cuh"

namespace qtt {

int64_t packed_size(const qtt_layout* L) {
  int64_t end = 0;
  for (int l = 0; l < L->d; ++l) {
    const int64_t sz = L->ranks[l] * L->rows[l] * L->cols[l] * L->ranks[l + 1];
    end = std::max(end, L->offsets[l] + sz);
  }
  return end;
}

void pack_offsets(qtt_layout* L) {
  int64_t off = 0;
  for (int l = 0; l < L->d; ++l) {
    L->offsets[l] = off;
    const int64_t sz = L->ranks[l] * L->rows[l] * L->cols[l] * L->ranks[l + 1];
    off += (sz + 31) / 32 * 32;
  }
}

// tt_ops.cu
int product(const qtt_layout*, const double*, const qtt_layout*, const double*, const qtt_layout*,
            double*, int, cudaStream_t);
int add(const qtt_layout*, const double*, const qtt_layout*, const double*, double,
        const qtt_layout*, double*, cudaStream_t);
int zkron(const qtt_layout*, const double*, const qtt_layout*, const double*, const qtt_layout*,
          double*, cudaStream_t);
int diag(const qtt_layout*, const double*, const qtt_layout*, double*, cudaStream_t);
int transpose_tt(const qtt_layout*, const double*, const qtt_layout*, double*, cudaStream_t);
int scale_copy(const qtt_layout*, const double*, double, double*, cudaStream_t);
int dot(const qtt_layout*, const double*, const qtt_layout*, const double*, double*, cudaStream_t);
// round.cu
int round_tt(const qtt_layout*, const double*, double, qtt_layout*, double*, cudaStream_t, double*);
int norm_orth(const qtt_layout*, const double*, double*, cudaStream_t);
int decompose(const double*, int, const int64_t*, double, qtt_layout*, double*, int64_t,
              cudaStream_t);
// dense.cu
int contract(const qtt_layout*, const double*, double*, cudaStream_t);
int dense_apply(const qtt_layout*, const double*, const double*, double*, cudaStream_t);
int zorder_perm(int, int64_t*, int, cudaStream_t);
int z_index(int, int64_t, const int64_t*, const int64_t*, int64_t*, cudaStream_t);

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }
bool valid(const qtt_layout* L) {
  if (!L || L->d < 1 || L->d > QTT_MAX_CORES) return false;
  if (L->ranks[0] != 1 || L->ranks[L->d] != 1) return false;
  for (int l = 0; l < L->d; ++l) {
    if (L->ranks[l] < 1 || L->rows[l] < 1 || L->cols[l] < 1) return false;
    if (L->offsets[l] < 0) return false;
  }
  return true;
}
}  // namespace

}  // namespace qtt

using namespace qtt;

extern "C" {

const char* qtt_version(void) { return "qtt_b200 0.1 sm_100a fp64"; }

long long qtt_launch_count(void) { return g_launches.load(); }

int qtt_profile_gemm(int32_t on) {
  pool_init();
  GemmProfile& p = gemm_profile();
  std::lock_guard<std::mutex> lk(p.mu);
  for (auto& e : p.events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  p.events.clear();
  p.launch_flops.clear();
  p.shapes.clear();
  p.flops = 0.0;
  p.on = on != 0;
  return QTT_OK;
}

int qtt_profile_gemm_read(double* flops, double* ms, int64_t* launches) {
  pool_init();
  GemmProfile& p = gemm_profile();
  std::lock_guard<std::mutex> lk(p.mu);
  double tot = 0.0;
  for (auto& e : p.events) {
    QTT_CUDA(cudaEventSynchronize(e.second));
    float t = 0.f;
    QTT_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
    tot += t;
  }
  if (getenv("QTT_GEMM_LOG"))  // per-launch shapes for tools/gemm_shapes.py
    for (size_t i = 0; i < p.events.size() && i < p.shapes.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, p.events[i].first, p.events[i].second);
      const auto& q = p.shapes[i];
      fprintf(stderr, "[gemm] %ld %ld %ld %ld %ld %ld %.4f %.6e\n", (long)q[0], (long)q[1], (long)q[2],
              (long)q[3], (long)q[4], (long)q[5], t, p.launch_flops[i]);
    }
  *flops = p.flops;
  *ms = tot;
  *launches = (int64_t)p.events.size();
  return QTT_OK;
}

int qtt_profile_gemm_shape(int64_t i, int64_t* out) {
  GemmProfile& p = gemm_profile();
  std::lock_guard<std::mutex> lk(p.mu);
  if (i < 0) i += (int64_t)p.shapes.size();
  if (i < 0 || i >= (int64_t)p.shapes.size()) return QTT_EINVAL;
  for (int j = 0; j < 7; ++j) out[j] = p.shapes[i][j];
  return QTT_OK;
}

int qtt_release_cached(void* stream) {
  pool_init();
  QTT_CUDA(cudaStreamSynchronize(S(stream)));
  int dev = 0;
  QTT_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  QTT_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  QTT_CUDA(cudaMemPoolTrimTo(pool, 0));
  trim_thread_pools();
  return QTT_OK;
}

int qtt_thread_shared_pool(int32_t shared) {
  pool_init();
  set_thread_shared_pool(shared != 0);
  return QTT_OK;
}

int64_t qtt_layout_size(const qtt_layout* lay) { return valid(lay) ? packed_size(lay) : -1; }

int qtt_matvec(const qtt_layout* A, const double* a, const qtt_layout* x, const double* xd,
               const qtt_layout* y, double* yd, void* stream) {
  pool_init();
  if (!valid(A) || !valid(x) || !valid(y) || !A->is_matrix || x->is_matrix) return QTT_EINVAL;
  return product(A, a, x, xd, y, yd, 0, S(stream));
}

int qtt_matmat(const qtt_layout* A, const double* a, const qtt_layout* B, const double* b,
               const qtt_layout* C, double* c, void* stream) {
  pool_init();
  if (!valid(A) || !valid(B) || !valid(C) || !A->is_matrix || !B->is_matrix) return QTT_EINVAL;
  return product(A, a, B, b, C, c, 0, S(stream));
}

int qtt_hadamard(const qtt_layout* A, const double* a, const qtt_layout* B, const double* b,
                 const qtt_layout* C, double* c, void* stream) {
  pool_init();
  if (!valid(A) || !valid(B) || !valid(C)) return QTT_EINVAL;
  return product(A, a, B, b, C, c, 1, S(stream));
}

int qtt_add(const qtt_layout* A, const double* a, const qtt_layout* B, const double* b,
            double beta, const qtt_layout* C, double* c, void* stream) {
  pool_init();
  if (!valid(A) || !valid(B) || !valid(C)) return QTT_EINVAL;
  return add(A, a, B, b, beta, C, c, S(stream));
}

int qtt_zkron(const qtt_layout* A, const double* a, const qtt_layout* B, const double* b,
              const qtt_layout* C, double* c, void* stream) {
  pool_init();
  if (!valid(A) || !valid(B) || !valid(C)) return QTT_EINVAL;
  return zkron(A, a, B, b, C, c, S(stream));
}

int qtt_diag(const qtt_layout* V, const double* v, const qtt_layout* D, double* dd, void* stream) {
  pool_init();
  if (!valid(V) || !valid(D)) return QTT_EINVAL;
  return diag(V, v, D, dd, S(stream));
}

int qtt_transpose(const qtt_layout* A, const double* a, const qtt_layout* T, double* t,
                  void* stream) {
  pool_init();
  if (!valid(A) || !valid(T)) return QTT_EINVAL;
  return transpose_tt(A, a, T, t, S(stream));
}

int qtt_scale(const qtt_layout* A, const double* a, double s, double* out, void* stream) {
  pool_init();
  if (!valid(A)) return QTT_EINVAL;
  return scale_copy(A, a, s, out, S(stream));
}

int qtt_round(const qtt_layout* in, const double* in_data, double eps, qtt_layout* out,
              double* out_data, void* stream) {
  pool_init();
  if (!valid(in) || !out || eps < 0) return QTT_EINVAL;
  return round_tt(in, in_data, eps, out, out_data, S(stream), nullptr);
}

int qtt_round_to_host(const qtt_layout* in, const double* in_data, double eps, qtt_layout* out,
                      double* out_data, double* host_data, void* stream) {
  pool_init();
  if (!valid(in) || !out || !host_data || eps < 0) return QTT_EINVAL;
  return round_tt(in, in_data, eps, out, out_data, S(stream), host_data);
}

int qtt_decompose(const double* dense, int32_t d, const int64_t* sizes, double eps,
                  qtt_layout* out, double* out_data, int64_t out_capacity, void* stream) {
  pool_init();
  if (!dense || !sizes || !out || eps < 0) return QTT_EINVAL;
  return decompose(dense, d, sizes, eps, out, out_data, out_capacity, S(stream));
}

int qtt_norm(const qtt_layout* A, const double* a, double* result, void* stream) {
  pool_init();
  if (!valid(A) || !result) return QTT_EINVAL;
  return norm_orth(A, a, result, S(stream));
}

int qtt_dot(const qtt_layout* A, const double* a, const qtt_layout* B, const double* b,
            double* result, void* stream) {
  pool_init();
  if (!valid(A) || !valid(B) || !result) return QTT_EINVAL;
  return dot(A, a, B, b, result, S(stream));
}

int qtt_contract(const qtt_layout* A, const double* a, double* dense, void* stream) {
  pool_init();
  if (!valid(A)) return QTT_EINVAL;
  return contract(A, a, dense, S(stream));
}

int qtt_dense_apply(const qtt_layout* A, const double* a, const double* v, double* out,
                    void* stream) {
  pool_init();
  if (!valid(A) || !A->is_matrix) return QTT_EINVAL;
  return dense_apply(A, a, v, out, S(stream));
}

int qtt_zorder_permutation(int32_t d, int64_t* perm, void* stream) {
  pool_init();
  if (d < 1 || d > 30) return QTT_EINVAL;
  return zorder_perm(d, perm, 0, S(stream));
}

int qtt_zorder_dof_permutation(int32_t d, int64_t* perm, void* stream) {
  pool_init();
  if (d < 1 || d > 30) return QTT_EINVAL;
  return zorder_perm(d, perm, 1, S(stream));
}

int qtt_z_index(int32_t d, int64_t count, const int64_t* i, const int64_t* j, int64_t* z,
                void* stream) {
  pool_init();
  if (d < 1 || d > 31 || count < 0) return QTT_EINVAL;
  return z_index(d, count, i, j, z, S(stream));
}

int qtt_gemm(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k, double alpha,
             const double* a, int64_t lda, const double* b, int64_t ldb, double beta, double* c,
             int64_t ldc, void* stream) {
  pool_init();
  if (m < 0 || n < 0 || k < 0 || m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff)
    return QTT_EINVAL;
  return dgemm(S(stream), trans_a, trans_b, (int)m, (int)n, (int)k, alpha, a, lda, b, ldb, beta, c,
               ldc);
}

int qtt_gemm_structured(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n, int64_t k,
                        double alpha, const double* a, int64_t lda, const double* b, int64_t ldb,
                        double beta, double* c, int64_t ldc, int32_t flags, void* stream) {
  pool_init();
  if (m < 0 || n < 0 || k < 0 || m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff ||
      (flags & ~31) != 0)
    return QTT_EINVAL;
  return dgemm(S(stream), trans_a, trans_b, (int)m, (int)n, (int)k, alpha, a, lda, b, ldb, beta, c,
               ldc, flags);
}

int qtt_qr(int64_t m, int64_t n, const double* a, int64_t lda, double* q, int64_t ldq, double* r,
           int64_t ldr, void* stream) {
  pool_init();
  if (m < 1 || n < 1 || m > 0x7fffffff || n > 0x7fffffff) return QTT_EINVAL;
  return qr(S(stream), (int)m, (int)n, a, lda, q, ldq, r, ldr);
}

int qtt_svd(int64_t m, int64_t n, const double* a, int64_t lda, double* s, double* u, int64_t ldu,
            void* stream) {
  pool_init();
  if (m < 1 || n < 1 || m > 0x7fffffff || n > 0x7fffffff) return QTT_EINVAL;
  cudaStream_t st = S(stream);
  const int M = (int)m, N = (int)n, k = std::min(M, N);
  // tall: A = Q R, R^T W = Z, U = Q W;  wide: A^T = Q2 R2, R2 W = Z, U = W.
  double *Q = nullptr, *R = nullptr, *X = nullptr, *W = nullptr, *tmp = nullptr;
  int* perm = nullptr;
  int* rank = nullptr;
  QTT_CUDA(malloc_async(&R, sizeof(double) * (int64_t)k * std::max(M, N), st));
  QTT_CUDA(malloc_async(&X, sizeof(double) * (int64_t)k * k, st));
  QTT_CUDA(malloc_async(&W, sizeof(double) * (int64_t)k * k, st));
  QTT_CUDA(malloc_async(&perm, sizeof(int) * (k + 2), st));
  rank = perm + k;
  if (M >= N) {
    QTT_CUDA(malloc_async(&Q, sizeof(double) * (int64_t)M * k, st));
    QTT_CUDA(malloc_async(&tmp, sizeof(double) * (int64_t)M * k, st));
    QTT_TRY(qr(st, M, N, a, lda, Q, M, R, k, nullptr, true));  // SVD inputs are ill-conditioned by design
    QTT_TRY(transpose(st, k, k, R, k, X, k));
    QTT_TRY(jacobi(st, k, k, X, k, W, k));
    QTT_TRY(sort_chop(st, k, k, X, k, s, perm, nullptr, 0.0, k, 0, rank));
    QTT_TRY(gather_columns(st, k, k, W, k, perm, X, k));
    QTT_TRY(dgemm(st, 0, 0, M, k, k, 1.0, Q, M, X, k, 0.0, u, ldu));
    QTT_CUDA(cudaFreeAsync(Q, st));
    QTT_CUDA(cudaFreeAsync(tmp, st));
  } else {
    QTT_CUDA(malloc_async(&tmp, sizeof(double) * (int64_t)M * N, st));
    QTT_TRY(transpose(st, M, N, a, lda, tmp, N));
    QTT_TRY(qr(st, N, M, tmp, N, nullptr, 1, R, k, nullptr, true));
    QTT_TRY(copy_matrix(st, k, k, R, k, X, k));
    QTT_TRY(jacobi(st, k, k, X, k, W, k));
    QTT_TRY(sort_chop(st, k, k, X, k, s, perm, nullptr, 0.0, k, 0, rank));
    QTT_TRY(gather_columns(st, k, k, W, k, perm, u, ldu));
    QTT_CUDA(cudaFreeAsync(tmp, st));
  }
  QTT_CUDA(cudaFreeAsync(R, st));
  QTT_CUDA(cudaFreeAsync(X, st));
  QTT_CUDA(cudaFreeAsync(W, st));
  QTT_CUDA(cudaFreeAsync(perm, st));
  return QTT_OK;
}

}  // extern "C"
