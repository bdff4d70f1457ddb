// Restarted GMRES for the AMEn local systems (row a13), replacing the
// scipy.sparse.linalg.gmres call of solver._solve_local (solver.py:186-195:
// restart 40, rtol, atol 0, warm start from the current core).
//
// The local operator is never formed: M x = sum_ab phi_l[:,a,:] A[a,:,:,b]
// phi_r[:,b,:] applied as three DMMA GEMMs and two index permutations
// (solver._proj_a).  The Arnoldi basis lives in HBM as (restart+1) rows of
// length dim; classical Gram-Schmidt is done twice (two GEMV-shaped GEMM
// pairs) for orthogonality.  Only the (j+2)-vector of Hessenberg entries
// crosses to the host per iteration, where the Givens rotations and the
// convergence test live; the whole cycle is driven from C++ so an iteration
// costs ~10 launches and one small D2H copy.
#include <cmath>
#include <vector>

#include "../../include/qtt_b200.h"
#include "linalg.cuh"

namespace qtt {
namespace {

// out = permutation of a row-major 4-D tensor: out dims are in dims
// (p0, p1, p2, p3); out[i0,i1,i2,i3] = in[j] with j_{p_k} = i_k.
struct Perm4 {
  int64_t od[4];       // output dims
  int64_t istride[4];  // input stride of the input dim feeding output dim k
};

__global__ void permute4_kernel(Perm4 P, int64_t total, const double* __restrict__ in,
                                double* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = o, src = 0;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      const int64_t i = rem % P.od[k];
      rem /= P.od[k];
      src += i * P.istride[k];
    }
    out[o] = in[src];
  }
}

int permute4(cudaStream_t s, const int64_t dims[4], const int p[4], const double* in, double* out) {
  int64_t stride[4];
  stride[3] = 1;
  for (int k = 2; k >= 0; --k) stride[k] = stride[k + 1] * dims[k + 1];
  Perm4 P;
  for (int k = 0; k < 4; ++k) {
    P.od[k] = dims[p[k]];
    P.istride[k] = stride[p[k]];
  }
  const int64_t total = dims[0] * dims[1] * dims[2] * dims[3];
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16 * num_sms()));
  permute4_kernel<<<grid, 256, 0, s>>>(P, total, in, out);
  QTT_CHECK_LAUNCH();
  return kOk;
}

// y = b - y (in place)
__global__ void rsub_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[i] - y[i];
}

// v *= 1 / *den  (no-op when *den == 0)
__global__ void scale_by_kernel(int64_t n, const double* __restrict__ den, double* __restrict__ v) {
  const double d = *den;
  if (d == 0.0) return;
  const double inv = 1.0 / d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] *= inv;
}


// Classical Gram-Schmidt building blocks (memory bound; replace GEMV-shaped
// GEMMs that waste 63/64 of a DMMA tile).  V is row-major (nv x dim).
constexpr int MD_THREADS = 256, MD_E = 4;  // up to MD_E elements per thread

// part[blk * nv + i] = sum over block chunk of V[i, t] * w[t]
__global__ void __launch_bounds__(MD_THREADS) mdot_partial_kernel(int nv, int64_t dim,
                                                                  const double* __restrict__ V,
                                                                  const double* __restrict__ w,
                                                                  double* __restrict__ part, int ce) {
  __shared__ double red[MD_THREADS / 32][64];
  const int64_t base = (int64_t)blockIdx.x * MD_THREADS * ce + threadIdx.x;
  double wv[MD_E];
#pragma unroll
  for (int e = 0; e < MD_E; ++e) {
    const int64_t t = base + e * MD_THREADS;
    wv[e] = (e < ce && t < dim) ? w[t] : 0.0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < nv; ++i) {
    const double* vi = V + (int64_t)i * dim;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < MD_E; ++e) {
      const int64_t t = base + e * MD_THREADS;
      if (e < ce && t < dim) acc = fma(vi[t], wv[e], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp][i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += MD_THREADS) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < MD_THREADS / 32; ++q) acc += red[q][i];
    part[(int64_t)blockIdx.x * nv + i] = acc;
  }
}

// c_i = sum_b part[b * nv + i] (fixed order); w[t] += sign * sum_i V[i,t] c_i.
// Block 0 stores c to cout (when given); with npart the block's partial
// of ||w_new||^2 goes to npart[blockIdx.x].
__global__ void __launch_bounds__(MD_THREADS) vcomb_kernel(int nv, int64_t dim,
                                                           const double* __restrict__ V,
                                                           const double* __restrict__ part,
                                                           int nblk, double sign, double* w,
                                                           double* __restrict__ cout,
                                                           double* __restrict__ npart, int ce) {
  __shared__ double c[64];
  __shared__ double tmp[MD_THREADS / 64][64];
  __shared__ double red[MD_THREADS / 32];
  {
    const int i = threadIdx.x & 63, grp = threadIdx.x >> 6;
    if (i < nv) {
      double acc = 0.0;
      for (int b = grp; b < nblk; b += MD_THREADS / 64) acc += part[(int64_t)b * nv + i];
      tmp[grp][i] = acc;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < MD_THREADS / 64; ++q) acc += tmp[q][threadIdx.x];
    c[threadIdx.x] = acc;
    if (cout && blockIdx.x == 0) cout[threadIdx.x] = acc;
  }
  __syncthreads();
  double nacc = 0.0;
  const int64_t base = (int64_t)blockIdx.x * MD_THREADS * ce + threadIdx.x;
#pragma unroll
  for (int e = 0; e < MD_E; ++e) {
    const int64_t t = base + e * MD_THREADS;
    if (e < ce && t < dim) {
      double acc = 0.0;
      for (int i = 0; i < nv; ++i) acc = fma(V[(int64_t)i * dim + t], c[i], acc);
      const double v = fma(sign, acc, w[t]);
      w[t] = v;
      nacc = fma(v, v, nacc);
    }
  }
  if (npart) {
    nacc = warp_sum(nacc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < MD_THREADS / 32; ++q) t += red[q];
      npart[blockIdx.x] = t;
    }
  }
}

// hv[i] = h[i] + h2[i] (i < nv), hv[nv] = sqrt(sum npart)
__global__ void hess_col_kernel(int nv, const double* __restrict__ h, const double* __restrict__ h2,
                                const double* __restrict__ npart, int nblk, double* __restrict__ hv) {
  __shared__ double red[32];
  double a = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) a += npart[b];
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) hv[nv] = sqrt(v);
  }
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hv[i] = h[i] + h2[i];
}

inline int elem_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 8 * num_sms()));
}

// Row-major C (M x N) = A (M x K) * op(B), op(B) = B (K x N) or, with tb,
// B^T for B stored row-major N x K.  Issued as the column-major C^T = op(B)^T A^T.
inline int mm_rm(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                 bool tb, double* C, double alpha = 1.0, double beta = 0.0) {
  return dgemm(s, tb ? 1 : 0, 0, (int)N, (int)M, (int)K, alpha, B, tb ? K : N, A, K, beta, C, N);
}

struct LocalOp {
  int64_t rl, n, rr, ra, rb;
  const double *phil, *ajib, *phir;
  double *t1, *p1;  // rl*ra*n*rr each (t2/p2 reuse them: rl*rr*n*rb)
};

// y = M x (solver._proj_a): x, y have rl*n*rr entries.
int local_apply(cudaStream_t s, const LocalOp& op, const double* x, double* y) {
  const int64_t z = op.rl, a = op.ra, n = op.n, R = op.rr, b = op.rb;
  QTT_TRY(mm_rm(s, z * a, n * R, z, op.phil, x, false, op.t1));  // (z,a,j,R)
  {
    const int64_t dims[4] = {z, a, n, R};
    const int p[4] = {0, 3, 1, 2};
    QTT_TRY(permute4(s, dims, p, op.t1, op.p1));  // (z,R,a,j)
  }
  QTT_TRY(mm_rm(s, z * R, n * b, a * n, op.p1, op.ajib, false, op.t1));  // (z,R,i,b)
  {
    const int64_t dims[4] = {z, R, n, b};
    const int p[4] = {0, 2, 3, 1};
    QTT_TRY(permute4(s, dims, p, op.t1, op.p1));  // (z,i,b,R)
  }
  return mm_rm(s, z * n, R, b * R, op.p1, op.phir, true, y);  // (z,i,Z)
}

struct DevMem {
  std::vector<std::pair<void*, cudaStream_t>> v;
  template <typename T>
  int get(cudaStream_t s, T** p, int64_t n) {
    QTT_CUDA(malloc_async(reinterpret_cast<void**>(p), sizeof(T) * std::max<int64_t>(n, 1), s));
    v.emplace_back(*p, s);
    return kOk;
  }
  ~DevMem() {
    for (auto& e : v) cudaFreeAsync(e.first, e.second);
  }
};

double* pinned_scratch(int64_t n) {
  thread_local double* buf = nullptr;
  thread_local int64_t cap = 0;
  if (n > cap) {
    if (buf) cudaFreeHost(buf);
    cap = std::max<int64_t>(n, 256);
    if (cudaMallocHost(&buf, sizeof(double) * cap) != cudaSuccess) {
      buf = nullptr;
      cap = 0;
    }
  }
  return buf;
}

}  // namespace

int local_gmres(cudaStream_t s, const LocalOp& op, const double* rhs, const double* x0, double* x,
                double rtol, int restart, int maxit, int abort_early, int* iters, int* converged) {
  const int64_t dim = op.rl * op.n * op.rr;
  *iters = 0;
  *converged = 0;
  DevMem mem;
  if (restart > 63) return kInvalid;  // Hessenberg columns live in 64-entry smem
  // elements per thread: enough blocks to cover the SMs at small dims
  const int ce = dim >= (int64_t)MD_THREADS * 4 * num_sms() ? 4 : dim >= (int64_t)MD_THREADS * 2 * num_sms() ? 2 : 1;
  const int nblk = (int)ceil_div(dim, (int64_t)MD_THREADS * ce);
  double *V, *h, *h2, *hv, *yv, *part, *npart;
  QTT_TRY(mem.get(s, &part, (int64_t)nblk * (restart + 1)));
  QTT_TRY(mem.get(s, &npart, nblk));
  QTT_TRY(mem.get(s, &V, (int64_t)(restart + 1) * dim));
  QTT_TRY(mem.get(s, &h, restart + 2));
  QTT_TRY(mem.get(s, &h2, restart + 2));
  QTT_TRY(mem.get(s, &hv, restart + 2));
  QTT_TRY(mem.get(s, &yv, restart + 2));
  double* host = pinned_scratch(restart + 2);
  if (!host) return kCuda;

  if (x != x0) QTT_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * dim, cudaMemcpyDeviceToDevice, s));
  QTT_TRY(frob_norm(s, dim, rhs, hv));
  QTT_CUDA(cudaMemcpyAsync(host, hv, sizeof(double), cudaMemcpyDeviceToHost, s));
  QTT_CUDA(cudaStreamSynchronize(s));
  const double bn = host[0];
  if (bn == 0.0) {
    QTT_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * dim, s));
    *converged = 1;
    return kOk;
  }
  const double target = rtol * bn;
  std::vector<double> H((size_t)(restart + 1) * restart), cs(restart), sn(restart), g(restart + 1),
      y(restart);
  auto Hat = [&](int i, int j) -> double& { return H[(size_t)j * (restart + 1) + i]; };
  int total = 0;
  while (true) {
    // r = b - M x -> V[0]; beta = ||r||
    QTT_TRY(local_apply(s, op, x, V));
    rsub_kernel<<<elem_grid(dim), 256, 0, s>>>(dim, rhs, V);
    QTT_CHECK_LAUNCH();
    QTT_TRY(frob_norm(s, dim, V, hv));
    QTT_CUDA(cudaMemcpyAsync(host, hv, sizeof(double), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    const double beta = host[0];
    if (beta <= target) {
      *converged = 1;
      break;
    }
    if (total >= maxit) break;
    scale_by_kernel<<<elem_grid(dim), 256, 0, s>>>(dim, hv, V);
    QTT_CHECK_LAUNCH();
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int jend = 0;
    for (int j = 0; j < restart; ++j) {
      double* w = V + (int64_t)(j + 1) * dim;
      QTT_TRY(local_apply(s, op, V + (int64_t)j * dim, w));
      // CGS2: h = V^T w, w -= V h (twice), then ||w|| (fused into the 2nd update)
      const int nv = j + 1;
      mdot_partial_kernel<<<nblk, MD_THREADS, 0, s>>>(nv, dim, V, w, part, ce);
      QTT_CHECK_LAUNCH();
      vcomb_kernel<<<nblk, MD_THREADS, 0, s>>>(nv, dim, V, part, nblk, -1.0, w, h, nullptr, ce);
      QTT_CHECK_LAUNCH();
      mdot_partial_kernel<<<nblk, MD_THREADS, 0, s>>>(nv, dim, V, w, part, ce);
      QTT_CHECK_LAUNCH();
      vcomb_kernel<<<nblk, MD_THREADS, 0, s>>>(nv, dim, V, part, nblk, -1.0, w, h2, npart, ce);
      QTT_CHECK_LAUNCH();
      hess_col_kernel<<<1, 256, 0, s>>>(nv, h, h2, npart, nblk, hv);
      QTT_CHECK_LAUNCH();
      QTT_CUDA(cudaMemcpyAsync(host, hv, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, s));
      scale_by_kernel<<<elem_grid(dim), 256, 0, s>>>(dim, hv + j + 1, w);
      QTT_CHECK_LAUNCH();
      QTT_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i < j + 2; ++i) Hat(i, j) = host[i];
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hat(i, j) + sn[i] * Hat(i + 1, j);
        Hat(i + 1, j) = -sn[i] * Hat(i, j) + cs[i] * Hat(i + 1, j);
        Hat(i, j) = t;
      }
      const double den = std::hypot(Hat(j, j), Hat(j + 1, j));
      if (den == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = Hat(j, j) / den;
        sn[j] = Hat(j + 1, j) / den;
      }
      Hat(j, j) = den;
      Hat(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      jend = j + 1;
      if (std::fabs(g[j + 1]) <= target || total >= maxit || host[j + 1] == 0.0) break;
    }
    // x += V[:jend]^T y with H y = g (upper triangular)
    for (int i = jend - 1; i >= 0; --i) {
      double acc = g[i];
      for (int l = i + 1; l < jend; ++l) acc -= Hat(i, l) * y[l];
      y[i] = acc / Hat(i, i);
    }
    for (int i = 0; i < jend; ++i) host[i] = y[i];
    QTT_CUDA(cudaMemcpyAsync(yv, host, sizeof(double) * jend, cudaMemcpyHostToDevice, s));
    vcomb_kernel<<<nblk, MD_THREADS, 0, s>>>(jend, dim, V, yv, 1, 1.0, x, nullptr, nullptr, ce);
    QTT_CHECK_LAUNCH();
    // the pinned buffer is reused by the next cycle: the H2D copy must land first
    QTT_CUDA(cudaStreamSynchronize(s));
    // Early abort (the caller has a dense fallback): project the iterations
    // still needed from this cycle's convergence rate.
    if (abort_early && jend == restart && std::fabs(g[jend]) > target) {
      const double rate = std::pow(std::fabs(g[jend]) / beta, 1.0 / jend);
      if (!(rate < 1.0)) break;
      const double need = std::log(target / std::fabs(g[jend])) / std::log(rate);
      if (total + need > 1.25 * maxit) break;
    }
  }
  *iters = total;
  return kOk;
}

}  // namespace qtt

extern "C" int qtt_local_gmres(int64_t rl, int64_t n, int64_t rr, int64_t ra, int64_t rb,
                               const double* phi_l, const double* a_jib, const double* phi_r,
                               const double* rhs, const double* x0, double* x, double rtol,
                               int32_t restart, int32_t maxit, int32_t abort_early, int32_t* iters,
                               int32_t* converged, void* stream) {
  qtt::pool_init();
  if (rl < 1 || n < 1 || rr < 1 || ra < 1 || rb < 1 || restart < 1 || maxit < 0 || !iters ||
      !converged)
    return QTT_EINVAL;
  const int64_t dim = rl * n * rr;
  const int64_t work = std::max(rl * ra * n * rr, rl * rr * n * rb);
  if (dim > 0x7fffffff || work > ((int64_t)1 << 40)) return QTT_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double *t1 = nullptr, *p1 = nullptr;
  QTT_CUDA(qtt::malloc_async(&t1, sizeof(double) * work, s));
  QTT_CUDA(qtt::malloc_async(&p1, sizeof(double) * work, s));
  qtt::LocalOp op{rl, n, rr, ra, rb, phi_l, a_jib, phi_r, t1, p1};
  int it = 0, conv = 0;
  const int st = qtt::local_gmres(s, op, rhs, x0, x, rtol, restart, maxit, abort_early, &it, &conv);
  cudaFreeAsync(t1, s);
  cudaFreeAsync(p1, s);
  *iters = it;
  *converged = conv;
  return st;
}

extern "C" int qtt_local_apply(int64_t rl, int64_t n, int64_t rr, int64_t ra, int64_t rb,
                               const double* phi_l, const double* a_jib, const double* phi_r,
                               const double* x, double* y, void* stream) {
  qtt::pool_init();
  if (rl < 1 || n < 1 || rr < 1 || ra < 1 || rb < 1) return QTT_EINVAL;
  const int64_t work = std::max(rl * ra * n * rr, rl * rr * n * rb);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double *t1 = nullptr, *p1 = nullptr;
  QTT_CUDA(qtt::malloc_async(&t1, sizeof(double) * work, s));
  QTT_CUDA(qtt::malloc_async(&p1, sizeof(double) * work, s));
  qtt::LocalOp op{rl, n, rr, ra, rb, phi_l, a_jib, phi_r, t1, p1};
  const int st = qtt::local_apply(s, op, x, y);
  cudaFreeAsync(t1, s);
  cudaFreeAsync(p1, s);
  return st;
}
