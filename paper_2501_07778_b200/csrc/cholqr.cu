// CholeskyQR2 for the large, well-conditioned unfoldings of TT rounding.
//
// Householder QR of an m x n matrix needs n sequential column reductions
// (the panel); for the 4096 x 2048 unfoldings of the BASELINE config-2
// rounding that latency dominates.  CholeskyQR2 replaces it with four large
// DMMA GEMMs (A^T A, A R1^{-1}, Q1^T Q1, Q1 R2^{-1}), two blocked Cholesky
// factorisations of the n x n Gram matrices and two triangular inversions.
// It is exact-arithmetic QR and numerically orthogonal to O(eps) whenever
// cond(A) is below ~eps^{-1/2}; the second pass is certified by checking
// ||Q1^T Q1 - I||_F <= 1/4 (then cond(Q1) <= 1.3 and Q = Q1 R2^{-1} is
// orthogonal to working accuracy).  Otherwise the caller falls back to
// Householder (rank-deficient assembly/solver unfoldings).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "linalg.cuh"

namespace qtt {
namespace {

constexpr int CB = 64;  // Cholesky block
constexpr int kDefectParts = 296;

// One block step of the blocked Cholesky, fused: every CTA factors the
// kb x kb diagonal block G11 = R11^T R11 in registers (redundantly; it is a
// few microseconds and saves a launch + a dependency), CTA 0 writes R11 to
// `rblk` (64 x 64, ld 64; copied into G after the last step, because other
// CTAs may still be reading G11), and each CTA solves 64 columns of the
// block row in place, G12 <- R11^{-T} G12, by forward substitution with four
// lanes per column: the pivot entry travels by warp shuffle, no barriers.
__global__ void __launch_bounds__(256) chol_panel_kernel(int kb, const double* __restrict__ G11,
                                                         int64_t ldg, double* __restrict__ rblk,
                                                         double* __restrict__ G12, int rest,
                                                         int* __restrict__ bad) {
  __shared__ double S[kBlk][kBlk + 1];
  __shared__ __align__(16) double line[256];
  __shared__ double dinv[kBlk];
  double a[16];
  blk_load(a, G11, ldg, kb);
  blk_factor<true>(a, line, bad);
  if (blockIdx.x == 0) blk_store(a, rblk, kBlk, kBlk);
  const int col = blockIdx.x * kBlk + blk_col();
  if (blockIdx.x * kBlk >= rest) return;
  blk_to_smem(a, S);
  __syncthreads();
  if (threadIdx.x < kBlk) dinv[threadIdx.x] = 1.0 / S[threadIdx.x][threadIdx.x];
  const int part = blk_part(), lane = threadIdx.x & 31;
  const bool act = col < rest;
  double x[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int i = part + 4 * q;
    x[q] = (act && i < kb) ? G12[i + (int64_t)col * ldg] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kBlk; ++j) {
    const int qj = j >> 2, pj = j & 3;
    const double v = x[qj] * dinv[j];
    const double xj = -__shfl_sync(0xffffffffu, v, (lane & ~3) | pj);
    const double* r = &S[j][part];
    if (part == pj) x[qj] = v;
    if (part > pj) x[qj] = fma(r[4 * qj], xj, x[qj]);
#pragma unroll
    for (int q = qj + 1; q < 16; ++q) x[q] = fma(r[4 * q], xj, x[q]);
  }
  if (act) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      if (i < kb) G12[i + (int64_t)col * ldg] = x[q];
    }
  }
}

// G(diag block b) <- rblk[b] (upper incl. diagonal; strictly lower zero) and
// zero block column b below its diagonal block.
__global__ void __launch_bounds__(256) chol_diag_writeback_kernel(int n, const double* __restrict__ rblk,
                                                                  double* __restrict__ G, int64_t ldg) {
  const int b0 = blockIdx.x * kBlk;
  const int kb = min(kBlk, n - b0);
  const double* src = rblk + (int64_t)blockIdx.x * kBlk * kBlk;
  if (blockIdx.y == 0)
    for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
      const int r = idx % kb, c = idx / kb;
      G[(b0 + r) + (int64_t)(b0 + c) * ldg] = src[r + c * kBlk];
    }
  const int below = n - b0 - kb;
  for (int64_t idx = blockIdx.y * blockDim.x + threadIdx.x; idx < (int64_t)below * kb;
       idx += (int64_t)gridDim.y * blockDim.x) {
    const int r = (int)(idx % below), c = (int)(idx / below);
    G[(b0 + kb + r) + (int64_t)(b0 + c) * ldg] = 0.0;
  }
}

// partial sums of squares of (G - I) for the orthogonality certificate
__global__ void gram_defect_kernel(int n, const double* __restrict__ G, int64_t ldg,
                                   double* out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n * n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % n), c = (int)(i / n);
    if (r > c) continue;  // G holds its upper triangle only
    const double v = G[r + (int64_t)c * ldg] - (r == c ? 1.0 : 0.0);
    a = fma(r == c ? v : 2.0 * v, v, a);
  }
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[blockIdx.x] = t;
  }
}

__global__ void sum_parts_kernel(int n, const double* __restrict__ part, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

// U <- split(G - I - W): strictly upper part of (G - I - W) plus half its
// diagonal (upper triangle of U, lower zeroed).  W may be null (W = 0).
__global__ void near_identity_split_kernel(int n, const double* __restrict__ G, int64_t ldg,
                                           const double* __restrict__ W, int64_t ldw,
                                           double* __restrict__ U, int64_t ldu) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % n), c = (int)(idx / n);
    double v = 0.0;
    if (r <= c) {
      v = G[r + (int64_t)c * ldg] - (r == c ? 1.0 : 0.0);
      if (W) v -= W[r + (int64_t)c * ldw];
      if (r == c) v *= 0.5;
    }
    U[r + (int64_t)c * ldu] = v;
  }
}

// G <- I + U (upper), in place.
__global__ void add_identity_kernel(int n, const double* __restrict__ U, int64_t ldu,
                                    double* __restrict__ G, int64_t ldg) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % n), c = (int)(idx / n);
    G[r + (int64_t)c * ldg] = U[r + (int64_t)c * ldu] + (r == c ? 1.0 : 0.0);
  }
}

// Cholesky factor of a Gram matrix close to the identity, G = I + E with
// ||E||_F = delta small (the second CholeskyQR pass), without the
// sequential factorisation: R = I + U with U upper triangular solving
// U + U^T = E - U^T U, by the fixed-point iteration
//   U_0 = split(E),  U_{k+1} = split(E - U_k^T U_k),
// split = strict upper part + half the diagonal.  The error contracts as
// delta^(k+2), so `iters` = smallest k with delta^(k+2) <= 1e-17; each
// iteration is one triangular DMMA GEMM (lower x upper, upper tiles only).
int chol_near_identity(cudaStream_t s, int n, double* G, int64_t ldg, double* U, double* W,
                       int iters) {
  const int64_t nn = n;
  const int blocks = (int)std::min<int64_t>(ceil_div(nn * nn, 256), 8 * num_sms());
  near_identity_split_kernel<<<blocks, 256, 0, s>>>(n, G, ldg, nullptr, 0, U, nn);
  QTT_CHECK_LAUNCH();
  for (int it = 0; it < iters; ++it) {
    QTT_TRY(dgemm(s, 1, 0, n, n, n, 1.0, U, nn, U, nn, 0.0, W, nn,
                  kGemmUpperC | kGemmLowA | kGemmTriB));
    near_identity_split_kernel<<<blocks, 256, 0, s>>>(n, G, ldg, W, nn, U, nn);
    QTT_CHECK_LAUNCH();
  }
  add_identity_kernel<<<blocks, 256, 0, s>>>(n, U, nn, G, ldg);
  QTT_CHECK_LAUNCH();
  return kOk;
}

// Blocked right-looking upper Cholesky G = R^T R (in place).  rblk: scratch
// for the ceil(n/64) diagonal factors (64 x 64 each).
//
// Look-ahead of depth one: the critical path (panel k = factor + block-row
// solve, then the update of block row k+1 only, "a_k") runs on the
// high-priority side stream, while the rest of the trailing update ("b_k",
// rows/cols beyond block k+1, upper tiles) runs on `s` concurrently with
// panel k+1.  Dependencies: a_k after b_{k-1} (both update block row k+1),
// b_k after panel k; disjoint writes otherwise.
int chol_upper(cudaStream_t s, int n, double* G, int64_t ldg, double* rblk, int* bad) {
  thread_local cudaEvent_t ev[6] = {};
  if (!ev[0])
    for (auto& e : ev) QTT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t *evP = ev, *evB = ev + 2, evStart = ev[4], evEnd = ev[5];
  cudaStream_t ss = side_stream();
  const bool ahead = ss != s && !getenv("QTT_NO_LOOKAHEAD");
  cudaStream_t sp = ahead ? ss : s;  // critical-path stream
  if (ahead) {
    QTT_CUDA(cudaEventRecord(evStart, s));
    QTT_CUDA(cudaStreamWaitEvent(ss, evStart, 0));
  }
  int nblk = 0;
  for (int k0 = 0; k0 < n; k0 += CB, ++nblk) {
    const int k = nblk;
    const int kb = std::min(CB, n - k0);
    const int rest = n - k0 - kb;
    const double* Gkk = G + k0 + (int64_t)k0 * ldg;
    double* G12 = G + k0 + (int64_t)(k0 + kb) * ldg;
    chol_panel_kernel<<<std::max(1, (int)ceil_div(rest, CB)), 256, 0, sp>>>(
        kb, Gkk, ldg, rblk + (int64_t)k * CB * CB, G12, rest, bad);
    QTT_CHECK_LAUNCH();
    if (rest <= 0) continue;
    const int kb1 = std::min(CB, rest), rest2 = rest - kb1;
    double* G22 = G + (k0 + kb) + (int64_t)(k0 + kb) * ldg;
    if (ahead) QTT_CUDA(cudaEventRecord(evP[k & 1], ss));
    // a_k: block row k+1 -= R12[:, :kb1]^T R12
    if (ahead && k > 0) QTT_CUDA(cudaStreamWaitEvent(ss, evB[(k - 1) & 1], 0));
    QTT_TRY(dgemm(sp, 1, 0, kb1, rest, kb, -1.0, G12, ldg, G12, ldg, 1.0, G22, ldg));
    if (rest2 <= 0) continue;
    // b_k: the rest of G22 (upper tiles)
    if (ahead) QTT_CUDA(cudaStreamWaitEvent(s, evP[k & 1], 0));
    const double* R12b = G12 + (int64_t)kb1 * ldg;
    QTT_TRY(dgemm(s, 1, 0, rest2, rest2, kb, -1.0, R12b, ldg, R12b, ldg, 1.0,
                  G22 + kb1 + (int64_t)kb1 * ldg, ldg, kGemmUpperC));
    if (ahead) QTT_CUDA(cudaEventRecord(evB[k & 1], s));
  }
  if (ahead) {
    QTT_CUDA(cudaEventRecord(evEnd, ss));
    QTT_CUDA(cudaStreamWaitEvent(s, evEnd, 0));
  }
  chol_diag_writeback_kernel<<<dim3(nblk, 16), 256, 0, s>>>(n, rblk, G, ldg);
  QTT_CHECK_LAUNCH();
  return kOk;
}

__global__ void gram_trace_kernel(int n, const double* __restrict__ G, int64_t ldg, double* out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += G[i + (int64_t)i * ldg];
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// sc[0] = ||X||_F^2 (trace of G), sc[1] = ||R^{-1}||_F
__global__ void gram_certificate_kernel(int p, int r, const double* sc, const int* bad,
                                        const double* delta_dev, double delta_scale, int* ok,
                                        int debug) {
  const double eps = 2.220446049250313e-16;
  const double x2 = sc[0], xn = sc[1];
  const double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
  const double thr = 1.25 * fmax(delta, sqrt(fmax(x2, 0.0)) * (double)max(r, 2) * eps);
  const double lower = 1.0 / (xn * xn) - 2.0 * (double)(p + r + 2) * eps * x2;
  const bool good = !*bad && isfinite(xn) && isfinite(x2) && xn > 0.0 && lower > thr * thr;
  *ok = good ? 1 : 0;
  if (debug)
    printf("[gram-cert] p=%d r=%d smin^2/|X|^2 >= %.3e thr^2/|X|^2=%.3e bad=%d good=%d\n", p, r,
           lower / x2, thr * thr / x2, *bad, (int)good);
}

}  // namespace

int gram_certificate(cudaStream_t s, int p, int r, const double* X, int64_t ldx,
                     const double* delta_dev, double delta_scale, int* ok_dev) {
  if (p < r || r <= 0) return kInvalid;
  const int64_t nn = r;
  double *G, *Ri, *rblk, *sc;
  int* bad;
  QTT_CUDA(cudaMallocAsync(&G, sizeof(double) * nn * nn, s));
  QTT_CUDA(cudaMallocAsync(&Ri, sizeof(double) * nn * nn, s));
  QTT_CUDA(cudaMallocAsync(&rblk, sizeof(double) * CB * CB * ceil_div(nn, CB), s));
  QTT_CUDA(cudaMallocAsync(&sc, sizeof(double) * 4, s));
  QTT_CUDA(cudaMallocAsync(&bad, sizeof(int), s));
  QTT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  int status = kOk;
  do {
    if ((status = dgemm(s, 1, 0, r, r, p, 1.0, X, ldx, X, ldx, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    gram_trace_kernel<<<1, 256, 0, s>>>(r, G, nn, sc);
    QTT_CHECK_LAUNCH();
    if ((status = chol_upper(s, r, G, nn, rblk, bad)) != kOk) break;
    if ((status = tri_inverse(s, r, G, nn, Ri)) != kOk) break;
    if ((status = frob_norm(s, nn * nn, Ri, sc + 1)) != kOk) break;
    static const int debug = getenv("QTT_CERT_DEBUG") ? 1 : 0;
    gram_certificate_kernel<<<1, 1, 0, s>>>(p, r, sc, bad, delta_dev, delta_scale, ok_dev, debug);
    QTT_CHECK_LAUNCH();
  } while (false);
  QTT_CUDA(cudaFreeAsync(G, s));
  QTT_CUDA(cudaFreeAsync(Ri, s));
  QTT_CUDA(cudaFreeAsync(rblk, s));
  QTT_CUDA(cudaFreeAsync(sc, s));
  QTT_CUDA(cudaFreeAsync(bad, s));
  return status;
}

int cholqr2(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
            double* R, int64_t ldr, int* ok) {
  *ok = 0;
  if (m < n || n <= 0) return kOk;
  const int64_t nn = n;
  double *G, *R1, *Ri, *Q1, *rblk, *scal, *parts;
  int* bad;
  QTT_CUDA(cudaMallocAsync(&G, sizeof(double) * nn * nn, s));
  QTT_CUDA(cudaMallocAsync(&R1, sizeof(double) * nn * nn, s));
  QTT_CUDA(cudaMallocAsync(&Ri, sizeof(double) * nn * nn, s));
  QTT_CUDA(cudaMallocAsync(&Q1, sizeof(double) * (int64_t)m * nn, s));
  QTT_CUDA(cudaMallocAsync(&rblk, sizeof(double) * CB * CB * ceil_div(nn, CB), s));
  QTT_CUDA(cudaMallocAsync(&scal, sizeof(double) * 4, s));
  QTT_CUDA(cudaMallocAsync(&parts, sizeof(double) * kDefectParts, s));
  QTT_CUDA(cudaMallocAsync(&bad, sizeof(int), s));
  QTT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  int status = kOk;
  do {
    // pass 1: G = A^T A = R1^T R1, Q1 = A R1^{-1}
    if ((status = dgemm(s, 1, 0, n, n, m, 1.0, A, lda, A, lda, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    if ((status = chol_upper(s, n, G, nn, rblk, bad)) != kOk) break;
    int hbad = 0;
    QTT_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    if (hbad) break;
    QTT_CUDA(cudaMemcpyAsync(R1, G, sizeof(double) * nn * nn, cudaMemcpyDeviceToDevice, s));
    if ((status = tri_inverse(s, n, R1, nn, Ri)) != kOk) break;
    if ((status = dgemm(s, 0, 0, m, n, n, 1.0, A, lda, Ri, nn, 0.0, Q1, m, kGemmTriB)) != kOk) break;
    // pass 2: certify cond(Q1) ~ 1, then G = Q1^T Q1 = R2^T R2, Q = Q1 R2^{-1}
    if ((status = dgemm(s, 1, 0, n, n, m, 1.0, Q1, m, Q1, m, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    gram_defect_kernel<<<kDefectParts, 256, 0, s>>>(n, G, nn, parts);
    QTT_CHECK_LAUNCH();
    sum_parts_kernel<<<1, 32, 0, s>>>(kDefectParts, parts, scal);
    QTT_CHECK_LAUNCH();
    double defect = 0.0;
    QTT_CUDA(cudaMemcpyAsync(&defect, scal, sizeof(double), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    if (getenv("QTT_QR_DEBUG")) fprintf(stderr, "[cholqr2] m=%d n=%d defect=%.3e\n", m, n, std::sqrt(defect));
    const double delta = std::sqrt(defect);
    if (!(delta <= 0.25)) break;
    if (delta <= 1e-2 && !getenv("QTT_NO_NEAR_IDENTITY")) {
      int iters = 0;
      while (iters < 8 && std::pow(std::max(delta, 1e-300), iters + 2) > 1e-17) ++iters;
      double *U, *W;
      QTT_CUDA(cudaMallocAsync(&U, sizeof(double) * nn * nn, s));
      QTT_CUDA(cudaMallocAsync(&W, sizeof(double) * nn * nn, s));
      status = chol_near_identity(s, n, G, nn, U, W, iters);
      QTT_CUDA(cudaFreeAsync(U, s));
      QTT_CUDA(cudaFreeAsync(W, s));
      if (status != kOk) break;
    } else {
      if ((status = chol_upper(s, n, G, nn, rblk, bad)) != kOk) break;
      QTT_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      QTT_CUDA(cudaStreamSynchronize(s));
      if (hbad) break;
    }
    if ((status = tri_inverse(s, n, G, nn, Ri)) != kOk) break;
    if ((status = dgemm(s, 0, 0, m, n, n, 1.0, Q1, m, Ri, nn, 0.0, Q, ldq, kGemmTriB)) != kOk) break;
    // R = R2 R1 (product of upper-triangular factors stays upper triangular)
    if ((status = dgemm(s, 0, 0, n, n, n, 1.0, G, nn, R1, nn, 0.0, R, ldr, kGemmTriA | kGemmTriB)) != kOk) break;
    *ok = 1;
  } while (false);
  QTT_CUDA(cudaFreeAsync(G, s));
  QTT_CUDA(cudaFreeAsync(R1, s));
  QTT_CUDA(cudaFreeAsync(Ri, s));
  QTT_CUDA(cudaFreeAsync(Q1, s));
  QTT_CUDA(cudaFreeAsync(rblk, s));
  QTT_CUDA(cudaFreeAsync(scal, s));
  QTT_CUDA(cudaFreeAsync(parts, s));
  QTT_CUDA(cudaFreeAsync(bad, s));
  return status;
}

}  // namespace qtt
