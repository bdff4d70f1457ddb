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
#ifdef QTT_PANEL_DEBUG
  const long long t0 = clock64();
#endif
  blk_load(a, G11, ldg, kb);
#ifdef QTT_PANEL_DEBUG
  const long long t1 = clock64();
#endif
  blk_factor<true>(a, line, bad);
#ifdef QTT_PANEL_DEBUG
  const long long t2 = clock64();
#endif
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
#ifdef QTT_PANEL_DEBUG
  const long long t3 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0 && rest > 1900)
    printf("[chol-panel] load %lld factor %lld solve %lld\n", t1 - t0, t2 - t1, t3 - t2);
#endif
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


// ---------------------------------------------------- small fused factor
// Cholesky factor AND its inverse of an n x n Gram matrix, n <= 128, in ONE
// CTA (the serial pivot chain of a small factorisation does not parallelise
// across CTAs, and one launch replaces ~12: panels, updates, write-back,
// diagonal inverses, doubling GEMMs).  G (upper triangle valid) = R^T R;
// writes R and Ri = R^{-1} (both n x n upper, strictly lower part zeroed).
// The matrix is handled as 2 x 2 blocks of 64: register factor of G11
// (common.cuh), forward substitution for R12 with four lanes per column,
// G22 - R12^T R12, register factor of R22, block inverses and
// X12 = -X11 R12 X22.
//
// defect_mode (second CholeskyQR pass, G = Q1^T Q1): defect_out[0] receives
// ||G - I||_F^2; if it is <= 1e-16 the factor is R = I + U, Ri = I - U with
// U = strict upper part of E plus half its diagonal (error ||U||^2), with no
// factorisation at all; above 1/16 (= (1/4)^2) the status flag is raised.
// *status |= 1 on a non-positive pivot or a failed defect test (sticky:
// speculative callers check it once per sweep).
constexpr int kCisSmem = (5 * kBlk * (kBlk + 1) + 256 + kBlk + 16) * (int)sizeof(double);

__device__ __forceinline__ double block_sum_256(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) t += red[w];
  return t;
}

typedef double (*CisBlk)[kBlk + 1];

// Inverse of the upper-triangular 2 x 2 block matrix [S11 S12; 0 S22] held in
// shared memory (identity padded): X11, X22 by register back substitution,
// X12 = -X11 S12 X22.  Writes the inverse to Ri (n = kb1 + kb2; may be null)
// and returns ||R^{-1}||_F^2 (of the unpadded n x n part).  S11 is
// overwritten.  All 256 threads of the CTA must call.
__device__ double cis_inverse(CisBlk S11, CisBlk S22, CisBlk S12, CisBlk X11, CisBlk X22, double* line,
                              double* dinv, double* red, int kb1, int kb2, double* __restrict__ Ri,
                              int64_t ldi) {
  const int c = blk_col(), part = blk_part();
  double a[16], x[16], y[16];
  double nrm = 0.0;
  blk_tri_inverse<false>(S11, x, y, line, dinv);
  if (Ri) blk_store(x, Ri, ldi, kb1);
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (part + 4 * q < kb1 && c < kb1) nrm = fma(x[q], x[q], nrm);
  if (kb2 > 0) {
    blk_to_smem(x, X11);
    __syncthreads();
    blk_tri_inverse<false>(S22, x, y, line, dinv);
    blk_to_smem(x, X22);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      if (i < kb2 && c < kb2) {
        nrm = fma(x[q], x[q], nrm);
        if (Ri) Ri[(kBlk + i) + (int64_t)(kBlk + c) * ldi] = x[q];
      }
    }
    __syncthreads();
    // T = S12 X22 (into S11, free now), X12 = -X11 T
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = 0.0;
    for (int k = 0; k <= c; ++k) {  // X22 upper triangular
      const double xc = X22[k][c];
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = fma(S12[part + 4 * q][k], xc, a[q]);
    }
    __syncthreads();
    blk_to_smem(a, S11);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = 0.0;
    for (int k = 0; k < kBlk; ++k) {
      const double tc = -S11[k][c];
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = fma(X11[part + 4 * q][k], tc, a[q]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      if (i < kb1 && c < kb2) {
        nrm = fma(a[q], a[q], nrm);
        if (Ri) Ri[i + (int64_t)(kBlk + c) * ldi] = a[q];
      }
    }
  }
  return block_sum_256(nrm, red);
}

__global__ void __launch_bounds__(256) chol_inv_small_kernel(int n, const double* __restrict__ G,
                                                             int64_t ldg, double* __restrict__ R,
                                                             int64_t ldr, double* __restrict__ Ri,
                                                             int64_t ldi, int defect_mode,
                                                             double* __restrict__ defect_out,
                                                             int* __restrict__ status) {
  extern __shared__ double cis_sm[];
  typedef double (*Blk)[kBlk + 1];
  Blk S11 = reinterpret_cast<Blk>(cis_sm);
  Blk S22 = reinterpret_cast<Blk>(cis_sm + 1 * kBlk * (kBlk + 1));
  Blk S12 = reinterpret_cast<Blk>(cis_sm + 2 * kBlk * (kBlk + 1));
  Blk X11 = reinterpret_cast<Blk>(cis_sm + 3 * kBlk * (kBlk + 1));
  Blk X22 = reinterpret_cast<Blk>(cis_sm + 4 * kBlk * (kBlk + 1));
  double* line = cis_sm + 5 * kBlk * (kBlk + 1);
  double* dinv = line + 256;
  double* red = dinv + kBlk;
  __shared__ int bad_s;
  const int tid = threadIdx.x;
  if (tid == 0) bad_s = 0;
  const int kb1 = min(kBlk, n), kb2 = n - kb1;
  const int c = blk_col(), part = blk_part(), lane = tid & 31;

  if (defect_mode) {
    double acc = 0.0;
    for (int idx = tid; idx < n * n; idx += 256) {
      const int i = idx % n, j = idx / n;
      if (i > j) continue;
      const double v = G[i + (int64_t)j * ldg] - (i == j ? 1.0 : 0.0);
      acc = fma(i == j ? v : 2.0 * v, v, acc);
    }
    const double d2 = block_sum_256(acc, red);
    if (tid == 0) {
      defect_out[0] = d2;
      defect_out[1] = (double)n;  // ||R2^{-1}||_F^2 on the shortcut path (R2 = I + O(delta))
    }
    if (!(d2 <= 0.0625)) {
      if (tid == 0) atomicOr(status, 1);
      return;
    }
    if (d2 <= 1e-16) {
      for (int idx = tid; idx < n * n; idx += 256) {
        const int i = idx % n, j = idx / n;
        double u = 0.0;
        if (i < j) u = G[i + (int64_t)j * ldg];
        else if (i == j) u = 0.5 * (G[i + (int64_t)j * ldg] - 1.0);
        const double e = (i == j) ? 1.0 : 0.0;
        R[i + (int64_t)j * ldr] = e + u;
        Ri[i + (int64_t)j * ldi] = e - u;
      }
      return;
    }
  }
  __syncthreads();
  if (defect_out && !defect_mode) {  // ||A||_F^2 = trace(G)
    double tr = 0.0;
    for (int i = tid; i < n; i += 256) tr += G[i + (int64_t)i * ldg];
    tr = block_sum_256(tr, red);
    if (tid == 0) defect_out[2] = tr;
  }

  // ---- R11
  double a[16], x[16];
  blk_load(a, G, ldg, kb1);
  blk_factor<true>(a, line, &bad_s);
  blk_to_smem(a, S11);
  blk_store(a, R, ldr, kb1);
  __syncthreads();
  if (kb2 > 0) {
    // ---- R12 = R11^{-T} G12 (column c of the second block column)
    if (tid < kBlk) dinv[tid] = 1.0 / S11[tid][tid];
    const bool act = c < kb2;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      x[q] = (act && i < kb1) ? G[i + (int64_t)(kBlk + c) * ldg] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBlk; ++j) {
      const int qj = j >> 2, pj = j & 3;
      const double v = x[qj] * dinv[j];
      const double xj = -__shfl_sync(0xffffffffu, v, (lane & ~3) | pj);
      const double* r = &S11[j][part];
      if (part == pj) x[qj] = v;
      if (part > pj) x[qj] = fma(r[4 * qj], xj, x[qj]);
#pragma unroll
      for (int q = qj + 1; q < 16; ++q) x[q] = fma(r[4 * q], xj, x[q]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      S12[i][c] = x[q];
      if (act && i < kb1) R[i + (int64_t)(kBlk + c) * ldr] = x[q];
    }
    __syncthreads();
    // ---- G22 - R12^T R12 (identity padded), then R22
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      a[q] = (i < kb2 && c < kb2) ? G[(kBlk + i) + (int64_t)(kBlk + c) * ldg] : (i == c ? 1.0 : 0.0);
    }
    for (int k = 0; k < kBlk; ++k) {
      const double rc = -S12[k][c];
      const double* rr = &S12[k][part];
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = fma(rr[4 * q], rc, a[q]);
    }
    __syncthreads();
    blk_factor<true>(a, line, &bad_s);
    blk_to_smem(a, S22);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = part + 4 * q;
      if (i < kb2) {
        if (c < kb2) R[(kBlk + i) + (int64_t)(kBlk + c) * ldr] = a[q];
        Ri[(kBlk + i) + (int64_t)c * ldi] = 0.0;  // lower-left blocks (kb1 = 64 columns)
        R[(kBlk + i) + (int64_t)c * ldr] = 0.0;
      }
    }
    __syncthreads();
  }
  const double inv2 = cis_inverse(S11, S22, S12, X11, X22, line, dinv, red, kb1, kb2, Ri, ldi);
  if (tid == 0 && defect_out) {
    defect_out[1] = inv2;  // ||R^{-1}||_F^2
  }
  __syncthreads();
  if (tid == 0 && bad_s) atomicOr(status, 1);
}

// No-truncation certificate for an upper-triangular R, k <= 128, in ONE CTA
// (replaces the inverse + two norms + decision kernels, ~12 launches):
// good iff 1 / ||R^{-1}||_F > 1.25 max(delta, ||R||_F max(k, 2) eps).
// ok_dev (optional) receives the verdict; sflag (optional, sticky) gets bit 2
// OR-ed in when the certificate fails (speculative sweeps).
__global__ void __launch_bounds__(256) cert_small_kernel(int k, const double* __restrict__ R, int64_t ldr,
                                                         const double* delta_dev, double delta_scale,
                                                         int* ok_dev, int* sflag, int debug) {
  extern __shared__ double cis_sm[];
  CisBlk S11 = reinterpret_cast<CisBlk>(cis_sm);
  CisBlk S22 = reinterpret_cast<CisBlk>(cis_sm + 1 * kBlk * (kBlk + 1));
  CisBlk S12 = reinterpret_cast<CisBlk>(cis_sm + 2 * kBlk * (kBlk + 1));
  CisBlk X11 = reinterpret_cast<CisBlk>(cis_sm + 3 * kBlk * (kBlk + 1));
  CisBlk X22 = reinterpret_cast<CisBlk>(cis_sm + 4 * kBlk * (kBlk + 1));
  double* line = cis_sm + 5 * kBlk * (kBlk + 1);
  double* dinv = line + 256;
  double* red = dinv + kBlk;
  const int kb1 = min(kBlk, k), kb2 = k - kb1;
  double rn = 0.0;
  for (int idx = threadIdx.x; idx < kBlk * kBlk; idx += 256) {
    const int i = idx % kBlk, c = idx / kBlk;
    const double e = (i == c) ? 1.0 : 0.0;
    const double v11 = (i < kb1 && c < kb1) ? (i <= c ? R[i + (int64_t)c * ldr] : 0.0) : e;
    const double v12 = (i < kb1 && c < kb2) ? R[i + (int64_t)(kBlk + c) * ldr] : 0.0;
    const double v22 = (i < kb2 && c < kb2) ? (i <= c ? R[(kBlk + i) + (int64_t)(kBlk + c) * ldr] : 0.0) : e;
    S11[i][c] = v11;
    S12[i][c] = v12;
    S22[i][c] = v22;
    if (i < kb1 && c < kb1) rn = fma(v11, v11, rn);
    rn = fma(v12, v12, rn);
    if (i < kb2 && c < kb2) rn = fma(v22, v22, rn);
  }
  rn = sqrt(block_sum_256(rn, red));
  const double inv2 = cis_inverse(S11, S22, S12, X11, X22, line, dinv, red, kb1, kb2, nullptr, 0);
  if (threadIdx.x == 0) {
    const double eps = 2.220446049250313e-16;
    const double xn = sqrt(inv2);
    const double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
    const double thr = fmax(delta, rn * (double)max(k, 2) * eps);
    const bool good = isfinite(xn) && isfinite(rn) && xn > 0.0 && (1.0 / xn) > 1.25 * thr;
    if (ok_dev) *ok_dev = good ? 1 : 0;
    if (sflag && !good) atomicOr(sflag, 2);
    if (debug) printf("[cert-small] k=%d smin/||R||>=%.3e thr/||R||=%.3e good=%d\n", k, 1.0 / xn / rn,
                      thr / rn, (int)good);
  }
}

// The same certificate for k <= 32 by ONE warp: lane l back-substitutes column
// l of R^{-1} out of registers (the small bonds at both ends of every TT).
__global__ void __launch_bounds__(32) cert_tiny_kernel(int k, const double* __restrict__ R, int64_t ldr,
                                                       const double* delta_dev, double delta_scale,
                                                       int* ok_dev, int* sflag, int debug) {
  __shared__ double S[32][33];
  const int l = threadIdx.x;
  double rn = 0.0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    double v = (i == l) ? 1.0 : 0.0;
    if (i < k && l < k) v = (i <= l) ? R[i + (int64_t)l * ldr] : 0.0;
    S[i][l] = v;
    if (i < k && l < k) rn = fma(v, v, rn);
  }
  __syncwarp();
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = 0.0;
#pragma unroll
  for (int k2 = 31; k2 >= 0; --k2) {
    const double dinv = 1.0 / S[k2][k2];
    const double xk = (l == k2) ? dinv : (l > k2 ? -v[k2] * dinv : 0.0);
    v[k2] = xk;
#pragma unroll
    for (int i = 0; i < k2; ++i) v[i] = fma(S[i][k2], xk, v[i]);
  }
  double xn = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < k && l < k) xn = fma(v[i], v[i], xn);
  rn = sqrt(warp_sum(rn));
  xn = sqrt(warp_sum(xn));
  if (l == 0) {
    const double eps = 2.220446049250313e-16;
    const double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
    const double thr = fmax(delta, rn * (double)max(k, 2) * eps);
    const bool good = isfinite(xn) && isfinite(rn) && xn > 0.0 && (1.0 / xn) > 1.25 * thr;
    if (ok_dev) *ok_dev = good ? 1 : 0;
    if (sflag && !good) atomicOr(sflag, 2);
    if (debug) printf("[cert-tiny] k=%d smin/||R||>=%.3e thr/||R||=%.3e good=%d\n", k, 1.0 / xn / rn,
                      thr / rn, (int)good);
  }
}

// ------------------------------------------------ small fused factor, v2
// Same contract as chol_inv_small_kernel, organised for latency: blocks of
// 32, the matrix in shared memory (row stride 129), and each 32 x 32 diagonal
// leaf factored AND inverted by ONE warp out of registers (lane l owns column
// l; the pivot row travels through a double-buffered shared line, so a pivot
// step costs one __syncwarp instead of a block barrier: ~180 cycles instead
// of ~500).  Panels (R_kj = X_kk^T G_kj), trailing updates and the
// off-diagonal inverse blocks (X_ij = -X_ii sum_k R_ik X_kj) are 32^3 block
// products spread over the 8 warps with warp-uniform (broadcast) left
// operands and branch-free, unrolled inner loops.  R lives in the upper
// triangle of M, the off-diagonal blocks of X = R^{-1} transposed in the
// lower block triangle, the diagonal blocks X_kk dense (zero below the
// diagonal) in Xd.
constexpr int kC2 = 32;             // block
constexpr int kC2N = 128;           // max n
constexpr int kC2Ld = kC2N + 1;     // row stride of M
constexpr int kC2Xd = kC2 * (kC2 + 1);
constexpr int kC2Smem =
    (kC2N * kC2Ld + 4 * kC2Xd + 2 * kC2 + kC2Xd + 16) * (int)sizeof(double);

// Factor + invert the 32 x 32 diagonal leaf at (k0, k0); executed by one warp.
// R_kk -> upper triangle of M, X_kk -> xdk (32 x 33, zero below the diagonal).
template <int LD, bool INV>
__device__ __forceinline__ void c2_leaf(double* M, double* xdk, double* rowbuf, int k0, int* bad) {
  const int l = threadIdx.x & 31;
  double col[kC2], dinv[kC2];
#pragma unroll
  for (int i = 0; i < kC2; ++i) col[i] = M[(k0 + i) * LD + k0 + l];
#pragma unroll
  for (int j = 0; j < kC2; ++j) {
    const double p = __shfl_sync(0xffffffffu, col[j], j);
    if (l == 0 && !(p > 0.0)) *bad = 1;
    const double inv = rsqrt_nr(p);
    dinv[j] = inv;
    const double r = (l >= j) ? col[j] * inv : 0.0;
    col[j] = r;
    double* rb = rowbuf + (j & 1) * kC2;
    rb[l] = r;
    __syncwarp();
#pragma unroll
    for (int i = j + 1; i < kC2; ++i) col[i] = fma(-rb[i], r, col[i]);
  }
#pragma unroll
  for (int i = 0; i < kC2; ++i)
    if (i <= l) M[(k0 + i) * LD + k0 + l] = col[i];
  __syncwarp();
  if constexpr (INV) {
    // column l of X = R^{-1}: v[i] accumulates sum_k R[i][k] x[k] until it becomes x[i]
    double v[kC2];
#pragma unroll
    for (int i = 0; i < kC2; ++i) v[i] = 0.0;
#pragma unroll
    for (int k2 = kC2 - 1; k2 >= 0; --k2) {
      const double xk = (l == k2) ? dinv[k2] : (l > k2 ? -v[k2] * dinv[k2] : 0.0);
      v[k2] = xk;
      const double* rcol = M + (size_t)k0 * LD + k0 + k2;  // R[i][k2], i < k2 (broadcast reads)
#pragma unroll
      for (int i = 0; i < k2; ++i) v[i] = fma(rcol[i * LD], xk, v[i]);
    }
#pragma unroll
    for (int i = 0; i < kC2; ++i) xdk[i * (kC2 + 1) + l] = v[i];  // zero for i > l
  }
}

__global__ void __launch_bounds__(256) chol_inv_small2_kernel(int n, const double* __restrict__ G,
                                                              int64_t ldg, double* __restrict__ R,
                                                              int64_t ldr, double* __restrict__ Ri,
                                                              int64_t ldi, int defect_mode,
                                                              double* __restrict__ defect_out,
                                                              int* __restrict__ status) {
  extern __shared__ double c2_sm[];
  double* M = c2_sm;
  double* Xd = M + kC2N * kC2Ld;        // 4 dense diagonal blocks of X
  double* rowbuf = Xd + 4 * kC2Xd;
  double* T = rowbuf + 2 * kC2;         // 32 x 33
  double* red = T + kC2Xd;
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) bad_s = 0;
  const int nb = (n + kC2 - 1) / kC2, np = nb * kC2;
  const int dbg = defect_mode & 256;
  defect_mode &= 255;
  long long tstamp[16];
  int nst = 0;
  const long long t00 = clock64();
#define C2_STAMP() do { if (dbg && tid == 0 && nst < 15) tstamp[nst++] = clock64() - t00; } while (0)

  // load: thread -> (row i = tid & 127 within a column pair, columns j = tid >> 7 + 2 t)
  // coalesced along i; all loads of a thread are independent (unrolled)
  {
    const int i = tid & (kC2N - 1), jh = tid >> 7;
    double acc = 0.0, tr = 0.0;
#pragma unroll 32
    for (int t = 0; t < kC2N / 2; ++t) {
      const int j = 2 * t + jh;
      double v = 0.0;
      if (i < n && j < n) v = G[i + (int64_t)j * ldg];
      if (i > j) v = 0.0;
      if (i == j) {
        if (i >= n) v = 1.0;
        else tr += v;
      }
      if (i < np && j < np) M[i * kC2Ld + j] = v;
      if (i <= j && j < n) {
        const double e = v - (i == j ? 1.0 : 0.0);
        acc = fma(i == j ? e : 2.0 * e, e, acc);
      }
    }
    tr = block_sum_256(tr, red);  // also the barrier after the load
    if (tid == 0 && defect_out && !defect_mode) defect_out[2] = tr;
    if (defect_mode) {
      const double d2 = block_sum_256(acc, red);
      if (tid == 0) {
        defect_out[0] = d2;
        defect_out[1] = (double)n;
      }
      if (!(d2 <= 0.0625)) {
        if (tid == 0) atomicOr(status, 1);
        return;
      }
      if (d2 <= 1e-16) {
#pragma unroll 8
        for (int t = 0; t < kC2N / 2; ++t) {
          const int j = 2 * t + jh;
          if (i < n && j < n) {
            const double g = M[i * kC2Ld + j];  // upper triangle of G, zero below
            const double e = (i == j) ? 1.0 : 0.0;
            const double u = (i == j) ? 0.5 * (g - 1.0) : g;
            R[i + (int64_t)j * ldr] = e + u;
            Ri[i + (int64_t)j * ldi] = e - u;
          }
        }
        return;
      }
    }
  }
  C2_STAMP();

  const int c = lane, i0 = warp * 4;  // thread tile: rows i0..i0+3 of a block, column c
  for (int kb = 0; kb < nb; ++kb) {
    const int k0 = kb * kC2;
    if (warp == 0) c2_leaf<kC2Ld, true>(M, Xd + kb * kC2Xd, rowbuf, k0, &bad_s);
    __syncthreads();
    C2_STAMP();
    const int nj = nb - kb - 1;
    if (nj == 0) break;
    // panel: R[kb][jb] = X_kk^T G[kb][jb]; out[i][c] = sum_k X[k][i] G[k][c]
    {
      double out[3][4];
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int q = 0; q < 4; ++q) out[b][q] = 0.0;
      const double* xk = Xd + kb * kC2Xd + i0;
      const double* gk = M + (size_t)k0 * kC2Ld + k0 + kC2 + c;
#pragma unroll 8
      for (int k2 = 0; k2 < kC2; ++k2) {
        const double x0 = xk[k2 * (kC2 + 1)], x1 = xk[k2 * (kC2 + 1) + 1], x2 = xk[k2 * (kC2 + 1) + 2],
                     x3 = xk[k2 * (kC2 + 1) + 3];
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (b < nj) {
            const double g = gk[k2 * kC2Ld + b * kC2];
            out[b][0] = fma(x0, g, out[b][0]);
            out[b][1] = fma(x1, g, out[b][1]);
            out[b][2] = fma(x2, g, out[b][2]);
            out[b][3] = fma(x3, g, out[b][3]);
          }
      }
      __syncthreads();
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b < nj)
#pragma unroll
          for (int q = 0; q < 4; ++q) M[(k0 + i0 + q) * kC2Ld + k0 + (b + 1) * kC2 + c] = out[b][q];
    }
    __syncthreads();
    // trailing update: G[ib][jb] -= R[kb][ib]^T R[kb][jb], kb < ib <= jb
    for (int ib = kb + 1; ib < nb; ++ib)
      for (int jb = ib; jb < nb; ++jb) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* ri = M + (size_t)k0 * kC2Ld + ib * kC2 + i0;
        const double* rj = M + (size_t)k0 * kC2Ld + jb * kC2 + c;
#pragma unroll 8
        for (int k2 = 0; k2 < kC2; ++k2) {
          const double rc = rj[k2 * kC2Ld];
          a0 = fma(ri[k2 * kC2Ld], rc, a0);
          a1 = fma(ri[k2 * kC2Ld + 1], rc, a1);
          a2 = fma(ri[k2 * kC2Ld + 2], rc, a2);
          a3 = fma(ri[k2 * kC2Ld + 3], rc, a3);
        }
        double* dst = M + (size_t)(ib * kC2 + i0) * kC2Ld + jb * kC2 + c;
        dst[0] -= a0;
        dst[kC2Ld] -= a1;
        dst[2 * kC2Ld] -= a2;
        dst[3 * kC2Ld] -= a3;
      }
    __syncthreads();
    C2_STAMP();
  }
  C2_STAMP();
  // off-diagonal blocks of X = R^{-1}: X[ib][jb] = -X_ii sum_{kb=ib+1..jb} R[ib][kb] X[kb][jb];
  // X[ib][jb][i][c] is stored at M[jb*32 + c][ib*32 + i]
  for (int jb = 1; jb < nb; ++jb)
    for (int ib = jb - 1; ib >= 0; --ib) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
      for (int kb = ib + 1; kb <= jb; ++kb) {
        // X[kb*32 + k2][jb*32 + c]: dense diagonal block or transposed lower storage
        const double* xp = (kb == jb) ? Xd + jb * kC2Xd + c : M + (size_t)(jb * kC2 + c) * kC2Ld + kb * kC2;
        const int xs = (kb == jb) ? (kC2 + 1) : 1;
        const double* rr = M + (size_t)(ib * kC2 + i0) * kC2Ld + kb * kC2;
#pragma unroll 8
        for (int k2 = 0; k2 < kC2; ++k2) {
          const double xv = xp[k2 * xs];
          t0 = fma(rr[k2], xv, t0);
          t1 = fma(rr[kC2Ld + k2], xv, t1);
          t2 = fma(rr[2 * kC2Ld + k2], xv, t2);
          t3 = fma(rr[3 * kC2Ld + k2], xv, t3);
        }
      }
      T[(i0 + 0) * (kC2 + 1) + c] = t0;
      T[(i0 + 1) * (kC2 + 1) + c] = t1;
      T[(i0 + 2) * (kC2 + 1) + c] = t2;
      T[(i0 + 3) * (kC2 + 1) + c] = t3;
      __syncthreads();
      double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
      const double* xi = Xd + ib * kC2Xd + i0 * (kC2 + 1);  // X_ii[i][k2]
#pragma unroll 8
      for (int k2 = 0; k2 < kC2; ++k2) {
        const double tv = T[k2 * (kC2 + 1) + c];
        x0 = fma(xi[k2], tv, x0);
        x1 = fma(xi[(kC2 + 1) + k2], tv, x1);
        x2 = fma(xi[2 * (kC2 + 1) + k2], tv, x2);
        x3 = fma(xi[3 * (kC2 + 1) + k2], tv, x3);
      }
      double* dst = M + (size_t)(jb * kC2 + c) * kC2Ld + ib * kC2 + i0;
      dst[0] = -x0;
      dst[1] = -x1;
      dst[2] = -x2;
      dst[3] = -x3;
      __syncthreads();
    }
  C2_STAMP();
  // write R, Ri (column-major, strictly lower zero) and ||Ri||_F^2
  double nrm = 0.0;
  {
    const int i = tid & (kC2N - 1), jh = tid >> 7;
#pragma unroll 16
    for (int t = 0; t < kC2N / 2; ++t) {
      const int j = 2 * t + jh;
      if (i < n && j < n) {
        const int ib = i >> 5, jb = j >> 5;
        const double rv = (i <= j) ? M[i * kC2Ld + j] : 0.0;
        double xv = 0.0;
        if (ib == jb) xv = Xd[ib * kC2Xd + (i & 31) * (kC2 + 1) + (j & 31)];
        else if (ib < jb) xv = M[j * kC2Ld + i];
        R[i + (int64_t)j * ldr] = rv;
        if (Ri) Ri[i + (int64_t)j * ldi] = xv;
        nrm = fma(xv, xv, nrm);
      }
    }
  }
  nrm = block_sum_256(nrm, red);
  if (tid == 0) {
    if (defect_out) defect_out[1] = nrm;
    if (bad_s) atomicOr(status, 1);
    if (dbg) {
      tstamp[nst++] = clock64() - t00;
      printf("[cis2] n=%d stamps:", n);
      for (int q = 0; q < nst; ++q) printf(" %lld", tstamp[q]);
      printf("\n");
    }
  }
#undef C2_STAMP
}

int chol_inv_small(cudaStream_t s, int n, const double* G, int64_t ldg, double* R, int64_t ldr,
                   double* Ri, int64_t ldi, int defect_mode, double* defect_out, int* status) {
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(chol_inv_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kCisSmem));
    configured.set();
  }
  static const bool v1 = getenv("QTT_CIS_V1") != nullptr;
  if (v1) {
    chol_inv_small_kernel<<<1, 256, kCisSmem, s>>>(n, G, ldg, R, ldr, Ri, ldi, defect_mode, defect_out,
                                                  status);
  } else {
    static DeviceFlag configured2;
    if (!configured2.test()) {
      QTT_CUDA(cudaFuncSetAttribute(chol_inv_small2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kC2Smem));
      configured2.set();
    }
    static const int dbg2 = getenv("QTT_CIS_DEBUG") ? 256 : 0;
    chol_inv_small2_kernel<<<1, 256, kC2Smem, s>>>(n, G, ldg, R, ldr, Ri, ldi, defect_mode | dbg2, defect_out,
                                                  status);
  }
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
    // (a variant with single-warp 32 x 32 register leaves for the diagonal factor, as in
    // chol_inv_small2_kernel, measured no faster here: 90.9 vs 89.1 ms serial config-2 step)
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

// Certificate from the by-products of cholqr2_small (sc[1] = ||R1^{-1}||_F^2,
// sc[2] = ||A||_F^2, sc[4] = ||Q1^T Q1 - I||_F^2): R = R2 R1 with
// sigma_min(R2)^2 = lambda_min(Q1^T Q1) >= 1 - delta, so
// sigma_min(R) >= sqrt(1 - delta) / ||R1^{-1}||_F; ||R||_F = ||A||_F.
__global__ void cert_factors_kernel(int k, const double* sc, const double* delta_dev, double delta_scale,
                                    int* sflag, int debug) {
  const double eps = 2.220446049250313e-16;
  const double rn = sqrt(fmax(sc[2], 0.0));
  const double lb = sqrt(fmax(1.0 - sqrt(fmax(sc[4], 0.0)), 0.0)) / sqrt(sc[1]);
  const double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
  const double thr = fmax(delta, rn * (double)max(k, 2) * eps);
  const bool good = isfinite(lb) && isfinite(rn) && lb > 1.25 * thr;
  if (!good) atomicOr(sflag, 2);
  if (debug) printf("[cert-factors] k=%d smin/||R||>=%.3e thr/||R||=%.3e good=%d\n", k, lb / rn, thr / rn,
                    (int)good);
}

int cert_factors(cudaStream_t s, int k, const double* sc, const double* delta_dev, double delta_scale,
                 int* sflag) {
  static const int debug = getenv("QTT_CERT_DEBUG") ? 1 : 0;
  cert_factors_kernel<<<1, 1, 0, s>>>(k, sc, delta_dev, delta_scale, sflag, debug);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int cert_small(cudaStream_t s, int k, const double* R, int64_t ldr, const double* delta_dev,
               double delta_scale, int* ok_dev, int* sflag) {
  if (k <= 0 || k > 2 * kBlk) return kInvalid;
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(cert_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCisSmem));
    configured.set();
  }
  static const int debug = getenv("QTT_CERT_DEBUG") ? 1 : 0;
  if (k <= 32) {
    cert_tiny_kernel<<<1, 32, 0, s>>>(k, R, ldr, delta_dev, delta_scale, ok_dev, sflag, debug);
    QTT_CHECK_LAUNCH();
    return kOk;
  }
  cert_small_kernel<<<1, 256, kCisSmem, s>>>(k, R, ldr, delta_dev, delta_scale, ok_dev, sflag, debug);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int gram_certificate(cudaStream_t s, int p, int r, const double* X, int64_t ldx,
                     const double* delta_dev, double delta_scale, int* ok_dev) {
  if (p < r || r <= 0) return kInvalid;
  const int64_t nn = r;
  double *G, *Ri, *rblk, *sc;
  int* bad;
  QTT_CUDA(malloc_async(&G, sizeof(double) * nn * nn, s));
  QTT_CUDA(malloc_async(&Ri, sizeof(double) * nn * nn, s));
  QTT_CUDA(malloc_async(&rblk, sizeof(double) * CB * CB * ceil_div(nn, CB), s));
  QTT_CUDA(malloc_async(&sc, sizeof(double) * 4, s));
  QTT_CUDA(malloc_async(&bad, sizeof(int), s));
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

// CholeskyQR2 of a small tall matrix (n <= 128) with NO host synchronisation:
// Gram (DMMA) -> fused factor+inverse -> Q1 = A Ri1 -> Gram -> fused
// factor+inverse with the near-identity shortcut -> Q = Q1 Ri2, R = R2 R1.
// Seven launches.  Failure (pivot breakdown, ||Q1^T Q1 - I||_F > 1/4) raises
// the sticky device flag *status and leaves unspecified output.
int cholqr2_small(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
                  double* R, int64_t ldr, int* status, double* scalars) {
  if (m < n || n <= 0 || n > 2 * kBlk) return kInvalid;
  const int64_t nn = n;
  double *buf, *Q1;
  QTT_CUDA(malloc_async(&buf, sizeof(double) * (4 * nn * nn + 8), s));
  QTT_CUDA(malloc_async(&Q1, sizeof(double) * (int64_t)m * nn, s));
  double *G = buf, *R1 = buf + nn * nn, *Ri = buf + 2 * nn * nn, *R2 = buf + 3 * nn * nn,
         *sc = scalars ? scalars : buf + 4 * nn * nn;
  int status_code = kOk;
  do {
    if ((status_code = dgemm(s, 1, 0, n, n, m, 1.0, A, lda, A, lda, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    if ((status_code = chol_inv_small(s, n, G, nn, R1, nn, Ri, nn, 0, sc, status)) != kOk) break;
    if ((status_code = dgemm(s, 0, 0, m, n, n, 1.0, A, lda, Ri, nn, 0.0, Q1, m, kGemmTriB)) != kOk) break;
    if ((status_code = dgemm(s, 1, 0, n, n, m, 1.0, Q1, m, Q1, m, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    if ((status_code = chol_inv_small(s, n, G, nn, R2, nn, Ri, nn, 1, sc + 4, status)) != kOk) break;
    if (Q && (status_code = dgemm(s, 0, 0, m, n, n, 1.0, Q1, m, Ri, nn, 0.0, Q, ldq, kGemmTriB)) != kOk) break;
    if (R && (status_code = dgemm(s, 0, 0, n, n, n, 1.0, R2, nn, R1, nn, 0.0, R, ldr, kGemmTriA | kGemmTriB)) != kOk) break;
  } while (false);
  QTT_CUDA(cudaFreeAsync(buf, s));
  QTT_CUDA(cudaFreeAsync(Q1, s));
  return status_code;
}

// Ri <- 2 I - G on the upper triangle (zero below): inverse of G = I + U to
// first order, exact to ||U||^2.
__global__ void neumann1_kernel(int n, const double* __restrict__ G, int64_t ldg,
                                double* __restrict__ Ri, int64_t ldi) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % n), c = (int)(idx / n);
    Ri[r + (int64_t)c * ldi] = (r > c) ? 0.0 : ((r == c ? 2.0 : 0.0) - G[r + (int64_t)c * ldg]);
  }
}

int cholqr2(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
            double* R, int64_t ldr, int* ok, QrInfo* info) {
  *ok = 0;
  if (info) info->valid = false;
  if (m < n || n <= 0) return kOk;
  const int64_t nn = n;
  double *G, *R1, *Ri, *Q1, *rblk, *scal, *parts;
  int* bad;
  QTT_CUDA(malloc_async(&G, sizeof(double) * nn * nn, s));
  QTT_CUDA(malloc_async(&R1, sizeof(double) * nn * nn, s));
  QTT_CUDA(malloc_async(&Ri, sizeof(double) * nn * nn, s));
  QTT_CUDA(malloc_async(&Q1, sizeof(double) * (int64_t)m * nn, s));
  QTT_CUDA(malloc_async(&rblk, sizeof(double) * CB * CB * ceil_div(nn, CB), s));
  QTT_CUDA(malloc_async(&scal, sizeof(double) * 4, s));
  QTT_CUDA(malloc_async(&parts, sizeof(double) * kDefectParts, s));
  QTT_CUDA(malloc_async(&bad, sizeof(int), s));
  QTT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  int status = kOk;
  PhaseTimer pt(s);
  do {
    // pass 1: G = A^T A = R1^T R1, Q1 = A R1^{-1}
    if ((status = dgemm(s, 1, 0, n, n, m, 1.0, A, lda, A, lda, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    gram_trace_kernel<<<1, 256, 0, s>>>(n, G, nn, scal + 1);  // ||A||_F^2
    QTT_CHECK_LAUNCH();
    pt.lap(" cq-gram1", 0, m, n, 0);
    if ((status = chol_upper(s, n, G, nn, rblk, bad)) != kOk) break;
    pt.lap(" cq-chol1", 0, m, n, 0);
    // no synchronisation here: a breakdown (bad pivot -> NaN) surfaces in the
    // defect below, which is read together with the flag
    QTT_CUDA(cudaMemcpyAsync(R1, G, sizeof(double) * nn * nn, cudaMemcpyDeviceToDevice, s));
    if ((status = tri_inverse(s, n, R1, nn, Ri)) != kOk) break;
    if ((status = frob_norm(s, nn * nn, Ri, scal + 2)) != kOk) break;  // ||R1^{-1}||_F
    pt.lap(" cq-inv1", 0, m, n, 0);
    if ((status = dgemm(s, 0, 0, m, n, n, 1.0, A, lda, Ri, nn, 0.0, Q1, m, kGemmTriB)) != kOk) break;
    pt.lap(" cq-q1", 0, m, n, 0);
    // pass 2: certify cond(Q1) ~ 1, then G = Q1^T Q1 = R2^T R2, Q = Q1 R2^{-1}
    if ((status = dgemm(s, 1, 0, n, n, m, 1.0, Q1, m, Q1, m, 0.0, G, nn, kGemmUpperC)) != kOk) break;
    gram_defect_kernel<<<kDefectParts, 256, 0, s>>>(n, G, nn, parts);
    QTT_CHECK_LAUNCH();
    sum_parts_kernel<<<1, 32, 0, s>>>(kDefectParts, parts, scal);
    QTT_CHECK_LAUNCH();
    double hs[3] = {0.0, 0.0, 0.0};  // defect^2, ||A||_F^2, ||R1^{-1}||_F
    int hbad = 0;
    QTT_CUDA(cudaMemcpyAsync(hs, scal, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    const double defect = hs[0];
    if (getenv("QTT_QR_DEBUG")) fprintf(stderr, "[cholqr2] m=%d n=%d defect=%.3e\n", m, n, std::sqrt(defect));
    const double delta = std::sqrt(defect);
    pt.lap(" cq-gram2", 0, m, n, (int)(-std::log10(std::max(delta, 1e-99))));
    if (hbad || !(delta <= 0.25)) break;
    bool near_id = false;
    if (delta <= 1e-2 && !getenv("QTT_NO_NEAR_IDENTITY")) {
      int iters = 0;
      while (iters < 8 && std::pow(std::max(delta, 1e-300), iters + 2) > 1e-17) ++iters;
      double *U, *W;
      QTT_CUDA(malloc_async(&U, sizeof(double) * nn * nn, s));
      QTT_CUDA(malloc_async(&W, sizeof(double) * nn * nn, s));
      status = chol_near_identity(s, n, G, nn, U, W, iters);
      QTT_CUDA(cudaFreeAsync(U, s));
      QTT_CUDA(cudaFreeAsync(W, s));
      if (status != kOk) break;
      near_id = true;
    } else {
      if ((status = chol_upper(s, n, G, nn, rblk, bad)) != kOk) break;
      QTT_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      QTT_CUDA(cudaStreamSynchronize(s));
      if (hbad) break;
    }
    pt.lap(" cq-chol2", 0, m, n, 0);
    if (Q) {
      if (near_id && delta <= 1e-9) {
        // R2 = I + U with ||U|| <= delta: R2^{-1} = I - U to delta^2 <= 1e-18
        const int blocks = (int)std::min<int64_t>(ceil_div(nn * nn, 256), 8 * num_sms());
        neumann1_kernel<<<blocks, 256, 0, s>>>(n, G, nn, Ri, nn);
        QTT_CHECK_LAUNCH();
      } else if ((status = tri_inverse(s, n, G, nn, Ri)) != kOk) {
        break;
      }
    }
    pt.lap(" cq-inv2", 0, m, n, 0);
    if (Q && (status = dgemm(s, 0, 0, m, n, n, 1.0, Q1, m, Ri, nn, 0.0, Q, ldq, kGemmTriB)) != kOk) break;
    pt.lap(" cq-q", 0, m, n, 0);
    // R = R2 R1 (product of upper-triangular factors stays upper triangular)
    if ((status = dgemm(s, 0, 0, n, n, n, 1.0, G, nn, R1, nn, 0.0, R, ldr, kGemmTriA | kGemmTriB)) != kOk) break;
    pt.lap(" cq-r", 0, m, n, 0);
    *ok = 1;
    if (info) {
      // sigma_min(R) >= sigma_min(R2) sigma_min(R1) >= sqrt(1 - delta) / ||R1^{-1}||_F
      info->valid = std::isfinite(hs[2]) && hs[2] > 0.0 && std::isfinite(hs[1]);
      info->sigma_lb = std::sqrt(std::max(1.0 - delta, 0.0)) / hs[2];
      info->anorm = std::sqrt(std::max(hs[1], 0.0));
    }
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
