// Element-level value grids for the QTT assembly (row a10).
//
// One launch evaluates, for every element (i, j) of the zero-padded
// 2^d x 2^d element grid, the 16 corner-pair stiffness couplings (x 4
// displacement components) and the 16 load weights of element.py:160-212,
// using the affine Jacobian expansion J(i,j) = J00 + i dJ10 + j dJ01 at each
// Gauss point (element.py:111-150).  Threads run over
// the OUTPUT index (Z-order or canonical), so the 80 output vectors are
// written with coalesced stores directly in the layout grid_to_qtt feeds to
// the TT-SVD (assembly.py:144-158).  An optional per-Gauss-point modulus
// multiplier grid implements the BASELINE config-4 E(x,y) extension.
#include "../../include/qtt_b200.h"
#include "common.cuh"

namespace qtt {
namespace {

struct ElemCoef {
  int ng;            // Gauss points (<= 4)
  int n_elem;        // elements per side
  int d;             // grid bits per side
  int zorder;        // 1: Z-order output, 0: canonical i + n j
  int paper_det;
  double j00[4][4];  // [g][entry] entries (x_xi, y_xi, x_eta, y_eta)
  double d10[4][4];
  double d01[4][4];
  double det00[4], det10[4], det01[4];  // paper determinant pieces
  double w[4];                          // Gauss weights (product)
  double grad[4][4][2];                 // [g][corner][dxi, deta]
  double val[4][4];                     // [g][corner]
  double C[3][3];
};

__device__ __forceinline__ int64_t squeeze_bits(int64_t z, int d) {
  int64_t x = 0;
  for (int b = 0; b < d; ++b) x |= ((z >> (2 * b)) & 1LL) << b;
  return x;
}

// grid (4 pair-groups): thread handles one output position and one corner a
// (4 partner corners b, 4 components each + 4 load weights).
__global__ void element_grids_kernel(const __grid_constant__ ElemCoef ec, const double* __restrict__ modulus,
                                     double* __restrict__ kout, double* __restrict__ gout,
                                     int* __restrict__ degenerate) {
  const int64_t npos = 1LL << (2 * ec.d);
  const int n = 1 << ec.d;
  const int64_t total = npos * 4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t / npos);
    const int64_t pos = t % npos;
    int64_t i, j;
    if (ec.zorder) {
      i = squeeze_bits(pos, ec.d);
      j = squeeze_bits(pos >> 1, ec.d);
    } else {
      i = pos % n;
      j = pos / n;
    }
    double k[4][4];
    double g[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      g[b] = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) k[b][c] = 0.0;
    }
    if (i < ec.n_elem && j < ec.n_elem) {
      const double fi = (double)i, fj = (double)j;
      for (int q = 0; q < ec.ng; ++q) {
        const double x_xi = ec.j00[q][0] + fi * ec.d10[q][0] + fj * ec.d01[q][0];
        const double y_xi = ec.j00[q][1] + fi * ec.d10[q][1] + fj * ec.d01[q][1];
        const double x_eta = ec.j00[q][2] + fi * ec.d10[q][2] + fj * ec.d01[q][2];
        const double y_eta = ec.j00[q][3] + fi * ec.d10[q][3] + fj * ec.d01[q][3];
        double det = ec.paper_det ? ec.det00[q] + fi * ec.det10[q] + fj * ec.det01[q]
                                  : x_xi * y_eta - y_xi * x_eta;
        if (!(det > 0.0)) atomicExch(degenerate, 1);
        const double e = modulus ? modulus[((int64_t)q * ec.n_elem + i) * ec.n_elem + j] : 1.0;
        const double wd = ec.w[q] * det;
        const double wk = wd * e;
        const double gxa = (ec.grad[q][a][0] * y_eta - ec.grad[q][a][1] * y_xi) / det;
        const double gya = (-ec.grad[q][a][0] * x_eta + ec.grad[q][a][1] * x_xi) / det;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double gxb = (ec.grad[q][b][0] * y_eta - ec.grad[q][b][1] * y_xi) / det;
          const double gyb = (-ec.grad[q][b][0] * x_eta + ec.grad[q][b][1] * x_xi) / det;
          k[b][0] += wk * (ec.C[0][0] * gxa * gxb + ec.C[2][2] * gya * gyb);
          k[b][1] += wk * (ec.C[0][1] * gxa * gyb + ec.C[2][2] * gya * gxb);
          k[b][2] += wk * (ec.C[0][1] * gya * gxb + ec.C[2][2] * gxa * gyb);
          k[b][3] += wk * (ec.C[1][1] * gya * gyb + ec.C[2][2] * gxa * gxb);
          g[b] += wd * ec.val[q][a] * ec.val[q][b];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int pair = a * 4 + b;
#pragma unroll
      for (int c = 0; c < 4; ++c) kout[(int64_t)(pair * 4 + c) * npos + pos] = k[b][c];
      gout[(int64_t)pair * npos + pos] = g[b];
    }
  }
}

}  // namespace
}  // namespace qtt

using namespace qtt;

extern "C" int qtt_element_grids(int32_t d, int32_t zorder, int32_t ngauss, const double* coef,
                                 const double* cmat, int32_t paper_det, const double* modulus,
                                 double* kout, double* gout, int32_t* degenerate, void* stream) {
  if (d < 1 || d > 15 || ngauss < 1 || ngauss > 4 || !coef || !cmat || !degenerate)
    return QTT_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  pool_init();
  ElemCoef ec;
  ec.ng = ngauss;
  ec.d = d;
  ec.n_elem = (1 << d) - 1;
  ec.zorder = zorder;
  ec.paper_det = paper_det;
  // coef layout per Gauss point: j00[4], d10[4], d01[4], w, grad[4][2], val[4]
  // (25 doubles), entries ordered (x_xi, y_xi, x_eta, y_eta).
  for (int q = 0; q < ngauss; ++q) {
    const double* c = coef + q * 25;
    for (int e = 0; e < 4; ++e) {
      ec.j00[q][e] = c[e];
      ec.d10[q][e] = c[4 + e];
      ec.d01[q][e] = c[8 + e];
    }
    ec.w[q] = c[12];
    for (int k = 0; k < 4; ++k) {
      ec.grad[q][k][0] = c[13 + 2 * k];
      ec.grad[q][k][1] = c[14 + 2 * k];
      ec.val[q][k] = c[21 + k];
    }
    auto det2 = [](const double* m) { return m[0] * m[3] - m[1] * m[2]; };
    ec.det00[q] = det2(c);
    ec.det10[q] = det2(c + 4);
    ec.det01[q] = det2(c + 8);
  }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) ec.C[r][c] = cmat[3 * r + c];
  int* flag;
  QTT_CUDA(malloc_async(&flag, sizeof(int), s));
  QTT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const int64_t total = (1LL << (2 * d)) * 4;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16 * num_sms()));
  element_grids_kernel<<<blocks, 256, 0, s>>>(ec, modulus, kout, gout, flag);
  QTT_CHECK_LAUNCH();
  int host = 0;
  QTT_CUDA(cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  QTT_CUDA(cudaFreeAsync(flag, s));
  QTT_CUDA(cudaStreamSynchronize(s));
  *degenerate = host;
  return QTT_OK;
}
