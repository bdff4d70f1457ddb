// Dense FP64 factorizations for the TT sweeps: blocked Householder QR with
// cluster (DSMEM) panels, one-sided Jacobi SVD, sort + _chop, and the
// triangular-inverse certificate that skips the SVD when no truncation can
// occur.  See linalg.cuh for the contracts.
#include <cooperative_groups.h>

#include <cstdlib>
#include <string>

#include "linalg.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr double kEps = 2.220446049250313e-16;

// ------------------------------------------------------------------ panel QR

constexpr int PTHREADS = 512;    // 16 warps per CTA
constexpr int PMAXROWS = 736;    // panel rows held per CTA (736*32*8 B = 184 KB)
constexpr int PMAXCLUSTER = 16;  // non-portable cluster size (B200: 16 SMs per cluster)

struct PanelArgs {
  int m, nb, rpc;
  double* A;
  int64_t lda;
  double* V;
  int64_t ldv;
  double* Y;
  int64_t ldy;
  double* Y2;
  int64_t ldy2;
  double* tau;
};

// One cluster reduction per column.  For column j every CTA pushes, over
// its rows g > j, the dots of column j with every panel column c:
//   c >= j : S_c = sum_g A[g,j] A[g,c]      (S_j = squared norm)
//   c <  j : Z_c = sum_g V[g,c] A[g,j]      (for the compact-WY T factor)
// and the owner of row j pushes that row.  With v = (x - beta e_j)/(alpha - beta)
// the reflector dots follow without a second reduction,
//   w_c = A[j,c] + scal S_c,   (V^T v_j)_c = V[j,c] + scal Z_c,
// so T (dlarft, forward, columnwise) is accumulated on the fly.  Partials are
// double buffered by column parity: one cluster barrier per column and none
// after the loop.
__device__ __forceinline__ void panel_barrier(cg::cluster_group& cl, int cs) {
  if (cs == 1) __syncthreads();
  else cl.sync();
}

template <int PNB>
__global__ void __launch_bounds__(PTHREADS) panel_qr_kernel(PanelArgs pa) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int ld = pa.rpc;
  const int row0 = crank * pa.rpc;
  const int nrows = max(0, min(pa.m - row0, pa.rpc));
  const int nb = pa.nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = PTHREADS / 32;
  constexpr int SLOT = 2 * PNB;  // per-CTA slot: [dots (PNB) | owner row (PNB)]

  double* P = smem;                                // ld * PNB
  double* part = P + (size_t)ld * PNB;             // [2][PMAXCLUSTER][SLOT]
  double* gS = part + 2 * PMAXCLUSTER * SLOT;      // PNB reduced dots
  double* gR = gS + PNB;                           // PNB row-j values
  double* T = gR + PNB;                            // PNB*PNB
  double* tau_s = T + PNB * PNB;                   // PNB

  for (int idx = tid; idx < nrows * nb; idx += PTHREADS) {
    const int r = idx % nrows, c = idx / nrows;
    P[r + c * ld] = pa.A[(row0 + r) + (int64_t)c * pa.lda];
  }
  for (int idx = tid; idx < PNB * PNB; idx += PTHREADS) T[idx] = 0.0;
  __syncthreads();

  for (int j = 0; j < nb; ++j) {
    double* pb = part + (j & 1) * PMAXCLUSTER * SLOT;
    const int rstart = max(0, j + 1 - row0);
    // (1) dots of column j with all panel columns over local rows g > j
    for (int c = warp; c < nb; c += NW) {
      double acc = 0.0;
      for (int r = rstart + lane; r < nrows; r += 32) acc = fma(P[r + j * ld], P[r + c * ld], acc);
      acc = warp_sum(acc);
      if (cs == 1) {
        if (lane == 0) pb[c] = acc;
      } else if (lane < cs) {
        cluster.map_shared_rank(pb, lane)[crank * SLOT + c] = acc;
      }
    }
    const bool owner = (j >= row0 && j < row0 + nrows);
    if (owner) {
      const int rj = j - row0;
      for (int idx = tid; idx < nb * cs; idx += PTHREADS) {
        const int c = idx % nb, q = idx / nb;
        double* dst = (cs == 1) ? pb : cluster.map_shared_rank(pb, q);
        dst[PNB + c] = P[rj + c * ld];  // owner row lands in slot 0's row half
      }
    }
    panel_barrier(cluster, cs);
    // (2) local reduction of the pushed partials (same order everywhere)
    for (int c = tid; c < nb; c += PTHREADS) {
      double sum = 0.0;
      for (int q = 0; q < cs; ++q) sum += pb[q * SLOT + c];
      gS[c] = sum;
      gR[c] = pb[PNB + c];
    }
    __syncthreads();
    // (3) reflector
    const double norm2 = gS[j];
    const double alpha = gR[j];
    double tau = 0.0, beta = alpha, scal = 1.0;
    if (norm2 > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, norm2));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    // (4) T column j (warp 0) while the other warps update the rows
    if (warp == NW - 1) {
      if (lane == 0) {
        tau_s[j] = tau;
        T[j + j * PNB] = tau;
      }
      if (lane < j) {
        double acc = 0.0;
        for (int l = lane; l < j; ++l) acc = fma(T[lane + l * PNB], fma(scal, gS[l], gR[l]), acc);
        T[lane + j * PNB] = -tau * acc;
      }
    }
    if (tau != 0.0) {
      for (int r = rstart + tid; r < nrows; r += PTHREADS) {
        const double v = P[r + j * ld] * scal;
        for (int c = j + 1; c < nb; ++c) {
          const double w = fma(scal, gS[c], gR[c]);
          P[r + c * ld] = fma(-tau * w, v, P[r + c * ld]);
        }
        P[r + j * ld] = v;
      }
      if (owner && tid == 0) {
        const int rj = j - row0;
        for (int c = j + 1; c < nb; ++c) P[rj + c * ld] -= tau * fma(scal, gS[c], gR[c]);
      }
    }
    if (owner && tid == 0) P[(j - row0) + j * ld] = beta;
    __syncthreads();
  }

  // ---- outputs: V (explicit), Y = V T^T, Y2 = V T, R rows, tau
  for (int idx = tid; idx < nrows * nb; idx += PTHREADS) {
    const int r = idx % nrows, q = idx / nrows;
    const int g = row0 + r;
    double y = 0.0, y2 = 0.0;
    const int pmax = min(nb - 1, g);
    for (int p = 0; p <= pmax; ++p) {
      const double v = (g == p) ? 1.0 : P[r + p * ld];
      y = fma(v, T[q + p * PNB], y);
      y2 = fma(v, T[p + q * PNB], y2);
    }
    const double vq = (g == q) ? 1.0 : (g > q ? P[r + q * ld] : 0.0);
    pa.V[g + (int64_t)q * pa.ldv] = vq;
    pa.Y[g + (int64_t)q * pa.ldy] = y;
    pa.Y2[g + (int64_t)q * pa.ldy2] = y2;
    if (g <= q) pa.A[g + (int64_t)q * pa.lda] = P[r + q * ld];
  }
  if (crank == 0 && tid < nb) pa.tau[tid] = tau_s[tid];
}

constexpr int PMAXROWS16 = 1600;  // rows per CTA for the 16-wide panels of very tall matrices

size_t panel_smem_bytes(int rpc, int pnb) {
  return sizeof(double) *
         ((size_t)rpc * pnb + 2 * PMAXCLUSTER * 2 * pnb + 2 * pnb + pnb * pnb + pnb);
}

template <int PNB>
int launch_panel_t(cudaStream_t s, const PanelArgs& pa0, int maxrows) {
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(panel_qr_kernel<PNB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)panel_smem_bytes(maxrows, PNB)));
    QTT_CUDA(cudaFuncSetAttribute(panel_qr_kernel<PNB>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured.set();
  }
  PanelArgs pa = pa0;
  // spread tall panels over up to 16 CTAs (>= 256 rows each) so the
  // per-column work per CTA stays small; single CTA below 384 rows.
  int cs = (int)std::max<int64_t>(ceil_div(pa.m, maxrows), std::min<int64_t>(16, pa.m / 256));
  cs = std::max(cs, 1);
  if (cs > PMAXCLUSTER) return kUnsupported;
  pa.rpc = (int)ceil_div(pa.m, cs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(PTHREADS, 1, 1);
  cfg.dynamicSmemBytes = panel_smem_bytes(pa.rpc, PNB);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QTT_CUDA(cudaLaunchKernelEx(&cfg, panel_qr_kernel<PNB>, pa));
  note_launch();
  return kOk;
}

// Panel width: 32 columns while a 16-CTA cluster holds the rows, else 16.
inline int panel_width(int m) { return m <= PMAXCLUSTER * PMAXROWS ? 32 : 16; }

int launch_panel(cudaStream_t s, const PanelArgs& pa) {
  return pa.nb > 16 || panel_width(pa.m + 0) == 32 ? launch_panel_t<32>(s, pa, PMAXROWS)
                                                   : launch_panel_t<16>(s, pa, PMAXROWS16);
}

__global__ void upper_copy_kernel(int k, int n, const double* __restrict__ A, int64_t lda,
                                  double* __restrict__ R, int64_t ldr) {
  const int64_t total = (int64_t)k * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % k);
    const int64_t c = i / k;
    R[r + c * ldr] = (r <= c) ? A[r + c * lda] : 0.0;
  }
}

__global__ void identity_kernel(int rows, int cols, double* A, int64_t lda) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows);
    const int64_t c = i / rows;
    A[r + c * lda] = (r == c) ? 1.0 : 0.0;
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 16 * num_sms()));
}

// ------------------------------------------------------------------- Jacobi
// Round-robin (circle method) pair of round r: positions of the list
// [0, 1 + (r mod kp-1), ...] paired first-with-last.
__device__ __forceinline__ void rr_pair(int kp, int r, int q, int& i, int& j) {
  const int m = kp - 1;
  auto at = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + r) % m); };
  i = at(q);
  j = at(kp - 1 - q);
  if (i > j) { int t = i; i = j; j = t; }
}

// One Jacobi rotation on columns (i, j) by one warp; returns 1 if rotated.
__device__ int jacobi_pair(double* X, int64_t ldx, double* W, int64_t ldw, int p, int k, int i,
                           int j, double tol, double noise2) {
  const int lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0, g = 0.0;
  double* xi = X + (int64_t)i * ldx;
  double* xj = X + (int64_t)j * ldx;
  for (int r = lane; r < p; r += 32) {
    const double u = xi[r], v = xj[r];
    a = fma(u, u, a);
    b = fma(v, v, b);
    g = fma(u, v, g);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  g = warp_sum(g);
  // Columns below the noise level eps*||X||_F sit far under the _chop floor
  // (s0 * max(k,2) * eps); rotating them only churns rounding noise.
  if (g == 0.0 || a < noise2 || b < noise2 || !(fabs(g) > tol * sqrt(a) * sqrt(b))) return 0;
  const double zeta = (b - a) / (2.0 * g);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  const double c = 1.0 / sqrt(fma(t, t, 1.0));
  const double sn = c * t;
  for (int r = lane; r < p; r += 32) {
    const double u = xi[r], v = xj[r];
    xi[r] = c * u - sn * v;
    xj[r] = sn * u + c * v;
  }
  double* wi = W + (int64_t)i * ldw;
  double* wj = W + (int64_t)j * ldw;
  for (int r = lane; r < k; r += 32) {
    const double u = wi[r], v = wj[r];
    wi[r] = c * u - sn * v;
    wj[r] = sn * u + c * v;
  }
  return 1;
}

// Optional rotation floor from the caller's truncation threshold: columns
// with ||x||^2 < (floor_scale * *floor_dev)^2 / k (the sum over all of them
// stays below 1e-6 delta^2 for floor_scale = 1e-3 * delta / ||t||) are
// certain to be discarded by _chop, and rotations among or against them
// cannot change the kept subspace beyond that energy, so they are skipped.
__device__ __forceinline__ double jacobi_floor2(const double* floor_dev, double floor_scale, int k) {
  if (!floor_dev) return 0.0;
  const double f = floor_scale * *floor_dev;
  return f * f / (double)max(k, 1);
}

constexpr int JMAXSWEEPS = 60;
__device__ int g_jacobi_sweeps;  // sweeps used by the last Jacobi launch (diagnostics)
constexpr int JTHREADS = 1024;

// Small problems: one CTA, X and W staged in shared memory.
__global__ void __launch_bounds__(JTHREADS) jacobi_smem_kernel(int p, int k, double* X,
                                                                int64_t ldx, double* W,
                                                                int64_t ldw, double tol,
                                                                const double* floor_dev,
                                                                double floor_scale) {
  extern __shared__ double sm[];
  __shared__ int rotated;
  double* Xs = sm;
  double* Ws = sm + (size_t)p * k;
  for (int idx = threadIdx.x; idx < p * k; idx += blockDim.x)
    Xs[idx] = X[(idx % p) + (int64_t)(idx / p) * ldx];
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x)
    Ws[idx] = ((idx % k) == (idx / k)) ? 1.0 : 0.0;
  const int kp = k + (k & 1);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double red[32];
  __shared__ double noise2;
  {
    double acc = 0.0;
    for (int idx = threadIdx.x; idx < p * k; idx += blockDim.x) acc = fma(Xs[idx], Xs[idx], acc);
    acc = warp_sum(acc);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[w];
      noise2 = fmax(t * kEps * kEps, jacobi_floor2(floor_dev, floor_scale, k));
    }
    __syncthreads();
  }
  for (int sweep = 0; sweep < JMAXSWEEPS; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    int any = 0;
    for (int r = 0; r < kp - 1; ++r) {
      for (int q = warp; q < kp / 2; q += nw) {
        int i, j;
        rr_pair(kp, r, q, i, j);
        if (j < k) any |= jacobi_pair(Xs, p, Ws, k, p, k, i, j, tol, noise2);
      }
      __syncthreads();
    }
    if (any && (threadIdx.x & 31) == 0) rotated = 1;
    __syncthreads();
    if (threadIdx.x == 0) g_jacobi_sweeps = sweep + 1;
    if (!rotated) break;
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < p * k; idx += blockDim.x)
    X[(idx % p) + (int64_t)(idx / p) * ldx] = Xs[idx];
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x)
    W[(idx % k) + (int64_t)(idx / k) * ldw] = Ws[idx];
}

// Mid-size problems: a thread-block cluster holds X and W in distributed
// shared memory, ROWS spread over the CTAs.  Per round every CTA computes the
// partial (alpha, beta, gamma) of all k/2 disjoint pairs over its rows, one
// cluster barrier publishes them, every CTA reduces the same partials in the
// same order (so all CTAs take identical rotation decisions) and rotates its
// own rows.  Partials are double buffered by round parity: one cluster
// barrier per round.
constexpr int JC_THREADS = 512;

__global__ void __launch_bounds__(JC_THREADS) jacobi_cluster_kernel(int p, int k, double* X,
                                                                     int64_t ldx, double* W,
                                                                     int64_t ldw, double tol,
                                                                     int px, int pw,
                                                                     const double* floor_dev,
                                                                     double floor_scale) {
  extern __shared__ double jc[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  const int kp = k + (k & 1);
  const int np = kp / 2;
  const int x0 = cr * px, nx = max(0, min(p - x0, px));
  const int w0 = cr * pw, nw = max(0, min(k - w0, pw));
  double* Xs = jc;                        // px x kp (column-major, ld px)
  double* Ws = Xs + (size_t)px * kp;      // pw x kp
  double* part = Ws + (size_t)pw * kp;    // [2][cs][np][3], pushed by every CTA
  double* rot = part + 2 * 3 * np * cs;   // [np][2] (c, s); c = 2 marks "no rotation"
  __shared__ int any_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = JC_THREADS / 32;
  for (int idx = tid; idx < px * kp; idx += JC_THREADS) {
    const int r = idx % px, c = idx / px;
    Xs[idx] = (r < nx && c < k) ? X[(x0 + r) + (int64_t)c * ldx] : 0.0;
  }
  for (int idx = tid; idx < pw * kp; idx += JC_THREADS) {
    const int r = idx % pw, c = idx / pw;
    Ws[idx] = (r < nw && c < k) ? ((w0 + r) == c ? 1.0 : 0.0) : 0.0;
  }
  __syncthreads();
  // ||X||_F^2: every CTA pushes its partial into slot [cr] of every CTA
  double* np2 = rot + 2 * np;  // [cs]
  {
    double acc = 0.0;
    for (int idx = tid; idx < px * kp; idx += JC_THREADS) acc = fma(Xs[idx], Xs[idx], acc);
    acc = warp_sum(acc);
    __shared__ double red[JC_THREADS / 32];
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid < cs) {
      double t = 0.0;
      for (int w = 0; w < NWARP; ++w) t += red[w];
      cluster.map_shared_rank(np2, tid)[cr] = t;
    }
  }
  cluster.sync();
  double noise2 = 0.0;
  for (int c = 0; c < cs; ++c) noise2 += np2[c];
  noise2 = fmax(noise2 * kEps * kEps, jacobi_floor2(floor_dev, floor_scale, k));
  int round_no = 0;
  for (int sweep = 0; sweep < JMAXSWEEPS; ++sweep) {
    if (tid == 0) any_rot = 0;
    for (int r = 0; r < kp - 1; ++r, ++round_no) {
      double* pb = part + (size_t)(round_no & 1) * 3 * np * cs;
      for (int q = warp; q < np; q += NWARP) {
        int i, j;
        rr_pair(kp, r, q, i, j);
        double a = 0.0, b = 0.0, g = 0.0;
        for (int rr = lane; rr < nx; rr += 32) {
          const double u = Xs[rr + i * px], v = Xs[rr + j * px];
          a = fma(u, u, a);
          b = fma(v, v, b);
          g = fma(u, v, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        // push this CTA's partials into slot [cr] of every CTA (remote
        // stores do not stall; the cluster barrier orders them)
        if (lane < cs) {
          double* dst = cluster.map_shared_rank(pb, lane) + 3 * ((size_t)cr * np + q);
          dst[0] = a;
          dst[1] = b;
          dst[2] = g;
        }
      }
      cluster.sync();
      for (int q = tid; q < np; q += JC_THREADS) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int c = 0; c < cs; ++c) {
          const double* rp = pb + 3 * ((size_t)c * np + q);
          a += rp[0];
          b += rp[1];
          g += rp[2];
        }
        int i, j;
        rr_pair(kp, r, q, i, j);
        double cc = 2.0, sn = 0.0;
        if (j < k && g != 0.0 && a >= noise2 && b >= noise2 && fabs(g) > tol * sqrt(a) * sqrt(b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          cc = 1.0 / sqrt(fma(t, t, 1.0));
          sn = cc * t;
          any_rot = 1;
        }
        rot[2 * q] = cc;
        rot[2 * q + 1] = sn;
      }
      __syncthreads();
      // rotate local rows of X and W
      const int totx = np * nx, totw = np * nw;
      for (int idx = tid; idx < totx + totw; idx += JC_THREADS) {
        const bool isx = idx < totx;
        const int e = isx ? idx : idx - totx;
        const int nr = isx ? nx : nw;
        const int q = e / nr, rr = e % nr;
        const double cc = rot[2 * q];
        if (cc == 2.0) continue;
        const double sn = rot[2 * q + 1];
        int i, j;
        rr_pair(kp, r, q, i, j);
        double* base = isx ? Xs : Ws;
        const int ld = isx ? px : pw;
        const double u = base[rr + i * ld], v = base[rr + j * ld];
        base[rr + i * ld] = cc * u - sn * v;
        base[rr + j * ld] = sn * u + cc * v;
      }
      __syncthreads();
    }
    const int done = !any_rot;
    __syncthreads();
    if (cr == 0 && tid == 0) g_jacobi_sweeps = sweep + 1;
    if (done) break;
  }
  cluster.sync();  // no CTA exits while others may read its partials
  for (int idx = tid; idx < nx * k; idx += JC_THREADS) {
    const int r = idx % nx, c = idx / nx;
    X[(x0 + r) + (int64_t)c * ldx] = Xs[r + c * px];
  }
  for (int idx = tid; idx < nw * k; idx += JC_THREADS) {
    const int r = idx % nw, c = idx / nw;
    W[(w0 + r) + (int64_t)c * ldw] = Ws[r + c * pw];
  }
}

size_t jacobi_cluster_smem(int px, int pw, int k, int cs) {
  const int kp = k + (k & 1);
  return sizeof(double) * ((size_t)(px + pw) * kp + 3 * (size_t)kp * cs + kp + 16);
}

// Ring one-sided Jacobi (Brent-Luk ordering), the default for p + k <= 640.
// A warp OWNS one column pair per round and holds both augmented columns
// [X(:,c); W(:,c)] in registers (lane l keeps rows l, l+32, ...), so the
// dots, the rotation decision and the rotation itself need no block-level
// reduction.  After the rotation the two columns are pushed straight into
// the (double-buffered, parity = round number) shared-memory slots of the
// pairs that own them in the next round: in the circle schedule the column
// at position pos moves to pos-1 (position 1 wraps to kp-1, 0 is fixed), so
// side-0 columns go to pair q-1 and side-1 columns to pair q+1, which is the
// same CTA except at the chunk edges (those stores cross DSMEM).  One cluster
// barrier per round and no partial-sum traffic; after a whole sweep
// (kp-1 rounds) every column is back at its starting position, so the
// output needs no permutation.  Convergence is agreed by pushing a per-sweep
// "rotated" flag to every CTA before the sweep's last barrier.
constexpr int JR_MAXL = 640;  // p + k limit (E = 20 registers-pairs per lane)

__device__ __forceinline__ void ring_dest(int q, int side, int np, int& dq, int& dside) {
  if (np == 1) {
    dq = 0;
    dside = side;
  } else if (side == 0) {
    dq = q <= 1 ? 0 : q - 1;
    dside = q == 1 ? 1 : 0;
  } else {
    dq = q == np - 1 ? q : q + 1;
    dside = q == np - 1 ? 0 : 1;
  }
}

template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT) jacobi_ring_kernel(int p, int k, double* X, int64_t ldx,
                                                           double* W, int64_t ldw, double tol,
                                                           int ppc, const double* floor_dev,
                                                           double floor_scale) {
  extern __shared__ double jr[];  // [2 parity][ppc][2 side][32 E]
  __shared__ double nrm[16];
  __shared__ int anyrot[2];
  constexpr int LP = 32 * E;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  const int kp = k + (k & 1), np = kp / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = cr * ppc + warp;
  const bool active = q < np;
  const int c0 = q, c1 = kp - 1 - q;  // columns at round 0 (and after every sweep)
  double u[E], v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int t = lane + 32 * e;
    double a = 0.0, b = 0.0;
    if (active) {
      if (t < p) {
        a = X[t + (int64_t)c0 * ldx];
        b = c1 < k ? X[t + (int64_t)c1 * ldx] : 0.0;
      } else if (t < p + k) {
        a = (t - p == c0) ? 1.0 : 0.0;
        b = (t - p == c1 && c1 < k) ? 1.0 : 0.0;
      }
    }
    u[e] = a;
    v[e] = b;
  }
  if (threadIdx.x < 2) anyrot[threadIdx.x] = 0;
  {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (lane + 32 * e < p) acc = fma(u[e], u[e], fma(v[e], v[e], acc));
    acc = warp_sum(acc);
    __shared__ double red[32];
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if ((int)threadIdx.x < cs) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      cluster.map_shared_rank(nrm, (int)threadIdx.x)[cr] = t;
    }
  }
  cluster.sync();
  double noise2 = 0.0;
  for (int c = 0; c < cs; ++c) noise2 += nrm[c];
  noise2 = fmax(noise2 * kEps * kEps, jacobi_floor2(floor_dev, floor_scale, k));
  const double tol2 = tol * tol;

  int dq0, ds0, dq1, ds1;
  ring_dest(q, 0, np, dq0, ds0);
  ring_dest(q, 1, np, dq1, ds1);
  // local stores stay st.shared; only chunk-edge columns cross DSMEM
  double* const base0 = dq0 / ppc == cr ? jr : cluster.map_shared_rank(jr, dq0 / ppc);
  double* const base1 = dq1 / ppc == cr ? jr : cluster.map_shared_rank(jr, dq1 / ppc);
  double* const dst0 = base0 + ((size_t)(dq0 % ppc) * 2 + ds0) * LP;
  double* const dst1 = base1 + ((size_t)(dq1 % ppc) * 2 + ds1) * LP;
  const size_t parity_stride = (size_t)ppc * 2 * LP;
  double* const mine = jr + (size_t)warp * 2 * LP;

  int sweep = 0, rn = 0;
  for (; sweep < JMAXSWEEPS; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < kp - 1; ++r, ++rn) {
      const size_t par = (size_t)(rn & 1) * parity_stride;
      if (active) {
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (lane + 32 * e < p) {
            a = fma(u[e], u[e], a);
            b = fma(v[e], v[e], b);
            g = fma(u[e], v[e], g);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        // same decision and rotation as jacobi_pair; the divisions and
        // square roots go through the Newton-refined hardware approximations
        // (the round's critical path is this scalar chain).
        if (g != 0.0 && a >= noise2 && b >= noise2 && g * g > tol2 * a * b) {
          const double zeta = (b - a) * rcp_nr(2.0 * g);
          const double az = fabs(zeta);
          double t;
          if (az < 1e100) {
            const double w = fma(zeta, zeta, 1.0);
            t = rcp_nr(az + w * rsqrt_nr(w));
          } else {
            t = 0.5 * rcp_nr(az);
          }
          t = zeta >= 0.0 ? t : -t;
          const double c = rsqrt_nr(fma(t, t, 1.0));
          const double sn = c * t;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double x = u[e], y = v[e];
            u[e] = c * x - sn * y;
            v[e] = sn * x + c * y;
          }
          rotated = 1;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          dst0[par + lane + 32 * e] = u[e];
          dst1[par + lane + 32 * e] = v[e];
        }
        if (r == kp - 2 && rotated && lane < cs)
          (lane == cr ? anyrot : cluster.map_shared_rank(anyrot, lane))[sweep & 1] = 1;
      }
      if (cs == 1) __syncthreads();
      else cluster.sync();
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          u[e] = mine[par + lane + 32 * e];
          v[e] = mine[par + LP + lane + 32 * e];
        }
      }
    }
    const int more = anyrot[sweep & 1];
    __syncthreads();
    if (threadIdx.x == 0) anyrot[sweep & 1] = 0;
    if (!more) break;
  }
  if (cr == 0 && threadIdx.x == 0) g_jacobi_sweeps = min(sweep + 1, JMAXSWEEPS);
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int t = lane + 32 * e;
      if (t < p) {
        X[t + (int64_t)c0 * ldx] = u[e];
        if (c1 < k) X[t + (int64_t)c1 * ldx] = v[e];
      } else if (t < p + k) {
        W[(t - p) + (int64_t)c0 * ldw] = u[e];
        if (c1 < k) W[(t - p) + (int64_t)c1 * ldw] = v[e];
      }
    }
  }
  cluster.sync();  // no CTA exits while a neighbour may still push into it
}

template <int E, int MAXT>
int launch_ring_t(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                  double tol, int cs, int ppc, size_t smem, const double* fd, double fs) {
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(jacobi_ring_kernel<E, MAXT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    QTT_CUDA(cudaFuncSetAttribute(jacobi_ring_kernel<E, MAXT>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured.set();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(ppc * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QTT_CUDA(cudaLaunchKernelEx(&cfg, jacobi_ring_kernel<E, MAXT>, p, k, X, ldx, W, ldw, tol, ppc, fd,
                              fs));
  note_launch();
  return kOk;
}

// Returns kUnsupported when the problem does not fit the ring kernel.
int jacobi_ring(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                double tol, const double* fd, double fs) {
  const int L = p + k;
  if (L > JR_MAXL || k < 1) return kUnsupported;
  const int E = (int)ceil_div(L, 32);
  const int Et = E <= 4 ? 4 : E <= 8 ? 8 : E <= 12 ? 12 : E <= 16 ? 16 : 20;
  const int maxw = Et <= 8 ? 32 : 16;  // register budget: 1024 threads need <= 64 regs
  const int np = (k + (k & 1)) / 2;
  for (int cs = 1; cs <= 16; ++cs) {
    const int ppc = (int)ceil_div(np, cs);
    const size_t smem = sizeof(double) * 4 * (size_t)ppc * 32 * Et;
    if (ppc > maxw || smem > 210 * 1024) continue;
    if (ceil_div(np, ppc) != cs) continue;  // every CTA of the cluster owns >= 1 pair
    switch (Et) {
      case 4: return launch_ring_t<4, 1024>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
      case 8: return launch_ring_t<8, 1024>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
      case 12: return launch_ring_t<12, 512>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
      case 16: return launch_ring_t<16, 512>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
      default: return launch_ring_t<20, 512>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
    }
  }
  return kUnsupported;
}

// Ring Jacobi for columns too long for shared-memory slots (p + k > 640,
// k <= 1024): the same warp-per-pair Brent-Luk schedule, but the slots live
// in a global (L2-resident) workspace, double buffered by round parity, and
// each round streams its two columns twice (dots over the X rows, then
// rotate-and-forward), so registers stay O(1).  Loads/stores bypass L1
// (.cg); the cluster barrier (release/acquire at cluster scope) orders them
// between CTAs.  Up to 16 CTAs x 32 warps.
constexpr int GR_U = 8;

__global__ void __launch_bounds__(1024) jacobi_gring_kernel(int p, int k, double* X, int64_t ldx,
                                                            double* W, int64_t ldw, double tol,
                                                            int ppc, double* slots,
                                                            const double* floor_dev,
                                                            double floor_scale) {
  __shared__ double nrm[16];
  __shared__ int anyrot[2];
  __shared__ double red[32];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  const int kp = k + (k & 1), np = kp / 2;
  const int64_t L = (int64_t)p + k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = cr * ppc + warp;
  const bool active = q < np;
  const int c0 = q, c1 = kp - 1 - q;
  auto slot = [&](int par, int qq, int side) {
    return slots + (((int64_t)par * np + qq) * 2 + side) * L;
  };
  double acc = 0.0;
  if (active) {
    double* s0 = slot(0, q, 0);
    double* s1 = slot(0, q, 1);
    for (int64_t t = lane; t < L; t += 32) {
      double a = 0.0, b = 0.0;
      if (t < p) {
        a = X[t + (int64_t)c0 * ldx];
        b = c1 < k ? X[t + (int64_t)c1 * ldx] : 0.0;
        acc = fma(a, a, fma(b, b, acc));
      } else {
        a = (t - p == c0) ? 1.0 : 0.0;
        b = (t - p == c1 && c1 < k) ? 1.0 : 0.0;
      }
      __stcg(s0 + t, a);
      __stcg(s1 + t, b);
    }
  }
  if (threadIdx.x < 2) anyrot[threadIdx.x] = 0;
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if ((int)threadIdx.x < cs) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    cluster.map_shared_rank(nrm, (int)threadIdx.x)[cr] = t;
  }
  cluster.sync();
  double noise2 = 0.0;
  for (int c = 0; c < cs; ++c) noise2 += nrm[c];
  noise2 = fmax(noise2 * kEps * kEps, jacobi_floor2(floor_dev, floor_scale, k));
  const double tol2 = tol * tol;
  int dq0, ds0, dq1, ds1;
  ring_dest(q, 0, np, dq0, ds0);
  ring_dest(q, 1, np, dq1, ds1);
  int sweep = 0, rn = 0;
  for (; sweep < JMAXSWEEPS; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < kp - 1; ++r, ++rn) {
      if (active) {
        const double* u = slot(rn & 1, q, 0);
        const double* v = slot(rn & 1, q, 1);
        double* du = slot((rn + 1) & 1, dq0, ds0);
        double* dv = slot((rn + 1) & 1, dq1, ds1);
        // 8 independent loads per lane in flight (L2 latency bound otherwise)
        double a = 0.0, b = 0.0, g = 0.0;
        for (int t0 = lane; t0 < p; t0 += 32 * GR_U) {
          double xs[GR_U], ys[GR_U];
#pragma unroll
          for (int e = 0; e < GR_U; ++e) {
            const int t = t0 + 32 * e;
            xs[e] = t < p ? __ldcg(u + t) : 0.0;
            ys[e] = t < p ? __ldcg(v + t) : 0.0;
          }
#pragma unroll
          for (int e = 0; e < GR_U; ++e) {
            a = fma(xs[e], xs[e], a);
            b = fma(ys[e], ys[e], b);
            g = fma(xs[e], ys[e], g);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        double c = 1.0, sn = 0.0;
        if (g != 0.0 && a >= noise2 && b >= noise2 && g * g > tol2 * a * b) {
          const double zeta = (b - a) * rcp_nr(2.0 * g);
          const double az = fabs(zeta);
          double t;
          if (az < 1e100) {
            const double w = fma(zeta, zeta, 1.0);
            t = rcp_nr(az + w * rsqrt_nr(w));
          } else {
            t = 0.5 * rcp_nr(az);
          }
          t = zeta >= 0.0 ? t : -t;
          c = rsqrt_nr(fma(t, t, 1.0));
          sn = c * t;
          rotated = 1;
        }
        for (int64_t t0 = lane; t0 < L; t0 += 32 * GR_U) {
          double xs[GR_U], ys[GR_U];
#pragma unroll
          for (int e = 0; e < GR_U; ++e) {
            const int64_t t = t0 + 32 * e;
            xs[e] = t < L ? __ldcg(u + t) : 0.0;
            ys[e] = t < L ? __ldcg(v + t) : 0.0;
          }
#pragma unroll
          for (int e = 0; e < GR_U; ++e) {
            const int64_t t = t0 + 32 * e;
            if (t < L) {
              __stcg(du + t, c * xs[e] - sn * ys[e]);
              __stcg(dv + t, sn * xs[e] + c * ys[e]);
            }
          }
        }
        if (r == kp - 2 && rotated && lane < cs)
          (lane == cr ? anyrot : cluster.map_shared_rank(anyrot, lane))[sweep & 1] = 1;
      }
      cluster.sync();
    }
    const int more = anyrot[sweep & 1];
    __syncthreads();
    if (threadIdx.x == 0) anyrot[sweep & 1] = 0;
    if (!more) break;
  }
  if (cr == 0 && threadIdx.x == 0) g_jacobi_sweeps = min(sweep + 1, JMAXSWEEPS);
  if (active) {
    const double* u = slot(rn & 1, q, 0);
    const double* v = slot(rn & 1, q, 1);
    for (int64_t t = lane; t < L; t += 32) {
      const double x = __ldcg(u + t), y = __ldcg(v + t);
      if (t < p) {
        X[t + (int64_t)c0 * ldx] = x;
        if (c1 < k) X[t + (int64_t)c1 * ldx] = y;
      } else {
        W[(t - p) + (int64_t)c0 * ldw] = x;
        if (c1 < k) W[(t - p) + (int64_t)c1 * ldw] = y;
      }
    }
  }
  cluster.sync();
}

// Ring Jacobi for long columns (p + k in (640, 1024]) with SINGLE-buffered
// shared-memory slots: every pair rotates its two columns in place, then the
// ring migration is done as a PULL in two halves (each lane stages half a
// column pair in registers, cluster barrier, writes its own slot), so a
// cluster of <= 16 CTAs holds the whole augmented matrix in shared memory
// (~15 KB per pair) at three cluster barriers per round and no L2 traffic.
template <int EH>
__global__ void __launch_bounds__(512) jacobi_pring_kernel(int p, int k, double* X, int64_t ldx,
                                                           double* W, int64_t ldw, double tol,
                                                           int ppc, const double* floor_dev,
                                                           double floor_scale) {
  extern __shared__ double jp[];  // [ppc][2][L]
  __shared__ double nrm[16];
  __shared__ int anyrot[2];
  __shared__ double red[32];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  const int kp = k + (k & 1), np = kp / 2;
  const int L = p + k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = cr * ppc + warp;
  const bool active = q < np;
  const int c0 = q, c1 = kp - 1 - q;
  double* const u = jp + (size_t)warp * 2 * L;
  double* const v = u + L;
  double acc = 0.0;
  if (active) {
    for (int t = lane; t < L; t += 32) {
      double a = 0.0, b = 0.0;
      if (t < p) {
        a = X[t + (int64_t)c0 * ldx];
        b = c1 < k ? X[t + (int64_t)c1 * ldx] : 0.0;
        acc = fma(a, a, fma(b, b, acc));
      } else {
        a = (t - p == c0) ? 1.0 : 0.0;
        b = (t - p == c1 && c1 < k) ? 1.0 : 0.0;
      }
      u[t] = a;
      v[t] = b;
    }
  }
  if (threadIdx.x < 2) anyrot[threadIdx.x] = 0;
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if ((int)threadIdx.x < cs) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    cluster.map_shared_rank(nrm, (int)threadIdx.x)[cr] = t;
  }
  cluster.sync();
  double noise2 = 0.0;
  for (int c = 0; c < cs; ++c) noise2 += nrm[c];
  noise2 = fmax(noise2 * kEps * kEps, jacobi_floor2(floor_dev, floor_scale, k));
  const double tol2 = tol * tol;
  // pull sources (inverse of ring_dest)
  int sq0, ss0, sq1, ss1;
  if (np == 1) {
    sq0 = 0; ss0 = 0; sq1 = 0; ss1 = 1;
  } else {
    sq0 = q == 0 ? 0 : (q == np - 1 ? np - 1 : q + 1);
    ss0 = (q == np - 1 && q != 0) ? 1 : 0;
    sq1 = q == 0 ? 1 : q - 1;
    ss1 = q == 0 ? 0 : 1;
  }
  const double* src0 = nullptr;
  const double* src1 = nullptr;
  if (active) {
    const double* b0 = sq0 / ppc == cr ? jp : cluster.map_shared_rank(jp, sq0 / ppc);
    const double* b1 = sq1 / ppc == cr ? jp : cluster.map_shared_rank(jp, sq1 / ppc);
    src0 = b0 + ((size_t)(sq0 % ppc) * 2 + ss0) * L;
    src1 = b1 + ((size_t)(sq1 % ppc) * 2 + ss1) * L;
  }
  const int half = (L + 1) / 2;
  int sweep = 0;
  for (; sweep < JMAXSWEEPS; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < kp - 1; ++r) {
      if (active) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int t = lane; t < p; t += 32) {
          const double x = u[t], y = v[t];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (g != 0.0 && a >= noise2 && b >= noise2 && g * g > tol2 * a * b) {
          const double zeta = (b - a) * rcp_nr(2.0 * g);
          const double az = fabs(zeta);
          double t;
          if (az < 1e100) {
            const double w = fma(zeta, zeta, 1.0);
            t = rcp_nr(az + w * rsqrt_nr(w));
          } else {
            t = 0.5 * rcp_nr(az);
          }
          t = zeta >= 0.0 ? t : -t;
          const double c = rsqrt_nr(fma(t, t, 1.0));
          const double sn = c * t;
          for (int t2 = lane; t2 < L; t2 += 32) {
            const double x = u[t2], y = v[t2];
            u[t2] = c * x - sn * y;
            v[t2] = sn * x + c * y;
          }
          rotated = 1;
        }
        if (r == kp - 2 && rotated && lane < cs)
          (lane == cr ? anyrot : cluster.map_shared_rank(anyrot, lane))[sweep & 1] = 1;
      }
      cluster.sync();  // B1: all rotations (and flags) done
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int lo = hh * half, hi = min(L, lo + half);
        double ru[EH], rv[EH];
        if (active) {
#pragma unroll
          for (int e = 0; e < EH; ++e) {
            const int t = lo + lane + 32 * e;
            ru[e] = t < hi ? src0[t] : 0.0;
            rv[e] = t < hi ? src1[t] : 0.0;
          }
        }
        cluster.sync();  // B2/B3: every reader of this half is done
        if (active) {
#pragma unroll
          for (int e = 0; e < EH; ++e) {
            const int t = lo + lane + 32 * e;
            if (t < hi) {
              u[t] = ru[e];
              v[t] = rv[e];
            }
          }
        }
      }
      __syncwarp();
    }
    const int more = anyrot[sweep & 1];
    __syncthreads();
    if (threadIdx.x == 0) anyrot[sweep & 1] = 0;
    if (!more) break;
  }
  if (cr == 0 && threadIdx.x == 0) g_jacobi_sweeps = min(sweep + 1, JMAXSWEEPS);
  if (active) {
    for (int t = lane; t < L; t += 32) {
      if (t < p) {
        X[t + (int64_t)c0 * ldx] = u[t];
        if (c1 < k) X[t + (int64_t)c1 * ldx] = v[t];
      } else {
        W[(t - p) + (int64_t)c0 * ldw] = u[t];
        if (c1 < k) W[(t - p) + (int64_t)c1 * ldw] = v[t];
      }
    }
  }
  cluster.sync();
}

template <int EH>
int launch_pring_t(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                   double tol, int cs, int ppc, size_t smem, const double* fd, double fs) {
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(jacobi_pring_kernel<EH>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    QTT_CUDA(cudaFuncSetAttribute(jacobi_pring_kernel<EH>,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured.set();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(ppc * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QTT_CUDA(cudaLaunchKernelEx(&cfg, jacobi_pring_kernel<EH>, p, k, X, ldx, W, ldw, tol, ppc, fd, fs));
  note_launch();
  return kOk;
}

int jacobi_pring(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                 double tol, const double* fd, double fs) {
  const int L = p + k;
  if (L > 1024 || k < 2) return kUnsupported;
  const int EH = (int)ceil_div((L + 1) / 2, 32);
  const int np = (k + (k & 1)) / 2;
  for (int cs = 1; cs <= 16; ++cs) {
    const int ppc = (int)ceil_div(np, cs);
    const size_t smem = sizeof(double) * 2 * (size_t)ppc * L;
    if (ppc > 16 || smem > 226 * 1024) continue;
    if (ceil_div(np, ppc) != cs) continue;
    if (EH <= 12) return launch_pring_t<12>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
    return launch_pring_t<16>(s, p, k, X, ldx, W, ldw, tol, cs, ppc, smem, fd, fs);
  }
  return kUnsupported;
}

int jacobi_gring(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                 double tol, const double* fd, double fs) {
  const int np = (k + (k & 1)) / 2;
  if (k < 2 || np > 16 * 32) return kUnsupported;
  int cs = (int)ceil_div(np, 32);
  const int ppc = (int)ceil_div(np, cs);
  cs = (int)ceil_div(np, ppc);
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(jacobi_gring_kernel,
                                  cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured.set();
  }
  double* slots;
  QTT_CUDA(malloc_async(&slots, sizeof(double) * 4 * (size_t)np * ((size_t)p + k), s));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(ppc * 32, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  QTT_CUDA(cudaLaunchKernelEx(&cfg, jacobi_gring_kernel, p, k, X, ldx, W, ldw, tol, ppc, slots, fd,
                              fs));
  note_launch();
  QTT_CUDA(cudaFreeAsync(slots, s));
  return kOk;
}

// Large problems: cooperative grid, columns stay in global memory (L2).
__global__ void __launch_bounds__(256) jacobi_grid_kernel(int p, int k, double* X, int64_t ldx,
                                                          double* W, int64_t ldw, double tol,
                                                          int* flags) {
  cg::grid_group grid = cg::this_grid();
  const int kp = k + (k & 1);
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  for (int sweep = 0; sweep < JMAXSWEEPS; ++sweep) {
    int any = 0;
    for (int r = 0; r < kp - 1; ++r) {
      for (int q = gw; q < kp / 2; q += nw) {
        int i, j;
        rr_pair(kp, r, q, i, j);
        if (j < k) any |= jacobi_pair(X, ldx, W, ldw, p, k, i, j, tol, 0.0);
      }
      grid.sync();
    }
    if (any && (threadIdx.x & 31) == 0) atomicOr(&flags[sweep], 1);
    grid.sync();
    if (flags[sweep] == 0) break;
  }
}

// --------------------------------------------------------------- sort/chop
constexpr int SORT_MAX = 8192;

__global__ void __launch_bounds__(1024) sort_chop_kernel(int p, int k, const double* X,
                                                         int64_t ldx, double* sigma, int* perm,
                                                         const double* delta_dev,
                                                         double delta_scale, int rmax,
                                                         int floor_rule, int* rank_dev) {
  extern __shared__ double sort_sm[];
  double* sv = sort_sm;
  double* ss = sort_sm + k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < k; c += nw) {
    double a = 0.0;
    for (int r = lane; r < p; r += 32) {
      const double x = X[r + (int64_t)c * ldx];
      a = fma(x, x, a);
    }
    a = warp_sum(a);
    if (lane == 0) sv[c] = sqrt(a);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double v = sv[i];
    int pos = 0;
    for (int j = 0; j < k; ++j) {
      const double w = sv[j];
      pos += (w > v) || (w == v && j < i);
    }
    ss[pos] = v;
    perm[pos] = i;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) sigma[i] = ss[i];
  if (threadIdx.x == 0) {
    double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
    if (floor_rule) delta = fmax(delta, ss[0] * (double)max(k, 2) * kEps);
    double acc = 0.0;
    int r = 1;
    for (int i = k - 1; i >= 0; --i) {
      acc += ss[i] * ss[i];
      if (sqrt(acc) > delta) { r = i + 1; break; }
    }
    *rank_dev = max(1, min(r, rmax));
  }
}

// ----------------------------------------------------------- certificate
constexpr int TRB = 64;

// Invert the 64x64 diagonal blocks of an upper-triangular R (one CTA each),
// block held in registers (common.cuh, blk_tri_inverse).
__global__ void __launch_bounds__(256) trinv_diag_kernel(int k, const double* __restrict__ R,
                                                         int64_t ldr, double* __restrict__ X,
                                                         int64_t ldx) {
  extern __shared__ double tri_sm[];
  double (*S)[kBlk + 1] = reinterpret_cast<double (*)[kBlk + 1]>(tri_sm);
  double* line = tri_sm + kBlk * (kBlk + 1);
  double* dinv = line + 256;
  const int b0 = blockIdx.x * TRB;
  const int nb = min(TRB, k - b0);
  double a[16], x[16], y[16];
  blk_load(a, R + b0 + (int64_t)b0 * ldr, ldr, nb);
  blk_to_smem(a, S);
  __syncthreads();
  blk_tri_inverse<false>(S, x, y, line, dinv);
  blk_store(x, X + b0 + (int64_t)b0 * ldx, ldx, nb);
}

// Deterministic two-stage sum of squares.
__global__ void sumsq_partial_kernel(int64_t n, const double* __restrict__ x,
                                     double* __restrict__ part) {
  __shared__ double red[32];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    a = fma(v, v, a);
  }
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void sum_final_kernel(int nparts, const double* __restrict__ part, double* out,
                                 int take_sqrt) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += part[i];
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(v) : v;
  }
}

__global__ void certificate_kernel(int k, const double* rnorm, const double* xnorm,
                                   const double* delta_dev, double delta_scale, int* ok,
                                   int debug) {
  const double rn = *rnorm, xn = *xnorm;
  const double delta = delta_dev ? (*delta_dev) * delta_scale : 0.0;
  const double thr = fmax(delta, rn * (double)max(k, 2) * kEps);
  const bool good = isfinite(xn) && isfinite(rn) && xn > 0.0 && (1.0 / xn) > 1.25 * thr;
  *ok = good ? 1 : 0;
  if (debug) printf("[cert] k=%d smin/||R||=%.3e thr/||R||=%.3e good=%d\n", k, 1.0 / xn / rn,
                    thr / rn, (int)good);
}

__global__ void gather_columns_kernel(int rows, int cols, const double* __restrict__ src,
                                      int64_t lds, const int* __restrict__ perm,
                                      double* __restrict__ dst, int64_t ldd) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows);
    const int64_t c = i / rows;
    dst[r + c * ldd] = src[r + (int64_t)perm[c] * lds];
  }
}

}  // namespace

int set_identity(cudaStream_t s, int rows, int cols, double* A, int64_t lda) {
  if (rows <= 0 || cols <= 0) return kOk;
  identity_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(rows, cols, A, lda);
  QTT_CHECK_LAUNCH();
  return kOk;
}

// Side stream for the look-ahead panel factorisation (one per process).
cudaStream_t side_stream() {
  thread_local cudaStream_t st = nullptr;
  if (!st) {
    // highest priority: the panel (critical path) is scheduled ahead of the
    // trailing-update GEMM blocks as soon as SMs free up
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi);
  }
  return st;
}

// ------------------------------------------------------------- small QR
// Whole Householder QR of a small matrix (n <= 64, m <= 256, A in shared
// memory) in ONE CTA, left-looking and dataflow-ordered: warp w owns columns
// w, w+16, w+32, w+48 and finishes them in increasing order; a column gets
// every published reflector applied as soon as its ready flag is up, then
// its own reflector is formed and published (v in A's lower part, tau,
// beta on the diagonal).  The serial chain per column is therefore
// flag -> one column update -> reflector -> flag, with no block barrier;
// the catch-up of a warp's next column overlaps the other warps' chain.
// The explicit Q is formed in registers, q_c = H_0 ... H_c e_c, with the
// owned columns interleaved so their warp reductions overlap.  Replaces the
// 32-wide cluster panel + compact-WY GEMMs for the small cores of a
// rounding sweep (~90 us of serial panel latency per 32 columns).
constexpr int SQ_THREADS = 512, SQ_WARPS = SQ_THREADS / 32, SQ_MAXN = 64, SQ_MAXM = 256;
constexpr int SQ_CPW = SQ_MAXN / SQ_WARPS;  // columns per warp

// Shared-memory flag handshake with release/acquire semantics at CTA scope
// (cheaper than a sequentially consistent __threadfence_block()).
__device__ __forceinline__ void flag_release(volatile int* f) {
  const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)f);
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(a), "r"(1) : "memory");
}
__device__ __forceinline__ int flag_acquire(volatile int* f) {
  const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)f);
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ void sq_apply(const double* v, double* col, double tj, int j, int m,
                                         int lane) {
  double w = 0.0;
  for (int r = j + 1 + lane; r < m; r += 32) w = fma(v[r], col[r], w);
  w = warp_sum(w) + col[j];
  const double tw = tj * w;
  for (int r = j + 1 + lane; r < m; r += 32) col[r] = fma(-tw, v[r], col[r]);
  __syncwarp();
  if (lane == 0) col[j] -= tw;
  __syncwarp();
}

__device__ __forceinline__ void sq_reflect(double* sa, int m, int j, double* tau_s,
                                           volatile int* ready, int lane) {
  double* col = sa + (int64_t)j * m;
  double nrm2 = 0.0;
  for (int r = j + 1 + lane; r < m; r += 32) nrm2 = fma(col[r], col[r], nrm2);
  nrm2 = warp_sum(nrm2);
  const double alpha = col[j];
  double tau = 0.0, beta = alpha, scal = 1.0;
  if (nrm2 > 0.0) {
    const double nrm = sqrt(fma(alpha, alpha, nrm2));
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  for (int r = j + 1 + lane; r < m; r += 32) col[r] *= scal;
  __syncwarp();
  if (lane == 0) {
    col[j] = beta;
    tau_s[j] = tau;
  }
  __syncwarp();
  if (lane == 0) flag_release(ready + j);
}

template <int E>
__global__ void __launch_bounds__(SQ_THREADS) small_qr_kernel(int m, int n, const double* A,
                                                              int64_t lda, double* Q, int64_t ldq,
                                                              double* R, int64_t ldr, int dbg,
                                                              int sq_sleep) {
  extern __shared__ double sa[];  // m x n, ld m
  __shared__ double tau_s[SQ_MAXN];
  __shared__ int ready_s[SQ_MAXN];
  __shared__ long long tpub[SQ_MAXN + 4];
  const long long t0 = clock64();
  volatile int* ready = ready_s;
  const int k = min(m, n);
  for (int idx = threadIdx.x; idx < m * n; idx += SQ_THREADS)
    sa[idx] = A[(idx % m) + (int64_t)(idx / m) * lda];
  if (threadIdx.x < SQ_MAXN) ready_s[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) tpub[SQ_MAXN] = clock64() - t0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < n; c += SQ_WARPS) {
    double* col = sa + (int64_t)c * m;
    const int jmax = min(c, k);
    for (int j = 0; j < jmax; ++j) {
      while (flag_acquire(ready + j) == 0) {
        if (sq_sleep) __nanosleep(sq_sleep);
      }
      const double tj = tau_s[j];
      if (tj != 0.0) sq_apply(sa + (int64_t)j * m, col, tj, j, m, lane);
    }
    if (c < k) sq_reflect(sa, m, c, tau_s, ready, lane);
    if (dbg && lane == 0 && c < SQ_MAXN) tpub[c] = clock64() - t0;
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) {
    printf("[sqr] m=%d n=%d load=%lld", m, n, tpub[SQ_MAXN]);
    for (int c = 0; c < k; c += max(1, k / 8)) printf(" T%d=%lld", c, tpub[c]);
    printf(" fact_end=%lld\n", clock64() - t0);
  }
  if (R) {
    for (int idx = threadIdx.x; idx < k * n; idx += SQ_THREADS) {
      const int r = idx % k, c = idx / k;
      R[r + (int64_t)c * ldr] = (r <= c) ? sa[r + (int64_t)c * m] : 0.0;
    }
  }
  if (!Q) return;
  // owned Q columns c_i = warp + 16 i (< k), all advanced together
  double q[SQ_CPW][E];
  int cmax = -1;
#pragma unroll
  for (int i = 0; i < SQ_CPW; ++i) {
    const int c = warp + SQ_WARPS * i;
    if (c < k) cmax = c;
#pragma unroll
    for (int e = 0; e < E; ++e) q[i][e] = (lane + 32 * e == c) ? 1.0 : 0.0;
  }
  for (int j = cmax; j >= 0; --j) {
    const double tj = tau_s[j];
    if (tj == 0.0) continue;
    const double* v = sa + (int64_t)j * m;
    double vr[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int r = lane + 32 * e;
      vr[e] = (r < m && r > j) ? v[r] : (r == j ? 1.0 : 0.0);
    }
    double w[SQ_CPW];
#pragma unroll
    for (int i = 0; i < SQ_CPW; ++i) {
      w[i] = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) w[i] = fma(vr[e], q[i][e], w[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < SQ_CPW; ++i) w[i] += __shfl_xor_sync(0xffffffffu, w[i], o);
#pragma unroll
    for (int i = 0; i < SQ_CPW; ++i) {
      // q_c is still e_c while j > c, and H_j e_c = e_c there
      if (warp + SQ_WARPS * i < j) continue;
      const double tw = tj * w[i];
#pragma unroll
      for (int e = 0; e < E; ++e) q[i][e] = fma(-tw, vr[e], q[i][e]);
    }
  }
#pragma unroll
  for (int i = 0; i < SQ_CPW; ++i) {
    const int c = warp + SQ_WARPS * i;
    if (c >= k) continue;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int r = lane + 32 * e;
      if (r < m) Q[r + (int64_t)c * ldq] = q[i][e];
    }
  }
}

bool small_qr_fits(int m, int n) { return n <= SQ_MAXN && m <= SQ_MAXM; }

int small_qr(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
             double* R, int64_t ldr) {
  const size_t smem = sizeof(double) * (size_t)m * n;
  static const int dbg = getenv("QTT_SQR_DEBUG") ? 1 : 0;
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(small_qr_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SQ_MAXM * SQ_MAXN * 8));
    QTT_CUDA(cudaFuncSetAttribute(small_qr_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SQ_MAXM * SQ_MAXN * 8));
    configured.set();
  }
  static const int slp = getenv("QTT_SQR_SLEEP") ? atoi(getenv("QTT_SQR_SLEEP")) : 0;
  if (m <= 128)
    small_qr_kernel<4><<<1, SQ_THREADS, smem, s>>>(m, n, A, lda, Q, ldq, R, ldr, dbg, slp);
  else
    small_qr_kernel<8><<<1, SQ_THREADS, smem, s>>>(m, n, A, lda, Q, ldq, R, ldr, dbg, slp);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int qr(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
       double* R, int64_t ldr, int* spec_dev, bool careful, QrInfo* info) {
  if (info) info->valid = false;
  if (m <= 0 || n <= 0) return kInvalid;
  const int k = std::min(m, n);
  static const bool use_small = getenv("QTT_NO_SMALLQR") == nullptr;
  // Small tall factors: sync-free CholeskyQR2 (7 launches) beats the serial
  // Householder chain of small_qr from n = 32 on (75 / 155 us at n = 32 / 64).
  static const bool use_cq_small = getenv("QTT_NO_CHOLQR_SMALL") == nullptr;
  if (use_cq_small && !careful && m >= n && n >= kCholQrSmallMin && n <= kCholQrSmallMax) {
    if (spec_dev) return cholqr2_small(s, m, n, A, lda, Q, ldq, R, ldr, spec_dev);
    int* st;
    QTT_CUDA(malloc_async(&st, sizeof(int), s));
    QTT_CUDA(cudaMemsetAsync(st, 0, sizeof(int), s));
    QTT_TRY(cholqr2_small(s, m, n, A, lda, Q, ldq, R, ldr, st));
    int hst = 0;
    QTT_CUDA(cudaMemcpyAsync(&hst, st, sizeof(int), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    QTT_CUDA(cudaFreeAsync(st, s));
    if (!hst) return kOk;
  }
  if (use_small && small_qr_fits(m, n)) return small_qr(s, m, n, A, lda, Q, ldq, R, ldr);
  // Large tall factors: try the GEMM-bound CholeskyQR2 first (certified, falls
  // back to Householder for ill-conditioned / rank-deficient inputs).
  static const bool use_chol = getenv("QTT_NO_CHOLQR") == nullptr;
  if (use_chol && m >= n && n >= 128) {
    double* Rt = R;
    if (!R) QTT_CUDA(malloc_async(&Rt, sizeof(double) * (int64_t)n * n, s));
    int ok = 0;
    QTT_TRY(cholqr2(s, m, n, A, lda, Q, Q ? ldq : m, Rt, R ? ldr : n, &ok, info));  // Q may be null (R only)
    if (!R) QTT_CUDA(cudaFreeAsync(Rt, s));
    static const bool dbg = getenv("QTT_QR_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "[qr] cholqr2 m=%d n=%d %s\n", m, n, ok ? "ok" : "fallback");
    if (ok) return kOk;
  }
  if (ceil_div(m, PMAXROWS16) > PMAXCLUSTER) return kUnsupported;
  const int PW = panel_width(m);
  double *Ac, *V, *Y, *Y2, *tau, *W, *W1;
  const int64_t mm = m;
  QTT_CUDA(malloc_async(&Ac, sizeof(double) * mm * n, s));
  QTT_CUDA(malloc_async(&V, sizeof(double) * mm * k, s));
  QTT_CUDA(malloc_async(&Y, sizeof(double) * mm * k, s));
  QTT_CUDA(malloc_async(&Y2, sizeof(double) * mm * k, s));
  QTT_CUDA(malloc_async(&tau, sizeof(double) * (k + 1), s));
  QTT_CUDA(malloc_async(&W, sizeof(double) * PW * (int64_t)std::max(n, k), s));
  QTT_CUDA(malloc_async(&W1, sizeof(double) * PW * PW, s));
  QTT_TRY(copy_matrix(s, m, n, A, lda, Ac, m));
  // Look-ahead: after panel p, update only panel p+1's columns, factor panel
  // p+1 on a side stream while the rest of the trailing matrix is updated,
  // so the latency-bound panel overlaps the DMMA update.
  thread_local cudaEvent_t ev_cols = nullptr, ev_panel = nullptr;
  if (!ev_cols) {
    QTT_CUDA(cudaEventCreateWithFlags(&ev_cols, cudaEventDisableTiming));
    QTT_CUDA(cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming));
  }
  cudaStream_t sb = side_stream();
  auto panel_args = [&](int j0) {
    const int nb = std::min(PW, k - j0);
    return PanelArgs{m - j0, nb, 0, Ac + j0 + (int64_t)j0 * m, mm, V + j0 + (int64_t)j0 * m, mm,
                     Y + j0 + (int64_t)j0 * m, mm, Y2 + j0 + (int64_t)j0 * m, mm, tau + j0};
  };
  static const bool lookahead = getenv("QTT_NO_LOOKAHEAD") == nullptr;
  if (!lookahead) {
    for (int j0 = 0; j0 < k; j0 += PW) {
      const int nb = std::min(PW, k - j0);
      const int mp = m - j0, nt = n - j0 - nb;
      QTT_TRY(launch_panel(s, panel_args(j0)));
      if (nt > 0) {
        double* At = Ac + j0 + (int64_t)(j0 + nb) * m;
        QTT_TRY(dgemm(s, 1, 0, nb, nt, mp, 1.0, V + j0 + (int64_t)j0 * m, mm, At, mm, 0.0, W, nb));
        QTT_TRY(dgemm(s, 0, 0, mp, nt, nb, -1.0, Y + j0 + (int64_t)j0 * m, mm, W, nb, 1.0, At, mm));
      }
    }
  } else {
  QTT_TRY(launch_panel(s, panel_args(0)));
  for (int j0 = 0; j0 < k; j0 += PW) {
    const int nb = std::min(PW, k - j0);
    const int mp = m - j0;
    const int nt = n - j0 - nb;
    if (nt <= 0) break;
    const double* Vp = V + j0 + (int64_t)j0 * m;
    const double* Yp = Y + j0 + (int64_t)j0 * m;
    const int jn = j0 + nb;
    const int nb_next = jn < k ? std::min(PW, k - jn) : 0;
    if (nb_next > 0) {
      double* An = Ac + j0 + (int64_t)jn * m;
      QTT_TRY(dgemm(s, 1, 0, nb, nb_next, mp, 1.0, Vp, mm, An, mm, 0.0, W1, nb));
      QTT_TRY(dgemm(s, 0, 0, mp, nb_next, nb, -1.0, Yp, mm, W1, nb, 1.0, An, mm));
      QTT_CUDA(cudaEventRecord(ev_cols, s));
      QTT_CUDA(cudaStreamWaitEvent(sb, ev_cols, 0));
      QTT_TRY(launch_panel(sb, panel_args(jn)));
      QTT_CUDA(cudaEventRecord(ev_panel, sb));
    }
    const int rest = nt - nb_next;
    if (rest > 0) {
      double* Ar = Ac + j0 + (int64_t)(jn + nb_next) * m;
      QTT_TRY(dgemm(s, 1, 0, nb, rest, mp, 1.0, Vp, mm, Ar, mm, 0.0, W, nb));
      QTT_TRY(dgemm(s, 0, 0, mp, rest, nb, -1.0, Yp, mm, W, nb, 1.0, Ar, mm));
    }
    if (nb_next > 0) QTT_CUDA(cudaStreamWaitEvent(s, ev_panel, 0));
  }
  }
  if (R) {
    upper_copy_kernel<<<grid_for((int64_t)k * n), 256, 0, s>>>(k, n, Ac, mm, R, ldr);
    QTT_CHECK_LAUNCH();
  }
  if (Q) {
    QTT_TRY(set_identity(s, m, k, Q, ldq));
    const int last = ((k - 1) / PW) * PW;
    for (int j0 = last; j0 >= 0; j0 -= PW) {
      const int nb = std::min(PW, k - j0);
      const int mp = m - j0, kc = k - j0;
      double* Qs = Q + j0 + (int64_t)j0 * ldq;
      QTT_TRY(dgemm(s, 1, 0, nb, kc, mp, 1.0, V + j0 + (int64_t)j0 * m, mm, Qs, ldq, 0.0, W, nb));
      QTT_TRY(dgemm(s, 0, 0, mp, kc, nb, -1.0, Y2 + j0 + (int64_t)j0 * m, mm, W, nb, 1.0, Qs, ldq));
    }
  }
  QTT_CUDA(cudaFreeAsync(Ac, s));
  QTT_CUDA(cudaFreeAsync(V, s));
  QTT_CUDA(cudaFreeAsync(Y, s));
  QTT_CUDA(cudaFreeAsync(Y2, s));
  QTT_CUDA(cudaFreeAsync(tau, s));
  QTT_CUDA(cudaFreeAsync(W, s));
  QTT_CUDA(cudaFreeAsync(W1, s));
  return kOk;
}

static int jacobi_impl(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                       const double* fd, double fs);

int jacobi(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
           const double* floor_dev, double floor_scale) {
  static const bool dbg = getenv("QTT_JACOBI_DEBUG") != nullptr;
  cudaEvent_t e0, e1;
  if (dbg) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  const int st = jacobi_impl(s, p, k, X, ldx, W, ldw, floor_dev, floor_scale);
  if (dbg) {
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    int sw = 0;
    cudaMemcpyFromSymbol(&sw, g_jacobi_sweeps, sizeof(int));
    fprintf(stderr, "[jacobi] p=%d k=%d sweeps=%d ms=%.3f\n", p, k, sw, ms);
  }
  return st;
}

static int jacobi_impl(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
                       const double* fd, double fs) {
  if (p <= 0 || k <= 0) return kInvalid;
  // Off-diagonal cosine threshold.  Rotating below ~32 sqrt(p) eps only churns
  // rounding noise: singular values move at second order (~1e-28) and the
  // singular vectors stay orthogonal to ~1e-14.
  const double tol = 32.0 * sqrt((double)std::max(p, 1)) * kEps;
  // QTT_JACOBI_KERNEL=legacy forces the row-distributed kernels (A/B checks).
  static const char* kern = getenv("QTT_JACOBI_KERNEL");
  static const bool legacy = kern && std::string(kern) == "legacy";
  if (!legacy) {
    int st = jacobi_ring(s, p, k, X, ldx, W, ldw, tol, fd, fs);
    if (st == kUnsupported) st = jacobi_pring(s, p, k, X, ldx, W, ldw, tol, fd, fs);
    if (st == kUnsupported) st = jacobi_gring(s, p, k, X, ldx, W, ldw, tol, fd, fs);
    if (st != kUnsupported) return st;
  }
  const size_t smem = sizeof(double) * ((size_t)p * k + (size_t)k * k);
  if (smem <= 200 * 1024) {
    static DeviceFlag configured;
    if (!configured.test()) {
      QTT_CUDA(cudaFuncSetAttribute(jacobi_smem_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      configured.set();
    }
    const int threads = std::min(JTHREADS, std::max(32, ((k + 1) / 2) * 32));
    jacobi_smem_kernel<<<1, threads, smem, s>>>(p, k, X, ldx, W, ldw, tol, fd, fs);
    QTT_CHECK_LAUNCH();
    return kOk;
  }
  // cluster path: smallest cluster whose per-CTA slice fits 200 KB
  for (int cs = 2; cs <= 16; ++cs) {
    const int px = (int)ceil_div(p, cs), pw = (int)ceil_div(k, cs);
    const size_t bytes = jacobi_cluster_smem(px, pw, k, cs);
    if (bytes > 200 * 1024) continue;
    static bool cconf = false;
    if (!cconf) {
      QTT_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      QTT_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cconf = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(JC_THREADS, 1, 1);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    QTT_CUDA(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel, p, k, X, ldx, W, ldw, tol, px, pw, fd,
                                fs));
    note_launch();
    return kOk;
  }
  QTT_TRY(set_identity(s, k, k, W, ldw));
  int* flags;
  QTT_CUDA(malloc_async(&flags, sizeof(int) * JMAXSWEEPS, s));
  QTT_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * JMAXSWEEPS, s));
  int dev = 0, per_sm = 0;
  QTT_CUDA(cudaGetDevice(&dev));
  QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, 256, 0));
  const int pairs = (k + 1) / 2;
  int blocks = std::max(1, std::min((int)ceil_div(pairs, 8), per_sm * num_sms()));
  double tol_v = tol;
  void* args[] = {&p, &k, &X, &ldx, &W, &ldw, &tol_v, &flags};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_grid_kernel, dim3(blocks), dim3(256), args, 0,
                                       s));
  note_launch();
  QTT_CUDA(cudaFreeAsync(flags, s));
  return kOk;
}

int sort_chop(cudaStream_t s, int p, int k, const double* X, int64_t ldx, double* sigma,
              int* perm, const double* delta_dev, double delta_scale, int rmax, int floor_rule,
              int* rank_dev) {
  if (k <= 0 || k > SORT_MAX) return kUnsupported;
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(sort_chop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(2 * SORT_MAX * sizeof(double))));
    configured.set();
  }
  sort_chop_kernel<<<1, 1024, 2 * k * sizeof(double), s>>>(p, k, X, ldx, sigma, perm, delta_dev, delta_scale, rmax,
                                      floor_rule, rank_dev);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int frob_norm(cudaStream_t s, int64_t n, const double* x, double* out_dev) {
  const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 1024), 1024));
  double* part;
  QTT_CUDA(malloc_async(&part, sizeof(double) * parts, s));
  sumsq_partial_kernel<<<parts, 256, 0, s>>>(n, x, part);
  QTT_CHECK_LAUNCH();
  sum_final_kernel<<<1, 1024, 0, s>>>(parts, part, out_dev, 1);
  QTT_CHECK_LAUNCH();
  QTT_CUDA(cudaFreeAsync(part, s));
  return kOk;
}

int tri_inverse(cudaStream_t s, int k, const double* R, int64_t ldr, double* X) {
  double* T;
  const int64_t kk = k;
  QTT_CUDA(malloc_async(&T, sizeof(double) * kk * kk, s));
  QTT_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * kk * kk, s));
  static DeviceFlag configured;
  const int tri_smem = (int)((kBlk * (kBlk + 1) + 256 + kBlk) * sizeof(double));
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(trinv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  tri_smem));
    configured.set();
  }
  trinv_diag_kernel<<<(int)ceil_div(k, TRB), 256, tri_smem, s>>>(k, R, ldr, X, kk);
  QTT_CHECK_LAUNCH();
  // Recursive doubling: X12 = -X11 * R12 * X22 for block pairs of size sz.
  // All full pairs of a level have the same shape and a constant stride
  // 2 sz (1 + ld) along the diagonal: one batched GEMM per product and level;
  // a trailing partial pair (c < sz) is issued separately.  X22 and X11 are
  // upper triangular, so each tile's reduction is clipped to their nonzeros
  // (kGemmTriB / kGemmTriA: half the flops, bitwise the same result).
  for (int sz = TRB; sz < k; sz *= 2) {
    const int full = (k / (2 * sz));  // pairs with c == sz
    if (full > 0) {
      GemmArgs g1{sz, sz, sz, 0, 0, 1.0, 0.0,
                  R + (int64_t)sz * ldr, ldr, 2 * (int64_t)sz * (1 + ldr),
                  X + sz + (int64_t)sz * kk, kk, 2 * (int64_t)sz * (1 + kk),
                  T, sz, (int64_t)sz * sz, full, kGemmTriB};
      QTT_TRY(gemm(g1, s));
      GemmArgs g2{sz, sz, sz, 0, 0, -1.0, 0.0,
                  X, kk, 2 * (int64_t)sz * (1 + kk),
                  T, sz, (int64_t)sz * sz,
                  X + (int64_t)sz * kk, kk, 2 * (int64_t)sz * (1 + kk), full, kGemmTriA};
      QTT_TRY(gemm(g2, s));
    }
    const int b = full * 2 * sz;
    if (b + sz < k) {
      const int c = k - b - sz;  // < sz
      const double* R12 = R + b + (int64_t)(b + sz) * ldr;
      const double* X22 = X + (b + sz) + (int64_t)(b + sz) * kk;
      const double* X11 = X + b + (int64_t)b * kk;
      double* X12 = X + b + (int64_t)(b + sz) * kk;
      QTT_TRY(dgemm(s, 0, 0, sz, c, c, 1.0, R12, ldr, X22, kk, 0.0, T, sz, kGemmTriB));
      QTT_TRY(dgemm(s, 0, 0, sz, c, sz, -1.0, X11, kk, T, sz, 0.0, X12, kk, kGemmTriA));
    }
  }
  QTT_CUDA(cudaFreeAsync(T, s));
  return kOk;
}

int no_truncation_certificate(cudaStream_t s, int k, const double* R, int64_t ldr,
                              const double* delta_dev, double delta_scale, int* ok_dev) {
  static const bool use_small = getenv("QTT_NO_CERT_SMALL") == nullptr;
  if (use_small && k <= 2 * kBlk) return cert_small(s, k, R, ldr, delta_dev, delta_scale, ok_dev, nullptr);
  double *X, *norms;
  const int64_t kk = k;
  QTT_CUDA(malloc_async(&X, sizeof(double) * kk * kk, s));
  QTT_CUDA(malloc_async(&norms, sizeof(double) * 2, s));
  QTT_TRY(tri_inverse(s, k, R, ldr, X));
  // ||R||_F (upper triangle of R as stored: caller guarantees zeros below)
  double* Rc;
  QTT_CUDA(malloc_async(&Rc, sizeof(double) * kk * kk, s));
  QTT_TRY(copy_matrix(s, k, k, R, ldr, Rc, kk));
  QTT_TRY(frob_norm(s, kk * kk, Rc, norms));
  QTT_TRY(frob_norm(s, kk * kk, X, norms + 1));
  static const int debug = getenv("QTT_CERT_DEBUG") ? 1 : 0;
  certificate_kernel<<<1, 1, 0, s>>>(k, norms, norms + 1, delta_dev, delta_scale, ok_dev, debug);
  QTT_CHECK_LAUNCH();
  QTT_CUDA(cudaFreeAsync(Rc, s));
  QTT_CUDA(cudaFreeAsync(X, s));
  QTT_CUDA(cudaFreeAsync(norms, s));
  return kOk;
}

int gather_columns(cudaStream_t s, int rows, int cols, const double* src, int64_t lds,
                   const int* perm, double* dst, int64_t ldd) {
  if (rows <= 0 || cols <= 0) return kOk;
  gather_columns_kernel<<<grid_for((int64_t)rows * cols), 256, 0, s>>>(rows, cols, src, lds, perm,
                                                                       dst, ldd);
  QTT_CHECK_LAUNCH();
  return kOk;
}

}  // namespace qtt
