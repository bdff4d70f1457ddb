// TT-SVD of a dense vector (row a6, ttcore.py:193-264) by device-resident
// supersteps.
//
// The reference sweeps d-1 sequential SVDs of the unfoldings
// M_l = reshape(carry_{l-1}, r_{l-1} n_l x rest) (ttcore.py:193-208), each a
// pass over the whole remaining data.  Here k consecutive steps are decided
// from ONE pass ("superstep"): with V = reshape(carry, p x N), p = r n_l ...
// n_{l+k-1} <= 64, every M_{l+s} equals a small matrix P_s times a matrix
// with orthonormal rows, where P_0 is built from any factor L with
// V V^T = L L^T.  So a pass only has to produce the p x p Gram matrix of V;
// the k SVDs, rank decisions (the reference's _chop rule, ttcore.py:175-190)
// and cores are computed on chip by one CTA, which also forms the composite
// basis Gc (p x r_{l+k-1}) whose projection Gc^T V is the next carry.  The
// next superstep's pass computes that projection and, from the same tile,
// the next Gram matrix: each element of the data is read once and written
// once per superstep.
//
// Accuracy.  A Gram matrix formed in FP64 loses every singular value below
// sqrt(eps_mach) ||V||.  The Gram here is accumulated in
// double-double (error-free products and sums, ~1e-32 relative), factored
// by a pivoted Cholesky in double-double, and only the Cholesky factor is
// rounded to FP64: the resulting L has backward error ~eps_mach ||V||, the
// same as the Householder QR that LAPACK's dgesdd applies first.  The step
// SVDs are one-sided Jacobi (backward stable) on the small P_s.
//
// Launch structure.  Each superstep is ONE kernel launch (grid-stride pass +
// last-CTA small phase) driven by a state block in device memory, so the
// host queues launches without synchronising and reads the ranks once at
// the end.  When r_l n_l > 64 the remaining steps are handed back to the
// per-step path in round.cu (decompose()).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/qtt_b200.h"
#include "linalg.cuh"

namespace qtt {

namespace {

constexpr int SV_PMAX = 64;                          // rows of a superstep column
constexpr int SV_P0 = 16;                            // rows in the first (largest) pass
constexpr int SV_NT = 512;                           // threads per CTA
constexpr int SV_NW = SV_NT / 32;
constexpr int SV_NE = SV_PMAX * (SV_PMAX + 1) / 2;   // Gram entries (upper triangle)
constexpr int SV_EPT = (SV_NE + SV_NT - 1) / SV_NT;  // entries per thread
constexpr int SV_CORE = SV_PMAX * SV_PMAX;           // staging doubles per core
constexpr int SV_TILE = 6144;                        // doubles of a source / carry tile
constexpr int SV_SMEM_DBL = 22528;                   // dynamic shared memory (176 KB)

enum SvMode { kGramInput = 0, kProjectGram = 1, kProjectOnly = 2, kDone = 3 };

struct SvState {
  int mode;
  int l;        // first step (decision index) of the superstep
  int k;        // steps decided by the superstep
  int r_in;     // rank entering the superstep (rows of the projected carry)
  int pg;       // rows of a Gram column: r_in * n_l ... n_{l+k-1}
  int gsz;      // carry columns per Gram column
  int p_src;    // rows of a source column
  int src_sel;  // 0: dense input, 1/2: carry buffer 0/1
  int dst_sel;  // carry buffer written by the projection (1/2)
  int handoff;  // kDone reached because r_l n_l > SV_PMAX
  int zero;     // the input is the zero vector
  int pad;
  long long n_src;  // source columns
  double delta;     // eps / sqrt(d-1) * ||v||
  unsigned int counter;
  int ranks[QTT_MAX_CORES + 1];
  long long clk[8];  // QTT_TTSVD_DEBUG: section timestamps of the last small phase
  int sweeps[QTT_MAX_CORES];  // Jacobi sweeps per step (diagnostics)
};

struct SvParams {
  int d;
  double eps_scale;                        // eps / sqrt(d-1)
  int64_t n[QTT_MAX_CORES];                // mode sizes
  int64_t rest[QTT_MAX_CORES + 1];         // rest[l] = prod_{t >= l} n_t
  const double* input;
  double* buf[2];
  double* partials;  // [grid][SV_NE][2]
  double* gc;        // [SV_PMAX * SV_PMAX] projection of the next pass
  double* stage;     // [d][SV_CORE] cores, C order (r, n, r')
  SvState* st;
};

// ------------------------------------------------------- double-double
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// hi + lo += a * b without rounding error in the product or the sum (Dot2,
// Ogita-Rump-Oishi): the correction lo collects both error terms.
__device__ __forceinline__ void dot2_acc(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  double s, e;
  two_sum(hi, p, s, e);
  hi = s;
  lo += e + pe;
}
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_norm(double hi, double lo) {
  const double s = hi + lo;
  return {s, lo - (s - hi)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  double s, e, t, f;
  two_sum(a.hi, b.hi, s, e);
  two_sum(a.lo, b.lo, t, f);
  e += t;
  dd r = dd_norm(s, e);
  r.lo += f;
  return dd_norm(r.hi, r.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return dd_norm(p, e);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  const dd r = dd_add(a, dd_neg(dd_mul({q1, 0.0}, b)));
  const double q2 = r.hi / b.hi;
  return dd_norm(q1, q2);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  const double x = sqrt(a.hi);
  const dd r = dd_add(a, dd_neg(dd_mul({x, 0.0}, {x, 0.0})));
  return dd_norm(x, r.hi / (2.0 * x));
}

__device__ __forceinline__ double warp_max_idx(double v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  return v;
}

// (i, j) of the upper-triangle entry e of a p x p matrix, row-major order.
__device__ __forceinline__ void tri_ij(int e, int p, int& i, int& j) {
  int row = 0, base = 0;
  while (base + (p - row) <= e) {
    base += p - row;
    ++row;
  }
  i = row;
  j = row + (e - base);
}

// Asynchronous global -> shared copy of n doubles (cp.async, 16-byte
// granules when both sides allow it); completion via cp_async_wait<N>.
__device__ __forceinline__ void async_copy(double* sdst, const double* gsrc, int n) {
  // shared-window address computed once (S2UR is slow), then offset
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sdst);
  const bool v16 = ((reinterpret_cast<uintptr_t>(gsrc) | (uintptr_t)sbase) & 15) == 0;
  if (v16) {
    const int n2 = n >> 1;
    for (int i = threadIdx.x; i < n2; i += SV_NT)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + 16u * i), "l"(gsrc + 2 * i));
    if ((n & 1) && threadIdx.x == 0)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * (n - 1)), "l"(gsrc + n - 1));
  } else {
    for (int i = threadIdx.x; i < n; i += SV_NT)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * i), "l"(gsrc + i));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------- one-sided Jacobi
// Orthogonalises the nv vectors X_v = X + v ld (length len, nv <= 64) by
// plane rotations accumulated into Acc (nv x nv, column-major, set to I):
// afterwards X_out = X_in Acc with mutually orthogonal X_out vectors.
// Brent-Luk round-robin pairs, one half-warp per pair (all pairs of a round
// at once).  Returns the number of sweeps.
__device__ int jacobi_vecs(double* X, int nv, int len, int ld, double* Acc, int* s_flag, double* s_red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hw = tid >> 4, hl = tid & 15;
  const unsigned hmask = 0xffffu << (16 * (lane >> 4));
  for (int idx = tid; idx < nv * nv; idx += SV_NT) Acc[idx] = (idx % nv == idx / nv) ? 1.0 : 0.0;
  double part = 0.0;
  for (int v = 0; v < nv; ++v)
    for (int i = tid; i < len; i += SV_NT) part = fma(X[v * ld + i], X[v * ld + i], part);
  part = warp_sum(part);
  if (lane == 0) s_red[warp] = part;
  __syncthreads();
  double fro2 = 0.0;
  for (int w = 0; w < SV_NW; ++w) fro2 += s_red[w];
  // vectors below eps ||X|| / 8 only carry rounding noise: they take no part
  // in rotations among themselves (the rank decisions never keep them)
  const double floor2 = fro2 * (1.1e-16 / 8) * (1.1e-16 / 8);
  // dgesvj-style threshold: the computed gamma of two orthogonal vectors
  // carries rounding noise ~ sqrt(len) eps sqrt(alpha beta)
  const double tol = fmax(1e-15, 2.0 * sqrt((double)len) * 1.1102230246251565e-16);
  const double tol2 = tol * tol;
  const int mm = nv + (nv & 1);
  if (mm < 2) return 0;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (tid == 0) *s_flag = 0;
    __syncthreads();
    for (int round = 0; round < mm - 1; ++round) {
      for (int pi = hw; pi < mm / 2; pi += 2 * SV_NW) {
        const int pa = pi, pb = mm - 1 - pi;
        const int p = pa == 0 ? 0 : ((round + pa - 1) % (mm - 1)) + 1;
        const int q = pb == 0 ? 0 : ((round + pb - 1) % (mm - 1)) + 1;
        if (p >= nv || q >= nv) continue;
        double* xp = X + (int64_t)p * ld;
        double* xq = X + (int64_t)q * ld;
        double al = 0.0, be = 0.0, ga = 0.0;
        double xr[4], yr[4];  // len <= 64: the pair stays in registers
        if (len <= 64) {
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const int j = hl + 16 * k2;
            xr[k2] = j < len ? xp[j] : 0.0;
            yr[k2] = j < len ? xq[j] : 0.0;
            al = fma(xr[k2], xr[k2], al);
            be = fma(yr[k2], yr[k2], be);
            ga = fma(xr[k2], yr[k2], ga);
          }
        } else {
          for (int j = hl; j < len; j += 16) {
            const double x = xp[j], y = xq[j];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          al += __shfl_xor_sync(hmask, al, o);
          be += __shfl_xor_sync(hmask, be, o);
          ga += __shfl_xor_sync(hmask, ga, o);
        }
        if (ga == 0.0 || fmin(al, be) < floor2) continue;
        if (ga * ga <= tol2 * al * be) continue;
        // rotation from the hardware reciprocal / rsqrt plus Newton steps
        // (full precision, no slow-path division or square root)
        const double zeta = (be - al) * rcp_nr(2.0 * ga);
        const double az = fabs(zeta);
        const double t = az > 1e100 ? 0.5 / zeta
                                     : copysign(1.0, zeta) * rcp_nr(az + (fma(zeta, zeta, 1.0)) * rsqrt_nr(fma(zeta, zeta, 1.0)));
        const double cs = rsqrt_nr(fma(t, t, 1.0));
        const double sn = cs * t;
        if (len <= 64) {
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const int j = hl + 16 * k2;
            if (j < len) {
              xp[j] = cs * xr[k2] - sn * yr[k2];
              xq[j] = sn * xr[k2] + cs * yr[k2];
            }
          }
        } else {
          for (int j = hl; j < len; j += 16) {
            const double x = xp[j], y = xq[j];
            xp[j] = cs * x - sn * y;
            xq[j] = sn * x + cs * y;
          }
        }
        double* up = Acc + (int64_t)p * nv;
        double* uq = Acc + (int64_t)q * nv;
        for (int j = hl; j < nv; j += 16) {
          const double x = up[j], y = uq[j];
          up[j] = cs * x - sn * y;
          uq[j] = sn * x + cs * y;
        }
        if (hl == 0) *s_flag = 1;
      }
      __syncthreads();
    }
    const int f = *s_flag;
    __syncthreads();
    if (!f) break;
  }
  return sweep + 1;
}

// --------------------------------------------------------- the superstep
// Shared-memory regions of the small phase (doubles).
constexpr int RA = 0;      // 8192: Gram hi/lo, later Pt (4096) + U (4096)
constexpr int RB = 8192;   // 4096: Cholesky factor R, later Gc (ping)
constexpr int RC = 12288;  // 4096: Gc (pong)
constexpr int RD = 16384;  // 4096: L / W (the current step matrix)
constexpr int RE = 20480;  // 2048: small vectors

__device__ void small_phase(const SvParams& P, SvState& S, double* sm, int64_t n_gram, int nparts) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pg = S.pg, kst = S.k, l0 = S.l, r_in = S.r_in, mode = S.mode, dst_sel = S.dst_sel;
  const int ne = pg * (pg + 1) / 2;
  double* Ghi = sm + RA;
  double* Glo = sm + RA + SV_PMAX * SV_PMAX;
  double* Rp = sm + RB;  // Cholesky rows, physical column order
  double* L = sm + RD;
  double* sig = sm + RE;                                  // 64
  double* rrow_hi = sm + RE + 64;                         // 64
  double* rrow_lo = sm + RE + 128;                        // 64
  double* red = sm + RE + 192;                            // 32
  int* pivoted = reinterpret_cast<int*>(sm + RE + 256);   // 64 ints
  int* order = reinterpret_cast<int*>(sm + RE + 384);     // 64 ints
  int* s_int = reinterpret_cast<int*>(sm + RE + 448);     // scratch ints
  double* s_dbl = sm + RE + 512;                          // scratch doubles
  if (tid == 0) S.clk[0] = clock64();

  // 1. Gram matrix: the partials of the CTAs that saw data, summed in a
  //    fixed order (deterministic); tpe threads per entry, then combined
  {
    const int tpe = ne <= SV_NT ? SV_NT / ne : 1;
    double* scratch = sm + RB;  // 2 * SV_NT doubles
    if (ne <= SV_NT) {
      if (tid < ne * tpe) {
        const int e = tid % ne, c = tid / ne;
        dd acc{0.0, 0.0};
        for (int b = c; b < nparts; b += tpe) {
          const double* pp = P.partials + ((int64_t)b * SV_NE + e) * 2;
          acc = dd_add(acc, {pp[0], pp[1]});
        }
        scratch[2 * tid] = acc.hi;
        scratch[2 * tid + 1] = acc.lo;
      }
      __syncthreads();
      if (tid < ne) {
        dd acc{0.0, 0.0};
        for (int c = 0; c < tpe; ++c) acc = dd_add(acc, {scratch[2 * (c * ne + tid)], scratch[2 * (c * ne + tid) + 1]});
        int i, j;
        tri_ij(tid, pg, i, j);
        Ghi[i * pg + j] = acc.hi;
        Glo[i * pg + j] = acc.lo;
        Ghi[j * pg + i] = acc.hi;
        Glo[j * pg + i] = acc.lo;
      }
    } else {
      for (int e = tid; e < ne; e += SV_NT) {
        dd acc{0.0, 0.0};
        for (int b = 0; b < nparts; ++b) {
          const double* pp = P.partials + ((int64_t)b * SV_NE + e) * 2;
          acc = dd_add(acc, {pp[0], pp[1]});
        }
        int i, j;
        tri_ij(e, pg, i, j);
        Ghi[i * pg + j] = acc.hi;
        Glo[i * pg + j] = acc.lo;
        Ghi[j * pg + i] = acc.hi;
        Glo[j * pg + i] = acc.lo;
      }
    }
  }
  if (tid < pg) pivoted[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    dd tr{0.0, 0.0};
    for (int i = 0; i < pg; ++i) tr = dd_add(tr, {Ghi[i * pg + i], Glo[i * pg + i]});
    s_dbl[0] = tr.hi;
    s_dbl[1] = tr.lo;
  }
  __syncthreads();
  const dd trace{s_dbl[0], s_dbl[1]};
  if (l0 == 0) {
    if (trace.hi <= 0.0) {  // zero vector: rank-1 zero cores (ttcore.py:231-233)
      for (int l = 0; l < P.d; ++l)
        for (int idx = tid; idx < (int)P.n[l]; idx += SV_NT) P.stage[(int64_t)l * SV_CORE + idx] = 0.0;
      if (tid == 0) {
        for (int l = 0; l <= P.d; ++l) S.ranks[l] = 1;
        S.zero = 1;
        S.mode = kDone;
      }
      return;
    }
    if (tid == 0) S.delta = P.eps_scale * dd_sqrt(trace).hi;
  }
  __syncthreads();
  const double delta = S.delta;
  if (tid == 0) S.clk[1] = clock64();

  // 2. pivoted Cholesky in double-double with the pivot order kept as an
  //    indirection: G = Pi R^T R Pi^T, Rp[t][rho] = R[t][Pi^-1 rho]
  // Stop once the energy left in the Schur complement, trace(S) = the
  // squared Frobenius norm of the remaining rows of R, is below
  // (1e-3 thr)^2 with thr the smallest threshold _chop can use here
  // (delta, or the eps_mach floor with s0^2 >= trace / pg): dropping it
  // moves every tail sum by at most 1e-3 thr (decisions change only at
  // near-ties) and shrinks the Jacobi problem to the significant rank.
  const double tol = trace.hi * 5e-32;
  const double thr_min = fmax(delta, 2.0 * 2.220446049250313e-16 * sqrt(trace.hi / pg));
  const double drop2 = (1e-3 * thr_min) * (1e-3 * thr_min);
  int b = 0;
  for (int j = 0; j < pg; ++j) {
    if (warp == 0) {
      double best = -1.0;
      int bi = pg;
      double rem = 0.0;  // remaining trace (a stopping test: FP64 is enough)
      for (int i = lane; i < pg; i += 32) {
        const double v = pivoted[i] ? -1.0 : Ghi[i * pg + i];
        if (!pivoted[i]) rem += Ghi[i * pg + i];
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      rem = warp_sum(rem);
      best = warp_max_idx(best, bi);
      if (lane == 0) {
        s_int[0] = bi;
        s_dbl[2] = best;
        s_dbl[3] = rem;
      }
    }
    __syncthreads();
    if (!(s_dbl[2] > tol) || s_dbl[3] <= drop2) break;  // uniform
    const int pj = s_int[0];
    const dd rjj = dd_sqrt({Ghi[pj * pg + pj], Glo[pj * pg + pj]});
    for (int rho = tid; rho < pg; rho += SV_NT) {
      dd v{0.0, 0.0};
      if (rho == pj) v = rjj;
      else if (!pivoted[rho]) v = dd_div({Ghi[pj * pg + rho], Glo[pj * pg + rho]}, rjj);
      rrow_hi[rho] = v.hi;
      rrow_lo[rho] = v.lo;
      Rp[j * pg + rho] = v.hi;
    }
    if (tid == 0) pivoted[pj] = 1;
    __syncthreads();
    for (int c1 = warp; c1 < pg; c1 += SV_NW) {
      if (pivoted[c1]) continue;
      const dd a1{rrow_hi[c1], rrow_lo[c1]};
      for (int c2 = lane; c2 < pg; c2 += 32) {
        if (pivoted[c2]) continue;
        const dd prod = dd_mul(a1, {rrow_hi[c2], rrow_lo[c2]});
        const dd g = dd_add({Ghi[c1 * pg + c2], Glo[c1 * pg + c2]}, dd_neg(prod));
        Ghi[c1 * pg + c2] = g.hi;
        Glo[c1 * pg + c2] = g.lo;
      }
    }
    __syncthreads();
    b = j + 1;
  }
  const int bdone = b;
  if (b == 0) b = 1;  // all-zero data: one zero column keeps the shapes valid
  // L (pg x b, column-major): L L^T = G
  for (int idx = tid; idx < pg * b; idx += SV_NT) {
    const int rho = idx % pg, t = idx / pg;
    L[idx] = t < bdone ? Rp[t * pg + rho] : 0.0;
  }
  __syncthreads();
  if (tid == 0) S.clk[2] = clock64();

  // 3. the k step SVDs of the superstep
  double* W = L;  // current step matrix, column-major (rowsW x b)
  double* X = sm + RA;             // Jacobi vectors (<= 4096)
  double* Acc = sm + RA + SV_CORE; // rotations (<= 4096)
  double* gc_cur = sm + RB;
  double* gc_nxt = sm + RC;
  int r_prev = r_in;
  int rowsW = pg;
  int rows_gc = r_in;  // gc_cur is (rows_gc x r_prev); identity before step 0
  for (int s = 0; s < kst; ++s) {
    const int ls = l0 + s;
    const int n = (int)P.n[ls];
    const int m = r_prev * n;
    const int c = (rowsW / m) * b;
    // P_s = W viewed column-major m x c.  c <= m: one-sided Jacobi on its
    // columns (the Cholesky factor's rows: graded, converges in a few
    // sweeps); else on its rows.
    const bool cols = c <= m;
    if (cols) {
      for (int idx = tid; idx < m * c; idx += SV_NT) X[idx] = W[idx];
    } else {
      for (int idx = tid; idx < m * c; idx += SV_NT) X[idx] = W[(idx / c) + (int64_t)m * (idx % c)];
    }
    __syncthreads();
    const int nv = cols ? c : m, len = cols ? m : c;
    const int nsw = jacobi_vecs(X, nv, len, len, Acc, s_int + 2, red);
    if (tid == 0) S.sweeps[ls] = nsw;
    for (int v = tid; v < nv; v += SV_NT) {
      double acc = 0.0;
      for (int j = 0; j < len; ++j) acc = fma(X[v * len + j], X[v * len + j], acc);
      sig[v] = sqrt(acc);
    }
    __syncthreads();
    for (int v = tid; v < nv; v += SV_NT) {
      int pos = 0;
      for (int j2 = 0; j2 < nv; ++j2) pos += (sig[j2] > sig[v]) || (sig[j2] == sig[v] && j2 < v);
      order[pos] = v;
    }
    __syncthreads();
    if (tid == 0) {  // _chop over the len = min(rows, cols) singular values
      const int64_t cols_total = P.rest[ls + 1];
      const int lenc = (int)min((int64_t)min(m, nv), cols_total);
      const double s0 = sig[order[0]];
      const double thr = fmax(delta, s0 * (double)max((int)min((int64_t)m, cols_total), 2) * 2.220446049250313e-16);
      int r = 1;
      double tail2 = 0.0;
      for (int kk = lenc - 1; kk >= 0; --kk) {
        const double sv = sig[order[kk]];
        tail2 += sv * sv;
        if (sqrt(tail2) > thr) {
          r = kk + 1;
          break;
        }
      }
      s_int[1] = r;
      S.ranks[ls + 1] = r;
    }
    __syncthreads();
    const int r = s_int[1];
    // u(:, b') -- column b' of the kept left singular basis (m entries)
    auto u_at = [&](int row, int bq) -> double {
      const int v = order[bq];
      if (cols) {
        const double sv = sig[v];
        return sv > 0.0 ? X[(int64_t)v * m + row] / sv : (row == bq ? 1.0 : 0.0);
      }
      return Acc[(int64_t)v * m + row];
    };
    // core (r_prev, n, r), C order: core[a, i, b'] = u[a + r_prev i, b']
    double* core = P.stage + (int64_t)ls * SV_CORE;
    for (int idx = tid; idx < m * r; idx += SV_NT) {
      const int bq = idx % r, ai = idx / r;  // ai = a * n + i
      const int a = ai / n, i = ai % n;
      core[idx] = u_at(a + r_prev * i, bq);
    }
    // next step matrix W' = U_keep^T P_s (r x c, column-major)
    if (s + 1 < kst) {
      for (int idx = tid; idx < r * c; idx += SV_NT) {
        const int bq = idx % r, jcol = idx / r;
        const int v = order[bq];
        W[idx] = cols ? sig[v] * Acc[(int64_t)v * c + jcol] : X[(int64_t)v * c + jcol];
      }
    }
    // composite basis: gc_nxt[rho + rows_gc i, b'] = sum_b gc_cur[rho, b] u[b + r_prev i, b']
    const int rows_nxt = rows_gc * n;
    for (int idx = tid; idx < rows_nxt * r; idx += SV_NT) {
      const int row = idx % rows_nxt, bq = idx / rows_nxt;
      const int rho = row % rows_gc, i = row / rows_gc;
      double acc;
      if (s == 0) {
        acc = u_at(rho + r_prev * i, bq);  // gc_cur = identity (rows_gc == r_prev)
      } else {
        acc = 0.0;
        for (int bb = 0; bb < r_prev; ++bb) acc = fma(gc_cur[rho + (int64_t)rows_gc * bb], u_at(bb + r_prev * i, bq), acc);
      }
      gc_nxt[idx] = acc;
    }
    __syncthreads();
    double* tmp = gc_cur;
    gc_cur = gc_nxt;
    gc_nxt = tmp;
    rows_gc = rows_nxt;
    rowsW = r * (rowsW / m);
    r_prev = r;
  }
  if (tid == 0) S.clk[3] = clock64();
  // 4. projection for the next pass and the next superstep's parameters
  for (int idx = tid; idx < rows_gc * r_prev; idx += SV_NT) P.gc[idx] = gc_cur[idx];
  __syncthreads();
  if (tid == 0) {
    const int l2 = l0 + kst;
    S.src_sel = mode == kGramInput ? 0 : dst_sel;
    S.dst_sel = S.src_sel == 1 ? 2 : 1;
    S.p_src = pg;
    S.n_src = n_gram;
    S.r_in = r_prev;
    S.l = l2;
    S.k = 0;
    S.gsz = 1;
    S.pg = r_prev;
    if (l2 >= P.d - 1) {
      S.mode = kProjectOnly;  // the carry is the last core
    } else if ((int64_t)r_prev * P.n[l2] > SV_PMAX) {
      S.mode = kProjectOnly;  // hand the carry to the per-step path
      S.handoff = 1;
    } else {
      // one step per superstep: P_0 is then the (graded) Cholesky factor
      S.mode = kProjectGram;
      S.k = 1;
      S.pg = (int)(r_prev * P.n[l2]);
      S.gsz = (int)P.n[l2];
    }
  }
  (void)lane;
}

__global__ void __launch_bounds__(SV_NT, 1) ttsvd_step_kernel(const SvParams P) {
  extern __shared__ double sm[];
  __shared__ SvState S;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  if (tid == 0) S = *P.st;
  __syncthreads();
  if (S.mode == kDone) return;
  const double* src = S.src_sel == 0 ? P.input : P.buf[S.src_sel - 1];
  const int mode = S.mode;
  const int p_src = S.p_src;
  const int r_out = S.r_in;
  const int64_t n_src = S.n_src;
  const bool project = mode != kGramInput;
  const int pg = mode == kProjectOnly ? r_out : S.pg;
  const int gsz = project ? S.gsz : 1;
  const int64_t n_gram = n_src / gsz;
  double* dst = project ? P.buf[S.dst_sel - 1] : nullptr;

  // tiles: TG Gram columns = TG * gsz source columns, double-buffered
  int TG = project ? SV_TILE / (gsz * max(p_src, r_out)) : SV_TILE / pg;
  TG = max(TG, 1);
  double* tiles[2] = {sm, sm + SV_TILE};  // source columns (cp.async ring)
  double* ctile = sm + 2 * SV_TILE;       // projected carry columns
  double* gcs = sm + 3 * SV_TILE;         // SV_PMAX^2: projection
  if (project) {
    for (int idx = tid; idx < p_src * r_out; idx += SV_NT) gcs[idx] = P.gc[idx];
  }
  // Gram entry ownership: ne <= SV_NT -> one entry per thread, SV_NT / ne
  // column groups; otherwise one group, entries tid, tid + SV_NT, ...
  const int ne = pg * (pg + 1) / 2;
  const bool gram = mode != kProjectOnly;
  int groups = 1, my_g = 0;
  if (ne <= SV_NT) {
    groups = SV_NT / ne;
    my_g = tid / ne;
  }
  const bool active = gram && my_g < groups;
  int ei[SV_EPT], ej[SV_EPT];
  double hi[SV_EPT], lo[SV_EPT];
  int nmine = 0;
#pragma unroll
  for (int q = 0; q < SV_EPT; ++q) {
    hi[q] = 0.0;
    lo[q] = 0.0;
    ei[q] = 0;
    ej[q] = 0;
    const int e = ne <= SV_NT ? (q == 0 ? tid % ne : ne) : tid + q * SV_NT;
    if (active && e < ne) {
      tri_ij(e, pg, ei[q], ej[q]);
      nmine = q + 1;
    }
  }
  __syncthreads();
  const int64_t ntiles = (n_gram + TG - 1) / TG;
  const int64_t src_cols_per_tile = (int64_t)TG * gsz;
  auto issue = [&](int64_t t, double* buf) {
    const int64_t g0 = t * TG;
    const int tg = (int)min((int64_t)TG, n_gram - g0);
    async_copy(buf, src + g0 * gsz * (int64_t)p_src, tg * gsz * p_src);
  };
  int cur = 0;
  if ((int64_t)blockIdx.x < ntiles) issue(blockIdx.x, tiles[0]);
  cp_async_commit();
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) issue(tn, tiles[cur ^ 1]);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double* tile = tiles[cur];
    const int64_t g0 = t * TG;
    const int tg = (int)min((int64_t)TG, n_gram - g0);
    const double* col0 = tile;  // Gram columns of this tile (pg rows each)
    if (project) {
      const int ns = tg * gsz;  // source columns
      // work item = (source column, chunk of 8 outputs): the 8 outputs stay
      // in registers; row i is visited in the rotated order (i + jc) mod
      // p_src so the lanes of a warp hit different shared-memory banks
      const int nchunk = (r_out + 7) >> 3;
      for (int it = tid; it < ns * nchunk; it += SV_NT) {
        const int jc = it / nchunk, b0 = (it % nchunk) * 8;
        const double* x = tile + (int64_t)jc * p_src;
        double acc[8];
#pragma unroll
        for (int bq = 0; bq < 8; ++bq) acc[bq] = 0.0;
        int i = jc % p_src;
        for (int k2 = 0; k2 < p_src; ++k2) {
          const double xi = x[i];
#pragma unroll
          for (int bq = 0; bq < 8; ++bq)
            if (b0 + bq < r_out) acc[bq] = fma(gcs[(b0 + bq) * p_src + i], xi, acc[bq]);
          i = i + 1 == p_src ? 0 : i + 1;
        }
#pragma unroll
        for (int bq = 0; bq < 8; ++bq)
          if (b0 + bq < r_out) ctile[jc * r_out + b0 + bq] = acc[bq];
      }
      __syncthreads();
      double* gdst = dst + g0 * gsz * (int64_t)r_out;
      for (int idx = tid; idx < ns * r_out; idx += SV_NT) gdst[idx] = ctile[idx];
      col0 = ctile;
    }
    if (active) {
      if (ne <= SV_NT) {
        // one entry per thread: SV_EPT interleaved column streams keep the
        // dependent double-double chains independent (latency, not FP64
        // throughput, bounds a single chain)
        const int i0 = ei[0], j0 = ej[0];
        int jc = my_g;
        for (; jc + (SV_EPT - 1) * groups < tg; jc += SV_EPT * groups) {
#pragma unroll
          for (int q = 0; q < SV_EPT; ++q) {
            const double* y = col0 + (int64_t)(jc + q * groups) * pg;
            dot2_acc(hi[q], lo[q], y[i0], y[j0]);
          }
        }
        for (; jc < tg; jc += groups) {
          const double* y = col0 + (int64_t)jc * pg;
          dot2_acc(hi[0], lo[0], y[i0], y[j0]);
        }
      } else {
        for (int jc = 0; jc < tg; ++jc) {
          const double* y = col0 + (int64_t)jc * pg;
#pragma unroll
          for (int q = 0; q < SV_EPT; ++q)
            if (q < nmine) dot2_acc(hi[q], lo[q], y[ei[q]], y[ej[q]]);
        }
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  cp_async_wait<0>();
  (void)src_cols_per_tile;
  if (gram) {
    // CTA partial: groups summed in a fixed order
    double* red = sm;  // 2 * SV_NT doubles (the tiles are no longer needed)
    if (ne <= SV_NT) {
      if (active) {
        dd acc = dd_norm(hi[0], lo[0]);
#pragma unroll
        for (int q = 1; q < SV_EPT; ++q) acc = dd_add(acc, dd_norm(hi[q], lo[q]));
        red[2 * tid] = acc.hi;
        red[2 * tid + 1] = acc.lo;
      }
      __syncthreads();
      if (tid < ne) {
        dd acc{0.0, 0.0};
        for (int g = 0; g < groups; ++g) acc = dd_add(acc, {red[2 * (g * ne + tid)], red[2 * (g * ne + tid) + 1]});
        double* pp = P.partials + ((int64_t)blockIdx.x * SV_NE + tid) * 2;
        pp[0] = acc.hi;
        pp[1] = acc.lo;
      }
    } else {
#pragma unroll
      for (int q = 0; q < SV_EPT; ++q) {
        const int e = tid + q * SV_NT;
        if (q < nmine && e < ne) {
          const dd v = dd_norm(hi[q], lo[q]);
          double* pp = P.partials + ((int64_t)blockIdx.x * SV_NE + e) * 2;
          pp[0] = v.hi;
          pp[1] = v.lo;
        }
      }
    }
  }
  // last CTA to finish runs the small phase
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&P.st->counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (mode == kProjectOnly) {
    if (!S.handoff) {  // the projected carry (r x n_{d-1}) is the last core (r, n, 1)
      const int nl = (int)P.n[P.d - 1];
      double* core = P.stage + (int64_t)(P.d - 1) * SV_CORE;
      for (int idx = tid; idx < r_out * nl; idx += SV_NT) {
        const int a = idx / nl, i = idx % nl;
        core[idx] = dst[a + (int64_t)r_out * i];
      }
    }
    if (tid == 0) {
      S.mode = kDone;
      S.counter = 0;
      *P.st = S;
    }
    return;
  }
  small_phase(P, S, sm, n_gram, (int)min((int64_t)gridDim.x, ntiles));
  __syncthreads();
  if (tid == 0) {
    S.counter = 0;
    *P.st = S;
  }
}

__global__ void ttsvd_pack_kernel(int d, const double* __restrict__ stage, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ len, double* __restrict__ out) {
  for (int l = blockIdx.y; l < d; l += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len[l];
         i += (int64_t)gridDim.x * blockDim.x)
      out[off[l] + i] = stage[(int64_t)l * SV_CORE + i];
}

}  // namespace

// Result of the device supersteps: done (all cores staged) or a handoff at
// step `l` with the carry (r x rest) in `carry`.
struct TtsvdFast {
  bool done = false, zero = false;
  int l = 0, r = 1;
  std::vector<int> ranks;
  double* stage = nullptr;   // [d][SV_CORE]
  double* carry = nullptr;   // handoff carry (column-major r x rest)
  double* owned[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t s = nullptr;
  void release() {
    for (auto& p : owned)
      if (p) cudaFreeAsync(p, s), p = nullptr;
  }
};

int ttsvd_fast(cudaStream_t s, const double* dense, int d, const int64_t* sizes, double eps,
               TtsvdFast& res) {
  res.s = s;
  if (d < 2 || d > QTT_MAX_CORES) return kUnsupported;
  if (getenv("QTT_TTSVD_LEGACY")) return kUnsupported;
  int64_t total = 1;
  for (int l = 0; l < d; ++l) total *= sizes[l];
  // first superstep: r_in = 1, as many steps as fit in SV_P0 rows
  int k0 = 0;
  int64_t p0 = 1;
  while (k0 < d - 1 && p0 * sizes[k0] <= SV_P0) p0 *= sizes[k0++];
  if (k0 == 0) return kUnsupported;
  static DeviceFlag configured;
  if (!configured.test()) {
    QTT_CUDA(cudaFuncSetAttribute(ttsvd_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  SV_SMEM_DBL * (int)sizeof(double)));
    configured.set();
  }
  const int grid = num_sms();
  SvParams P{};
  P.d = d;
  P.eps_scale = eps / std::sqrt((double)std::max(d - 1, 1));
  for (int l = 0; l < d; ++l) P.n[l] = sizes[l];
  P.rest[d] = 1;
  for (int l = d - 1; l >= 0; --l) P.rest[l] = P.rest[l + 1] * sizes[l];
  P.input = dense;
  // carry buffers: every projected carry has at most `total` entries
  QTT_CUDA(malloc_async(&res.owned[0], sizeof(double) * total, s));
  QTT_CUDA(malloc_async(&res.owned[1], sizeof(double) * total, s));
  const size_t small = (size_t)grid * SV_NE * 2 + SV_PMAX * SV_PMAX + (size_t)d * SV_CORE;
  QTT_CUDA(malloc_async(&res.owned[2], sizeof(double) * small, s));
  QTT_CUDA(malloc_async(&res.owned[3], sizeof(SvState), s));
  P.buf[0] = res.owned[0];
  P.buf[1] = res.owned[1];
  P.partials = res.owned[2];
  P.gc = P.partials + (size_t)grid * SV_NE * 2;
  P.stage = P.gc + SV_PMAX * SV_PMAX;
  P.st = reinterpret_cast<SvState*>(res.owned[3]);
  res.stage = P.stage;
  SvState st{};
  st.mode = kGramInput;
  st.l = 0;
  st.k = k0;
  st.r_in = 1;
  st.pg = (int)p0;
  st.gsz = 1;
  st.p_src = (int)p0;
  st.src_sel = 0;
  st.dst_sel = 1;
  st.n_src = total / p0;
  st.ranks[0] = 1;
  st.ranks[d] = 1;
  thread_local SvState* host_st = nullptr;
  if (!host_st) QTT_CUDA(cudaMallocHost(&host_st, sizeof(SvState)));
  *host_st = st;
  QTT_CUDA(cudaMemcpyAsync(P.st, host_st, sizeof(SvState), cudaMemcpyHostToDevice, s));
  const size_t smem = SV_SMEM_DBL * sizeof(double);
  // queue supersteps in batches; each launch reads its parameters from the
  // device state (no host round trip between supersteps)
  static const bool dbg = getenv("QTT_TTSVD_DEBUG") != nullptr;
  for (int launched = 0; launched < 2 * d + 2;) {
    const int batch = dbg ? 1 : (launched == 0 ? 4 : 3);
    for (int b = 0; b < batch; ++b, ++launched) {
      ttsvd_step_kernel<<<grid, SV_NT, smem, s>>>(P);
      QTT_CHECK_LAUNCH();
    }
    QTT_CUDA(cudaMemcpyAsync(host_st, P.st, sizeof(SvState), cudaMemcpyDeviceToHost, s));
    QTT_CUDA(cudaStreamSynchronize(s));
    if (dbg) {
      const SvState& h = *host_st;
      fprintf(stderr, "[ttsvd] after launch %d: mode %d l %d k %d r_in %d pg %d n_src %lld | reduce %lld chol %lld "
              "steps %lld cyc | sweeps", launched, h.mode, h.l, h.k, h.r_in, h.pg, h.n_src, h.clk[1] - h.clk[0],
              h.clk[2] - h.clk[1], h.clk[3] - h.clk[2]);
      for (int l = 0; l < d; ++l) fprintf(stderr, " %d", h.sweeps[l]);
      fprintf(stderr, "\n");
    }
    if (host_st->mode == kDone) break;
  }
  const SvState& fin = *host_st;
  if (fin.mode != kDone) return kCuda;
  res.zero = fin.zero != 0;
  res.ranks.assign(fin.ranks, fin.ranks + d + 1);
  res.ranks[0] = 1;
  if (fin.handoff) {
    res.done = false;
    res.l = fin.l;
    res.r = fin.r_in;
    res.carry = P.buf[fin.dst_sel - 1];
  } else {
    res.done = true;
    res.ranks[d] = 1;
  }
  return kOk;
}

int ttsvd_pack(cudaStream_t s, int d, const double* stage, const qtt_layout* out, double* out_data) {
  std::vector<int64_t> hv(2 * d);
  for (int l = 0; l < d; ++l) {
    hv[l] = out->offsets[l];
    hv[d + l] = out->ranks[l] * out->rows[l] * out->ranks[l + 1];
  }
  int64_t* dv = nullptr;
  QTT_CUDA(malloc_async(&dv, sizeof(int64_t) * 2 * d, s));
  QTT_CUDA(cudaMemcpyAsync(dv, hv.data(), sizeof(int64_t) * 2 * d, cudaMemcpyHostToDevice, s));
  ttsvd_pack_kernel<<<dim3(8, std::min(d, 64)), 256, 0, s>>>(d, stage, dv, dv + d, out_data);
  QTT_CHECK_LAUNCH();
  QTT_CUDA(cudaFreeAsync(dv, s));
  return kOk;
}

}  // namespace qtt
