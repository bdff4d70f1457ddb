// Core-wise TT products and structural TT algebra (rows a2-a4, a7, a8).
//
// qtt_matvec / qtt_matmat / qtt_hadamard run ALL d cores in one launch:
// the output cores are cut into 4096-element units, a block per unit, and
// every thread streams 16-byte stores (st.global.cs) over consecutive
// element pairs of its unit.  Inputs are tiny next to the outputs (the
// output rank is the product of input ranks) and stay in L1/L2; the kernel
// is bound by HBM write bandwidth (~0.5 flop/B).
#include "common.cuh"
#include "../../include/qtt_b200.h"

namespace qtt {
namespace {


constexpr int kProdThreads = 256;

struct ProdCore {
  int64_t a_off, b_off, c_off;
  int ra0, ra1, rb0, rb1;  // ranks of the two operands
  int n, m, k;             // out rows n, contracted m, out cols k (1 = vector)
  int mode;                // 0: sum over j (product), 1: hadamard (no sum)
  int64_t unit_begin;
};

struct ProdDesc {
  int ncores;
  int64_t total_units;
  ProdCore c[QTT_MAX_CORES];
};

__device__ __forceinline__ void st_cs2(double* p, double x, double y) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
}

// Slab-structured product.  For fixed (c, i, kk) the output entries
// y[(a,c), i, kk, (b,e)] = sum_j A[a,i,j,b] B[c,j,kk,e] form a "slab" of
// ra0 rows.  One block per slab: the A slice A[:, i, :, :] is staged once in
// shared memory (broadcast reads), every thread keeps its column pair
// B[c, :, kk, e:e+2] in registers for the whole slab and loops over (a, b):
// 2m FMAs and one 16-byte streaming store per iteration, no per-element
// index arithmetic.  (mode 1 = hadamard: no j sum, B indexed by i.)
constexpr int kSlabA = 4096;  // doubles of the staged A slice (32 KB)

__global__ void __launch_bounds__(kProdThreads) core_product_kernel(const __grid_constant__ ProdDesc desc,
                                                                     const double* __restrict__ A,
                                                                     const double* __restrict__ B,
                                                                     double* __restrict__ C) {
  __shared__ double As[kSlabA];
  for (int64_t u = blockIdx.x; u < desc.total_units; u += gridDim.x) {
    int ci = 0;
    while (ci + 1 < desc.ncores && desc.c[ci + 1].unit_begin <= u) ++ci;
    const ProdCore& pc = desc.c[ci];
    const int rb1 = pc.rb1, ra1 = pc.ra1, ra0 = pc.ra0;
    const int m = pc.mode == 1 ? 1 : pc.m;
    const int64_t slab = u - pc.unit_begin;  // (c, i, kk)
    const int kk = (int)(slab % pc.k);
    const int i = (int)((slab / pc.k) % pc.n);
    const int cc = (int)(slab / ((int64_t)pc.k * pc.n));
    const int64_t Q = (int64_t)ra1 * rb1;
    const double* a = A + pc.a_off;
    const double* bb = B + pc.b_off;
    double* c = C + pc.c_off;
    // stage A[:, i, :, :] as As[(aa * m + j) * ra1 + b]
    const int aslice = ra0 * m * ra1;
    const bool staged = aslice <= kSlabA;
    __syncthreads();
    if (staged) {
      for (int t = threadIdx.x; t < aslice; t += kProdThreads) {
        const int bq = t % ra1, rest = t / ra1, j = rest % m, aa = rest / m;
        As[t] = pc.mode == 1 ? a[((int64_t)aa * pc.n + i) * ra1 + bq]
                             : a[(((int64_t)aa * pc.n + i) * pc.m + j) * ra1 + bq];
      }
    }
    __syncthreads();
    const int ep_count = (rb1 + 1) / 2;
    const int ep_lanes = min(ep_count, kProdThreads);
    const int b_lanes = kProdThreads / ep_lanes;
    const int tid = threadIdx.x;
    if (tid >= ep_lanes * b_lanes) continue;
    const int ep0 = tid % ep_lanes, bl = tid / ep_lanes;
    const bool aligned = ((rb1 & 1) == 0) && ((pc.c_off & 1) == 0);
    for (int ep = ep0; ep < ep_count; ep += ep_lanes) {
      const int e = 2 * ep;
      const bool two = e + 1 < rb1;
      double x0[4], x1[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x0[j] = x1[j] = 0.0;
        if (j < m) {
          const double* bp = pc.mode == 1 ? bb + ((int64_t)cc * pc.n + i) * rb1 + e
                                          : bb + (((int64_t)cc * pc.m + j) * pc.k + kk) * rb1 + e;
          x0[j] = __ldg(bp);
          x1[j] = two ? __ldg(bp + 1) : 0.0;
        }
      }
      for (int aa = 0; aa < ra0; ++aa) {
        const int64_t row = (((int64_t)aa * pc.rb0 + cc) * pc.n + i) * pc.k + kk;
        double* crow = c + row * Q + e;
        for (int b = bl; b < ra1; b += b_lanes) {
          double y0 = 0.0, y1 = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (j < m) {
              const double av = staged ? As[(aa * m + j) * ra1 + b]
                                       : (pc.mode == 1 ? __ldg(a + ((int64_t)aa * pc.n + i) * ra1 + b)
                                                       : __ldg(a + (((int64_t)aa * pc.n + i) * pc.m + j) * ra1 + b));
              y0 = fma(av, x0[j], y0);
              y1 = fma(av, x1[j], y1);
            }
          }
          double* dst = crow + (int64_t)b * rb1;
          if (aligned && two) {
            st_cs2(dst, y0, y1);
          } else {
            dst[0] = y0;
            if (two) dst[1] = y1;
          }
        }
      }
    }
  }
}

int launch_product(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b,
                   const qtt_layout* LC, double* c, int mode, cudaStream_t s) {
  const int d = LA->d;
  if (d < 1 || d > QTT_MAX_CORES || LB->d != d || LC->d != d) return kInvalid;
  ProdDesc desc;
  desc.ncores = d;
  int64_t units = 0;
  for (int l = 0; l < d; ++l) {
    ProdCore& pc = desc.c[l];
    pc.a_off = LA->offsets[l];
    pc.b_off = LB->offsets[l];
    pc.c_off = LC->offsets[l];
    pc.ra0 = (int)LA->ranks[l];
    pc.ra1 = (int)LA->ranks[l + 1];
    pc.rb0 = (int)LB->ranks[l];
    pc.rb1 = (int)LB->ranks[l + 1];
    pc.mode = mode;
    if (mode == 1) {
      pc.n = (int)(LA->rows[l] * LA->cols[l]);
      pc.m = 1;
      pc.k = 1;
    } else {
      pc.n = (int)LA->rows[l];
      pc.m = (int)LA->cols[l];
      pc.k = LB->is_matrix ? (int)LB->cols[l] : 1;
      if (LB->rows[l] != pc.m) return kInvalid;
      if (pc.m > 4) return kUnsupported;
    }
    if (LC->ranks[l] != (int64_t)pc.ra0 * pc.rb0 || LC->ranks[l + 1] != (int64_t)pc.ra1 * pc.rb1)
      return kInvalid;
    pc.unit_begin = units;
    units += (int64_t)pc.rb0 * pc.n * pc.k;  // one block per (c, i, kk) slab
  }
  desc.total_units = units;
  if (units == 0) return kOk;
  const int grid = (int)std::min<int64_t>(units, (int64_t)num_sms() * 32);
  core_product_kernel<<<grid, kProdThreads, 0, s>>>(desc, a, b, c);
  QTT_CHECK_LAUNCH();
  return kOk;
}

// ------------------------------------------------------------ structural ops
// One descriptor per output core; the kernel gathers every output element.
enum StructOp : int { kOpAdd = 0, kOpZFast = 1, kOpZSlow = 2, kOpDiag = 3, kOpTrans = 4, kOpCopy = 5 };

struct StructCore {
  int op;
  int64_t out_off, x_off, y_off;
  int out_r0, out_n, out_r1;  // output as order-3 (merged modes)
  int xr0, xn, xr1;           // first operand (merged order-3 view)
  int yr0, yr1;               // second operand ranks (add)
  int aux;                    // zkron: identity size; diag/trans: row mode n
  int aux2;                   // trans: col mode m
  double sx, sy;              // scalings
  int64_t begin;              // prefix of output elements
};

struct StructDesc {
  int ncores;
  int64_t total;
  StructCore c[QTT_MAX_CORES * 2];
};

__global__ void struct_kernel(const __grid_constant__ StructDesc desc, const double* __restrict__ X,
                              const double* __restrict__ Y, double* __restrict__ O) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < desc.total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int ci = 0;
    while (ci + 1 < desc.ncores && desc.c[ci + 1].begin <= g) ++ci;
    const StructCore& sc = desc.c[ci];
    const int64_t f = g - sc.begin;
    const int q = (int)(f % sc.out_r1);
    const int64_t t = f / sc.out_r1;
    const int i = (int)(t % sc.out_n);
    const int p = (int)(t / sc.out_n);
    double v = 0.0;
    switch (sc.op) {
      case kOpAdd: {
        // block-diagonal: x in [0:xr0, :, 0:xr1], y in [x0:, :, x1:]
        const bool first = sc.out_r0 == 1 && sc.xr0 == 1 && sc.yr0 == 1;
        const bool last = sc.out_r1 == 1 && sc.xr1 == 1 && sc.yr1 == 1;
        const int o0 = first ? 0 : sc.xr0;
        const int o1 = last ? 0 : sc.xr1;
        if (p < sc.xr0 && q < sc.xr1)
          v += sc.sx * X[sc.x_off + ((int64_t)p * sc.xn + i) * sc.xr1 + q];
        if (p >= o0 && p < o0 + sc.yr0 && q >= o1 && q < o1 + sc.yr1)
          v += sc.sy * Y[sc.y_off + ((int64_t)(p - o0) * sc.xn + i) * sc.yr1 + (q - o1)];
        break;
      }
      case kOpZFast: {
        // out[(b*I + a), n, (c*I + a')] = delta(a,a') * S[b, n, c]
        const int I = sc.aux;
        const int b = p / I, a = p % I, c = q / I, a2 = q % I;
        if (a == a2) v = sc.sx * X[sc.x_off + ((int64_t)b * sc.xn + i) * sc.xr1 + c];
        break;
      }
      case kOpZSlow: {
        // out[(c*R0 + a), n, (c'*R1 + b)] = delta(c,c') * S[a, n, b]
        const int R0 = sc.xr0, R1 = sc.xr1;
        const int c = p / R0, a = p % R0, c2 = q / R1, b = q % R1;
        if (c == c2) v = sc.sx * X[sc.x_off + ((int64_t)a * sc.xn + i) * sc.xr1 + b];
        break;
      }
      case kOpDiag: {
        // out (r0, n, n, r1) merged as i_out = ii*n + jj (row-major (n, n))
        const int n = sc.aux;
        const int ii = i / n, jj = i % n;
        if (ii == jj) v = sc.sx * X[sc.x_off + ((int64_t)p * sc.xn + ii) * sc.xr1 + q];
        break;
      }
      case kOpTrans: {
        // out (r0, m, n, r1) from x (r0, n, m, r1)
        const int n = sc.aux, m = sc.aux2;
        const int jo = i / n, io = i % n;  // out row mode index jo (m), col io (n)
        v = sc.sx * X[sc.x_off + ((int64_t)p * sc.xn + (io * m + jo)) * sc.xr1 + q];
        break;
      }
      default: {  // copy with scale
        v = sc.sx * X[sc.x_off + f];
      }
    }
    O[sc.out_off + f] = v;
  }
}

int launch_struct(StructDesc& desc, const double* x, const double* y, double* o, cudaStream_t s) {
  int64_t tot = 0;
  for (int l = 0; l < desc.ncores; ++l) {
    desc.c[l].begin = tot;
    tot += (int64_t)desc.c[l].out_r0 * desc.c[l].out_n * desc.c[l].out_r1;
  }
  desc.total = tot;
  if (tot == 0) return kOk;
  const int grid = (int)std::min<int64_t>(ceil_div(tot, 256), (int64_t)num_sms() * 16);
  struct_kernel<<<grid, 256, 0, s>>>(desc, x, y ? y : x, o);
  QTT_CHECK_LAUNCH();
  return kOk;
}

inline int64_t merged_n(const qtt_layout* L, int l) { return L->rows[l] * L->cols[l]; }

// ----------------------------------------------------------- norm / dot
// Gram sweep for <a, b>, core by core with GEMMs (ttcore.py:355-363):
//   G_{l+1}[c, d] = sum_{a, b, n} G_l[a, b] A_l[a, n, c] B_l[b, n, d]
int gram_dot(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b,
             double* result, cudaStream_t s) {
  const int d = LA->d;
  int64_t maxr = 1, maxtmp = 1;
  for (int l = 0; l <= d; ++l) maxr = std::max(maxr, LA->ranks[l] * LB->ranks[l]);
  for (int l = 0; l < d; ++l)
    maxtmp = std::max(maxtmp, LA->ranks[l] * merged_n(LB, l) * LB->ranks[l + 1]);
  double *G = nullptr, *T = nullptr;
  QTT_CUDA(malloc_async(&G, sizeof(double) * (maxr + 1), s));
  QTT_CUDA(malloc_async(&T, sizeof(double) * maxtmp, s));
  QTT_TRY(fill(s, G, 1, 1.0));
  for (int l = 0; l < d; ++l) {
    const int ra0 = (int)LA->ranks[l], ra1 = (int)LA->ranks[l + 1];
    const int rb0 = (int)LB->ranks[l], rb1 = (int)LB->ranks[l + 1];
    const int n = (int)merged_n(LA, l);
    // G is (ra0 x rb0) column-major with G[a + ra0*b].  B_l viewed column-major
    // as (n*rb1 x rb0): T (ra0 x n*rb1) = G * B^T  -> T[a, (n, d)]
    QTT_TRY(dgemm(s, 0, 1, ra0, n * rb1, rb0, 1.0, G, ra0, b + LB->offsets[l], (int64_t)n * rb1,
                  0.0, T, ra0));
    // G'(ra1 x rb1) = sum_i A_i^T T_i with A_i = A[:, i, :] (column-major
    // (ra1 x ra0) at offset i*ra1, ld n*ra1) and T_i = T[:, i*rb1:(i+1)*rb1].
    for (int i = 0; i < n; ++i)
      QTT_TRY(dgemm(s, 0, 0, ra1, rb1, ra0, 1.0, a + LA->offsets[l] + (int64_t)i * ra1,
                    (int64_t)n * ra1, T + (int64_t)ra0 * i * rb1, ra0, i == 0 ? 0.0 : 1.0, G,
                    ra1));
  }
  double host = 0.0;
  QTT_CUDA(cudaMemcpyAsync(&host, G, sizeof(double), cudaMemcpyDeviceToHost, s));
  QTT_CUDA(cudaFreeAsync(G, s));
  QTT_CUDA(cudaFreeAsync(T, s));
  QTT_CUDA(cudaStreamSynchronize(s));
  *result = host;
  return kOk;
}

}  // namespace

int product(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b,
            const qtt_layout* LC, double* c, int mode, cudaStream_t s) {
  return launch_product(LA, a, LB, b, LC, c, mode, s);
}

int add(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b, double beta,
        const qtt_layout* LC, double* c, cudaStream_t s) {
  const int d = LA->d;
  if (d < 1 || d > QTT_MAX_CORES || LB->d != d || LC->d != d) return kInvalid;
  StructDesc desc;
  desc.ncores = d;
  for (int l = 0; l < d; ++l) {
    StructCore& sc = desc.c[l];
    sc.op = kOpAdd;
    sc.out_off = LC->offsets[l];
    sc.x_off = LA->offsets[l];
    sc.y_off = LB->offsets[l];
    sc.out_r0 = (int)LC->ranks[l];
    sc.out_r1 = (int)LC->ranks[l + 1];
    sc.out_n = (int)merged_n(LC, l);
    sc.xr0 = (int)LA->ranks[l];
    sc.xr1 = (int)LA->ranks[l + 1];
    sc.xn = sc.out_n;
    sc.yr0 = (int)LB->ranks[l];
    sc.yr1 = (int)LB->ranks[l + 1];
    sc.sx = 1.0;
    sc.sy = (l == 0) ? beta : 1.0;  // scaling the first core scales the TT
    sc.aux = sc.aux2 = 0;
  }
  return launch_struct(desc, a, b, c, s);
}

int zkron(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b,
          const qtt_layout* LC, double* c, cudaStream_t s) {
  const int d = LA->d;
  if (d < 1 || LB->d != d || LC->d != 2 * d || 2 * d > QTT_MAX_CORES) return kInvalid;
  // zkron writes its two inputs' cores into the output; both read from
  // separate buffers, so run two launches (fast cores from B, slow from A).
  StructDesc fast, slow;
  fast.ncores = d;
  slow.ncores = d;
  for (int k = 0; k < d; ++k) {
    const int ra0 = (int)LA->ranks[k], ra1 = (int)LA->ranks[k + 1];
    const int rb0 = (int)LB->ranks[k], rb1 = (int)LB->ranks[k + 1];
    StructCore& f = fast.c[k];
    f.op = kOpZFast;
    f.out_off = LC->offsets[2 * k];
    f.x_off = LB->offsets[k];
    f.out_r0 = rb0 * ra0;
    f.out_n = (int)merged_n(LB, k);
    f.out_r1 = rb1 * ra0;
    f.xr0 = rb0;
    f.xn = f.out_n;
    f.xr1 = rb1;
    f.aux = ra0;
    f.sx = 1.0;
    StructCore& w = slow.c[k];
    w.op = kOpZSlow;
    w.out_off = LC->offsets[2 * k + 1];
    w.x_off = LA->offsets[k];
    w.out_r0 = rb1 * ra0;
    w.out_n = (int)merged_n(LA, k);
    w.out_r1 = rb1 * ra1;
    w.xr0 = ra0;
    w.xn = w.out_n;
    w.xr1 = ra1;
    w.sx = 1.0;
    if (LC->ranks[2 * k] != f.out_r0 || LC->ranks[2 * k + 1] != f.out_r1 ||
        LC->ranks[2 * k + 2] != w.out_r1)
      return kInvalid;
  }
  QTT_TRY(launch_struct(fast, b, nullptr, c, s));
  return launch_struct(slow, a, nullptr, c, s);
}

int diag(const qtt_layout* LV, const double* v, const qtt_layout* LD, double* dd, cudaStream_t s) {
  const int d = LV->d;
  if (d < 1 || d > QTT_MAX_CORES || LD->d != d) return kInvalid;
  StructDesc desc;
  desc.ncores = d;
  for (int l = 0; l < d; ++l) {
    StructCore& sc = desc.c[l];
    const int n = (int)LV->rows[l];
    sc.op = kOpDiag;
    sc.out_off = LD->offsets[l];
    sc.x_off = LV->offsets[l];
    sc.out_r0 = (int)LV->ranks[l];
    sc.out_r1 = (int)LV->ranks[l + 1];
    sc.out_n = n * n;
    sc.xr0 = sc.out_r0;
    sc.xr1 = sc.out_r1;
    sc.xn = n;
    sc.aux = n;
    sc.sx = 1.0;
  }
  return launch_struct(desc, v, nullptr, dd, s);
}

int transpose_tt(const qtt_layout* LA, const double* a, const qtt_layout* LT, double* t,
                 cudaStream_t s) {
  const int d = LA->d;
  if (d < 1 || d > QTT_MAX_CORES || LT->d != d) return kInvalid;
  StructDesc desc;
  desc.ncores = d;
  for (int l = 0; l < d; ++l) {
    StructCore& sc = desc.c[l];
    sc.op = kOpTrans;
    sc.out_off = LT->offsets[l];
    sc.x_off = LA->offsets[l];
    sc.out_r0 = (int)LA->ranks[l];
    sc.out_r1 = (int)LA->ranks[l + 1];
    sc.out_n = (int)merged_n(LA, l);
    sc.xr0 = sc.out_r0;
    sc.xr1 = sc.out_r1;
    sc.xn = sc.out_n;
    sc.aux = (int)LA->rows[l];
    sc.aux2 = (int)LA->cols[l];
    sc.sx = 1.0;
  }
  return launch_struct(desc, a, nullptr, t, s);
}

int scale_copy(const qtt_layout* LA, const double* a, double sc0, double* out, cudaStream_t s) {
  const int d = LA->d;
  if (d < 1 || d > QTT_MAX_CORES) return kInvalid;
  StructDesc desc;
  desc.ncores = d;
  for (int l = 0; l < d; ++l) {
    StructCore& sc = desc.c[l];
    sc.op = kOpCopy;
    sc.out_off = LA->offsets[l];
    sc.x_off = LA->offsets[l];
    sc.out_r0 = (int)LA->ranks[l];
    sc.out_r1 = (int)LA->ranks[l + 1];
    sc.out_n = (int)merged_n(LA, l);
    sc.sx = l == 0 ? sc0 : 1.0;
  }
  return launch_struct(desc, a, nullptr, out, s);
}

int dot(const qtt_layout* LA, const double* a, const qtt_layout* LB, const double* b,
        double* result, cudaStream_t s) {
  if (LA->d < 1 || LA->d != LB->d) return kInvalid;
  return gram_dot(LA, a, LB, b, result, s);
}

}  // namespace qtt
