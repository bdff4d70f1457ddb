// FP64 GEMM on the DMMA tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// B200 has no tcgen05 kind for f64: the FP64 tensor path is the DMMA unit
// fed from registers, so this kernel stages 64x64x16 tiles through shared
// memory with cp.async double buffering and runs 2x2 warps of 32x32 warp
// tiles (16 DMMA accumulators per warp).  Column-major operands, optional
// transposes, strided batching.  Used for every dense contraction of the
// TT hot path: rounding carries, compact-WY updates, Jacobi rotations,
// AMEn environment contractions and the dense residual.
#include "common.cuh"

#include <cstdlib>

namespace qtt {
namespace {

constexpr int BK = 16, PAD = 4;

// CTA tile configurations: WM x WN warps, each owning a (8 TM) x (8 TN) block
// of DMMA m8n8 tiles; CTA tile (8 WM TM) x (8 WN TN); STG-deep pipeline.
template <int WM_, int WN_, int TM_, int TN_, int STG_>
struct TileCfg {
  static constexpr int WM = WM_, WN = WN_, TM = TM_, TN = TN_, STG = STG_;
  static constexpr int BM = 8 * WM * TM, BN = 8 * WN * TN, THREADS = 32 * WM * WN;
  static constexpr int SMEM = STG * BK * (BM + PAD + BN + PAD) * (int)sizeof(double);
  static_assert(STG >= 3, "pipeline needs >= 3 stages");
};
// 64 x 64 CTA tile, 2 x 2 warps of 32 x 32, 4 stages.  (Measured against
// 128 x 64, 64 x 128, 128 x 128 and 64 x 32 tiles with 4-8 warps: none is
// faster once the tile loads are hoisted; 8192^3 runs at cuBLAS speed.)
using CfgSmall = TileCfg<2, 2, 4, 4, 4>;
// 32 x 32 CTA tile (2 x 2 warps of 16 x 16) for small outputs with a short
// reduction (k < 1024; QTT_GEMM_TINY_K overrides), where the 64 x 64 grid
// leaves most SMs idle: 4x the CTAs beats a 2-way split-K at k = 512-768
// (tools/tiny_ab.py; config-2 serial step 148 -> 145 ms).
using CfgTiny = TileCfg<2, 2, 2, 2, 4>;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <int TA, int TB, class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS) gemm_kernel(GemmArgs g, int mt, int kchunk, double* ws) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, THREADS = Cfg::THREADS, STAGES = Cfg::STG;
  constexpr int TM = Cfg::TM, TN = Cfg::TN;
  extern __shared__ double gemm_sm[];
  double (*As)[BK][BM + PAD] = reinterpret_cast<double (*)[BK][BM + PAD]>(gemm_sm);
  double (*Bs)[BK][BN + PAD] = reinterpret_cast<double (*)[BK][BN + PAD]>(gemm_sm + STAGES * BK * (BM + PAD));

  // Grouped tile order: consecutive CTAs cover GROUP m-tiles x all n-tiles
  // column by column, so the A panels of a wave stay in L2.
  constexpr int GROUP = 8;
  const int tile = blockIdx.x;
  const int nt = (g.n + BN - 1) / BN;
  const int first_m = (tile / (GROUP * nt)) * GROUP;
  const int gsz = min(mt - first_m, GROUP);
  const int in_group = tile % (GROUP * nt);
  int mi = first_m + in_group % gsz, ni = in_group / gsz;
  // Triangular operands make tiles unequal: issue the longest reductions
  // first (kGemmTriB / kGemmLowA: K grows with n / m) so they do not form
  // the tail of the last wave.
  if (g.flags & kGemmTriB) ni = nt - 1 - ni;
  if (g.flags & kGemmLowA) mi = mt - 1 - mi;
  const int m0 = mi * BM;
  const int n0 = ni * BN;
  const int bz = blockIdx.y;
  const double* A = g.a + bz * g.stride_a;
  const double* B = g.b + bz * g.stride_b;
  double* C = g.c + bz * g.stride_c;
  const int M = g.m, N = g.n;
  int kbeg = blockIdx.z * kchunk;
  int K = min(g.k, kbeg + kchunk);  // tiles cover [kbeg, K)
  if (g.flags) {
    if ((g.flags & kGemmUpperC) && m0 >= n0 + BN) {
      if (ws == nullptr) return;
      K = kbeg;  // split-K partial of a skipped tile: zeros
    }
    if (g.flags & kGemmTriA) kbeg = max(kbeg, m0);
    if (g.flags & kGemmTriB) K = min(K, n0 + BN);
    if (g.flags & kGemmLowA) K = min(K, m0 + BM);
    if (g.flags & kGemmLowB) kbeg = max(kbeg, n0);
  }
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = (warp % Cfg::WM) * (8 * TM), wn = (warp / Cfg::WM) * (8 * TN);

  // Global -> shared tile loads.  Every thread owns a fixed row (or column)
  // of the tile and a fixed set of k offsets, so the addresses are one base
  // pointer plus compile-time multiples of a precomputed stride, and the
  // row predicate is hoisted; only the K bound is tested per stage.
  static_assert(THREADS % BM == 0 && THREADS % BN == 0 && THREADS % BK == 0, "tile/thread shape");
  constexpr int A_E = (BM * BK) / THREADS, B_E = (BN * BK) / THREADS;
  // TA == 0: A(m, k) at a + m + k lda, thread -> m = t % BM, k = t / BM + e (THREADS / BM)
  // TA == 1: A(m, k) at a + k + m lda, thread -> k = t % BK, m = t / BK + e (THREADS / BK)
  const int a_m = TA == 0 ? t % BM : t / BK, a_k = TA == 0 ? t / BM : t % BK;
  const int b_n = TB == 0 ? t / BK : t % BN, b_k = TB == 0 ? t % BK : t / BN;
  const double* pa = A + (TA == 0 ? (int64_t)(m0 + a_m) + (int64_t)(kbeg + a_k) * g.lda
                                   : (int64_t)(kbeg + a_k) + (int64_t)(m0 + a_m) * g.lda);
  const double* pb = B + (TB == 0 ? (int64_t)(kbeg + b_k) + (int64_t)(n0 + b_n) * g.ldb
                                   : (int64_t)(n0 + b_n) + (int64_t)(kbeg + b_k) * g.ldb);
  const int64_t a_es = TA == 0 ? (int64_t)(THREADS / BM) * g.lda : (int64_t)(THREADS / BK) * g.lda;
  const int64_t b_es = TB == 0 ? (int64_t)(THREADS / BK) * g.ldb : (int64_t)(THREADS / BN) * g.ldb;
  const int64_t a_ks = TA == 0 ? (int64_t)BK * g.lda : BK;  // per stage
  const int64_t b_ks = TB == 0 ? BK : (int64_t)BK * g.ldb;
  // row predicates (TA == 1 / TB == 0: the owned rows/columns vary with e)
  unsigned a_rows = 0, b_cols = 0;
#pragma unroll
  for (int e = 0; e < A_E; ++e) {
    const int m = TA == 0 ? a_m : a_m + e * (THREADS / BK);
    if (m0 + m < M) a_rows |= 1u << e;
  }
#pragma unroll
  for (int e = 0; e < B_E; ++e) {
    const int nn = TB == 0 ? b_n + e * (THREADS / BK) : b_n;
    if (n0 + nn < N) b_cols |= 1u << e;
  }
  auto load_tile = [&](int buf, int st) {
    const int k0 = kbeg + st * BK;
    const double* qa = pa + st * a_ks;
    const double* qb = pb + st * b_ks;
#pragma unroll
    for (int e = 0; e < A_E; ++e) {
      const int kk = TA == 0 ? a_k + e * (THREADS / BM) : a_k;
      const int mm = TA == 0 ? a_m : a_m + e * (THREADS / BK);
      const bool ok = ((a_rows >> e) & 1u) && k0 + kk < K;
      cp_async8(&As[buf][kk][mm], ok ? qa + e * a_es : A, ok);
    }
#pragma unroll
    for (int e = 0; e < B_E; ++e) {
      const int kk = TB == 0 ? b_k : b_k + e * (THREADS / BN);
      const int nn = TB == 0 ? b_n + e * (THREADS / BK) : b_n;
      const bool ok = ((b_cols >> e) & 1u) && k0 + kk < K;
      cp_async8(&Bs[buf][kk][nn], ok ? qb + e * b_es : B, ok);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = (K - kbeg + BK - 1) / BK;
  // STAGES-deep cp.async pipeline (one commit group per stage; empty groups
  // at the tail keep the wait counts uniform) with register double-buffered
  // fragments: the fragments of k-step s+1 are loaded while the DMMAs of
  // k-step s issue; the single barrier per stage sits before the last
  // k-step, when the next stage's first fragments are fetched.
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < ktiles) load_tile(st, st);
    cp_async_commit();
  }
  constexpr int KS = BK / 4;
  double af[2][TM], bf[2][TN];
  auto load_frag = [&](int buf, int ks, int slot) {
    const int kr = ks * 4 + (lane & 3);
#pragma unroll
    for (int i = 0; i < TM; ++i) af[slot][i] = As[buf][kr][wm + i * 8 + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < TN; ++j) bf[slot][j] = Bs[buf][kr][wn + j * 8 + (lane >> 2)];
  };
  if (ktiles > 0) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load_frag(0, 0, 0);
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt % STAGES;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int cur = ks & 1;
      if (ks == KS - 1) {
        // stage kt+1 landed (groups 0..kt+STAGES-2 committed) and every
        // thread is past its reads of stage kt-1, whose buffer is refilled
        cp_async_wait<STAGES - 3>();
        __syncthreads();
        const int nxt = kt + STAGES - 1;
        if (nxt < ktiles) load_tile(nxt % STAGES, nxt);
        cp_async_commit();
        if (kt + 1 < ktiles) load_frag((kt + 1) % STAGES, 0, cur ^ 1);
      } else {
        load_frag(buf, ks + 1, cur ^ 1);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma(acc[i][j], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();

  if (ws != nullptr) {
    // split-K partial: plain accumulator into ws[(z * batch + b) * M * N]
    double* W = ws + ((int64_t)blockIdx.z * gridDim.y + bz) * (int64_t)M * N;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int row = m0 + wm + i * 8 + (lane >> 2);
      if (row >= M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = n0 + wn + j * 8 + 2 * (lane & 3) + h;
          if (col < N) W[row + (int64_t)col * M] = acc[i][j][h];
        }
    }
    return;
  }
  const double alpha = g.alpha, beta = g.beta;
  if (beta != 0.0) {
    // all C loads in flight before the first store (no load-store chain)
    double cv[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int row = m0 + wm + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = n0 + wn + j * 8 + 2 * (lane & 3) + h;
          cv[i][j][h] = (row < M && col < N) ? __ldg(C + row + (int64_t)col * g.ldc) : 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][j][h] = fma(alpha, acc[i][j][h], beta * cv[i][j][h]);
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][j][h] *= alpha;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = m0 + wm + i * 8 + (lane >> 2);
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (col < N) C[row + (int64_t)col * g.ldc] = acc[i][j][h];
      }
    }
  }
}

__global__ void splitk_reduce_kernel(GemmArgs g, int splits, const double* __restrict__ ws) {
  const int64_t mn = (int64_t)g.m * g.n;
  const int64_t total = mn * g.batch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / mn, e = i % mn;
    const int r = (int)(e % g.m);
    const int64_t c = e / g.m;
    double acc = 0.0;
    for (int s = 0; s < splits; ++s) acc += ws[((int64_t)s * g.batch + b) * mn + e];
    double* p = g.c + b * g.stride_c + r + c * g.ldc;
    double v = g.alpha * acc;
    if (g.beta != 0.0) v += g.beta * *p;
    *p = v;
  }
}

__global__ void scale_kernel(GemmArgs g) {
  // k == 0 (or alpha == 0): C = beta * C
  int64_t total = (int64_t)g.m * g.n;
  double* C = g.c + blockIdx.y * g.stride_c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = i % g.m;
    int64_t c = i / g.m;
    double* p = C + r + c * g.ldc;
    *p = g.beta == 0.0 ? 0.0 : g.beta * *p;
  }
}

__global__ void transpose_kernel(int rows, int cols, const double* __restrict__ src, int64_t lds,
                                 double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) tile[j][threadIdx.x] = src[r + (int64_t)c * lds];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    int c = c0 + threadIdx.x, r = r0 + j;
    if (r < rows && c < cols) dst[c + (int64_t)r * ldd] = tile[threadIdx.x][j];
  }
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void copy_matrix_kernel(int rows, int cols, const double* __restrict__ src, int64_t lds,
                                   double* __restrict__ dst, int64_t ldd) {
  int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = i % rows;
    int64_t c = i / rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}

}  // namespace

void pool_init() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

namespace {
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;
}  // namespace

namespace {
thread_local bool t_shared_pool = false;
}  // namespace

void set_thread_shared_pool(bool shared) { t_shared_pool = shared; }

cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s) {
  // QTT_SHARED_POOL=1 / =0: every thread on the device's default pool / on a private one (A/B)
  static const char* env = getenv("QTT_SHARED_POOL");
  const bool shared = env ? env[0] != '0' : t_shared_pool;
  if (shared) return cudaMallocAsync(p, bytes, s);
  thread_local cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  dev &= 63;
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    e = cudaMemPoolCreate(&pools[dev], &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pools.push_back(pools[dev]);
  }
  return cudaMallocFromPoolAsync(p, bytes, pools[dev], s);
}

void trim_thread_pools() {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (cudaMemPool_t pool : g_pools) cudaMemPoolTrimTo(pool, 0);
}

GemmProfile& gemm_profile() {
  static GemmProfile p;
  return p;
}

int gemm(const GemmArgs& g, cudaStream_t stream) {
  if (g.m < 0 || g.n < 0 || g.k < 0 || g.batch < 0) return kInvalid;
  if (g.m == 0 || g.n == 0 || g.batch == 0) return kOk;
  if (g.batch > 65535) return kUnsupported;
  if (g.k == 0 || g.alpha == 0.0) {
    dim3 grid((unsigned)std::min<int64_t>(ceil_div((int64_t)g.m * g.n, 256), 4096), g.batch);
    scale_kernel<<<grid, 256, 0, stream>>>(g);
    QTT_CHECK_LAUNCH();
    return kOk;
  }
  static const bool tiny_ok = getenv("QTT_GEMM_NO_TINY") == nullptr;
  const int64_t tiles64 = ceil_div(g.m, CfgSmall::BM) * ceil_div(g.n, CfgSmall::BN);
  static const int tiny_k = getenv("QTT_GEMM_TINY_K") ? atoi(getenv("QTT_GEMM_TINY_K")) : 1024;
  const bool tiny = tiny_ok && tiles64 * g.batch < num_sms() && g.k < tiny_k;
  const int BM = tiny ? CfgTiny::BM : CfgSmall::BM, BN = tiny ? CfgTiny::BN : CfgSmall::BN;
  const int mt = (int)ceil_div(g.m, BM);
  const int64_t tiles = (int64_t)mt * ceil_div(g.n, BN);
  if (tiles > 0x7fffffff) return kUnsupported;
  dim3 grid((unsigned)tiles, g.batch);
  GemmProfile& prof = gemm_profile();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof.on) {
    QTT_CUDA(cudaEventCreate(&e0));
    QTT_CUDA(cudaEventCreate(&e1));
    QTT_CUDA(cudaEventRecord(e0, stream));
  }
  // Split K when the tile grid cannot fill the SMs (skinny outputs with a
  // long reduction, e.g. V^T A in the compact-WY updates); the partial sums
  // are reduced in a fixed order, so results stay deterministic.
  // kGemmUpperC grids count only the tiles that compute (the strictly lower
  // ones exit at once), so a Gram matrix with a long reduction splits too.
  int splits = 1;
  int64_t work_tiles = tiles;
  if (g.flags & kGemmUpperC) {
    const int64_t nt = ceil_div(g.n, BN);
    work_tiles = 0;
    for (int64_t ni = 0; ni < nt; ++ni) work_tiles += std::min<int64_t>(mt, ceil_div((ni + 1) * BN, BM));
  }
  const int64_t ctas = work_tiles * g.batch;
  static const int split_fill = getenv("QTT_GEMM_SPLIT_FILL") ? atoi(getenv("QTT_GEMM_SPLIT_FILL")) : 1;
  if (!tiny && ctas < split_fill * num_sms() && g.k >= 512) {
    splits = (int)std::min<int64_t>({16, ceil_div((split_fill + 1) * num_sms(), ctas), g.k / 256});
    splits = std::max(splits, 1);
  }
  const int kchunk = splits > 1 ? (int)(ceil_div(ceil_div(g.k, splits), BK) * BK) : g.k;
  if (splits > 1) splits = (int)ceil_div(g.k, kchunk);
  double* ws = nullptr;
  if (splits > 1)
    QTT_CUDA(malloc_async(&ws, sizeof(double) * splits * g.batch * (int64_t)g.m * g.n, stream));
  grid.z = splits;
  static DeviceFlag configured;
  if (!configured.test()) {
#define QTT_CFG_ATTR(TA_, TB_, CF)                                                                   \
  QTT_CUDA(cudaFuncSetAttribute(gemm_kernel<TA_, TB_, CF>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                CF::SMEM));
    QTT_CFG_ATTR(0, 0, CfgSmall) QTT_CFG_ATTR(0, 1, CfgSmall) QTT_CFG_ATTR(1, 0, CfgSmall) QTT_CFG_ATTR(1, 1, CfgSmall)
    QTT_CFG_ATTR(0, 0, CfgTiny) QTT_CFG_ATTR(0, 1, CfgTiny) QTT_CFG_ATTR(1, 0, CfgTiny) QTT_CFG_ATTR(1, 1, CfgTiny)
#undef QTT_CFG_ATTR
    configured.set();
  }
#define QTT_LAUNCH(CF)                                                                             \
  do {                                                                                             \
    if (!g.trans_a && !g.trans_b) gemm_kernel<0, 0, CF><<<grid, CF::THREADS, CF::SMEM, stream>>>(g, mt, kchunk, ws); \
    else if (!g.trans_a && g.trans_b) gemm_kernel<0, 1, CF><<<grid, CF::THREADS, CF::SMEM, stream>>>(g, mt, kchunk, ws); \
    else if (g.trans_a && !g.trans_b) gemm_kernel<1, 0, CF><<<grid, CF::THREADS, CF::SMEM, stream>>>(g, mt, kchunk, ws); \
    else gemm_kernel<1, 1, CF><<<grid, CF::THREADS, CF::SMEM, stream>>>(g, mt, kchunk, ws);       \
  } while (0)
  if (tiny)
    QTT_LAUNCH(CfgTiny);
  else
    QTT_LAUNCH(CfgSmall);
#undef QTT_LAUNCH
  QTT_CHECK_LAUNCH();
  if (splits > 1) {
    const int64_t total = (int64_t)g.m * g.n * g.batch;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 16 * num_sms());
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(g, splits, ws);
    QTT_CHECK_LAUNCH();
    QTT_CUDA(cudaFreeAsync(ws, stream));
  }
  if (e0) {
    QTT_CUDA(cudaEventRecord(e1, stream));
    std::lock_guard<std::mutex> lk(prof.mu);
    prof.events.emplace_back(e0, e1);
    double f = 2.0 * g.m * (double)g.n * g.k * g.batch;
    if (g.flags) {  // multiply-adds of the tiles actually computed
      f = 0.0;
      for (int mi = 0; mi < mt; ++mi)
        for (int64_t ni = 0; ni < tiles / mt; ++ni) {
          if ((g.flags & kGemmUpperC) && (int64_t)mi * BM >= (ni + 1) * BN) continue;
          const int64_t klo = (g.flags & kGemmTriA) ? (int64_t)mi * BM : 0;
          int64_t khi = (g.flags & kGemmTriB) ? std::min<int64_t>(g.k, (ni + 1) * BN) : g.k;
          if (g.flags & kGemmLowA) khi = std::min<int64_t>(khi, (int64_t)(mi + 1) * BM);
          const int64_t klo2 = (g.flags & kGemmLowB) ? std::max<int64_t>(klo, ni * BN) : klo;
          if (khi > klo2)
            f += 2.0 * std::min(BM, g.m - mi * BM) * std::min<int64_t>(BN, g.n - ni * BN) * (khi - klo2);
        }
      f *= g.batch;
    }
    prof.launch_flops.push_back(f);
    prof.shapes.push_back({g.m, g.n, g.k, g.batch, g.flags, splits, BM});
    prof.flops += f;
  }
  return kOk;
}

int transpose(cudaStream_t s, int rows, int cols, const double* src, int64_t lds, double* dst,
              int64_t ldd) {
  if (rows <= 0 || cols <= 0) return kOk;
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(cols, 32));
  if (grid.y > 65535) return kUnsupported;
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(rows, cols, src, lds, dst, ldd);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int fill(cudaStream_t s, double* p, int64_t n, double v) {
  if (n <= 0) return kOk;
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 8 * num_sms());
  fill_kernel<<<blocks, 256, 0, s>>>(p, n, v);
  QTT_CHECK_LAUNCH();
  return kOk;
}

int copy_matrix(cudaStream_t s, int rows, int cols, const double* src, int64_t lds, double* dst,
                int64_t ldd) {
  if (rows <= 0 || cols <= 0) return kOk;
  int blocks = (int)std::min<int64_t>(ceil_div((int64_t)rows * cols, 256), 8 * num_sms());
  copy_matrix_kernel<<<blocks, 256, 0, s>>>(rows, cols, src, lds, dst, ldd);
  QTT_CHECK_LAUNCH();
  return kOk;
}

}  // namespace qtt
