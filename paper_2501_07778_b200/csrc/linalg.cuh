// Dense FP64 building blocks for TT rounding / TT-SVD / AMEn (sm_100a).
#pragma once
#include "common.cuh"

#include <cstdlib>

namespace qtt {
// QTT_ROUND_TRACE=1: synchronising per-phase timer (diagnostics only).
struct PhaseTimer {
  bool on;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  explicit PhaseTimer(cudaStream_t st) : on(getenv("QTT_ROUND_TRACE") != nullptr), s(st) {
    if (on) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
  }
  void lap(const char* what, int k, int a, int b, int c) {
    if (!on) return;
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "[round] %-10s k=%2d %5d x %5d (%5d) %8.3f ms\n", what, k, a, b, c, ms);
    cudaEventRecord(e0, s);
  }
  ~PhaseTimer() {
    if (on) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
};


// Householder QR of a column-major m x n matrix A (lda).  Writes the
// explicit thin factor Q (m x k, ldq) and R (k x n upper triangular, ldr),
// k = min(m, n).  A is not modified.  Blocked: panels of 32 columns are
// factorised by one thread-block cluster (rows spread over up to 16 CTAs,
// reductions through distributed shared memory), trailing updates and the
// explicit-Q accumulation are compact-WY DMMA GEMMs.
//
// spec_dev (optional, device int): speculative mode.  Small well-conditioned
// factors (32 <= n <= 128, m >= n) then run as CholeskyQR2 with no host
// synchronisation; a breakdown ORs 1 into *spec_dev and leaves unspecified
// output, and the caller redoes the call with careful = true (Householder /
// synchronous CholeskyQR2 only) once it has read the flag.  Without spec_dev
// the same path is used but checked (one synchronisation) and falls back
// internally.
struct QrInfo;
int qr(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
       double* R, int64_t ldr, int* spec_dev = nullptr, bool careful = false, QrInfo* info = nullptr);

// One-sided (Hestenes) Jacobi on the p x k column-major matrix X (ldx, in
// place): X <- X W with W (k x k, ldw) orthogonal, so that the columns of X
// become mutually orthogonal.  W is initialised to the identity here.
// With floor_dev (device scalar) columns whose squared norm stays below
// (floor_scale * *floor_dev)^2 / k take no part in rotations (see
// jacobi_floor2 in linalg.cu); callers pass 1e-3 * delta.
int jacobi(cudaStream_t s, int p, int k, double* X, int64_t ldx, double* W, int64_t ldw,
           const double* floor_dev = nullptr, double floor_scale = 0.0);

// Column norms of X (p x k) sorted descending: sigma[k] and perm[k] (device).
// rank = chop(sigma, delta) (ttcore.py:175-190) with delta read from
// *delta_dev (device scalar) times delta_scale, clamped to rmax; floor_rule
// selects the reference rounding rule (eps floor) or the solver rule
// without floor (solver.py:221-236).  *rank_dev receives the kept rank.
int sort_chop(cudaStream_t s, int p, int k, const double* X, int64_t ldx, double* sigma,
              int* perm, const double* delta_dev, double delta_scale, int rmax, int floor_rule,
              int* rank_dev);

// Certificate that truncation cannot happen: with R (k x k upper triangular)
// sets *ok_dev = 1 iff 1/||R^{-1}||_F > 1.25 * max(delta, ||R||_F*max(k,2)*eps),
// i.e. the smallest singular value of R provably exceeds the _chop threshold.
// QTT_CERT_DEBUG=1 prints the per-bond margins.
int no_truncation_certificate(cudaStream_t s, int k, const double* R, int64_t ldr,
                              const double* delta_dev, double delta_scale, int* ok_dev);

// The same certificate for k <= 128 in ONE single-CTA launch.  ok_dev
// (optional) receives the verdict; sflag (optional) is a sticky device flag
// that gets bit 2 OR-ed in on failure (speculative sweeps check it once).
int cert_small(cudaStream_t s, int k, const double* R, int64_t ldr, const double* delta_dev,
               double delta_scale, int* ok_dev, int* sflag);

// X = R^{-1} for an upper-triangular k x k R (X: k x k, ld k): 64x64 diagonal
// blocks inverted in shared memory, recursive doubling with DMMA GEMMs.
int tri_inverse(cudaStream_t s, int k, const double* R, int64_t ldr, double* X);

// CholeskyQR2 (Gram -> Cholesky -> A R^{-1}, twice) for m >= n.  GEMM-bound
// replacement of the latency-bound Householder panels for well-conditioned
// tall matrices.  Returns kOk and sets *ok = 1 on success; *ok = 0 when the
// Cholesky breaks down or the first-pass Q is too far from orthonormal
// (||Q1^T Q1 - I||_F > 1/4), in which case the caller falls back to Householder.
// info (optional): on success, a lower bound of sigma_min(R) and ||R||_F =
// ||A||_F from the factorisation's own by-products, so the caller can decide
// the no-truncation certificate on the host without another pass.
struct QrInfo {
  bool valid = false;
  double sigma_lb = 0.0;  // sigma_min(R) >= sigma_lb
  double anorm = 0.0;     // ||A||_F = ||R||_F
};
int cholqr2(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
            double* R, int64_t ldr, int* ok, QrInfo* info = nullptr);

// Cheap no-truncation certificate for a tall column-major X (p x r, p >= r)
// from its Gram matrix: G = X^T X = R^T R (blocked Cholesky), and
//   sigma_min(X)^2 >= 1 / ||R^{-1}||_F^2 - 2 (p + r + 2) eps_mach ||X||_F^2
// (the subtracted term bounds the rounding error of forming and factoring
// G).  *ok_dev = 1 iff that lower bound exceeds
// (1.25 max(delta, ||X||_F max(r, 2) eps_mach))^2, delta = *delta_dev *
// delta_scale; 0 also when the Cholesky breaks down (caller falls back to a
// QR-based certificate: the Gram route cannot resolve sigma_min below
// ~sqrt(p eps_mach) ||X||).
int gram_certificate(cudaStream_t s, int p, int r, const double* X, int64_t ldx,
                     const double* delta_dev, double delta_scale, int* ok_dev);

// CholeskyQR2 for n <= 128 without host synchronisation (seven launches, the
// two n x n factorisations + inverses fused into one single-CTA kernel
// each).  Q and/or R may be null.  On breakdown the sticky device flag
// *status_dev is OR-ed with 1 and the outputs are unspecified: the caller
// checks the flag at its next synchronisation point and redoes the
// factorisation with qr(..., careful = true).
//
// scalars (optional, 8 device doubles) receives the by-products
// [1] = ||R1^{-1}||_F^2, [2] = ||A||_F^2, [4] = ||Q1^T Q1 - I||_F^2, from which
// cert_factors() evaluates the no-truncation certificate of R without
// another pass (ORs 2 into the sticky flag when it fails).
int cholqr2_small(cudaStream_t s, int m, int n, const double* A, int64_t lda, double* Q, int64_t ldq,
                  double* R, int64_t ldr, int* status_dev, double* scalars = nullptr);
int cert_factors(cudaStream_t s, int k, const double* scalars, const double* delta_dev,
                 double delta_scale, int* sflag);
constexpr int kCholQrSmallMin = 32, kCholQrSmallMax = 128;  // n range of cholqr2_small inside qr()

// Process-wide high-priority side stream used for look-ahead factorisation
// of the next panel / diagonal block while the trailing update runs.
cudaStream_t side_stream();

// Gather columns: dst[:, c] = src[:, perm[c]] for c < cols (device perm).
int gather_columns(cudaStream_t s, int rows, int cols, const double* src, int64_t lds,
                   const int* perm, double* dst, int64_t ldd);

// Frobenius norm of a contiguous array into a device scalar.
int frob_norm(cudaStream_t s, int64_t n, const double* x, double* out_dev);

// Identity into a column-major rows x cols matrix.
int set_identity(cudaStream_t s, int rows, int cols, double* A, int64_t lda);

}  // namespace qtt
