/*
 * qtt_b200.h — C ABI of the B200-native QTT hot path (libqttb200.so).
 *
 * Drop-in boundary for the tensor-train linear algebra of the reference
 * package `qttfem` (arXiv 2501.07778).  The reference is pure Python over
 * numpy/LAPACK, so its "FFI" for this path is the set of module functions
 * listed next to every entry point below; the Python mirror
 * (paper_2501_07778_b200/*.py) binds these symbols with ctypes and keeps the
 * reference signatures, argument meanings and ValueError/TypeError behaviour.
 *
 * Conventions
 *   - All numeric buffers are device pointers to FP64 data.
 *   - A TT object is a packed buffer of cores plus a host-side qtt_layout:
 *     vector cores (r_l, n_l, r_{l+1}) and matrix cores (r_l, n_l, m_l,
 *     r_{l+1}), C-contiguous, exactly the reference core layouts
 *     (ttcore.py:55-138); core l starts at data + offsets[l] (element offset,
 *     multiple of 32 so every core is 256-byte aligned).
 *   - Mode 1 is the least significant index bit (ttcore.py:3-10).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Return value: QTT_OK or one of the QTT_E* codes.  Entry points that
 *     return data-dependent ranks write them into the caller's out layout;
 *     they synchronise `stream` once to do so.
 *   - The caller owns every output buffer.  Temporary device memory comes
 *     from the CUDA stream-ordered allocator on `stream`.
 */
#ifndef QTT_B200_H_
#define QTT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QTT_MAX_CORES 64

enum {
  QTT_OK = 0,
  QTT_EINVAL = 1,      /* shape / argument error (Python raises ValueError) */
  QTT_ECUDA = 2,       /* CUDA runtime error                               */
  QTT_EWORKSPACE = 3,  /* output buffer too small                          */
  QTT_EUNSUPPORTED = 4 /* size outside the kernels' envelope              */
};

typedef struct qtt_layout {
  int32_t d;                         /* number of cores                     */
  int32_t is_matrix;                 /* 0: vector cores, 1: matrix cores    */
  int64_t ranks[QTT_MAX_CORES + 1];  /* r_0 .. r_d (r_0 = r_d = 1)          */
  int64_t rows[QTT_MAX_CORES];       /* n_l                                 */
  int64_t cols[QTT_MAX_CORES];       /* m_l (1 for vectors)                 */
  int64_t offsets[QTT_MAX_CORES];    /* element offset of core l            */
} qtt_layout;

/* Library identification; returns a static string. */
const char* qtt_version(void);

/* Kernel launches issued by the library since load (bench.py evidence). */
long long qtt_launch_count(void);

/* DMMA GEMM profiling: qtt_profile_gemm(1) starts recording CUDA events
 * around every GEMM launch (on its stream); _read returns the summed
 * algorithmic FLOPs (2mnk), the summed event time and the launch count. */
int qtt_profile_gemm(int32_t on);
int qtt_profile_gemm_read(double* flops, double* ms, int64_t* launches);
/* Dispatch record of the i-th profiled GEMM launch (negative i counts from
 * the end): out[7] = {m, n, k, batch, flags, k-splits, tile rows BM}.  Lets
 * the parity tests assert which kernel configuration a shape reached. */
int qtt_profile_gemm_shape(int64_t i, int64_t* out);

/* Number of doubles a packed buffer for `lay` needs (with alignment). */
int64_t qtt_layout_size(const qtt_layout* lay);

/* Synchronise `stream` and return the unused memory cached by the library's
 * stream-ordered pool to the driver (no reference counterpart: host-side
 * memory management for growing AMEn local systems, solver.py:148-171). */
int qtt_release_cached(void* stream);
/* Memory-pool policy of the CALLING host thread for the library's
 * stream-ordered temporaries: 1 = the device's shared default pool (what the
 * concurrent chain workers of the Python mirror use), 0 = a pool private to
 * the thread (the default; see csrc/common.cuh for the measurements). */
int qtt_thread_shared_pool(int32_t shared);

/* ---------------------------------------------------------------- (a2,a3)
 * Exact core-wise products, all cores in ONE launch.
 * qtt_matvec  replaces ttcore.tt_matvec  (ttcore.py:443-455):
 *   y_l[(a,c), i, (b,e)] = sum_j A_l[a,i,j,b] x_l[c,j,e]
 * qtt_matmat  replaces ttcore.tt_matmat  (ttcore.py:458-470).
 * qtt_hadamard replaces ttcore.tt_hadamard (ttcore.py:421-440); for matrix
 *   operands the modes are the merged (i,j) pairs.
 * Output layouts (ranks = products) are computed by the caller. */
int qtt_matvec(const qtt_layout* A, const double* a, const qtt_layout* x,
               const double* xd, const qtt_layout* y, double* yd, void* stream);
int qtt_matmat(const qtt_layout* A, const double* a, const qtt_layout* B,
               const double* b, const qtt_layout* C, double* c, void* stream);
int qtt_hadamard(const qtt_layout* A, const double* a, const qtt_layout* B,
                 const double* b, const qtt_layout* C, double* c, void* stream);

/* ------------------------------------------------------------------- (a4)
 * Structural algebra, one launch each.
 * qtt_add      replaces tt_add      (ttcore.py:380-411), scales b by beta.
 * qtt_zkron    replaces tt_zkron    (ttcore.py:501-539).
 * qtt_diag     replaces tt_diag     (ttcore.py:478-486).
 * qtt_transpose replaces tt_transpose (ttcore.py:473-475).
 * qtt_scale    replaces tt_scale    (ttcore.py:414-418): copy, core 0 * s. */
int qtt_add(const qtt_layout* A, const double* a, const qtt_layout* B,
            const double* b, double beta, const qtt_layout* C, double* c,
            void* stream);
int qtt_zkron(const qtt_layout* A, const double* a, const qtt_layout* B,
              const double* b, const qtt_layout* C, double* c, void* stream);
int qtt_diag(const qtt_layout* V, const double* v, const qtt_layout* D,
             double* dd, void* stream);
int qtt_transpose(const qtt_layout* A, const double* a, const qtt_layout* T,
                  double* t, void* stream);
int qtt_scale(const qtt_layout* A, const double* a, double s, double* out,
              void* stream);

/* ------------------------------------------------------------------- (a5)
 * TT rounding, replaces ttcore.tt_round (ttcore.py:322-338):
 * right-to-left QR sweep, then left-to-right truncated SVD sweep with
 * delta = eps/sqrt(d-1)*||t|| and the _chop rule (ttcore.py:175-190).  Same
 * ranks and the same tensor within eps as the reference; how it gets there
 * (DESIGN.md section 4): structurally full-rank cores are folded into
 * identities, a bond whose triangular factor provably has no singular value
 * at or below the _chop threshold keeps its QR factors instead of an SVD
 * (one certificate covers every bond of the leading identity zone),
 * otherwise one-sided Jacobi; factors of dimension <= 128 run without host
 * synchronisation (a sticky device flag sends the call back to the examined
 * path).  QTT_ROUND_NO_SPEC=1 / QTT_ROUND_NO_ZONE=1 switch those two off,
 * QTT_ROUND_TRACE=1 prints per-phase device times.
 * `out` receives the final ranks/offsets; out_data needs
 * qtt_layout_size(in) doubles (ranks never increase). */
int qtt_round(const qtt_layout* in, const double* in_data, double eps,
              qtt_layout* out, double* out_data, void* stream);
/* qtt_round that also streams the result to pinned host memory: every core is
 * copied device -> host (at the same packed offsets as in out_data) on a
 * second stream as soon as it is final, while the sweep continues, so the
 * read-back overlaps the computation (the reference's tt_round returns host
 * arrays; this is the drop-in's way of doing the same without a serial
 * D2H pass).  host_data: page-locked, at least as large as out_data. */
int qtt_round_to_host(const qtt_layout* in, const double* in_data, double eps,
                      qtt_layout* out, double* out_data, double* host_data,
                      void* stream);

/* ------------------------------------------------------------------- (a6)
 * TT-SVD of a dense vector, replaces ttcore.tt_decompose for 1-D input
 * (ttcore.py:211-235, _tt_svd 193-208).  `sizes` are the d mode sizes;
 * `dense` is read only.  `out` receives ranks/offsets; out_data must hold
 * `out_capacity` doubles. */
int qtt_decompose(const double* dense, int32_t d, const int64_t* sizes,
                  double eps, qtt_layout* out, double* out_data,
                  int64_t out_capacity, void* stream);

/* ------------------------------------------------------------------- (a7)
 * Norm / inner product (ttcore.py:341-363); results land in host memory. */
int qtt_norm(const qtt_layout* A, const double* a, double* result,
             void* stream);
int qtt_dot(const qtt_layout* A, const double* a, const qtt_layout* B,
            const double* b, double* result, void* stream);

/* ------------------------------------------------------------- (a8,a14)
 * Dense realisation (ttcore.tt_contract, ttcore.py:267-293) and dense
 * operator application (solver.apply_tt_matrix, solver.py:57-78). */
int qtt_contract(const qtt_layout* A, const double* a, double* dense,
                 void* stream);
int qtt_dense_apply(const qtt_layout* A, const double* a, const double* v,
                    double* out, void* stream);

/* ------------------------------------------------------------------- (a9)
 * Index maps, bit exact (indexing.py:58-112).  perm has 4^d (node) or
 * 2*4^d (dof) int64 entries on the device. */
int qtt_zorder_permutation(int32_t d, int64_t* perm, void* stream);
int qtt_zorder_dof_permutation(int32_t d, int64_t* perm, void* stream);
int qtt_z_index(int32_t d, int64_t count, const int64_t* i, const int64_t* j,
                int64_t* z, void* stream);

/* ------------------------------------------------------------------ (a10)
 * Element value grids, replaces element.element_stiffness_block /
 * element_load_block (element.py:160-212) for all 16 corner pairs at once.
 * coef: per Gauss point 25 doubles = J00[4], dJ10[4], dJ01[4] (entries
 * x_xi, y_xi, x_eta, y_eta), weight, shape gradients [4][2], shape values
 * [4]; cmat: 3x3 row-major C.  modulus (device, optional): [g][i][j]
 * multiplier of the stiffness integrand (config-4 E(x,y) extension).
 * kout: 64 vectors (pair a*4+b, component alpha*2+beta) and gout: 16
 * vectors of length 4^d, zero-padded, in Z-order (zorder=1) or canonical
 * order.  *degenerate = 1 if any |J| <= 0 (Python raises ValueError). */
int qtt_element_grids(int32_t d, int32_t zorder, int32_t ngauss,
                      const double* coef, const double* cmat,
                      int32_t paper_det, const double* modulus, double* kout,
                      double* gout, int32_t* degenerate, void* stream);

/* ------------------------------------------------------------------ (a13)
 * Dense local solve of the AMEn sweep, replaces np.linalg.solve in
 * solver._solve_local (solver.py:162-173): blocked LU without pivoting on
 * [M | b] with DMMA updates, residual check, Householder-QR fallback.
 * M is n x n column-major (ldm); b, x have n entries (device).
 * *fallback = 1 if the QR path was taken. */
int qtt_dense_solve(int64_t n, const double* m, int64_t ldm, const double* b,
                    double* x, int32_t* fallback, void* stream);

/* Restarted GMRES on the structured AMEn local operator, replaces the
 * scipy.sparse.linalg.gmres call of solver._solve_local (solver.py:186-195:
 * restart, rtol, atol = 0, warm start x0).  The operator
 *   M[(x,i,g),(y,j,h)] = sum_ab phi_l[x,a,y] A[a,i,j,b] phi_r[g,b,h]
 * is applied without being formed (solver._proj_a): phi_l (rl,ra,rl),
 * a_jib = A permuted to (a,j,i,b) as a row-major (ra*n) x (n*rb) matrix,
 * phi_r (rr,rb,rr), rhs/x0/x (rl,n,rr), all C-order on the device (x may
 * alias x0).  abort_early != 0 stops once the first cycles' rate projects
 * past maxit (the caller then solves densely).  *iters / *converged report
 * the outcome; non-convergence is not an error. */
int qtt_local_gmres(int64_t rl, int64_t n, int64_t rr, int64_t ra, int64_t rb,
                    const double* phi_l, const double* a_jib, const double* phi_r,
                    const double* rhs, const double* x0, double* x, double rtol,
                    int32_t restart, int32_t maxit, int32_t abort_early,
                    int32_t* iters, int32_t* converged, void* stream);
/* y = M x for the same operator (solver._local_matvec, solver.py:136-139). */
int qtt_local_apply(int64_t rl, int64_t n, int64_t rr, int64_t ra, int64_t rb,
                    const double* phi_l, const double* a_jib, const double* phi_r,
                    const double* x, double* y, void* stream);

/* ------------------------------------------------------ dense primitives
 * Exposed for the parity tests of the building blocks. */
int qtt_gemm(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
             int64_t k, double alpha, const double* a, int64_t lda,
             const double* b, int64_t ldb, double beta, double* c,
             int64_t ldc, void* stream);
/* qtt_gemm with the internal structure flags of the rounding/Cholesky
 * products (bit 1: only entries of C with row <= col are defined -- tiles entirely
 * below the diagonal are skipped, so strictly-lower entries of diagonal
 * tiles may be left unwritten;
 * 2 / 4: op(A) / op(B) upper triangular; 8 / 16: lower triangular), so the
 * parity tests reach the clipped-reduction, split-K and tile-order paths. */
int qtt_gemm_structured(int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
                        int64_t k, double alpha, const double* a, int64_t lda,
                        const double* b, int64_t ldb, double beta, double* c,
                        int64_t ldc, int32_t flags, void* stream);
/* QR of a column-major m x n matrix: explicit thin Q (m x k) and upper
 * triangular R (k x n), k = min(m, n); q may be null (R only).  Tall
 * well-conditioned inputs take CholeskyQR2 (certified: pivot breakdown or
 * ||Q1^T Q1 - I||_F > 1/4 falls back), everything else blocked Householder
 * (single-CTA kernel below 64 columns, cluster panels + compact-WY above). */
int qtt_qr(int64_t m, int64_t n, const double* a, int64_t lda, double* q,
           int64_t ldq, double* r, int64_t ldr, void* stream);
/* Singular values (descending) and left singular vectors (u, m x min(m,n))
 * of a column-major m x n matrix via QR + one-sided Jacobi. */
int qtt_svd(int64_t m, int64_t n, const double* a, int64_t lda, double* s,
            double* u, int64_t ldu, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QTT_B200_H_ */
