/*
 * mpeig_b200.h -- C ABI of the B200-native (sm_100a) LOBPCG / PINVIT hot path.
 *
 * Drop-in boundary for the reference library `mpeig` (arXiv 2302.12528
 * artifact).  Every entry point cites the reference interface it replaces
 * (paths relative to the reference's proj/ directory).  Plain pointers and
 * sizes only: no C++ or torch types cross this boundary.
 *
 * Memory model: block vectors are column-major (dense_matrix.hpp:38-41)
 * device arrays with a caller-chosen leading dimension.  Host arrays are
 * named *_host.  All work is ordered on the context's CUDA stream.
 *
 * Errors: every function returns an mpeig_status.  Codes 1..8 are 1:1 with
 * the reference exception types thrown on the solver path (errors.hpp:10-62);
 * mpeig_last_error() returns the message and the index payload
 * (NotPositiveDefinite::index, SingularTriangular::index,
 * RankDeficient::column).  Non-convergence within maxit is NOT an error
 * (converged = 0), as in eigensolvers.hpp:248-262.
 */
#ifndef MPEIG_B200_H
#define MPEIG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
typedef enum {
  MPEIG_OK = 0,
  MPEIG_E_DIMENSION = 1,       /* DimensionMismatch      errors.hpp:11   */
  MPEIG_E_CONFIG = 2,          /* ConfigError            errors.hpp:15   */
  MPEIG_E_NOT_PD = 3,          /* NotPositiveDefinite    errors.hpp:24   */
  MPEIG_E_SINGULAR_TRI = 4,    /* SingularTriangular     errors.hpp:30   */
  MPEIG_E_RANK_DEFICIENT = 5,  /* RankDeficient          errors.hpp:36   */
  MPEIG_E_RANK_COLLAPSE = 6,   /* RankCollapse           errors.hpp:46   */
  MPEIG_E_NO_CONVERGENCE = 7,  /* NoConvergence          errors.hpp:50   */
  MPEIG_E_OVERFLOW = 8,        /* OverflowError          errors.hpp:55   */
  MPEIG_E_CALLBACK = 20,       /* a user callback returned nonzero      */
  MPEIG_E_CUDA = 30,
  MPEIG_E_CUSOLVER = 31,
  MPEIG_E_COMM = 32,
  MPEIG_E_OTHER = 99
} mpeig_status;

/* Variant (solver_types.hpp:11) */
typedef enum {
  MPEIG_DLOBPCG_DCHOL = 0,
  MPEIG_DLOBPCG_SCHOL = 1,
  MPEIG_MPLOBPCG_SCHOL = 2,
  MPEIG_PINVIT = 3
} mpeig_variant;

/* Precision (precision.hpp:14) */
typedef enum { MPEIG_WORKING = 0, MPEIG_LOWER = 1 } mpeig_precision;

typedef struct mpeig_ctx mpeig_ctx;
typedef struct mpeig_op mpeig_op;

/* SolverConfig (solver_types.hpp:31-57).  block == 0 picks (3k+1)/2. */
typedef struct {
  int64_t k;
  int64_t block;
  int64_t maxit;
  double tol;
  double lower_tol;
  uint64_t seed;
  int32_t variant;       /* mpeig_variant */
  int64_t sketch_rows;
} mpeig_cfg;

/* StageOptions (eigensolvers.hpp:176-181) */
typedef struct {
  double tol;
  int32_t use_mixed_qr;
  int32_t stagnation_exit;
  int32_t tag;           /* mpeig_precision of the history records */
} mpeig_stage_opts;

/* IterationRecord (solver_types.hpp:59-66); passed to the history sink once
 * per iteration.  Arrays are valid only during the callback. */
typedef struct {
  int32_t stage;         /* mpeig_precision */
  int64_t m;
  const double* ritz_values;
  const double* residual_norms;
  int64_t n_converged;
  int64_t w_columns_dropped;
  int32_t basis_rotation_fallback;
} mpeig_iter_record;
typedef void (*mpeig_history_sink)(void* user, const mpeig_iter_record* rec);

/* StageTimings (solver_types.hpp:68-74), seconds, accumulated */
typedef struct {
  double factorize;
  double precond_apply;
  double orthogonalize;
  double projected_eig;
  double total;
} mpeig_timings;

/* StageOutcome (eigensolvers.hpp:183-190).  X is a caller-owned device
 * buffer (n x m, ld ldx) of the stage's precision; theta / residual_norms
 * are caller-owned host arrays of length m. */
typedef struct {
  void* X;
  int64_t ldx;
  double* theta;
  double* residual_norms;
  int64_t iterations;
  int32_t converged;
} mpeig_stage_out;

/* EigResult (solver_types.hpp:76-88).  Caller-owned host arrays of length k;
 * X optional (device, n x k fp64, ld ldx; NULL to skip). */
typedef struct {
  double* theta;
  double* residual_norms;
  double* X;
  int64_t ldx;
  int64_t iterations_lower;
  int64_t iterations_working;
  int32_t converged;
  double a_norm_estimate;
  mpeig_timings timings;
} mpeig_result;

/* ------------------------------------------------------------- context */
/* One context per (GPU, stream); not thread-safe per context, independent
 * contexts may run concurrently (SPEC.md:526 / SURVEY §8b threading). */
/* cuda_stream NULL: the context creates its own stream and orders every call
 * after earlier, and before later, work on the legacy default stream. */
int mpeig_ctx_create(int device, void* cuda_stream, mpeig_ctx** out);
void mpeig_ctx_destroy(mpeig_ctx* ctx);
/* message of the last failure on this context; *index gets the payload */
const char* mpeig_last_error(mpeig_ctx* ctx, int64_t* index);
/* number of kernels this library launched on ctx since creation / reset */
int64_t mpeig_launch_count(mpeig_ctx* ctx, int reset);
/* device stream the context orders its work on */
void* mpeig_ctx_stream(mpeig_ctx* ctx);
/* execution options (results are bitwise identical across them unless noted):
 *   "spec_mode"   1 (default): one host sync per iteration, breakdowns rolled
 *                 back to the careful path; 0: eager, one sync per decision
 *   "use_graphs"  1 (default): replay the steady-state iteration as a CUDA graph
 *   "eig_backend" 0 (default): one-CTA tridiagonal + QL eigensolver (the
 *                 reference's algorithm) for 3m <= 96, cuSOLVER syevd above;
 *                 1: cuSOLVER syevd always; 2: cuSOLVER syevj (diagnostic)
 *   "spec_qr"     1 (default): the speculative body orthonormalises W by
 *                 Cholesky-QR twice with a conditioning guard (a column with
 *                 < 1e-5 (fp64) / 1e-2 (fp32) of its norm outside the span of
 *                 the columns before it fails the guard and the iteration is
 *                 repeated on the careful path with the reference's QR);
 *                 0: the TSQR-based QR in the speculative body too.  Same
 *                 results to rounding (not bitwise).
 *   "ql_exact"    QL rotation formulas of the one-CTA Rayleigh-Ritz
 *                 eigensolver (-1 default; see syev.cu); per context */
int mpeig_ctx_set_option(mpeig_ctx* ctx, const char* key, int value);
/* speculative iterations this context repeated on the careful path (a
 * breakdown or a failed guard inside the speculative body) */
int64_t mpeig_spec_rollbacks(mpeig_ctx* ctx, int reset);

/* device memory for callers without the CUDA runtime headers (the C++ layer
 * include/mpeig_b200.hpp): allocation on the context's device, and a copy in
 * any direction (cudaMemcpyDefault; unified addressing) ordered on the
 * context's stream and complete on return */
int mpeig_buffer_alloc(mpeig_ctx* ctx, int64_t bytes, void** out);
void mpeig_buffer_free(mpeig_ctx* ctx, void* p);
int mpeig_copy(mpeig_ctx* ctx, void* dst, const void* src, int64_t bytes);

/* -------------------------------------------------------- row sharding */
/* the n x . blocks are row-sharded over the ranks (z-slabs of
 * the stencil).  Per iteration the ranks sum-allreduce the small Gram
 * matrices and column norms, allgather their TSQR R factors, exchange the
 * stencil's boundary planes with the slab neighbours and max-reduce the
 * status words; the Rayleigh-Ritz step and all small factorisations run
 * replicated.  A context attached to a communicator solves its rank's rows.
 * NCCL (one process per GPU; rank 0 creates the id, broadcasts it):        */
int mpeig_nccl_unique_id(void* out, int64_t cap);  /* cap >= 128 bytes */
int mpeig_ctx_attach_nccl(mpeig_ctx* ctx, int rank, int nranks, const void* unique_id);
/* ranks as threads of one process, host-staged sums in rank order (tests) */
int mpeig_host_group_create(int nranks, void** out);
void mpeig_host_group_destroy(void* group);
int mpeig_ctx_attach_host_comm(mpeig_ctx* ctx, void* group, int rank);

/* ------------------------------------------------------------ operators */
/* BlockOperator<T> (dense_kernels.hpp:15-16).  Device callback: Y = op(X),
 * X/Y device column-major n_local x ncols, stream-ordered on `stream`,
 * must not synchronise the device.  Return 0 on success. */
typedef int (*mpeig_apply_fn)(void* user, int64_t n_local, int64_t ncols,
                              const void* X, int64_t ldx, void* Y, int64_t ldy,
                              void* stream);
/* Host BlockOperator adapter: contiguous column-major host arrays (n x ncols).
 * Lets a reference-style CPU callback run unchanged (D2H, call, H2D). */
typedef int (*mpeig_host_apply_fn)(void* user, int64_t n, int64_t ncols,
                                   const void* X_host, void* Y_host);

/* Built-in operators.  Each provides a working (fp64) and a lower (fp32)
 * apply; the lower one uses to_lower() of the coefficients
 * (csr_matrix.hpp:136-146), overflow -> MPEIG_E_OVERFLOW. */
/* 3-D 7-point Dirichlet Laplacian, diag 6 / off -1, row = x + nx(y + ny z),
 * entries summed in ascending column order like spmv_block
 * (sparse_kernels.hpp:16-33) -> bitwise equal to the reference's CSR apply */
int mpeig_op_lap3d(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, mpeig_op** out);
/* this rank's z-slab [z0, z0 + nz_local) of the nx x ny x nz_global 7-point
 * Laplacian (rows row0 = nx ny z0 ...), halo planes exchanged through the
 * context's communicator; sharded rank r must hold slab r in z order */
int mpeig_op_lap3d_slab(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz_global, int64_t z0,
                        int64_t nz_local, mpeig_op** out);
/* the same 7-point stencil with a variable diagonal: H = -Laplacian + V, row
 * i's diagonal diag_host[i] = 6 + V_i (the KS-like cfg5 family; host array of
 * n values), off-diagonals -1, sums in the CSR column order (bitwise the
 * reference's spmv_block on the CSR form) */
int mpeig_op_lap3d_diag(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz,
                        const double* diag_host, mpeig_op** out);
/* this rank's z-slab of the variable-diagonal 7-pt operator; diag_local_host
 * = the slab's n_local diagonal values (rows row0 .. row0 + n_local) */
int mpeig_op_lap3d_slab_diag(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz_global, int64_t z0,
                             int64_t nz_local, const double* diag_local_host, mpeig_op** out);
/* gen_laplace2d (generators.cpp:13-30) applied matrix-free */
int mpeig_op_lap2d(mpeig_ctx* ctx, int64_t nx, int64_t ny, mpeig_op** out);
/* CsrMatrix<double> (csr_matrix.hpp:13-146): int64 row_ptr/col_idx, sorted
 * columns, host arrays (copied to the device) */
int mpeig_op_csr(mpeig_ctx* ctx, int64_t n, const int64_t* row_ptr_host,
                 const int64_t* col_idx_host, const double* vals_host, mpeig_op** out);
/* this rank's row block [row0, row0 + n_local) of an n_global x n_global CSR
 * matrix (row-sharded): row_ptr over the local rows, GLOBAL
 * column indices, sorted per row.  Rank r must hold the r-th contiguous
 * block (collective over the context's communicator: the ranks agree on the
 * partition and on the ghost-row lists, the other ranks' rows this block's
 * entries touch).  Each apply packs the rows the peers need, exchanges them
 * (NCCL send / recv, or host-staged) on a side stream while the rows without
 * ghost entries are computed, then the boundary rows: every row's sum keeps
 * the global column order, bitwise the unsharded apply.  A sharded solve
 * needs every block at least as tall as the search basis is wide (3m). */
int mpeig_op_csr_rows(mpeig_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local,
                      const int64_t* row_ptr_host, const int64_t* col_idx_host,
                      const double* vals_host, mpeig_op** out);
/* dense symmetric n x n, herm_product (dense_kernels.hpp:66-72); host array */
int mpeig_op_dense(mpeig_ctx* ctx, int64_t n, const double* A_host, int64_t lda,
                   mpeig_op** out);
/* user device callbacks (either may be NULL if that precision is unused) */
int mpeig_op_device_callback(mpeig_ctx* ctx, int64_t n, mpeig_apply_fn apply_working,
                             mpeig_apply_fn apply_lower, void* user, mpeig_op** out);
/* user host callbacks (the CPU BlockOperator adapter) */
int mpeig_op_host_callback(mpeig_ctx* ctx, int64_t n, mpeig_host_apply_fn apply_working,
                           mpeig_host_apply_fn apply_lower, void* user, mpeig_op** out);
/* Jacobi preconditioner f_T = diag(A)^-1 built at `precision`
 * (Preconditioner<T>::build, precond.hpp:33-77, with a diagonal factor):
 *   WORKING: apply(R) = R .* dinv                       (fp64)
 *   LOWER:   apply(R) = to_working(to_lower(R) .* dinvf) (precond.hpp:92-100)
 *            apply_lower(R) = R .* dinvf                (precond.hpp:103-109)
 * The solver fuses it with the residual and the conversions (one HBM pass). */
int mpeig_precond_jacobi(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision,
                         mpeig_op** out);
/* Dense Cholesky preconditioner f_T = L^-T L^-1 of an explicit dense operator
 * (Preconditioner<T>::build(DenseMatrix, prec), precond.hpp:33-50; the
 * reference's own preconditioner for dense systems):
 *   WORKING: L = chol(A) in fp64; apply(R) = L^-T L^-1 R        (precond.hpp:98)
 *   LOWER:   L = chol(to_lower(A)) in fp32, on NotPositiveDefinite / Overflow
 *            one retry with A + 10 u_l ||A||_est I (retry_dense, :140-146);
 *            apply(R) = to_working(L^-T L^-1 to_lower(R))        (:99)
 *            apply_lower(R) = L^-T L^-1 R                        (:103-109)
 * A must come from mpeig_op_dense. Errors: MPEIG_E_NOT_PD (index = pivot),
 * MPEIG_E_OVERFLOW, MPEIG_E_SINGULAR_TRI on apply (check_tri_diag). */
int mpeig_precond_dense_chol(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision,
                             mpeig_op** out);
/* Preconditioner::shift_applied() (precond.hpp:114): the retry shift, else 0 */
double mpeig_precond_shift(const mpeig_op* op);
/* Sparse Cholesky preconditioner f_T = Pi L^-T L^-1 Pi^T of a CSR operator
 * (Preconditioner<T>::build(CsrMatrix, prec[, perm]), precond.hpp:55-77):
 * ordering 0 = reverse Cuthill-McKee (rcm_ordering, rcm.cpp:8-57), 1 = identity
 * (the system was permuted upstream, drivers.hpp:195-197), 2 = `perm` (n entries,
 * perm[k] = original index of factored row k).  Up-looking factorisation on the
 * host (sparse_kernels.hpp:92-170): fp64 at WORKING; fp32 of to_lower(A) at LOWER
 * with retry_sparse's one shifted retry (precond.hpp:148-159).  Each apply runs the
 * two triangular sweeps on the device, permutation and lower()/working() fused
 * (sparse_tri_solve, sparse_kernels.hpp:178-225).  A must come from mpeig_op_csr. */
int mpeig_precond_sparse_chol(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision,
                              int32_t ordering, const int64_t* perm, mpeig_op** out);
/* Preconditioner::factor_nnz() (precond.hpp:116-119) */
int64_t mpeig_precond_factor_nnz(const mpeig_op* op);
/* rcm_ordering_pattern (rcm.cpp:8-57), host arrays; perm_out has n entries */
int mpeig_rcm_ordering(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                       int64_t* perm_out);
void mpeig_op_destroy(mpeig_op* op);
int64_t mpeig_op_n(const mpeig_op* op);
/* Y = op(X) in working (fp64) or lower (fp32) precision, device arrays */
int mpeig_op_apply(mpeig_ctx* ctx, const mpeig_op* op, int32_t precision, int64_t ncols,
                   const void* X, int64_t ldx, void* Y, int64_t ldy);

/* ------------------------------------------------------ solver entry points */
/* spectral_norm_estimate (norm_estimate.hpp:15-24): Omega drawn on the host
 * with the reference PCG64/Box-Muller stream (bit-exact), one device apply */
int mpeig_spectral_norm_estimate(mpeig_ctx* ctx, const mpeig_op* A, int64_t sketch_rows,
                                 uint64_t seed, double* out);

/* lobpcg_stage<double> / <float> (eigensolvers.hpp:195-321).  X0 is an
 * orthonormal device block (n x m, ld ldx0) of the stage precision.  The
 * preconditioner T is applied as T.apply (f64) or T.apply_lower (f32). */
int mpeig_lobpcg_stage_f64(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0,
                           int64_t ldx0, int64_t m, const mpeig_cfg* cfg, const mpeig_op* T,
                           double a_norm_est, const mpeig_stage_opts* opt,
                           mpeig_history_sink sink, void* sink_user,
                           mpeig_stage_out* out, mpeig_timings* tim);
int mpeig_lobpcg_stage_f32(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const float* X0,
                           int64_t ldx0, int64_t m, const mpeig_cfg* cfg, const mpeig_op* T,
                           double a_norm_est, const mpeig_stage_opts* opt,
                           mpeig_history_sink sink, void* sink_user,
                           mpeig_stage_out* out, mpeig_timings* tim);

/* pinvit<double> (eigensolvers.hpp:326-390), with the preconditioner as an
 * operator (generalises the reference's concrete Preconditioner<T>&).
 * a_norm_est <= 0 computes the sketch as the reference does. */
int mpeig_pinvit_f64(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0,
                     int64_t ldx0, int64_t m, const mpeig_cfg* cfg, const mpeig_op* T,
                     double a_norm_est, mpeig_history_sink sink, void* sink_user,
                     mpeig_result* out);

/* solve() (drivers.hpp:158-181) + run_variant (drivers.hpp:57-111):
 * sketch, X0 = orthonormal_q(gaussian_matrix(n, m, seed), true), then the
 * variant's stage(s).  T must be built at the variant's precision
 * (DLOBPCG_DCHOL: WORKING, others: LOWER; drivers.hpp:113-116). */
int mpeig_solve(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T, const mpeig_cfg* cfg,
                mpeig_history_sink sink, void* sink_user, mpeig_result* out);

/* solve() from device-resident raw inputs: X0raw = gaussian_matrix(n, m, seed)
 * (NOT yet orthonormal, device n x m) and Omega = gaussian_matrix(n,
 * sketch_rows, seed ^ 0x9e3779b97f4a7c15) (device); omega_fro = ||Omega||_F
 * (<= 0: computed on the device).  Equivalent to mpeig_solve minus the host
 * RNG and uploads; this is the timed region of the benchmark. */
int mpeig_solve_prepared(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T,
                         const mpeig_cfg* cfg, const double* X0raw, int64_t ldx0,
                         const double* omega, int64_t ldo, double omega_fro,
                         mpeig_history_sink sink, void* sink_user, mpeig_result* out);

/* solve(CsrMatrix, cfg) (drivers.hpp:183-210): the reference's stock sparse
 * driver.  One RCM permutation of the system (rcm.cpp:8-57), the sparse
 * Cholesky preconditioner of the permuted system at the variant's precision
 * (Preconditioner::build(As, prec, {}), precond.hpp:59-77, with retry_sparse's
 * shift), the norm sketch and seeded start block on the permuted system, then
 * run_variant; out->X (device, optional) comes back in the ORIGINAL row order
 * (unpermute_rows).  Host CSR arrays, columns sorted per row.  *precond_shift
 * (optional) = P.shift_applied(); out->timings.factorize = the factor time. */
int mpeig_solve_csr(mpeig_ctx* ctx, int64_t n, const int64_t* row_ptr_host,
                    const int64_t* col_idx_host, const double* vals_host, const mpeig_cfg* cfg,
                    mpeig_history_sink sink, void* sink_user, mpeig_result* out,
                    double* precond_shift);

/* run_variant on an explicit start block X0 (device fp64, n x m) with a
 * precomputed norm estimate (drivers.hpp:57-111; mixed_lobpcg :122-152) */
int mpeig_run_variant(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T,
                      const mpeig_cfg* cfg, const double* X0, int64_t ldx0,
                      double a_norm_est, mpeig_history_sink sink, void* sink_user,
                      mpeig_result* out);

/* ----------------------------------------------- kernel-level entry points
 * (used by the parity tests; each mirrors one reference routine) */
/* gaussian_matrix<double> (dense_matrix.hpp:144-161) drawn on the host with
 * the reference stream, written to a host array (rows x cols) */
int mpeig_gaussian_matrix_host(int64_t rows, int64_t cols, uint64_t seed, double* out_host);
/* rows [row0, row0 + rows) of gaussian_matrix<double>(n_global, cols, seed):
 * a row-shard's part of the start block / sketch (rows x cols, column-major) */
int mpeig_gaussian_matrix_rows_host(int64_t n_global, int64_t cols, uint64_t seed, int64_t row0,
                                    int64_t rows, double* out_host);
/* detail::orthonormal_q (eigensolvers.hpp:55-70): mixed_qr with Householder
 * fallback (use_mixed, fp64) or Householder-equivalent QR.  In place on W. */
int mpeig_orthonormal_q_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                            int32_t use_mixed);
int mpeig_orthonormal_q_f32(mpeig_ctx* ctx, int64_t n, int64_t m, float* W, int64_t ldw);
/* mixed_qr (ortho.hpp:173-186, Alg. 2): Q in place on W, R (m x m) to R_out */
int mpeig_mixed_qr_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                       double* R_out);
/* householder_qr (ortho.hpp:127-140) equivalent: unique Q with diag(R) > 0 */
int mpeig_householder_qr_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                             double* R_out);
/* orthonormal_q_dropping (eigensolvers.hpp:74-85): returns kept column count */
int mpeig_orthonormal_q_dropping_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W,
                                     int64_t ldw, int32_t use_mixed, int64_t* kept);
/* G = A^T B (adjoint_matmul, dense_kernels.hpp:36-52); G ka x kb, ld ka */
int mpeig_gram_f64(mpeig_ctx* ctx, int64_t n, int64_t ka, const double* A, int64_t lda,
                   int64_t kb, const double* B, int64_t ldb, double* G);
/* Y = beta Z + alpha A C (matmul, dense_kernels.hpp:20-34) */
int mpeig_gemm_f64(mpeig_ctx* ctx, int64_t n, int64_t k, int64_t c, double alpha,
                   const double* A, int64_t lda, const double* Cm, int64_t ldc, double beta,
                   const double* Z, int64_t ldz, double* Y, int64_t ldy);
/* Process-wide kernel-selection knobs (diagnostics and tests; NOT per
 * context -- set them before any solve runs):
 *   "gram_tc" / "gemm_tc" / "tc" (both): the binary32 Gram / block update
 *              on the tcgen05 tensor cores (exact 3-way bf16 split, fp32
 *              accumulation): 1 = for products with n * k * c >= 2^28
 *              (default), 0 = never (SIMT FFMA kernels), 2 = always.
 *   "gram_tma":  TMA-fed tensor-core Gram (1, default) or the cp.async one (0).
 *   "gemm_tma2": tensor-core block update with C split once per call (1,
 *              default) or the per-tile split (0; in place only c <= 128).
 *   "pdl":      programmatic kernel -> kernel edges in the captured iteration
 *              graphs (1, default; 0 = ordinary edges; bitwise identical).
 *   "spchol_threads": host threads of the sparse-Cholesky factorisation (0 =
 *              the hardware's, capped at 32; the factor is bitwise the same
 *              for any count).
 * Diagnostics of the tensor-core kernels (results change with "tc_nprod",
 * "tc_twoacc" and "tc_ablate"; never set them for a real solve):
 *   "tc_nprod" part products (8), "tc_twoacc" second accumulator (1),
 *   "tc_stage" staged TMA-store epilogue (1), "g2_depth" ring depths as RSD
 *   digits (0 = by shared memory), "tc_ablate" bit mask that removes data
 *   paths (1 C copies / loads, 2 split, 4 stores, 8 A loads, 16 TMEM drain;
 *   bits 16+: CTA cap) to find what bounds a kernel. */
int mpeig_set_process_option(const char* key, int value);
/* the same two products in binary32 (the lower-precision stage's kernels) */
int mpeig_gram_f32(mpeig_ctx* ctx, int64_t n, int64_t ka, const float* A, int64_t lda,
                   int64_t kb, const float* B, int64_t ldb, float* G);
int mpeig_gemm_f32(mpeig_ctx* ctx, int64_t n, int64_t k, int64_t c, float alpha,
                   const float* A, int64_t lda, const float* Cm, int64_t ldc, float beta,
                   const float* Z, int64_t ldz, float* Y, int64_t ldy);
/* block_project_out (ortho.hpp:190-200): W -= B (B^T W), `passes` times */
int mpeig_project_out_f64(mpeig_ctx* ctx, int64_t n, int64_t b, const double* B,
                          int64_t ldb, int64_t w, double* W, int64_t ldw, int32_t passes);
/* small_herm_eig (small_eig.hpp:92-218) on device: the reference's Householder
 * tridiagonalisation + implicit QL (k_small_ql3) for s <= 96, cuSOLVER syevd above:
 * M device s x s, values (device, ascending), vectors (device s x s) */
int mpeig_small_eig_f64(mpeig_ctx* ctx, int64_t s, const double* M, double* values,
                        double* vectors);
/* hl_update (eigensolvers.hpp:148-174): coefficient block [c_x c_pv]
 * (device s x (m+p), ld s) from eigenvectors C (device s x s); returns p
 * and the rotation-fallback flag */
int mpeig_hl_coeffs_f64(mpeig_ctx* ctx, int64_t s, int64_t m, const double* C,
                        double* coef, int64_t* p, int32_t* fallback);
/* residual_block + column norms + f_T (eigensolvers.hpp:104-129,
 * precond.hpp:92-100) fused: W = T(AX - X diag(theta)); norms to host */
int mpeig_residual_precond_f64(mpeig_ctx* ctx, const mpeig_op* T, int64_t n, int64_t m,
                               const double* X, int64_t ldx, const double* AX,
                               int64_t ldax, const double* theta_host, double* W,
                               int64_t ldw, double* rnorm_host, double* xnorm_host);

/* ------------------------------------------------------ instrumentation
 * Per-kernel-class CUDA-event timing (off by default): every launch of a
 * class is bracketed by events on its stream and its algorithmic bytes and
 * flops are recorded.  Used by bench.py for the roofline figures. */
void mpeig_profile_enable(int on);
void mpeig_profile_reset(void);
int mpeig_profile_names(char* buf, int64_t cap);
int mpeig_profile_query(const char* name, int64_t* count, double* ms, double* bytes,
                        double* flops);

#ifdef __cplusplus
}
#endif
#endif /* MPEIG_B200_H */
