/*
 * mp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Common C ABI of the two CPU checkers used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs:
 *
 *   mpref_*  oracle/_ref/libmpeig_ref.so  -- the UNMODIFIED reference library
 *            (/root/reference/proj headers + src/rng.cpp, src/generators.cpp),
 *            driven through its own lobpcg_stage / BlockOperator callbacks by
 *            oracle/ref_harness.cpp (recipe: oracle/Makefile).
 *   mporc_*  oracle/liboracle.so -- oracle/mp_oracle.c, a plain-C restatement
 *            of the reference algorithm, pinned against mpref_* and the
 *            reference's golden vectors (tests/test_oracle.py).
 *
 * Nothing in the product (paper_2302_12528_b200/) includes, links or calls
 * anything declared here.
 */
#ifndef MP_ORACLE_H
#define MP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variant ids follow mpeig::Variant (solver_types.hpp:11). */
enum { MP_DLOBPCG_DCHOL = 0, MP_DLOBPCG_SCHOL = 1, MP_MPLOBPCG_SCHOL = 2, MP_PINVIT = 3 };

/* Problem kinds. Matrix-defined problems are materialised as CSR with
 * sorted columns (csr_matrix.hpp:31-58) so both checkers see the same bytes. */
enum { MP_PROB_LAP3D = 0, MP_PROB_LAP2D = 1, MP_PROB_CSR = 2, MP_PROB_DENSE = 3 };

typedef struct {
  int32_t kind;
  int64_t nx, ny, nz;          /* grid sides for LAP3D / LAP2D           */
  int64_t n;                   /* order (CSR / DENSE)                      */
  const int64_t* row_ptr;      /* CSR, n+1                                 */
  const int64_t* col_idx;      /* CSR, nnz, sorted per row                 */
  const double* vals;          /* CSR, nnz                                 */
  const double* dense;         /* DENSE, n*n column-major                  */
} mp_problem;

/* SolverConfig (solver_types.hpp:31-57). block == 0 picks (3k+1)/2. */
typedef struct {
  int64_t k, block, maxit;
  double tol, lower_tol;
  uint64_t seed;
  int64_t sketch_rows;
  /* optional: the n x m start block before orthonormal_q (column-major),
   * replacing gaussian_matrix(n, m, seed) -- used to measure the reference's
   * iteration-count envelope under 1-ulp perturbations of X0 */
  const double* x0;
} mp_cfg;

/* Output of one solve. Caller owns every array; capacities in *_cap. */
typedef struct {
  int32_t converged;
  int32_t status;              /* 0 ok, else an MP_E* code (below)         */
  int64_t iters_lower, iters_working;
  double a_norm_est;
  double* theta;               /* k                                        */
  double* resid;               /* k                                        */
  double* X;                   /* n*k column-major, or NULL                */
  int64_t hist_cap, hist_len;  /* IterationRecord sink (solver_types:59)   */
  int32_t* hist_stage;         /* 0 working, 1 lower                       */
  int64_t* hist_nc;
  int64_t* hist_dropped;
  int32_t* hist_fallback;
  double* hist_ritz;           /* hist_cap*m                               */
  double* hist_resid;          /* hist_cap*m                               */
  double t_total;              /* seconds inside the solve                 */
  double t_setup;              /* norm sketch + initial QR                 */
  double t_stage1;             /* fp32 stage + hand-off QR (mixed only)    */
  char msg[256];
} mp_result;

/* Error codes 1:1 with errors.hpp types used on the solver path. */
enum {
  MP_OK = 0, MP_E_DIMENSION = 1, MP_E_CONFIG = 2, MP_E_NOT_PD = 3,
  MP_E_SINGULAR_TRI = 4, MP_E_RANK_DEFICIENT = 5, MP_E_RANK_COLLAPSE = 6,
  MP_E_NO_CONVERGENCE = 7, MP_E_OVERFLOW = 8, MP_E_OTHER = 99
};

#define MP_ORACLE_DECLS(P)                                                          \
  int P##solve(const mp_problem* prob, int variant, const mp_cfg* cfg,              \
               mp_result* out);                                                     \
  void P##pcg64_u64(uint64_t seed, int64_t count, uint64_t* out);                   \
  void P##gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out);         \
  double P##norm_estimate(const mp_problem* prob, int64_t sketch_rows,             \
                          uint64_t seed);                                           \
  int P##householder_qr(int64_t n, int64_t m, const double* A, double* Q,           \
                        double* R);                                                 \
  int P##householder_qr_f32(int64_t n, int64_t m, const float* A, float* Q,         \
                            float* R);                                              \
  int P##mixed_qr(int64_t n, int64_t m, const double* A, double* Q, double* R);     \
  int P##cholesky_qr(int64_t n, int64_t m, const double* A, double* Q,              \
                     double* R);                                                    \
  int P##small_herm_eig(int64_t n, const double* M, double* vals, double* vecs);    \
  int P##hl_update(int64_t n, int64_t s, int64_t m, const double* S,                \
                   const double* C, double* X, double* P, double* c_pv,             \
                   int32_t* fallback);                                              \
  void P##project_out(int64_t n, int64_t b, int64_t w, const double* B,             \
                      double* W, int passes);                                       \
  int64_t P##ortho_dropping(int64_t n, int64_t w, const double* W, double tol,     \
                            double* Q);                                             \
  void P##apply_op(const mp_problem* prob, int64_t ncols, const double* X,          \
                   double* Y);                                                      \
  int64_t P##converged_count(int64_t n, int64_t m, double a_norm_est,               \
                             const double* X, const double* theta,                  \
                             const double* R, double tol);

MP_ORACLE_DECLS(mpref_)
MP_ORACLE_DECLS(mporc_)

#ifdef __cplusplus
}
#endif
#endif
