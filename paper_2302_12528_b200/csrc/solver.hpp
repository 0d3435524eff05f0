// solver.hpp -- internal declarations of the device LOBPCG / PINVIT drivers.
#pragma once

#include <vector>

#include "context.hpp"

namespace mpb {

// Per-stage device workspace.  S/AS (and the ping-pong S2/AS2) hold up to
// smax = 3m columns with leading dimension ld = padded_ld(n).
template <typename T>
struct Work {
  mpeig_ctx* ctx;
  cudaStream_t s;
  int64_t n, ld, m, smax;
  DevBuf<T> S, AS, S2, AS2;
  DevBuf<T> V;        // n x m scratch (QR V, plain residual R)
  DevBuf<T> G;        // smax x smax Gram / projected matrix / eigenvectors
  DevBuf<T> evals;    // smax
  DevBuf<T> coef;     // smax x (m + p) HL coefficients
  DevBuf<T> small;    // m x m factors + HL scratch
  DevBuf<float> smallf;
  DevBuf<T> gramw;    // split-n Gram partials
  DevBuf<T> tsqr_w;   // TSQR tree in T
  DevBuf<float> tsqr_f;  // TSQR tree in fp32 (mixed_qr)
  DevBuf<double> rw;  // residual partials + norms
  DevBuf<T> theta;    // current Ritz values (device)
  DevBuf<T> theta_prev;  // Ritz values before the last speculative update
  DevBuf<T> eigw;
  int lwork = 0;
  // row-sharded mode: gathered per-rank R factors, stacked, and the TSQR
  // workspace of the (nranks m) x m stack
  DevBuf<T> rstk, rstk2, tsqr_w2;
  DevBuf<float> rstkf, rstk2f, tsqr_f2;

  Work(mpeig_ctx* c, int64_t n_, int64_t m_, int64_t smax_);
  T* L();
  T* Uinv();
  T* Rw();
  T* Rinv();
  T* Lt();
  T* scratch();
  double* rnorm();
  double* xnorm();
  double* dscal();
};

struct StageResult {
  std::vector<double> theta, resid;
  int64_t iterations = 0;
  bool converged = false;
};

template <typename T>
void precond_apply(mpeig_ctx* ctx, const mpeig_op* T_op, int64_t ncols, const T* R, int64_t ldr,
                   T* W, int64_t ldw);
template <typename T>
void small_eig(Work<T>& w, int64_t sdim, T* G, int64_t ldg, T* vals);
template <typename T>
void orthonormal_q(Work<T>& w, int64_t m, T* W, int64_t ldw, bool use_mixed);
template <typename T>
int64_t orthonormal_q_dropping(Work<T>& w, int64_t m, T* W, int64_t ldw, bool use_mixed,
                               int64_t* dropped, bool second = false);
template <typename T>
void project_out(Work<T>& w, const T* B, int64_t b, int64_t ldb, T* W, int64_t wc, int64_t ldw,
                 int passes);
int qr_with_r(Work<double>& w, int64_t m, double* W, int64_t ldw, bool lower, double* Rout,
              int64_t* idx);

template <typename T>
StageResult lobpcg_stage(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const T* X0, int64_t ldx0,
                         int64_t m, const mpeig_cfg& cfg, const mpeig_op* T_op, double a_norm_est,
                         const mpeig_stage_opts& opt, mpeig_history_sink sink, void* sink_user,
                         T* Xout, int64_t ldxout, mpeig_timings* tim);
StageResult pinvit(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0, int64_t ldx0,
                   int64_t m, const mpeig_cfg& cfg, const mpeig_op* T_op, double a_norm_est,
                   mpeig_history_sink sink, void* sink_user, double* Xout, int64_t ldxout,
                   mpeig_timings* tim);
double spectral_norm_estimate(mpeig_ctx* ctx, const mpeig_op* A, int64_t sketch_rows,
                              uint64_t seed);
void run_variant(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
                 const double* X0, int64_t ldx0, double a_norm_est, mpeig_history_sink sink,
                 void* sink_user, mpeig_result* out);
void solve(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
           mpeig_history_sink sink, void* sink_user, mpeig_result* out);
void solve_prepared(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
                    const double* X0raw, int64_t ldx0, const double* omega, int64_t ldo,
                    double omega_fro, mpeig_history_sink sink, void* sink_user, mpeig_result* out);
// Preconditioner<T>::build(DenseMatrix, prec) (precond.hpp:33-50): fills op (kOpDenseChol)
void dense_chol_build(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, mpeig_op* op);
// Preconditioner<T>::build(CsrMatrix, prec[, perm]) (precond.hpp:55-77): fills op (kOpSparseChol)
// ordering: 0 = RCM (rcm_ordering), 1 = identity, 2 = `perm`
void sparse_chol_build(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, int32_t ordering,
                       const int64_t* perm, mpeig_op* op);
void validate_cfg(const mpeig_cfg& cfg, int64_t n);

}  // namespace mpb
