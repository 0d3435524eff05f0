// mpeig_b200.hpp -- the reference's C++ solver entry points on the B200 path.
//
// A header-only layer over the C ABI of libmpeig_b200.so (mpeig_b200.h) that
// restores the signatures of the reference library `mpeig` (proj/include/mpeig)
// with its own types (DenseMatrix, CsrMatrix, SolverConfig, StageOptions,
// StageOutcome, EigResult, IterationRecord, StageTimings, Preconditioner,
// BlockOperator) and its own exception types.  A maintainer switches a call
// site by qualifying it:
//
//     mpeig::lobpcg_stage<double>(...)   ->  mpeig::b200::lobpcg_stage<double>(...)
//     mpeig::solve(A, cfg)               ->  mpeig::b200::solve(A, cfg)
//
// Include after the reference's headers; link -lmpeig_b200 (no CUDA headers
// or runtime flags needed: device memory goes through mpeig_buffer_* /
// mpeig_copy).  Replaced interfaces (reference file:line):
//
//   lobpcg_stage<T>           eigensolvers.hpp:195-321  -> mpeig_lobpcg_stage_f64 / _f32
//   pinvit<T>                 eigensolvers.hpp:326-390  -> mpeig_pinvit_f64
//   mixed_lobpcg(Dense/Csr)   drivers.hpp:122-152       -> mpeig_run_variant
//   solve(DenseMatrix)        drivers.hpp:158-181       -> mpeig_solve
//   solve(CsrMatrix)          drivers.hpp:183-210       -> mpeig_solve_csr
//   spectral_norm_estimate<T> norm_estimate.hpp:15-24   -> mpeig_spectral_norm_estimate
//   BlockOperator<T>          dense_kernels.hpp:15-16   -> mpeig_op_host_callback
//   Preconditioner<T>         precond.hpp:24-130        -> host callback of P.apply /
//                                                         P.apply_lower, or the device
//                                                         factors (mpeig_precond_*)
//   errors                    errors.hpp:10-62          -> MPEIG_E_* rethrown as the same types
//
// Operators passed as BlockOperator run on the host through the adapter
// (D2H, call, H2D per apply) so reference callbacks work unchanged; the
// matrix overloads (solve, mixed_lobpcg) keep A·X and the preconditioner on
// the device.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <initializer_list>
#include <limits>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <mpeig/drivers.hpp>
#include <mpeig/eigensolvers.hpp>

#include "mpeig_b200.h"

namespace mpeig::b200 {

// ------------------------------------------------------------------ errors
// MPEIG_E_* -> the reference's exception types (errors.hpp:10-62), with the
// index payload where the reference carries one.
[[noreturn]] inline void throw_status(mpeig_ctx* ctx, int rc) {
  int64_t idx = -1;
  const char* m = ctx ? mpeig_last_error(ctx, &idx) : "mpeig_b200: context creation failed";
  const std::string msg = m ? m : "";
  const std::size_t at = idx < 0 ? 0 : static_cast<std::size_t>(idx);
  switch (rc) {
    case MPEIG_E_DIMENSION: throw DimensionMismatch(msg);
    case MPEIG_E_CONFIG: throw ConfigError(msg);
    case MPEIG_E_NOT_PD: throw NotPositiveDefinite(at, msg);
    case MPEIG_E_SINGULAR_TRI: throw SingularTriangular(at, msg);
    case MPEIG_E_RANK_DEFICIENT: throw RankDeficient(at, msg);
    case MPEIG_E_RANK_COLLAPSE: throw RankCollapse(msg);
    case MPEIG_E_NO_CONVERGENCE: throw NoConvergence(msg);
    case MPEIG_E_OVERFLOW: throw OverflowError(msg);
    default: throw std::runtime_error("mpeig_b200 (" + std::to_string(rc) + "): " + msg);
  }
}

inline void check(mpeig_ctx* ctx, int rc) {
  if (rc != MPEIG_OK) throw_status(ctx, rc);
}

// ----------------------------------------------------------------- context
// One device context per thread (the reference runs one solve per thread,
// SPEC.md:526); device 0 unless set_device() is called before the first use.
class Context {
 public:
  explicit Context(int device = 0) {
    mpeig_ctx* c = nullptr;
    const int rc = mpeig_ctx_create(device, nullptr, &c);
    if (rc != MPEIG_OK) throw_status(nullptr, rc);
    h_ = c;
  }
  ~Context() { mpeig_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mpeig_ctx* get() const { return h_; }

 private:
  mpeig_ctx* h_ = nullptr;
};

inline int& thread_device() {
  static thread_local int dev = 0;
  return dev;
}
inline void set_device(int device) { thread_device() = device; }
inline mpeig_ctx* ctx() {
  static thread_local Context c(thread_device());
  return c.get();
}

// -------------------------------------------------------- RAII helpers
struct Op {
  mpeig_op* p = nullptr;
  Op() = default;
  Op(const Op&) = delete;
  Op& operator=(const Op&) = delete;
  ~Op() { mpeig_op_destroy(p); }
};

template <class T>
struct DeviceBlock {  // n x c, column-major, ld = n
  void* p = nullptr;
  std::size_t n = 0, c = 0;
  DeviceBlock(std::size_t rows, std::size_t cols) : n(rows), c(cols) {
    check(ctx(), mpeig_buffer_alloc(ctx(), static_cast<int64_t>(sizeof(T) * n * c), &p));
  }
  explicit DeviceBlock(const DenseMatrix<T>& M) : DeviceBlock(M.rows(), M.cols()) {
    check(ctx(), mpeig_copy(ctx(), p, M.data().data(), static_cast<int64_t>(sizeof(T) * n * c)));
  }
  DeviceBlock(const DeviceBlock&) = delete;
  DeviceBlock& operator=(const DeviceBlock&) = delete;
  ~DeviceBlock() { mpeig_buffer_free(ctx(), p); }
  DenseMatrix<T> download(std::size_t cols) const {
    DenseMatrix<T> M(n, cols);
    check(ctx(), mpeig_copy(ctx(), M.data().data(), p, static_cast<int64_t>(sizeof(T) * n * cols)));
    return M;
  }
};

// BlockOperator<T> -> mpeig_host_apply_fn: contiguous n x c column-major host
// arrays in and out; an exception inside the callback aborts the stage
// (MPEIG_E_CALLBACK) and is rethrown by the caller below.
struct CallbackState {
  const void* op = nullptr;
  std::exception_ptr error;
};

template <class T>
inline int host_apply(void* user, int64_t n, int64_t c, const void* X, void* Y) {
  auto* st = static_cast<CallbackState*>(user);
  try {
    const auto& op = *static_cast<const BlockOperator<T>*>(st->op);
    DenseMatrix<T> in(static_cast<std::size_t>(n), static_cast<std::size_t>(c));
    std::memcpy(in.data().data(), X, sizeof(T) * static_cast<std::size_t>(n * c));
    const DenseMatrix<T> out = op(in);
    if (out.rows() != static_cast<std::size_t>(n) || out.cols() != static_cast<std::size_t>(c))
      throw DimensionMismatch("BlockOperator returned a block of the wrong shape");
    std::memcpy(Y, out.data().data(), sizeof(T) * static_cast<std::size_t>(n * c));
    return 0;
  } catch (...) {
    st->error = std::current_exception();
    return 1;
  }
}

template <class T>
inline void make_host_op(const BlockOperator<T>& f, std::size_t n, CallbackState& st, Op& op) {
  st.op = &f;
  if constexpr (sizeof(real_t<T>) == 8)
    check(ctx(), mpeig_op_host_callback(ctx(), static_cast<int64_t>(n), &host_apply<T>, nullptr,
                                        &st, &op.p));
  else
    check(ctx(), mpeig_op_host_callback(ctx(), static_cast<int64_t>(n), nullptr, &host_apply<T>,
                                        &st, &op.p));
}

inline void rethrow_callbacks(int rc, std::initializer_list<const CallbackState*> states) {
  if (rc == MPEIG_OK) return;
  for (const CallbackState* s : states)
    if (s && s->error) std::rethrow_exception(s->error);
  throw_status(ctx(), rc);
}

inline mpeig_cfg to_c(const SolverConfig& cfg) {
  mpeig_cfg c{};
  c.k = static_cast<int64_t>(cfg.k);
  c.block = static_cast<int64_t>(cfg.block);
  c.maxit = static_cast<int64_t>(cfg.maxit);
  c.tol = cfg.tol;
  c.lower_tol = cfg.lower_tol;
  c.seed = cfg.seed;
  c.variant = static_cast<int32_t>(cfg.variant);
  c.sketch_rows = static_cast<int64_t>(cfg.sketch_rows);
  return c;
}

// the history sink: one IterationRecord per call (solver_types.hpp:59-66)
inline void push_record(void* user, const mpeig_iter_record* r) {
  auto& h = *static_cast<std::vector<IterationRecord>*>(user);
  IterationRecord rec;
  rec.stage = r->stage == MPEIG_LOWER ? Precision::Lower : Precision::Working;
  rec.ritz_values.assign(r->ritz_values, r->ritz_values + r->m);
  rec.residual_norms.assign(r->residual_norms, r->residual_norms + r->m);
  rec.n_converged = static_cast<std::size_t>(r->n_converged);
  rec.w_columns_dropped = static_cast<std::size_t>(r->w_columns_dropped);
  rec.basis_rotation_fallback = r->basis_rotation_fallback != 0;
  h.push_back(std::move(rec));
}

inline void add_timings(StageTimings& t, const mpeig_timings& c) {
  t.factorize += c.factorize;
  t.precond_apply += c.precond_apply;
  t.orthogonalize += c.orthogonalize;
  t.projected_eig += c.projected_eig;
}

// ----------------------------------------------------------- entry points
// lobpcg_stage<T> (eigensolvers.hpp:195-201): same arguments, same outcome;
// history appended and timings accumulated by reference.
template <class T>
StageOutcome<T> lobpcg_stage(const BlockOperator<T>& apply_A, std::size_t n,
                             const DenseMatrix<T>& X0, const SolverConfig& cfg,
                             const BlockOperator<T>& apply_precond, double a_norm_est,
                             const StageOptions& opt, std::vector<IterationRecord>& history,
                             StageTimings& tim) {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>,
                "mpeig::b200::lobpcg_stage: real double / float only");
  if (X0.rows() != n) throw DimensionMismatch("lobpcg_stage: X0 has wrong rows");
  const std::size_t m = X0.cols();
  CallbackState sa, st;
  Op A, P;
  make_host_op<T>(apply_A, n, sa, A);
  make_host_op<T>(apply_precond, n, st, P);
  DeviceBlock<T> dX0(X0), dX(n, m);
  const mpeig_cfg c = to_c(cfg);
  mpeig_stage_opts o{};
  o.tol = opt.tol;
  o.use_mixed_qr = opt.use_mixed_qr ? 1 : 0;
  o.stagnation_exit = opt.stagnation_exit ? 1 : 0;
  o.tag = opt.tag == Precision::Lower ? MPEIG_LOWER : MPEIG_WORKING;
  std::vector<double> theta(m), resid(m);
  mpeig_stage_out so{};
  so.X = dX.p;
  so.ldx = static_cast<int64_t>(n);
  so.theta = theta.data();
  so.residual_norms = resid.data();
  mpeig_timings t{};
  int rc;
  if constexpr (std::is_same_v<T, double>)
    rc = mpeig_lobpcg_stage_f64(ctx(), A.p, static_cast<int64_t>(n),
                                static_cast<const double*>(dX0.p), static_cast<int64_t>(n),
                                static_cast<int64_t>(m), &c, P.p, a_norm_est, &o, &push_record,
                                &history, &so, &t);
  else
    rc = mpeig_lobpcg_stage_f32(ctx(), A.p, static_cast<int64_t>(n),
                                static_cast<const float*>(dX0.p), static_cast<int64_t>(n),
                                static_cast<int64_t>(m), &c, P.p, a_norm_est, &o, &push_record,
                                &history, &so, &t);
  rethrow_callbacks(rc, {&sa, &st});
  add_timings(tim, t);
  StageOutcome<T> out;
  out.X = dX.download(m);
  out.theta.assign(theta.begin(), theta.end());
  out.residual_norms.assign(resid.begin(), resid.end());
  out.iterations = static_cast<std::size_t>(so.iterations);
  out.converged = so.converged != 0;
  return out;
}

// spectral_norm_estimate<T> (norm_estimate.hpp:15-24)
template <class T>
double spectral_norm_estimate(const BlockOperator<T>& apply_A, std::size_t n,
                              std::size_t sketch_rows, std::uint64_t seed) {
  static_assert(std::is_same_v<T, double>, "mpeig::b200::spectral_norm_estimate: double only");
  if (sketch_rows < 1) throw ConfigError("spectral_norm_estimate: sketch_rows < 1");
  CallbackState sa;
  Op A;
  make_host_op<T>(apply_A, n, sa, A);
  double est = 0;
  rethrow_callbacks(mpeig_spectral_norm_estimate(ctx(), A.p, static_cast<int64_t>(sketch_rows),
                                                 seed, &est),
                    {&sa});
  return est;
}

namespace detail {

inline EigResult<double> finish(const mpeig_result& r, std::vector<double>& theta,
                                std::vector<double>& resid, DeviceBlock<double>* X,
                                std::size_t k, std::vector<IterationRecord>&& hist) {
  EigResult<double> out;
  out.theta = theta;
  out.residual_norms = resid;
  if (X) out.X = X->download(k);
  out.iterations_lower = static_cast<std::size_t>(r.iterations_lower);
  out.iterations_working = static_cast<std::size_t>(r.iterations_working);
  out.history = std::move(hist);
  out.converged = r.converged != 0;
  out.timings.factorize = r.timings.factorize;
  out.timings.precond_apply = r.timings.precond_apply;
  out.timings.orthogonalize = r.timings.orthogonalize;
  out.timings.projected_eig = r.timings.projected_eig;
  out.timings.total = r.timings.total;
  out.a_norm_estimate = r.a_norm_estimate;
  return out;
}

struct ResultBuffers {
  std::vector<double> theta, resid;
  DeviceBlock<double> X;
  std::vector<IterationRecord> hist;
  mpeig_result r{};
  ResultBuffers(std::size_t n, std::size_t k) : theta(k), resid(k), X(n, k) {
    r.theta = theta.data();
    r.residual_norms = resid.data();
    r.X = static_cast<double*>(X.p);
    r.ldx = static_cast<int64_t>(n);
  }
  EigResult<double> take(std::size_t k) { return finish(r, theta, resid, &X, k, std::move(hist)); }
};

inline void dense_op(const DenseMatrix<double>& A, Op& op) {
  if (A.rows() != A.cols()) throw DimensionMismatch("herm_product: A not square");
  check(ctx(), mpeig_op_dense(ctx(), static_cast<int64_t>(A.rows()), A.data().data(),
                              static_cast<int64_t>(A.rows()), &op.p));
}

inline void csr_op(const CsrMatrix<double>& A, Op& op) {
  check(ctx(), mpeig_op_csr(ctx(), static_cast<int64_t>(A.n()), A.row_ptr().data(),
                            A.col_idx().data(), A.values().data(), &op.p));
}

inline int32_t build_precision(Variant v) {
  return v == Variant::DLOBPCG_dchol ? MPEIG_WORKING : MPEIG_LOWER;  // drivers.hpp:113-116
}

template <class Clock = std::chrono::steady_clock>
inline double since(typename Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// mixed_lobpcg body (drivers.hpp:122-152): factor at LOWER, sketch, run_variant on X0
inline EigResult<double> mixed_on_device(const Op& A, bool sparse, const DenseMatrix<double>& X0,
                                         SolverConfig cfg) {
  cfg.variant = Variant::MPLOBPCG_schol;
  const std::size_t n = static_cast<std::size_t>(mpeig_op_n(A.p));
  cfg.validate(n);
  if (X0.rows() != n || X0.cols() != cfg.block_size())
    throw DimensionMismatch("mixed_lobpcg: X0 must be n x block_size");
  const auto t0 = std::chrono::steady_clock::now();
  Op P;
  if (sparse)
    check(ctx(), mpeig_precond_sparse_chol(ctx(), A.p, MPEIG_LOWER, 0, nullptr, &P.p));
  else
    check(ctx(), mpeig_precond_dense_chol(ctx(), A.p, MPEIG_LOWER, &P.p));
  const double t_factor = since(t0);
  double est = 0;
  check(ctx(), mpeig_spectral_norm_estimate(ctx(), A.p, static_cast<int64_t>(cfg.sketch_rows),
                                            cfg.seed ^ 0x9e3779b97f4a7c15ULL, &est));
  DeviceBlock<double> dX0(X0);
  ResultBuffers b(n, cfg.k);
  const mpeig_cfg c = to_c(cfg);
  check(ctx(), mpeig_run_variant(ctx(), A.p, P.p, &c, static_cast<const double*>(dX0.p),
                                 static_cast<int64_t>(n), est, &push_record, &b.hist, &b.r));
  EigResult<double> out = b.take(cfg.k);
  out.timings.factorize = t_factor;
  out.precond_shift = mpeig_precond_shift(P.p);
  return out;
}

}  // namespace detail

// pinvit<T> (eigensolvers.hpp:326-390) with the reference's Preconditioner<T>
// applied on the host (P.apply); a_norm_est <= 0 -> sketched on the device.
template <class T>
EigResult<T> pinvit(const BlockOperator<T>& apply_A, std::size_t n, const DenseMatrix<T>& X0,
                    const SolverConfig& cfg, const Preconditioner<T>& P, double a_norm_est = 0) {
  static_assert(std::is_same_v<T, double>, "pinvit iterates at working precision (double)");
  cfg.validate(n);
  if (X0.rows() != n) throw DimensionMismatch("pinvit: X0 has wrong rows");
  const BlockOperator<T> apply_P = [&P](const DenseMatrix<T>& R) { return P.apply(R); };
  CallbackState sa, sp;
  Op A, T_op;
  make_host_op<T>(apply_A, n, sa, A);
  make_host_op<T>(apply_P, n, sp, T_op);
  DeviceBlock<double> dX0(X0);
  detail::ResultBuffers b(n, cfg.k);
  const mpeig_cfg c = to_c(cfg);
  const int rc = mpeig_pinvit_f64(ctx(), A.p, static_cast<int64_t>(n),
                                  static_cast<const double*>(dX0.p), static_cast<int64_t>(n),
                                  static_cast<int64_t>(X0.cols()), &c, T_op.p, a_norm_est,
                                  &push_record, &b.hist, &b.r);
  rethrow_callbacks(rc, {&sa, &sp});
  EigResult<T> out = b.take(cfg.k);
  out.precond_shift = P.shift_applied();
  return out;
}

// mixed_lobpcg (drivers.hpp:122-152): A and its fp32 Cholesky preconditioner on the device
template <class T>
EigResult<T> mixed_lobpcg(const DenseMatrix<T>& A, const DenseMatrix<T>& X0, SolverConfig cfg) {
  static_assert(std::is_same_v<T, double>, "mixed_lobpcg: real double systems");
  Op op;
  detail::dense_op(A, op);
  return detail::mixed_on_device(op, false, X0, cfg);
}

template <class T>
EigResult<T> mixed_lobpcg(const CsrMatrix<T>& A, const DenseMatrix<T>& X0, SolverConfig cfg) {
  static_assert(std::is_same_v<T, double>, "mixed_lobpcg: real double systems");
  Op op;
  detail::csr_op(A, op);
  return detail::mixed_on_device(op, true, X0, cfg);
}

// solve(DenseMatrix, cfg) (drivers.hpp:158-181): Preconditioner::build at the
// variant's precision, sketch, seeded start block, run_variant
template <class T>
EigResult<T> solve(const DenseMatrix<T>& A, const SolverConfig& cfg) {
  static_assert(std::is_same_v<T, double>, "solve: real double systems");
  const std::size_t n = A.rows();
  cfg.validate(n);
  Op op, P;
  detail::dense_op(A, op);
  const auto t0 = std::chrono::steady_clock::now();
  check(ctx(), mpeig_precond_dense_chol(ctx(), op.p, detail::build_precision(cfg.variant), &P.p));
  const double t_factor = detail::since(t0);
  detail::ResultBuffers b(n, cfg.k);
  const mpeig_cfg c = to_c(cfg);
  check(ctx(), mpeig_solve(ctx(), op.p, P.p, &c, &push_record, &b.hist, &b.r));
  EigResult<T> out = b.take(cfg.k);
  out.timings.factorize = t_factor;
  out.precond_shift = mpeig_precond_shift(P.p);
  return out;
}

// solve(CsrMatrix, cfg) (drivers.hpp:183-210): RCM permutation, sparse Cholesky
// on the permuted system, solve, eigenvectors in the original row order
template <class T>
EigResult<T> solve(const CsrMatrix<T>& A, const SolverConfig& cfg) {
  static_assert(std::is_same_v<T, double>, "solve: real double systems");
  const std::size_t n = A.n();
  detail::ResultBuffers b(n, cfg.k);
  const mpeig_cfg c = to_c(cfg);
  double shift = 0;
  check(ctx(), mpeig_solve_csr(ctx(), static_cast<int64_t>(n), A.row_ptr().data(),
                               A.col_idx().data(), A.values().data(), &c, &push_record, &b.hist,
                               &b.r, &shift));
  EigResult<T> out = b.take(cfg.k);
  out.precond_shift = shift;
  return out;
}

}  // namespace mpeig::b200
