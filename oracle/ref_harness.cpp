// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (see mp_oracle.h).
//
// Drives the UNMODIFIED reference library under /root/reference/proj through
// its own public entry points and BlockOperator callbacks, and exports the
// result over the plain C ABI in mp_oracle.h (prefix mpref_).  Nothing here
// re-implements reference numerics: every numeric call below is a reference
// function (lobpcg_stage, orthonormal_q, ritz_rotate, residual_block,
// converged_count, spectral_norm_estimate, gaussian_matrix, spmv_block, ...).
// The only harness-defined pieces are the ones the reference does not have
// (SURVEY.md §8c): the 3-D 7-point Laplacian, the Jacobi preconditioner as a
// BlockOperator, the two-stage hand-off restated from drivers.hpp:79-108 for
// callback preconditioners, and PINVIT with a callback preconditioner
// (eigensolvers.hpp:326-390 takes a concrete Preconditioner<T>).
//
// Built by oracle/Makefile into oracle/_ref/libmpeig_ref.so with the
// reference's Release flags (proj/CMakeLists.txt:8-12).

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "mpeig/drivers.hpp"
#include "mpeig/run_record.hpp"
#include "mpeig/eigensolvers.hpp"
#include "mpeig/generators.hpp"
#include "mpeig/norm_estimate.hpp"
#include "mpeig/ortho.hpp"
#include "mpeig/small_eig.hpp"
#include "mpeig/sparse_kernels.hpp"

#include "mp_oracle.h"

using namespace mpeig;

namespace {

using clk = std::chrono::steady_clock;
double secs(clk::time_point t0) {
  return std::chrono::duration<double>(clk::now() - t0).count();
}

// ---------------------------------------------------------------- problems
CsrMatrix<double> lap3d(std::size_t nx, std::size_t ny, std::size_t nz) {
  const std::size_t n = nx * ny * nz;
  std::vector<Triplet<double>> t;
  t.reserve(7 * n);
  for (std::size_t z = 0; z < nz; ++z)
    for (std::size_t y = 0; y < ny; ++y)
      for (std::size_t x = 0; x < nx; ++x) {
        const index_t p = static_cast<index_t>(x + nx * (y + ny * z));
        const index_t sx = 1, sy = static_cast<index_t>(nx),
                      sz = static_cast<index_t>(nx * ny);
        if (z > 0) t.push_back({p, p - sz, -1.0});
        if (y > 0) t.push_back({p, p - sy, -1.0});
        if (x > 0) t.push_back({p, p - sx, -1.0});
        t.push_back({p, p, 6.0});
        if (x + 1 < nx) t.push_back({p, p + sx, -1.0});
        if (y + 1 < ny) t.push_back({p, p + sy, -1.0});
        if (z + 1 < nz) t.push_back({p, p + sz, -1.0});
      }
  return CsrMatrix<double>::from_triplets(n, std::move(t));
}

struct System {
  std::size_t n = 0;
  bool dense = false;
  CsrMatrix<double> A;
  CsrMatrix<float> Al;
  DenseMatrix<double> D;
  DenseMatrix<float> Dl;
  std::vector<double> dinv;
  std::vector<float> dinvf;
  BlockOperator<double> op() const {
    if (dense) return [this](const DenseMatrix<double>& X) { return herm_product(D, X); };
    return [this](const DenseMatrix<double>& X) { return spmv_block(A, X); };
  }
  BlockOperator<float> op_lower() const {
    if (dense) return [this](const DenseMatrix<float>& X) { return herm_product(Dl, X); };
    return [this](const DenseMatrix<float>& X) { return spmv_block(Al, X); };
  }
};

std::unique_ptr<System> make_system(const mp_problem* p, bool need_lower) {
  auto s = std::make_unique<System>();
  switch (p->kind) {
    case MP_PROB_LAP3D:
      s->A = lap3d(p->nx, p->ny, p->nz);
      break;
    case MP_PROB_LAP2D:
      s->A = gen_laplace2d(p->nx, p->ny);
      break;
    case MP_PROB_CSR: {
      std::vector<Triplet<double>> t;
      for (int64_t i = 0; i < p->n; ++i)
        for (int64_t q = p->row_ptr[i]; q < p->row_ptr[i + 1]; ++q)
          t.push_back({i, p->col_idx[q], p->vals[q]});
      s->A = CsrMatrix<double>::from_triplets(p->n, std::move(t));
      break;
    }
    case MP_PROB_DENSE: {
      s->dense = true;
      s->D = DenseMatrix<double>(p->n, p->n);
      std::memcpy(s->D.data().data(), p->dense, sizeof(double) * p->n * p->n);
      break;
    }
    default:
      throw ConfigError("unknown problem kind");
  }
  s->n = s->dense ? s->D.rows() : s->A.n();
  s->dinv.resize(s->n);
  s->dinvf.resize(s->n);
  for (std::size_t i = 0; i < s->n; ++i) {
    const double d = s->dense ? s->D(i, i) : *s->A.find(i, static_cast<index_t>(i));
    s->dinv[i] = 1.0 / d;
    s->dinvf[i] = static_cast<float>(s->dinv[i]);
  }
  if (need_lower) {
    if (s->dense)
      s->Dl = to_lower(s->D);
    else
      s->Al = to_lower(s->A);
  }
  return s;
}

// ------------------------------------------------------- Jacobi f_T variants
// working:            W = R .* dinv                       (fp64 f_T)
// schol / mixed / pv: W = to_working(to_lower(R) .* dinvf) (fp32 f_T sandwich,
//                     the shape of Preconditioner::apply, precond.hpp:92-100)
// lower stage:        W = R .* dinvf                      (apply_lower, :103-109)
BlockOperator<double> jacobi_working(const System& s) {
  return [&s](const DenseMatrix<double>& R) {
    DenseMatrix<double> W(R.rows(), R.cols());
    for (std::size_t j = 0; j < R.cols(); ++j)
      for (std::size_t i = 0; i < R.rows(); ++i) W(i, j) = R(i, j) * s.dinv[i];
    return W;
  };
}
BlockOperator<double> jacobi_sandwich(const System& s) {
  return [&s](const DenseMatrix<double>& R) {
    DenseMatrix<float> Rl = to_lower(R);
    for (std::size_t j = 0; j < Rl.cols(); ++j)
      for (std::size_t i = 0; i < Rl.rows(); ++i) Rl(i, j) = Rl(i, j) * s.dinvf[i];
    return to_working(Rl);
  };
}
BlockOperator<float> jacobi_lower(const System& s) {
  return [&s](const DenseMatrix<float>& R) {
    DenseMatrix<float> W(R.rows(), R.cols());
    for (std::size_t j = 0; j < R.cols(); ++j)
      for (std::size_t i = 0; i < R.rows(); ++i) W(i, j) = R(i, j) * s.dinvf[i];
    return W;
  };
}

// PINVIT with a callback preconditioner: eigensolvers.hpp:326-390 with
// `P.apply(R)` replaced by `apply_precond(R)`; all numerics are reference calls.
EigResult<double> pinvit_cb(const BlockOperator<double>& apply_A, std::size_t n,
                            const DenseMatrix<double>& X0, const SolverConfig& cfg,
                            const BlockOperator<double>& apply_precond,
                            double a_norm_est) {
  EigResult<double> out;
  out.a_norm_estimate = a_norm_est;
  DenseMatrix<double> Xt = X0;
  (void)n;
  for (std::size_t iter = 0;; ++iter) {
    DenseMatrix<double> X;
    try {
      X = detail::orthonormal_q(Xt, true);
    } catch (const RankDeficient&) {
      throw RankCollapse("pinvit: iterate block lost rank");
    }
    DenseMatrix<double> AX = apply_A(X);
    std::vector<double> theta = detail::ritz_rotate(X, AX);
    const DenseMatrix<double> Rblk = detail::residual_block(AX, X, theta);
    const std::size_t n_c = converged_count(a_norm_est, X, theta, Rblk, cfg.tol);
    out.history.push_back(detail::make_record(Precision::Working, theta, Rblk, n_c));
    const bool done = n_c >= cfg.k;
    if (done || iter >= cfg.maxit) {
      out.converged = done;
      out.iterations_working = iter;
      out.theta.assign(theta.begin(), theta.begin() + cfg.k);
      out.X = X.slice_cols(0, cfg.k);
      for (std::size_t j = 0; j < cfg.k; ++j)
        out.residual_norms.push_back(Rblk.col_norm(j));
      return out;
    }
    const DenseMatrix<double> W = apply_precond(Rblk);
    Xt = subtract(X, W);
  }
}

int code_of(const std::exception& e) {
  if (dynamic_cast<const DimensionMismatch*>(&e)) return MP_E_DIMENSION;
  if (dynamic_cast<const ConfigError*>(&e)) return MP_E_CONFIG;
  if (dynamic_cast<const NotPositiveDefinite*>(&e)) return MP_E_NOT_PD;
  if (dynamic_cast<const SingularTriangular*>(&e)) return MP_E_SINGULAR_TRI;
  if (dynamic_cast<const RankDeficient*>(&e)) return MP_E_RANK_DEFICIENT;
  if (dynamic_cast<const RankCollapse*>(&e)) return MP_E_RANK_COLLAPSE;
  if (dynamic_cast<const NoConvergence*>(&e)) return MP_E_NO_CONVERGENCE;
  if (dynamic_cast<const OverflowError*>(&e)) return MP_E_OVERFLOW;
  return MP_E_OTHER;
}

template <class F>
int guarded(F&& f, char* msg = nullptr) {
  try {
    f();
    return MP_OK;
  } catch (const std::exception& e) {
    if (msg) std::snprintf(msg, 256, "%s", e.what());
    return code_of(e);
  }
}

void export_history(const std::vector<IterationRecord>& h, std::size_t m, mp_result* out) {
  out->hist_len = static_cast<int64_t>(h.size());
  const std::size_t cap = out->hist_cap > 0 ? static_cast<std::size_t>(out->hist_cap) : 0;
  for (std::size_t i = 0; i < h.size() && i < cap; ++i) {
    const IterationRecord& r = h[i];
    if (out->hist_stage) out->hist_stage[i] = r.stage == Precision::Lower ? 1 : 0;
    if (out->hist_nc) out->hist_nc[i] = static_cast<int64_t>(r.n_converged);
    if (out->hist_dropped) out->hist_dropped[i] = static_cast<int64_t>(r.w_columns_dropped);
    if (out->hist_fallback) out->hist_fallback[i] = r.basis_rotation_fallback ? 1 : 0;
    for (std::size_t j = 0; j < m; ++j) {
      if (out->hist_ritz) out->hist_ritz[i * m + j] = j < r.ritz_values.size() ? r.ritz_values[j] : NAN;
      if (out->hist_resid) out->hist_resid[i * m + j] = j < r.residual_norms.size() ? r.residual_norms[j] : NAN;
    }
  }
}

SolverConfig to_cfg(const mp_cfg* c, int variant) {
  SolverConfig cfg;
  cfg.k = static_cast<std::size_t>(c->k);
  cfg.block = static_cast<std::size_t>(c->block);
  cfg.maxit = static_cast<std::size_t>(c->maxit);
  cfg.tol = c->tol;
  cfg.lower_tol = c->lower_tol;
  cfg.seed = c->seed;
  cfg.sketch_rows = static_cast<std::size_t>(c->sketch_rows);
  cfg.variant = static_cast<Variant>(variant);
  return cfg;
}

DenseMatrix<double> wrap(int64_t r, int64_t c, const double* p) {
  DenseMatrix<double> M(r, c);
  if (r > 0 && c > 0) std::memcpy(M.data().data(), p, sizeof(double) * r * c);
  return M;
}
template <class T>
void unwrap(const DenseMatrix<T>& M, T* p) {
  if (p && !M.data().empty()) std::memcpy(p, M.data().data(), sizeof(T) * M.data().size());
}

}  // namespace

extern "C" {

int mpref_solve(const mp_problem* prob, int variant, const mp_cfg* c, mp_result* out) {
  out->status = guarded([&] {
    const SolverConfig cfg = to_cfg(c, variant);
    const bool mixed = variant == MP_MPLOBPCG_SCHOL;
    auto sys = make_system(prob, mixed);
    const std::size_t n = sys->n;
    cfg.validate(n);
    const std::size_t m = cfg.block_size();
    const auto t0 = clk::now();
    // drivers.hpp:164-169 (solve): sketch, then the orthonormal start block
    const double est = spectral_norm_estimate<double>(sys->op(), n, cfg.sketch_rows,
                                                      cfg.seed ^ 0x9e3779b97f4a7c15ULL);
    const DenseMatrix<double> X0 = detail::orthonormal_q(
        c->x0 ? wrap(static_cast<int64_t>(n), static_cast<int64_t>(m), c->x0)
              : gaussian_matrix<double>(n, m, cfg.seed),
        true);
    out->t_setup = secs(t0);
    out->t_stage1 = 0;
    EigResult<double> r;
    r.a_norm_estimate = est;
    if (variant == MP_PINVIT) {
      r = pinvit_cb(sys->op(), n, X0, cfg, jacobi_sandwich(*sys), est);
    } else {
      // drivers.hpp:79-108 (run_variant), preconditioner as a callback
      DenseMatrix<double> X = X0;
      if (mixed) {
        StageOptions lo;
        lo.tol = cfg.lower_tol;
        lo.use_mixed_qr = false;
        lo.stagnation_exit = true;
        lo.tag = Precision::Lower;
        const auto t1 = clk::now();
        StageOutcome<float> st1 = lobpcg_stage<float>(sys->op_lower(), n, to_lower(X), cfg,
                                                      jacobi_lower(*sys), est, lo,
                                                      r.history, r.timings);
        r.iterations_lower = st1.iterations;
        X = detail::orthonormal_q(to_working(st1.X), true);
        out->t_stage1 = secs(t1);
      }
      StageOptions hi;
      hi.tol = cfg.tol;
      hi.use_mixed_qr = mixed;
      hi.tag = Precision::Working;
      const BlockOperator<double> T = variant == MP_DLOBPCG_DCHOL
                                          ? jacobi_working(*sys)
                                          : jacobi_sandwich(*sys);
      StageOutcome<double> st = lobpcg_stage<double>(sys->op(), n, X, cfg, T, est, hi,
                                                     r.history, r.timings);
      r.iterations_working = st.iterations;
      r.converged = st.converged;
      for (std::size_t j = 0; j < cfg.k; ++j) {
        r.theta.push_back(st.theta[j]);
        r.residual_norms.push_back(st.residual_norms[j]);
      }
      r.X = st.X.slice_cols(0, cfg.k);
      r.a_norm_estimate = est;
    }
    out->t_total = secs(t0);
    out->converged = r.converged ? 1 : 0;
    out->iters_lower = static_cast<int64_t>(r.iterations_lower);
    out->iters_working = static_cast<int64_t>(r.iterations_working);
    out->a_norm_est = est;
    for (std::size_t j = 0; j < cfg.k; ++j) {
      out->theta[j] = r.theta[j];
      out->resid[j] = r.residual_norms[j];
    }
    unwrap(r.X, out->X);
    export_history(r.history, m, out);
  }, out->msg);
  return out->status;
}

// The reference's stock drivers: solve(DenseMatrix, cfg) (drivers.hpp:158-181)
// and solve(CsrMatrix, cfg) (:183-210) with their own Cholesky preconditioners
// (Preconditioner<T>::build, precond.hpp:33-77) -- the golden source for the
// device dense / sparse Cholesky f_T.  Same outputs as mpref_solve.
int mpref_solve_native(const mp_problem* prob, int variant, const mp_cfg* c, mp_result* out) {
  out->status = guarded([&] {
    const SolverConfig cfg = to_cfg(c, variant);
    auto sys = make_system(prob, false);
    const std::size_t m = cfg.block_size();
    const auto t0 = clk::now();
    // dense: Cholesky f_T; CSR: RCM-permuted system + sparse Cholesky f_T
    EigResult<double> r = sys->dense ? solve(sys->D, cfg) : solve(sys->A, cfg);
    out->t_total = secs(t0);
    out->t_setup = r.timings.factorize;
    out->t_stage1 = r.precond_shift;  // (field reused: the retry shift)
    out->converged = r.converged ? 1 : 0;
    out->iters_lower = static_cast<int64_t>(r.iterations_lower);
    out->iters_working = static_cast<int64_t>(r.iterations_working);
    out->a_norm_est = r.a_norm_estimate;
    for (std::size_t j = 0; j < cfg.k && j < r.theta.size(); ++j) {
      out->theta[j] = r.theta[j];
      out->resid[j] = r.residual_norms[j];
    }
    unwrap(r.X, out->X);
    export_history(r.history, m, out);
  }, out->msg);
  return out->status;
}

// format_shortest (run_record.cpp:97-102): std::to_chars shortest round trip
int mpref_format_shortest(double v, char* buf, int cap) {
  const std::string t = format_shortest(v);
  std::snprintf(buf, static_cast<std::size_t>(cap), "%s", t.c_str());
  return static_cast<int>(t.size());
}

// rcm_ordering_pattern (rcm.cpp:8-57) on a CSR pattern
void mpref_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* out) {
  std::vector<index_t> r(rp, rp + n + 1), c(ci, ci + rp[n]);
  const std::vector<index_t> p = rcm_ordering_pattern(static_cast<std::size_t>(n), r, c);
  for (int64_t k = 0; k < n; ++k) out[k] = p[k];
}

void mpref_pcg64_u64(uint64_t seed, int64_t count, uint64_t* o) {
  Pcg64 g(seed);
  for (int64_t i = 0; i < count; ++i) o[i] = g.next_u64();
}

void mpref_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* o) {
  unwrap(gaussian_matrix<double>(rows, cols, seed), o);
}

double mpref_norm_estimate(const mp_problem* prob, int64_t sketch_rows, uint64_t seed) {
  auto sys = make_system(prob, false);
  return spectral_norm_estimate<double>(sys->op(), sys->n, sketch_rows, seed);
}

int mpref_householder_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  return guarded([&] {
    auto f = householder_qr(wrap(n, m, A));
    unwrap(f.Q, Q);
    unwrap(f.R, R);
  });
}

int mpref_householder_qr_f32(int64_t n, int64_t m, const float* A, float* Q, float* R) {
  return guarded([&] {
    DenseMatrix<float> M(n, m);
    std::memcpy(M.data().data(), A, sizeof(float) * n * m);
    auto f = householder_qr(M);
    unwrap(f.Q, Q);
    unwrap(f.R, R);
  });
}

int mpref_mixed_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  return guarded([&] {
    auto f = mixed_qr(wrap(n, m, A));
    unwrap(f.Q, Q);
    unwrap(f.R, R);
  });
}

int mpref_cholesky_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  return guarded([&] {
    auto f = cholesky_qr(wrap(n, m, A));
    unwrap(f.Q, Q);
    unwrap(f.R, R);
  });
}

int mpref_small_herm_eig(int64_t n, const double* M, double* vals, double* vecs) {
  return guarded([&] {
    auto e = small_herm_eig(wrap(n, n, M));
    for (int64_t i = 0; i < n; ++i) vals[i] = e.values[i];
    unwrap(e.vectors, vecs);
  });
}

int mpref_hl_update(int64_t n, int64_t s, int64_t m, const double* S, const double* C,
                    double* X, double* P, double* c_pv, int32_t* fallback) {
  return guarded([&] {
    std::vector<double> D(s, 0.0);
    auto up = hl_update(wrap(n, s, S), wrap(s, s, C), D, m);
    unwrap(up.X, X);
    unwrap(up.P, P);
    unwrap(up.c_pv, c_pv);
    *fallback = up.rotation_fallback ? 1 : 0;
  });
}

void mpref_project_out(int64_t n, int64_t b, int64_t w, const double* B, double* W,
                       int passes) {
  auto Y = block_project_out(wrap(n, w, W), wrap(n, b, B), passes);
  unwrap(Y, W);
}

int64_t mpref_ortho_dropping(int64_t n, int64_t w, const double* W, double tol, double* Q) {
  std::size_t dropped = 0;
  auto R = orthonormalize_dropping(wrap(n, w, W), tol, &dropped);
  unwrap(R, Q);
  return static_cast<int64_t>(R.cols());
}

void mpref_apply_op(const mp_problem* prob, int64_t ncols, const double* X, double* Y) {
  auto sys = make_system(prob, false);
  unwrap(sys->op()(wrap(sys->n, ncols, X)), Y);
}

int64_t mpref_converged_count(int64_t n, int64_t m, double a_norm_est, const double* X,
                              const double* theta, const double* R, double tol) {
  std::vector<double> th(theta, theta + m);
  return static_cast<int64_t>(
      converged_count(a_norm_est, wrap(n, m, X), th, wrap(n, m, R), tol));
}

}  // extern "C"
