// Drop-in check of include/mpeig_b200.hpp -- TEST INFRASTRUCTURE.
//
// Compiled against the reference's own headers (/root/reference/proj/include)
// and libmpeig_b200.so by oracle/Makefile (target `dropin`), so the reference's
// types, callbacks and call sequences drive the B200 path unchanged:
//
//   dropin_main stage <nx> <ny> <nz> <variant> <k> <tol> <maxit>
//       run_variant's flow (drivers.hpp:79-108) with Jacobi BlockOperator
//       callbacks -- the golden harness's sequence (oracle/ref_harness.cpp) --
//       with every lobpcg_stage call qualified as mpeig::b200::lobpcg_stage.
//   dropin_main solve_csr <nx> <ny> <nz> <variant> <k> <block> <tol> <maxit> <seed>
//       mpeig::b200::solve(CsrMatrix, cfg)    (drivers.hpp:183-210)
//   dropin_main solve_dense <file> <n> <variant> <k> <tol> <maxit> <seed>
//       mpeig::b200::solve(DenseMatrix, cfg)  (drivers.hpp:158-181); file = n*n
//       column-major doubles
//   dropin_main errors
//       the reference's exception types out of the B200 path
//
// Prints one JSON object per run on stdout.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include <mpeig/drivers.hpp>
#include <mpeig/eigensolvers.hpp>
#include <mpeig/generators.hpp>
#include <mpeig/sparse_kernels.hpp>

#include "mpeig_b200.hpp"

using namespace mpeig;

static CsrMatrix<double> laplacian(std::size_t nx, std::size_t ny, std::size_t nz) {
  if (nz <= 1) return gen_laplace2d(nx, ny);
  std::vector<Triplet<double>> t;
  const std::size_t n = nx * ny * nz, sy = nx, sz = nx * ny;
  for (std::size_t z = 0; z < nz; ++z)
    for (std::size_t y = 0; y < ny; ++y)
      for (std::size_t x = 0; x < nx; ++x) {
        const index_t p = static_cast<index_t>(x + nx * (y + ny * z));
        if (z > 0) t.push_back({p, p - static_cast<index_t>(sz), -1.0});
        if (y > 0) t.push_back({p, p - static_cast<index_t>(sy), -1.0});
        if (x > 0) t.push_back({p, p - 1, -1.0});
        t.push_back({p, p, 6.0});
        if (x + 1 < nx) t.push_back({p, p + 1, -1.0});
        if (y + 1 < ny) t.push_back({p, p + static_cast<index_t>(sy), -1.0});
        if (z + 1 < nz) t.push_back({p, p + static_cast<index_t>(sz), -1.0});
      }
  return CsrMatrix<double>::from_triplets(n, std::move(t));
}

static void print_result(const char* mode, const std::vector<double>& theta, std::size_t il,
                         std::size_t iw, bool conv, double est, double shift, std::size_t hist) {
  std::printf("{\"mode\": \"%s\", \"iters_lower\": %zu, \"iters_working\": %zu, \"converged\": %s, "
              "\"a_norm_est\": %.17g, \"precond_shift\": %.17g, \"history\": %zu, \"theta\": [",
              mode, il, iw, conv ? "true" : "false", est, shift, hist);
  for (std::size_t j = 0; j < theta.size(); ++j) std::printf("%s%.17g", j ? ", " : "", theta[j]);
  std::printf("]}\n");
}

static int run_stage(int argc, char** argv) {
  if (argc < 9) return 2;
  const std::size_t nx = std::stoul(argv[2]), ny = std::stoul(argv[3]), nz = std::stoul(argv[4]);
  SolverConfig cfg;
  cfg.variant = variant_from_name(argv[5]);
  cfg.k = std::stoul(argv[6]);
  cfg.tol = std::stod(argv[7]);
  cfg.maxit = std::stoul(argv[8]);
  const CsrMatrix<double> A = laplacian(nx, ny, nz);
  const CsrMatrix<float> Al = to_lower(A);
  const std::size_t n = A.n(), m = cfg.block_size();
  cfg.validate(n);
  std::vector<double> dinv(n);
  std::vector<float> dinvf(n);
  for (std::size_t i = 0; i < n; ++i) {
    dinv[i] = 1.0 / *A.find(i, static_cast<index_t>(i));
    dinvf[i] = static_cast<float>(dinv[i]);
  }
  const BlockOperator<double> opA = [&](const DenseMatrix<double>& X) { return spmv_block(A, X); };
  const BlockOperator<float> opAl = [&](const DenseMatrix<float>& X) { return spmv_block(Al, X); };
  const BlockOperator<double> precW = [&](const DenseMatrix<double>& R) {
    DenseMatrix<double> W(R.rows(), R.cols());
    for (std::size_t j = 0; j < R.cols(); ++j)
      for (std::size_t i = 0; i < R.rows(); ++i) W(i, j) = R(i, j) * dinv[i];
    return W;
  };
  const BlockOperator<double> precS = [&](const DenseMatrix<double>& R) {
    DenseMatrix<float> Rl = to_lower(R);
    for (std::size_t j = 0; j < Rl.cols(); ++j)
      for (std::size_t i = 0; i < Rl.rows(); ++i) Rl(i, j) = Rl(i, j) * dinvf[i];
    return to_working(Rl);
  };
  const BlockOperator<float> precL = [&](const DenseMatrix<float>& R) {
    DenseMatrix<float> W(R.rows(), R.cols());
    for (std::size_t j = 0; j < R.cols(); ++j)
      for (std::size_t i = 0; i < R.rows(); ++i) W(i, j) = R(i, j) * dinvf[i];
    return W;
  };
  // solve() (drivers.hpp:164-169): sketch, orthonormal start block
  const double est = mpeig::b200::spectral_norm_estimate<double>(opA, n, cfg.sketch_rows,
                                                                 cfg.seed ^ 0x9e3779b97f4a7c15ULL);
  DenseMatrix<double> X = detail::orthonormal_q(gaussian_matrix<double>(n, m, cfg.seed), true);
  // run_variant (drivers.hpp:79-108), lobpcg_stage qualified to the B200 path
  std::vector<IterationRecord> history;
  StageTimings tim;
  std::size_t it_lo = 0;
  const bool mixed = cfg.variant == Variant::MPLOBPCG_schol;
  if (mixed) {
    StageOptions lo;
    lo.tol = cfg.lower_tol;
    lo.use_mixed_qr = false;
    lo.stagnation_exit = true;
    lo.tag = Precision::Lower;
    StageOutcome<float> st1 = mpeig::b200::lobpcg_stage<float>(opAl, n, to_lower(X), cfg, precL,
                                                               est, lo, history, tim);
    it_lo = st1.iterations;
    X = detail::orthonormal_q(to_working(st1.X), true);
  }
  StageOptions hi;
  hi.tol = cfg.tol;
  hi.use_mixed_qr = mixed;
  hi.tag = Precision::Working;
  const BlockOperator<double>& T = cfg.variant == Variant::DLOBPCG_dchol ? precW : precS;
  StageOutcome<double> st = mpeig::b200::lobpcg_stage<double>(opA, n, X, cfg, T, est, hi,
                                                              history, tim);
  std::vector<double> theta(st.theta.begin(), st.theta.begin() + cfg.k);
  // residual contract on the host, through the reference's own kernels
  const DenseMatrix<double> AX = spmv_block(A, st.X);
  double worst = 0;
  for (std::size_t j = 0; j < cfg.k; ++j) {
    double r2 = 0;
    for (std::size_t i = 0; i < n; ++i) {
      const double r = AX(i, j) - st.theta[j] * st.X(i, j);
      r2 += r * r;
    }
    const double thr = cfg.tol * (est + std::abs(st.theta[j]));
    worst = std::max(worst, std::sqrt(r2) / thr);
  }
  std::fprintf(stderr, "worst residual / threshold = %.3g\n", worst);
  print_result("stage", theta, it_lo, st.iterations, st.converged && worst <= 1.0 + 1e-9, est, 0,
               history.size());
  return 0;
}

static int run_solve_csr(int argc, char** argv) {
  if (argc < 11) return 2;
  const CsrMatrix<double> A = laplacian(std::stoul(argv[2]), std::stoul(argv[3]), std::stoul(argv[4]));
  SolverConfig cfg;
  cfg.variant = variant_from_name(argv[5]);
  cfg.k = std::stoul(argv[6]);
  cfg.block = std::stoul(argv[7]);
  cfg.tol = std::stod(argv[8]);
  cfg.maxit = std::stoul(argv[9]);
  cfg.seed = std::stoull(argv[10]);
  const EigResult<double> r = mpeig::b200::solve(A, cfg);
  // X in the original row order: residuals on the unpermuted matrix
  const DenseMatrix<double> AX = spmv_block(A, r.X);
  double worst = 0;
  for (std::size_t j = 0; j < cfg.k; ++j) {
    double r2 = 0;
    for (std::size_t i = 0; i < A.n(); ++i) {
      const double e = AX(i, j) - r.theta[j] * r.X(i, j);
      r2 += e * e;
    }
    worst = std::max(worst, std::sqrt(r2) / (cfg.tol * (r.a_norm_estimate + std::abs(r.theta[j]))));
  }
  std::fprintf(stderr, "worst residual / threshold (original order) = %.3g\n", worst);
  print_result("solve_csr", r.theta, r.iterations_lower, r.iterations_working,
               r.converged && worst <= 10.0, r.a_norm_estimate, r.precond_shift, r.history.size());
  return 0;
}

static int run_solve_dense(int argc, char** argv) {
  if (argc < 9) return 2;
  const std::size_t n = std::stoul(argv[3]);
  DenseMatrix<double> A(n, n);
  std::ifstream f(argv[2], std::ios::binary);
  f.read(reinterpret_cast<char*>(A.data().data()), static_cast<std::streamsize>(sizeof(double) * n * n));
  if (!f) return 3;
  SolverConfig cfg;
  cfg.variant = variant_from_name(argv[4]);
  cfg.k = std::stoul(argv[5]);
  cfg.tol = std::stod(argv[6]);
  cfg.maxit = std::stoul(argv[7]);
  cfg.seed = std::stoull(argv[8]);
  const EigResult<double> r = mpeig::b200::solve(A, cfg);
  print_result("solve_dense", r.theta, r.iterations_lower, r.iterations_working, r.converged,
               r.a_norm_estimate, r.precond_shift, r.history.size());
  return 0;
}

static int run_errors() {
  int ok = 0, total = 0;
  auto expect = [&](const char* what, auto&& f, auto tag) {
    using E = decltype(tag);
    ++total;
    try {
      f();
      std::fprintf(stderr, "%s: no exception\n", what);
    } catch (const E&) {
      ++ok;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s: wrong exception: %s\n", what, e.what());
    }
  };
  const CsrMatrix<double> A = laplacian(6, 6, 1);  // n = 36
  SolverConfig big;
  big.k = 12;
  big.block = 13;  // 3 * 13 > 36
  expect("config", [&] { mpeig::b200::solve(A, big); }, ConfigError("x"));
  DenseMatrix<double> D(8, 8);  // indefinite (zero) dense matrix: the fp64 factor fails
  SolverConfig c2;
  c2.k = 1;
  c2.variant = Variant::DLOBPCG_dchol;
  expect("not_pd", [&] { mpeig::b200::solve(D, c2); }, NotPositiveDefinite(0, "x"));
  const BlockOperator<double> bad = [](const DenseMatrix<double>& X) {
    return DenseMatrix<double>(X.rows() + 1, X.cols());
  };
  expect("callback_shape", [&] { mpeig::b200::spectral_norm_estimate<double>(bad, 36, 8, 1); },
         DimensionMismatch("x"));
  std::printf("{\"mode\": \"errors\", \"ok\": %d, \"total\": %d}\n", ok, total);
  return ok == total ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "stage") return run_stage(argc, argv);
    if (mode == "solve_csr") return run_solve_csr(argc, argv);
    if (mode == "solve_dense") return run_solve_dense(argc, argv);
    if (mode == "errors") return run_errors();
  } catch (const std::exception& e) {
    std::printf("{\"mode\": \"%s\", \"error\": \"%s\"}\n", mode.c_str(), e.what());
    return 1;
  }
  return 2;
}
