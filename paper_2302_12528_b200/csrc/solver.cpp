// solver.cpp -- the LOBPCG / PINVIT iteration on the device (host orchestration).
//
// Mirrors the reference solver step for step:
//   lobpcg_stage<T>  eigensolvers.hpp:195-321
//   pinvit<T>        eigensolvers.hpp:326-390
//   run_variant      drivers.hpp:57-111,   solve() drivers.hpp:158-181
// Every block vector stays on the device; per iteration the host receives
// only theta, the residual / column norms and a few status words (needed for
// the prefix convergence rule and the history record), exactly the data the
// reference's IterationRecord carries.
//
// Device layout: S = [X | P | W] and AS = [AX | AP | AW] are
// single column-major allocations (ld = n rounded up to 32), so the
// reference's hconcat copies (dense_matrix.hpp:90-107) vanish; the next X, P,
// AX, AP are written to a second pair of buffers and the pairs swap.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <utility>
#include <vector>

#include "context.hpp"
#include "solver.hpp"
#include "spchol.hpp"

namespace mpb {

std::atomic<int64_t> g_launches{0};

// ------------------------------------------------------------------ status
void status_clear(mpeig_ctx* ctx) {
  MPB_CUDA(cudaMemsetAsync(ctx->d_status, 0, 16 * sizeof(int), ctx->stream));
}

void status_fetch(mpeig_ctx* ctx) {
  // row-sharded: every rank sees every rank's failures, so all take the same branch
  if (Comm* c = dist(ctx)) c->allreduce_max(ctx->d_status, 16, ctx->stream);
  MPB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, 16 * sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
  MPB_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void cusolver_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS)
    throw Error(MPEIG_E_CUSOLVER, std::string(what) + " failed (cusolver status " +
                                      std::to_string(static_cast<int>(st)) + ")");
}

static void cublas_check(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS)
    throw Error(MPEIG_E_CUDA, std::string(what) + " failed (cublas status " +
                                  std::to_string(static_cast<int>(st)) + ")");
}

// --------------------------------------------------------------- operators
// ------------------------------------------- dense Cholesky f_T
// Preconditioner<T>::Kind::DenseChol (precond.hpp:33-50, 92-109, 121-126):
// T(R) = L^-T L^-1 R with L the lower Cholesky factor of A (or of to_lower(A)).
// Built once per solve: cuSOLVER potrf (the reference's dense_cholesky, same
// failure semantics), then potri turns the factor into M = L^-T L^-1 in the
// build precision, stored as a full symmetric n x n matrix.  Each apply is then
// ONE GEMM M R (cuBLAS, no TF32) instead of two triangular solves: the same
// 2 n^2 c flops, but at GEMM throughput instead of trsm's column-serial sweep
// (cfg3, n = 16384, c = 96: trsm pair 10.6 ms -> SGEMM, scripts/cfg3_dense.py).
// Rounding differs from the reference's substitutions at the level of the
// preconditioner's own accuracy (kappa eps_T); parity is the solver-level bar
// (tests/test_gpu_precond.py).  The lower()/working() conversions of an fp32
// factor run around the GEMM.

// dense_cholesky (dense_kernels.hpp:128-152) on L in place: failure index and
// the reference's error types (non-finite pivot -> OverflowError, nonpositive
// -> NotPositiveDefinite(j)); check_tri_diag (:163-170) recorded for the applies
template <typename F>
static void chol_factor(mpeig_ctx* ctx, F* L, int64_t n, mpeig_op* op) {
  cudaStream_t s = ctx->stream;
  const int ni = static_cast<int>(n);
  int lwork = 0;
  if constexpr (sizeof(F) == 8)
    cusolver_check(cusolverDnDpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, &lwork),
                   "cusolverDnDpotrf_bufferSize");
  else
    cusolver_check(cusolverDnSpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, &lwork),
                   "cusolverDnSpotrf_bufferSize");
  DevBuf<F> work(static_cast<size_t>(std::max(lwork, 1)), s);
  DevBuf<int> info(1, s);
  if constexpr (sizeof(F) == 8)
    cusolver_check(cusolverDnDpotrf(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, work.p, lwork, info.p),
                   "cusolverDnDpotrf");
  else
    cusolver_check(cusolverDnSpotrf(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, work.p, lwork, info.p),
                   "cusolverDnSpotrf");
  int h_info = 0;
  std::vector<F> d(static_cast<size_t>(n));
  MPB_CUDA(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaMemcpy2DAsync(d.data(), sizeof(F), L, sizeof(F) * (n + 1), sizeof(F), n,
                             cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  const int64_t fail = h_info > 0 ? h_info - 1 : n;
  for (int64_t j = 0; j < fail; ++j)
    if (!std::isfinite(static_cast<double>(d[j])))
      throw Error(MPEIG_E_OVERFLOW, "dense_cholesky: pivot " + std::to_string(j) + " is not finite", j);
  if (h_info > 0)
    throw Error(MPEIG_E_NOT_PD, "dense_cholesky: nonpositive pivot at " + std::to_string(fail), fail);
  op->tri_singular = -1;
  for (int64_t j = 0; j < n; ++j) {
    const F a = std::abs(d[j]);
    if (a == 0 || a < std::numeric_limits<F>::min()) {
      op->tri_singular = j;
      return;  // every apply throws SingularTriangular (check_tri_diag)
    }
  }
  // M = L^-T L^-1 (lower triangle), then mirrored to the upper one
  lwork = 0;
  if constexpr (sizeof(F) == 8)
    cusolver_check(cusolverDnDpotri_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, &lwork),
                   "cusolverDnDpotri_bufferSize");
  else
    cusolver_check(cusolverDnSpotri_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, &lwork),
                   "cusolverDnSpotri_bufferSize");
  work.alloc(static_cast<size_t>(std::max(lwork, 1)), s);
  if constexpr (sizeof(F) == 8)
    cusolver_check(cusolverDnDpotri(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, work.p, lwork, info.p),
                   "cusolverDnDpotri");
  else
    cusolver_check(cusolverDnSpotri(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, L, ni, work.p, lwork, info.p),
                   "cusolverDnSpotri");
  MPB_CUDA(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  if (h_info > 0)
    throw Error(MPEIG_E_SINGULAR_TRI, "tri_solve: zero or subnormal diagonal", h_info - 1);
  symmetrize_lower<F>(n, L, n, s);
}

void dense_chol_build(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, mpeig_op* op) {
  if (!A || A->kind != kOpDense)
    throw Error(MPEIG_E_CONFIG, "dense_chol: operator is not an explicit dense matrix");
  const int64_t n = A->n;
  cudaStream_t s = ctx->stream;
  op->precision = precision;
  if (precision == MPEIG_WORKING) {  // precond.hpp:38-41: no retry in working precision
    MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&op->Lw), sizeof(double) * n * n));
    copy_block<double>(n, n, A->A, A->lda, op->Lw, n, s);
    chol_factor<double>(ctx, op->Lw, n, op);
    return;
  }
  MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&op->Ll), sizeof(float) * n * n));
  auto attempt = [&](double shift) {
    if (shift == 0.0) {  // dense_cholesky(to_lower(A))
      if (A->lower_overflow) throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
      copy_block<float>(n, n, A->Al, A->lda, op->Ll, n, s);
    } else {  // retry_dense: to_lower(A + shift I), the shift added in fp64
      DevBuf<double> As(static_cast<size_t>(n * n), s);
      copy_block<double>(n, n, A->A, A->lda, As.p, n, s);
      add_diag_f64(n, As.p, n, shift, s);
      status_clear(ctx);
      convert_f64_to_f32(n, n, As.p, n, op->Ll, n, ctx->d_status + 2, s);
      status_fetch(ctx);
      if (ctx->h_status[2]) throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
    }
    chol_factor<float>(ctx, op->Ll, n, op);
  };
  try {
    attempt(0.0);
  } catch (const Error& e) {  // precond.hpp:42-48: one retry on NotPositiveDefinite / OverflowError
    if (e.code != MPEIG_E_NOT_PD && e.code != MPEIG_E_OVERFLOW) throw;
    // retry_shift (precond.hpp:128-132): 10 u_l ||A||_est, sketch seed kShiftSeed (:161)
    op->shift = 10.0 * 0x1p-24 * spectral_norm_estimate(ctx, A, 8, 0x5eed0123ULL);
    attempt(op->shift);
  }
}

// Y = M B (n x c), M = L^-T L^-1 symmetric n x n: dense_solve (precond.hpp:115-120,
// tri_solve Forward then BackwardAdjoint) as one GEMM.  Y must not alias B.
template <typename F>
static void chol_apply_gemm(mpeig_ctx* ctx, const F* M, int64_t n, int64_t c, const F* B,
                            int64_t ldb, F* Y, int64_t ldy) {
  const int ni = static_cast<int>(n), ci = static_cast<int>(c);
  const F one = 1, zero = 0;
  ProfScope prof("precond_chol", ctx->stream, double(sizeof(F)) * (double(n) * n + 2.0 * n * c),
                 2.0 * n * double(n) * c);
  if constexpr (sizeof(F) == 8) {
    // fp64: cuBLAS DGEMM, a plain library GEMM (35 TF/s at n = 16384, c = 96
    // against 28.4 for the library's own deep-K DMMA GEMM, scripts/dense_ax_bench.py)
    cublas_check(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, ni, ci, ni, &one, M, ni, B,
                             static_cast<int>(ldb), &zero, Y, static_cast<int>(ldy)),
                 "cublasDgemm");
  } else {
    // fp32: the tcgen05 block update (exact 3-way bf16 split; 96 TF/s at
    // n = 16384, c = 96 against cuBLAS SGEMM's 46, profiles/r02_dense_ax.json)
    (void)one;
    (void)zero;
    (void)ni;
    (void)ci;
    gemm_tn<float>(n, n, c, 1.f, M, n, B, ldb, 0.f, nullptr, 0, Y, ldy, ctx->stream);
  }
}

// fp32 scratch of the op, at least `need` elements
static float* op_scratch(mpeig_ctx* ctx, const mpeig_op* op, size_t need) {
  if (op->scratch_elems < need) {
    if (op->scratch) {
      MPB_CUDA(cudaStreamSynchronize(ctx->stream));
      MPB_CUDA(cudaFree(op->scratch));
      op->scratch = nullptr;
    }
    MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&op->scratch), sizeof(float) * need));
    op->scratch_elems = need;
  }
  return op->scratch;
}

// Preconditioner::apply (T = double) / apply_lower (T = float), precond.hpp:92-109
// ------------------------------------------- sparse Cholesky f_T
// Preconditioner<T>::build(CsrMatrix, prec[, perm]) (precond.hpp:55-77): the
// ordering (RCM by default, rcm.cpp:8-57) and the up-looking factorisation run
// on the host once per solve (spchol_host.cpp), as in the reference; the factor
// lives on the device and every apply is the two sweeps of spchol.cu.
template <typename V>
static V* sp_upload(const V* host, size_t count, cudaStream_t s) {
  V* d = nullptr;
  MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), count * sizeof(V)));
  MPB_CUDA(cudaMemcpyAsync(d, host, count * sizeof(V), cudaMemcpyHostToDevice, s));
  return d;
}

template <typename F>
static void upload_sparse_factor(mpeig_ctx* ctx, const HostFactor<F>& L, int64_t n, mpeig_op* op) {
  const int64_t nnz = static_cast<int64_t>(L.ci.size());
  if (nnz > INT32_MAX) throw Error(MPEIG_E_CONFIG, "sparse_chol: factor above 2^31 entries");
  std::vector<int> lrp(static_cast<size_t>(n + 1)), lci(static_cast<size_t>(nnz));
  std::vector<int> urp(static_cast<size_t>(n + 1), 0), uci(static_cast<size_t>(nnz));
  std::vector<F> uv(static_cast<size_t>(nnz));
  op->tri_singular = -1;
  for (int64_t i = 0; i < n; ++i) {
    lrp[i] = static_cast<int>(L.rp[i]);
    for (int64_t p = L.rp[i]; p < L.rp[i + 1]; ++p) {
      lci[p] = static_cast<int>(L.ci[p]);
      ++urp[L.ci[p] + 1];
    }
    const F d = std::abs(L.v[L.rp[i + 1] - 1]);  // check_tri_diag (sparse_kernels.hpp:186-192)
    if (op->tri_singular < 0 && (d == F(0) || d < std::numeric_limits<F>::min())) op->tri_singular = i;
  }
  lrp[n] = static_cast<int>(nnz);
  for (int64_t j = 0; j < n; ++j) urp[j + 1] += urp[j];
  std::vector<int> fill(urp.begin(), urp.end() - 1);
  for (int64_t i = 0; i < n; ++i)  // rows ascending: U row j starts with L(j, j)
    for (int64_t p = L.rp[i]; p < L.rp[i + 1]; ++p) {
      const int q = fill[L.ci[p]]++;
      uci[q] = static_cast<int>(i);
      uv[q] = L.v[p];
    }
  // block split points of the blocked sweeps (spchol.cu): rows in blocks of 32
  // lsp = [Lsp | Lsp2], usp = [Usp | Usp2] (n each): Lsp2 / Usp2 bound the entries
  // of the neighbouring block (previous for L, next for U)
  std::vector<int> lsp(static_cast<size_t>(2 * n)), usp(static_cast<size_t>(2 * n));
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b0 = i & ~int64_t{31}, b1 = b0 + 32;
    int64_t p = L.rp[i];
    while (p < L.rp[i + 1] - 1 && L.ci[p] < b0 - 32) ++p;
    lsp[n + i] = static_cast<int>(p);
    while (p < L.rp[i + 1] - 1 && L.ci[p] < b0) ++p;
    lsp[i] = static_cast<int>(p);
    int q = urp[i] + 1;
    while (q < urp[i + 1] && uci[q] < b1) ++q;
    usp[i] = q;
    while (q < urp[i + 1] && uci[q] < b1 + 32) ++q;
    usp[n + i] = q;
  }
  cudaStream_t s = ctx->stream;
  op->sp_Lsp = sp_upload(lsp.data(), lsp.size(), s);
  op->sp_Usp = sp_upload(usp.data(), usp.size(), s);
  op->sp_Lrp = sp_upload(lrp.data(), lrp.size(), s);
  op->sp_Lci = sp_upload(lci.data(), lci.size(), s);
  op->sp_Urp = sp_upload(urp.data(), urp.size(), s);
  op->sp_Uci = sp_upload(uci.data(), uci.size(), s);
  op->sp_Lv = sp_upload(L.v.data(), L.v.size(), s);
  op->sp_Uv = sp_upload(uv.data(), uv.size(), s);
  op->sp_nnz = nnz;
  MPB_CUDA(cudaStreamSynchronize(s));
}

void sparse_chol_build(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, int32_t ordering,
                       const int64_t* user_perm, mpeig_op* op) {
  if (!A || A->kind != kOpCsr)
    throw Error(MPEIG_E_CONFIG, "sparse_chol: operator is not an explicit CSR matrix");
  const int64_t n = A->n;
  if (n > INT32_MAX) throw Error(MPEIG_E_CONFIG, "sparse_chol: n above 2^31");
  cudaStream_t s = ctx->stream;
  std::vector<int64_t> rp(static_cast<size_t>(n + 1));
  MPB_CUDA(cudaMemcpyAsync(rp.data(), A->rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> ci(static_cast<size_t>(rp[n]));
  std::vector<double> v(static_cast<size_t>(rp[n]));
  MPB_CUDA(cudaMemcpyAsync(ci.data(), A->ci, sizeof(int64_t) * rp[n], cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaMemcpyAsync(v.data(), A->vals, sizeof(double) * rp[n], cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> perm;
  if (ordering == 0) {
    perm = rcm_ordering(n, rp.data(), ci.data());
  } else if (ordering == 2) {
    if (!user_perm) throw Error(MPEIG_E_CONFIG, "sparse_chol: null permutation");
    perm.assign(user_perm, user_perm + n);
    std::vector<char> hit(static_cast<size_t>(n), 0);
    for (int64_t k = 0; k < n; ++k) {
      if (perm[k] < 0 || perm[k] >= n || hit[perm[k]])
        throw Error(MPEIG_E_DIMENSION, "sparse_cholesky: bad permutation");
      hit[perm[k]] = 1;
    }
  } else if (ordering != 1) {
    throw Error(MPEIG_E_CONFIG, "sparse_chol: unknown ordering");
  }
  std::vector<int64_t> brp, bci;
  std::vector<double> bv;
  csr_permute<double>(n, rp.data(), ci.data(), v.data(), perm, brp, bci, bv);
  op->precision = precision;
  if (precision == MPEIG_WORKING) {  // no retry in working precision (precond.hpp:64-67)
    upload_sparse_factor(ctx, sparse_cholesky_host<double>(n, brp, bci, bv), n, op);
  } else {
    auto attempt = [&](double shift) {
      std::vector<double> sv = bv;
      if (shift != 0.0) {  // retry_sparse (precond.hpp:148-159): A + shift I, every diagonal present
        for (int64_t k = 0; k < n; ++k) {
          int64_t d = -1;
          for (int64_t p = brp[k]; p < brp[k + 1]; ++p)
            if (bci[p] == k) d = p;
          const int64_t orig = perm.empty() ? k : perm[k];
          if (d < 0)
            throw Error(MPEIG_E_NOT_PD, "precond: missing diagonal entry at " + std::to_string(orig), orig);
          sv[d] += shift;
        }
      }
      std::vector<float> fv(sv.size());
      for (size_t q = 0; q < sv.size(); ++q) {  // to_lower (precision.hpp:102-107)
        fv[q] = static_cast<float>(sv[q]);
        if (std::isinf(fv[q]) && !std::isinf(sv[q]))
          throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
      }
      upload_sparse_factor(ctx, sparse_cholesky_host<float>(n, brp, bci, fv), n, op);
    };
    try {
      attempt(0.0);
    } catch (const Error& e) {
      if (e.code != MPEIG_E_NOT_PD && e.code != MPEIG_E_OVERFLOW) throw;
      op->shift = 10.0 * 0x1p-24 * spectral_norm_estimate(ctx, A, 8, 0x5eed0123ULL);
      attempt(op->shift);
    }
  }
  if (!perm.empty()) {
    std::vector<int> p32(perm.begin(), perm.end());
    op->sp_perm = sp_upload(p32.data(), p32.size(), s);
    MPB_CUDA(cudaStreamSynchronize(s));
  }
}

// sparse_tri_solve(F, R, true) (sparse_kernels.hpp:178-225) as Preconditioner::apply
// (T = double) / apply_lower (T = float)
template <typename T>
static void sparse_chol_apply(mpeig_ctx* ctx, const mpeig_op* op, int64_t ncols, const T* R,
                              int64_t ldr, T* W, int64_t ldw) {
  const int64_t n = op->n;
  cudaStream_t s = ctx->stream;
  if (op->tri_singular >= 0)
    throw Error(MPEIG_E_SINGULAR_TRI, "sparse_tri_solve: bad diagonal", op->tri_singular);
  if (ncols <= 0) return;
  const int ni = static_cast<int>(n), ci = static_cast<int>(ncols);
  const bool wide = op->precision == MPEIG_WORKING;
  // global-memory column scratch only when a column exceeds shared memory
  const size_t fbytes = wide ? sizeof(double) : sizeof(float);
  float* gy = fbytes * n > 200 * 1024 ? op_scratch(ctx, op, (fbytes / 4) * n * ncols) : nullptr;
  ProfScope prof("precond_spchol", s, double(fbytes) * 2.0 * (op->sp_nnz * 2 + n) +
                 2.0 * sizeof(T) * n * ncols, 4.0 * op->sp_nnz * ncols);
  if (wide) {
    if constexpr (sizeof(T) == 4) {
      throw Error(MPEIG_E_CONFIG, "precond apply_lower: factor was built at working precision");
    } else {
      spchol_solve<double, double, double>(ni, ci, op->sp_Lrp, op->sp_Lci,
                                           static_cast<const double*>(op->sp_Lv), op->sp_Lsp,
                                           op->sp_Urp, op->sp_Uci,
                                           static_cast<const double*>(op->sp_Uv), op->sp_Usp,
                                           op->sp_perm, R, ldr, W, ldw, ctx->d_status + 2,
                                           reinterpret_cast<double*>(gy), s);
    }
    return;
  }
  const float* lv = static_cast<const float*>(op->sp_Lv);
  const float* uv = static_cast<const float*>(op->sp_Uv);
  if constexpr (sizeof(T) == 4) {
    spchol_solve<float, float, float>(ni, ci, op->sp_Lrp, op->sp_Lci, lv, op->sp_Lsp, op->sp_Urp,
                                      op->sp_Uci, uv, op->sp_Usp, op->sp_perm, R, ldr, W, ldw, ctx->d_status + 2, gy, s);
  } else {  // to_working(sparse_tri_solve(L, to_lower(R))), conversions fused
    status_clear(ctx);
    spchol_solve<double, float, double>(ni, ci, op->sp_Lrp, op->sp_Lci, lv, op->sp_Lsp,
                                        op->sp_Urp, op->sp_Uci, uv, op->sp_Usp, op->sp_perm, R, ldr, W, ldw, ctx->d_status + 2, gy, s);
    status_fetch(ctx);
    if (ctx->h_status[2]) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
  }
}

template <typename T>
static void dense_chol_apply(mpeig_ctx* ctx, const mpeig_op* op, int64_t ncols, const T* R,
                             int64_t ldr, T* W, int64_t ldw) {
  const int64_t n = op->n;
  cudaStream_t s = ctx->stream;
  if (op->tri_singular >= 0)
    throw Error(MPEIG_E_SINGULAR_TRI, "tri_solve: zero or subnormal diagonal", op->tri_singular);
  if (ncols <= 0) return;
  const size_t blk = static_cast<size_t>(n * ncols);
  if (op->precision == MPEIG_WORKING) {
    if constexpr (sizeof(T) == 4) {
      throw Error(MPEIG_E_CONFIG, "precond apply_lower: factor was built at working precision");
    } else {
      const double* B = R;
      int64_t ldb = ldr;
      if (W == R) {  // in place: GEMM input from a copy
        double* t = reinterpret_cast<double*>(op_scratch(ctx, op, 2 * blk));
        copy_block<double>(n, ncols, R, ldr, t, n, s);
        B = t;
        ldb = n;
      }
      chol_apply_gemm<double>(ctx, op->Lw, n, ncols, B, ldb, W, ldw);
    }
    return;
  }
  if constexpr (sizeof(T) == 4) {  // apply_lower
    const float* B = R;
    int64_t ldb = ldr;
    if (W == R) {
      float* t = op_scratch(ctx, op, blk);
      copy_block<float>(n, ncols, R, ldr, t, n, s);
      B = t;
      ldb = n;
    }
    chol_apply_gemm<float>(ctx, op->Ll, n, ncols, B, ldb, W, ldw);
  } else {  // to_working(dense_solve(L, to_lower(R)))
    float* lo = op_scratch(ctx, op, 2 * blk);
    float* hi = lo + blk;
    status_clear(ctx);
    convert_f64_to_f32(n, ncols, R, ldr, lo, n, ctx->d_status + 2, s);
    status_fetch(ctx);
    if (ctx->h_status[2]) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
    chol_apply_gemm<float>(ctx, op->Ll, n, ncols, lo, n, hi, n);
    convert_f32_to_f64(n, ncols, hi, n, W, ldw, s);
  }
}

template <typename T>
void op_apply(mpeig_ctx* ctx, const mpeig_op* op, int64_t ncols, const T* X, int64_t ldx, T* Y,
              int64_t ldy) {
  constexpr bool kW = sizeof(T) == 8;
  cudaStream_t s = ctx->stream;
  if (ncols <= 0) return;
  switch (op->kind) {
    case kOpLap3d: {
      Comm* c = dist(ctx);
      const T* dg = nullptr;  // -Laplacian + V: the row's diagonal 6 + V_i (else 6)
      if constexpr (kW) {
        dg = op->dgw;
      } else {
        if (op->dgw && op->lower_overflow)
          throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
        dg = op->dgl;
      }
      if (!op->slab || !c) {
        stencil7<T>(op->nx, op->ny, op->nz, ncols, X, ldx, Y, ldy, s, nullptr, nullptr, dg);
        return;
      }
      // z-slab of a row-sharded Laplacian: swap the boundary planes with
      // the neighbouring ranks (SURVEY §8e halo exchange), then one pass
      const int64_t sz = op->nx * op->ny;
      const size_t plane = sizeof(T) * static_cast<size_t>(sz * ncols);
      if (op->halo_bytes < 4 * plane) {
        if (op->halo) MPB_CUDA(cudaFreeAsync(op->halo, s));
        MPB_CUDA(cudaMallocAsync(&op->halo, 4 * plane, s));
        op->halo_bytes = 4 * plane;
      }
      char* h = static_cast<char*>(op->halo);
      T* slo = reinterpret_cast<T*>(h);
      T* shi = reinterpret_cast<T*>(h + plane);
      T* rlo = reinterpret_cast<T*>(h + 2 * plane);
      T* rhi = reinterpret_cast<T*>(h + 3 * plane);
      MPB_CUDA(cudaMemcpy2DAsync(slo, sizeof(T) * sz, X, sizeof(T) * ldx, sizeof(T) * sz, ncols,
                                 cudaMemcpyDeviceToDevice, s));
      MPB_CUDA(cudaMemcpy2DAsync(shi, sizeof(T) * sz, X + (op->nz - 1) * sz, sizeof(T) * ldx,
                                 sizeof(T) * sz, ncols, cudaMemcpyDeviceToDevice, s));
      // the exchange runs on a side stream while the interior planes (every
      // neighbour inside the slab) are computed; the two boundary planes
      // follow once the neighbours' planes have arrived.  Each point's sum
      // order is unchanged, so the sharded apply stays bitwise the global one.
      if (!op->halo_stream) {
        MPB_CUDA(cudaStreamCreateWithFlags(&op->halo_stream, cudaStreamNonBlocking));
        MPB_CUDA(cudaEventCreateWithFlags(&op->ev_packed, cudaEventDisableTiming));
        MPB_CUDA(cudaEventCreateWithFlags(&op->ev_halo, cudaEventDisableTiming));
      }
      MPB_CUDA(cudaEventRecord(op->ev_packed, s));
      MPB_CUDA(cudaStreamWaitEvent(op->halo_stream, op->ev_packed, 0));
      c->exchange(slo, shi, rlo, rhi, static_cast<int64_t>(plane), op->halo_stream);
      MPB_CUDA(cudaEventRecord(op->ev_halo, op->halo_stream));
      const int64_t nz = op->nz;
      const T* lo_halo = c->rank > 0 ? rlo : nullptr;
      const T* hi_halo = c->rank + 1 < c->nranks ? rhi : nullptr;
      auto dgz = [&](int64_t z) -> const T* { return dg ? dg + z * sz : nullptr; };
      if (nz >= 3)  // interior planes 1 .. nz-2: z-neighbours are X's own planes
        stencil7<T>(op->nx, op->ny, nz - 2, ncols, X + sz, ldx, Y + sz, ldy, s, X,
                    X + (nz - 1) * sz, dgz(1), ldx, ldx);
      MPB_CUDA(cudaStreamWaitEvent(s, op->ev_halo, 0));
      if (nz == 1) {
        stencil7<T>(op->nx, op->ny, 1, ncols, X, ldx, Y, ldy, s, lo_halo, hi_halo, dgz(0));
      } else {
        // plane 0: below = the lower neighbour's plane (packed), above = X's plane 1;
        // plane nz-1: below = X's plane nz-2, above = the upper neighbour's plane
        stencil7<T>(op->nx, op->ny, 1, ncols, X, ldx, Y, ldy, s, lo_halo, X + sz, dgz(0), 0, ldx);
        stencil7<T>(op->nx, op->ny, 1, ncols, X + (nz - 1) * sz, ldx, Y + (nz - 1) * sz, ldy, s,
                    X + (nz - 2) * sz, hi_halo, dgz(nz - 1), ldx, 0);
      }
      return;
    }
    case kOpLap2d:
      stencil5<T>(op->nx, op->ny, ncols, X, ldx, Y, ldy, s);
      return;
    case kOpCsr: {
      const T* vals;
      if constexpr (kW) {
        vals = op->vals;
      } else {
        if (op->lower_overflow) throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
        vals = op->vals_l;
      }
      Comm* c = dist(ctx);
      if (!op->slab || !c) {
        csr_spmm<T>(op->n, op->rp32, op->ci32, vals, op->nnz, ncols, X, ldx, Y, ldy, s);
        return;
      }
      // row block of a sharded CSR matrix (SURVEY §8e ghost rows): pack the
      // rows the peers need, exchange them on a side stream while the rows
      // without ghost entries are computed, then the boundary rows
      const int nr = c->nranks;
      const size_t row_bytes = sizeof(T) * static_cast<size_t>(ncols);
      const size_t need = row_bytes * static_cast<size_t>(op->n_send + 2 * op->n_ghost);
      if (op->halo_bytes < need) {
        if (op->halo) MPB_CUDA(cudaFreeAsync(op->halo, s));
        MPB_CUDA(cudaMallocAsync(&op->halo, std::max<size_t>(need, 16), s));
        op->halo_bytes = std::max<size_t>(need, 16);
      }
      T* sendb = static_cast<T*>(op->halo);
      T* recvb = sendb + op->n_send * ncols;  // per peer: rows_q x ncols blocks
      T* G = recvb + op->n_ghost * ncols;     // the ghost rows, ld n_ghost
      for (int q = 0; q < nr; ++q)
        gather_rows<T>(op->gx_send_rows[q], op->gx_send_idx + op->gx_send_off[q], ncols, X, ldx,
                       sendb + op->gx_send_off[q] * ncols, op->gx_send_rows[q], s);
      if (!op->halo_stream) {
        MPB_CUDA(cudaStreamCreateWithFlags(&op->halo_stream, cudaStreamNonBlocking));
        MPB_CUDA(cudaEventCreateWithFlags(&op->ev_packed, cudaEventDisableTiming));
        MPB_CUDA(cudaEventCreateWithFlags(&op->ev_halo, cudaEventDisableTiming));
      }
      MPB_CUDA(cudaEventRecord(op->ev_packed, s));
      MPB_CUDA(cudaStreamWaitEvent(op->halo_stream, op->ev_packed, 0));
      std::vector<int64_t> sb(nr), so(nr), rb(nr), ro(nr);
      for (int q = 0; q < nr; ++q) {
        sb[q] = static_cast<int64_t>(row_bytes) * op->gx_send_rows[q];
        so[q] = static_cast<int64_t>(row_bytes) * op->gx_send_off[q];
        rb[q] = static_cast<int64_t>(row_bytes) * op->gx_recv_rows[q];
        ro[q] = static_cast<int64_t>(row_bytes) * op->gx_recv_off[q];
      }
      c->alltoallv(sendb, sb.data(), so.data(), recvb, rb.data(), ro.data(), op->halo_stream);
      for (int q = 0; q < nr; ++q)
        if (op->gx_recv_rows[q] > 0)
          MPB_CUDA(cudaMemcpy2DAsync(G + op->gx_recv_off[q], sizeof(T) * op->n_ghost,
                                     recvb + op->gx_recv_off[q] * ncols,
                                     sizeof(T) * op->gx_recv_rows[q], sizeof(T) * op->gx_recv_rows[q],
                                     ncols, cudaMemcpyDeviceToDevice, op->halo_stream));
      MPB_CUDA(cudaEventRecord(op->ev_halo, op->halo_stream));
      csr_spmm_rows<T>(op->n_inner, op->rows_inner, op->rp32, op->ci32, vals, ncols, X, ldx, op->n,
                       nullptr, 0, Y, ldy, s);
      MPB_CUDA(cudaStreamWaitEvent(s, op->ev_halo, 0));
      csr_spmm_rows<T>(op->n_bnd, op->rows_bnd, op->rp32, op->ci32, vals, ncols, X, ldx, op->n,
                       op->n_ghost ? G : nullptr, op->n_ghost, Y, ldy, s);
      return;
    }
    case kOpDense: {
      // herm_product (dense_kernels.hpp:66-72): a plain library GEMM (cuBLAS
      // DGEMM 35 TF/s = 95 % of the DMMA peak at cfg3, scripts/dense_ax_bench.py)
      const int n = static_cast<int>(op->n), c = static_cast<int>(ncols);
      ProfScope prof("dense_apply", s, double(sizeof(T)) * (double(n) * n + 2.0 * n * c),
                     2.0 * n * double(n) * c);
      if constexpr (kW) {
        const double one = 1.0, zero = 0.0;
        cublas_check(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, n, c, n, &one, op->A,
                                 static_cast<int>(op->lda), X, static_cast<int>(ldx), &zero, Y,
                                 static_cast<int>(ldy)),
                     "cublasDgemm");
      } else {
        // the fp32 stage's A X: the tcgen05 block update (faster than cuBLAS SGEMM here)
        if (op->lower_overflow) throw Error(MPEIG_E_OVERFLOW, "to_lower: matrix exceeds binary32 range");
        gemm_tn<float>(op->n, op->n, ncols, 1.f, op->Al, op->lda, X, ldx, 0.f, nullptr, 0, Y, ldy, s);
      }
      return;
    }
    case kOpDeviceCb: {
      mpeig_apply_fn f = kW ? op->dev_w : op->dev_l;
      if (!f) throw Error(MPEIG_E_CONFIG, "operator callback missing for this precision");
      const int rc = f(op->user, op->n, ncols, X, ldx, Y, ldy, s);
      if (rc != 0) throw Error(MPEIG_E_CALLBACK, "operator callback failed", rc);
      return;
    }
    case kOpHostCb: {
      mpeig_host_apply_fn f = kW ? op->host_w : op->host_l;
      if (!f) throw Error(MPEIG_E_CONFIG, "host operator callback missing for this precision");
      std::vector<T> hx(static_cast<size_t>(op->n * ncols)), hy(hx.size());
      MPB_CUDA(cudaMemcpy2DAsync(hx.data(), sizeof(T) * op->n, X, sizeof(T) * ldx, sizeof(T) * op->n,
                                 ncols, cudaMemcpyDeviceToHost, s));
      MPB_CUDA(cudaStreamSynchronize(s));
      const int rc = f(op->user, op->n, ncols, hx.data(), hy.data());
      if (rc != 0) throw Error(MPEIG_E_CALLBACK, "host operator callback failed", rc);
      MPB_CUDA(cudaMemcpy2DAsync(Y, sizeof(T) * ldy, hy.data(), sizeof(T) * op->n, sizeof(T) * op->n,
                                 ncols, cudaMemcpyHostToDevice, s));
      MPB_CUDA(cudaStreamSynchronize(s));
      return;
    }
    case kOpJacobi:
      precond_apply<T>(ctx, op, ncols, X, ldx, Y, ldy);
      return;
    case kOpDenseChol:
      dense_chol_apply<T>(ctx, op, ncols, X, ldx, Y, ldy);
      return;
    case kOpSparseChol:
      sparse_chol_apply<T>(ctx, op, ncols, X, ldx, Y, ldy);
      return;
  }
}

// Jacobi mode for a block of precision T (Preconditioner::apply / apply_lower)
template <typename T>
static int jacobi_mode(const mpeig_op* op, const void** dinv) {
  if constexpr (sizeof(T) == 8) {
    if (op->precision == MPEIG_WORKING) {
      *dinv = op->dinv;
      return kResidJacobiT;
    }
    *dinv = op->dinvf;
    return kResidSandwich;
  } else {
    if (op->precision != MPEIG_LOWER)
      throw Error(MPEIG_E_CONFIG, "precond apply_lower: factor was built at working precision");
    *dinv = op->dinvf;
    return kResidJacobiT;
  }
}

template <typename T>
void precond_apply(mpeig_ctx* ctx, const mpeig_op* T_op, int64_t ncols, const T* R, int64_t ldr,
                   T* W, int64_t ldw) {
  if (T_op->kind != kOpJacobi) {
    op_apply<T>(ctx, T_op, ncols, R, ldr, W, ldw);
    return;
  }
  const void* dinv = nullptr;
  const int mode = jacobi_mode<T>(T_op, &dinv);
  status_clear(ctx);
  jacobi_apply<T>(mode, T_op->n, ncols, R, ldr, dinv, W, ldw, ctx->d_status + 2, ctx->stream);
  status_fetch(ctx);
  if (ctx->h_status[2]) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
}

// ---------------------------------------------------------------- workspace
template <typename T>
Work<T>::Work(mpeig_ctx* c, int64_t n_, int64_t m_, int64_t smax_) : ctx(c), n(n_), m(m_), smax(smax_) {
  s = ctx->stream;
  ld = padded_ld(n);
  S.alloc(static_cast<size_t>(ld * smax), s);
  AS.alloc(static_cast<size_t>(ld * smax), s);
  S2.alloc(static_cast<size_t>(ld * smax), s);
  AS2.alloc(static_cast<size_t>(ld * smax), s);
  V.alloc(static_cast<size_t>(ld * m), s);
  G.alloc(static_cast<size_t>(smax * smax), s);
  evals.alloc(static_cast<size_t>(smax), s);
  coef.alloc(static_cast<size_t>(smax * smax), s);
  small.alloc(static_cast<size_t>(8 * m * m + 4 * smax * smax), s);
  smallf.alloc(static_cast<size_t>(2 * m * m), s);
  int64_t gw = 0;
  gw = std::max(gw, gram_workspace_elems<T>(n, smax, smax));
  gw = std::max(gw, gram_workspace_elems<T>(n, 2 * m, m));
  gw = std::max(gw, gram_workspace_elems<T>(n, m, m));
  gw = std::max(gw, gram_workspace_elems<T>(n, m, 1));
  gramw.alloc_zero(static_cast<size_t>(gw), s);
  tsqr_w.alloc_zero(static_cast<size_t>(tsqr_workspace_elems<T, T>(n, m)), s);
  if constexpr (sizeof(T) == 8)
    tsqr_f.alloc_zero(static_cast<size_t>(tsqr_workspace_elems<double, float>(n, m)), s);
  rw.alloc(static_cast<size_t>(std::max<int64_t>(resid_workspace_elems(n, m), kNumSMs * 2) + 4 * m + 8), s);
  theta.alloc(static_cast<size_t>(smax), s);
  theta_prev.alloc(static_cast<size_t>(smax), s);
  // cuSOLVER syevd workspace for the largest projected problem
  int lw = 0;
  if constexpr (sizeof(T) == 8)
    cusolver_check(cusolverDnDsyevd_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, static_cast<int>(smax), G.p,
                                               static_cast<int>(smax), evals.p, &lw),
                   "syevd_bufferSize");
  else
    cusolver_check(cusolverDnSsyevd_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, static_cast<int>(smax), G.p,
                                               static_cast<int>(smax), evals.p, &lw),
                   "syevd_bufferSize");
  lwork = lw;
  eigw.alloc(static_cast<size_t>(lw > 0 ? lw : 1), s);
  if (Comm* c = dist(ctx)) {
    const int64_t P = c->nranks, mm = m * m;
    rstk.alloc(static_cast<size_t>(P * mm), s);
    rstk2.alloc(static_cast<size_t>(P * mm), s);
    tsqr_w2.alloc_zero(static_cast<size_t>(tsqr_workspace_elems<T, T>(P * m, m)), s);
    rstkf.alloc(static_cast<size_t>(P * mm), s);
    rstk2f.alloc(static_cast<size_t>(P * mm), s);
    tsqr_f2.alloc_zero(static_cast<size_t>(tsqr_workspace_elems<float, float>(P * m, m)), s);
  }
}

template <typename T>
T* Work<T>::L() { return small.p; }
template <typename T>
T* Work<T>::Uinv() { return small.p + m * m; }
template <typename T>
T* Work<T>::Rw() { return small.p + 2 * m * m; }
template <typename T>
T* Work<T>::Rinv() { return small.p + 3 * m * m; }
template <typename T>
T* Work<T>::Lt() { return small.p + 4 * m * m; }
template <typename T>
T* Work<T>::scratch() { return small.p + 8 * m * m; }
template <typename T>
double* Work<T>::rnorm() { return rw.p + (rw.count - 4 * m - 8); }
template <typename T>
double* Work<T>::xnorm() { return rnorm() + m; }
template <typename T>
double* Work<T>::dscal() { return rnorm() + 2 * m; }

// ----------------------------------------------------------- small eig
// small_herm_eig (small_eig.hpp:92-218) -> cuSOLVER syevd on the device:
// ascending values, vectors overwrite G.  info > 0 -> NoConvergence.
template <typename T>
void small_eig(Work<T>& w, int64_t sdim, T* G, int64_t ldg, T* vals) {
  mpeig_ctx* ctx = w.ctx;
  if (ctx->eig_backend == 0 && small_syev_supported<T>(sdim)) {
    small_syev<T>(sdim, G, ldg, vals, ctx->d_status + 3, w.s, ctx->ql_exact);
    return;
  }
  ProfScope prof("small_eig_cusolver", w.s, 0, 0);
  if (ctx->eig_backend == 2) {  // diagnostic: cuSOLVER's Jacobi (syevj)
    syevjInfo_t jp;
    cusolverDnCreateSyevjInfo(&jp);
    cusolverDnXsyevjSetTolerance(jp, 0.0);
    cusolverDnXsyevjSetMaxSweeps(jp, 100);
    int lw = 0;
    if constexpr (sizeof(T) == 8)
      cusolverDnDsyevj_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  static_cast<int>(sdim), G, static_cast<int>(ldg), vals, &lw, jp);
    else
      cusolverDnSsyevj_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                  static_cast<int>(sdim), G, static_cast<int>(ldg), vals, &lw, jp);
    DevBuf<T> wk(static_cast<size_t>(lw > 0 ? lw : 1), w.s);
    if constexpr (sizeof(T) == 8)
      cusolverDnDsyevj(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                       static_cast<int>(sdim), G, static_cast<int>(ldg), vals, wk.p, lw,
                       ctx->d_status + 3, jp);
    else
      cusolverDnSsyevj(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                       static_cast<int>(sdim), G, static_cast<int>(ldg), vals, wk.p, lw,
                       ctx->d_status + 3, jp);
    MPB_CUDA(cudaStreamSynchronize(w.s));
    cusolverDnDestroySyevjInfo(jp);
    return;
  }
  if constexpr (sizeof(T) == 8)
    cusolver_check(cusolverDnDsyevd(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    static_cast<int>(sdim), G, static_cast<int>(ldg), vals, w.eigw.p,
                                    w.lwork, ctx->d_status + 3),
                   "cusolverDnDsyevd");
  else
    cusolver_check(cusolverDnSsyevd(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                    static_cast<int>(sdim), G, static_cast<int>(ldg), vals, w.eigw.p,
                                    w.lwork, ctx->d_status + 3),
                   "cusolverDnSsyevd");
}

// ---------------------------------------------------- row-sharded helpers
// G = A^T B summed over the ranks' rows (then hermitized): the Gram products
// are the solver's only O(n)-reductions besides the column norms.
template <typename T>
static void dgram(Work<T>& w, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B,
                  int64_t ldb, T* G, int64_t ldg, int sym) {
  Comm* c = dist(w.ctx);
  if (!c) {
    gram<T>(w.n, ka, A, lda, kb, B, ldb, G, ldg, sym, w.gramw.p, w.s);
    return;
  }
  if (ldg != ka) throw Error(MPEIG_E_OTHER, "dgram: Gram leading dimension must equal its rows");
  gram<T>(w.n, ka, A, lda, kb, B, ldb, G, ldg, 0, w.gramw.p, w.s);
  c->allreduce_sum(G, ka * kb, w.s);
  if (sym) small_symmetrize<T>(ka, G, ldg, w.s);
}

// ||x||^2 of one column, summed over the ranks
template <typename T>
static void dfrob(Work<T>& w, int64_t n, const T* v, int64_t ld, double* d2) {
  frob_sq<T>(n, 1, v, ld, d2, w.rw.p, w.s);
  if (Comm* c = dist(w.ctx)) c->allreduce_sum(d2, 1, w.s);
}

// residual + norms (+ fused f_T); the norms' sums of squares are reduced over
// the ranks before the square root
template <typename T>
static void dresidual(Work<T>& w, int mode, int64_t m, const T* X, const T* AX, const void* dinv,
                      T* Wdst, int* ovf) {
  Comm* c = dist(w.ctx);
  residual_precond<T>(mode, w.n, m, X, w.ld, AX, w.ld, w.theta.p, dinv, Wdst, w.ld, w.rnorm(),
                      w.xnorm(), ovf, w.rw.p, w.s, c ? 1 : 0);
  if (c) {
    c->allreduce_sum(w.rnorm(), 2 * m, w.s);  // rnorm, xnorm are adjacent
    norms_sqrt<T>(2 * m, w.rnorm(), w.s);
  }
}

// R of the row-sharded block: each rank's TSQR R, gathered, stacked and
// factored again (a TSQR tree whose top level spans the ranks); every rank
// computes the same global R, then Rw = R (working precision), Rinv = R^-1.
template <typename T>
static void dgram(Work<T>& w, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B,
                  int64_t ldb, T* G, int64_t ldg, int sym);

template <typename T>
static void tsqr_R(Work<T>& w, int64_t m, T* W, int64_t ldw, bool lower, int* status) {
  const int64_t n = w.n;
  cudaStream_t s = w.s;
  Comm* c = dist(w.ctx);
  if (!tsqr_fits<T, T>(n, m) || (lower && !tsqr_fits<T, float>(n, m))) {
    // blocks too wide for a one-CTA Householder tree (cfg5's m = 192): R from
    // the Cholesky factor of W^T W, R = L^T, R^-1 = L^-T.  Any R that makes
    // W R^-1 well conditioned serves the next CholQR pass of qr_core; a
    // breakdown (cond(W) ~ u^-1/2) is reported as NotPositiveDefinite like
    // mixed_qr's (ortho.hpp:173-186) and falls back the same way.
    dgram<T>(w, m, W, ldw, m, W, ldw, w.G.p, m, 1);
    small_cholesky_inv<T>(m, w.G.p, m, w.L(), w.Rinv(), status, s);
    small_transpose<T>(m, m, w.L(), m, w.Rw(), m, s);
    return;
  }
  if (!c) {
    if constexpr (sizeof(T) == 8) {
      if (lower) {
        // fp32 R_l, then R_l in fp64 and R_l^-1 (fused into the TSQR root)
        tsqr_r<double, float>(n, m, W, ldw, w.smallf.p, m, w.tsqr_f.p, status, s, w.Rw(), w.Rinv());
        return;
      }
    }
    tsqr_r<T, T>(n, m, W, ldw, w.Rw(), m, w.tsqr_w.p, status, s, nullptr, w.Rinv());
    return;
  }
  const int64_t P = c->nranks, mm = m * m;
  if constexpr (sizeof(T) == 8) {
    if (lower) {
      tsqr_r<double, float>(n, m, W, ldw, w.smallf.p, m, w.tsqr_f.p, status, s, nullptr, nullptr, 0);
      c->allgather(w.smallf.p, w.rstkf.p, static_cast<int64_t>(sizeof(float)) * mm, s);
      for (int64_t r = 0; r < P; ++r)
        MPB_CUDA(cudaMemcpy2DAsync(w.rstk2f.p + r * m, sizeof(float) * P * m, w.rstkf.p + r * mm,
                                   sizeof(float) * m, sizeof(float) * m, m, cudaMemcpyDeviceToDevice,
                                   s));
      tsqr_r<float, float>(P * m, m, w.rstk2f.p, P * m, w.smallf.p, m, w.tsqr_f2.p, status, s,
                           nullptr, nullptr, 0);
      tsqr_epilogue<double, float>(m, w.smallf.p, m, w.Rw(), w.Rinv(), status, s);
      return;
    }
  }
  tsqr_r<T, T>(n, m, W, ldw, w.Rw(), m, w.tsqr_w.p, status, s, nullptr, nullptr, 0);
  c->allgather(w.Rw(), w.rstk.p, static_cast<int64_t>(sizeof(T)) * mm, s);
  for (int64_t r = 0; r < P; ++r)
    MPB_CUDA(cudaMemcpy2DAsync(w.rstk2.p + r * m, sizeof(T) * P * m, w.rstk.p + r * mm,
                               sizeof(T) * m, sizeof(T) * m, m, cudaMemcpyDeviceToDevice, s));
  tsqr_r<T, T>(P * m, m, w.rstk2.p, P * m, w.Rw(), m, w.tsqr_w2.p, status, s, nullptr, w.Rinv());
}

// CholQR's Gram + Cholesky of X (default w.V), fused on one GPU; tau2 > 0 is
// the conditioning guard of the speculative CholQR (warp_cholesky_inv)
template <typename T>
static void gram_chol(Work<T>& w, int64_t m, int* status, const T* X = nullptr, int64_t ldx = 0,
                      T tau2 = T(0)) {
  if (!X) {
    X = w.V.p;
    ldx = w.ld;
  }
  if (!dist(w.ctx) &&
      gram_cholesky<T>(w.n, m, X, ldx, w.G.p, w.gramw.p, w.L(), w.Uinv(), status, w.s, tau2))
    return;
  dgram<T>(w, m, X, ldx, m, X, ldx, w.G.p, m, 1);
  small_cholesky_inv<T>(m, w.G.p, m, w.L(), w.Uinv(), status, w.s, tau2);
}

// guard of the CholQR first pass (option "spec_qr" = k > 0: fp64 1e-k)
template <typename T>
static T cholqr_tau2(const mpeig_ctx* ctx) {
  return sizeof(T) == 8 ? T(std::pow(10.0, -std::max(1, ctx->spec_qr))) : T(1e-4);
}
// guard of the single CholQR pass of the second project + QR round (fp64
// stage): every equilibrated pivot >= 1/2, i.e. cond(W) ~ 1, so one pass is
// orthonormal to ~eps * cond^2 ~ eps (W is the first round's Q minus an
// O(u cond) overlap).  The fp32 stage keeps both passes: its length is set by
// how well the fp32 iteration holds orthogonality, and one
// fp32 pass measurably lengthens it (lap2d 5x500: 880 vs 797 iterations).
template <typename T>
constexpr T kCholQrSingleTau2 = T(0.25);

// W <- W C (m x m) in place.  Every GEMM kernel reads a row block's inputs
// before writing it only within ONE output column tile (<= 64 columns:
// kernels.cuh gemm_tn); a wider block would let a later column tile read
// columns an earlier tile of the same rows already overwrote, so above that
// the product goes through the QR scratch w.V and is copied back.
template <typename T>
static void gemm_right_inplace(Work<T>& w, int64_t m, T* W, int64_t ldw, const T* C) {
  if (gemm_inplace_ok(sizeof(T) == 8, w.n, m, m)) {
    gemm_tn<T>(w.n, m, m, T(1), W, ldw, C, m, T(0), nullptr, 0, W, ldw, w.s);
    return;
  }
  gemm_tn<T>(w.n, m, m, T(1), W, ldw, C, m, T(0), nullptr, 0, w.V.p, w.ld, w.s);
  copy_block<T>(w.n, m, w.V.p, w.ld, W, ldw, w.s);
}

// ------------------------------------------------------------- QR family
// Q (in place) by "R from a Householder TSQR, then Cholesky-QR of W R^-1":
//   lower = true  (T = double): Alg. 2 / mixed_qr (ortho.hpp:173-186) --
//                 fp32 Householder R_l, V = W R_l^-1 in fp64, CholQR(V).
//   lower = false: Householder QR (ortho.hpp:127-140) equivalent -- the same
//                 structure with an R of the block's own precision; Q is the
//                 unique positive-diagonal Q to rounding.
// Returns the status {code, index}; W is overwritten only on success.
template <typename T>
static int qr_core(Work<T>& w, int64_t m, T* W, int64_t ldw, bool lower, T* Rout, int64_t* idx) {
  mpeig_ctx* ctx = w.ctx;
  cudaStream_t s = w.s;
  const int64_t n = w.n;
  status_clear(ctx);
  tsqr_R<T>(w, m, W, ldw, lower, ctx->d_status);
  gemm_tn<T>(n, m, m, T(1), W, ldw, w.Rinv(), m, T(0), nullptr, 0, w.V.p, w.ld, s);
  gram_chol<T>(w, m, ctx->d_status);
  status_fetch(ctx);
  const int code = ctx->h_status[0];
  *idx = ctx->h_status[1];
  if (code != 0) return code;
  gemm_tn<T>(n, m, m, T(1), w.V.p, w.ld, w.Uinv(), m, T(0), nullptr, 0, W, ldw, s);
  if (Rout) {
    // R = R_chol R_w with R_chol = L^T   (ortho.hpp:184)
    small_transpose<T>(m, m, w.L(), m, w.Lt(), m, s);
    small_matmul<T>(m, m, m, w.Lt(), m, w.Rw(), m, Rout, m, s);
  }
  return 0;
}

// detail::orthonormal_q (eigensolvers.hpp:55-70)
template <typename T>
void orthonormal_q(Work<T>& w, int64_t m, T* W, int64_t ldw, bool use_mixed) {
  int64_t idx = 0;
  if constexpr (sizeof(T) == 8) {
    if (use_mixed) {
      const int st = qr_core<T>(w, m, W, ldw, true, nullptr, &idx);
      if (st == 0) return;
      if (st == MPEIG_E_RANK_DEFICIENT) throw Error(st, "householder_qr: column vanished", idx);
      if (st == MPEIG_E_SINGULAR_TRI) throw Error(st, "tri_solve: zero or subnormal diagonal", idx);
      // NotPositiveDefinite / OverflowError -> Householder at working precision
    }
  }
  const int st = qr_core<T>(w, m, W, ldw, false, nullptr, &idx);
  if (st == 0) return;
  // a vanished column (or a numerically singular block) is rank deficiency
  throw Error(MPEIG_E_RANK_DEFICIENT, "householder_qr: column vanished",
              st == MPEIG_E_RANK_DEFICIENT || st == MPEIG_E_SINGULAR_TRI ? idx : m - 1);
}

// Q in place by two Cholesky-QR passes, the first guarded on the equilibrated
// pivots (cholqr_tau2); true on success, W untouched otherwise (the caller then
// runs the reference's QR chain).  Q of a full-rank W is unique to rounding, so
// this is the reference's mixed_qr / householder_qr Q without the TSQR's
// column-serial chain.
template <typename T>
static bool guarded_cholqr2(Work<T>& w, int64_t m, T* W, int64_t ldw) {
  cudaStream_t s = w.s;
  status_clear(w.ctx);
  gram_chol<T>(w, m, w.ctx->d_status, W, ldw, cholqr_tau2<T>(w.ctx));
  gemm_tn<T>(w.n, m, m, T(1), W, ldw, w.Uinv(), m, T(0), nullptr, 0, w.V.p, w.ld, s);
  gram_chol<T>(w, m, w.ctx->d_status);
  status_fetch(w.ctx);
  if (w.ctx->h_status[0] != 0) return false;
  gemm_tn<T>(w.n, m, m, T(1), w.V.p, w.ld, w.Uinv(), m, T(0), nullptr, 0, W, ldw, s);
  return true;
}

// orthonormalize_dropping (ortho.hpp:205-250): two-pass Gram-Schmidt that
// drops columns whose projected norm falls below drop_tol * original norm.
template <typename T>
int64_t ortho_dropping(Work<T>& w, int64_t m, T* W, int64_t ldw, T drop_tol) {
  mpeig_ctx* ctx = w.ctx;
  cudaStream_t s = w.s;
  const int64_t n = w.n;
  T* v = w.V.p;  // column 0 of the QR scratch
  T* g = w.G.p;
  double* d2 = w.dscal();
  double h2 = 0;
  int64_t kept = 0;
  for (int64_t j = 0; j < m; ++j) {
    copy_block<T>(n, 1, W + j * ldw, ldw, v, w.ld, s);
    dfrob<T>(w, n, v, w.ld, d2);
    MPB_CUDA(cudaMemcpyAsync(&h2, d2, sizeof(double), cudaMemcpyDeviceToHost, s));
    MPB_CUDA(cudaStreamSynchronize(s));
    const T n0 = static_cast<T>(std::sqrt(h2));
    if (n0 == T(0)) continue;
    for (int pass = 0; pass < 2 && kept > 0; ++pass) {
      dgram<T>(w, kept, W, ldw, 1, v, w.ld, g, kept, 0);
      gemm_tn<T>(n, kept, 1, T(-1), W, ldw, g, kept, T(1), v, w.ld, v, w.ld, s);
    }
    dfrob<T>(w, n, v, w.ld, d2);
    MPB_CUDA(cudaMemcpyAsync(&h2, d2, sizeof(double), cudaMemcpyDeviceToHost, s));
    MPB_CUDA(cudaStreamSynchronize(s));
    const T nv = static_cast<T>(std::sqrt(h2));
    if (nv <= drop_tol * n0) continue;
    scale_block<T>(n, 1, T(1) / nv, v, w.ld, W + kept * ldw, ldw, s);
    ++kept;
  }
  return kept;
}

// detail::orthonormal_q_dropping (eigensolvers.hpp:74-85)
template <typename T>
int64_t orthonormal_q_dropping(Work<T>& w, int64_t m, T* W, int64_t ldw, bool use_mixed,
                               int64_t* dropped, bool second) {
  *dropped = 0;
  if (w.ctx->spec_qr && m > 0 && second && sizeof(T) == 8) {
    // second round (qr_spec): one guarded CholQR pass, in place
    cudaStream_t s = w.s;
    status_clear(w.ctx);
    gram_chol<T>(w, m, w.ctx->d_status, W, ldw, kCholQrSingleTau2<T>);
    status_fetch(w.ctx);
    if (w.ctx->h_status[0] == 0) {
      gemm_right_inplace<T>(w, m, W, ldw, w.Uinv());
      return m;
    }
  } else if (w.ctx->spec_qr && m > 0) {
    // the guarded Cholesky-QR of qr_spec first (so the eager, careful and
    // speculative paths take identical steps); W is overwritten only when
    // both passes succeed, else the reference's QR chain below runs on it
    if (guarded_cholqr2<T>(w, m, W, ldw)) return m;
  }
  try {
    orthonormal_q<T>(w, m, W, ldw, use_mixed);
    return m;
  } catch (const Error& e) {
    if (e.code != MPEIG_E_RANK_DEFICIENT) throw;
  }
  const T tol = std::sqrt(std::numeric_limits<T>::epsilon());
  const int64_t kept = ortho_dropping<T>(w, m, W, ldw, tol);
  *dropped = m - kept;
  return kept;
}

// block_project_out (ortho.hpp:190-200): W -= B (B^T W), `passes` times
template <typename T>
void project_out(Work<T>& w, const T* B, int64_t b, int64_t ldb, T* W, int64_t wc, int64_t ldw,
                 int passes) {
  if (b == 0 || wc == 0) return;
  for (int p = 0; p < passes; ++p) {
    dgram<T>(w, b, B, ldb, wc, W, ldw, w.G.p, b, 0);
    gemm_tn<T>(w.n, b, wc, T(-1), B, ldb, w.G.p, b, T(1), W, ldw, W, ldw, w.s);
  }
}

// detail::ritz_rotate (eigensolvers.hpp:89-102): X <- X V, AX <- AX V,
// theta = eig(X^T AX).  Reads S/AS column block 0, writes S2/AS2, swaps.
template <typename T>
void ritz_rotate(Work<T>& w) {
  const int64_t m = w.m;
  dgram<T>(w, m, w.S.p, w.ld, m, w.AS.p, w.ld, w.G.p, m, 1);
  small_eig<T>(w, m, w.G.p, m, w.evals.p);
  gemm_tn_pair<T>(w.n, m, m, w.S.p, w.AS.p, w.ld, w.G.p, m, w.S2.p, w.AS2.p, w.ld, w.s);
  MPB_CUDA(cudaMemcpyAsync(w.theta.p, w.evals.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, w.s));
  std::swap(w.S, w.S2);
  std::swap(w.AS, w.AS2);
}

// ------------------------------------------------------------ iteration
// Residual + norms (+ fused Jacobi f_T into Wdst when possible), then one
// D2H of {theta, ||r||, ||x||, status}.  Returns true if f_T was fused.
template <typename T>
static bool residual_step(Work<T>& w, const mpeig_op* T_op, const T* X, const T* AX, T* Wdst,
                          std::vector<double>& theta, std::vector<double>& rn,
                          std::vector<double>& xn, bool* overflow) {
  mpeig_ctx* ctx = w.ctx;
  const int64_t m = w.m;
  const bool fused = T_op && T_op->kind == kOpJacobi;
  const void* dinv = nullptr;
  int mode = kResidPlain;
  if (fused) mode = jacobi_mode<T>(T_op, &dinv);
  status_clear(ctx);
  dresidual<T>(w, mode, m, X, AX, dinv, fused ? Wdst : w.V.p, ctx->d_status + 2);
  std::vector<T> th(static_cast<size_t>(m));
  MPB_CUDA(cudaMemcpyAsync(th.data(), w.theta.p, sizeof(T) * m, cudaMemcpyDeviceToHost, w.s));
  MPB_CUDA(cudaMemcpyAsync(ctx->h_pinned, w.rnorm(), sizeof(double) * 2 * m, cudaMemcpyDeviceToHost,
                           w.s));
  status_fetch(ctx);
  theta.resize(m);
  rn.resize(m);
  xn.resize(m);
  for (int64_t j = 0; j < m; ++j) {
    theta[j] = static_cast<double>(th[j]);
    // col_norm is computed in real_t<T> (dense_matrix.hpp:74-82)
    rn[j] = static_cast<double>(static_cast<T>(ctx->h_pinned[j]));
    xn[j] = static_cast<double>(static_cast<T>(ctx->h_pinned[m + j]));
  }
  *overflow = ctx->h_status[2] != 0;
  return fused;
}

// converged_count (eigensolvers.hpp:25-43): prefix rule
static int64_t converged_prefix(double a_norm_est, const std::vector<double>& theta,
                                const std::vector<double>& rn, const std::vector<double>& xn,
                                double tol) {
  int64_t n_c = 0;
  for (size_t j = 0; j < theta.size(); ++j) {
    const double thr = tol * (a_norm_est + std::abs(theta[j])) * xn[j];
    if (rn[j] <= thr)
      ++n_c;
    else
      break;
  }
  return n_c;
}

struct EvTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit EvTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EvTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start() { cudaEventRecord(a, s); }
  double stop() {  // seconds; synchronises on the end event
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
  }
};

// Eager reference-shaped stage: one host round trip per decision point.  Used
// when the operator or preconditioner cannot run without the host (host
// BlockOperator adapter, user callbacks that synchronise) and as the
// semantic baseline of the speculative stage below.
template <typename T>
StageResult lobpcg_stage_eager(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const T* X0,
                               int64_t ldx0, int64_t m, const mpeig_cfg& cfg, const mpeig_op* T_op,
                               double a_norm_est, const mpeig_stage_opts& opt,
                               mpeig_history_sink sink, void* sink_user, T* Xout, int64_t ldxout,
                               mpeig_timings* tim) {
  if (n <= 0 || m <= 0) throw Error(MPEIG_E_DIMENSION, "lobpcg_stage: empty block");
  const int64_t smax = 3 * m;
  Work<T> w(ctx, n, m, smax);
  cudaStream_t s = w.s;
  EvTimer timer(s);
  mpeig_timings local{};
  mpeig_timings& tm = tim ? *tim : local;

  // X = X0, AX = A X, Ritz rotation (eigensolvers.hpp:207-216)
  copy_block<T>(n, m, X0, ldx0, w.S.p, w.ld, s);
  op_apply<T>(ctx, A, m, w.S.p, w.ld, w.AS.p, w.ld);
  timer.start();
  ritz_rotate<T>(w);
  tm.projected_eig += timer.stop();
  int64_t p = 0;

  double best_metric = std::numeric_limits<double>::infinity();
  int64_t since_improvement = 0;
  constexpr int64_t kStagnationWindow = 40;

  std::vector<double> theta, rn, xn;
  StageResult res;
  for (int64_t iter = 0;; ++iter) {
    T* X = w.S.p;
    T* AX = w.AS.p;
    T* Wslot = w.S.p + (m + p) * w.ld;
    bool overflow = false;
    const bool fused = residual_step<T>(w, T_op, X, AX, Wslot, theta, rn, xn, &overflow);
    const int64_t n_c = converged_prefix(a_norm_est, theta, rn, xn, opt.tol);

    if (opt.stagnation_exit) {
      double metric = 0;
      for (int64_t j = 0; j < cfg.k && j < m; ++j) {
        const double denom = (a_norm_est + std::abs(theta[j])) * xn[j];
        const double ratio = denom > 0 ? rn[j] / denom : std::numeric_limits<double>::infinity();
        if (ratio > metric) metric = ratio;
      }
      if (metric < 0.99 * best_metric) {
        best_metric = metric;
        since_improvement = 0;
      } else {
        ++since_improvement;
      }
    }
    mpeig_iter_record rec{};
    rec.stage = opt.tag;
    rec.m = m;
    rec.ritz_values = theta.data();
    rec.residual_norms = rn.data();
    rec.n_converged = n_c;

    const bool done = n_c >= cfg.k;
    const bool out_of_iters = iter >= cfg.maxit;
    const bool stalled = opt.stagnation_exit && since_improvement >= kStagnationWindow;
    if (done || out_of_iters || stalled) {
      if (sink) sink(sink_user, &rec);
      if (Xout) copy_block<T>(n, m, X, w.ld, Xout, ldxout, s);
      MPB_CUDA(cudaStreamSynchronize(s));
      res.theta = theta;
      res.resid = rn;
      res.iterations = iter;
      res.converged = done;
      return res;
    }

    // W = T(R)  (eigensolvers.hpp:266-271)
    timer.start();
    if (overflow) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
    if (!fused) precond_apply<T>(ctx, T_op, m, w.V.p, w.ld, Wslot, w.ld);
    tm.precond_apply += timer.stop();

    // project + QR, twice (eigensolvers.hpp:272-291)
    timer.start();
    const int64_t b = m + p;
    int64_t dropped = 0, wc = m;
    project_out<T>(w, w.S.p, b, w.ld, Wslot, wc, w.ld, 2);
    wc = orthonormal_q_dropping<T>(w, wc, Wslot, w.ld, opt.use_mixed_qr != 0, &dropped);
    if (wc > 0) {
      int64_t more = 0;
      project_out<T>(w, w.S.p, b, w.ld, Wslot, wc, w.ld, 1);
      wc = orthonormal_q_dropping<T>(w, wc, Wslot, w.ld, opt.use_mixed_qr != 0, &more, true);
      dropped += more;
    }
    rec.w_columns_dropped = dropped;
    tm.orthogonalize += timer.stop();
    if (wc == 0 && p == 0) {
      if (sink) sink(sink_user, &rec);
      throw Error(MPEIG_E_RANK_COLLAPSE, "lobpcg_stage: no usable search directions left");
    }

    // AW = A W; Rayleigh-Ritz on S = [X P W] (eigensolvers.hpp:297-311)
    op_apply<T>(ctx, A, wc, Wslot, w.ld, w.AS.p + (m + p) * w.ld, w.ld);
    timer.start();
    const int64_t sdim = m + p + wc;
    status_clear(ctx);
    dgram<T>(w, sdim, w.S.p, w.ld, sdim, w.AS.p, w.ld, w.G.p, sdim, 1);
    small_eig<T>(w, sdim, w.G.p, sdim, w.evals.p);
    const int64_t pn = std::min(m, sdim - m);
    if constexpr (sizeof(T) == 8)
      hl_coeffs(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + 4, s);
    else
      hl_coeffs_f32(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + 4, s);
    // X, P = S [c_x c_pv]; AX, AP = AS [c_x c_pv] (eigensolvers.hpp:315-319)
    gemm_tn_pair<T>(n, sdim, m + pn, w.S.p, w.AS.p, w.ld, w.coef.p, sdim, w.S2.p, w.AS2.p, w.ld,
                    s);
    MPB_CUDA(cudaMemcpyAsync(w.theta.p, w.evals.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
    status_fetch(ctx);
    tm.projected_eig += timer.stop();
    if (ctx->h_status[3] > 0) throw Error(MPEIG_E_NO_CONVERGENCE, "small_herm_eig: syevd did not converge");
    if (ctx->h_status[3] < 0) throw Error(MPEIG_E_CUSOLVER, "syevd: invalid argument", -ctx->h_status[3]);
    rec.basis_rotation_fallback = ctx->h_status[4];
    if (sink) sink(sink_user, &rec);
    std::swap(w.S, w.S2);
    std::swap(w.AS, w.AS2);
    p = pn;
  }
}

// ----------------------------------------------------- speculative stage
// Status slots (ctx->d_status) written by one speculative iteration.
enum : int { kSlotOvf = 2, kSlotEig = 3, kSlotHl = 4, kSlotQr1 = 6, kSlotQr2 = 8 };

// Q in place without host synchronisation: same kernels as qr_core, Q is
// written unconditionally and failures only land in `status` (the caller
// rolls the iteration back and repeats it on the careful path).
template <typename T>
static void qr_spec(Work<T>& w, int64_t m, T* W, int64_t ldw, bool lower, int* status,
                    bool second = false) {
  cudaStream_t s = w.s;
  const int64_t n = w.n;
  if (w.ctx->spec_qr && second && sizeof(T) == 8) {
    // second round: W is already orthonormal up to the scrubbed overlap, so
    // one guarded CholQR pass (in place: every GEMM kernel reads all of a
    // row's inputs before it writes the row)
    gram_chol<T>(w, m, status, W, ldw, kCholQrSingleTau2<T>);
    gemm_right_inplace<T>(w, m, W, ldw, w.Uinv());
    return;
  }
  if (w.ctx->spec_qr) {
    // First pass as a guarded Cholesky-QR instead of the TSQR R: one Gram
    // (no column-serial reduction chain).  Cholesky is invariant to column
    // scaling, so the guard tests the equilibrated pivots: every column must
    // keep >= 1e-5 (fp64) / 1e-2 (fp32) of its norm outside the span of the
    // ones before it.  Then V = W R1^-1 is orthonormal to ~eps * cond^2 <<
    // 1 and the second pass makes Q orthonormal to rounding, as the
    // reference's QR does.  A failed guard rolls the iteration back to the
    // careful path (the reference's mixed_qr / householder_qr).
    gram_chol<T>(w, m, status, W, ldw, cholqr_tau2<T>(w.ctx));
    gemm_tn<T>(n, m, m, T(1), W, ldw, w.Uinv(), m, T(0), nullptr, 0, w.V.p, w.ld, s);
  } else {
    tsqr_R<T>(w, m, W, ldw, lower, status);
    gemm_tn<T>(n, m, m, T(1), W, ldw, w.Rinv(), m, T(0), nullptr, 0, w.V.p, w.ld, s);
  }
  gram_chol<T>(w, m, status);
  gemm_tn<T>(n, m, m, T(1), w.V.p, w.ld, w.Uinv(), m, T(0), nullptr, 0, W, ldw, s);
}

// Residual of the block in (X, AX) = (S, AS) column block 0, f_T fused into
// the W slot (or R into w.V), then the per-iteration record to pinned host
// memory: rnorm, xnorm (double) and theta (T).
template <typename T>
static void resid_launch(Work<T>& w, const mpeig_op* T_op, const T* S, const T* AS, T* Wslot) {
  mpeig_ctx* ctx = w.ctx;
  const int64_t m = w.m;
  const bool fused = T_op && T_op->kind == kOpJacobi;
  const void* dinv = nullptr;
  int mode = kResidPlain;
  if (fused) mode = jacobi_mode<T>(T_op, &dinv);
  dresidual<T>(w, mode, m, S, AS, dinv, fused ? Wslot : w.V.p, ctx->d_status + kSlotOvf);
  MPB_CUDA(cudaMemcpyAsync(ctx->h_pinned, w.rnorm(), sizeof(double) * 2 * m,
                           cudaMemcpyDeviceToHost, w.s));
  MPB_CUDA(cudaMemcpyAsync(ctx->h_pinned + 2 * m, w.theta.p, sizeof(T) * m, cudaMemcpyDeviceToHost,
                           w.s));
  if (Comm* c = dist(ctx)) c->allreduce_max(ctx->d_status, 16, w.s);
  MPB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, 16 * sizeof(int), cudaMemcpyDeviceToHost,
                           w.s));
}

template <typename T>
static void read_record(Work<T>& w, std::vector<double>& theta, std::vector<double>& rn,
                        std::vector<double>& xn) {
  mpeig_ctx* ctx = w.ctx;
  const int64_t m = w.m;
  const T* th = reinterpret_cast<const T*>(ctx->h_pinned + 2 * m);
  theta.resize(m);
  rn.resize(m);
  xn.resize(m);
  for (int64_t j = 0; j < m; ++j) {
    theta[j] = static_cast<double>(th[j]);
    rn[j] = static_cast<double>(static_cast<T>(ctx->h_pinned[j]));
    xn[j] = static_cast<double>(static_cast<T>(ctx->h_pinned[m + j]));
  }
}

struct PhaseEvents {
  cudaEvent_t e[4];
  bool on = true;  // record phase boundaries inside the body (eager bodies only)
  PhaseEvents() {
    for (auto& x : e) cudaEventCreate(&x);
  }
  ~PhaseEvents() {
    for (auto& x : e) cudaEventDestroy(x);
  }
  float ms(int a, int b) const {
    float t = 0;
    cudaEventElapsedTime(&t, e[a], e[b]);
    return t;
  }
};

// Speculative iteration body: project + QR twice, A W, Rayleigh-Ritz, HL
// update into (S2, AS2), theta update, and the NEXT iteration's residual and
// record copy.  No host synchronisation; graph-capturable when A is.
template <typename T>
static void spec_body(Work<T>& w, const mpeig_op* A, const mpeig_op* T_op, int64_t p, bool mixed,
                      T* S, T* AS, T* S2, T* AS2, PhaseEvents& ev) {
  mpeig_ctx* ctx = w.ctx;
  cudaStream_t s = w.s;
  const int64_t m = w.m, ld = w.ld, n = w.n;
  T* Wslot = S + (m + p) * ld;
  if (ev.on) MPB_CUDA(cudaEventRecord(ev.e[0], s));
  MPB_CUDA(cudaMemsetAsync(ctx->d_status, 0, 16 * sizeof(int), s));
  MPB_CUDA(cudaMemcpyAsync(w.theta_prev.p, w.theta.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
  project_out<T>(w, S, m + p, ld, Wslot, m, ld, 2);
  qr_spec<T>(w, m, Wslot, ld, mixed, ctx->d_status + kSlotQr1);
  project_out<T>(w, S, m + p, ld, Wslot, m, ld, 1);
  qr_spec<T>(w, m, Wslot, ld, mixed, ctx->d_status + kSlotQr2, true);
  if (ev.on) MPB_CUDA(cudaEventRecord(ev.e[1], s));
  op_apply<T>(ctx, A, m, Wslot, ld, AS + (m + p) * ld, ld);
  const int64_t sdim = 2 * m + p;
  dgram<T>(w, sdim, S, ld, sdim, AS, ld, w.G.p, sdim, 1);
  small_syev<T>(sdim, w.G.p, sdim, w.evals.p, ctx->d_status + kSlotEig, s, ctx->ql_exact);
  const int64_t pn = std::min(m, sdim - m);
  if constexpr (sizeof(T) == 8)
    hl_coeffs(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + kSlotHl, s);
  else
    hl_coeffs_f32(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + kSlotHl, s);
  gemm_tn_pair<T>(n, sdim, m + pn, S, AS, ld, w.coef.p, sdim, S2, AS2, ld, s);
  MPB_CUDA(cudaMemcpyAsync(w.theta.p, w.evals.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
  if (ev.on) MPB_CUDA(cudaEventRecord(ev.e[2], s));
  resid_launch<T>(w, T_op, S2, AS2, S2 + (m + pn) * ld);
  if (ev.on) MPB_CUDA(cudaEventRecord(ev.e[3], s));
}

// Programmatic dependent launch inside the iteration graph: every kernel ->
// kernel edge becomes a programmatic edge, so a kernel is launched while its
// predecessor's CTAs drain and waits in MPB_PDL_WAIT (every kernel's first
// statement) for the predecessor to complete with its memory visible.
// Memset / memcpy edges keep full ordering.  Results are bitwise unchanged;
// cfg1 0.4467 -> 0.4420 s (scripts/pdl_ab.py).  g_pdl = 2 (diagnostic): the
// launch-completion port, dependents resident from the predecessor's start --
// 0.484 s, they crowd the SMs the chain still needs.
int g_pdl = 1;

static void make_kernel_edges_programmatic(cudaGraph_t graph) {
  size_t ne = 0;
  MPB_CUDA(cudaGraphGetEdges_v2(graph, nullptr, nullptr, nullptr, &ne));
  if (ne == 0) return;
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  std::vector<cudaGraphEdgeData> data(ne);
  MPB_CUDA(cudaGraphGetEdges_v2(graph, from.data(), to.data(), data.data(), &ne));
  for (size_t e = 0; e < ne; ++e) {
    cudaGraphNodeType tf, tt;
    MPB_CUDA(cudaGraphNodeGetType(from[e], &tf));
    MPB_CUDA(cudaGraphNodeGetType(to[e], &tt));
    if (tf != cudaGraphNodeTypeKernel || tt != cudaGraphNodeTypeKernel) continue;
    if (data[e].type != cudaGraphDependencyTypeDefault) continue;
    MPB_CUDA(cudaGraphRemoveDependencies_v2(graph, &from[e], &to[e], &data[e], 1));
    cudaGraphEdgeData pd{};
    pd.from_port = g_pdl == 2 ? cudaGraphKernelNodePortLaunchCompletion : cudaGraphKernelNodePortProgrammatic;
    pd.to_port = 0;
    pd.type = cudaGraphDependencyTypeProgrammatic;
    MPB_CUDA(cudaGraphAddDependencies_v2(graph, &from[e], &to[e], &pd, 1));
  }
}

static bool graph_capturable(const mpeig_op* op) {
  return op && (op->kind == kOpLap3d || op->kind == kOpLap2d || op->kind == kOpCsr ||
                op->kind == kOpJacobi);
}

// lobpcg_stage<T> (eigensolvers.hpp:195-321), speculative form: one host
// synchronisation per iteration (the record the reference's convergence test
// and IterationRecord need), the iteration body replayed as a CUDA graph in
// the steady state.  A breakdown flagged by the body (mixed_qr Cholesky
// failure, rank deficiency, eigensolver non-convergence) rolls the iteration
// back -- S/AS are untouched, theta is restored -- and repeats it on the
// careful path with the reference's fallbacks (orthonormal_q,
// orthonormal_q_dropping, RankCollapse), so the semantics are unchanged.
template <typename T>
StageResult lobpcg_stage(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const T* X0, int64_t ldx0,
                         int64_t m, const mpeig_cfg& cfg, const mpeig_op* T_op, double a_norm_est,
                         const mpeig_stage_opts& opt, mpeig_history_sink sink, void* sink_user,
                         T* Xout, int64_t ldxout, mpeig_timings* tim) {
  if (n <= 0 || m <= 0) throw Error(MPEIG_E_DIMENSION, "lobpcg_stage: empty block");
  const bool spec_ok = ctx->spec_mode != 0 && graph_capturable(A) && T_op &&
                       T_op->kind == kOpJacobi && small_syev_supported<T>(3 * m);
  if (!spec_ok)
    return lobpcg_stage_eager<T>(ctx, A, n, X0, ldx0, m, cfg, T_op, a_norm_est, opt, sink,
                                 sink_user, Xout, ldxout, tim);
  Work<T> w(ctx, n, m, 3 * m);
  cudaStream_t s = w.s;
  EvTimer timer(s);
  PhaseEvents ev;
  mpeig_timings local{};
  mpeig_timings& tm = tim ? *tim : local;
  const bool mixed = opt.use_mixed_qr != 0;
  // row-sharded runs: the body's collectives and halo / ghost exchanges are
  // captured with it over NCCL (stream-ordered); the host-staged transport
  // synchronises inside the body and runs it eagerly
  const bool use_graphs = ctx->use_graphs != 0 && !g_prof_on && (!dist(ctx) || dist(ctx)->capturable());

  copy_block<T>(n, m, X0, ldx0, w.S.p, w.ld, s);
  op_apply<T>(ctx, A, m, w.S.p, w.ld, w.AS.p, w.ld);
  timer.start();
  ritz_rotate<T>(w);
  tm.projected_eig += timer.stop();
  int64_t p = 0;
  MPB_CUDA(cudaMemsetAsync(ctx->d_status, 0, 16 * sizeof(int), s));
  resid_launch<T>(w, T_op, w.S.p, w.AS.p, w.S.p + m * w.ld);
  MPB_CUDA(cudaStreamSynchronize(s));

  struct GraphKey {
    const void* S;
    int64_t p;
  };
  struct CachedGraph {
    GraphKey key;
    cudaGraphExec_t exec;
    int64_t kernels;  // library kernels per replay (counted into g_launches)
  };
  std::vector<CachedGraph> graphs;
  auto cleanup = [&] {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  };

  double best_metric = std::numeric_limits<double>::infinity();
  int64_t since_improvement = 0;
  constexpr int64_t kStagnationWindow = 40;
  std::vector<double> theta, rn, xn;
  StageResult res;
  try {
    for (int64_t iter = 0;; ++iter) {
      read_record<T>(w, theta, rn, xn);
      const int64_t n_c = converged_prefix(a_norm_est, theta, rn, xn, opt.tol);
      if (opt.stagnation_exit) {
        double metric = 0;
        for (int64_t j = 0; j < cfg.k && j < m; ++j) {
          const double denom = (a_norm_est + std::abs(theta[j])) * xn[j];
          const double ratio = denom > 0 ? rn[j] / denom : std::numeric_limits<double>::infinity();
          if (ratio > metric) metric = ratio;
        }
        if (metric < 0.99 * best_metric) {
          best_metric = metric;
          since_improvement = 0;
        } else {
          ++since_improvement;
        }
      }
      mpeig_iter_record rec{};
      rec.stage = opt.tag;
      rec.m = m;
      rec.ritz_values = theta.data();
      rec.residual_norms = rn.data();
      rec.n_converged = n_c;
      const bool done = n_c >= cfg.k;
      const bool out_of_iters = iter >= cfg.maxit;
      const bool stalled = opt.stagnation_exit && since_improvement >= kStagnationWindow;
      if (done || out_of_iters || stalled) {
        if (sink) sink(sink_user, &rec);
        if (Xout) copy_block<T>(n, m, w.S.p, w.ld, Xout, ldxout, s);
        MPB_CUDA(cudaStreamSynchronize(s));
        res.theta = theta;
        res.resid = rn;
        res.iterations = iter;
        res.converged = done;
        cleanup();
        return res;
      }
      if (ctx->h_status[kSlotOvf])
        throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");

      // ---- speculative body (graph in the steady state)
      cudaGraphExec_t exec = nullptr;
      if (use_graphs && p == m) {
        int64_t nk = 0;
        for (auto& g : graphs)
          if (g.key.S == w.S.p && g.key.p == p) {
            exec = g.exec;
            nk = g.kernels;
          }
        if (!exec) {
          cudaGraph_t graph;
          ev.on = false;
          const int64_t c0 = g_launches.load();
          MPB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
          try {
            spec_body<T>(w, A, T_op, p, mixed, w.S.p, w.AS.p, w.S2.p, w.AS2.p, ev);
          } catch (...) {
            cudaStreamEndCapture(s, &graph);
            throw;
          }
          MPB_CUDA(cudaStreamEndCapture(s, &graph));
          if (g_pdl) make_kernel_edges_programmatic(graph);
          MPB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
          cudaGraphDestroy(graph);
          // capture records launches without running them: count them per replay
          nk = g_launches.load() - c0;
          g_launches.fetch_sub(nk);
          graphs.push_back({{w.S.p, p}, exec, nk});
        }
        MPB_CUDA(cudaEventRecord(ev.e[0], s));
        MPB_CUDA(cudaGraphLaunch(exec, s));
        g_launches.fetch_add(nk);
        MPB_CUDA(cudaEventRecord(ev.e[3], s));
        MPB_CUDA(cudaStreamSynchronize(s));
        tm.projected_eig += ev.ms(0, 3) * 1e-3;  // whole body (no phase split in a graph)
      } else {
        ev.on = true;
        spec_body<T>(w, A, T_op, p, mixed, w.S.p, w.AS.p, w.S2.p, w.AS2.p, ev);
        MPB_CUDA(cudaStreamSynchronize(s));
        tm.orthogonalize += ev.ms(0, 1) * 1e-3;
        tm.projected_eig += ev.ms(1, 2) * 1e-3;
        tm.precond_apply += ev.ms(2, 3) * 1e-3;
      }
      const bool failed = ctx->h_status[kSlotQr1] || ctx->h_status[kSlotQr2] ||
                          ctx->h_status[kSlotEig];
      int64_t dropped = 0, pn = std::min(m, m + p);
      if (failed) {
        ++ctx->spec_rollbacks;
        // ---- roll back and repeat on the careful path
        MPB_CUDA(cudaMemcpyAsync(w.theta.p, w.theta_prev.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
        T* Wslot = w.S.p + (m + p) * w.ld;
        const void* dinv = nullptr;
        const int mode = jacobi_mode<T>(T_op, &dinv);
        dresidual<T>(w, mode, m, w.S.p, w.AS.p, dinv, Wslot, ctx->d_status + kSlotOvf);
        timer.start();
        const int64_t b = m + p;
        int64_t wc = m;
        project_out<T>(w, w.S.p, b, w.ld, Wslot, wc, w.ld, 2);
        wc = orthonormal_q_dropping<T>(w, wc, Wslot, w.ld, mixed, &dropped);
        if (wc > 0) {
          int64_t more = 0;
          project_out<T>(w, w.S.p, b, w.ld, Wslot, wc, w.ld, 1);
          wc = orthonormal_q_dropping<T>(w, wc, Wslot, w.ld, mixed, &more, true);
          dropped += more;
        }
        tm.orthogonalize += timer.stop();
        rec.w_columns_dropped = dropped;
        if (wc == 0 && p == 0) {
          if (sink) sink(sink_user, &rec);
          throw Error(MPEIG_E_RANK_COLLAPSE, "lobpcg_stage: no usable search directions left");
        }
        op_apply<T>(ctx, A, wc, Wslot, w.ld, w.AS.p + (m + p) * w.ld, w.ld);
        timer.start();
        const int64_t sdim = m + p + wc;
        status_clear(ctx);
        dgram<T>(w, sdim, w.S.p, w.ld, sdim, w.AS.p, w.ld, w.G.p, sdim, 1);
        small_eig<T>(w, sdim, w.G.p, sdim, w.evals.p);
        pn = std::min(m, sdim - m);
        if constexpr (sizeof(T) == 8)
          hl_coeffs(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + kSlotHl, s);
        else
          hl_coeffs_f32(sdim, m, pn, w.G.p, sdim, w.coef.p, w.scratch(), ctx->d_status + kSlotHl, s);
        gemm_tn_pair<T>(n, sdim, m + pn, w.S.p, w.AS.p, w.ld, w.coef.p, sdim, w.S2.p, w.AS2.p,
                        w.ld, s);
        MPB_CUDA(cudaMemcpyAsync(w.theta.p, w.evals.p, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
        status_fetch(ctx);
        tm.projected_eig += timer.stop();
        if (ctx->h_status[kSlotEig] > 0)
          throw Error(MPEIG_E_NO_CONVERGENCE, "small_herm_eig: QL sweep budget exhausted");
        const int hl_fb = ctx->h_status[kSlotHl];
        MPB_CUDA(cudaMemsetAsync(ctx->d_status, 0, 16 * sizeof(int), s));
        resid_launch<T>(w, T_op, w.S2.p, w.AS2.p, w.S2.p + (m + pn) * w.ld);
        MPB_CUDA(cudaStreamSynchronize(s));
        ctx->h_status[kSlotHl] = hl_fb;
      }
      rec.w_columns_dropped = dropped;
      rec.basis_rotation_fallback = ctx->h_status[kSlotHl];
      if (sink) sink(sink_user, &rec);
      std::swap(w.S, w.S2);
      std::swap(w.AS, w.AS2);
      p = pn;
    }
  } catch (...) {
    cleanup();
    throw;
  }
}

// pinvit<double> (eigensolvers.hpp:326-390) with an operator preconditioner
StageResult pinvit(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0, int64_t ldx0,
                   int64_t m, const mpeig_cfg& cfg, const mpeig_op* T_op, double a_norm_est,
                   mpeig_history_sink sink, void* sink_user, double* Xout, int64_t ldxout,
                   mpeig_timings* tim) {
  using T = double;
  Work<T> w(ctx, n, m, m);
  cudaStream_t s = w.s;
  EvTimer timer(s);
  mpeig_timings local{};
  mpeig_timings& tm = tim ? *tim : local;
  // Xt lives in S2 column block 0 between iterations (ritz_rotate swaps S/S2)
  T* Xt = w.S2.p;
  copy_block<T>(n, m, X0, ldx0, Xt, w.ld, s);
  std::vector<double> theta, rn, xn;
  StageResult res;
  for (int64_t iter = 0;; ++iter) {
    timer.start();
    copy_block<T>(n, m, Xt, w.ld, w.S.p, w.ld, s);
    try {
      // X = orthonormal_q(Xt, true) (eigensolvers.hpp:342-347): the guarded
      // Cholesky-QR first (the iterate is X minus a small correction, well
      // conditioned), the reference's mixed_qr chain when the guard fails
      if (!(ctx->spec_qr && guarded_cholqr2<T>(w, m, w.S.p, w.ld)))
        orthonormal_q<T>(w, m, w.S.p, w.ld, true);
    } catch (const Error& e) {
      if (e.code == MPEIG_E_RANK_DEFICIENT)
        throw Error(MPEIG_E_RANK_COLLAPSE, "pinvit: iterate block lost rank");
      throw;
    }
    tm.orthogonalize += timer.stop();
    op_apply<T>(ctx, A, m, w.S.p, w.ld, w.AS.p, w.ld);
    timer.start();
    ritz_rotate<T>(w);  // X, AX now in S, AS
    tm.projected_eig += timer.stop();
    bool overflow = false;
    T* W = w.AS2.p;  // free after ritz_rotate's swap
    const bool fused = residual_step<T>(w, T_op, w.S.p, w.AS.p, W, theta, rn, xn, &overflow);
    const int64_t n_c = converged_prefix(a_norm_est, theta, rn, xn, cfg.tol);
    mpeig_iter_record rec{};
    rec.stage = MPEIG_WORKING;
    rec.m = m;
    rec.ritz_values = theta.data();
    rec.residual_norms = rn.data();
    rec.n_converged = n_c;
    if (sink) sink(sink_user, &rec);
    const bool done = n_c >= cfg.k;
    if (done || iter >= cfg.maxit) {
      if (Xout) copy_block<T>(n, m, w.S.p, w.ld, Xout, ldxout, s);
      MPB_CUDA(cudaStreamSynchronize(s));
      res.theta = theta;
      res.resid = rn;
      res.iterations = iter;
      res.converged = done;
      return res;
    }
    timer.start();
    if (overflow) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
    if (!fused) precond_apply<T>(ctx, T_op, m, w.V.p, w.ld, W, w.ld);
    tm.precond_apply += timer.stop();
    Xt = w.S2.p;
    subtract<T>(n, m, w.S.p, w.ld, W, w.ld, Xt, w.ld, s);  // Xt = X - W (:388)
  }
}

// spectral_norm_estimate (norm_estimate.hpp:15-24)
double spectral_norm_estimate(mpeig_ctx* ctx, const mpeig_op* A, int64_t sketch_rows,
                              uint64_t seed) {
  if (sketch_rows < 1) throw Error(MPEIG_E_CONFIG, "spectral_norm_estimate: sketch_rows < 1");
  const int64_t n = A->n;
  const int64_t ld = padded_ld(n);
  std::vector<double> om(static_cast<size_t>(n * sketch_rows));
  if (A->n_global > n)  // this rank's rows of the global sketch
    gaussian_fill_rows(A->n_global, sketch_rows, seed, A->row0, n, om.data());
  else
    gaussian_fill(n, sketch_rows, seed, om.data());
  double den2 = 0;  // frobenius_norm, sequential like the reference
  for (double v : om) den2 += std::abs(v) * std::abs(v);
  cudaStream_t s = ctx->stream;
  DevBuf<double> O(static_cast<size_t>(ld * sketch_rows), s), Y(static_cast<size_t>(ld * sketch_rows), s),
      wk(kNumSMs * 2 + 2, s);
  MPB_CUDA(cudaMemcpy2DAsync(O.p, sizeof(double) * ld, om.data(), sizeof(double) * n,
                             sizeof(double) * n, sketch_rows, cudaMemcpyHostToDevice, s));
  op_apply<double>(ctx, A, sketch_rows, O.p, ld, Y.p, ld);
  frob_sq<double>(n, sketch_rows, Y.p, ld, wk.p + kNumSMs * 2, wk.p, s);
  double h[2] = {0, den2};
  if (Comm* c = dist(ctx)) {
    MPB_CUDA(cudaMemcpyAsync(wk.p + kNumSMs * 2 + 1, &h[1], sizeof(double), cudaMemcpyHostToDevice, s));
    c->allreduce_sum(wk.p + kNumSMs * 2, 2, s);
    MPB_CUDA(cudaMemcpyAsync(h, wk.p + kNumSMs * 2, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  } else {
    MPB_CUDA(cudaMemcpyAsync(h, wk.p + kNumSMs * 2, sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  MPB_CUDA(cudaStreamSynchronize(s));
  const double denom = std::sqrt(h[1]);
  if (denom == 0) return 0;
  return std::sqrt(h[0]) / denom;
}

// run_variant (drivers.hpp:57-111) on a device start block
void run_variant(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
                 const double* X0, int64_t ldx0, double a_norm_est, mpeig_history_sink sink,
                 void* sink_user, mpeig_result* out) {
  const int64_t n = A->n;
  const int64_t m = cfg.block != 0 ? cfg.block : (3 * cfg.k + 1) / 2;
  cudaStream_t s = ctx->stream;
  out->a_norm_estimate = a_norm_est;
  out->iterations_lower = 0;
  out->iterations_working = 0;
  const int64_t ld = padded_ld(n);
  DevBuf<double> Xf(static_cast<size_t>(ld * m), s);
  StageResult st;
  if (cfg.variant == MPEIG_PINVIT) {
    st = pinvit(ctx, A, n, X0, ldx0, m, cfg, T_op, a_norm_est, sink, sink_user, Xf.p, ld,
                &out->timings);
    out->iterations_working = st.iterations;
  } else {
    DevBuf<double> X(static_cast<size_t>(ld * m), s);
    copy_block<double>(n, m, X0, ldx0, X.p, ld, s);
    const bool mixed = cfg.variant == MPEIG_MPLOBPCG_SCHOL;
    if (mixed) {
      // stage 1: everything in binary32 to lower_tol, stagnation exit
      mpeig_stage_opts lo{cfg.lower_tol, 0, 1, MPEIG_LOWER};
      StageResult st1;
      {
        DevBuf<float> Xl(static_cast<size_t>(ld * m), s), X1(static_cast<size_t>(ld * m), s);
        status_clear(ctx);
        convert_f64_to_f32(n, m, X.p, ld, Xl.p, ld, ctx->d_status + 5, s);
        status_fetch(ctx);
        if (ctx->h_status[5]) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
        st1 = lobpcg_stage<float>(ctx, A, n, Xl.p, ld, m, cfg, T_op, a_norm_est, lo, sink, sink_user,
                                  X1.p, ld, &out->timings);
        out->iterations_lower = st1.iterations;
        // a stalled or capped first stage still hands over its block
        convert_f32_to_f64(n, m, X1.p, ld, X.p, ld, s);
      }
      Work<double> w(ctx, n, m, m);
      orthonormal_q<double>(w, m, X.p, ld, true);
    }
    mpeig_stage_opts hi{cfg.tol, mixed ? 1 : 0, 0, MPEIG_WORKING};
    st = lobpcg_stage<double>(ctx, A, n, X.p, ld, m, cfg, T_op, a_norm_est, hi, sink, sink_user,
                              Xf.p, ld, &out->timings);
    out->iterations_working = st.iterations;
  }
  out->converged = st.converged ? 1 : 0;
  for (int64_t j = 0; j < cfg.k; ++j) {
    if (out->theta) out->theta[j] = st.theta[j];
    if (out->residual_norms) out->residual_norms[j] = st.resid[j];
  }
  if (out->X) copy_block<double>(n, cfg.k, Xf.p, ld, out->X, out->ldx, s);
  MPB_CUDA(cudaStreamSynchronize(s));
}

// solve (drivers.hpp:158-181): sketch, seeded start block, run_variant
void solve(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
           mpeig_history_sink sink, void* sink_user, mpeig_result* out) {
  const int64_t n = A->n;
  validate_cfg(cfg, A->n_global > n ? A->n_global : n);
  const int64_t m = cfg.block != 0 ? cfg.block : (3 * cfg.k + 1) / 2;
  const auto t0 = std::chrono::steady_clock::now();
  const double est =
      spectral_norm_estimate(ctx, A, cfg.sketch_rows, cfg.seed ^ 0x9e3779b97f4a7c15ULL);
  std::vector<double> g(static_cast<size_t>(n * m));
  if (A->n_global > n)  // this rank's rows of the global start block
    gaussian_fill_rows(A->n_global, m, cfg.seed, A->row0, n, g.data());
  else
    gaussian_fill(n, m, cfg.seed, g.data());
  const int64_t ld = padded_ld(n);
  cudaStream_t s = ctx->stream;
  DevBuf<double> X0(static_cast<size_t>(ld * m), s);
  MPB_CUDA(cudaMemcpy2DAsync(X0.p, sizeof(double) * ld, g.data(), sizeof(double) * n,
                             sizeof(double) * n, m, cudaMemcpyHostToDevice, s));
  {
    Work<double> w(ctx, n, m, m);
    orthonormal_q<double>(w, m, X0.p, ld, true);
  }
  run_variant(ctx, A, T_op, cfg, X0.p, ld, est, sink, sink_user, out);
  out->timings.total =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// solve() from device-resident raw inputs: the Gaussian start block X0raw
// (n x m, not yet orthonormal) and the sketch Omega (n x sketch_rows), as
// drawn by gaussian_matrix on the host.  omega_fro = ||Omega||_F (computed on
// the device when <= 0).  This is the timed region of bench.py:
// sketch apply, initial orthonormalisation and both stages.
void solve_prepared(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T_op, const mpeig_cfg& cfg,
                    const double* X0raw, int64_t ldx0, const double* omega, int64_t ldo,
                    double omega_fro, mpeig_history_sink sink, void* sink_user, mpeig_result* out) {
  const int64_t n = A->n;
  validate_cfg(cfg, A->n_global > n ? A->n_global : n);
  const int64_t m = cfg.block != 0 ? cfg.block : (3 * cfg.k + 1) / 2;
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = ctx->stream;
  const int64_t ld = padded_ld(n);
  const int64_t sr = cfg.sketch_rows;
  double est = 0;
  {
    DevBuf<double> Y(static_cast<size_t>(ld * sr), s), wk(kNumSMs * 2 + 4, s);
    op_apply<double>(ctx, A, sr, omega, ldo, Y.p, ld);
    frob_sq<double>(n, sr, Y.p, ld, wk.p + kNumSMs * 2, wk.p, s);
    if (omega_fro <= 0) frob_sq<double>(n, sr, omega, ldo, wk.p + kNumSMs * 2 + 1, wk.p, s);
    if (Comm* c = dist(ctx)) c->allreduce_sum(wk.p + kNumSMs * 2, omega_fro <= 0 ? 2 : 1, s);
    double h[2] = {0, 0};
    MPB_CUDA(cudaMemcpyAsync(h, wk.p + kNumSMs * 2, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
    MPB_CUDA(cudaStreamSynchronize(s));
    const double den = omega_fro > 0 ? omega_fro : std::sqrt(h[1]);
    est = den == 0 ? 0 : std::sqrt(h[0]) / den;
  }
  DevBuf<double> X0(static_cast<size_t>(ld * m), s);
  copy_block<double>(n, m, X0raw, ldx0, X0.p, ld, s);
  {
    Work<double> w(ctx, n, m, m);
    orthonormal_q<double>(w, m, X0.p, ld, true);
  }
  run_variant(ctx, A, T_op, cfg, X0.p, ld, est, sink, sink_user, out);
  out->timings.total =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// SolverConfig::validate (solver_types.hpp:43-56)
void validate_cfg(const mpeig_cfg& cfg, int64_t n) {
  const int64_t m = cfg.block != 0 ? cfg.block : (3 * cfg.k + 1) / 2;
  if (cfg.k < 1) throw Error(MPEIG_E_CONFIG, "config: k must be at least 1");
  if (m < cfg.k) throw Error(MPEIG_E_CONFIG, "config: block size below k");
  if (3 * m > n)
    throw Error(MPEIG_E_CONFIG, "config: block size " + std::to_string(m) + " too large for n=" +
                                    std::to_string(n) + " (need 3*block <= n)");
  if (!(cfg.tol > 0) || !(cfg.tol < 1)) throw Error(MPEIG_E_CONFIG, "config: tol outside (0,1)");
  if (!(cfg.lower_tol > 0) || !(cfg.lower_tol < 1))
    throw Error(MPEIG_E_CONFIG, "config: lower_tol outside (0,1)");
  if (cfg.maxit < 1) throw Error(MPEIG_E_CONFIG, "config: maxit must be at least 1");
  if (cfg.sketch_rows < 1) throw Error(MPEIG_E_CONFIG, "config: sketch_rows must be at least 1");
}

// explicit instantiations
template void op_apply<double>(mpeig_ctx*, const mpeig_op*, int64_t, const double*, int64_t, double*,
                               int64_t);
template void op_apply<float>(mpeig_ctx*, const mpeig_op*, int64_t, const float*, int64_t, float*,
                              int64_t);
template void precond_apply<double>(mpeig_ctx*, const mpeig_op*, int64_t, const double*, int64_t,
                                    double*, int64_t);
template void precond_apply<float>(mpeig_ctx*, const mpeig_op*, int64_t, const float*, int64_t,
                                   float*, int64_t);
template struct Work<double>;
template struct Work<float>;
template void orthonormal_q<double>(Work<double>&, int64_t, double*, int64_t, bool);
template void orthonormal_q<float>(Work<float>&, int64_t, float*, int64_t, bool);
template int64_t orthonormal_q_dropping<double>(Work<double>&, int64_t, double*, int64_t, bool,
                                                int64_t*, bool);
template void project_out<double>(Work<double>&, const double*, int64_t, int64_t, double*, int64_t,
                                  int64_t, int);
template void small_eig<double>(Work<double>&, int64_t, double*, int64_t, double*);
template StageResult lobpcg_stage<double>(mpeig_ctx*, const mpeig_op*, int64_t, const double*,
                                          int64_t, int64_t, const mpeig_cfg&, const mpeig_op*,
                                          double, const mpeig_stage_opts&, mpeig_history_sink,
                                          void*, double*, int64_t, mpeig_timings*);
template StageResult lobpcg_stage<float>(mpeig_ctx*, const mpeig_op*, int64_t, const float*,
                                         int64_t, int64_t, const mpeig_cfg&, const mpeig_op*,
                                         double, const mpeig_stage_opts&, mpeig_history_sink,
                                         void*, float*, int64_t, mpeig_timings*);

int qr_with_r(Work<double>& w, int64_t m, double* W, int64_t ldw, bool lower, double* Rout,
              int64_t* idx) {
  return qr_core<double>(w, m, W, ldw, lower, Rout, idx);
}

}  // namespace mpb
