// kernels.cuh -- launcher declarations for the sm_100a kernels.
//
// All block vectors are column-major device arrays with explicit leading
// dimensions.  Every launcher is stream-ordered and never synchronises.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace mpb {

// ----------------------------------------------------------------- dense
// Workspace (device) needed by gram(): floats of type T.
template <typename T>
int64_t gram_workspace_elems(int64_t n, int64_t ka, int64_t kb);

// G (ka x kb, ld ldg) = A^T B over n rows (adjoint_matmul,
// dense_kernels.hpp:36-52).  Split-n partial products reduced in a fixed
// order -> bitwise deterministic for a given n.  `sym` != 0 additionally
// symmetrises G in place like hermitize (dense_kernels.hpp:77-88); needs
// ka == kb.  work: gram_workspace_elems<T>() elements, zeroed before first
// use (its head holds the reduction-tree counters, which reset themselves).
template <typename T>
void gram(int64_t n, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B,
          int64_t ldb, T* G, int64_t ldg, int sym, T* work, cudaStream_t s);

// Y (n x c) = beta Z + alpha A (n x k) C (k x c)   (matmul, dense_kernels.hpp:20-34)
// Y may alias Z (elementwise read-before-write).  Y may alias A only when
// c <= kGemmInplaceCols: each CTA then owns whole rows (one column tile) and
// reads all of them before it writes; wider outputs span several CTAs per row
// block and an in-place call would race.
constexpr int64_t kGemmInplaceCols = 64;
// Y = A C in place for wider c: binary64 c <= 96 (one DMMA column tile),
// binary32 c <= 256 on the tensor-core path when it applies (gemm_tn checks)
bool gemm_inplace_ok(bool f64, int64_t n, int64_t k, int64_t c);
bool gemm_tc_inplace_ok(int64_t c);
// frees the tensor-core scratch of a stream about to be destroyed
void tc_scratch_release(cudaStream_t s);
template <typename T>
void gemm_tn(int64_t n, int64_t k, int64_t c, T alpha, const T* A, int64_t lda, const T* C,
             int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y, int64_t ldy, cudaStream_t s);
// binary32 Gram chunk partials on the tcgen05 tensor cores (tc.cu); the
// caller combines the returned number of chunks
bool gram_tc_eligible(int64_t n, int64_t ka, int64_t kb, int64_t lda, int64_t ldb, const float* A,
                      const float* B);
int64_t gram_tc_f32(int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb, const float* B,
                    int64_t ldb, int64_t max_chunks, float* part, cudaStream_t s);
// binary32 Y = beta Z + alpha A C (+ the paired A2 C) on tcgen05 (tc.cu)
bool gemm_tc_eligible(int64_t n, int64_t k, int64_t c, int64_t lda, int64_t ldc, const float* A,
                      const float* C);
// returns false (nothing launched) when `inplace` (Y aliases A) and no
// single-column-tile kernel is available for c
bool gemm_tc_f32(int64_t n, int64_t k, int64_t c, float alpha, const float* A, int64_t lda,
                 const float* C, int64_t ldc, float beta, const float* Z, int64_t ldz, float* Y,
                 int64_t ldy, const float* A2, float* Y2, bool inplace, cudaStream_t s);
// policy: the tensor-core path for Grams big enough to be bandwidth/compute
// bound (the m = 16 cfg1 shapes stay on the latency-lean SIMT kernel);
// g_gram_tc: 1 = by size (default), 0 = never, 2 = always (tests)
extern int g_gram_tc, g_gemm_tc;
extern int g_gemm_tma2, g_tc_twoacc, g_tc_ablate, g_g2_depth, g_tc_stage;
extern int g_tc_nprod, g_tc_store;
extern int g_gram_tma;
extern int g_pdl;  // programmatic edges in the captured iteration graphs (solver.cpp)  // TMA-fed tensor-core Gram (1, default) or the cp.async one (0)
// (crossovers measured at n = 2M, scripts/dense_shapes.py: the tensor-core
// Gram wins from 32 x 16 up, the tensor-core block update once k * c reaches
// the m = 48 project-out's 96 x 48; narrower updates stay on the FFMA kernel)
inline bool gram_tc_wanted(int64_t n, int64_t ka, int64_t kb) {
  return g_gram_tc == 2 ||
         (g_gram_tc == 1 && n * ka * kb >= (int64_t(1) << 28) && ka * kb > 256);
}
inline bool gemm_tc_wanted(int64_t n, int64_t k, int64_t c) {
  return g_gemm_tc == 2 ||
         (g_gemm_tc == 1 && n * k * c >= (int64_t(1) << 28) && k * c >= 96 * 48);
}
// CholQR's Gram and factorization in one pass (m <= 16): G = V^T V
// (hermitized), then L L^T = G and Uinv = L^{-T} by the last CTA of the
// combine; returns false (nothing launched) when m > 16.
template <typename T>
bool gram_cholesky(int64_t n, int64_t m, const T* V, int64_t ldv, T* G, T* work, T* L, T* Uinv,
                   int* status, cudaStream_t s, T tau2 = T(0));

// Y1 = A1 C and Y2 = A2 C in one launch (the S C / AS C update pair)
template <typename T>
void gemm_tn_pair(int64_t n, int64_t k, int64_t c, const T* A1, const T* A2, int64_t lda,
                  const T* C, int64_t ldc, T* Y1, T* Y2, int64_t ldy, cudaStream_t s);

// dst = (To) src, elementwise over an n x c block; to_lower() narrowing sets
// *overflow_flag = 1 on finite -> inf (precision.hpp:102-107).
void convert_f64_to_f32(int64_t n, int64_t c, const double* src, int64_t lds, float* dst,
                        int64_t ldd, int* overflow_flag, cudaStream_t s);
// A(j, i) = A(i, j) for i > j (mirror the lower triangle of a symmetric n x n matrix)
template <typename T>
void symmetrize_lower(int64_t n, T* A, int64_t lda, cudaStream_t s);
// A(i, i) += shift, i < n (retry_dense's shifted copy, precond.hpp:140-146)
void add_diag_f64(int64_t n, double* A, int64_t lda, double shift, cudaStream_t s);
void convert_f32_to_f64(int64_t n, int64_t c, const float* src, int64_t lds, double* dst,
                        int64_t ldd, cudaStream_t s);
template <typename T>
void copy_block(int64_t n, int64_t c, const T* src, int64_t lds, T* dst, int64_t ldd,
                cudaStream_t s);

// Y = alpha X (elementwise; Y may alias X)
// dst(perm[i], j) = src(i, j): unpermute_rows (drivers.hpp:209) of an n x c block
void scatter_rows_f64(int64_t n, int64_t c, const double* src, int64_t lds, const int64_t* perm,
                      double* dst, int64_t ldd, cudaStream_t s);
template <typename T>
void scale_block(int64_t n, int64_t c, T alpha, const T* X, int64_t ldx, T* Y, int64_t ldy,
                 cudaStream_t s);

// sum of squares of every entry of an n x c block -> *out (device, double)
template <typename T>
void frob_sq(int64_t n, int64_t c, const T* X, int64_t ldx, double* out, double* work,
             cudaStream_t s);

// ------------------------------------------------------------- residual
// Jacobi/f_T modes of the fused residual kernel
enum ResidMode {
  kResidPlain = 0,     // W = R
  kResidJacobiT = 1,   // W = R .* dinv (dinv in T)
  kResidSandwich = 2,  // W = to_working(to_lower(R) .* dinvf)   (T = double)
};
int64_t resid_workspace_elems(int64_t n, int64_t m);
// R = AX - X diag(theta) (residual_block, eigensolvers.hpp:104-115); column
// norms of R and X (col_norm, dense_matrix.hpp:74-82) -> rnorm/xnorm (device
// double, length m); W = f(R) by mode.  dinv is T or float per mode.
template <typename T>
void residual_precond(int mode, int64_t n, int64_t m, const T* X, int64_t ldx, const T* AX,
                      int64_t ldax, const T* theta, const void* dinv, T* W, int64_t ldw,
                      double* rnorm, double* xnorm, int* overflow_flag, double* work,
                      cudaStream_t s, int raw_sums = 0);
// v = sqrt(v) in real_t<T> (after the row-sharded sums of squares were reduced)
template <typename T>
void norms_sqrt(int64_t count, double* v, cudaStream_t s);
// W = f_T(R) without residual (generic Jacobi apply on a block)
template <typename T>
void jacobi_apply(int mode, int64_t n, int64_t c, const T* R, int64_t ldr, const void* dinv,
                  T* W, int64_t ldw, int* overflow_flag, cudaStream_t s);
// Y = X - W (subtract, dense_kernels.hpp:54-62)
template <typename T>
void subtract(int64_t n, int64_t c, const T* X, int64_t ldx, const T* W, int64_t ldw, T* Y,
              int64_t ldy, cudaStream_t s);

// ------------------------------------------------------------- operators
// 3-D 7-point / 2-D 5-point Laplacian, matrix-free, reference summation order
// (hlo / hhi: the z-planes adjacent to the slab -- the neighbouring ranks'
//  received planes, column j at + j * ldl / ldu (0: nx*ny, packed), or planes
//  of X itself when a sub-slab is applied; nullptr at the domain boundary;
//  dg: the variable diagonal, else 6)
template <typename T>
void stencil7(int64_t nx, int64_t ny, int64_t nz, int64_t c, const T* X, int64_t ldx, T* Y,
              int64_t ldy, cudaStream_t s, const T* hlo = nullptr, const T* hhi = nullptr,
              const T* dg = nullptr, int64_t ldl = 0, int64_t ldu = 0);
template <typename T>
void stencil5(int64_t nx, int64_t ny, int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy,
              cudaStream_t s);
// CSR SpMM (spmv_block, sparse_kernels.hpp:16-33), ascending-column order
template <typename T>
void csr_spmm(int64_t n, const int* row_ptr, const int* col_idx, const T* vals, int64_t nnz,
              int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy, cudaStream_t s);
// the row-sharded CSR apply: rows of a list, ghost columns (>= nown) from G
template <typename T>
void csr_spmm_rows(int64_t nrows, const int* rows, const int* row_ptr, const int* col_idx,
                   const T* vals, int64_t c, const T* X, int64_t ldx, int64_t nown, const T* G,
                   int64_t ldg, T* Y, int64_t ldy, cudaStream_t s);
template <typename T>
void gather_rows(int64_t nrows, const int* idx, int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy,
                 cudaStream_t s);

// ---------------------------------------------------------- small dense
// Small (<= ~600) matrices, single-CTA kernels working in global memory.
// status layout (device int[2]): [0] code, [1] index; the first error wins.
template <typename T>
void small_symmetrize(int64_t s, T* G, int64_t ldg, cudaStream_t st);
// lower Cholesky G = L L^T (dense_cholesky, dense_kernels.hpp:128-152) and
// Uinv = L^{-T} (upper).  On failure status = {NOT_PD|OVERFLOW, index}.
template <typename T>
void small_cholesky_inv(int64_t m, const T* G, int64_t ldg, T* L, T* Uinv, int* status,
                        cudaStream_t st, T tau2 = T(0));
// Rinv = R^{-1} for upper-triangular R (check_tri_diag, dense_kernels.hpp:163-170)
template <typename T>
void small_upper_inverse(int64_t m, const T* R, int64_t ldr, T* Rinv, int* status,
                         cudaStream_t st);
// C = A B for small square/rect blocks (all device, col-major)
template <typename T>
void small_matmul(int64_t r, int64_t k, int64_t c, const T* A, int64_t lda, const T* B,
                  int64_t ldb, T* C, int64_t ldc, cudaStream_t st);
// B = A^T
template <typename T>
void small_transpose(int64_t r, int64_t c, const T* A, int64_t lda, T* B, int64_t ldb,
                     cudaStream_t st);
// Hetmaniuk-Lehoucq coefficient block (eigensolvers.hpp:148-174):
// coef = [C(:,0:m) | C(:,m:m+p) V], V from householder_qr_square of
// C(0:m, m:m+p)^T (ortho.hpp:114-121); rank-deficient -> V = I, flag.
void hl_coeffs(int64_t s, int64_t m, int64_t p, const double* C, int64_t ldc, double* coef,
               double* scratch, int* fallback, cudaStream_t st);
void hl_coeffs_f32(int64_t s, int64_t m, int64_t p, const float* C, int64_t ldc, float* coef,
                   float* scratch, int* fallback, cudaStream_t st);

// Symmetric eigendecomposition of a small s x s matrix in one CTA (syev.cu):
// ascending values, vectors overwrite G.  info = 1 on QL non-convergence.
constexpr int64_t kSyevMax = 96;
template <typename T>
bool small_syev_supported(int64_t s);
template <typename T>
void small_syev(int64_t s, T* G, int64_t ldg, T* vals, int* info, cudaStream_t st, int exact = -1);
// same, with per-phase clock64 counters (tridiag, QL, sort, sweeps, chain) into prof
template <typename T>
void small_syev_prof(int64_t s, T* G, int64_t ldg, T* vals, int* info, long long* prof,
                     cudaStream_t st, int exact = -1);

// ------------------------------------------------------------------ TSQR
// R factor (m x m, upper, positive diagonal) of a tall n x m block by a
// Householder TSQR tree in precision Tq; the input is read in Tin and
// narrowed on load when Tin != Tq (to_lower with overflow check).
// status: [0] = RANK_DEFICIENT / OVERFLOW, [1] = column index.
template <typename Tin, typename Tq>
int64_t tsqr_workspace_elems(int64_t n, int64_t m);
template <typename Tin, typename Tq>
bool tsqr_fits(int64_t n, int64_t m);
template <typename Tin, typename Tq>
void tsqr_r(int64_t n, int64_t m, const Tin* W, int64_t ldw, Tq* R, int64_t ldr, Tq* work,
            int* status, cudaStream_t s, Tin* Rw_out = nullptr, Tin* Rinv_out = nullptr,
            int rank_check = -1);
// (rank_check: -1 numeric check iff Tin == Tq (default), 0 exact zeros only,
//  1 numeric; a row-shard's local R factor uses 0 -- only the global R counts)
// R (Tq) -> Rw (Tin, m x m) and Rinv = R^-1 (Tin), for an R already formed
template <typename Tin, typename Tq>
void tsqr_epilogue(int64_t m, const Tq* R, int64_t ldr, Tin* Rw, Tin* Rinv, int* status,
                   cudaStream_t s);
// (Rinv_out != nullptr: also R in Tin (Rw_out, m x m) and R^{-1} (m x m) --
//  fused into the TSQR root for m <= 16)

}  // namespace mpb
