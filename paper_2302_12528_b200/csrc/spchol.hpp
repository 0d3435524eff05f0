// Sparse Cholesky preconditioner: host factorisation
// (spchol_host.cpp) and device triangular solves (spchol.cu).
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace mpb {

template <typename F>
struct HostFactor {  // CSR lower factor, diagonal last in each row
  std::vector<int64_t> rp, ci;
  std::vector<F> v;
};

// host factorisation threads (process option "spchol_threads"; 0 = hardware)
extern int g_spchol_threads;
std::vector<int64_t> rcm_ordering(int64_t n, const int64_t* rp, const int64_t* ci);
template <typename V>
void csr_permute(int64_t n, const int64_t* rp, const int64_t* ci, const V* v,
                 const std::vector<int64_t>& perm, std::vector<int64_t>& brp,
                 std::vector<int64_t>& bci, std::vector<V>& bv);
template <typename F>
HostFactor<F> sparse_cholesky_host(int64_t n, const std::vector<int64_t>& rp,
                                   const std::vector<int64_t>& ci, const std::vector<F>& v);

// W = Pi L^-T L^-1 Pi^T R on the device (sparse_tri_solve, sparse_kernels.hpp:178-225):
// one CTA per block column, rows in blocks of 32; Tin -> F narrowing (overflow
// flag) and F -> Tout widening fused into the gather / scatter.  L rows: diagonal
// last, Lsp[i] = first entry of row i inside row i's 32-row block (Lsp[n + i]: first
// entry of the previous block); U = L^T rows: diagonal first, Usp[i] = first entry
// right of row i's block (Usp[n + i]: first entry two blocks right).  perm may be null
// (identity).  gy: n x c scratch of F used when a column exceeds shared memory.
template <typename Tin, typename F, typename Tout>
void spchol_solve(int n, int c, const int* Lrp, const int* Lci, const F* Lv, const int* Lsp,
                  const int* Urp, const int* Uci, const F* Uv, const int* Usp, const int* perm,
                  const Tin* B, int64_t ldb, Tout* Y, int64_t ldy, int* overflow, F* gy,
                  cudaStream_t s);

}  // namespace mpb
