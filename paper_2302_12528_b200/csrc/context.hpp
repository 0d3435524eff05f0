// context.hpp -- context, operators and device buffers (host side).
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdint>
#include <string>
#include <vector>

#include "comm.hpp"
#include "common.cuh"
#include "kernels.cuh"

struct mpeig_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // own stream (created for a NULL stream argument): every C-ABI call is
  // ordered after prior work on the legacy default stream and before later
  // work there, through these two events
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  cublasHandle_t cublas = nullptr;
  std::string last_msg;
  int64_t last_index = -1;
  int* d_status = nullptr;      // 16 ints of device status slots
  int* h_status = nullptr;      // pinned mirror
  double* h_pinned = nullptr;   // pinned staging for per-iteration records
  int64_t h_pinned_elems = 0;
  int eig_backend = 0;          // 0 auto (one-CTA syev for s <= kSyevMax), 1 cuSOLVER
  int spec_mode = 1;            // speculative iteration (1 host sync / iteration)
  int use_graphs = 1;           // replay the steady-state iteration as a CUDA graph
  int spec_qr = 10;             // speculative body's QR: k > 0 guarded CholQR2 (fp64 guard 1e-k), 0 TSQR
  int ql_exact = -1;            // QL rotation formulas of the one-CTA eigensolver (syev.cu)
  int64_t spec_rollbacks = 0;   // speculative iterations repeated on the careful path
  mpb::Comm* comm = nullptr;    // row-sharded mode (owned), nullptr: single GPU
};

enum OpKind { kOpLap3d, kOpLap2d, kOpCsr, kOpDense, kOpDeviceCb, kOpHostCb, kOpJacobi, kOpDenseChol, kOpSparseChol };

struct mpeig_op {
  OpKind kind;
  mpeig_ctx* ctx = nullptr;
  int64_t n = 0, nx = 0, ny = 0, nz = 0;
  // row sharding: this rank holds global rows [row0, row0 + n) of n_global
  // (z-slab [z0, z0 + nz) of nz_global for the stencil)
  int64_t n_global = 0, row0 = 0, z0 = 0, nz_global = 0;
  bool slab = false;
  mutable void* halo = nullptr;  // send/recv planes of the slab exchange
  mutable size_t halo_bytes = 0;
  mutable cudaStream_t halo_stream = nullptr;  // the overlapped halo exchange
  mutable cudaEvent_t ev_packed = nullptr, ev_halo = nullptr;
  // CSR (device)
  int64_t* rp = nullptr;
  int64_t* ci = nullptr;
  double* dgw = nullptr;  // 7-pt stencil with a variable diagonal (-Laplacian + V): 6 + V_i
  float* dgl = nullptr;   // to_lower of it
  std::vector<double> dg_host;
  int* rp32 = nullptr;  // the same pattern with int32 indices (the SpMM's; n, nnz < 2^31)
  int* ci32 = nullptr;
  int64_t nnz = 0;
  double* vals = nullptr;
  float* vals_l = nullptr;
  // row-sharded CSR (mpeig_op_csr_rows): local column indices, owned rows
  // first then the ghost rows (other ranks' rows this rank's entries touch),
  // grouped by owner; per peer the rows sent / received (host, in rows)
  int64_t n_ghost = 0, n_send = 0;
  std::vector<int64_t> gx_send_rows, gx_send_off, gx_recv_rows, gx_recv_off;
  int* gx_send_idx = nullptr;  // local rows packed for the peers, peer order
  int* rows_inner = nullptr;   // rows without ghost entries (computed during the exchange)
  int* rows_bnd = nullptr;     // rows with ghost entries (after it)
  int64_t n_inner = 0, n_bnd = 0;
  // dense (device)
  double* A = nullptr;
  float* Al = nullptr;
  int64_t lda = 0;
  // callbacks
  mpeig_apply_fn dev_w = nullptr, dev_l = nullptr;
  mpeig_host_apply_fn host_w = nullptr, host_l = nullptr;
  void* user = nullptr;
  // Jacobi
  int32_t precision = MPEIG_WORKING;
  double* dinv = nullptr;   // 1 / diag, fp64
  float* dinvf = nullptr;   // to_lower(1 / diag)
  bool lower_overflow = false;  // to_lower of the coefficients overflowed
  // dense Cholesky f_T (Preconditioner::Kind::DenseChol, precond.hpp:33-50):
  // lower factor L (n x n, ld n) in the build precision
  double* Lw = nullptr;
  float* Ll = nullptr;
  double shift = 0.0;          // retry_dense's diagonal shift (precond.hpp:140-146)
  int64_t tri_singular = -1;   // first zero / subnormal diag(L) (check_tri_diag)
  mutable float* scratch = nullptr;  // to_lower(R) of a working-precision apply
  mutable size_t scratch_elems = 0;
  // sparse Cholesky f_T (Kind::SparseCholKind, precond.hpp:55-77): L rows with
  // the diagonal last, U = L^T rows with the diagonal first, int32 indices;
  // values in the build precision; perm[k] = original index of row k
  int* sp_Lrp = nullptr;
  int* sp_Lci = nullptr;
  int* sp_Urp = nullptr;
  int* sp_Uci = nullptr;
  int* sp_perm = nullptr;
  int* sp_Lsp = nullptr;  // per row: first L entry inside the row's 32-row block
  int* sp_Usp = nullptr;  // per row: first U entry right of the row's block
  void* sp_Lv = nullptr;
  void* sp_Uv = nullptr;
  int64_t sp_nnz = 0;
};

namespace mpb {

// RAII stream-ordered device buffer
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  void alloc(size_t n, cudaStream_t st) {
    release();
    s = st;
    count = n;
    if (n) MPB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st));
  }
  // workspaces holding self-resetting tree counters (gram, tsqr) start zeroed
  void alloc_zero(size_t n, cudaStream_t st) {
    alloc(n, st);
    if (n) MPB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    count = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count), s(o.s) { o.p = nullptr; o.count = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p;
    count = o.count;
    s = o.s;
    o.p = nullptr;
    o.count = 0;
    return *this;
  }
  T* get() const { return p; }
};

// host-side gaussian block generation (rng.cpp)
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out);
// rows [row0, row0 + rows) of the n_global x cols block gaussian_fill draws
void gaussian_fill_rows(int64_t n_global, int64_t cols, uint64_t seed, int64_t row0, int64_t rows,
                        double* out);

// the communicator when the context runs row-sharded (any attached comm,
// a 1-rank one included: that runs the sharded code path on one GPU)
inline Comm* dist(const mpeig_ctx* ctx) { return ctx->comm; }
uint64_t pcg64_draw(uint64_t seed, uint64_t index);

// operator application (ops dispatch in solver.cpp)
template <typename T>
void op_apply(mpeig_ctx* ctx, const mpeig_op* op, int64_t ncols, const T* X, int64_t ldx, T* Y,
              int64_t ldy);

// status helpers
void status_clear(mpeig_ctx* ctx);
void status_fetch(mpeig_ctx* ctx);  // synchronises the stream

}  // namespace mpb
