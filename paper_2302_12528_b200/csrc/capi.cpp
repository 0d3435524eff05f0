// capi.cpp -- the extern "C" boundary (include/mpeig_b200.h).
//
// Every entry point catches mpb::Error and CUDA failures and maps them to an
// mpeig_status (1:1 with the reference exception types, errors.hpp:10-62),
// keeping the message and index payload on the context.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "context.hpp"
#include "solver.hpp"
#include "spchol.hpp"

using namespace mpb;

namespace {

// a context on its own stream joins the legacy default stream around each call
struct LegacyOrder {
  mpeig_ctx* ctx;
  explicit LegacyOrder(mpeig_ctx* c) : ctx(c && c->own_stream && c->ev_in ? c : nullptr) {
    if (!ctx) return;
    cudaEventRecord(ctx->ev_in, cudaStreamLegacy);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0);
  }
  ~LegacyOrder() {
    if (!ctx) return;
    cudaEventRecord(ctx->ev_out, ctx->stream);
    cudaStreamWaitEvent(cudaStreamLegacy, ctx->ev_out, 0);
  }
};

template <typename F>
int guard(mpeig_ctx* ctx, F&& f) {
  // A non-sticky error left in the runtime's per-thread slot by a call outside
  // this entry point (another library, a context torn down by the garbage
  // collector) must not be reported by this call's launch checks; sticky
  // errors still surface on the next runtime call.
  (void)cudaGetLastError();
  try {
    LegacyOrder order(ctx);
    f();
    if (ctx) {
      ctx->last_msg.clear();
      ctx->last_index = -1;
    }
    return MPEIG_OK;
  } catch (const Error& e) {
    if (ctx) {
      ctx->last_msg = e.what();
      ctx->last_index = e.index;
    }
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_msg = "host allocation failed";
    return MPEIG_E_OTHER;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_msg = e.what();
    return MPEIG_E_OTHER;
  }
}

void set_device(mpeig_ctx* ctx) { MPB_CUDA(cudaSetDevice(ctx->device)); }

mpeig_op* new_op(mpeig_ctx* ctx, OpKind k, int64_t n) {
  auto* op = new mpeig_op();
  op->kind = k;
  op->ctx = ctx;
  op->n = n;
  return op;
}

template <typename T>
T* upload(const T* host, size_t count, cudaStream_t s) {
  T* d = nullptr;
  MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), count * sizeof(T)));
  MPB_CUDA(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return d;
}

// to_lower of a coefficient array (precision.hpp:102-107); false on overflow
bool narrow(const double* src, size_t count, std::vector<float>& dst) {
  dst.resize(count);
  bool ok = true;
  for (size_t i = 0; i < count; ++i) {
    const float y = static_cast<float>(src[i]);
    if (std::isfinite(src[i]) && !std::isfinite(y)) ok = false;
    dst[i] = y;
  }
  return ok;
}

}  // namespace

extern "C" {

int mpeig_ctx_create(int device, void* cuda_stream, mpeig_ctx** out) {
  auto* ctx = new mpeig_ctx();
  ctx->device = device;
  const int rc = guard(ctx, [&] {
    MPB_CUDA(cudaSetDevice(device));
    if (cuda_stream) {
      ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
      MPB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      MPB_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
      MPB_CUDA(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
      ctx->own_stream = true;
    }
    if (cusolverDnCreate(&ctx->cusolver) != CUSOLVER_STATUS_SUCCESS)
      throw Error(MPEIG_E_CUSOLVER, "cusolverDnCreate failed");
    cusolverDnSetStream(ctx->cusolver, ctx->stream);
    if (cublasCreate(&ctx->cublas) != CUBLAS_STATUS_SUCCESS)
      throw Error(MPEIG_E_CUDA, "cublasCreate failed");
    cublasSetStream(ctx->cublas, ctx->stream);
    cublasSetMathMode(ctx->cublas, CUBLAS_PEDANTIC_MATH);  // no TF32 in the fp32 stage
    MPB_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->d_status), 16 * sizeof(int)));
    MPB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_status), 16 * sizeof(int)));
    ctx->h_pinned_elems = 4096;
    MPB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_pinned),
                            static_cast<size_t>(ctx->h_pinned_elems) * sizeof(double)));
    // keep freed stage buffers cached in the stream-ordered pool
    cudaMemPool_t pool;
    MPB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  });
  if (rc != MPEIG_OK) {
    mpeig_ctx_destroy(ctx);
    *out = nullptr;
    return rc;
  }
  *out = ctx;
  return MPEIG_OK;
}

void mpeig_ctx_destroy(mpeig_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->cusolver) cusolverDnDestroy(ctx->cusolver);
  if (ctx->cublas) cublasDestroy(ctx->cublas);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->own_stream && ctx->stream) {
    tc_scratch_release(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  delete ctx->comm;
  delete ctx;
  (void)cudaGetLastError();  // teardown must not leave an error for the next caller
}

const char* mpeig_last_error(mpeig_ctx* ctx, int64_t* index) {
  if (!ctx) return "null context";
  if (index) *index = ctx->last_index;
  return ctx->last_msg.c_str();
}

int64_t mpeig_launch_count(mpeig_ctx* ctx, int reset) {
  (void)ctx;
  return reset ? g_launches.exchange(0) : g_launches.load();
}

void* mpeig_ctx_stream(mpeig_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

// ---- row sharding (comm.hpp)
int mpeig_host_group_create(int nranks, void** out) {
  if (!out || nranks < 1) return MPEIG_E_CONFIG;
  *out = new mpb::HostGroup(nranks);
  return MPEIG_OK;
}

void mpeig_host_group_destroy(void* group) { delete static_cast<mpb::HostGroup*>(group); }

int mpeig_ctx_attach_host_comm(mpeig_ctx* ctx, void* group, int rank) {
  return guard(ctx, [&] {
    auto* g = static_cast<mpb::HostGroup*>(group);
    if (!g || rank < 0 || rank >= g->nranks) throw Error(MPEIG_E_CONFIG, "bad host group / rank");
    delete ctx->comm;
    ctx->comm = new mpb::HostComm(g, rank);
  });
}

int mpeig_nccl_unique_id(void* out, int64_t cap) {
  if (!out || cap < 128) return MPEIG_E_CONFIG;
  try {
    mpb::nccl_unique_id(out);
  } catch (const Error& e) {
    return e.code;
  }
  return MPEIG_OK;
}

int mpeig_ctx_attach_nccl(mpeig_ctx* ctx, int rank, int nranks, const void* id) {
  return guard(ctx, [&] {
    if (!id || rank < 0 || rank >= nranks) throw Error(MPEIG_E_CONFIG, "bad NCCL rank / id");
    MPB_CUDA(cudaSetDevice(ctx->device));
    mpb::Comm* c = mpb::make_nccl_comm(rank, nranks, id);
    delete ctx->comm;
    ctx->comm = c;
  });
}

int64_t mpeig_spec_rollbacks(mpeig_ctx* ctx, int reset) {
  if (!ctx) return 0;
  const int64_t v = ctx->spec_rollbacks;
  if (reset) ctx->spec_rollbacks = 0;
  return v;
}

int mpeig_ctx_set_option(mpeig_ctx* ctx, const char* key, int value) {
  if (!ctx || !key) return MPEIG_E_CONFIG;
  const std::string k(key);
  if (k == "eig_backend") ctx->eig_backend = value;
  else if (k == "spec_mode") ctx->spec_mode = value;
  else if (k == "use_graphs") ctx->use_graphs = value;
  else if (k == "spec_qr") ctx->spec_qr = value;
  else if (k == "ql_exact") ctx->ql_exact = value;
  else return MPEIG_E_CONFIG;
  return MPEIG_OK;
}

// ---------------------------------------------------------------- operators
int mpeig_op_lap3d(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, mpeig_op** out) {
  return guard(ctx, [&] {
    if (nx < 1 || ny < 1 || nz < 1) throw Error(MPEIG_E_CONFIG, "lap3d: grid sides must be >= 1");
    mpeig_op* op = new_op(ctx, kOpLap3d, nx * ny * nz);
    op->nx = nx;
    op->ny = ny;
    op->nz = nz;
    *out = op;
  });
}

int mpeig_op_lap3d_slab(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz_global, int64_t z0,
                        int64_t nz_local, mpeig_op** out) {
  return guard(ctx, [&] {
    if (nx < 1 || ny < 1 || nz_local < 1 || z0 < 0 || z0 + nz_local > nz_global)
      throw Error(MPEIG_E_CONFIG, "lap3d_slab: bad slab");
    mpeig_op* op = new_op(ctx, kOpLap3d, nx * ny * nz_local);
    op->nx = nx;
    op->ny = ny;
    op->nz = nz_local;
    op->slab = true;
    op->z0 = z0;
    op->nz_global = nz_global;
    op->n_global = nx * ny * nz_global;
    op->row0 = nx * ny * z0;
    *out = op;
  });
}

namespace {
// the variable diagonal (6 + V_i) of a 7-pt operator: host copy, fp64 and
// to_lower'd fp32 device copies
void attach_diag(mpeig_ctx* ctx, mpeig_op* op, const double* diag_host) {
  const int64_t n = op->n;
  op->dg_host.assign(diag_host, diag_host + n);
  cudaStream_t s = ctx->stream;
  op->dgw = upload(diag_host, static_cast<size_t>(n), s);
  std::vector<float> dl;
  op->lower_overflow = !narrow(diag_host, static_cast<size_t>(n), dl);
  op->dgl = upload(dl.data(), dl.size(), s);
  MPB_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

int mpeig_op_lap3d_slab_diag(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz_global, int64_t z0,
                             int64_t nz_local, const double* diag_local_host, mpeig_op** out) {
  mpeig_op* op = nullptr;
  int rc = mpeig_op_lap3d_slab(ctx, nx, ny, nz_global, z0, nz_local, &op);
  if (rc != MPEIG_OK) return rc;
  rc = guard(ctx, [&] {
    set_device(ctx);
    if (!diag_local_host) throw Error(MPEIG_E_CONFIG, "lap3d_slab_diag: null diagonal");
    attach_diag(ctx, op, diag_local_host);
  });
  if (rc != MPEIG_OK) {
    mpeig_op_destroy(op);
    return rc;
  }
  *out = op;
  return MPEIG_OK;
}

int mpeig_op_lap3d_diag(mpeig_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, const double* diag_host,
                        mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (nx < 1 || ny < 1 || nz < 1) throw Error(MPEIG_E_CONFIG, "lap3d: grid sides must be >= 1");
    if (!diag_host) throw Error(MPEIG_E_CONFIG, "lap3d_diag: null diagonal");
    const int64_t n = nx * ny * nz;
    mpeig_op* op = new_op(ctx, kOpLap3d, n);
    op->nx = nx;
    op->ny = ny;
    op->nz = nz;
    attach_diag(ctx, op, diag_host);
    *out = op;
  });
}

int mpeig_op_lap2d(mpeig_ctx* ctx, int64_t nx, int64_t ny, mpeig_op** out) {
  return guard(ctx, [&] {
    if (nx < 1 || ny < 1) throw Error(MPEIG_E_CONFIG, "gen_laplace2d: grid sides must be >= 1");
    mpeig_op* op = new_op(ctx, kOpLap2d, nx * ny);
    op->nx = nx;
    op->ny = ny;
    op->nz = 1;
    *out = op;
  });
}

int mpeig_op_csr(mpeig_ctx* ctx, int64_t n, const int64_t* row_ptr_host,
                 const int64_t* col_idx_host, const double* vals_host, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (n < 1) throw Error(MPEIG_E_DIMENSION, "csr: n must be >= 1");
    const int64_t nnz = row_ptr_host[n];
    for (int64_t i = 0; i < n; ++i) {
      if (row_ptr_host[i + 1] < row_ptr_host[i]) throw Error(MPEIG_E_DIMENSION, "csr: row_ptr not monotone");
      for (int64_t q = row_ptr_host[i]; q < row_ptr_host[i + 1]; ++q) {
        if (col_idx_host[q] < 0 || col_idx_host[q] >= n)
          throw Error(MPEIG_E_DIMENSION, "from_triplets: index out of range");
        if (q > row_ptr_host[i] && col_idx_host[q] <= col_idx_host[q - 1])
          throw Error(MPEIG_E_DIMENSION, "csr: columns must be sorted and unique per row");
      }
    }
    mpeig_op* op = new_op(ctx, kOpCsr, n);
    cudaStream_t s = ctx->stream;
    if (n >= INT32_MAX || nnz >= INT32_MAX)
      throw Error(MPEIG_E_CONFIG, "csr: n and nnz must stay below 2^31 (int32 device indices)");
    op->rp = upload(row_ptr_host, static_cast<size_t>(n + 1), s);
    op->ci = upload(col_idx_host, static_cast<size_t>(nnz), s);
    op->nnz = nnz;
    {
      std::vector<int> rp32(row_ptr_host, row_ptr_host + n + 1), ci32(col_idx_host, col_idx_host + nnz);
      op->rp32 = upload(rp32.data(), rp32.size(), s);
      op->ci32 = upload(ci32.data(), ci32.size(), s);
      MPB_CUDA(cudaStreamSynchronize(s));  // the host staging vectors go out of scope
    }
    op->vals = upload(vals_host, static_cast<size_t>(nnz), s);
    std::vector<float> vl;
    op->lower_overflow = !narrow(vals_host, static_cast<size_t>(nnz), vl);
    op->vals_l = upload(vl.data(), vl.size(), s);
    MPB_CUDA(cudaStreamSynchronize(s));
    *out = op;
  });
}

namespace {
// small host vectors through the communicator's device-side collectives
std::vector<int64_t> allgather_host(Comm* c, const std::vector<int64_t>& mine, cudaStream_t s) {
  const size_t cnt = mine.size();
  DevBuf<int64_t> d(cnt, s), all(cnt * c->nranks, s);
  MPB_CUDA(cudaMemcpyAsync(d.p, mine.data(), sizeof(int64_t) * cnt, cudaMemcpyHostToDevice, s));
  c->allgather(d.p, all.p, static_cast<int64_t>(sizeof(int64_t) * cnt), s);
  std::vector<int64_t> out(cnt * c->nranks);
  MPB_CUDA(cudaMemcpyAsync(out.data(), all.p, sizeof(int64_t) * out.size(), cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  return out;
}
}  // namespace

int mpeig_op_csr_rows(mpeig_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local,
                      const int64_t* row_ptr_host, const int64_t* col_idx_host,
                      const double* vals_host, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    Comm* c = dist(ctx);
    const int nr = c ? c->nranks : 1, me = c ? c->rank : 0;
    if (!c && (row0 != 0 || n_local != n_global))
      throw Error(MPEIG_E_CONFIG, "csr_rows: a partial row block needs a communicator");
    // validate locally, then agree: a rank with a bad block must not leave the
    // others waiting in the partition exchange, so every rank throws together
    int bad_code = MPEIG_OK;
    std::string bad_msg;
    const auto fail = [&](int code, const char* msg) {
      if (bad_code == MPEIG_OK) {
        bad_code = code;
        bad_msg = msg;
      }
    };
    if (n_local < 1 || row0 < 0 || row0 + n_local > n_global) fail(MPEIG_E_DIMENSION, "csr_rows: bad row range");
    const int64_t nnz = bad_code == MPEIG_OK ? row_ptr_host[n_local] : 0;
    for (int64_t i = 0; bad_code == MPEIG_OK && i < n_local; ++i) {
      if (row_ptr_host[i + 1] < row_ptr_host[i]) fail(MPEIG_E_DIMENSION, "csr: row_ptr not monotone");
      for (int64_t q = row_ptr_host[i]; bad_code == MPEIG_OK && q < row_ptr_host[i + 1]; ++q) {
        if (col_idx_host[q] < 0 || col_idx_host[q] >= n_global)
          fail(MPEIG_E_DIMENSION, "from_triplets: index out of range");
        else if (q > row_ptr_host[i] && col_idx_host[q] <= col_idx_host[q - 1])
          fail(MPEIG_E_DIMENSION, "csr: columns must be sorted and unique per row");
      }
    }
    if (bad_code == MPEIG_OK && (n_global >= INT32_MAX || nnz >= INT32_MAX))
      fail(MPEIG_E_CONFIG, "csr: n and nnz must stay below 2^31 (int32 device indices)");
    cudaStream_t s = ctx->stream;
    // the rank partition: contiguous row blocks in rank order covering n_global
    std::vector<int64_t> start(static_cast<size_t>(nr) + 1, 0);
    if (c) {
      const std::vector<int64_t> rr = allgather_host(c, {row0, n_local, bad_code}, s);
      if (bad_code != MPEIG_OK) throw Error(bad_code, bad_msg);
      for (int q = 0; q < nr; ++q)
        if (rr[3 * q + 2] != MPEIG_OK)
          throw Error(static_cast<int>(rr[3 * q + 2]), "csr_rows: rank " + std::to_string(q) + "'s row block is invalid");
      for (int q = 0; q < nr; ++q) {
        if (rr[3 * q] != start[q])
          throw Error(MPEIG_E_CONFIG, "csr_rows: rank row blocks must be contiguous in rank order");
        start[q + 1] = rr[3 * q] + rr[3 * q + 1];
      }
    } else {
      if (bad_code != MPEIG_OK) throw Error(bad_code, bad_msg);
      start[1] = n_global;
    }
    if (start[nr] != n_global) throw Error(MPEIG_E_CONFIG, "csr_rows: row blocks do not cover n_global");
    // ghost columns (sorted, hence grouped by owner) and local column indices
    std::vector<int64_t> ghosts;
    for (int64_t q = 0; q < nnz; ++q) {
      const int64_t g = col_idx_host[q];
      if (g < row0 || g >= row0 + n_local) ghosts.push_back(g);
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    const int64_t ng = static_cast<int64_t>(ghosts.size());
    std::vector<int> ci32(static_cast<size_t>(nnz)), rp32(row_ptr_host, row_ptr_host + n_local + 1);
    std::vector<int> inner, bnd;
    for (int64_t i = 0; i < n_local; ++i) {
      bool has_ghost = false;
      for (int64_t q = row_ptr_host[i]; q < row_ptr_host[i + 1]; ++q) {
        const int64_t g = col_idx_host[q];
        if (g >= row0 && g < row0 + n_local) {
          ci32[q] = static_cast<int>(g - row0);
        } else {
          ci32[q] = static_cast<int>(n_local + (std::lower_bound(ghosts.begin(), ghosts.end(), g) -
                                                ghosts.begin()));
          has_ghost = true;
        }
      }
      (has_ghost ? bnd : inner).push_back(static_cast<int>(i));
    }
    mpeig_op* op = new_op(ctx, kOpCsr, n_local);
    op->n_global = n_global;
    op->row0 = row0;
    op->nnz = nnz;
    op->n_ghost = ng;
    // per peer: the rows this rank receives (its ghosts owned by q) ...
    op->gx_recv_rows.assign(nr, 0);
    op->gx_recv_off.assign(nr, 0);
    for (int64_t g : ghosts) {
      const int q = static_cast<int>(std::upper_bound(start.begin(), start.end(), g) - start.begin()) - 1;
      ++op->gx_recv_rows[q];
    }
    for (int q = 1; q < nr; ++q) op->gx_recv_off[q] = op->gx_recv_off[q - 1] + op->gx_recv_rows[q - 1];
    // ... and the rows it sends: the count matrix, then the index lists
    op->gx_send_rows.assign(nr, 0);
    op->gx_send_off.assign(nr, 0);
    std::vector<int64_t> send_idx;
    if (c) {
      const std::vector<int64_t> cm = allgather_host(c, op->gx_recv_rows, s);  // cm[r * nr + q]
      for (int q = 0; q < nr; ++q) op->gx_send_rows[q] = cm[static_cast<size_t>(q) * nr + me];
      for (int q = 1; q < nr; ++q) op->gx_send_off[q] = op->gx_send_off[q - 1] + op->gx_send_rows[q - 1];
      op->n_send = op->gx_send_off[nr - 1] + op->gx_send_rows[nr - 1];
      // rank r asks owner q for its ghost list's q-part (global row indices)
      std::vector<int64_t> sb(nr), so(nr), rb(nr), ro(nr);
      for (int q = 0; q < nr; ++q) {
        sb[q] = 8 * op->gx_recv_rows[q];
        so[q] = 8 * op->gx_recv_off[q];
        rb[q] = 8 * op->gx_send_rows[q];
        ro[q] = 8 * op->gx_send_off[q];
      }
      DevBuf<int64_t> dreq(static_cast<size_t>(std::max<int64_t>(ng, 1)), s);
      DevBuf<int64_t> dgot(static_cast<size_t>(std::max<int64_t>(op->n_send, 1)), s);
      if (ng) MPB_CUDA(cudaMemcpyAsync(dreq.p, ghosts.data(), 8 * ng, cudaMemcpyHostToDevice, s));
      c->alltoallv(dreq.p, sb.data(), so.data(), dgot.p, rb.data(), ro.data(), s);
      send_idx.resize(static_cast<size_t>(op->n_send));
      if (op->n_send)
        MPB_CUDA(cudaMemcpyAsync(send_idx.data(), dgot.p, 8 * op->n_send, cudaMemcpyDeviceToHost, s));
      MPB_CUDA(cudaStreamSynchronize(s));
      for (int64_t& g : send_idx) {
        if (g < row0 || g >= row0 + n_local) throw Error(MPEIG_E_COMM, "csr_rows: ghost request for a foreign row");
        g -= row0;
      }
    }
    std::vector<int> send32(send_idx.begin(), send_idx.end());
    op->rp = upload(row_ptr_host, static_cast<size_t>(n_local + 1), s);
    op->ci = upload(col_idx_host, static_cast<size_t>(nnz), s);  // global (Jacobi's diagonal)
    op->rp32 = upload(rp32.data(), rp32.size(), s);
    op->ci32 = upload(ci32.data(), ci32.size(), s);
    op->gx_send_idx = upload(send32.data(), send32.size(), s);
    op->rows_inner = upload(inner.data(), inner.size(), s);
    op->rows_bnd = upload(bnd.data(), bnd.size(), s);
    op->n_inner = static_cast<int64_t>(inner.size());
    op->n_bnd = static_cast<int64_t>(bnd.size());
    op->vals = upload(vals_host, static_cast<size_t>(nnz), s);
    std::vector<float> vl;
    op->lower_overflow = !narrow(vals_host, static_cast<size_t>(nnz), vl);
    op->vals_l = upload(vl.data(), vl.size(), s);
    MPB_CUDA(cudaStreamSynchronize(s));  // host staging vectors go out of scope
    op->slab = c != nullptr;
    *out = op;
  });
}

int mpeig_op_dense(mpeig_ctx* ctx, int64_t n, const double* A_host, int64_t lda, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (n < 1 || lda < n) throw Error(MPEIG_E_DIMENSION, "dense: bad shape");
    mpeig_op* op = new_op(ctx, kOpDense, n);
    std::vector<double> a(static_cast<size_t>(n * n));
    for (int64_t j = 0; j < n; ++j) std::memcpy(&a[j * n], A_host + j * lda, sizeof(double) * n);
    cudaStream_t s = ctx->stream;
    op->A = upload(a.data(), a.size(), s);
    op->lda = n;
    std::vector<float> al;
    op->lower_overflow = !narrow(a.data(), a.size(), al);
    op->Al = upload(al.data(), al.size(), s);
    MPB_CUDA(cudaStreamSynchronize(s));
    *out = op;
  });
}

int mpeig_op_device_callback(mpeig_ctx* ctx, int64_t n, mpeig_apply_fn apply_working,
                             mpeig_apply_fn apply_lower, void* user, mpeig_op** out) {
  return guard(ctx, [&] {
    mpeig_op* op = new_op(ctx, kOpDeviceCb, n);
    op->dev_w = apply_working;
    op->dev_l = apply_lower;
    op->user = user;
    *out = op;
  });
}

int mpeig_op_host_callback(mpeig_ctx* ctx, int64_t n, mpeig_host_apply_fn apply_working,
                           mpeig_host_apply_fn apply_lower, void* user, mpeig_op** out) {
  return guard(ctx, [&] {
    mpeig_op* op = new_op(ctx, kOpHostCb, n);
    op->host_w = apply_working;
    op->host_l = apply_lower;
    op->user = user;
    *out = op;
  });
}

int mpeig_precond_jacobi(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    const int64_t n = A->n;
    std::vector<double> d(static_cast<size_t>(n));
    cudaStream_t s = ctx->stream;
    switch (A->kind) {
      case kOpLap3d:
        if (!A->dg_host.empty())
          d = A->dg_host;
        else
          std::fill(d.begin(), d.end(), 6.0);
        break;
      case kOpLap2d:
        std::fill(d.begin(), d.end(), 4.0);
        break;
      case kOpCsr: {
        std::vector<int64_t> rp(static_cast<size_t>(n + 1));
        MPB_CUDA(cudaMemcpyAsync(rp.data(), A->rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
        MPB_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> ci(static_cast<size_t>(rp[n]));
        std::vector<double> v(static_cast<size_t>(rp[n]));
        MPB_CUDA(cudaMemcpyAsync(ci.data(), A->ci, sizeof(int64_t) * rp[n], cudaMemcpyDeviceToHost, s));
        MPB_CUDA(cudaMemcpyAsync(v.data(), A->vals, sizeof(double) * rp[n], cudaMemcpyDeviceToHost, s));
        MPB_CUDA(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < n; ++i) {  // (global column indices: row0 + i on a shard)
          d[i] = 0.0;
          for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
            if (ci[q] == A->row0 + i) d[i] = v[q];
        }
        break;
      }
      case kOpDense: {
        for (int64_t i = 0; i < n; ++i)
          MPB_CUDA(cudaMemcpyAsync(&d[i], A->A + i + i * A->lda, sizeof(double), cudaMemcpyDeviceToHost, s));
        MPB_CUDA(cudaStreamSynchronize(s));
        break;
      }
      default:
        throw Error(MPEIG_E_CONFIG, "jacobi: operator has no explicit diagonal");
    }
    std::vector<double> dinv(static_cast<size_t>(n));
    std::vector<float> dinvf(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      if (!(d[i] != 0.0)) throw Error(MPEIG_E_NOT_PD, "jacobi: zero diagonal", i);
      dinv[i] = 1.0 / d[i];
      dinvf[i] = static_cast<float>(dinv[i]);
    }
    mpeig_op* op = new_op(ctx, kOpJacobi, n);
    op->precision = precision;
    op->dinv = upload(dinv.data(), dinv.size(), s);
    op->dinvf = upload(dinvf.data(), dinvf.size(), s);
    MPB_CUDA(cudaStreamSynchronize(s));
    *out = op;
  });
}

int mpeig_precond_dense_chol(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (!A) throw Error(MPEIG_E_CONFIG, "dense_chol: null operator");
    if (precision != MPEIG_WORKING && precision != MPEIG_LOWER)
      throw Error(MPEIG_E_CONFIG, "dense_chol: unknown precision");
    mpeig_op* op = new_op(ctx, kOpDenseChol, A->n);
    try {
      dense_chol_build(ctx, A, precision, op);
    } catch (...) {
      mpeig_op_destroy(op);
      throw;
    }
    *out = op;
  });
}

double mpeig_precond_shift(const mpeig_op* op) { return op ? op->shift : 0.0; }

int mpeig_precond_sparse_chol(mpeig_ctx* ctx, const mpeig_op* A, int32_t precision,
                              int32_t ordering, const int64_t* perm, mpeig_op** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (!A) throw Error(MPEIG_E_CONFIG, "sparse_chol: null operator");
    if (precision != MPEIG_WORKING && precision != MPEIG_LOWER)
      throw Error(MPEIG_E_CONFIG, "sparse_chol: unknown precision");
    mpeig_op* op = new_op(ctx, kOpSparseChol, A->n);
    try {
      sparse_chol_build(ctx, A, precision, ordering, perm, op);
    } catch (...) {
      mpeig_op_destroy(op);
      throw;
    }
    *out = op;
  });
}

int64_t mpeig_precond_factor_nnz(const mpeig_op* op) {
  if (!op) return 0;
  if (op->kind == kOpSparseChol) return op->sp_nnz;
  if (op->kind == kOpDenseChol) return op->n * (op->n + 1) / 2;
  return 0;
}

int mpeig_rcm_ordering(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, int64_t* perm_out) {
  try {
    const std::vector<int64_t> p = rcm_ordering(n, row_ptr, col_idx);
    std::copy(p.begin(), p.end(), perm_out);
    return MPEIG_OK;
  } catch (const std::exception&) {
    return MPEIG_E_OTHER;
  }
}

void mpeig_op_destroy(mpeig_op* op) {
  if (!op) return;
  if (op->ctx && op->ctx->stream) cudaStreamSynchronize(op->ctx->stream);
  cudaFree(op->rp);
  cudaFree(op->ci);
  cudaFree(op->rp32);
  cudaFree(op->ci32);
  cudaFree(op->dgw);
  cudaFree(op->dgl);
  cudaFree(op->vals);
  cudaFree(op->vals_l);
  cudaFree(op->A);
  cudaFree(op->Al);
  cudaFree(op->dinv);
  cudaFree(op->dinvf);
  cudaFree(op->Lw);
  cudaFree(op->Ll);
  cudaFree(op->scratch);
  cudaFree(op->sp_Lrp);
  cudaFree(op->sp_Lci);
  cudaFree(op->sp_Urp);
  cudaFree(op->sp_Uci);
  cudaFree(op->sp_perm);
  cudaFree(op->sp_Lsp);
  cudaFree(op->sp_Usp);
  cudaFree(op->sp_Lv);
  cudaFree(op->sp_Uv);
  cudaFree(op->gx_send_idx);
  cudaFree(op->rows_inner);
  cudaFree(op->rows_bnd);
  if (op->halo) cudaFree(op->halo);
  if (op->halo_stream) cudaStreamDestroy(op->halo_stream);
  if (op->ev_packed) cudaEventDestroy(op->ev_packed);
  if (op->ev_halo) cudaEventDestroy(op->ev_halo);
  delete op;
}

int64_t mpeig_op_n(const mpeig_op* op) { return op ? op->n : 0; }

int mpeig_op_apply(mpeig_ctx* ctx, const mpeig_op* op, int32_t precision, int64_t ncols,
                   const void* X, int64_t ldx, void* Y, int64_t ldy) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (precision == MPEIG_WORKING)
      op_apply<double>(ctx, op, ncols, static_cast<const double*>(X), ldx, static_cast<double*>(Y), ldy);
    else
      op_apply<float>(ctx, op, ncols, static_cast<const float*>(X), ldx, static_cast<float*>(Y), ldy);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------------------------ solvers
int mpeig_spectral_norm_estimate(mpeig_ctx* ctx, const mpeig_op* A, int64_t sketch_rows,
                                 uint64_t seed, double* out) {
  return guard(ctx, [&] {
    set_device(ctx);
    *out = spectral_norm_estimate(ctx, A, sketch_rows, seed);
  });
}

static void fill_stage_out(const StageResult& r, int64_t m, mpeig_stage_out* out) {
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  for (int64_t j = 0; j < m; ++j) {
    if (out->theta) out->theta[j] = r.theta[j];
    if (out->residual_norms) out->residual_norms[j] = r.resid[j];
  }
}

int mpeig_lobpcg_stage_f64(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0,
                           int64_t ldx0, int64_t m, const mpeig_cfg* cfg, const mpeig_op* T,
                           double a_norm_est, const mpeig_stage_opts* opt,
                           mpeig_history_sink sink, void* sink_user, mpeig_stage_out* out,
                           mpeig_timings* tim) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (A->n != n) throw Error(MPEIG_E_DIMENSION, "lobpcg_stage: X0 has wrong rows");
    const StageResult r = lobpcg_stage<double>(ctx, A, n, X0, ldx0, m, *cfg, T, a_norm_est, *opt, sink,
                                               sink_user, static_cast<double*>(out->X), out->ldx, tim);
    fill_stage_out(r, m, out);
  });
}

int mpeig_lobpcg_stage_f32(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const float* X0,
                           int64_t ldx0, int64_t m, const mpeig_cfg* cfg, const mpeig_op* T,
                           double a_norm_est, const mpeig_stage_opts* opt,
                           mpeig_history_sink sink, void* sink_user, mpeig_stage_out* out,
                           mpeig_timings* tim) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (A->n != n) throw Error(MPEIG_E_DIMENSION, "lobpcg_stage: X0 has wrong rows");
    const StageResult r = lobpcg_stage<float>(ctx, A, n, X0, ldx0, m, *cfg, T, a_norm_est, *opt, sink,
                                              sink_user, static_cast<float*>(out->X), out->ldx, tim);
    fill_stage_out(r, m, out);
  });
}

int mpeig_pinvit_f64(mpeig_ctx* ctx, const mpeig_op* A, int64_t n, const double* X0, int64_t ldx0,
                     int64_t m, const mpeig_cfg* cfg, const mpeig_op* T, double a_norm_est,
                     mpeig_history_sink sink, void* sink_user, mpeig_result* out) {
  return guard(ctx, [&] {
    set_device(ctx);
    validate_cfg(*cfg, n);
    if (m < cfg->k) throw Error(MPEIG_E_CONFIG, "pinvit: X0 has fewer columns than k");
    if (a_norm_est <= 0)
      a_norm_est = spectral_norm_estimate(ctx, A, cfg->sketch_rows, cfg->seed ^ 0x9e3779b97f4a7c15ULL);
    const int64_t ld = padded_ld(n);
    DevBuf<double> Xf(static_cast<size_t>(ld * m), ctx->stream);
    const StageResult r = pinvit(ctx, A, n, X0, ldx0, m, *cfg, T, a_norm_est, sink, sink_user, Xf.p,
                                 ld, &out->timings);
    out->a_norm_estimate = a_norm_est;
    out->iterations_lower = 0;
    out->iterations_working = r.iterations;
    out->converged = r.converged ? 1 : 0;
    for (int64_t j = 0; j < cfg->k; ++j) {
      if (out->theta) out->theta[j] = r.theta[j];
      if (out->residual_norms) out->residual_norms[j] = r.resid[j];
    }
    if (out->X) copy_block<double>(n, cfg->k, Xf.p, ld, out->X, out->ldx, ctx->stream);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_solve(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T, const mpeig_cfg* cfg,
                mpeig_history_sink sink, void* sink_user, mpeig_result* out) {
  return guard(ctx, [&] {
    set_device(ctx);
    out->timings = mpeig_timings{};
    solve(ctx, A, T, *cfg, sink, sink_user, out);
  });
}

int mpeig_solve_prepared(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T,
                         const mpeig_cfg* cfg, const double* X0raw, int64_t ldx0,
                         const double* omega, int64_t ldo, double omega_fro,
                         mpeig_history_sink sink, void* sink_user, mpeig_result* out) {
  return guard(ctx, [&] {
    set_device(ctx);
    out->timings = mpeig_timings{};
    solve_prepared(ctx, A, T, *cfg, X0raw, ldx0, omega, ldo, omega_fro, sink, sink_user, out);
  });
}

int mpeig_buffer_alloc(mpeig_ctx* ctx, int64_t bytes, void** out) {
  return guard(ctx, [&] {
    set_device(ctx);
    *out = nullptr;
    if (bytes > 0) MPB_CUDA(cudaMalloc(out, static_cast<size_t>(bytes)));
  });
}

void mpeig_buffer_free(mpeig_ctx* ctx, void* p) {
  if (!p) return;
  if (ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
  }
  cudaFree(p);
}

int mpeig_copy(mpeig_ctx* ctx, void* dst, const void* src, int64_t bytes) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (bytes <= 0) return;
    MPB_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault, ctx->stream));
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_solve_csr(mpeig_ctx* ctx, int64_t n, const int64_t* row_ptr_host,
                    const int64_t* col_idx_host, const double* vals_host, const mpeig_cfg* cfg,
                    mpeig_history_sink sink, void* sink_user, mpeig_result* out,
                    double* precond_shift) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (!cfg || !out || !row_ptr_host || n < 1) throw Error(MPEIG_E_CONFIG, "solve_csr: null argument");
    validate_cfg(*cfg, n);  // cfg.validate(n) first (drivers.hpp:185-186)
    // one RCM permutation of the system (drivers.hpp:187-188)
    const std::vector<int64_t> perm = rcm_ordering(n, row_ptr_host, col_idx_host);
    std::vector<int64_t> brp, bci;
    std::vector<double> bv;
    csr_permute<double>(n, row_ptr_host, col_idx_host, vals_host, perm, brp, bci, bv);
    auto rethrow = [&](int rc) {
      if (rc != MPEIG_OK) throw Error(rc, ctx->last_msg, ctx->last_index);
    };
    struct OpPtr {
      mpeig_op* p = nullptr;
      ~OpPtr() { mpeig_op_destroy(p); }
    } As, T;
    rethrow(mpeig_op_csr(ctx, n, brp.data(), bci.data(), bv.data(), &As.p));
    // the preconditioner on the permuted system, identity ordering (:190-192)
    const int32_t prec = cfg->variant == MPEIG_DLOBPCG_DCHOL ? MPEIG_WORKING : MPEIG_LOWER;
    const auto t0 = std::chrono::steady_clock::now();
    rethrow(mpeig_precond_sparse_chol(ctx, As.p, prec, 1, nullptr, &T.p));
    const double t_factor =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (precond_shift) *precond_shift = T.p->shift;
    out->timings = mpeig_timings{};
    solve(ctx, As.p, T.p, *cfg, sink, sink_user, out);
    out->timings.factorize = t_factor;
    if (out->X) {  // unpermute_rows (drivers.hpp:209): X(perm[i], :) = Xs(i, :)
      cudaStream_t s = ctx->stream;
      DevBuf<double> Xs(static_cast<size_t>(n * cfg->k), s);
      DevBuf<int64_t> dp(static_cast<size_t>(n), s);
      copy_block<double>(n, cfg->k, out->X, out->ldx, Xs.p, n, s);
      MPB_CUDA(cudaMemcpyAsync(dp.p, perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
      scatter_rows_f64(n, cfg->k, Xs.p, n, dp.p, out->X, out->ldx, s);
      MPB_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int mpeig_run_variant(mpeig_ctx* ctx, const mpeig_op* A, const mpeig_op* T, const mpeig_cfg* cfg,
                      const double* X0, int64_t ldx0, double a_norm_est, mpeig_history_sink sink,
                      void* sink_user, mpeig_result* out) {
  return guard(ctx, [&] {
    set_device(ctx);
    validate_cfg(*cfg, A->n);
    out->timings = mpeig_timings{};
    run_variant(ctx, A, T, *cfg, X0, ldx0, a_norm_est, sink, sink_user, out);
  });
}

// ----------------------------------------------------- kernel-level entries
int mpeig_gaussian_matrix_host(int64_t rows, int64_t cols, uint64_t seed, double* out_host) {
  return guard(nullptr, [&] { gaussian_fill(rows, cols, seed, out_host); });
}

int mpeig_gaussian_matrix_rows_host(int64_t n_global, int64_t cols, uint64_t seed, int64_t row0,
                                    int64_t rows, double* out_host) {
  return guard(nullptr, [&] {
    if (row0 < 0 || rows < 0 || row0 + rows > n_global) throw Error(MPEIG_E_CONFIG, "bad row range");
    gaussian_fill_rows(n_global, cols, seed, row0, rows, out_host);
  });
}

int mpeig_orthonormal_q_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                            int32_t use_mixed) {
  return guard(ctx, [&] {
    set_device(ctx);
    Work<double> w(ctx, n, m, m);
    orthonormal_q<double>(w, m, W, ldw, use_mixed != 0);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_orthonormal_q_f32(mpeig_ctx* ctx, int64_t n, int64_t m, float* W, int64_t ldw) {
  return guard(ctx, [&] {
    set_device(ctx);
    Work<float> w(ctx, n, m, m);
    orthonormal_q<float>(w, m, W, ldw, false);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

static int qr_entry(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw, double* R_out,
                    bool lower) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (n < m) throw Error(MPEIG_E_DIMENSION, "qr: more columns than rows");
    Work<double> w(ctx, n, m, m);
    int64_t idx = 0;
    DevBuf<double> R(static_cast<size_t>(m * m), ctx->stream);
    const int st = qr_with_r(w, m, W, ldw, lower, R.p, &idx);
    if (st != 0) throw Error(st, lower ? "mixed_qr failed" : "householder_qr failed", idx);
    if (R_out) MPB_CUDA(cudaMemcpyAsync(R_out, R.p, sizeof(double) * m * m, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_mixed_qr_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw, double* R_out) {
  return qr_entry(ctx, n, m, W, ldw, R_out, true);
}

int mpeig_householder_qr_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                             double* R_out) {
  return qr_entry(ctx, n, m, W, ldw, R_out, false);
}

int mpeig_orthonormal_q_dropping_f64(mpeig_ctx* ctx, int64_t n, int64_t m, double* W, int64_t ldw,
                                     int32_t use_mixed, int64_t* kept) {
  return guard(ctx, [&] {
    set_device(ctx);
    Work<double> w(ctx, n, m, m);
    int64_t dropped = 0;
    *kept = orthonormal_q_dropping<double>(w, m, W, ldw, use_mixed != 0, &dropped);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_gram_f64(mpeig_ctx* ctx, int64_t n, int64_t ka, const double* A, int64_t lda, int64_t kb,
                   const double* B, int64_t ldb, double* G) {
  return guard(ctx, [&] {
    set_device(ctx);
    DevBuf<double> wk;
    wk.alloc_zero(static_cast<size_t>(gram_workspace_elems<double>(n, ka, kb)), ctx->stream);
    gram<double>(n, ka, A, lda, kb, B, ldb, G, ka, 0, wk.p, ctx->stream);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_gemm_f64(mpeig_ctx* ctx, int64_t n, int64_t k, int64_t c, double alpha, const double* A,
                   int64_t lda, const double* Cm, int64_t ldc, double beta, const double* Z,
                   int64_t ldz, double* Y, int64_t ldy) {
  return guard(ctx, [&] {
    set_device(ctx);
    gemm_tn<double>(n, k, c, alpha, A, lda, Cm, ldc, beta, Z, ldz, Y, ldy, ctx->stream);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_set_process_option(const char* key, int value) {
  const std::string k = key ? key : "";
  if (k == "gram_tma") { g_gram_tma = value; return MPEIG_OK; }
  if (k == "pdl") { g_pdl = value; return MPEIG_OK; }
  if (k == "spchol_threads") { g_spchol_threads = value; return MPEIG_OK; }
  if (k == "gemm_tma2") { g_gemm_tma2 = value; return MPEIG_OK; }
  if (k == "tc_twoacc") { g_tc_twoacc = value; return MPEIG_OK; }
  if (k == "tc_ablate") { g_tc_ablate = value; return MPEIG_OK; }
  if (k == "g2_depth") { g_g2_depth = value; return MPEIG_OK; }
  if (k == "tc_stage") { g_tc_stage = value; return MPEIG_OK; }
  if (k == "tc_nprod") { g_tc_nprod = value; return MPEIG_OK; }
  if (k == "tc_store") { g_tc_store = value; return MPEIG_OK; }
  if (k == "gram_tc" || k == "gemm_tc" || k == "tc") {
    if (value < 0 || value > 2) return MPEIG_E_CONFIG;
    if (k != "gemm_tc") g_gram_tc = value;
    if (k != "gram_tc") g_gemm_tc = value;
    return MPEIG_OK;
  }
  return MPEIG_E_CONFIG;
}

int mpeig_gram_f32(mpeig_ctx* ctx, int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb,
                   const float* B, int64_t ldb, float* G) {
  return guard(ctx, [&] {
    set_device(ctx);
    DevBuf<float> wk;
    wk.alloc_zero(static_cast<size_t>(gram_workspace_elems<float>(n, ka, kb)), ctx->stream);
    gram<float>(n, ka, A, lda, kb, B, ldb, G, ka, 0, wk.p, ctx->stream);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_gemm_f32(mpeig_ctx* ctx, int64_t n, int64_t k, int64_t c, float alpha, const float* A,
                   int64_t lda, const float* Cm, int64_t ldc, float beta, const float* Z,
                   int64_t ldz, float* Y, int64_t ldy) {
  return guard(ctx, [&] {
    set_device(ctx);
    gemm_tn<float>(n, k, c, alpha, A, lda, Cm, ldc, beta, Z, ldz, Y, ldy, ctx->stream);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_project_out_f64(mpeig_ctx* ctx, int64_t n, int64_t b, const double* B, int64_t ldb,
                          int64_t wc, double* W, int64_t ldw, int32_t passes) {
  return guard(ctx, [&] {
    set_device(ctx);
    Work<double> w(ctx, n, std::max(b, wc), std::max(b, wc));
    project_out<double>(w, B, b, ldb, W, wc, ldw, passes);
    MPB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mpeig_small_eig_f64(mpeig_ctx* ctx, int64_t s, const double* M, double* values,
                        double* vectors) {
  return guard(ctx, [&] {
    set_device(ctx);
    Work<double> w(ctx, 3 * s, s, s);
    MPB_CUDA(cudaMemcpyAsync(vectors, M, sizeof(double) * s * s, cudaMemcpyDeviceToDevice, ctx->stream));
    status_clear(ctx);
    small_eig<double>(w, s, vectors, s, values);
    status_fetch(ctx);
    if (ctx->h_status[3] > 0) throw Error(MPEIG_E_NO_CONVERGENCE, "small_herm_eig: syevd did not converge");
  });
}

int mpeig_hl_coeffs_f64(mpeig_ctx* ctx, int64_t s, int64_t m, const double* C, double* coef,
                        int64_t* p, int32_t* fallback) {
  return guard(ctx, [&] {
    set_device(ctx);
    if (s < m) throw Error(MPEIG_E_DIMENSION, "hl_update: fewer columns than m");
    const int64_t pn = std::min(m, s - m);
    DevBuf<double> scratch(static_cast<size_t>(pn * m + 2 * pn * pn + pn + 1), ctx->stream);
    status_clear(ctx);
    hl_coeffs(s, m, pn, C, s, coef, scratch.p, ctx->d_status + 4, ctx->stream);
    status_fetch(ctx);
    *p = pn;
    *fallback = ctx->h_status[4];
  });
}

int mpeig_residual_precond_f64(mpeig_ctx* ctx, const mpeig_op* T, int64_t n, int64_t m,
                               const double* X, int64_t ldx, const double* AX, int64_t ldax,
                               const double* theta_host, double* W, int64_t ldw, double* rnorm_host,
                               double* xnorm_host) {
  return guard(ctx, [&] {
    set_device(ctx);
    cudaStream_t s = ctx->stream;
    DevBuf<double> th(static_cast<size_t>(m), s);
    DevBuf<double> wk(static_cast<size_t>(resid_workspace_elems(n, m) + 2 * m), s);
    MPB_CUDA(cudaMemcpyAsync(th.p, theta_host, sizeof(double) * m, cudaMemcpyHostToDevice, s));
    const void* dinv = nullptr;
    int mode = kResidPlain;
    if (T) {
      if (T->kind != kOpJacobi) throw Error(MPEIG_E_CONFIG, "residual_precond: T must be Jacobi");
      if (T->precision == MPEIG_WORKING) {
        mode = kResidJacobiT;
        dinv = T->dinv;
      } else {
        mode = kResidSandwich;
        dinv = T->dinvf;
      }
    }
    status_clear(ctx);
    double* norms = wk.p + resid_workspace_elems(n, m);
    residual_precond<double>(mode, n, m, X, ldx, AX, ldax, th.p, dinv, W, ldw, norms, norms + m,
                             ctx->d_status + 2, wk.p, s);
    std::vector<double> h(static_cast<size_t>(2 * m));
    MPB_CUDA(cudaMemcpyAsync(h.data(), norms, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost, s));
    status_fetch(ctx);
    for (int64_t j = 0; j < m; ++j) {
      rnorm_host[j] = h[j];
      xnorm_host[j] = h[m + j];
    }
    if (ctx->h_status[2]) throw Error(MPEIG_E_OVERFLOW, "to_lower: value exceeds binary32 range");
  });
}

}  // extern "C"
