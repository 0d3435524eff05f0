// comm.cpp -- host-staged and NCCL transports for the row-sharded solver.
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace mpb {

// ------------------------------------------------------------ host group
void HostGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const uint64_t gen = generation;
  if (++arrived == nranks) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

template <typename T, typename Op>
void HostComm::reduce(T* d, int64_t count, cudaStream_t s, Op op) {
  const size_t bytes = sizeof(T) * static_cast<size_t>(count);
  auto& mine = group->slots[rank];
  mine.resize(bytes);
  MPB_CUDA(cudaMemcpyAsync(mine.data(), d, bytes, cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  group->barrier();
  // every rank combines the slots in rank order: identical bits everywhere
  std::vector<T> acc(static_cast<size_t>(count));
  std::memcpy(acc.data(), group->slots[0].data(), bytes);
  for (int r = 1; r < nranks; ++r) {
    const T* v = reinterpret_cast<const T*>(group->slots[r].data());
    for (int64_t i = 0; i < count; ++i) acc[i] = op(acc[i], v[i]);
  }
  group->barrier();  // all reads done before any slot is reused
  MPB_CUDA(cudaMemcpyAsync(d, acc.data(), bytes, cudaMemcpyHostToDevice, s));
  MPB_CUDA(cudaStreamSynchronize(s));
}

void HostComm::allreduce_sum(double* d, int64_t count, cudaStream_t s) {
  reduce(d, count, s, [](double a, double b) { return a + b; });
}
void HostComm::allreduce_sum(float* d, int64_t count, cudaStream_t s) {
  reduce(d, count, s, [](float a, float b) { return a + b; });
}
void HostComm::allreduce_max(int* d, int64_t count, cudaStream_t s) {
  reduce(d, count, s, [](int a, int b) { return a > b ? a : b; });
}

void HostComm::allgather(const void* send, void* recv, int64_t bytes, cudaStream_t s) {
  auto& mine = group->slots[rank];
  mine.resize(static_cast<size_t>(bytes));
  MPB_CUDA(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  group->barrier();
  std::vector<char> all(static_cast<size_t>(bytes) * nranks);
  for (int r = 0; r < nranks; ++r)
    std::memcpy(all.data() + static_cast<size_t>(bytes) * r, group->slots[r].data(), bytes);
  group->barrier();
  MPB_CUDA(cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, s));
  MPB_CUDA(cudaStreamSynchronize(s));
}

void HostComm::exchange(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi,
                        int64_t bytes, cudaStream_t s) {
  auto& lo = group->slots[rank];
  auto& hi = group->slots2[rank];
  lo.resize(static_cast<size_t>(bytes));
  hi.resize(static_cast<size_t>(bytes));
  if (rank > 0) MPB_CUDA(cudaMemcpyAsync(lo.data(), send_lo, bytes, cudaMemcpyDeviceToHost, s));
  if (rank + 1 < nranks)
    MPB_CUDA(cudaMemcpyAsync(hi.data(), send_hi, bytes, cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  group->barrier();
  std::vector<char> a, b;
  if (rank > 0) a = group->slots2[rank - 1];          // rank-1's upper plane
  if (rank + 1 < nranks) b = group->slots[rank + 1];  // rank+1's lower plane
  group->barrier();
  if (rank > 0) MPB_CUDA(cudaMemcpyAsync(recv_lo, a.data(), bytes, cudaMemcpyHostToDevice, s));
  if (rank + 1 < nranks)
    MPB_CUDA(cudaMemcpyAsync(recv_hi, b.data(), bytes, cudaMemcpyHostToDevice, s));
  MPB_CUDA(cudaStreamSynchronize(s));
}

void HostComm::alltoallv(const void* send, const int64_t* send_bytes, const int64_t* send_off,
                         void* recv, const int64_t* recv_bytes, const int64_t* recv_off,
                         cudaStream_t s) {
  // slots[r]: rank r's whole send buffer; slots2[r]: its (offset, bytes) table
  int64_t extent = 0;
  for (int q = 0; q < nranks; ++q)
    if (send_bytes[q] > 0) extent = std::max(extent, send_off[q] + send_bytes[q]);
  auto& mine = group->slots[rank];
  auto& table = group->slots2[rank];
  mine.resize(static_cast<size_t>(extent));
  table.resize(sizeof(int64_t) * 2 * nranks);
  int64_t* t = reinterpret_cast<int64_t*>(table.data());
  for (int q = 0; q < nranks; ++q) {
    t[q] = send_off[q];
    t[nranks + q] = send_bytes[q];
  }
  if (extent > 0) MPB_CUDA(cudaMemcpyAsync(mine.data(), send, extent, cudaMemcpyDeviceToHost, s));
  MPB_CUDA(cudaStreamSynchronize(s));
  group->barrier();
  for (int q = 0; q < nranks; ++q) {
    if (recv_bytes[q] <= 0) continue;
    const int64_t* tq = reinterpret_cast<const int64_t*>(group->slots2[q].data());
    if (tq[nranks + rank] != recv_bytes[q]) throw Error(MPEIG_E_COMM, "alltoallv: size mismatch");
    MPB_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + recv_off[q], group->slots[q].data() + tq[rank],
                             recv_bytes[q], cudaMemcpyHostToDevice, s));
  }
  MPB_CUDA(cudaStreamSynchronize(s));
  group->barrier();  // all reads done before any slot is reused
}

// ------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};

const NcclApi& api() {
  static NcclApi a = [] {
    NcclApi r;
    // prefer the NCCL already in the process (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
#define MPB_SYM(field, name) r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, name))
    MPB_SYM(get_unique_id, "ncclGetUniqueId");
    MPB_SYM(init_rank, "ncclCommInitRank");
    MPB_SYM(destroy, "ncclCommDestroy");
    MPB_SYM(allreduce, "ncclAllReduce");
    MPB_SYM(allgather, "ncclAllGather");
    MPB_SYM(send, "ncclSend");
    MPB_SYM(recv, "ncclRecv");
    MPB_SYM(group_start, "ncclGroupStart");
    MPB_SYM(group_end, "ncclGroupEnd");
    MPB_SYM(errstr, "ncclGetErrorString");
#undef MPB_SYM
    r.ok = r.get_unique_id && r.init_rank && r.destroy && r.allreduce && r.allgather && r.send &&
           r.recv && r.group_start && r.group_end;
    return r;
  }();
  return a;
}

void nccl_check(ncclResult_t rc, const char* what) {
  if (rc != ncclSuccess) {
    const char* m = api().errstr ? api().errstr(rc) : "";
    throw Error(MPEIG_E_COMM, std::string(what) + " failed: " + m);
  }
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  ~NcclComm() override {
    if (comm) api().destroy(comm);
  }
  void allreduce_sum(double* d, int64_t count, cudaStream_t s) override {
    nccl_check(api().allreduce(d, d, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, s),
               "ncclAllReduce");
  }
  void allreduce_sum(float* d, int64_t count, cudaStream_t s) override {
    nccl_check(api().allreduce(d, d, static_cast<size_t>(count), ncclFloat32, ncclSum, comm, s),
               "ncclAllReduce");
  }
  void allreduce_max(int* d, int64_t count, cudaStream_t s) override {
    nccl_check(api().allreduce(d, d, static_cast<size_t>(count), ncclInt32, ncclMax, comm, s),
               "ncclAllReduce");
  }
  void allgather(const void* send, void* recv, int64_t bytes, cudaStream_t s) override {
    nccl_check(api().allgather(send, recv, static_cast<size_t>(bytes), ncclUint8, comm, s),
               "ncclAllGather");
  }
  void exchange(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi,
                int64_t bytes, cudaStream_t s) override {
    const size_t b = static_cast<size_t>(bytes);
    nccl_check(api().group_start(), "ncclGroupStart");
    if (rank > 0) {
      nccl_check(api().send(send_lo, b, ncclUint8, rank - 1, comm, s), "ncclSend");
      nccl_check(api().recv(recv_lo, b, ncclUint8, rank - 1, comm, s), "ncclRecv");
    }
    if (rank + 1 < nranks) {
      nccl_check(api().send(send_hi, b, ncclUint8, rank + 1, comm, s), "ncclSend");
      nccl_check(api().recv(recv_hi, b, ncclUint8, rank + 1, comm, s), "ncclRecv");
    }
    nccl_check(api().group_end(), "ncclGroupEnd");
  }
  void alltoallv(const void* send, const int64_t* send_bytes, const int64_t* send_off, void* recv,
                 const int64_t* recv_bytes, const int64_t* recv_off, cudaStream_t s) override {
    nccl_check(api().group_start(), "ncclGroupStart");
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) continue;
      if (send_bytes[q] > 0)
        nccl_check(api().send(static_cast<const char*>(send) + send_off[q],
                              static_cast<size_t>(send_bytes[q]), ncclUint8, q, comm, s),
                   "ncclSend");
      if (recv_bytes[q] > 0)
        nccl_check(api().recv(static_cast<char*>(recv) + recv_off[q], static_cast<size_t>(recv_bytes[q]),
                              ncclUint8, q, comm, s),
                   "ncclRecv");
    }
    nccl_check(api().group_end(), "ncclGroupEnd");
  }
};

}  // namespace

bool nccl_available() { return api().ok; }

void nccl_unique_id(void* out128) {
  if (!api().ok) throw Error(MPEIG_E_COMM, "libnccl.so.2 not available");
  ncclUniqueId id;
  nccl_check(api().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
}

Comm* make_nccl_comm(int rank, int nranks, const void* id128) {
  if (!api().ok) throw Error(MPEIG_E_COMM, "libnccl.so.2 not available");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* c = new NcclComm;
  c->rank = rank;
  c->nranks = nranks;
  try {
    nccl_check(api().init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

}  // namespace mpb
