// comm.hpp -- the row-sharded (multi-GPU) exchange steps of the solver.
//
// every n x . block is row-sharded (z-slabs of the stencil);
// the only cross-rank data per iteration are the small Gram matrices and
// column norms (sum-allreduce), the per-rank TSQR factors (allgather), the
// stencil halo planes (neighbour exchange) and the status words (max).  The
// Rayleigh-Ritz eigensolver and every small factorisation then run
// replicated on identical inputs, so all ranks take the same decisions.
//
// Two transports:
//  * NcclComm: NCCL over NVLink / NVSwitch (one process per GPU), libnccl
//    resolved at run time (the process's already-loaded NCCL, e.g. torch's).
//  * HostComm: ranks as threads of one process with host-staged sums in rank
//    order -- the transport of the multi-rank CPU-orchestrated tests.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

namespace mpb {

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() = default;
  // in-place, stream-ordered (may synchronise the stream)
  virtual void allreduce_sum(double* d, int64_t count, cudaStream_t s) = 0;
  virtual void allreduce_sum(float* d, int64_t count, cudaStream_t s) = 0;
  virtual void allreduce_max(int* d, int64_t count, cudaStream_t s) = 0;
  // recv = concat over ranks of send (bytes each), rank order
  virtual void allgather(const void* send, void* recv, int64_t bytes, cudaStream_t s) = 0;
  // slab neighbours: send_lo goes to rank-1 (arrives in its recv_hi), send_hi
  // to rank+1 (its recv_lo); a missing neighbour sends / receives nothing
  virtual void exchange(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi,
                        int64_t bytes, cudaStream_t s) = 0;
  // point-to-point to any peers (the CSR ghost rows): send_bytes[q] bytes at
  // send + send_off[q] go to rank q, which receives them at recv + recv_off[me];
  // sizes agreed beforehand (recv_bytes[q] == rank q's send_bytes[me])
  virtual void alltoallv(const void* send, const int64_t* send_bytes, const int64_t* send_off,
                         void* recv, const int64_t* recv_bytes, const int64_t* recv_off,
                         cudaStream_t s) = 0;
  // every exchange is stream-ordered without host synchronisation (NCCL), so
  // an iteration body containing them can be captured into a CUDA graph
  virtual bool capturable() const { return false; }
};

// ---- ranks as threads of one process ------------------------------------
struct HostGroup {
  explicit HostGroup(int n) : nranks(n), slots(n), slots2(n) {}
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<char>> slots, slots2;
  void barrier();
};

struct HostComm final : Comm {
  explicit HostComm(HostGroup* g, int r) : group(g) {
    rank = r;
    nranks = g->nranks;
  }
  HostGroup* group;
  void allreduce_sum(double* d, int64_t count, cudaStream_t s) override;
  void allreduce_sum(float* d, int64_t count, cudaStream_t s) override;
  void allreduce_max(int* d, int64_t count, cudaStream_t s) override;
  void allgather(const void* send, void* recv, int64_t bytes, cudaStream_t s) override;
  void exchange(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi,
                int64_t bytes, cudaStream_t s) override;
  void alltoallv(const void* send, const int64_t* send_bytes, const int64_t* send_off, void* recv,
                 const int64_t* recv_bytes, const int64_t* recv_off, cudaStream_t s) override;

 private:
  template <typename T, typename Op>
  void reduce(T* d, int64_t count, cudaStream_t s, Op op);
};

// ---- NCCL ------------------------------------------------------------------
bool nccl_available();
void nccl_unique_id(void* out128);
Comm* make_nccl_comm(int rank, int nranks, const void* id128);

}  // namespace mpb
