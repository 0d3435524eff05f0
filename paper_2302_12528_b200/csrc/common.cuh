// common.cuh -- shared definitions for the sm_100a LOBPCG hot path.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "mpeig_b200.h"

namespace mpb {

// Exception carrying an mpeig_status code (1:1 with the reference's
// errors.hpp types, see include/mpeig_b200.h) and an optional index payload.
struct Error : std::runtime_error {
  int code;
  int64_t index;
  Error(int c, const std::string& m, int64_t idx = -1)
      : std::runtime_error(m), code(c), index(idx) {}
};

#define MPB_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      throw ::mpb::Error(MPEIG_E_CUDA, std::string(#call) + ": " +              \
                                           cudaGetErrorString(e_));             \
  } while (0)

// Dynamic shared memory above 48 KB needs a per-function opt-in, which is
// per device context: set it once per (kernel, current device); thread-safe.
void smem_opt_in(const void* kernel, size_t bytes);

// Kernels launched by this library (reported as gpu_launches by bench.py).
extern std::atomic<int64_t> g_launches;

// Programmatic dependent launch: every kernel waits here for the grids it
// depends on (complete, memory visible) before touching global memory, so a
// captured iteration graph may launch it early (programmatic edges, solver.cpp);
// a no-op for an ordinary launch
#define MPB_PDL_WAIT() asm volatile("griddepcontrol.wait;\n" ::: "memory")

#define MPB_LAUNCH_CHECK()                      \
  do {                                          \
    ::mpb::g_launches.fetch_add(1, std::memory_order_relaxed); \
    MPB_CUDA(cudaGetLastError());               \
  } while (0)

// Per-kernel-class device timing (bench.py roofline): when enabled, every
// launcher brackets its kernel(s) with CUDA events on the launching stream and
// records the algorithmic bytes / flops of that launch.
void prof_begin(const char* name, cudaStream_t s, double bytes, double flops);
void prof_end(const char* name, cudaStream_t s);
extern bool g_prof_on;
struct ProfScope {
  const char* name;
  cudaStream_t s;
  ProfScope(const char* n, cudaStream_t st, double bytes, double flops) : name(n), s(st) {
    if (g_prof_on) prof_begin(n, st, bytes, flops);
  }
  ~ProfScope() {
    if (g_prof_on) prof_end(name, s);
  }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

constexpr int kNumSMs = 148;  // B200

// Leading dimension of every device block vector: rows padded to 32
// elements (256 B for fp64) so every column starts 256-B aligned.
inline int64_t padded_ld(int64_t n) { return round_up(n, 32); }

}  // namespace mpb
