// prof.cpp -- CUDA-event timing per kernel class (used by bench.py's roofline).
#include <map>
#include <mutex>
#include <set>
#include <utility>
#include <string>
#include <vector>

#include "common.cuh"

namespace mpb {

bool g_prof_on = false;

namespace {

struct Entry {
  std::vector<cudaEvent_t> start, stop;
  double bytes = 0, flops = 0;
  int64_t count = 0;
};

std::mutex g_mu;
std::map<std::string, Entry>& table() {
  static std::map<std::string, Entry> t;
  return t;
}

}  // namespace

void smem_opt_in(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  MPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert({kernel, dev}).second) return;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bytes));
  if (e != cudaSuccess) {
    done.erase({kernel, dev});
    MPB_CUDA(e);
  }
}

void prof_begin(const char* name, cudaStream_t s, double bytes, double flops) {
  std::lock_guard<std::mutex> lk(g_mu);
  Entry& e = table()[name];
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, s);
  e.start.push_back(ev);
  e.bytes += bytes;
  e.flops += flops;
  e.count += 1;
}

void prof_end(const char* name, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  Entry& e = table()[name];
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, s);
  e.stop.push_back(ev);
}

}  // namespace mpb

extern "C" {

void mpeig_profile_enable(int on) { mpb::g_prof_on = on != 0; }

void mpeig_profile_reset(void) {
  std::lock_guard<std::mutex> lk(mpb::g_mu);
  for (auto& kv : mpb::table()) {
    for (auto ev : kv.second.start) cudaEventDestroy(ev);
    for (auto ev : kv.second.stop) cudaEventDestroy(ev);
  }
  mpb::table().clear();
}

// Newline-separated kernel-class names into buf; returns the count.
int mpeig_profile_names(char* buf, int64_t cap) {
  std::lock_guard<std::mutex> lk(mpb::g_mu);
  std::string all;
  for (auto& kv : mpb::table()) all += kv.first + "\n";
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(all.size(), static_cast<size_t>(cap - 1));
    all.copy(buf, n);
    buf[n] = 0;
  }
  return static_cast<int>(mpb::table().size());
}

// Totals for one kernel class; synchronises on its events.
int mpeig_profile_query(const char* name, int64_t* count, double* ms, double* bytes,
                        double* flops) {
  std::lock_guard<std::mutex> lk(mpb::g_mu);
  auto it = mpb::table().find(name);
  if (it == mpb::table().end()) return 1;
  mpb::Entry& e = it->second;
  double tot = 0;
  for (size_t i = 0; i < e.start.size() && i < e.stop.size(); ++i) {
    cudaEventSynchronize(e.stop[i]);
    float t = 0;
    cudaEventElapsedTime(&t, e.start[i], e.stop[i]);
    tot += t;
  }
  *count = e.count;
  *ms = tot;
  *bytes = e.bytes;
  *flops = e.flops;
  return 0;
}


}  // extern "C"
