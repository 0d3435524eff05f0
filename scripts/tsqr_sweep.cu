// tsqr_sweep.cu -- TSQR latency vs rows (tree depth) at fixed width.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2302_12528_b200/csrc \
//        scripts/tsqr_sweep.cu -L paper_2302_12528_b200 -lmpeig_b200 -o build/tsqr_sweep
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

using namespace mpb;

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

template <typename F>
static double time_us(F f, int reps, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaStreamSynchronize(s));
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b, s);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1e3 * ms / reps;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 16;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  const int64_t nmax = 1 << 20;
  double* W;
  CK(cudaMalloc(&W, nmax * m * 8));
  std::vector<double> h(nmax);
  for (int j = 0; j < m; ++j) {
    for (int64_t i = 0; i < nmax; ++i) h[i] = ((i * (j + 3) * 2654435761ULL) % 1000003) * 1e-6 - 0.5;
    CK(cudaMemcpy(W + j * nmax, h.data(), nmax * 8, cudaMemcpyHostToDevice));
  }
  int* st;
  CK(cudaMalloc(&st, 64));
  CK(cudaMemset(st, 0, 64));
  double *R, *Rw, *Ri;
  CK(cudaMalloc(&R, m * m * 8));
  CK(cudaMalloc(&Rw, m * m * 8));
  CK(cudaMalloc(&Ri, m * m * 8));
  for (int64_t n : {256L, 2048L, 4096L, 8192L, 32768L, 65536L, 262144L, 1048576L}) {
    const int64_t w64 = tsqr_workspace_elems<double, double>(n, m);
    const int64_t w32 = tsqr_workspace_elems<double, float>(n, m);
    double* tw;
    float* tf;
    CK(cudaMalloc(&tw, w64 * 8 + 64));
    CK(cudaMemset(tw, 0, w64 * 8 + 64));
    CK(cudaMalloc(&tf, w32 * 4 + 64));
    CK(cudaMemset(tf, 0, w32 * 4 + 64));
    const double t64 = time_us([&] { tsqr_r<double, double>(n, m, W, nmax, R, m, tw, st, s); }, 50, s);
    const double t32 = time_us(
        [&] { tsqr_r<double, float>(n, m, W, nmax, reinterpret_cast<float*>(R), m, tf, st, s); }, 50, s);
    const double t64e = time_us(
        [&] { tsqr_r<double, double>(n, m, W, nmax, R, m, tw, st, s, Rw, Ri); }, 50, s);
    printf("m=%d n=%8ld  fp64 %8.2f us  fp32(R) %8.2f us  fp64+Rinv %8.2f us\n", m, (long)n, t64, t32, t64e);
    CK(cudaFree(tw));
    CK(cudaFree(tf));
  }
  int hs[2];
  CK(cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost));
  printf("status %d %d\n", hs[0], hs[1]);
  return 0;
}
