// gram_chol_bench.cu -- CholQR building blocks at cfg1 shapes: Gram alone,
// Gram + fused Cholesky / L^-T epilogue, the GEMM that applies it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2302_12528_b200/csrc \
//        scripts/gram_chol_bench.cu -L paper_2302_12528_b200 -lmpeig_b200 -o build/gram_chol_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

using namespace mpb;

template <typename F>
static double time_us(F f, int reps, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1e3 * ms / reps;
}

template <typename T>
static void run(int64_t n, int64_t m, cudaStream_t s) {
  T *W, *G, *L, *U, *Y, *work;
  int* st;
  cudaMalloc(&W, n * m * sizeof(T));
  cudaMalloc(&Y, n * m * sizeof(T));
  std::vector<T> h(n * m);
  for (int64_t i = 0; i < n * m; ++i) h[i] = T(((i * 2654435761ULL) % 1000003) * 1e-6 - 0.5);
  cudaMemcpy(W, h.data(), n * m * sizeof(T), cudaMemcpyHostToDevice);
  cudaMalloc(&G, m * m * sizeof(T));
  cudaMalloc(&L, m * m * sizeof(T));
  cudaMalloc(&U, m * m * sizeof(T));
  const int64_t gw = gram_workspace_elems<T>(n, m, m);
  cudaMalloc(&work, gw * sizeof(T) + 64);
  cudaMemset(work, 0, gw * sizeof(T) + 64);
  cudaMalloc(&st, 64);
  cudaMemset(st, 0, 64);
  const double tg = time_us([&] { gram<T>(n, m, W, n, m, W, n, G, m, 1, work, s); }, 100, s);
  const double tc = time_us([&] { gram_cholesky<T>(n, m, W, n, G, work, L, U, st, s); }, 100, s);
  const double tl = time_us([&] { small_cholesky_inv<T>(m, G, m, L, U, st, s); }, 100, s);
  const double tm = time_us([&] { gemm_tn<T>(n, m, m, T(1), W, n, U, m, T(0), nullptr, 0, Y, n, s); }, 100, s);
  int hs[2];
  cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost);
  printf("%s n=%ld m=%ld  gram %7.2f us  gram+chol %7.2f us  chol alone %7.2f us  gemm %7.2f us  status %d\n",
         sizeof(T) == 8 ? "f64" : "f32", (long)n, (long)m, tg, tc, tl, tm, hs[0]);
  cudaFree(W); cudaFree(Y); cudaFree(G); cudaFree(L); cudaFree(U); cudaFree(work); cudaFree(st);
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int64_t n : {32768L, 262144L, 1048576L}) {
    run<double>(n, 16, s);
    run<float>(n, 16, s);
  }
  return 0;
}
