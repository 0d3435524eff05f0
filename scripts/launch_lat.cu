// launch_lat.cu -- per-kernel cost of back-to-back dependent launches in a CUDA graph
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/launch_lat.cu -o build/launch_lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(double* x, int iters) {
  double v = x[threadIdx.x];
  for (int i = 0; i < iters; ++i) v = v * 0.999 + 0.001;
  x[threadIdx.x] = v;
}
__global__ void k_wide(double* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.5 + 1.0;
}

int main() {
  double* x;
  cudaMalloc(&x, 1 << 24);
  cudaMemset(x, 0, 1 << 24);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int kind = 0; kind < 3; ++kind) {
    const int N = 100;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      if (kind == 0) k_tiny<<<1, 32, 0, s>>>(x, 1);
      if (kind == 1) k_tiny<<<1, 32, 0, s>>>(x, 1000);
      if (kind == 2) k_wide<<<1024, 256, 0, s>>>(x, 1 << 18);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("kind %d (%s): %.2f us per kernel in a graph\n", kind,
           kind == 0 ? "1 warp, trivial" : kind == 1 ? "1 warp, 1000 dependent DFMA" : "1024x256 elementwise 2 MB",
           ms * 1000 / (10 * N));
    // plain stream launches
    cudaEventRecord(a, s);
    for (int r = 0; r < 10 * N; ++r) {
      if (kind == 0) k_tiny<<<1, 32, 0, s>>>(x, 1);
      if (kind == 1) k_tiny<<<1, 32, 0, s>>>(x, 1000);
      if (kind == 2) k_wide<<<1024, 256, 0, s>>>(x, 1 << 18);
    }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("kind %d: %.2f us per kernel, stream launches\n", kind, ms * 1000 / (10 * N));
  }
  return 0;
}
