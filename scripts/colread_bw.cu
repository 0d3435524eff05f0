// Read bandwidth of a tall column-major block when each CTA streams a row
// chunk of ALL its columns, KC rows per column per step (the Gram / GEMM
// access pattern).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 colread_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KC>
__global__ void k_read(const float* __restrict__ A, long n, long ld, int ncol, long rows_per_cta,
                       float* out) {
  const long r0 = blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
  float acc = 0.f;
  constexpr int V = KC / 4;  // float4 per column per step
  for (long r = r0; r < r1; r += KC) {
    for (int e = threadIdx.x; e < ncol * V; e += blockDim.x) {
      const int c = e / V, v = e % V;
      const float4 x = __ldg(reinterpret_cast<const float4*>(A + c * ld + r) + v);
      acc += x.x + x.y + x.z + x.w;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const long n = 1L << 21;
  const int maxc = 256;
  float* A;
  cudaMalloc(&A, sizeof(float) * n * maxc);
  cudaMemset(A, 0, sizeof(float) * n * maxc);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ncol : {96, 256}) {
    for (int ctas : {148, 296, 592}) {
      auto run = [&](auto kc_tag) {
        constexpr int KC = decltype(kc_tag)::value;
        const long rpc = ((n + ctas - 1) / ctas + KC - 1) / KC * KC;
        k_read<KC><<<ctas, 256>>>(A, n, n, ncol, rpc, out);
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) k_read<KC><<<ctas, 256>>>(A, n, n, ncol, rpc, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("ncol %3d ctas %3d KC %4d: %.3f ms  %.0f GB/s\n", ncol, ctas, KC, ms,
               4.0 * n * ncol / (ms * 1e6));
      };
      run(std::integral_constant<int, 32>());
      run(std::integral_constant<int, 128>());
      run(std::integral_constant<int, 512>());
    }
  }
  return 0;
}
