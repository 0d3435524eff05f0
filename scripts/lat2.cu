// lat2.cu -- latencies of the primitives on the small kernels' serial chains:
// dependent shared-memory load, warp shuffle (32 / 64-bit), xor-tree warp sum
// (fp64), CTA barrier (256 / 512 threads), and a barrier round trip with a
// shared-memory handoff between two warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/lat2.cu -o build/lat2
#include <cstdio>

__global__ void k_lat(long long* out, int iters) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 1024; i += blockDim.x) {
    sm[i] = 1.0 + i * 1e-9;
    si[i] = (i + 1) & 1023;
  }
  __syncthreads();
  long long t0, t1;
  // 1. dependent LDS chain (int pointer chase)
  int p = tid & 31;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = si[p];
  t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / iters;
  // 2. dependent shfl (32-bit)
  int v = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / iters;
  // 3. dependent shfl of a double
  double dv = lane * 1.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) dv = __shfl_xor_sync(0xffffffffu, dv, 1) + 1e-30;
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / iters;
  // 4. fp64 xor-tree warp sum
  double acc = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    acc *= 1e-3;
  }
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0) / iters;
  // 5. __syncthreads alone
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0) / iters;
  // 6. handoff: warp (i % nw) writes, barrier, everyone reads
  const int nw = blockDim.x >> 5;
  double x = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if ((tid >> 5) == (i % nw) && lane == 0) sm[i & 1] = x + 1.0;
    __syncthreads();
    x = sm[i & 1];
  }
  t1 = clock64();
  if (tid == 0) out[5] = (t1 - t0) / iters;
  // 7. dependent LDS of a double + DFMA
  double y = 1.0;
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    y = fma(y, sm[idx], 1e-9);
    idx = (idx + (y > 5.0 ? 1 : 0)) & 1023;
  }
  t1 = clock64();
  if (tid == 0) out[6] = (t1 - t0) / iters;
  // 8. sqrt + div chain (double)
  double z = 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) z = 2.0 / sqrt(z + 1.0) + 1.0;
  t1 = clock64();
  if (tid == 0) out[7] = (t1 - t0) / iters;
  if (p == -1 || v == -1 || dv == -1 || acc == -1 || x == -1 || y == -1 || z == -1) out[9] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  long long h[16];
  for (int nt : {32, 256, 512}) {
    k_lat<<<1, nt>>>(d, 1000);
    k_lat<<<1, nt>>>(d, 1000);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads %3d: lds-chain %lld  shfl32 %lld  shfl64 %lld  warpsum64 %lld  bar %lld  "
           "handoff %lld  lds+dfma %lld  sqrt+div %lld\n",
           nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
