// tridiag_lat.cu -- cycles per column of the tridiagonalisation's matvec
// phase (p = beta A_trail v over a shared-memory 48 x 48 block, 256 threads,
// one barrier) under several thread mappings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/tridiag_lat.cu -o build/tridiag_lat
#include <cstdio>

constexpr int S = 48, LD = S + 1, NT = 256;

template <int V>
__global__ void __launch_bounds__(NT) k_mv(const double* Ain, long long* out) {
  __shared__ double A[S * LD], hp[S], hv[S];
  const int tid = threadIdx.x;
  for (int i = tid; i < S * LD; i += NT) A[i] = Ain[i % (S * S)];
  for (int i = tid; i < S; i += NT) hv[i] = 0.01 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep)
    for (int k = 0; k + 2 < S; ++k) {
      const int len = S - k - 1;
      const double beta = 1.0 + 1e-3 * k;
      if (V == 0) {  // current: 4 lanes per row, strided columns, 3 chains
        for (int base = 0; base < len; base += NT / 4) {
          const int row = base + (tid >> 2), q = tid & 3;
          double a0 = 0, a1 = 0, a2 = 0;
          if (row < len) {
            const double* arow = A + (k + 1 + row) + (k + 1) * LD;
            int j = q;
            for (; j + 8 < len; j += 12) {
              a0 = fma(arow[j * LD], hv[j], a0);
              a1 = fma(arow[(j + 4) * LD], hv[j + 4], a1);
              a2 = fma(arow[(j + 8) * LD], hv[j + 8], a2);
            }
            for (; j < len; j += 4) a0 = fma(arow[j * LD], hv[j], a0);
          }
          double acc = (a0 + a1) + a2;
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          if (q == 0 && row < len) hp[row] = beta * acc;
        }
      } else if (V == 1) {  // 4 lanes per row, fully unrolled predicated (12 per lane)
        const int row = tid >> 2, q = tid & 3;
        double a[4] = {0, 0, 0, 0};
        if (row < len) {
          const double* arow = A + (k + 1 + row) + (k + 1) * LD;
#pragma unroll
          for (int t = 0; t < 12; ++t) {
            const int j = q + 4 * t;
            if (j < len) a[t & 3] = fma(arow[j * LD], hv[j], a[t & 3]);
          }
        }
        double acc = (a[0] + a[1]) + (a[2] + a[3]);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (q == 0 && row < len) hp[row] = beta * acc;
      } else if (V == 3) {  // 4 lanes per row, loads first, products, pairwise tree
        const int row = tid >> 2, q = tid & 3;
        double pr[12];
        const double* arow = A + (k + 1 + min(row, len - 1)) + (k + 1) * LD;
#pragma unroll
        for (int t = 0; t < 12; ++t) {
          const int j = q + 4 * t;
          pr[t] = (j < len) ? arow[j * LD] * hv[j] : 0.0;
        }
#pragma unroll
        for (int w = 1; w < 12; w <<= 1)
#pragma unroll
          for (int t = 0; t + w < 12; t += 2 * w) pr[t] += pr[t + w];
        double acc = pr[0];
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (q == 0 && row < len) hp[row] = beta * acc;
      } else if (V == 2) {  // 8 lanes per row over 2 passes? no: 5 lanes -> use 8 lanes, rows < 32 per pass
        for (int base = 0; base < len; base += NT / 8) {
          const int row = base + (tid >> 3), q = tid & 7;
          double a[3] = {0, 0, 0};
          if (row < len) {
            const double* arow = A + (k + 1 + row) + (k + 1) * LD;
#pragma unroll
            for (int t = 0; t < 6; ++t) {
              const int j = q + 8 * t;
              if (j < len) a[t % 3] = fma(arow[j * LD], hv[j], a[t % 3]);
            }
          }
          double acc = (a[0] + a[1]) + a[2];
          acc += __shfl_xor_sync(0xffffffffu, acc, 1);
          acc += __shfl_xor_sync(0xffffffffu, acc, 2);
          acc += __shfl_xor_sync(0xffffffffu, acc, 4);
          if (q == 0 && row < len) hp[row] = beta * acc;
        }
      }
      __syncthreads();
      if (tid == 0) hv[k % S] += hp[0] * 1e-30;
    }
  long long t1 = clock64();
  if (tid == 0) out[V] = (t1 - t0) / (4 * (S - 2));
}

int main() {
  double* A;
  long long* out;
  cudaMalloc(&A, S * S * 8);
  cudaMemset(A, 0, S * S * 8);
  cudaMalloc(&out, 64);
  k_mv<0><<<1, NT>>>(A, out);
  k_mv<1><<<1, NT>>>(A, out);
  k_mv<2><<<1, NT>>>(A, out);
  k_mv<0><<<1, NT>>>(A, out);
  k_mv<1><<<1, NT>>>(A, out);
  k_mv<2><<<1, NT>>>(A, out);
  k_mv<3><<<1, NT>>>(A, out);
  long long h[8];
  cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
  printf("matvec+barrier cycles/column: current %lld  unrolled-4lanes %lld  8lanes %lld  tree %lld\n", h[0], h[1], h[2], h[3]);
  return 0;
}
