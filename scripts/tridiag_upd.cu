// tridiag_upd.cu -- cycles per column of the tridiagonalisation's update
// phase (kappa, rank-2 trailing update, next reflector by warp 0, barrier) as
// written in k_small_ql3, and variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/tridiag_upd.cu -o build/tridiag_upd
#include <cstdio>

constexpr int S = 48, LD = S + 1, NT = 256, kMaxT = 6;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <int V>
__global__ void __launch_bounds__(NT) k_upd(const double* Ain, long long* out) {
  __shared__ double A[S * LD], hp[S], hb[S], e[S], part[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < S * LD; i += NT) A[i] = Ain[i % (S * S)] + (i % 7) * 0.01;
  for (int i = tid; i < S; i += NT) hp[i] = 0.02 * i;
  __syncthreads();
  const auto reflector = [&](int k) {
    const int len = S - k - 1;
    double* hv = A + (k + 1) + k * LD;
    double p = 0;
    for (int i = 1 + lane; i < len; i += 32) p = fma(hv[i], hv[i], p);
    const double tail2 = wsum(p);
    const double x0 = hv[0];
    const double nrm = sqrt(fma(x0, x0, tail2));
    if (lane == 0) {
      const double ph = x0 >= 0 ? 1.0 : -1.0;
      const double v0 = x0 + ph * nrm;
      hb[k] = 2.0 / fma(v0, v0, tail2);
      e[k] = -ph * nrm;
      hv[0] = v0;
    }
  };
  long long t0 = clock64(), tk = 0, tu = 0, tr = 0;
  for (int rep = 0; rep < 4; ++rep)
    for (int k = 0; k + 2 < S; ++k) {
      const int len = S - k - 1;
      const double* hv = A + (k + 1) + k * LD;
      const double beta = hb[k] * 1e-3 + 1e-3;
      long long a0 = clock64();
      double kappa;
      if (V == 0) {
        double vp = 0;
        for (int i = lane; i < len; i += 32) vp = fma(hv[i], hp[i], vp);
        kappa = beta * wsum(vp) / 2;
      } else {
        kappa = beta * part[0] / 2;  // (V1: kappa precomputed elsewhere)
      }
      long long a1 = clock64();
      {
        const int tx = tid & 15, ty = tid >> 4;
        double vi[kMaxT], wi[kMaxT];
#pragma unroll
        for (int a = 0; a < kMaxT; ++a) {
          const int i = tx + 16 * a;
          vi[a] = i < len ? hv[i] : 0.0;
          wi[a] = i < len ? hp[i] - kappa * vi[a] : 0.0;
        }
#pragma unroll
        for (int b2 = 0; b2 < kMaxT; ++b2) {
          const int j = ty + 16 * b2;
          if (j >= len) break;
          const double vj = hv[j], wj = hp[j] - kappa * vj;
          double* acol = A + (k + 1) + (k + 1 + j) * LD;
#pragma unroll
          for (int a = 0; a < kMaxT; ++a) {
            const int i = tx + 16 * a;
            if (i < len) acol[i] -= vi[a] * wj * 1e-9 + wi[a] * vj * 1e-9;
          }
        }
      }
      long long a2 = clock64();
      if (warp == 0 && k + 3 < S) {
        __syncwarp();
        reflector(k + 1);
      }
      long long a3 = clock64();
      __syncthreads();
      tk += a1 - a0;
      tu += a2 - a1;
      tr += a3 - a2;
    }
  long long t1 = clock64();
  if (tid == 0) {
    out[0] = (t1 - t0) / (4 * (S - 2));
    out[1] = tk / (4 * (S - 2));
    out[2] = tu / (4 * (S - 2));
    out[3] = tr / (4 * (S - 2));
  }
}

int main() {
  double* A;
  long long* out;
  cudaMalloc(&A, S * S * 8);
  cudaMemset(A, 0, S * S * 8);
  cudaMalloc(&out, 64);
  long long h[4];
  for (int it = 0; it < 2; ++it) {
    k_upd<0><<<1, NT>>>(A, out);
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  }
  printf("update phase cycles/column: total %lld = kappa %lld + update %lld + reflector %lld (+barrier)\n",
         h[0], h[1], h[2], h[3]);
  return 0;
}
