// Device half of the sparse Cholesky preconditioner: the two
// triangular sweeps of sparse_tri_solve (sparse_kernels.hpp:178-225) with the
// permutation and the lower()/working() conversions fused into the gather and
// the scatter.  One warp owns one block column: it gathers the column
// (permuted, narrowed) into shared memory, runs the forward sweep over the
// rows of L and the backward sweep over the rows of U = L^T, and scatters the
// result (widened).  Each row is a lane-strided dot product + a warp shuffle
// reduction; the rows are a dependent chain (the RCM etree is close to a
// path), so the sweep is latency-bound, like the reference's.
#include <cmath>

#include "common.cuh"
#include "spchol.hpp"

namespace mpb {
namespace {

template <typename F>
__device__ __forceinline__ F warp_sum_f(F v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename Tin, typename F, typename Tout>
__global__ void __launch_bounds__(32)
k_spchol_solve(int n, const int* __restrict__ Lrp, const int* __restrict__ Lci,
               const F* __restrict__ Lv, const int* __restrict__ Urp, const int* __restrict__ Uci,
               const F* __restrict__ Uv, const int* __restrict__ perm, const Tin* __restrict__ B,
               int64_t ldb, Tout* __restrict__ Y, int64_t ldy, int* overflow, F* gy, int use_smem) {
  extern __shared__ __align__(16) unsigned char raw[];
  const int col = blockIdx.x, lane = threadIdx.x;
  F* y = use_smem ? reinterpret_cast<F*>(raw) : gy + static_cast<int64_t>(col) * n;
  const Tin* b = B + static_cast<int64_t>(col) * ldb;
  int ovf = 0;
  for (int k = lane; k < n; k += 32) {
    const Tin v = b[perm ? perm[k] : k];
    const F f = static_cast<F>(v);
    if (sizeof(Tin) > sizeof(F) && isinf(f) && !isinf(v)) ovf = 1;  // to_lower overflow
    y[k] = f;
  }
  if (__any_sync(0xffffffffu, ovf) && lane == 0) *overflow = 1;
  __syncwarp();
  // forward: L z = y, rows ascending, diagonal last
  for (int i = 0; i < n; ++i) {
    const int p0 = Lrp[i], pd = Lrp[i + 1] - 1;
    F part = F(0);
    for (int p = p0 + lane; p < pd; p += 32) part = fma(Lv[p], y[Lci[p]], part);
    part = warp_sum_f(part);
    if (lane == 0) y[i] = (y[i] - part) / Lv[pd];
    __syncwarp();
  }
  // backward: L^T w = z, rows of U = L^T descending, diagonal first
  for (int i = n - 1; i >= 0; --i) {
    const int q0 = Urp[i], q1 = Urp[i + 1];
    F part = F(0);
    for (int q = q0 + 1 + lane; q < q1; q += 32) part = fma(Uv[q], y[Uci[q]], part);
    part = warp_sum_f(part);
    if (lane == 0) y[i] = (y[i] - part) / Uv[q0];
    __syncwarp();
  }
  Tout* out = Y + static_cast<int64_t>(col) * ldy;
  for (int k = lane; k < n; k += 32) out[perm ? perm[k] : k] = static_cast<Tout>(y[k]);
}

}  // namespace

template <typename Tin, typename F, typename Tout>
void spchol_solve(int n, int c, const int* Lrp, const int* Lci, const F* Lv, const int* Urp,
                  const int* Uci, const F* Uv, const int* perm, const Tin* B, int64_t ldb,
                  Tout* Y, int64_t ldy, int* overflow, F* gy, cudaStream_t s) {
  if (n <= 0 || c <= 0) return;
  const size_t bytes = sizeof(F) * static_cast<size_t>(n);
  const int use = bytes <= 200 * 1024;
  if (use && bytes > 48 * 1024)
    MPB_CUDA(cudaFuncSetAttribute(k_spchol_solve<Tin, F, Tout>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
  k_spchol_solve<Tin, F, Tout><<<c, 32, use ? bytes : 0, s>>>(n, Lrp, Lci, Lv, Urp, Uci, Uv, perm,
                                                             B, ldb, Y, ldy, overflow, gy, use);
  MPB_LAUNCH_CHECK();
}

template void spchol_solve<double, double, double>(int, int, const int*, const int*, const double*,
                                                   const int*, const int*, const double*, const int*,
                                                   const double*, int64_t, double*, int64_t, int*,
                                                   double*, cudaStream_t);
template void spchol_solve<double, float, double>(int, int, const int*, const int*, const float*,
                                                  const int*, const int*, const float*, const int*,
                                                  const double*, int64_t, double*, int64_t, int*,
                                                  float*, cudaStream_t);
template void spchol_solve<float, float, float>(int, int, const int*, const int*, const float*,
                                                const int*, const int*, const float*, const int*,
                                                const float*, int64_t, float*, int64_t, int*,
                                                float*, cudaStream_t);

}  // namespace mpb
