// Device half of the sparse Cholesky preconditioner: the two
// triangular sweeps of sparse_tri_solve (sparse_kernels.hpp:178-225) with the
// permutation and the lower()/working() conversions fused into the gather and
// the scatter.  One CTA owns one block column: it gathers the column
// (permuted, narrowed) into shared memory, runs the forward sweep over the
// rows of L and the backward sweep over the rows of U = L^T in blocks of 32
// rows, and scatters the result (widened).  The RCM etree is close to a path,
// so the rows form one dependent chain; blocking shortens that chain to 32
// register steps per block, the rest of each row being a parallel dot product.
#include <cmath>

#include "common.cuh"
#include "spchol.hpp"

namespace mpb {
namespace {

// one warp per row of a 32-row block: 32 rows' dot products in flight at once
constexpr int kSpThreads = 1024, kSpWarps = kSpThreads / 32;

template <typename F>
__device__ __forceinline__ F warp_sum_f(F v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum over p in [p0, p1), lane-strided, of v[p] * y[ci[p]]: each lane's terms in
// ascending order (one fma chain), the index / value loads of 16 terms issued
// ahead of their use so a long profile row streams instead of paying one
// memory latency per term
template <typename F>
__device__ __forceinline__ F row_dot(int p0, int p1, int lane, const int* __restrict__ ci,
                                     const F* __restrict__ v, const F* y) {
  constexpr int U = 16;
  F part = F(0);
  int p = p0 + lane;
  for (; p + (U - 1) * 32 < p1; p += U * 32) {
    int c[U];
    F a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ci[p + u * 32];
      a[u] = v[p + u * 32];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) part = fma(a[u], y[c[u]], part);
  }
  if (p + 7 * 32 < p1) {
    int c[8];
    F a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      c[u] = ci[p + u * 32];
      a[u] = v[p + u * 32];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) part = fma(a[u], y[c[u]], part);
    p += 8 * 32;
  }
  for (; p < p1; p += 32) part = fma(v[p], y[ci[p]], part);
  return part;
}

// Blocked sweeps: the rows go in blocks of 32.  Per block, (A) all 8 warps
// form each row's dot product with the ALREADY FINAL part of y (columns
// outside the block: the bulk of an RCM profile row) and scatter the row's
// in-block entries into a dense 32 x 32 shared tile; (B) warp 0 finishes the
// block's 32 x 32 triangular solve from registers (lane t = row t, one
// shuffle broadcast per column) while warps 1..31 already stream the next
// block's products with the entries that are final (all but the current
// block's), so phase A's bulk hides behind phase B.  The serial chain is 32 short steps per
// block instead of one full row per step.
template <typename Tin, typename F, typename Tout>
__global__ void __launch_bounds__(kSpThreads)
k_spchol_solve(int n, const int* __restrict__ Lrp, const int* __restrict__ Lci,
               const F* __restrict__ Lv, const int* __restrict__ Lsp, const int* __restrict__ Lsp2,
               const int* __restrict__ Urp, const int* __restrict__ Uci, const F* __restrict__ Uv,
               const int* __restrict__ Usp, const int* __restrict__ Usp2, const int* __restrict__ perm, const Tin* __restrict__ B, int64_t ldb,
               Tout* __restrict__ Y, int64_t ldy, int* overflow, F* gy, int use_smem) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ double tile_raw[32 * 33];
  __shared__ double acc_raw[32], dg_raw[32];
  F* tile = reinterpret_cast<F*>(tile_raw);
  F* acc = reinterpret_cast<F*>(acc_raw);
  F* dg = reinterpret_cast<F*>(dg_raw);
  const int col = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  F* y = use_smem ? reinterpret_cast<F*>(raw) : gy + static_cast<int64_t>(col) * n;
  const Tin* b = B + static_cast<int64_t>(col) * ldb;
  int ovf = 0;
  for (int k = tid; k < n; k += kSpThreads) {
    const Tin v = b[perm ? perm[k] : k];
    const F f = static_cast<F>(v);
    if (sizeof(Tin) > sizeof(F) && isinf(f) && !isinf(v)) ovf = 1;  // to_lower overflow
    y[k] = f;
  }
  if (__any_sync(0xffffffffu, ovf) && lane == 0) *overflow = 1;
  const int nblk = (n + 31) / 32;
  // accE[buf][r]: row r's product with the entries two or more blocks back,
  // formed by warps 1..31 while warp 0 runs the previous block's phase B
  __shared__ double accE_raw[2][32];
  F* accE0 = reinterpret_cast<F*>(accE_raw[0]);
  F* accE1 = reinterpret_cast<F*>(accE_raw[1]);
  if (tid < 32) accE0[tid] = F(0);
  // forward: L z = y, blocks ascending; row i: [Lrp, Lsp2) two+ blocks back,
  // [Lsp2, Lsp) the previous block, [Lsp, diag) inside, diag last
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = blk * 32, nb = min(32, n - b0);
    F* accE = (blk & 1) ? accE1 : accE0;
    F* accN = (blk & 1) ? accE0 : accE1;
    for (int e = tid; e < 32 * 33; e += kSpThreads) tile[e] = F(0);
    __syncthreads();
    for (int r = warp; r < nb; r += kSpWarps) {
      const int i = b0 + r, ps2 = Lsp2[i], ps = Lsp[i], pd = Lrp[i + 1] - 1;
      F part = row_dot<F>(ps2, ps, lane, Lci, Lv, y);
      for (int p = ps + lane; p < pd; p += 32) tile[r * 33 + (Lci[p] - b0)] = Lv[p];
      part = warp_sum_f(part);
      if (lane == 0) {
        acc[r] = accE[r] + part;
        dg[r] = Lv[pd];
      }
    }
    __syncthreads();
    if (warp == 0) {
      F s = lane < nb ? y[b0 + lane] - acc[lane] : F(0);
      for (int j = 0; j < nb; ++j) {
        if (lane == j) s = s / dg[j];
        const F yj = __shfl_sync(0xffffffffu, s, j);
        if (lane > j) s = fma(-tile[lane * 33 + j], yj, s);
      }
      if (lane < nb) y[b0 + lane] = s;
    } else if (blk + 1 < nblk) {  // next block's rows: entries before this block (final)
      const int c0 = b0 + 32, nc = min(32, n - c0);
      for (int r = warp - 1; r < nc; r += kSpWarps - 1) {
        const int i = c0 + r;
        F part = warp_sum_f(row_dot<F>(Lrp[i], Lsp2[i], lane, Lci, Lv, y));
        if (lane == 0) accN[r] = part;
      }
    }
    __syncthreads();
  }
  // backward: L^T w = z, blocks descending; U row i: diag, [+1, Usp) inside,
  // [Usp, Usp2) the next block, [Usp2, end) two+ blocks ahead
  if (tid < 32) accE0[tid] = F(0);
  __syncthreads();
  for (int k = 0; k < nblk; ++k) {
    const int blk = nblk - 1 - k;
    const int b0 = blk * 32, nb = min(32, n - b0);
    F* accE = (k & 1) ? accE1 : accE0;
    F* accN = (k & 1) ? accE0 : accE1;
    for (int e = tid; e < 32 * 33; e += kSpThreads) tile[e] = F(0);
    __syncthreads();
    for (int r = warp; r < nb; r += kSpWarps) {
      const int i = b0 + r, q0 = Urp[i], qs = Usp[i], qs2 = Usp2[i];
      F part = row_dot<F>(qs, qs2, lane, Uci, Uv, y);
      for (int q = q0 + 1 + lane; q < qs; q += 32) tile[r * 33 + (Uci[q] - b0)] = Uv[q];
      part = warp_sum_f(part);
      if (lane == 0) {
        acc[r] = accE[r] + part;
        dg[r] = Uv[q0];
      }
    }
    __syncthreads();
    if (warp == 0) {
      F s = lane < nb ? y[b0 + lane] - acc[lane] : F(0);
      for (int j = nb - 1; j >= 0; --j) {
        if (lane == j) s = s / dg[j];
        const F yj = __shfl_sync(0xffffffffu, s, j);
        if (lane < j) s = fma(-tile[lane * 33 + j], yj, s);
      }
      if (lane < nb) y[b0 + lane] = s;
    } else if (blk > 0) {  // previous block's rows: entries after this block (final)
      const int c0 = b0 - 32;
      for (int r = warp - 1; r < 32; r += kSpWarps - 1) {
        const int i = c0 + r;
        F part = warp_sum_f(row_dot<F>(Usp2[i], Urp[i + 1], lane, Uci, Uv, y));
        if (lane == 0) accN[r] = part;
      }
    }
    __syncthreads();
  }
  Tout* out = Y + static_cast<int64_t>(col) * ldy;
  for (int k = tid; k < n; k += kSpThreads) out[perm ? perm[k] : k] = static_cast<Tout>(y[k]);
}

}  // namespace

template <typename Tin, typename F, typename Tout>
void spchol_solve(int n, int c, const int* Lrp, const int* Lci, const F* Lv, const int* Lsp,
                  const int* Urp, const int* Uci, const F* Uv, const int* Usp, const int* perm,
                  const Tin* B, int64_t ldb, Tout* Y, int64_t ldy, int* overflow, F* gy,
                  cudaStream_t s) {
  if (n <= 0 || c <= 0) return;
  const size_t bytes = sizeof(F) * static_cast<size_t>(n);
  const int use = bytes <= 200 * 1024;
  if (use && bytes > 48 * 1024)
    MPB_CUDA(cudaFuncSetAttribute(k_spchol_solve<Tin, F, Tout>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
  k_spchol_solve<Tin, F, Tout><<<c, kSpThreads, use ? bytes : 0, s>>>(
      n, Lrp, Lci, Lv, Lsp, Lsp + n, Urp, Uci, Uv, Usp, Usp + n, perm, B, ldb, Y, ldy, overflow,
      gy, use);
  MPB_LAUNCH_CHECK();
}

template void spchol_solve<double, double, double>(int, int, const int*, const int*, const double*, const int*,
    const int*, const int*, const double*, const int*, const int*, const double*, int64_t, double*,
    int64_t, int*, double*, cudaStream_t);
template void spchol_solve<double, float, double>(int, int, const int*, const int*, const float*, const int*,
    const int*, const int*, const float*, const int*, const int*, const double*, int64_t, double*,
    int64_t, int*, float*, cudaStream_t);
template void spchol_solve<float, float, float>(int, int, const int*, const int*, const float*, const int*,
    const int*, const int*, const float*, const int*, const int*, const float*, int64_t, float*,
    int64_t, int*, float*, cudaStream_t);

}  // namespace mpb
