// smallwarp.cuh -- one-warp triangular routines shared by several kernels.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace mpb {

// R^{-1} of an upper-triangular m x m R (m <= MAXM <= 32) by one warp:
// column c of R^{-1} by lane c (back substitution), row k of R broadcast from
// lane k.  R is read as TS and converted to T; Rw (optional) receives that
// converted copy.  A zero or subnormal pivot is SingularTriangular
// (tri_solve, dense_kernels.hpp:177-194): status = {code, index}, first error
// wins; returns false then.  Called by all 32 lanes of one warp.
template <typename T, typename TS, int MAXM>
__device__ __forceinline__ bool warp_upper_inverse(int m, const TS* __restrict__ R, int64_t ldr,
                                                   T* __restrict__ Rw, T* __restrict__ Rinv,
                                                   int* status) {
  const int lane = threadIdx.x & 31;
  const T tiny = sizeof(T) == 8 ? T(DBL_MIN) : T(FLT_MIN);
  T r[MAXM];  // row `lane` of R
#pragma unroll
  for (int l = 0; l < MAXM; ++l)
    r[l] = (lane < m && l < m && l >= lane) ? static_cast<T>(R[lane + static_cast<int64_t>(l) * ldr])
                                            : T(0);
  if (Rw && lane < m) {
#pragma unroll
    for (int l = 0; l < MAXM; ++l)
      if (l < m) Rw[lane + l * m] = r[l];
  }
  T rdl = T(0);
#pragma unroll
  for (int l = 0; l < MAXM; ++l)
    if (l == lane) rdl = r[l];
  const bool bad = lane < m && (fabs(rdl) == T(0) || fabs(rdl) < tiny);
  const unsigned badm = __ballot_sync(0xffffffffu, bad);
  if (badm) {
    if (lane == 0 && status[0] == 0) {
      status[0] = MPEIG_E_SINGULAR_TRI;
      status[1] = __ffs(badm) - 1;
    }
    return false;
  }
  const T rinv_l = lane < m ? T(1) / rdl : T(0);
  T y[MAXM];
  const int c = lane;
#pragma unroll
  for (int k = MAXM - 1; k >= 0; --k) {
    y[k] = T(0);
    if (k >= m) continue;
    T s = k == c ? T(1) : T(0);
#pragma unroll
    for (int l = k + 1; l < MAXM; ++l) {
      if (l >= m) break;
      s = fma(-__shfl_sync(0xffffffffu, r[l], k), y[l], s);
    }
    const T rk = __shfl_sync(0xffffffffu, rinv_l, k);  // all lanes take part
    y[k] = k <= c ? s * rk : T(0);
  }
  if (c < m) {
#pragma unroll
    for (int k = 0; k < MAXM; ++k)
      if (k < m) Rinv[k + c * m] = y[k];
  }
  return true;
}

// G = L L^T and Uinv = L^{-T} (dense_cholesky, dense_kernels.hpp:128-152) by
// one warp for m <= MAXM <= 32: lane i holds row i.  G is read through L2
// (__ldcg: it may have been written by other CTAs of the calling kernel).
// Failure -> status {NOT_PD | OVERFLOW, column}, returns false.  tau2 > 0
// (conditioning guard of the speculative CholQR): a pivot below tau2 * G_jj,
// i.e. column j with less than sqrt(tau2) of its norm outside the span of the
// columns before it, also fails as NOT_PD.
template <typename T, int MAXM>
__device__ __forceinline__ bool warp_cholesky_inv(int m, const T* __restrict__ G, int64_t ldg,
                                                  T* __restrict__ L, T* __restrict__ Uinv,
                                                  int* status, T tau2 = T(0)) {
  const int lane = threadIdx.x & 31;
  T a[MAXM];
#pragma unroll
  for (int j = 0; j < MAXM; ++j)
    a[j] = (lane < m && j < m && lane >= j) ? __ldcg(G + lane + static_cast<int64_t>(j) * ldg) : T(0);
  T gdiag = T(0);  // G(lane, lane) before the elimination
  T rdiag = T(0);  // 1 / L(lane, lane)
#pragma unroll
  for (int j = 0; j < MAXM; ++j)
    if (j == lane) gdiag = a[j];
#pragma unroll
  for (int j = 0; j < MAXM; ++j) {
    if (j >= m) break;
    const T d2 = __shfl_sync(0xffffffffu, a[j], j);
    const T gjj = __shfl_sync(0xffffffffu, gdiag, j);
    if (!isfinite(static_cast<double>(d2)) || !(d2 > T(0)) || (tau2 > T(0) && !(d2 >= tau2 * gjj))) {
      if (lane == 0 && status[0] == 0) {
        status[0] = isfinite(static_cast<double>(d2)) ? MPEIG_E_NOT_PD : MPEIG_E_OVERFLOW;
        status[1] = j;
      }
      return false;
    }
    // one reciprocal square root on the serial chain (not sqrt + divide)
    T rd = rsqrt(d2);
    if constexpr (sizeof(T) == 4) {
      // rsqrtf: a 2-ulp approximation with a one-sided bias; one Newton step
      const T h = d2 * rd;
      rd = rd * fma(T(-0.5) * h, rd, T(1.5));
    }
    const T d = d2 * rd;
    const T lij = lane > j ? a[j] * rd : (lane == j ? d : T(0));
    if (lane == j) rdiag = rd;
    a[j] = lij;
#pragma unroll
    for (int k = j + 1; k < MAXM; ++k) {
      const T lkj = __shfl_sync(0xffffffffu, lij, k);
      if (lane >= k) a[k] = fma(-lij, lkj, a[k]);
    }
  }
  if (lane < m) {
#pragma unroll
    for (int j = 0; j < MAXM; ++j)
      if (j < m) L[lane + j * m] = a[j];
  }
  if (!Uinv) return true;
  // X = L^{-1}, column c by lane c, right-looking: x_l is final once the
  // updates of rows < l are in, then every later row's sum takes its term
  // at once (independent FMAs), so the serial chain is one multiply and one
  // FMA per row.  The L(i, l) broadcasts do not depend on x.  Uinv(c, i) = X(i, c).
  const int c = lane;
  T acc[MAXM];
#pragma unroll
  for (int i = 0; i < MAXM; ++i) acc[i] = i == c ? T(1) : T(0);
#pragma unroll
  for (int l = 0; l < MAXM; ++l) {
    if (l >= m) break;
    const T xl = acc[l] * __shfl_sync(0xffffffffu, rdiag, l);
    if (c < m) Uinv[c + l * m] = xl;
#pragma unroll
    for (int i = l + 1; i < MAXM; ++i) {
      const T lil = __shfl_sync(0xffffffffu, a[l], i);
      if (i < m) acc[i] = fma(-lil, xl, acc[i]);
    }
  }
  return true;
}

}  // namespace mpb
