// small.cu -- single-CTA kernels for the small (<= 3m x 3m) dense steps.
//
// These run once or twice per iteration on matrices of order <= 576 and are
// latency-bound: each stages its matrices in shared memory (global scratch
// only when they do not fit) and spreads every step over the CTA (warp
// reductions, trailing updates in parallel) so that the serial chain is one
// barrier and one scalar op (sqrt / reciprocal) per column.  They follow the
// reference's small factorizations step for step (dense_cholesky,
// dense_kernels.hpp:128-152; householder_qr_square, ortho.hpp:30-121;
// matmul :20-34); sums are formed in parallel, so results agree to rounding.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "rn.cuh"
#include "smallwarp.cuh"

namespace mpb {
namespace {

constexpr int kSmallThreads = 256;
constexpr size_t kSmemCap = 200 * 1024;
// k_hl_coeffs's dynamic shared memory (p = m = 96: 217 KB) + its ~2 KB static
constexpr size_t kHlSmemCap = 224 * 1024;
constexpr int kMaxHlP = 256;  // largest P block (block size m) of the HL update

template <typename T>
__global__ void k_symmetrize(int64_t s, T* G, int64_t ldg) {
  MPB_PDL_WAIT();
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < s * s;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % s, j = idx / s;
    if (i < j) {
      const T v = (G[i + j * ldg] + G[j + i * ldg]) / T(2);
      G[i + j * ldg] = v;
      G[j + i * ldg] = v;
    }
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum_s(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Right-looking Cholesky G = L L^T (dense_cholesky, dense_kernels.hpp:128-152)
// with the trailing update spread over the CTA, then Uinv = L^{-T}: L^{-1}
// by forward substitution, one thread per column.  status = {code, index},
// first error wins.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
k_cholesky_inv(int m, const T* __restrict__ G, int64_t ldg, T* __restrict__ L,
               T* __restrict__ Uinv, int* status, int use_smem, T tau2) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char raw[];
  T* As = use_smem ? reinterpret_cast<T*>(raw) : L;  // working lower triangle -> L
  T* Us = use_smem ? As + m * m : Uinv;
  __shared__ int fail;
  __shared__ T sh_rd;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  for (int idx = tid; idx < m * m; idx += nt) {
    const int i = idx % m, j = idx / m;
    As[idx] = i >= j ? G[i + static_cast<int64_t>(j) * ldg] : T(0);
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (tid == 0) {
      const T s = As[j + j * m];
      if (!isfinite(static_cast<double>(s))) {
        fail = 1;
        if (status[0] == 0) {
          status[0] = MPEIG_E_OVERFLOW;
          status[1] = j;
        }
      } else if (!(s > T(0)) || (tau2 > T(0) && !(s >= tau2 * G[j + static_cast<int64_t>(j) * ldg]))) {
        fail = 1;
        if (status[0] == 0) {
          status[0] = MPEIG_E_NOT_PD;
          status[1] = j;
        }
      } else {
        const T d = sqrt(s);
        As[j + j * m] = d;
        sh_rd = T(1) / d;
      }
    }
    __syncthreads();
    if (fail) return;
    const T rd = sh_rd;
    // trailing lower triangle (i >= k > j): A(i,k) -= A(i,j) A(k,j) / d^2;
    // column j is scaled after (it is read here)
    const int len = m - j - 1;
    for (int idx = tid; idx < len * len; idx += nt) {
      const int i = j + 1 + idx % len, k = j + 1 + idx / len;
      if (i >= k) As[i + k * m] = fma(-(As[i + j * m] * rd), As[k + j * m] * rd, As[i + k * m]);
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < m; i += nt) As[i + j * m] *= rd;
    __syncthreads();
  }
  if (Uinv) {
    // X = L^{-1} (lower), column c by thread c; Uinv = X^T (upper)
    for (int c = tid; c < m; c += nt) {
      for (int k = 0; k < c; ++k) Us[c + k * m] = T(0);
      const T xc = T(1) / As[c + c * m];
      Us[c + c * m] = xc;  // Us(c, k) holds X(k, c)
      for (int k = c + 1; k < m; ++k) {
        T s0 = T(0), s1 = T(0);
        int l = c;
        for (; l + 1 < k; l += 2) {
          s0 = fma(As[k + l * m], Us[c + l * m], s0);
          s1 = fma(As[k + (l + 1) * m], Us[c + (l + 1) * m], s1);
        }
        if (l < k) s0 = fma(As[k + l * m], Us[c + l * m], s0);
        Us[c + k * m] = -(s0 + s1) / As[k + k * m];
      }
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int idx = tid; idx < m * m; idx += nt) {
      L[idx] = As[idx];
      if (Uinv) Uinv[idx] = Us[idx];
    }
  }
}

// R^{-1} of an upper-triangular R: column c of R^{-1} by thread c (back
// substitution).  A zero or subnormal pivot is SingularTriangular.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
k_upper_inverse(int m, const T* __restrict__ R, int64_t ldr, T* __restrict__ Rinv, int* status,
                int use_smem) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char raw[];
  T* Rs = reinterpret_cast<T*>(raw);
  T* Is = use_smem ? Rs + m * m : Rinv;
  T* rdiag = use_smem ? Is + m * m : nullptr;
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  __syncthreads();
  const T tiny = sizeof(T) == 8 ? T(DBL_MIN) : T(FLT_MIN);
  if (use_smem)
    for (int idx = tid; idx < m * m; idx += nt) Rs[idx] = R[(idx % m) + static_cast<int64_t>(idx / m) * ldr];
  for (int j = tid; j < m; j += nt) {
    const T a = R[j + static_cast<int64_t>(j) * ldr];
    if (fabs(a) == T(0) || fabs(a) < tiny) fail = 1;
    if (rdiag) rdiag[j] = T(1) / a;
  }
  __syncthreads();
  if (fail) {
    if (tid == 0 && status[0] == 0) {
      for (int j = 0; j < m; ++j) {
        const T a = fabs(R[j + static_cast<int64_t>(j) * ldr]);
        if (a == T(0) || a < tiny) {
          status[0] = MPEIG_E_SINGULAR_TRI;
          status[1] = j;
          break;
        }
      }
    }
    return;
  }
  const T* Rr = use_smem ? Rs : R;
  const int64_t ld = use_smem ? m : ldr;
  for (int c = tid; c < m; c += nt) {
    for (int k = c + 1; k < m; ++k) Is[k + c * m] = T(0);
    const T rc = rdiag ? rdiag[c] : T(1) / Rr[c + c * ld];
    Is[c + c * m] = rc;
    for (int k = c - 1; k >= 0; --k) {
      T s0 = T(0), s1 = T(0);
      int l = k + 1;
      for (; l + 1 <= c; l += 2) {
        s0 = fma(Rr[k + l * ld], Is[l + c * m], s0);
        s1 = fma(Rr[k + (l + 1) * ld], Is[l + 1 + c * m], s1);
      }
      if (l <= c) s0 = fma(Rr[k + l * ld], Is[l + c * m], s0);
      Is[k + c * m] = -(s0 + s1) * (rdiag ? rdiag[k] : T(1) / Rr[k + k * ld]);
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int idx = tid; idx < m * m; idx += nt) Rinv[idx] = Is[idx];
  }
}

template <typename T>
__global__ void k_small_transpose(int r, int c, const T* __restrict__ A, int64_t lda,
                                  T* __restrict__ B, int64_t ldb) {
  MPB_PDL_WAIT();
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       idx < static_cast<int64_t>(r) * c; idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(idx % r), j = static_cast<int>(idx / r);
    B[j + i * ldb] = A[i + j * lda];
  }
}

template <typename T>
__global__ void k_small_matmul(int r, int k, int c, const T* __restrict__ A, int64_t lda,
                               const T* __restrict__ B, int64_t ldb, T* __restrict__ C, int64_t ldc) {
  MPB_PDL_WAIT();
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       idx < static_cast<int64_t>(r) * c; idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(idx % r), j = static_cast<int>(idx / r);
    T s = T(0);
    for (int l = 0; l < k; ++l) s = fma(A[i + l * lda], B[l + j * ldb], s);
    C[i + j * ldc] = s;
  }
}

// Hetmaniuk-Lehoucq coefficients, single CTA.  Work layout (T), in shared
// memory when it fits, else in `scratch`:
//   M  p x m   (C(0:m, m:m+p)^T, reduced in place to R)
//   V  p x p   (reflector j in column j, rows j..p-1)
//   Q  p x p
//   beta p
template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
k_hl_coeffs(int s, int m, int p, const T* __restrict__ C, int64_t ldc, T* __restrict__ coef,
            T* __restrict__ scratch, int* fallback, int use_smem, T* __restrict__ qout) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char raw[];
  T* M = use_smem ? reinterpret_cast<T*>(raw) : scratch;
  T* V = M + p * m;
  T* Q = V + p * p;
  // Reflector scalars in fp64 for both precisions (bitwise the reference's
  // for T = double; for T = float, 2/|v|^2 would overflow binary32 once a
  // column of C is tiny, which the Jacobi eigensolver's near-unit
  // eigenvectors produce).
  __shared__ double beta[kMaxHlP];
  __shared__ int fb;
  __shared__ double sh_beta;
  __shared__ T sh_diag;
  const int tid = threadIdx.x, nt = blockDim.x;
  // c_x = C(:, 0:m)
  for (int64_t idx = tid; idx < static_cast<int64_t>(s) * m; idx += nt) {
    const int i = static_cast<int>(idx % s), j = static_cast<int>(idx / s);
    coef[i + static_cast<int64_t>(j) * s] = C[i + static_cast<int64_t>(j) * ldc];
  }
  if (p == 0) return;
  if (tid == 0) fb = 0;
  // M(a, b) = C(b, m + a)   (a < p rows, b < m cols): top^*
  for (int idx = tid; idx < p * m; idx += nt) {
    const int a = idx % p, b = idx / p;
    M[a + b * p] = C[b + static_cast<int64_t>(m + a) * ldc];
  }
  __syncthreads();
  // householder_reduce (ortho.hpp:30-76) on the p x m block, steps = p;
  // warp 0 forms each reflector, the 8 warps apply it (a column per warp,
  // rows over lanes)
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int j = 0; j < p; ++j) {
    const int len = p - j;
    if (warp == 0) {
      double part = 0.0;
      for (int i = j + 1 + lane; i < p; i += 32) {
        const double a = static_cast<double>(M[i + j * p]);
        part = fma(a, a, part);
      }
      const double tail = warp_sum_s(part);
      const double x0 = static_cast<double>(M[j + j * p]);
      const double nrm = sqrt(fma(x0, x0, tail));
      if (nrm == 0.0) {
        if (lane == 0) fb = 1;
      } else {
        const double phase = x0 > 0.0 ? 1.0 : (x0 < 0.0 ? -1.0 : 1.0);
        const double v0 = x0 + phase * nrm;
        T* v = V + j * p + j;
        for (int i = lane; i < len; i += 32) v[i] = i == 0 ? static_cast<T>(v0) : M[j + i + j * p];
        if (lane == 0) {
          sh_beta = 2.0 / fma(v0, v0, tail);
          beta[j] = sh_beta;
          sh_diag = static_cast<T>(-phase * nrm);  // R(j,j) after the reflection (ortho.hpp:72)
        }
      }
    }
    __syncthreads();
    if (fb) break;
    const double b = sh_beta;
    const T* v = V + j * p + j;
    for (int c = j + 1 + warp; c < m; c += nw) {
      T* col = M + c * p + j;
      T part = T(0);
      for (int i = lane; i < len; i += 32) part = fma(v[i], col[i], part);
      const T f = static_cast<T>(static_cast<double>(warp_sum_s(part)) * b);
      for (int i = lane; i < len; i += 32) col[i] = fma(-f, v[i], col[i]);
    }
    if (warp == 0)
      for (int i = j + lane; i < p; i += 32) M[i + j * p] = i == j ? sh_diag : T(0);
    __syncthreads();
  }
  if (!fb) {
    // Q = I, reflectors applied last to first (apply_reflectors_to, ortho.hpp:78-92)
    for (int idx = tid; idx < p * p; idx += nt) Q[idx] = (idx % p) == (idx / p) ? T(1) : T(0);
    __syncthreads();
    for (int jj = p - 1; jj >= 0; --jj) {
      const int len = p - jj;
      const T* v = V + jj * p + jj;
      const double b = beta[jj];
      for (int c = warp; c < p; c += nw) {
        T* qc = Q + c * p + jj;
        T part = T(0);
        for (int i = lane; i < len; i += 32) part = fma(v[i], qc[i], part);
        const T f = static_cast<T>(static_cast<double>(warp_sum_s(part)) * b);
        for (int i = lane; i < len; i += 32) qc[i] = fma(-f, v[i], qc[i]);
      }
      __syncthreads();
    }
    // fix_diagonal_phases (ortho.hpp:95-110): steps = min(p, m) = p
    if (tid == 0) {
      for (int j = 0; j < p; ++j)
        if (M[j + j * p] == T(0)) fb = 1;
    }
    __syncthreads();
    if (!fb) {
      for (int idx = tid; idx < p * p; idx += nt) {
        const int j = idx / p;
        if (M[j + j * p] < T(0)) Q[idx] = -Q[idx];
      }
    }
    __syncthreads();
  }
  if (tid == 0) *fallback = fb;
  if (qout) {  // c_pv by k_hl_cpv across the GPU
    if (Q != qout && !fb)
      for (int idx = tid; idx < p * p; idx += nt) qout[idx] = Q[idx];
    return;
  }
  // c_pv = C(:, m:m+p) V  (V = I on fallback)
  for (int64_t idx = tid; idx < static_cast<int64_t>(s) * p; idx += nt) {
    const int i = static_cast<int>(idx % s), j = static_cast<int>(idx / s);
    T acc;
    if (fb) {
      acc = C[i + static_cast<int64_t>(m + j) * ldc];
    } else {
      // matmul(cp, Q) (dense_kernels.hpp:20-34)
      T a0 = T(0), a1 = T(0);
      int l = 0;
      for (; l + 1 < p; l += 2) {
        a0 = fma(C[i + static_cast<int64_t>(m + l) * ldc], Q[l + j * p], a0);
        a1 = fma(C[i + static_cast<int64_t>(m + l + 1) * ldc], Q[l + 1 + j * p], a1);
      }
      if (l < p) a0 = fma(C[i + static_cast<int64_t>(m + l) * ldc], Q[l + j * p], a0);
      acc = a0 + a1;
    }
    coef[i + static_cast<int64_t>(m + j) * s] = acc;
  }
}

// c_pv = C(:, m:m+p) Q (V = I on fallback) for k_hl_coeffs's Q: a thread per
// entry, rows in consecutive lanes (coalesced C columns), Q broadcast; the same
// two-way split sum as the single-CTA loop above, so results are identical.
template <typename T>
__global__ void __launch_bounds__(256)
k_hl_cpv(int s, int m, int p, const T* __restrict__ C, int64_t ldc, const T* __restrict__ Q,
         T* __restrict__ coef, const int* fallback) {
  MPB_PDL_WAIT();
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(s) * p) return;
  const int i = static_cast<int>(idx % s), j = static_cast<int>(idx / s);
  const T* cp = C + static_cast<int64_t>(m) * ldc + i;
  T acc;
  if (*fallback) {
    acc = cp[static_cast<int64_t>(j) * ldc];
  } else {
    const T* q = Q + static_cast<int64_t>(j) * p;
    T a0 = T(0), a1 = T(0);
    int l = 0;
    for (; l + 1 < p; l += 2) {
      a0 = fma(cp[static_cast<int64_t>(l) * ldc], q[l], a0);
      a1 = fma(cp[static_cast<int64_t>(l + 1) * ldc], q[l + 1], a1);
    }
    if (l < p) a0 = fma(cp[static_cast<int64_t>(l) * ldc], q[l], a0);
    acc = a0 + a1;
  }
  coef[i + static_cast<int64_t>(m + j) * s] = acc;
}

// ---- one-warp forms for m <= 32 ---------------------------------------------
// Lane i holds row i in registers; the per-column serial chain is a shuffle
// broadcast and one sqrt / reciprocal, with no CTA barrier at all.

// G = L L^T and Uinv = L^{-T} (dense_cholesky, dense_kernels.hpp:128-152)
template <typename T, int MAXM>
__global__ void __launch_bounds__(32)
k_cholesky_inv_warp(int m, const T* __restrict__ G, int64_t ldg, T* __restrict__ L,
                    T* __restrict__ Uinv, int* status, T tau2) {
  MPB_PDL_WAIT();
  warp_cholesky_inv<T, MAXM>(m, G, ldg, L, Uinv, status, tau2);
}

// R^{-1} of an upper-triangular R, one warp (smallwarp.cuh)
template <typename T, int MAXM>
__global__ void __launch_bounds__(32)
k_upper_inverse_warp(int m, const T* __restrict__ R, int64_t ldr, T* __restrict__ Rinv,
                     int* status) {
  MPB_PDL_WAIT();
  warp_upper_inverse<T, T, MAXM>(m, R, ldr, nullptr, Rinv, status);
}

// Hetmaniuk-Lehoucq coefficients (hl_update, eigensolvers.hpp:148-174) for
// m, p <= MAXM.  householder_qr_square of top^* (p x m) by warp 0 with the
// COLUMNS in lanes: lane c holds column c, so the reflector of column j is
// formed by lane j alone and every other column's dot product is lane-local
// (no shuffles); reflectors go to shared memory.  Then every thread takes a
// row of C_p and applies Q = H_0 ... H_{p-1} and the phase fix from the
// right, again lane-local: c_pv(r, :) = C_p(r, :) Q.
template <typename T, int MAXM>
__global__ void __launch_bounds__(kSmallThreads)
k_hl_coeffs_warp(int s, int m, int p, const T* __restrict__ C, int64_t ldc, T* __restrict__ coef,
                 int* fallback) {
  MPB_PDL_WAIT();
  __shared__ T Vs[MAXM][MAXM + 1];  // Vs[j][a]: reflector j, component a (a >= j)
  __shared__ double Bs[MAXM];       // reflector scalars (fp64)
  __shared__ T Sg[MAXM];            // sign of R(j, j)
  __shared__ int fb;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t idx = tid; idx < static_cast<int64_t>(s) * m; idx += nt) {
    const int i = static_cast<int>(idx % s), j = static_cast<int>(idx / s);
    coef[i + static_cast<int64_t>(j) * s] = C[i + static_cast<int64_t>(j) * ldc];
  }
  if (p == 0) return;
  if (tid < 32) {
    const int lane = tid;
    // column `lane` of M = top^*: M(a, c) = C(c, m + a), a < p
    T mc[MAXM];
#pragma unroll
    for (int a = 0; a < MAXM; ++a)
      mc[a] = (lane < m && a < p) ? C[lane + static_cast<int64_t>(m + a) * ldc] : T(0);
    int bad = 0;
#pragma unroll
    for (int j = 0; j < MAXM; ++j) {
      if (j < p && !bad) {  // guards, not break: the loops stay fully unrolled
        if (lane == j) {
          // four partial sums: the reduction is on the serial path
          double tp[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int a = j + 1; a < MAXM; ++a)
            tp[a & 3] = fma(static_cast<double>(mc[a]), static_cast<double>(mc[a]), tp[a & 3]);
          const double tail = (tp[0] + tp[1]) + (tp[2] + tp[3]);
          const double x0 = static_cast<double>(mc[j]);
          const double nrm = sqrt(fma(x0, x0, tail));
          if (nrm == 0.0) {
            Bs[j] = -1.0;  // rank deficient: fallback
          } else {
            const double phase = x0 < 0.0 ? -1.0 : 1.0;
            const double v0 = x0 + phase * nrm;
            Bs[j] = 2.0 / fma(v0, v0, tail);
#pragma unroll
            for (int a = 0; a < MAXM; ++a)
              Vs[j][a] = a < j ? T(0) : (a == j ? static_cast<T>(v0) : mc[a]);
            const T d = static_cast<T>(-phase * nrm);  // R(j,j) (ortho.hpp:72)
            Sg[j] = d < T(0) ? T(-1) : T(1);
#pragma unroll
            for (int a = j; a < MAXM; ++a) mc[a] = a == j ? d : T(0);
          }
        }
        __syncwarp();
        const double beta = Bs[j];
        if (beta < 0.0) bad = 1;
        if (!bad && lane > j && lane < m) {
          T dp[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int a = j; a < MAXM; ++a) dp[a & 3] = fma(Vs[j][a], mc[a], dp[a & 3]);
          const T dot = (dp[0] + dp[1]) + (dp[2] + dp[3]);
          const T f = static_cast<T>(static_cast<double>(dot) * beta);
#pragma unroll
          for (int a = j; a < MAXM; ++a) mc[a] = fma(-f, Vs[j][a], mc[a]);
        }
        __syncwarp();
      }
    }
    if (lane == 0) fb = bad;
  }
  __syncthreads();
  if (tid == 0) *fallback = fb;
  // c_pv(r, :) = C_p(r, :) H_0 H_1 ... H_{p-1} diag(sign R(j,j))  (V = I on fallback)
  const bool use_q = !fb;
  for (int r = tid; r < s; r += nt) {
    T y[MAXM];
#pragma unroll
    for (int a = 0; a < MAXM; ++a)
      y[a] = a < p ? C[r + static_cast<int64_t>(m + a) * ldc] : T(0);
    if (use_q) {
#pragma unroll
      for (int j = 0; j < MAXM; ++j) {
        if (j < p) {
          T dp[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int a = j; a < MAXM; ++a) dp[a & 3] = fma(y[a], Vs[j][a], dp[a & 3]);
          const T dot = (dp[0] + dp[1]) + (dp[2] + dp[3]);
          const T f = static_cast<T>(static_cast<double>(dot) * Bs[j]);
#pragma unroll
          for (int a = j; a < MAXM; ++a) y[a] = fma(-f, Vs[j][a], y[a]);
        }
      }
#pragma unroll
      for (int a = 0; a < MAXM; ++a)
        if (a < p) y[a] *= Sg[a];
    }
#pragma unroll
    for (int a = 0; a < MAXM; ++a)
      if (a < p) coef[r + static_cast<int64_t>(m + a) * s] = y[a];
  }
}


template <typename K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    MPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

template <typename T>
void hl_coeffs_t(int64_t s, int64_t m, int64_t p, const T* C, int64_t ldc, T* coef, T* scratch,
                 int* fallback, cudaStream_t st) {
  ProfScope prof("hl_coeffs", st, 0, 0);
  if (p > kMaxHlP) throw Error(MPEIG_E_CONFIG, "hl_update: block size above 256 not supported");
  if (m <= 16 && p <= 16) {
    k_hl_coeffs_warp<T, 16><<<1, kSmallThreads, 0, st>>>(static_cast<int>(s), static_cast<int>(m),
                                                        static_cast<int>(p), C, ldc, coef, fallback);
    MPB_LAUNCH_CHECK();
    return;
  }
  if constexpr (sizeof(T) == 4) {
    if (m <= 32 && p <= 32) {
      k_hl_coeffs_warp<T, 32><<<1, kSmallThreads, 0, st>>>(static_cast<int>(s), static_cast<int>(m),
                                                          static_cast<int>(p), C, ldc, coef, fallback);
      MPB_LAUNCH_CHECK();
      return;
    }
  }
  const size_t bytes = static_cast<size_t>(p * m + 2 * p * p + p) * sizeof(T);
  const int use = bytes <= kHlSmemCap;
  if (use) allow_smem(k_hl_coeffs<T>, bytes);
  // Q lands where the global-memory layout keeps it (scratch + p m + p p)
  T* qout = scratch + static_cast<int64_t>(p) * m + static_cast<int64_t>(p) * p;
  k_hl_coeffs<T><<<1, kSmallThreads, use ? bytes : 0, st>>>(
      static_cast<int>(s), static_cast<int>(m), static_cast<int>(p), C, ldc, coef, scratch,
      fallback, use, qout);
  MPB_LAUNCH_CHECK();
  k_hl_cpv<T><<<static_cast<unsigned>(ceil_div(s * p, 256)), 256, 0, st>>>(
      static_cast<int>(s), static_cast<int>(m), static_cast<int>(p), C, ldc, qout, coef, fallback);
  MPB_LAUNCH_CHECK();
}

}  // namespace

template <typename T>
void small_symmetrize(int64_t s, T* G, int64_t ldg, cudaStream_t st) {
  if (s <= 1) return;
  k_symmetrize<T><<<static_cast<unsigned>(ceil_div(s * s, 256) > 64 ? 64 : ceil_div(s * s, 256)), 256,
                    0, st>>>(s, G, ldg);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void small_cholesky_inv(int64_t m, const T* G, int64_t ldg, T* L, T* Uinv, int* status,
                        cudaStream_t st, T tau2) {
  if (m <= 0) return;
  ProfScope prof("small_chol", st, 0, 0);
  if ((m <= 16 || (sizeof(T) == 4 && m <= 32))) {
    if (m <= 16)
      k_cholesky_inv_warp<T, 16><<<1, 32, 0, st>>>(static_cast<int>(m), G, ldg, L, Uinv, status, tau2);
    else
      k_cholesky_inv_warp<T, 32><<<1, 32, 0, st>>>(static_cast<int>(m), G, ldg, L, Uinv, status, tau2);
    MPB_LAUNCH_CHECK();
    return;
  }
  const size_t bytes = static_cast<size_t>(2 * m * m) * sizeof(T);
  const int use = bytes <= kSmemCap;
  if (use) allow_smem(k_cholesky_inv<T>, bytes);
  k_cholesky_inv<T><<<1, kSmallThreads, use ? bytes : 0, st>>>(static_cast<int>(m), G, ldg, L, Uinv,
                                                               status, use, tau2);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void small_upper_inverse(int64_t m, const T* R, int64_t ldr, T* Rinv, int* status,
                         cudaStream_t st) {
  if (m <= 0) return;
  ProfScope prof("small_trinv", st, 0, 0);
  if ((m <= 16 || (sizeof(T) == 4 && m <= 32))) {
    if (m <= 16)
      k_upper_inverse_warp<T, 16><<<1, 32, 0, st>>>(static_cast<int>(m), R, ldr, Rinv, status);
    else
      k_upper_inverse_warp<T, 32><<<1, 32, 0, st>>>(static_cast<int>(m), R, ldr, Rinv, status);
    MPB_LAUNCH_CHECK();
    return;
  }
  const size_t bytes = static_cast<size_t>(2 * m * m + m) * sizeof(T);
  const int use = bytes <= kSmemCap;
  if (use) allow_smem(k_upper_inverse<T>, bytes);
  k_upper_inverse<T><<<1, kSmallThreads, use ? bytes : 0, st>>>(static_cast<int>(m), R, ldr, Rinv,
                                                                status, use);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void small_matmul(int64_t r, int64_t k, int64_t c, const T* A, int64_t lda, const T* B,
                  int64_t ldb, T* C, int64_t ldc, cudaStream_t st) {
  if (r * c <= 0) return;
  int64_t g = ceil_div(r * c, 256);
  if (g > 256) g = 256;
  k_small_matmul<T><<<static_cast<unsigned>(g), 256, 0, st>>>(
      static_cast<int>(r), static_cast<int>(k), static_cast<int>(c), A, lda, B, ldb, C, ldc);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void small_transpose(int64_t r, int64_t c, const T* A, int64_t lda, T* B, int64_t ldb,
                     cudaStream_t st) {
  if (r * c <= 0) return;
  int64_t g = ceil_div(r * c, 256);
  if (g > 256) g = 256;
  k_small_transpose<T><<<static_cast<unsigned>(g), 256, 0, st>>>(static_cast<int>(r),
                                                                 static_cast<int>(c), A, lda, B, ldb);
  MPB_LAUNCH_CHECK();
}

void hl_coeffs(int64_t s, int64_t m, int64_t p, const double* C, int64_t ldc, double* coef,
               double* scratch, int* fallback, cudaStream_t st) {
  hl_coeffs_t<double>(s, m, p, C, ldc, coef, scratch, fallback, st);
}

void hl_coeffs_f32(int64_t s, int64_t m, int64_t p, const float* C, int64_t ldc, float* coef,
                   float* scratch, int* fallback, cudaStream_t st) {
  hl_coeffs_t<float>(s, m, p, C, ldc, coef, scratch, fallback, st);
}

#define MPB_INST(T)                                                                            \
  template void small_symmetrize<T>(int64_t, T*, int64_t, cudaStream_t);                       \
  template void small_cholesky_inv<T>(int64_t, const T*, int64_t, T*, T*, int*, cudaStream_t, T); \
  template void small_upper_inverse<T>(int64_t, const T*, int64_t, T*, int*, cudaStream_t);    \
  template void small_matmul<T>(int64_t, int64_t, int64_t, const T*, int64_t, const T*,        \
                                int64_t, T*, int64_t, cudaStream_t);                            \
  template void small_transpose<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
