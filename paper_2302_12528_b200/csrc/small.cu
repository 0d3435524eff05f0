// small.cu -- single-CTA kernels for the small (<= 3m x 3m) dense steps.
//
// These run once or twice per iteration on matrices of order <= 576.  They
// are latency-bound, so each stages its matrices in shared memory (global
// scratch only when they do not fit) and keeps the reference's sequential
// inner-product order with separately rounded operations: for identical
// inputs they reproduce the reference's small factorizations
// (dense_cholesky, dense_kernels.hpp:128-152; householder_qr_square,
// ortho.hpp:30-121; matmul :20-34) bit for bit.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"
#include "rn.cuh"

namespace mpb {
namespace {

constexpr int kSmallThreads = 256;
constexpr size_t kSmemCap = 200 * 1024;
constexpr int kMaxHlP = 256;  // largest P block (block size m) of the HL update

template <typename T>
__global__ void k_symmetrize(int64_t s, T* G, int64_t ldg) {
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

// Left-looking Cholesky G = L L^T: column j after columns < j, rows of a
// column in parallel; then Uinv = L^{-T} by forward substitution (thread per
// column of L^{-1}).  status = {code, index}, first error wins.
template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
k_cholesky_inv(int m, const T* __restrict__ G, int64_t ldg, T* __restrict__ L,
               T* __restrict__ Uinv, int* status, int use_smem) {
  extern __shared__ __align__(16) unsigned char raw[];
  T* Ls = use_smem ? reinterpret_cast<T*>(raw) : L;
  T* Us = use_smem ? Ls + m * m : Uinv;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = 0;
  for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) Ls[idx] = T(0);
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (threadIdx.x == 0) {
      T s = G[j + static_cast<int64_t>(j) * ldg];
      for (int k = 0; k < j; ++k) {
        const T ljk = Ls[j + k * m];
        s = sub_rn(s, mul_rn(ljk, ljk));
      }
      if (!isfinite(static_cast<double>(s))) {
        fail = 1;
        if (status[0] == 0) {
          status[0] = MPEIG_E_OVERFLOW;
          status[1] = j;
        }
      } else if (!(s > T(0))) {
        fail = 1;
        if (status[0] == 0) {
          status[0] = MPEIG_E_NOT_PD;
          status[1] = j;
        }
      } else {
        Ls[j + j * m] = sqrt(s);
      }
    }
    __syncthreads();
    if (fail) return;
    const T djj = Ls[j + j * m];
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) {
      T s = G[i + static_cast<int64_t>(j) * ldg];
      for (int k = 0; k < j; ++k) s = sub_rn(s, mul_rn(Ls[i + k * m], Ls[j + k * m]));
      Ls[i + j * m] = s / djj;
    }
    __syncthreads();
  }
  if (Uinv) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      for (int k = 0; k < m; ++k) Us[c + k * m] = T(0);
      for (int k = c; k < m; ++k) {
        T s = (k == c) ? T(1) : T(0);
        for (int l = c; l < k; ++l) s = sub_rn(s, mul_rn(Ls[k + l * m], Us[c + l * m]));
        Us[c + k * m] = s / Ls[k + k * m];
      }
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      L[idx] = Ls[idx];
      if (Uinv) Uinv[idx] = Us[idx];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kSmallThreads)
k_upper_inverse(int m, const T* __restrict__ R, int64_t ldr, T* __restrict__ Rinv, int* status,
                int use_smem) {
  extern __shared__ __align__(16) unsigned char raw[];
  T* Rs = reinterpret_cast<T*>(raw);
  T* Is = use_smem ? Rs + m * m : Rinv;
  __shared__ int fail;
  if (use_smem)
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x)
      Rs[idx] = R[(idx % m) + static_cast<int64_t>(idx / m) * ldr];
  if (threadIdx.x == 0) {
    fail = 0;
    const T tiny = sizeof(T) == 8 ? T(DBL_MIN) : T(FLT_MIN);
    for (int j = 0; j < m; ++j) {
      const T a = fabs(R[j + static_cast<int64_t>(j) * ldr]);
      if (a == T(0) || a < tiny) {
        fail = 1;
        if (status[0] == 0) {
          status[0] = MPEIG_E_SINGULAR_TRI;
          status[1] = j;
        }
        break;
      }
    }
  }
  __syncthreads();
  if (fail) return;
  const T* Rr = use_smem ? Rs : R;
  const int64_t ld = use_smem ? m : ldr;
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    for (int k = c + 1; k < m; ++k) Is[k + c * m] = T(0);
    Is[c + c * m] = T(1) / Rr[c + c * ld];
    for (int k = c - 1; k >= 0; --k) {
      T s = T(0);
      for (int l = k + 1; l <= c; ++l) s = add_rn(s, mul_rn(Rr[k + l * ld], Is[l + c * m]));
      Is[k + c * m] = -s / Rr[k + k * ld];
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) Rinv[idx] = Is[idx];
  }
}

template <typename T>
__global__ void k_small_transpose(int r, int c, const T* __restrict__ A, int64_t lda,
                                  T* __restrict__ B, int64_t ldb) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       idx < static_cast<int64_t>(r) * c; idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(idx % r), j = static_cast<int>(idx / r);
    B[j + i * ldb] = A[i + j * lda];
  }
}

template <typename T>
__global__ void k_small_matmul(int r, int k, int c, const T* __restrict__ A, int64_t lda,
                               const T* __restrict__ B, int64_t ldb, T* __restrict__ C, int64_t ldc) {
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
            T* __restrict__ scratch, int* fallback, int use_smem) {
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
  // householder_reduce (ortho.hpp:30-76) on the p x m block, steps = p
  for (int j = 0; j < p; ++j) {
    const int len = p - j;
    if (tid == 0) {
      double nrm2 = 0.0;
      for (int i = j; i < p; ++i) {
        const double a = fabs(static_cast<double>(M[i + j * p]));
        nrm2 = add_rn(nrm2, mul_rn(a, a));
      }
      const double nrm = sqrt(nrm2);
      if (nrm == 0.0) {
        fb = 1;
      } else {
        const double x0 = static_cast<double>(M[j + j * p]);
        const double ax0 = fabs(x0);
        const double phase = ax0 > 0.0 ? x0 / ax0 : 1.0;
        T* v = V + j * p + j;
        v[0] = static_cast<T>(add_rn(x0, mul_rn(phase, nrm)));
        for (int i = 1; i < len; ++i) v[i] = M[j + i + j * p];
        double vn2 = 0.0;
        for (int i = 0; i < len; ++i) {
          const double a = fabs(static_cast<double>(v[i]));
          vn2 = add_rn(vn2, mul_rn(a, a));
        }
        sh_beta = 2.0 / vn2;
        beta[j] = sh_beta;
        sh_diag = static_cast<T>(-phase * nrm);  // R(j,j) after the reflection (ortho.hpp:72)
      }
    }
    __syncthreads();
    if (fb) break;
    const double b = sh_beta;
    const T* v = V + j * p + j;
    for (int c = j + tid; c < m; c += nt) {
      T* col = M + c * p + j;
      T sdot = T(0);
      for (int i = 0; i < len; ++i) sdot = add_rn(sdot, mul_rn(v[i], col[i]));
      sdot = static_cast<T>(mul_rn(static_cast<double>(sdot), b));
      for (int i = 0; i < len; ++i) col[i] = sub_rn(col[i], mul_rn(sdot, v[i]));
    }
    __syncthreads();
    if (tid == 0) {
      M[j + j * p] = sh_diag;
      for (int i = j + 1; i < p; ++i) M[i + j * p] = T(0);
    }
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
      for (int c = tid; c < p; c += nt) {
        T* qc = Q + c * p + (p - len);
        T sdot = T(0);
        for (int i = 0; i < len; ++i) sdot = add_rn(sdot, mul_rn(v[i], qc[i]));
        sdot = static_cast<T>(mul_rn(static_cast<double>(sdot), b));
        for (int i = 0; i < len; ++i) qc[i] = sub_rn(qc[i], mul_rn(sdot, v[i]));
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
  // c_pv = C(:, m:m+p) V  (V = I on fallback)
  for (int64_t idx = tid; idx < static_cast<int64_t>(s) * p; idx += nt) {
    const int i = static_cast<int>(idx % s), j = static_cast<int>(idx / s);
    T acc;
    if (fb) {
      acc = C[i + static_cast<int64_t>(m + j) * ldc];
    } else {
      // matmul(cp, Q): ascending l, separately rounded (dense_kernels.hpp:20-34)
      acc = T(0);
      for (int l = 0; l < p; ++l)
        acc = add_rn(acc, mul_rn(C[i + static_cast<int64_t>(m + l) * ldc], Q[l + j * p]));
    }
    coef[i + static_cast<int64_t>(m + j) * s] = acc;
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
  const size_t bytes = static_cast<size_t>(p * m + 2 * p * p + p) * sizeof(T);
  const int use = bytes <= kSmemCap;
  if (use) allow_smem(k_hl_coeffs<T>, bytes);
  k_hl_coeffs<T><<<1, kSmallThreads, use ? bytes : 0, st>>>(
      static_cast<int>(s), static_cast<int>(m), static_cast<int>(p), C, ldc, coef, scratch,
      fallback, use);
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
                        cudaStream_t st) {
  if (m <= 0) return;
  ProfScope prof("small_chol", st, 0, 0);
  const size_t bytes = static_cast<size_t>(2 * m * m) * sizeof(T);
  const int use = bytes <= kSmemCap;
  if (use) allow_smem(k_cholesky_inv<T>, bytes);
  k_cholesky_inv<T><<<1, kSmallThreads, use ? bytes : 0, st>>>(static_cast<int>(m), G, ldg, L, Uinv,
                                                               status, use);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void small_upper_inverse(int64_t m, const T* R, int64_t ldr, T* Rinv, int* status,
                         cudaStream_t st) {
  if (m <= 0) return;
  ProfScope prof("small_trinv", st, 0, 0);
  const size_t bytes = static_cast<size_t>(2 * m * m) * sizeof(T);
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
  template void small_cholesky_inv<T>(int64_t, const T*, int64_t, T*, T*, int*, cudaStream_t); \
  template void small_upper_inverse<T>(int64_t, const T*, int64_t, T*, int*, cudaStream_t);    \
  template void small_matmul<T>(int64_t, int64_t, int64_t, const T*, int64_t, const T*,        \
                                int64_t, T*, int64_t, cudaStream_t);                            \
  template void small_transpose<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
