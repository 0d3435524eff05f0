// resid.cu -- fused residual / column norms / f_T kernel (K2) and helpers.
//
// One HBM pass over X and AX produces, per column j:
//   R(:,j) = AX(:,j) - theta_j X(:,j)          residual_block (eigensolvers.hpp:104-115)
//   ||R(:,j)||, ||X(:,j)||                     col_norm (dense_matrix.hpp:74-82) used by
//                                              converged_count / make_record (:25-43,:117-129)
//   W(:,j) = f_T(R(:,j))                       Preconditioner::apply (precond.hpp:92-100)
// with f_T = Jacobi; in the sandwich mode R is narrowed to fp32 (to_lower,
// precision.hpp:102-107, overflow flagged), scaled in fp32 and widened back
// (to_working, :113-117), so R never exists in HBM.  The elementwise
// arithmetic is explicitly rounded -> bitwise equal to the reference's.
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "rn.cuh"

namespace mpb {
namespace {

constexpr int kColGroup = 2;  // columns per CTA: 8 -> 2 took n = 2M, m = 80 from 3.97 to 6.16 TB/s
                              // (fewer concurrent column streams per CTA, more CTAs)
constexpr int kThreads = 256;

struct ResidPlan {
  int64_t nchunk, rows_per_chunk;
};

ResidPlan resid_plan(int64_t n, int64_t m) {
  const int64_t groups = ceil_div(m, kColGroup);
  int64_t nchunk = ceil_div(static_cast<int64_t>(kNumSMs) * 8, groups);
  const int64_t maxc = ceil_div(n, 2 * kThreads);  // >= 512 rows per chunk
  if (nchunk > maxc) nchunk = maxc;
  if (nchunk < 1) nchunk = 1;
  ResidPlan p;
  p.rows_per_chunk = round_up(ceil_div(n, nchunk), kThreads);
  p.nchunk = ceil_div(n, p.rows_per_chunk);
  if (p.nchunk < 1) p.nchunk = 1;
  return p;
}

template <typename T, int MODE>
__device__ __forceinline__ T apply_ft(T r, const void* dinv, int64_t i, int* overflow) {
  if constexpr (MODE == kResidPlain) {
    return r;
  } else if constexpr (MODE == kResidJacobiT) {
    return mul_rn(r, static_cast<const T*>(dinv)[i]);
  } else {
    const float rl = __double2float_rn(static_cast<double>(r));
    if (isfinite(static_cast<double>(r)) && !isfinite(rl)) *overflow = 1;
    const float wl = __fmul_rn(rl, static_cast<const float*>(dinv)[i]);
    return static_cast<T>(wl);
  }
}

template <typename T, int MODE, bool VEC>
__global__ void __launch_bounds__(kThreads)
k_residual(int64_t n, int m, const T* __restrict__ X, int64_t ldx, const T* __restrict__ AX,
           int64_t ldax, const T* __restrict__ theta, const void* __restrict__ dinv,
           T* __restrict__ W, int64_t ldw, int64_t rows_per_chunk, double* __restrict__ part,
           int* overflow) {
  MPB_PDL_WAIT();
  // norms accumulate in real_t<T> like DenseMatrix<T>::col_norm
  // (dense_matrix.hpp:74-82): fp32 sums in the fp32 stage, fp64 otherwise
  using Acc = T;
  __shared__ Acc red[kThreads / 32][2 * kColGroup];
  const int j0 = blockIdx.y * kColGroup;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.x) * rows_per_chunk;
  const int64_t r_end = min(n, r_begin + rows_per_chunk);
  Acc rr[kColGroup], xx[kColGroup];
  T th[kColGroup];
#pragma unroll
  for (int q = 0; q < kColGroup; ++q) {
    rr[q] = 0;
    xx[q] = 0;
    th[q] = (j0 + q < m) ? theta[j0 + q] : T(0);
  }
  int ovf = 0;
  // two consecutive rows per thread with 2-wide loads / stores (rows are
  // contiguous per column; chunks start at multiples of 256 rows, ld % 32 == 0)
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  constexpr int kStep = VEC ? 2 : 1;
  for (int64_t i = r_begin + kStep * threadIdx.x; i < r_end; i += kStep * kThreads) {
    const bool pair = VEC && i + 1 < r_end;
#pragma unroll
    for (int q = 0; q < kColGroup; ++q) {
      const int j = j0 + q;
      if (j < m) {
        T x0, x1 = T(0), a0, a1 = T(0);
        if (pair) {
          const V2 xv = *reinterpret_cast<const V2*>(X + i + j * ldx);
          const V2 av = *reinterpret_cast<const V2*>(AX + i + j * ldax);
          x0 = xv.x;
          x1 = xv.y;
          a0 = av.x;
          a1 = av.y;
        } else {
          x0 = X[i + j * ldx];
          a0 = AX[i + j * ldax];
        }
        const T r0 = sub_rn(a0, mul_rn(th[q], x0));
        const T r1 = sub_rn(a1, mul_rn(th[q], x1));
        rr[q] = fma(static_cast<Acc>(r0), static_cast<Acc>(r0), rr[q]);
        xx[q] = fma(static_cast<Acc>(x0), static_cast<Acc>(x0), xx[q]);
        if (pair) {
          rr[q] = fma(static_cast<Acc>(r1), static_cast<Acc>(r1), rr[q]);
          xx[q] = fma(static_cast<Acc>(x1), static_cast<Acc>(x1), xx[q]);
        }
        if (W) {
          const T w0 = apply_ft<T, MODE>(r0, dinv, i, &ovf);
          if (pair) {
            V2 wv;
            wv.x = w0;
            wv.y = apply_ft<T, MODE>(r1, dinv, i + 1, &ovf);
            *reinterpret_cast<V2*>(W + i + j * ldw) = wv;
          } else {
            W[i + j * ldw] = w0;
          }
        }
      }
    }
  }
  if (ovf) atomicExch(overflow, 1);
  // block reduction of the 2*kColGroup sums, fixed order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kColGroup; ++q) {
    Acc a = rr[q], b = xx[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, off);
      b += __shfl_down_sync(0xffffffffu, b, off);
    }
    if (lane == 0) {
      red[warp][q] = a;
      red[warp][kColGroup + q] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * kColGroup) {
    Acc s = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s += red[w][threadIdx.x];
    const int q = threadIdx.x % kColGroup;
    const int which = threadIdx.x / kColGroup;  // 0: r, 1: x
    const int j = j0 + q;
    if (j < m) part[(static_cast<int64_t>(blockIdx.x) * m + j) * 2 + which] = s;
  }
}

// a warp per (column, r|x): lanes take chunks lane, lane+32, ... in order,
// then a fixed xor tree -> deterministic
template <typename Acc>
__global__ void k_resid_norms(int64_t nchunk, int m, const double* __restrict__ part,
                              double* __restrict__ rnorm, double* __restrict__ xnorm, int raw) {
  MPB_PDL_WAIT();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= 2 * m) return;
  const int j = t >> 1, which = t & 1;
  Acc s = 0;
  for (int64_t c = lane; c < nchunk; c += 32) s += static_cast<Acc>(part[(c * m + j) * 2 + which]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) (which ? xnorm : rnorm)[j] = raw ? static_cast<double>(s) : static_cast<double>(sqrt(s));
}

// sqrt in real_t<T> after the row-sharded sums were allreduced
template <typename Acc>
__global__ void k_norms_sqrt(int64_t count, double* __restrict__ v) {
  MPB_PDL_WAIT();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < count) v[i] = static_cast<double>(sqrt(static_cast<Acc>(v[i])));
}

template <typename T, int MODE>
__global__ void k_jacobi(int64_t n, int64_t c, const T* __restrict__ R, int64_t ldr,
                         const void* __restrict__ dinv, T* __restrict__ W, int64_t ldw,
                         int* overflow) {
  MPB_PDL_WAIT();
  int ovf = 0;
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    W[i + j * ldw] = apply_ft<T, MODE>(R[i + j * ldr], dinv, i, &ovf);
  }
  if (ovf) atomicExch(overflow, 1);
}

template <typename T>
__global__ void k_subtract(int64_t n, int64_t c, const T* __restrict__ X, int64_t ldx,
                           const T* __restrict__ W, int64_t ldw, T* __restrict__ Y,
                           int64_t ldy) {
  MPB_PDL_WAIT();
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    Y[i + j * ldy] = sub_rn(X[i + j * ldx], W[i + j * ldw]);
  }
}

int ew_grid(int64_t total) {
  int64_t g = ceil_div(total, 256);
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

template <typename T, int MODE, typename... Args>
void launch_resid(bool vec, dim3 grid, cudaStream_t s, Args... args) {
  if (vec)
    k_residual<T, MODE, true><<<grid, kThreads, 0, s>>>(args...);
  else
    k_residual<T, MODE, false><<<grid, kThreads, 0, s>>>(args...);
}

int64_t resid_workspace_elems(int64_t n, int64_t m) {
  return resid_plan(n, m).nchunk * m * 2;
}

template <typename T>
void residual_precond(int mode, int64_t n, int64_t m, const T* X, int64_t ldx, const T* AX,
                      int64_t ldax, const T* theta, const void* dinv, T* W, int64_t ldw,
                      double* rnorm, double* xnorm, int* overflow_flag, double* work,
                      cudaStream_t s, int raw_sums) {
  if (m <= 0) return;
  ProfScope prof("residual_ft", s, double(sizeof(T)) * n * m * (W ? 3 : 2), 6.0 * n * m);
  const ResidPlan p = resid_plan(n, m);
  dim3 grid(static_cast<unsigned>(p.nchunk), static_cast<unsigned>(ceil_div(m, kColGroup)));
  const size_t al = 2 * sizeof(T);
  const bool vec = ldx % 2 == 0 && ldax % 2 == 0 && (W == nullptr || ldw % 2 == 0) &&
                   reinterpret_cast<uintptr_t>(X) % al == 0 &&
                   reinterpret_cast<uintptr_t>(AX) % al == 0 &&
                   reinterpret_cast<uintptr_t>(W) % al == 0;
  const int mi = static_cast<int>(m);
  switch (mode) {
    case kResidPlain:
      launch_resid<T, kResidPlain>(vec, grid, s, n, mi, X, ldx, AX, ldax, theta, dinv, W,
                                                           ldw, p.rows_per_chunk, work, overflow_flag);
      break;
    case kResidJacobiT:
      launch_resid<T, kResidJacobiT>(vec, grid, s, 
          n, mi, X, ldx, AX, ldax, theta, dinv, W, ldw, p.rows_per_chunk, work, overflow_flag);
      break;
    default:
      if constexpr (sizeof(T) == 8) {
        launch_resid<T, kResidSandwich>(vec, grid, s, 
            n, mi, X, ldx, AX, ldax, theta, dinv, W, ldw, p.rows_per_chunk, work, overflow_flag);
      } else {
        throw Error(MPEIG_E_CONFIG, "sandwich f_T needs a working-precision block");
      }
  }
  MPB_LAUNCH_CHECK();
  k_resid_norms<T><<<static_cast<unsigned>(ceil_div(2 * m, 4)), 128, 0, s>>>(p.nchunk, mi, work,
                                                                          rnorm, xnorm, raw_sums);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void norms_sqrt(int64_t count, double* v, cudaStream_t s) {
  if (count <= 0) return;
  k_norms_sqrt<T><<<static_cast<unsigned>(ceil_div(count, 128)), 128, 0, s>>>(count, v);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void jacobi_apply(int mode, int64_t n, int64_t c, const T* R, int64_t ldr, const void* dinv, T* W,
                  int64_t ldw, int* overflow_flag, cudaStream_t s) {
  if (n * c <= 0) return;
  if (mode == kResidJacobiT) {
    k_jacobi<T, kResidJacobiT><<<ew_grid(n * c), 256, 0, s>>>(n, c, R, ldr, dinv, W, ldw,
                                                               overflow_flag);
  } else if (mode == kResidSandwich) {
    if constexpr (sizeof(T) == 8) {
      k_jacobi<T, kResidSandwich><<<ew_grid(n * c), 256, 0, s>>>(n, c, R, ldr, dinv, W, ldw,
                                                                  overflow_flag);
    } else {
      throw Error(MPEIG_E_CONFIG, "sandwich f_T needs a working-precision block");
    }
  } else {
    copy_block<T>(n, c, R, ldr, W, ldw, s);
    return;
  }
  MPB_LAUNCH_CHECK();
}

template <typename T>
void subtract(int64_t n, int64_t c, const T* X, int64_t ldx, const T* W, int64_t ldw, T* Y,
              int64_t ldy, cudaStream_t s) {
  if (n * c <= 0) return;
  k_subtract<T><<<ew_grid(n * c), 256, 0, s>>>(n, c, X, ldx, W, ldw, Y, ldy);
  MPB_LAUNCH_CHECK();
}

#define MPB_INST(T)                                                                             \
  template void residual_precond<T>(int, int64_t, int64_t, const T*, int64_t, const T*, int64_t, \
                                    const T*, const void*, T*, int64_t, double*, double*, int*,  \
                                    double*, cudaStream_t, int);                                 \
  template void norms_sqrt<T>(int64_t, double*, cudaStream_t);                                  \
  template void jacobi_apply<T>(int, int64_t, int64_t, const T*, int64_t, const void*, T*,       \
                                int64_t, int*, cudaStream_t);                                    \
  template void subtract<T>(int64_t, int64_t, const T*, int64_t, const T*, int64_t, T*, int64_t, \
                            cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
