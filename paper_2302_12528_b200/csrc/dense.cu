// dense.cu -- tall-skinny Gram products and block updates (fp64 / fp32).
//
// Shapes on the hot path: n rows (up to ~16.7M per GPU), k, c <= 3m <= 576.
//   gram    : G = A^T B      (adjoint_matmul, dense_kernels.hpp:36-52)
//   gemm_tn : Y = bZ + a A C (matmul, dense_kernels.hpp:20-34; subtract :54-62)
// Both are register-tiled (64 x 64 output tile per 256-thread CTA, 4 x 4 per
// thread) with shared-memory staged K panels.  The Gram splits n into a fixed
// number of chunks and reduces the partials in chunk order, so results are
// bitwise reproducible run to run (SURVEY §8e determinism).
#include "common.cuh"
#include "kernels.cuh"

namespace mpb {
namespace {

constexpr int kTile = 64;
constexpr int kGramBK = 32;
constexpr int kGemmBK = 16;
constexpr int kTargetCTAs = kNumSMs * 4;

struct GramPlan {
  int64_t tiles_m, tiles_n, nchunk, rows_per_chunk;
};

GramPlan gram_plan(int64_t n, int64_t ka, int64_t kb) {
  GramPlan p;
  p.tiles_m = ceil_div(ka, kTile);
  p.tiles_n = ceil_div(kb, kTile);
  const int64_t ntiles = p.tiles_m * p.tiles_n;
  int64_t nchunk = ceil_div(kTargetCTAs, ntiles);
  // >= 512 rows per chunk: the chunk partials are summed sequentially per entry
  const int64_t max_chunks = ceil_div(n, 512);
  if (nchunk > max_chunks) nchunk = max_chunks;
  if (nchunk < 1) nchunk = 1;
  p.rows_per_chunk = round_up(ceil_div(n, nchunk), kGramBK);
  if (p.rows_per_chunk < kGramBK) p.rows_per_chunk = kGramBK;
  p.nchunk = ceil_div(n, p.rows_per_chunk);
  if (p.nchunk < 1) p.nchunk = 1;
  return p;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gram_partial(int64_t n, int ka, int kb, const T* __restrict__ A, int64_t lda,
               const T* __restrict__ B, int64_t ldb, int64_t rows_per_chunk, int tiles_n,
               T* __restrict__ part) {
  __shared__ T As[kGramBK][kTile + 1];
  __shared__ T Bs[kGramBK][kTile + 1];
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * kTile, j0 = tn * kTile;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r_end = min(n, r_begin + rows_per_chunk);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);

  for (int64_t r0 = r_begin; r0 < r_end; r0 += kGramBK) {
#pragma unroll
    for (int e = threadIdx.x; e < kGramBK * kTile; e += 256) {
      const int r = e % kGramBK, c = e / kGramBK;
      const int64_t row = r0 + r;
      const bool rin = row < r_end;
      As[r][c] = (rin && i0 + c < ka) ? A[row + static_cast<int64_t>(i0 + c) * lda] : T(0);
      Bs[r][c] = (rin && j0 + c < kb) ? B[row + static_cast<int64_t>(j0 + c) * ldb] : T(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < kGramBK; ++r) {
      T av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[r][ty + 16 * q];
        bv[q] = Bs[r][tx + 16 * q];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  T* out = part + static_cast<int64_t>(blockIdx.y) * ka * kb;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i < ka && j < kb) out[i + static_cast<int64_t>(j) * ka] = acc[a][b];
    }
}

template <typename T>
__global__ void k_gram_reduce(int64_t nchunk, int ka, int kb, const T* __restrict__ part,
                              T* __restrict__ G, int64_t ldg, int sym) {
  const int64_t total = static_cast<int64_t>(ka) * kb;
  const int64_t stride = static_cast<int64_t>(ka) * kb;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(idx % ka), j = static_cast<int>(idx / ka);
    T s = T(0);
    for (int64_t c = 0; c < nchunk; ++c) s += part[c * stride + idx];
    if (sym) {
      T t = T(0);
      const int64_t tidx = j + static_cast<int64_t>(i) * ka;
      for (int64_t c = 0; c < nchunk; ++c) t += part[c * stride + tidx];
      s = (s + t) / T(2);
    }
    G[i + static_cast<int64_t>(j) * ldg] = s;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gemm_tn(int64_t n, int k, int c, T alpha, const T* __restrict__ A, int64_t lda,
          const T* __restrict__ Cm, int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y,
          int64_t ldy) {
  __shared__ T As[kGemmBK][kTile + 1];
  __shared__ T Cs[kGemmBK][kTile + 1];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int j0 = blockIdx.y * kTile;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);

  for (int l0 = 0; l0 < k; l0 += kGemmBK) {
#pragma unroll
    for (int e = threadIdx.x; e < kGemmBK * kTile; e += 256) {
      const int i = e % kTile, l = e / kTile;
      const int64_t row = i0 + i;
      As[l][i] = (row < n && l0 + l < k) ? A[row + static_cast<int64_t>(l0 + l) * lda] : T(0);
      const int lj = e % kGemmBK, jj = e / kGemmBK;
      Cs[lj][jj] = (l0 + lj < k && j0 + jj < c) ? Cm[(l0 + lj) + static_cast<int64_t>(j0 + jj) * ldc]
                                                : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < kGemmBK; ++l) {
      T av[4], cv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = As[l][tx + 16 * q];
        cv[q] = Cs[l][ty + 16 * q];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], cv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = j0 + ty + 16 * b;
    if (j >= c) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t i = i0 + tx + 16 * a;
      if (i >= n) continue;
      T v = alpha * acc[a][b];
      if (beta != T(0)) v = beta * Z[i + j * ldz] + v;
      Y[i + j * ldy] = v;
    }
  }
}

__global__ void k_f64_to_f32(int64_t n, int64_t c, const double* __restrict__ src, int64_t lds,
                             float* __restrict__ dst, int64_t ldd, int* overflow) {
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const double x = src[i + j * lds];
    const float y = __double2float_rn(x);
    if (isfinite(x) && !isfinite(y)) atomicExch(overflow, 1);
    dst[i + j * ldd] = y;
  }
}

__global__ void k_f32_to_f64(int64_t n, int64_t c, const float* __restrict__ src, int64_t lds,
                             double* __restrict__ dst, int64_t ldd) {
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    dst[i + j * ldd] = static_cast<double>(src[i + j * lds]);
  }
}

template <typename T>
__global__ void k_copy_block(int64_t n, int64_t c, const T* __restrict__ src, int64_t lds,
                             T* __restrict__ dst, int64_t ldd) {
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

template <typename T>
__global__ void k_scale(int64_t n, int64_t c, T alpha, const T* __restrict__ X, int64_t ldx,
                        T* __restrict__ Y, int64_t ldy) {
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    Y[i + j * ldy] = X[i + j * ldx] * alpha;
  }
}

template <typename T>
__global__ void k_frob_partial(int64_t n, int64_t c, const T* __restrict__ X, int64_t ldx,
                               double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0;
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    const double v = static_cast<double>(X[i + j * ldx]);
    acc = fma(v, v, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum_partials(int64_t np, const double* __restrict__ part, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0;
    for (int64_t i = 0; i < np; ++i) s += part[i];
    *out = s;
  }
}

int grid_for(int64_t total, int threads = 256, int64_t cap = kNumSMs * 8) {
  int64_t g = ceil_div(total, threads);
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

template <typename T>
int64_t gram_workspace_elems(int64_t n, int64_t ka, int64_t kb) {
  const GramPlan p = gram_plan(n, ka, kb);
  return p.nchunk * ka * kb;
}

template <typename T>
void gram(int64_t n, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B, int64_t ldb,
          T* G, int64_t ldg, int sym, T* work, cudaStream_t s) {
  if (ka <= 0 || kb <= 0) return;
  if (n <= 0) {
    for (int64_t j = 0; j < kb; ++j)
      MPB_CUDA(cudaMemsetAsync(G + j * ldg, 0, sizeof(T) * ka, s));
    return;
  }
  ProfScope prof("gram", s, double(sizeof(T)) * n * (A == B ? ka : ka + kb),
                 2.0 * n * ka * kb);
  const GramPlan p = gram_plan(n, ka, kb);
  dim3 grid(static_cast<unsigned>(p.tiles_m * p.tiles_n), static_cast<unsigned>(p.nchunk));
  k_gram_partial<T><<<grid, 256, 0, s>>>(n, static_cast<int>(ka), static_cast<int>(kb), A, lda, B,
                                         ldb, p.rows_per_chunk, static_cast<int>(p.tiles_n), work);
  MPB_LAUNCH_CHECK();
  k_gram_reduce<T><<<grid_for(ka * kb), 256, 0, s>>>(p.nchunk, static_cast<int>(ka),
                                                     static_cast<int>(kb), work, G, ldg, sym);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void gemm_tn(int64_t n, int64_t k, int64_t c, T alpha, const T* A, int64_t lda, const T* C,
             int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y, int64_t ldy, cudaStream_t s) {
  if (n <= 0 || c <= 0) return;
  if (k <= 0) {
    // Y = beta Z
    if (beta == T(0)) {
      for (int64_t j = 0; j < c; ++j) MPB_CUDA(cudaMemsetAsync(Y + j * ldy, 0, sizeof(T) * n, s));
    } else if (Y != Z) {
      copy_block<T>(n, c, Z, ldz, Y, ldy, s);
    }
    return;
  }
  ProfScope prof("gemm", s, double(sizeof(T)) * n * (k + (beta != T(0) ? 2 : 1) * c),
                 2.0 * n * k * c);
  dim3 grid(static_cast<unsigned>(ceil_div(n, kTile)), static_cast<unsigned>(ceil_div(c, kTile)));
  k_gemm_tn<T><<<grid, 256, 0, s>>>(n, static_cast<int>(k), static_cast<int>(c), alpha, A, lda, C,
                                    ldc, beta, Z, ldz, Y, ldy);
  MPB_LAUNCH_CHECK();
}

void convert_f64_to_f32(int64_t n, int64_t c, const double* src, int64_t lds, float* dst,
                        int64_t ldd, int* overflow_flag, cudaStream_t s) {
  if (n * c <= 0) return;
  k_f64_to_f32<<<grid_for(n * c), 256, 0, s>>>(n, c, src, lds, dst, ldd, overflow_flag);
  MPB_LAUNCH_CHECK();
}

void convert_f32_to_f64(int64_t n, int64_t c, const float* src, int64_t lds, double* dst,
                        int64_t ldd, cudaStream_t s) {
  if (n * c <= 0) return;
  k_f32_to_f64<<<grid_for(n * c), 256, 0, s>>>(n, c, src, lds, dst, ldd);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void copy_block(int64_t n, int64_t c, const T* src, int64_t lds, T* dst, int64_t ldd,
                cudaStream_t s) {
  if (n * c <= 0 || src == dst) return;
  if (lds == n && ldd == n) {
    MPB_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n * c, cudaMemcpyDeviceToDevice, s));
    return;
  }
  MPB_CUDA(cudaMemcpy2DAsync(dst, sizeof(T) * ldd, src, sizeof(T) * lds, sizeof(T) * n, c,
                             cudaMemcpyDeviceToDevice, s));
}

template <typename T>
void scale_block(int64_t n, int64_t c, T alpha, const T* X, int64_t ldx, T* Y, int64_t ldy,
                 cudaStream_t s) {
  if (n * c <= 0) return;
  k_scale<T><<<grid_for(n * c), 256, 0, s>>>(n, c, alpha, X, ldx, Y, ldy);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void frob_sq(int64_t n, int64_t c, const T* X, int64_t ldx, double* out, double* work,
             cudaStream_t s) {
  const int g = grid_for(n * c, 256, kNumSMs * 2);
  k_frob_partial<T><<<g, 256, 0, s>>>(n, c, X, ldx, work);
  MPB_LAUNCH_CHECK();
  k_sum_partials<<<1, 32, 0, s>>>(g, work, out);
  MPB_LAUNCH_CHECK();
}

#define MPB_INST(T)                                                                            \
  template int64_t gram_workspace_elems<T>(int64_t, int64_t, int64_t);                         \
  template void gram<T>(int64_t, int64_t, const T*, int64_t, int64_t, const T*, int64_t, T*,   \
                        int64_t, int, T*, cudaStream_t);                                        \
  template void gemm_tn<T>(int64_t, int64_t, int64_t, T, const T*, int64_t, const T*, int64_t, \
                           T, const T*, int64_t, T*, int64_t, cudaStream_t);                    \
  template void copy_block<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t); \
  template void frob_sq<T>(int64_t, int64_t, const T*, int64_t, double*, double*, cudaStream_t); \
  template void scale_block<T>(int64_t, int64_t, T, const T*, int64_t, T*, int64_t, cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
