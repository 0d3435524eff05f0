// dense.cu -- tall-skinny Gram products and block updates (fp64 / fp32).
//
// Shapes on the hot path: n rows (up to ~16.7M per GPU), k, c <= 3m <= 576.
//   gram    : G = A^T B      (adjoint_matmul, dense_kernels.hpp:36-52)
//   gemm_tn : Y = bZ + a A C (matmul, dense_kernels.hpp:20-34; subtract :54-62)
// Both are register-tiled (64 x 64 output tile per 256-thread CTA, 4 x 4 per
// thread) with shared-memory staged K panels.  The Gram splits n into a fixed
// number of chunks and reduces the partials in chunk order, so results are
// bitwise reproducible run to run (SURVEY §8e determinism).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "smallwarp.cuh"

namespace mpb {
namespace {

constexpr int kTile = 64;
constexpr int kGramBK = 32;
constexpr int kGemmBK = 16;

// ---- Gram G = A^T B ---------------------------------------------------------
// One CTA per (output tile, row chunk) writes its chunk's partial product; a
// second kernel combines the partials GPU-wide in a fixed order (bitwise
// reproducible) and hermitizes.  The output tile is 16*MT square (MT = 1..4)
// so that narrow blocks (k = 16, 32, 48) waste no MMA / FMA work on padding.

template <typename T>
constexpr int64_t kGramHead = 16 / sizeof(T);  // elements before the partials

struct GramPlan {
  int mt;  // output tile = 16 * mt
  int64_t tiles_m, tiles_n, nchunk, rows_per_chunk, level_elems;
};

GramPlan gram_plan(int64_t n, int64_t ka, int64_t kb) {
  GramPlan p;
  const int64_t kmax = std::max(ka, kb);
  if (kmax <= 64) {
    p.mt = kmax <= 16 ? 1 : kmax <= 32 ? 2 : kmax <= 48 ? 3 : 4;  // one tile
  } else {
    // wide Grams: the 16*mt tile (mt = 3..5) that wastes the least MMA work on
    // padding -- 240 = 3 x 80, 160 x 80 = 2 x 1 x 80, 144 = 3 x 48 -- ties to
    // the larger tile (fewer re-reads of the tall operands)
    int64_t best = -1;
    for (int mt = 5; mt >= 3; --mt) {
      const int64_t t = 16 * mt;
      const int64_t area = ceil_div(ka, t) * ceil_div(kb, t) * t * t;
      if (best < 0 || area < best) {
        best = area;
        p.mt = mt;
      }
    }
  }
  const int64_t tile = 16 * p.mt;
  p.tiles_m = ceil_div(ka, tile);
  p.tiles_n = ceil_div(kb, tile);
  // one wave: a single-tile Gram uses one CTA per SM (two reduction levels),
  // multi-tile Grams two CTAs per SM
  int64_t nchunk = kNumSMs;  // combine_body's unrolled loads assume nchunk <= kNumSMs
  const int64_t max_chunks = ceil_div(n, 64);  // >= 64 rows per chunk
  if (nchunk > max_chunks) nchunk = max_chunks;
  if (nchunk < 1) nchunk = 1;
  p.rows_per_chunk = round_up(ceil_div(n, nchunk), kGramBK);
  p.nchunk = ceil_div(n, p.rows_per_chunk);
  if (p.nchunk < 1) p.nchunk = 1;
  // chunk partials, combined by k_gram_combine
  p.level_elems = p.nchunk * ka * kb;
  return p;
}

// the SIMT kernel's tiles (TM <= 4): the single-tile policy up to 64, then 64
GramPlan gram_plan_simt(int64_t n, int64_t ka, int64_t kb) {
  GramPlan p = gram_plan(n, std::min<int64_t>(ka, 64), std::min<int64_t>(kb, 64));
  p.mt = 4;
  p.tiles_m = ceil_div(ka, 64);
  p.tiles_n = ceil_div(kb, 64);
  p.level_elems = p.nchunk * ka * kb;
  return p;
}

template <typename T>
__device__ __forceinline__ void combine_body(int64_t nchunk, int ka, int kb,
                                             const T* __restrict__ part, T* __restrict__ G,
                                             int64_t ldg, int sym) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t tot = static_cast<int64_t>(ka) * kb;
  int i, j;
  if (sym) {
    // pair index w -> (i <= j), column-major over the upper triangle
    if (w >= static_cast<int64_t>(ka) * (ka + 1) / 2) return;
    j = static_cast<int>((sqrt(8.0 * static_cast<double>(w) + 1.0) - 1.0) / 2.0);
    while ((static_cast<int64_t>(j) + 1) * (j + 2) / 2 <= w) ++j;
    while (static_cast<int64_t>(j) * (j + 1) / 2 > w) --j;
    i = static_cast<int>(w - static_cast<int64_t>(j) * (j + 1) / 2);
  } else {
    if (w >= tot) return;
    i = static_cast<int>(w % ka);
    j = static_cast<int>(w / ka);
  }
  const int64_t o1 = i + static_cast<int64_t>(j) * ka, o2 = j + static_cast<int64_t>(i) * ka;
  T a = T(0), b = T(0);
  // nchunk <= kNumSMs: every lane's chunk loads issued before the (ordered) sums
  constexpr int kPer = (kNumSMs + 31) / 32;
  T va[kPer], vb[kPer];
#pragma unroll
  for (int t = 0; t < kPer; ++t) {
    const int64_t c = lane + 32 * t;
    va[t] = c < nchunk ? __ldg(part + c * tot + o1) : T(0);
    vb[t] = (sym && c < nchunk) ? __ldg(part + c * tot + o2) : T(0);
  }
#pragma unroll
  for (int t = 0; t < kPer; ++t) {
    a += va[t];
    b += vb[t];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if (lane == 0) {
    if (sym) {
      const T v = (a + b) / T(2);
      G[i + static_cast<int64_t>(j) * ldg] = v;
      G[j + static_cast<int64_t>(i) * ldg] = v;
    } else {
      G[i + static_cast<int64_t>(j) * ldg] = a;
    }
  }
}

// Deterministic combine of the chunk partials, spread over the whole GPU: a
// warp per output entry (per symmetric pair when hermitizing), lanes sum
// chunks lane, lane+32, ... in order, then a fixed xor tree.  G = sum, or
// G(i,j) = G(j,i) = (sum_ij + sum_ji) / 2 (hermitize, eigensolvers.hpp:302-308).
//
// chol != 0 (CholQR, ka = kb <= 16): the last CTA to finish (ticket) also
// factors G = L L^T and forms L^{-T} (warp_cholesky_inv), saving the
// separate small-kernel launch of the reference's cholesky_qr step.
template <typename T>
__global__ void __launch_bounds__(256)
k_gram_combine(int64_t nchunk, int ka, int kb, const T* __restrict__ part, T* __restrict__ G,
               int64_t ldg, int sym, int* __restrict__ ticket, T* __restrict__ L,
               T* __restrict__ Uinv, int* status, T tau2) {
  MPB_PDL_WAIT();
  combine_body(nchunk, ka, kb, part, G, ldg, sym);
  if (!ticket) return;
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    s_last = atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1;
    if (s_last) *ticket = 0;  // ready for the next call / graph replay
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if ((threadIdx.x >> 5) == 0 && *reinterpret_cast<volatile int*>(status) == 0)
    warp_cholesky_inv<T, 16>(ka, G, ldg, L, Uinv, status, tau2);
}


// SIMT Gram (fp32, and fp64 operands that are not 16-B aligned): 256 threads
// as 16 x 16, TM x TM outputs per thread, 32-row panels staged through
// registers so the next panel's loads overlap this one's FMAs.
template <typename T, int TM>
__global__ void __launch_bounds__(256)
k_gram_partial(int64_t n, int ka, int kb, const T* __restrict__ A, int64_t lda,
               const T* __restrict__ B, int64_t ldb, int64_t rows_per_chunk, int tiles_n,
               int64_t nchunk, T* __restrict__ part, int* __restrict__ ctr, T* G, int64_t ldg,
               int sym) {
  MPB_PDL_WAIT();
  constexpr int TILE = 16 * TM;
  constexpr int kSm = 2 * kGramBK * (TILE + 1) > TILE * TILE ? 2 * kGramBK * (TILE + 1) : TILE * TILE;
  __shared__ T sm[kSm];
  auto As = reinterpret_cast<T(*)[TILE + 1]>(sm);
  auto Bs = reinterpret_cast<T(*)[TILE + 1]>(sm + kGramBK * (TILE + 1));
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * TILE, j0 = tn * TILE;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r_end = min(n, r_begin + rows_per_chunk);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[TM][TM];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TM; ++b) acc[a][b] = T(0);

  constexpr int kPer = kGramBK * TILE / 256;
  T ra[kPer], rb[kPer];
  auto fetch = [&](int64_t r0) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + 256 * t;
      const int r = e % kGramBK, c = e / kGramBK;
      const int64_t row = r0 + r;
      const bool rin = row < r_end;
      ra[t] = (rin && i0 + c < ka) ? __ldg(A + row + static_cast<int64_t>(i0 + c) * lda) : T(0);
      rb[t] = (rin && j0 + c < kb) ? __ldg(B + row + static_cast<int64_t>(j0 + c) * ldb) : T(0);
    }
  };
  if (r_begin < r_end) fetch(r_begin);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kGramBK) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = threadIdx.x + 256 * t;
      As[e % kGramBK][e / kGramBK] = ra[t];
      Bs[e % kGramBK][e / kGramBK] = rb[t];
    }
    __syncthreads();
    if (r0 + kGramBK < r_end) fetch(r0 + kGramBK);
#pragma unroll 8
    for (int r = 0; r < kGramBK; ++r) {
      T av[TM], bv[TM];
#pragma unroll
      for (int q = 0; q < TM; ++q) {
        av[q] = As[r][ty + 16 * q];
        bv[q] = Bs[r][tx + 16 * q];
      }
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TM; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  const bool direct = nchunk == 1 && !sym;
  T* out = direct ? G : part + static_cast<int64_t>(blockIdx.y) * ka * kb;
  const int64_t ldo = direct ? ldg : ka;
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TM; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i < ka && j < kb) out[i + static_cast<int64_t>(j) * ldo] = acc[a][b];
    }
}

// ---- fp64 tensor-core (DMMA) Gram -------------------------------------------
// mma.sync.m8n8k4.f64: the legacy fp64 tensor path (tcgen05 has no f64 kind).
// CTA = 4 warps (2 x 2), output tile 16*MT, each warp (8 MT)^2 = MT x MT MMA
// tiles; K (= the row dimension n) streamed in 16-row panels through a
// kGramStages-deep cp.async ring.  Column-major panels are copied verbatim
// (16-B chunks of contiguous rows); the smem row pitch 20 (doubles) makes the
// fragment reads 2-way (the minimum for 8-B lanes).
constexpr int kDBK = 16;
constexpr int kDPitch = kDBK + 4;
constexpr int kGramStages = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Load a 16-row x TILE-column panel of a column-major matrix (rows r0..,
// cols c0..) into smem [col][row]; out-of-range rows/cols are zero-filled.
template <int TILE>
__device__ __forceinline__ void load_panel(double (*dst)[kDPitch], const double* __restrict__ M,
                                           int64_t ld, int64_t r0, int64_t r_end, int c0, int ncols) {
  // TILE cols x 8 chunks of 2 doubles, 128 threads
#pragma unroll
  for (int t = 0; t < TILE / 16; ++t) {
    const int e = threadIdx.x + 128 * t;
    const int col = e >> 3, ch = e & 7;
    const int64_t row = r0 + 2 * ch;
    const bool cin = c0 + col < ncols;
    int bytes = 0;
    if (cin && row < r_end) bytes = row + 1 < r_end ? 16 : 8;
    const double* src = bytes ? M + row + static_cast<int64_t>(c0 + col) * ld : M;
    cp_async16(&dst[col][2 * ch], src, bytes);
  }
}

template <int MT>
constexpr size_t gram_dmma_smem() {
  constexpr size_t ring = sizeof(double) * 2 * kGramStages * (16 * MT) * kDPitch;
  constexpr size_t scratch = sizeof(double) * (16 * MT) * (16 * MT);
  return ring > scratch ? ring : scratch;
}

template <int MT>
__global__ void __launch_bounds__(128)
k_gram_dmma(int64_t n, int ka, int kb, const double* __restrict__ A, int64_t lda,
            const double* __restrict__ B, int64_t ldb, int64_t rows_per_chunk, int tiles_n,
            int64_t nchunk, double* __restrict__ part, int* __restrict__ ctr, double* G,
            int64_t ldg, int sym) {
  MPB_PDL_WAIT();
  constexpr int TILE = 16 * MT;
  extern __shared__ __align__(16) unsigned char gsm[];
  auto As = reinterpret_cast<double(*)[TILE][kDPitch]>(gsm);
  auto Bs = As + kGramStages;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * TILE, j0 = tn * TILE;
  const int64_t r_begin = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r_end = min(n, r_begin + rows_per_chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 8 * MT, wn = (warp & 1) * 8 * MT;
  double acc[MT][MT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < MT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // kGramStages-deep cp.async ring: stages-1 panels in flight ahead of the MMA
  const int npanel = static_cast<int>((r_end - r_begin + kDBK - 1) / kDBK);
#pragma unroll
  for (int q = 0; q < kGramStages - 1; ++q) {
    if (q < npanel) {
      const int64_t r1 = r_begin + static_cast<int64_t>(q) * kDBK;
      load_panel<TILE>(As[q], A, lda, r1, r_end, i0, ka);
      load_panel<TILE>(Bs[q], B, ldb, r1, r_end, j0, kb);
    }
    cp_async_commit();
  }
  for (int p = 0; p < npanel; ++p) {
    const int buf = p % kGramStages;
    cp_async_wait<kGramStages - 2>();
    __syncthreads();
    {
      const int q = p + kGramStages - 1;
      if (q < npanel) {
        const int64_t r1 = r_begin + static_cast<int64_t>(q) * kDBK;
        load_panel<TILE>(As[q % kGramStages], A, lda, r1, r_end, i0, ka);
        load_panel<TILE>(Bs[q % kGramStages], B, ldb, r1, r_end, j0, kb);
      }
      cp_async_commit();
    }
#pragma unroll
    for (int kk = 0; kk < kDBK; kk += 4) {
      double af[MT], bf[MT];
#pragma unroll
      for (int q = 0; q < MT; ++q) {
        af[q] = As[buf][wm + 8 * q + g][kk + t4];
        bf[q] = Bs[buf][wn + 8 * q + g][kk + t4];
      }
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < MT; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  const bool direct = nchunk == 1 && !sym;
  double* out = direct ? G : part + static_cast<int64_t>(blockIdx.y) * ka * kb;
  const int64_t ldo = direct ? ldg : ka;
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < MT; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + wm + 8 * a + g, j = j0 + wn + 8 * b + 2 * t4 + h;
        if (i < ka && j < kb) out[i + static_cast<int64_t>(j) * ldo] = acc[a][b][h];
      }
}

// ---- fp64 tensor-core (DMMA) block update Y = beta Z + alpha A C ------------
// A: n x k column-major (the tall operand), C: k x c (small).  CTA = 4 warps
// (2 x 2), 64 rows x 16*NT columns of Y (NT = 1..4 sized to c), each warp
// 32 x 8*NT; K in 16-wide panels through a cp.async ring, 4 stages for the
// k <= 64 products of the hot path every load is in flight at once (deep
// K uses a 2-stage ring: less shared memory, more CTAs per SM).  A panel
// smem layout [k][row] with pitch 72 (fragment reads 2-way), C panel [col][k]
// with pitch 20.
constexpr int kAPitch = kTile + 8;
template <int NT, int kGemmStages>
__global__ void __launch_bounds__(128)
k_gemm_dmma(int64_t n, int k, int c, double alpha, const double* __restrict__ A, int64_t lda,
            const double* __restrict__ Cm, int64_t ldc, double beta, const double* Z, int64_t ldz,
            double* Y, int64_t ldy, const double* __restrict__ A2, double* Y2) {
  MPB_PDL_WAIT();
  constexpr int TN = 16 * NT;
  if (blockIdx.z) {  // paired product Y2 = alpha A2 C (same C, k, c; beta = 0)
    A = A2;
    Y = Y2;
  }
  extern __shared__ __align__(16) unsigned char gemm_sm[];
  auto As = reinterpret_cast<double(*)[kDBK][kAPitch]>(gemm_sm);
  auto Cs = reinterpret_cast<double(*)[TN][kDPitch]>(gemm_sm + sizeof(double) * kGemmStages * kDBK * kAPitch);
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int j0 = blockIdx.y * TN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 8 * NT;
  double acc[4][NT][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto load = [&](int buf, int k0) {
    // A panel: 16 k-columns x 64 rows = 16 x 32 chunks of 2 doubles
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = threadIdx.x + 128 * t;
      const int kc = e >> 5, ch = e & 31;
      const int64_t row = i0 + 2 * ch;
      int bytes = 0;
      if (k0 + kc < k && row < n) bytes = row + 1 < n ? 16 : 8;
      const double* src = bytes ? A + row + static_cast<int64_t>(k0 + kc) * lda : A;
      cp_async16(&As[buf][kc][2 * ch], src, bytes);
    }
    // C panel: TN cols x 16 k = TN x 8 chunks
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int e = threadIdx.x + 128 * t;
      const int col = e >> 3, ch = e & 7;
      const int kr = k0 + 2 * ch;
      int bytes = 0;
      if (j0 + col < c && kr < k) bytes = kr + 1 < k ? 16 : 8;
      const double* src = bytes ? Cm + kr + static_cast<int64_t>(j0 + col) * ldc : Cm;
      cp_async16(&Cs[buf][col][2 * ch], src, bytes);
    }
  };

  const int npanel = (k + kDBK - 1) / kDBK;
#pragma unroll
  for (int q = 0; q < kGemmStages - 1; ++q) {
    if (q < npanel) load(q, q * kDBK);
    cp_async_commit();
  }
  for (int p = 0; p < npanel; ++p) {
    const int buf = p % kGemmStages;
    cp_async_wait<kGemmStages - 2>();
    __syncthreads();
    {
      const int q = p + kGemmStages - 1;
      if (q < npanel) load(q % kGemmStages, q * kDBK);
      cp_async_commit();
    }
#pragma unroll
    for (int kk = 0; kk < kDBK; kk += 4) {
      double af[4], bf[NT];
#pragma unroll
      for (int q = 0; q < 4; ++q) af[q] = As[buf][kk + t4][wm + 8 * q + g];
#pragma unroll
      for (int q = 0; q < NT; ++q) bf[q] = Cs[buf][wn + 8 * q + g][kk + t4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = i0 + wm + 8 * a + g;
        const int j = j0 + wn + 8 * b + 2 * t4 + h;
        if (i < n && j < c) {
          double v = alpha * acc[a][b][h];
          if (beta != 0.0) v = beta * Z[i + j * ldz] + v;
          Y[i + j * ldy] = v;
        }
      }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_gemm_tn(int64_t n, int k, int c, T alpha, const T* __restrict__ A, int64_t lda,
          const T* __restrict__ Cm, int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y,
          int64_t ldy, const T* __restrict__ A2, T* Y2) {
  MPB_PDL_WAIT();
  if (blockIdx.z) {
    A = A2;
    Y = Y2;
  }
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

// Tall-skinny times small, fp32 (and unaligned fp64): one thread per row of Y
// with all c <= CT outputs in registers; C (k x c) staged once in shared
// memory and read as broadcasts; the row's k values of A are independent,
// coalesced loads (8 in flight).  Pair mode via blockIdx.z as k_gemm_tn.
template <typename T, int CT>
__global__ void __launch_bounds__(128)
k_gemm_rows(int64_t n, int k, int c, T alpha, const T* __restrict__ A, int64_t lda,
            const T* __restrict__ Cm, int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y,
            int64_t ldy, const T* __restrict__ A2, T* Y2) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char rows_sm[];
  T* Cs = reinterpret_cast<T*>(rows_sm);  // k x CT, row l contiguous
  if (blockIdx.z) {
    A = A2;
    Y = Y2;
  }
  for (int e = threadIdx.x; e < k * CT; e += blockDim.x) {
    const int l = e / CT, jj = e % CT;
    Cs[e] = jj < c ? Cm[l + static_cast<int64_t>(jj) * ldc] : T(0);
  }
  __syncthreads();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  T acc[CT];
#pragma unroll
  for (int jj = 0; jj < CT; ++jj) acc[jj] = T(0);
  const T* a = A + i;
  int l = 0;
  // 16 loads in flight: the next batch is requested before this one is used
  constexpr int B = 16;
  T nxt[B];
  if (k >= B) {
#pragma unroll
    for (int u = 0; u < B; ++u) nxt[u] = __ldg(a + static_cast<int64_t>(u) * lda);
  }
  for (; l + B <= k; l += B) {
    T av[B];
#pragma unroll
    for (int u = 0; u < B; ++u) av[u] = nxt[u];
    if (l + 2 * B <= k) {
#pragma unroll
      for (int u = 0; u < B; ++u) nxt[u] = __ldg(a + static_cast<int64_t>(l + B + u) * lda);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const T* cr = Cs + (l + u) * CT;
#pragma unroll
      for (int jj = 0; jj < CT; ++jj) acc[jj] = fma(av[u], cr[jj], acc[jj]);
    }
  }
  for (; l < k; ++l) {
    const T av = __ldg(a + static_cast<int64_t>(l) * lda);
    const T* cr = Cs + l * CT;
#pragma unroll
    for (int jj = 0; jj < CT; ++jj) acc[jj] = fma(av, cr[jj], acc[jj]);
  }
#pragma unroll
  for (int jj = 0; jj < CT; ++jj) {
    if (jj < c) {
      T v = alpha * acc[jj];
      if (beta != T(0)) v = beta * Z[i + jj * ldz] + v;
      Y[i + jj * ldy] = v;
    }
  }
}

__global__ void k_f64_to_f32(int64_t n, int64_t c, const double* __restrict__ src, int64_t lds,
                             float* __restrict__ dst, int64_t ldd, int* overflow) {
  MPB_PDL_WAIT();
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
  MPB_PDL_WAIT();
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
  MPB_PDL_WAIT();
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
  MPB_PDL_WAIT();
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
  MPB_PDL_WAIT();
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
  MPB_PDL_WAIT();
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
void gram_combine(const GramPlan& p, int64_t ka, int64_t kb, const T* part, T* G, int64_t ldg, int sym,
                  cudaStream_t s, int* ticket = nullptr, T* L = nullptr, T* Uinv = nullptr,
                  int* status = nullptr, T tau2 = T(0), bool force = false) {
  if (p.nchunk == 1 && !sym && !force) return;  // the kernel wrote G directly
  const int64_t warps = sym ? ka * (ka + 1) / 2 : ka * kb;
  k_gram_combine<T><<<static_cast<unsigned>(ceil_div(warps, 8)), 256, 0, s>>>(
      p.nchunk, static_cast<int>(ka), static_cast<int>(kb), part, G, ldg, sym, ticket, L, Uinv,
      status, tau2);
  MPB_LAUNCH_CHECK();
}

template <typename T>
int64_t gram_workspace_elems(int64_t n, int64_t ka, int64_t kb) {
  const GramPlan p = gram_plan(n, ka, kb);
  return p.level_elems + kGramHead<T>;  // + the CholQR ticket (zero at allocation)
}

template <typename T>
static void gram_impl(int64_t n, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B,
                      int64_t ldb, T* G, int64_t ldg, int sym, T* work, cudaStream_t s, T* L,
                      T* Uinv, int* status, T tau2 = T(0)) {
  if (ka <= 0 || kb <= 0) return;
  if (n <= 0) {
    for (int64_t j = 0; j < kb; ++j)
      MPB_CUDA(cudaMemsetAsync(G + j * ldg, 0, sizeof(T) * ka, s));
    return;
  }
  ProfScope prof(sizeof(T) == 8 ? "gram" : "gram_f32", s, double(sizeof(T)) * n * (A == B ? ka : ka + kb),
                 2.0 * n * ka * kb);
  const GramPlan p = gram_plan(n, ka, kb);
  // workspace: [CholQR ticket (16 B, fixed place for every shape) | partials]
  int* ctr = nullptr;  // (unused)
  int* ticket = reinterpret_cast<int*>(work);
  T* part = work + kGramHead<T>;
  dim3 grid(static_cast<unsigned>(p.tiles_m * p.tiles_n), static_cast<unsigned>(p.nchunk));
  const bool aligned = (lda % 2 == 0) && (ldb % 2 == 0) &&
                       (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  const int kai = static_cast<int>(ka), kbi = static_cast<int>(kb), tn = static_cast<int>(p.tiles_n);
  if constexpr (sizeof(T) == 8) {
    if (aligned) {
      auto launch = [&](auto mt_tag) {
        constexpr int MT = decltype(mt_tag)::value;
        constexpr size_t smem = gram_dmma_smem<MT>();
        smem_opt_in(reinterpret_cast<const void*>(k_gram_dmma<MT>), smem);
        k_gram_dmma<MT><<<grid, 128, smem, s>>>(n, kai, kbi, A, lda, B, ldb, p.rows_per_chunk, tn,
                                                p.nchunk, part, ctr, G, ldg, sym);
      };
      switch (p.mt) {
        case 1: launch(std::integral_constant<int, 1>()); break;
        case 2: launch(std::integral_constant<int, 2>()); break;
        case 3: launch(std::integral_constant<int, 3>()); break;
        case 4: launch(std::integral_constant<int, 4>()); break;
        default: launch(std::integral_constant<int, 5>()); break;
      }
      MPB_LAUNCH_CHECK();
      gram_combine<T>(p, ka, kb, part, G, ldg, sym, s, L ? ticket : nullptr, L, Uinv, status, tau2);
      return;
    }
  }
  if constexpr (sizeof(T) == 4) {
    // binary32 on the tcgen05 tensor cores (tc.cu: exact 3-way bf16 split)
    if (gram_tc_wanted(n, ka, kb) && gram_tc_eligible(n, ka, kb, lda, ldb, A, B)) {
      GramPlan pt = p;
      pt.nchunk = gram_tc_f32(n, ka, A, lda, kb, B, ldb, p.nchunk, part, s);
      gram_combine<T>(pt, ka, kb, part, G, ldg, sym, s, L ? ticket : nullptr, L, Uinv, status, tau2,
                      /*force=*/true);
      return;
    }
  }
  (void)aligned;
  const GramPlan ps = p.mt <= 4 ? p : gram_plan_simt(n, ka, kb);
  grid = dim3(static_cast<unsigned>(ps.tiles_m * ps.tiles_n), static_cast<unsigned>(ps.nchunk));
  const int tns = static_cast<int>(ps.tiles_n);
  switch (ps.mt) {
    case 1:
      k_gram_partial<T, 1><<<grid, 256, 0, s>>>(n, kai, kbi, A, lda, B, ldb, ps.rows_per_chunk, tns,
                                                ps.nchunk, part, ctr, G, ldg, sym);
      break;
    case 2:
      k_gram_partial<T, 2><<<grid, 256, 0, s>>>(n, kai, kbi, A, lda, B, ldb, ps.rows_per_chunk, tns,
                                                ps.nchunk, part, ctr, G, ldg, sym);
      break;
    case 3:
      k_gram_partial<T, 3><<<grid, 256, 0, s>>>(n, kai, kbi, A, lda, B, ldb, ps.rows_per_chunk, tns,
                                                ps.nchunk, part, ctr, G, ldg, sym);
      break;
    default:
      k_gram_partial<T, 4><<<grid, 256, 0, s>>>(n, kai, kbi, A, lda, B, ldb, ps.rows_per_chunk, tns,
                                                ps.nchunk, part, ctr, G, ldg, sym);
      break;
  }
  MPB_LAUNCH_CHECK();
  gram_combine<T>(ps, ka, kb, part, G, ldg, sym, s, L ? ticket : nullptr, L, Uinv, status, tau2);
}

template <typename T>
void gram(int64_t n, int64_t ka, const T* A, int64_t lda, int64_t kb, const T* B, int64_t ldb,
          T* G, int64_t ldg, int sym, T* work, cudaStream_t s) {
  gram_impl<T>(n, ka, A, lda, kb, B, ldb, G, ldg, sym, work, s, nullptr, nullptr, nullptr);
}

template <typename T>
bool gram_cholesky(int64_t n, int64_t m, const T* V, int64_t ldv, T* G, T* work, T* L, T* Uinv,
                   int* status, cudaStream_t s, T tau2) {
  if (m > 16 || n <= 0) return false;
  gram_impl<T>(n, m, V, ldv, m, V, ldv, G, m, 1, work, s, L, Uinv, status, tau2);
  return true;
}

bool gemm_inplace_ok(bool f64, int64_t n, int64_t k, int64_t c) {
  if (c <= kGemmInplaceCols) return true;
  if (f64) return c <= 96;
  return gemm_tc_wanted(n, k, c) && gemm_tc_inplace_ok(c);
}

template <typename T>
static void gemm_impl(int64_t n, int64_t k, int64_t c, T alpha, const T* A, int64_t lda, const T* C,
                      int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y, int64_t ldy, const T* A2,
                      T* Y2, cudaStream_t s) {
  const unsigned nz = A2 ? 2u : 1u;
  if (n <= 0 || c <= 0) return;
  bool inplace = false;
  if (c > kGemmInplaceCols && k > 0) {
    // Y aliasing A: only legal within one output column tile (kernels.cuh)
    const auto lo = [](const T* p) { return reinterpret_cast<uintptr_t>(p); };
    const uintptr_t a0 = lo(A), a1 = lo(A + (k - 1) * lda + n), y0 = lo(Y), y1 = lo(Y + (c - 1) * ldy + n);
    inplace = a0 < y1 && y0 < a1;
    if (inplace && (A2 || !gemm_inplace_ok(sizeof(T) == 8, n, k, c)))
      throw Error(MPEIG_E_DIMENSION, "gemm_tn: output overlaps A beyond the in-place column limit");
  }
  if (k <= 0) {
    // Y = beta Z
    if (beta == T(0)) {
      for (int64_t j = 0; j < c; ++j) MPB_CUDA(cudaMemsetAsync(Y + j * ldy, 0, sizeof(T) * n, s));
    } else if (Y != Z) {
      copy_block<T>(n, c, Z, ldz, Y, ldy, s);
    }
    return;
  }
  ProfScope prof(sizeof(T) == 8 ? "gemm" : "gemm_f32", s, double(sizeof(T)) * n * (k + (beta != T(0) ? 2 : 1) * c),
                 2.0 * n * k * c);
  dim3 grid(static_cast<unsigned>(ceil_div(n, kTile)), static_cast<unsigned>(ceil_div(c, kTile)), nz);
  if constexpr (sizeof(T) == 8) {
    const bool aligned = (lda % 2 == 0) && (ldc % 2 == 0) &&
                         (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(C) % 16 == 0);
    if (aligned) {
      // output tile 16 * nt columns: the least padding, ties to the wider tile
      // (80 | 160 at m = 80, 48 | 96 | 144 at m = 48)
      int nt = 1;
      int64_t best = -1;
      for (int t = 5; t >= 1; --t) {
        const int64_t w = ceil_div(c, 16 * t) * 16 * t;
        if (best < 0 || w < best) {
          best = w;
          nt = t;
        }
      }
      // deep K (the dense operator A X, K = n): one column tile up to 96 wide,
      // so the n x n operand streams from HBM once instead of once per tile
      const bool deep = k > 4 * kDBK;
      if ((deep || inplace) && c > 16 * nt && c <= 96) nt = static_cast<int>(ceil_div(c, 16));
      const dim3 g2(static_cast<unsigned>(ceil_div(n, kTile)),
                    static_cast<unsigned>(ceil_div(c, 16 * nt)), nz);
      const int ki = static_cast<int>(k), ci = static_cast<int>(c);
      const bool shallow = !deep;
      auto launch = [&](auto nt_tag) {
        constexpr int NT = decltype(nt_tag)::value;
        auto go = [&](auto st_tag) {
          constexpr int ST = decltype(st_tag)::value;
          constexpr size_t smem = sizeof(double) * ST * (kDBK * kAPitch + 16 * NT * kDPitch);
          smem_opt_in(reinterpret_cast<const void*>(k_gemm_dmma<NT, ST>), smem);
          k_gemm_dmma<NT, ST><<<g2, 128, smem, s>>>(n, ki, ci, alpha, A, lda, C, ldc, beta, Z, ldz,
                                                    Y, ldy, A2, Y2);
        };
        // shallow K: every panel in flight at once; deep K: a 3-stage ring
        // (two panels of A in flight from HBM while the third is consumed)
        if (shallow)
          go(std::integral_constant<int, 4>());
        else
          go(std::integral_constant<int, 3>());
      };
      switch (nt) {
        case 1: launch(std::integral_constant<int, 1>()); break;
        case 2: launch(std::integral_constant<int, 2>()); break;
        case 3: launch(std::integral_constant<int, 3>()); break;
        case 4: launch(std::integral_constant<int, 4>()); break;
        case 5: launch(std::integral_constant<int, 5>()); break;
        default: launch(std::integral_constant<int, 6>()); break;
      }
      MPB_LAUNCH_CHECK();
      return;
    }
    if (inplace) throw Error(MPEIG_E_DIMENSION, "gemm_tn: in-place product needs 16-B aligned operands");
  }
  if constexpr (sizeof(T) == 4) {
    // binary32 on the tcgen05 tensor cores (tc.cu: exact 3-way bf16 split);
    // one CTA covers whole rows of every column tile it writes after reading
    // all of its rows of A, so the Y = A in-place contract (c <= 64) holds
    if (gemm_tc_wanted(n, k, c) && gemm_tc_eligible(n, k, c, lda, ldc, A, C) &&
        (!A2 || gemm_tc_eligible(n, k, c, lda, ldc, A2, C)) &&
        gemm_tc_f32(n, k, c, alpha, A, lda, C, ldc, beta, Z, ldz, Y, ldy, A2, Y2, inplace, s))
      return;
    if (inplace) throw Error(MPEIG_E_DIMENSION, "gemm_tn: in-place product needs the tensor-core path");
  }
  if (c <= 64 && k <= 1024) {
    const int ct = c <= 16 ? 16 : c <= 32 ? 32 : c <= 48 ? 48 : 64;
    const size_t smem = sizeof(T) * static_cast<size_t>(k) * ct;
    const dim3 g3(static_cast<unsigned>(ceil_div(n, 128)), 1, nz);
    const int ki = static_cast<int>(k), ci = static_cast<int>(c);
    auto go = [&](auto ct_tag) {
      constexpr int CT = decltype(ct_tag)::value;
      if (smem > 48 * 1024)
        MPB_CUDA(cudaFuncSetAttribute(k_gemm_rows<T, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      k_gemm_rows<T, CT><<<g3, 128, smem, s>>>(n, ki, ci, alpha, A, lda, C, ldc, beta, Z, ldz, Y,
                                               ldy, A2, Y2);
    };
    switch (ct) {
      case 16: go(std::integral_constant<int, 16>()); break;
      case 32: go(std::integral_constant<int, 32>()); break;
      case 48: go(std::integral_constant<int, 48>()); break;
      default: go(std::integral_constant<int, 64>()); break;
    }
    MPB_LAUNCH_CHECK();
    return;
  }
  k_gemm_tn<T><<<grid, 256, 0, s>>>(n, static_cast<int>(k), static_cast<int>(c), alpha, A, lda, C,
                                    ldc, beta, Z, ldz, Y, ldy, A2, Y2);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void gemm_tn(int64_t n, int64_t k, int64_t c, T alpha, const T* A, int64_t lda, const T* C,
             int64_t ldc, T beta, const T* Z, int64_t ldz, T* Y, int64_t ldy, cudaStream_t s) {
  gemm_impl<T>(n, k, c, alpha, A, lda, C, ldc, beta, Z, ldz, Y, ldy, nullptr, nullptr, s);
}

template <typename T>
void gemm_tn_pair(int64_t n, int64_t k, int64_t c, const T* A1, const T* A2, int64_t lda,
                  const T* C, int64_t ldc, T* Y1, T* Y2, int64_t ldy, cudaStream_t s) {
  if (k <= 0) {
    gemm_tn<T>(n, k, c, T(1), A1, lda, C, ldc, T(0), nullptr, 0, Y1, ldy, s);
    gemm_tn<T>(n, k, c, T(1), A2, lda, C, ldc, T(0), nullptr, 0, Y2, ldy, s);
    return;
  }
  gemm_impl<T>(n, k, c, T(1), A1, lda, C, ldc, T(0), nullptr, 0, Y1, ldy, A2, Y2, s);
}

void convert_f64_to_f32(int64_t n, int64_t c, const double* src, int64_t lds, float* dst,
                        int64_t ldd, int* overflow_flag, cudaStream_t s) {
  if (n * c <= 0) return;
  k_f64_to_f32<<<grid_for(n * c), 256, 0, s>>>(n, c, src, lds, dst, ldd, overflow_flag);
  MPB_LAUNCH_CHECK();
}

__global__ void k_add_diag(int64_t n, double* __restrict__ A, int64_t lda, double shift) {
  MPB_PDL_WAIT();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) A[i + i * lda] = __dadd_rn(A[i + i * lda], shift);
}

// A(j, i) = A(i, j) for i > j: 32 x 32 tiles through shared memory so both
// the lower-triangle reads and the upper-triangle writes are coalesced
template <typename T>
__global__ void k_symmetrize_lower(int64_t n, T* __restrict__ A, int64_t lda) {
  MPB_PDL_WAIT();
  __shared__ T tile[32][33];
  const int64_t bi = blockIdx.x, bj = blockIdx.y;  // tile row / column
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bi * 32 + tx, j = bj * 32 + r;
    if (i < n && j < n) tile[r][tx] = A[i + j * lda];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = bj * 32 + tx, j = bi * 32 + r;  // write A(i, j) = A(j, i), i < j
    if (i < n && j < n && i < j) A[i + j * lda] = tile[tx][r];
  }
}

template <typename T>
void symmetrize_lower(int64_t n, T* A, int64_t lda, cudaStream_t s) {
  if (n <= 1) return;
  const unsigned t = static_cast<unsigned>((n + 31) / 32);
  k_symmetrize_lower<T><<<dim3(t, t), dim3(32, 8), 0, s>>>(n, A, lda);
  MPB_LAUNCH_CHECK();
}
template void symmetrize_lower<double>(int64_t, double*, int64_t, cudaStream_t);
template void symmetrize_lower<float>(int64_t, float*, int64_t, cudaStream_t);

// A(i, i) += shift (retry_dense, precond.hpp:140-146)
void add_diag_f64(int64_t n, double* A, int64_t lda, double shift, cudaStream_t s) {
  if (n <= 0) return;
  k_add_diag<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(n, A, lda, shift);
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

__global__ void k_scatter_rows(int64_t n, int64_t c, const double* __restrict__ src, int64_t lds,
                               const int64_t* __restrict__ perm, double* __restrict__ dst,
                               int64_t ldd) {
  MPB_PDL_WAIT();
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= n * c) return;
  const int64_t i = t % n, j = t / n;
  dst[perm[i] + j * ldd] = src[i + j * lds];
}

void scatter_rows_f64(int64_t n, int64_t c, const double* src, int64_t lds, const int64_t* perm,
                      double* dst, int64_t ldd, cudaStream_t s) {
  if (n * c <= 0) return;
  k_scatter_rows<<<grid_for(n * c), 256, 0, s>>>(n, c, src, lds, perm, dst, ldd);
  MPB_LAUNCH_CHECK();
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
  template bool gram_cholesky<T>(int64_t, int64_t, const T*, int64_t, T*, T*, T*, T*, int*,   \
                                 cudaStream_t, T);                                             \
  template void gemm_tn_pair<T>(int64_t, int64_t, int64_t, const T*, const T*, int64_t, const T*, \
                                int64_t, T*, T*, int64_t, cudaStream_t);                          \
  template void copy_block<T>(int64_t, int64_t, const T*, int64_t, T*, int64_t, cudaStream_t); \
  template void frob_sq<T>(int64_t, int64_t, const T*, int64_t, double*, double*, cudaStream_t); \
  template void scale_block<T>(int64_t, int64_t, T, const T*, int64_t, T*, int64_t, cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
