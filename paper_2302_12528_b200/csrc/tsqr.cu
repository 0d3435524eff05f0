// tsqr.cu -- R factor of a tall-skinny block by a Householder TSQR tree.
//
// The reference factors the whole n x m block with a sequential Householder
// QR (householder_reduce, ortho.hpp:30-76) -- in fp32 for step 1 of mixed_qr
// (Alg. 2, ortho.hpp:173-186) and for the lower stage, in fp64 for the
// working-precision modes.  On the GPU the same reflections run on
// shared-memory row blocks (leaves) and then on stacked leaf R factors (tree
// levels); only R is formed.  R is unique up to row signs; the final step
// makes diag(R) positive like fix_diagonal_phases (ortho.hpp:95-110).
//
// The fp64 -> fp32 narrowing of mixed_qr's to_lower (precision.hpp:102-107)
// happens as the leaf loads W, with the overflow check.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "smallwarp.cuh"

namespace mpb {
namespace {

constexpr int kThreads = 256;
constexpr int64_t kSmemBudget = 100 * 1024;  // 2 CTAs / SM

template <typename Tq>
int64_t max_rows(int64_t m) {
  int64_t b = kSmemBudget / (m * static_cast<int64_t>(sizeof(Tq)));
  b = (b / 32) * 32;
  if (b > 1024) b = 1024;
  return b;
}

template <typename Tq>
struct TsqrPlan {
  int64_t leaf_rows;  // rows per leaf
  int64_t group;      // R factors stacked per tree node
  int64_t nleaf;
  bool ok;
};

template <typename Tq>
TsqrPlan<Tq> tsqr_plan(int64_t n, int64_t m) {
  TsqrPlan<Tq> p;
  const int64_t mr = round_up(m, 32);
  const int64_t bmax = max_rows<Tq>(m);
  p.ok = bmax >= mr;
  int64_t b = bmax;
  if (!p.ok) {
    // large m: one 227 KB CTA per leaf as long as m rows fit
    b = mr;
    p.ok = b * m * static_cast<int64_t>(sizeof(Tq)) <= 220 * 1024;
  } else {
    // short leaves: the per-column Householder step is latency-bound, so many
    // small leaves in parallel beat few tall ones; the tree nodes stack as
    // many R factors as shared memory allows.
    b = std::min(bmax, std::max<int64_t>(round_up(2 * m, 32), 128));
  }
  p.leaf_rows = b;
  p.group = std::max<int64_t>(2, (p.ok && bmax >= mr ? bmax : b) / m);
  if (p.group * m * static_cast<int64_t>(sizeof(Tq)) * m > 220 * 1024) p.group = 2;
  p.nleaf = ceil_div(n, b);
  return p;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return v;
}

// Householder reduction of the b x m tile (column-major, ld b) in shared
// memory.  On exit the upper triangle holds R.  A column whose remaining
// norm is zero gets no reflector (R(j,j) = 0; rank is judged on the final R).
// The reflector scalars (norm, beta = 2 / v^T v, the projection coefficient)
// are formed in fp64 even for an fp32 tile: beta = 2/|v|^2 overflows binary32
// once a column norm drops below ~1e-19, which happens for residual columns
// of converged Ritz pairs.
template <typename Tq>
__device__ void householder_tile(Tq* t, int b, int m) {
  __shared__ double red[kThreads / 32];
  __shared__ double sh_beta;
  __shared__ Tq sh_diag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int steps = min(b, m);
  for (int j = 0; j < steps; ++j) {
    Tq* cj = t + static_cast<int64_t>(j) * b;
    double part = 0.0;
    for (int i = j + 1 + tid; i < b; i += kThreads) {
      const double v = static_cast<double>(cj[i]);
      part = fma(v, v, part);
    }
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double tail2 = 0.0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) tail2 += red[w];
      const double x0 = static_cast<double>(cj[j]);
      const double nrm = sqrt(fma(x0, x0, tail2));
      if (nrm == 0.0) {
        sh_beta = 0.0;
        sh_diag = Tq(0);
      } else {
        const double phase = x0 >= 0.0 ? 1.0 : -1.0;
        const double v0 = x0 + phase * nrm;
        sh_beta = 2.0 / fma(v0, v0, tail2);
        sh_diag = static_cast<Tq>(-phase * nrm);
        cj[j] = static_cast<Tq>(v0);
      }
    }
    __syncthreads();
    const double beta = sh_beta;
    if (beta != 0.0) {
      for (int c = j + 1 + warp; c < m; c += kThreads / 32) {
        Tq* cc = t + static_cast<int64_t>(c) * b;
        Tq s = Tq(0);
        for (int i = j + lane; i < b; i += 32) s = fma(cj[i], cc[i], s);
        s = warp_sum(s);
        s = static_cast<Tq>(static_cast<double>(__shfl_sync(0xffffffffu, s, 0)) * beta);
        for (int i = j + lane; i < b; i += 32) cc[i] = fma(-s, cj[i], cc[i]);
      }
    }
    __syncthreads();
    if (tid == 0) cj[j] = sh_diag;
    __syncthreads();
  }
}

template <typename Tin, typename Tq>
__device__ __forceinline__ Tq narrow(Tin x, int* ovf) {
  if constexpr (sizeof(Tin) > sizeof(Tq)) {
    const Tq y = static_cast<Tq>(x);
    if (isfinite(static_cast<double>(x)) && !isfinite(static_cast<double>(y))) *ovf = 1;
    return y;
  } else {
    return static_cast<Tq>(x);
  }
}

template <typename Tin, typename Tq>
__global__ void __launch_bounds__(kThreads)
k_tsqr_leaf(int64_t n, int m, const Tin* __restrict__ W, int64_t ldw, int b, Tq* __restrict__ Rout,
            int* status) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tq* t = reinterpret_cast<Tq*>(smem_raw);
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * b;
  int ovf = 0;
  for (int j = 0; j < m; ++j)
    for (int i = threadIdx.x; i < b; i += kThreads) {
      const int64_t row = r0 + i;
      t[i + static_cast<int64_t>(j) * b] = row < n ? narrow<Tin, Tq>(W[row + j * ldw], &ovf) : Tq(0);
    }
  if (ovf) atomicCAS(status, 0, MPEIG_E_OVERFLOW);
  __syncthreads();
  householder_tile<Tq>(t, b, m);
  Tq* R = Rout + static_cast<int64_t>(blockIdx.x) * m * m;
  for (int64_t idx = threadIdx.x; idx < static_cast<int64_t>(m) * m; idx += kThreads) {
    const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
    R[idx] = (i <= j && i < b) ? t[i + static_cast<int64_t>(j) * b] : Tq(0);
  }
}

template <typename Tq>
__global__ void __launch_bounds__(kThreads)
k_tsqr_node(int64_t nR, int m, int group, const Tq* __restrict__ Rin, Tq* __restrict__ Rout) {
  MPB_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tq* t = reinterpret_cast<Tq*>(smem_raw);
  const int b = group * m;
  for (int g = 0; g < group; ++g) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * group + g;
    for (int64_t idx = threadIdx.x; idx < static_cast<int64_t>(m) * m; idx += kThreads) {
      const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
      t[g * m + i + static_cast<int64_t>(j) * b] = q < nR ? Rin[q * m * m + idx] : Tq(0);
    }
  }
  __syncthreads();
  householder_tile<Tq>(t, b, m);
  Tq* R = Rout + static_cast<int64_t>(blockIdx.x) * m * m;
  for (int64_t idx = threadIdx.x; idx < static_cast<int64_t>(m) * m; idx += kThreads) {
    const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
    R[idx] = i <= j ? t[i + static_cast<int64_t>(j) * b] : Tq(0);
  }
}

// positive diagonal (fix_diagonal_phases), rank check, copy to R (ld ldr)
template <typename Tq>
__global__ void k_tsqr_finish(int m, const Tq* __restrict__ Rin, Tq* __restrict__ R, int64_t ldr,
                              int* status, int numeric_rank_check) {
  MPB_PDL_WAIT();
  for (int64_t idx = threadIdx.x; idx < static_cast<int64_t>(m) * m; idx += blockDim.x) {
    const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
    const Tq d = Rin[i + static_cast<int64_t>(i) * m];
    const Tq v = Rin[idx];
    R[i + static_cast<int64_t>(j) * ldr] = d < Tq(0) ? -v : v;
  }
  if (threadIdx.x == 0 && status[0] == 0) {
    // Exact zero pivot: the reference's householder_reduce throws
    // RankDeficient (ortho.hpp:43-45).  A non-finite pivot is overflow.  With
    // numeric_rank_check (Householder-equivalent QR, R and the block in one
    // precision) a pivot below m*eps*max|R_ii| also counts as rank deficient:
    // Q = W R^-1 cannot represent the null directions a Householder Q fills
    // with rounding noise, so the caller takes the reference's rank-dropping
    // fallback (orthonormalize_dropping, ortho.hpp:205-250) instead.
    Tq dmax = Tq(0);
    for (int j = 0; j < m; ++j) dmax = fmax(dmax, fabs(Rin[j + static_cast<int64_t>(j) * m]));
    const Tq eps = sizeof(Tq) == 8 ? Tq(2.220446049250313e-16) : Tq(1.1920929e-7f);
    for (int j = 0; j < m; ++j) {
      const Tq d = fabs(Rin[j + static_cast<int64_t>(j) * m]);
      if (!isfinite(static_cast<double>(d))) {
        status[0] = MPEIG_E_OVERFLOW;
        status[1] = j;
        break;
      }
      if (d == Tq(0) || (numeric_rank_check && d <= Tq(m) * eps * dmax)) {
        status[0] = MPEIG_E_RANK_DEFICIENT;
        status[1] = j;
        break;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Register-resident TSQR: one launch for the whole tree.
//
// A CTA of NW warps holds a b x m tile (b = 32*RPL) in registers: warp w owns
// columns c = w + NW*q (q < MPW), lane l owns rows l + 32*i (i < RPL).  Step j
// of the Householder reduction is formed by the warp owning column j (warp
// reductions, fp64 scalars), published through a double-buffered shared
// vector, and applied by every warp to its own columns with one barrier per
// step.  Leaves factor row blocks of W; the last leaf of each group of G
// (atomic counter; the workspace starts zeroed and each counter is reset
// by the CTA that consumes it) stacks the G leaf R factors into its tile
// and factors them again, and so on up to the root, which also applies the
// positive-diagonal and rank checks of k_tsqr_finish.
// ---------------------------------------------------------------------------
template <typename Tq, int NW, int RPL, int MPW>
struct RegTile {
  static constexpr int B = 32 * RPL;
  Tq a[MPW][RPL];

  template <typename T>
  static __device__ __forceinline__ T xor_sum(T v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  }

  // Householder reduction of the tile; on exit rows <= c of column c hold R
  // and the rows below are zero.
  __device__ void factor(int m, Tq (*vbuf)[B], double* sbeta) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < m; ++j) {
      const int buf = j & 1;
      if (warp == (j % NW)) {
        const int qj = j / NW;
#pragma unroll
        for (int q = 0; q < MPW; ++q) {
          if (q != qj) continue;  // compile-time q: the tile stays in registers
          // 4 independent partial sums: the reduction is on the serial path
          double tp[4] = {0.0, 0.0, 0.0, 0.0}, xj = 0.0;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = lane + 32 * i;
            const double v = static_cast<double>(a[q][i]);
            if (r > j) tp[i & 3] = fma(v, v, tp[i & 3]);
            if (r == j) xj = v;
          }
          double tail = xor_sum((tp[0] + tp[1]) + (tp[2] + tp[3]));
          const double x0 = __shfl_sync(0xffffffffu, xj, j & 31);
          const double nrm = sqrt(fma(x0, x0, tail));
          double beta = 0.0, diag = 0.0, v0 = 0.0;
          if (nrm != 0.0) {
            const double phase = x0 >= 0.0 ? 1.0 : -1.0;
            v0 = x0 + phase * nrm;
            beta = 2.0 / fma(v0, v0, tail);
            diag = -phase * nrm;
          }
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = lane + 32 * i;
            vbuf[buf][r] = r < j ? Tq(0) : (r == j ? static_cast<Tq>(v0) : a[q][i]);
            a[q][i] = r < j ? a[q][i] : (r == j ? static_cast<Tq>(diag) : Tq(0));
          }
          if (lane == 0) sbeta[buf] = beta;
        }
      }
      __syncthreads();
      const double beta = sbeta[buf];
      if (beta == 0.0) continue;
      const Tq* v = vbuf[buf] + lane;
      const int i0 = j >> 5;  // row blocks above j hold zeros of v
#pragma unroll
      for (int q = 0; q < MPW; ++q) {
        const int c = warp + NW * q;
        if (c > j && c < m) {
          Tq sp[4] = {Tq(0), Tq(0), Tq(0), Tq(0)};
#pragma unroll
          for (int i = 0; i < RPL; ++i)
            if (i >= i0) sp[i & 3] = fma(v[32 * i], a[q][i], sp[i & 3]);
          const Tq sacc = xor_sum((sp[0] + sp[1]) + (sp[2] + sp[3]));
          const Tq f = static_cast<Tq>(static_cast<double>(sacc) * beta);
#pragma unroll
          for (int i = 0; i < RPL; ++i)
            if (i >= i0) a[q][i] = fma(-f, v[32 * i], a[q][i]);
        }
      }
    }
  }

  __device__ void store_r(int m, Tq* __restrict__ R) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < MPW; ++q) {
      const int c = warp + NW * q;
      if (c >= m) continue;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        if (r < m) R[r + static_cast<int64_t>(c) * m] = a[q][i];
      }
    }
  }
};

template <typename Tin, typename Tq, int NW, int RPL, int MPW>
__global__ void __launch_bounds__(NW * 32, 1)
k_tsqr_reg(int64_t n, int m, const Tin* __restrict__ W, int64_t ldw, Tq* __restrict__ Rbuf,
           int* __restrict__ counters, int64_t nleaf, int G, Tq* __restrict__ Rfinal, int64_t ldr,
           int* status, int numeric_rank_check, Tin* __restrict__ Rw_out, Tin* __restrict__ Rinv_out) {
  MPB_PDL_WAIT();
  using Tile = RegTile<Tq, NW, RPL, MPW>;
  constexpr int B = Tile::B;
  __shared__ __align__(16) Tq vbuf[2][B];
  __shared__ double sbeta[2];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Tile t;
  {
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * B;
    int ovf = 0;
#pragma unroll
    for (int q = 0; q < MPW; ++q) {
      const int c = warp + NW * q;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int64_t row = r0 + lane + 32 * i;
        t.a[q][i] = (c < m && row < n) ? narrow<Tin, Tq>(__ldg(W + row + c * ldw), &ovf) : Tq(0);
      }
    }
    if (ovf) atomicCAS(status, 0, MPEIG_E_OVERFLOW);
  }
  t.factor(m, vbuf, sbeta);
  const int64_t mm = static_cast<int64_t>(m) * m;
  int64_t idx = blockIdx.x, cnt = nleaf;
  Tq* level = Rbuf;   // R factors of the current level
  int* ctr = counters;
  while (cnt > 1) {
    t.store_r(m, level + idx * mm);
    const int64_t parent = idx / G;
    const int nchild = static_cast<int>(min(static_cast<int64_t>(G), cnt - parent * G));
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(ctr + parent, 1);
      s_last = old == nchild - 1;
      if (s_last) ctr[parent] = 0;  // ready for the next call / graph replay
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const Tq* kids = level + parent * G * mm;
#pragma unroll
    for (int q = 0; q < MPW; ++q) {
      const int c = warp + NW * q;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        const int g = r / m, rr = r - g * m;
        t.a[q][i] = (c < m && g < nchild && rr <= c) ? __ldcg(kids + g * mm + rr + c * m) : Tq(0);
      }
    }
    level += cnt * mm;
    ctr += ceil_div(cnt, static_cast<int64_t>(G));
    cnt = ceil_div(cnt, static_cast<int64_t>(G));
    idx = parent;
    t.factor(m, vbuf, sbeta);
  }
  // root: this CTA holds R of the whole block in registers.  Diagonal to
  // shared memory, then R with rows of positive diagonal (fix_diagonal_phases)
  // straight from the registers, and the k_tsqr_finish checks by one warp.
  Tq* sdiag = vbuf[0];  // the reflector buffers are free now (b >= m)
  __syncthreads();
#pragma unroll
  for (int q = 0; q < MPW; ++q) {
    const int c = warp + NW * q;
    if (c < m) {
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if (lane + 32 * i == c) sdiag[c] = t.a[q][i];
    }
  }
  __syncthreads();
  Tq* sR = vbuf[1];  // signed R for the fused epilogue (m <= 16: m*m <= b)
  const bool stage = Rinv_out != nullptr && m * m <= B;
#pragma unroll
  for (int q = 0; q < MPW; ++q) {
    const int c = warp + NW * q;
    if (c >= m) continue;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = lane + 32 * i;
      if (r < m) {
        const Tq v = r <= c ? (sdiag[r] < Tq(0) ? -t.a[q][i] : t.a[q][i]) : Tq(0);
        Rfinal[r + static_cast<int64_t>(c) * ldr] = v;
        if (stage) sR[r + c * m] = v;
      }
    }
  }
  if (warp == 0 && *reinterpret_cast<volatile int*>(status) == 0) {
    Tq dmax = Tq(0);
    for (int j = lane; j < m; j += 32) dmax = fmax(dmax, fabs(sdiag[j]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    const Tq eps = sizeof(Tq) == 8 ? Tq(2.220446049250313e-16) : Tq(1.1920929e-7f);
    // the first failing column decides the code, as the serial scan would
    int first = 0x7fffffff, code = 0;
    for (int j = lane; j < m; j += 32) {
      const Tq d = fabs(sdiag[j]);
      int cj = 0;
      if (!isfinite(static_cast<double>(d)))
        cj = MPEIG_E_OVERFLOW;
      else if (d == Tq(0) || (numeric_rank_check && d <= Tq(m) * eps * dmax))
        cj = MPEIG_E_RANK_DEFICIENT;
      if (cj && j < first) {
        first = j;
        code = cj;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const int of = __shfl_xor_sync(0xffffffffu, first, off);
      const int oc = __shfl_xor_sync(0xffffffffu, code, off);
      if (of < first) {
        first = of;
        code = oc;
      }
    }
    if (lane == 0 && code) {
      status[0] = code;
      status[1] = first;
    }
  }
  if (Rinv_out) {
    // fused epilogue of the QR's next two steps for m <= 16: R in the
    // working precision (Rw_out) and R^{-1} (Rinv_out), by warp 0
    __syncthreads();
    if (warp == 0 && *reinterpret_cast<volatile int*>(status) == 0) {
      if (stage)
        warp_upper_inverse<Tin, Tq, 16>(m, sR, m, Rw_out, Rinv_out, status);
      else
        warp_upper_inverse<Tin, Tq, 16>(m, Rfinal, ldr, Rw_out, Rinv_out, status);
    }
  }
}

// ---------------------------------------------------------------------------
// Throughput leaves for long blocks: one WARP factors one b x m leaf (b =
// 32*RPL) held in shared memory, with warp-synchronous steps only (no CTA
// barrier) and the dot products of four columns interleaved, so many leaves'
// latency chains overlap on each SM.  Each leaf writes its R (m x m) into a
// stacked, column-major (nleaf m) x m block, which the next pass (or the
// register TSQR above) factors again.
// ---------------------------------------------------------------------------
template <typename Tin, typename Tq, int RPL>
__global__ void __launch_bounds__(128)
k_tsqr_warpleaf(int64_t rows, int m, const Tin* __restrict__ W, int64_t ldw, int64_t nleaf,
                Tq* __restrict__ out, int* status) {
  MPB_PDL_WAIT();
  constexpr int B = 32 * RPL;
  extern __shared__ __align__(16) unsigned char wl_sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t leaf = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
  if (leaf >= nleaf) return;
  Tq* t = reinterpret_cast<Tq*>(wl_sm) + static_cast<int64_t>(warp) * B * m;
  const int64_t r0 = leaf * B;
  int ovf = 0;
  // four columns' loads in flight before their stores (one DRAM round trip
  // per four columns, not per column)
  for (int c0 = 0; c0 < m; c0 += 4) {
    Tin buf[4][RPL];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int64_t row = r0 + lane + 32 * i;
        buf[u][i] = (c0 + u < m && row < rows) ? __ldg(W + row + (c0 + u) * ldw) : Tin(0);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < m)
#pragma unroll
        for (int i = 0; i < RPL; ++i) t[(c0 + u) * B + lane + 32 * i] = narrow<Tin, Tq>(buf[u][i], &ovf);
  }
  if (ovf) atomicCAS(status, 0, MPEIG_E_OVERFLOW);
  __syncwarp();
  const int steps = m < B ? m : B;
  for (int j = 0; j < steps; ++j) {
    Tq v[RPL];
    double tail = 0.0, xj = 0.0;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = lane + 32 * i;
      v[i] = t[j * B + r];
      const double x = static_cast<double>(v[i]);
      if (r > j) tail = fma(x, x, tail);
      if (r == j) xj = x;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) tail += __shfl_xor_sync(0xffffffffu, tail, off);
    const double x0 = __shfl_sync(0xffffffffu, xj, j & 31);
    const double nrm = sqrt(fma(x0, x0, tail));
    double beta = 0.0, diag = 0.0, v0 = 0.0;
    if (nrm != 0.0) {
      const double phase = x0 >= 0.0 ? 1.0 : -1.0;
      v0 = x0 + phase * nrm;
      beta = 2.0 / fma(v0, v0, tail);
      diag = -phase * nrm;
    }
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = lane + 32 * i;
      v[i] = r < j ? Tq(0) : (r == j ? static_cast<Tq>(v0) : v[i]);
      if (r >= j) t[j * B + r] = r == j ? static_cast<Tq>(diag) : Tq(0);
    }
    if (beta != 0.0) {
      for (int c = j + 1; c < m; c += 4) {
        Tq d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          d[u] = Tq(0);
          if (c + u < m) {
            const Tq* col = t + (c + u) * B + lane;
#pragma unroll
            for (int i = 0; i < RPL; ++i) d[u] = fma(v[i], col[32 * i], d[u]);
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int u = 0; u < 4; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], off);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c + u < m) {
            const Tq f = static_cast<Tq>(static_cast<double>(d[u]) * beta);
            Tq* col = t + (c + u) * B + lane;
#pragma unroll
            for (int i = 0; i < RPL; ++i) col[32 * i] = fma(-f, v[i], col[32 * i]);
          }
        }
      }
    }
    __syncwarp();
  }
  // R (rows < m of the tile) -> rows [leaf m, leaf m + m) of the stack
  const int64_t ldo = nleaf * m;
  for (int c = 0; c < m; ++c)
    for (int r = lane; r < m; r += 32)
      out[leaf * m + r + c * ldo] = r <= c && r < B ? t[c * B + r] : Tq(0);
}

constexpr int kWarpLeafRPL = 8;  // b = 256 rows per leaf

template <typename Tq>
int warpleaf_warps(int64_t m) {  // warps (leaves) per CTA within 200 KB of shared memory
  const int64_t per = 32 * kWarpLeafRPL * m * static_cast<int64_t>(sizeof(Tq));
  int64_t w = (200 * 1024) / std::max<int64_t>(per, 1);
  return static_cast<int>(std::min<int64_t>(4, w));
}

// passes of the warp-leaf reduction for an n x m block: rows of each pass's
// input (the last entry is what the register TSQR finishes)
template <typename Tq>
std::vector<int64_t> warpleaf_passes(int64_t n, int64_t m) {
  std::vector<int64_t> rows{n};
  // (fp64 leaves: the register TSQR is faster -- 2.5 vs 3.6 ms at n = 1 M, m = 48)
  if (sizeof(Tq) != 4 || m > 64 || warpleaf_warps<Tq>(m) < 1) return rows;
  const int64_t b = 32 * kWarpLeafRPL;
  // worth it once there are several leaves per warp slot of the GPU
  while (rows.back() >= 8 * kNumSMs * b && b >= 2 * m)
    rows.push_back(ceil_div(rows.back(), b) * m);
  return rows;
}

struct RegCfg {
  int nw, rpl, mpw;  // 0 = not supported
};

// tile shape per (precision, width): b = 32*RPL >= 2m so a tree node stacks
// at least two R factors; the register tile stays <= 96 32-bit registers.
template <typename Tq>
RegCfg reg_cfg(int64_t m) {
  // The per-column step is a latency chain (two warp reductions, sqrt, a
  // barrier), so the tree is kept shallow: tall tiles (b = 32*RPL rows) and
  // wide fan-in G = b/m.  One column per warp where m allows.
  if (sizeof(Tq) == 4) {
    if (m <= 16) return {16, 8, 1};
    if (m <= 32) return {16, 16, 2};
    if (m <= 48) return {16, 16, 3};
    if (m <= 64) return {16, 16, 4};
    if (m <= 96) return {16, 8, 6};
    if (m <= 128) return {16, 8, 8};
  } else {
    if (m <= 16) return {16, 8, 1};
    if (m <= 32) return {16, 16, 2};
    if (m <= 48) return {16, 8, 3};
    if (m <= 64) return {16, 8, 4};
    if (m <= 96) return {16, 6, 6};
  }
  return {0, 0, 0};
}

template <typename Tin, typename Tq>
using RegKernel = void (*)(int64_t, int, const Tin*, int64_t, Tq*, int*, int64_t, int, Tq*, int64_t,
                           int*, int, Tin*, Tin*);

template <typename Tin, typename Tq>
RegKernel<Tin, Tq> reg_kernel(const RegCfg& c) {
#define MPB_REG(NW, RPL, MPW) \
  if (c.nw == NW && c.rpl == RPL && c.mpw == MPW) return k_tsqr_reg<Tin, Tq, NW, RPL, MPW>;
  if constexpr (sizeof(Tq) == 4) {
    MPB_REG(16, 32, 1) MPB_REG(16, 16, 1) MPB_REG(16, 8, 1) MPB_REG(16, 16, 2) MPB_REG(16, 16, 3)
    MPB_REG(16, 16, 4) MPB_REG(16, 8, 6)
    MPB_REG(16, 8, 8)
  } else {
    MPB_REG(16, 16, 1) MPB_REG(16, 8, 1) MPB_REG(16, 16, 2) MPB_REG(16, 8, 3) MPB_REG(16, 8, 4)
    MPB_REG(16, 6, 6)
  }
#undef MPB_REG
  return nullptr;
}

struct RegPlan {
  RegCfg cfg;
  int64_t nleaf, G, r_elems, n_ctr;
};

template <typename Tq>
RegPlan reg_plan(int64_t n, int64_t m) {
  RegPlan p{};
  p.cfg = reg_cfg<Tq>(m);
  if (p.cfg.nw == 0) return p;
  const int64_t b = 32 * p.cfg.rpl;
  p.G = b / m;
  p.nleaf = std::max<int64_t>(1, ceil_div(n, b));
  int64_t cnt = p.nleaf;
  p.r_elems = m * m;  // root
  p.n_ctr = 0;
  while (cnt > 1) {
    p.r_elems += cnt * m * m;
    cnt = ceil_div(cnt, p.G);
    p.n_ctr += cnt;
  }
  return p;
}


}  // namespace

// R -> Rw (working precision) and R^{-1} when the epilogue is not fused
template <typename Tin, typename Tq>
void tsqr_epilogue(int64_t m, const Tq* R, int64_t ldr, Tin* Rw, Tin* Rinv, int* status,
                   cudaStream_t s) {
  if constexpr (sizeof(Tin) != sizeof(Tq)) {
    convert_f32_to_f64(m, m, R, ldr, Rw, m, s);
    small_upper_inverse<Tin>(m, Rw, m, Rinv, status, s);
  } else {
    if (Rw && Rw != R) copy_block<Tin>(m, m, R, ldr, Rw, m, s);
    small_upper_inverse<Tin>(m, R, ldr, Rinv, status, s);
  }
}

template <typename Tin, typename Tq>
int64_t tsqr_workspace_elems(int64_t n, int64_t m) {
  const std::vector<int64_t> passes = warpleaf_passes<Tq>(n, m);
  if (passes.size() > 1) {
    // two ping-pong stacks (the first pass's output is the largest), then the
    // register TSQR of the last stack
    int64_t st = passes[1] * m;
    const int64_t last = passes.back();
    const TsqrPlan<Tq> p = tsqr_plan<Tq>(last, m);
    const int64_t smem_path = (p.nleaf + ceil_div(p.nleaf, p.group) + 1) * m * m;
    const RegPlan r = reg_plan<Tq>(last, m);
    const int64_t reg_path = r.r_elems + ceil_div(r.n_ctr * static_cast<int64_t>(sizeof(int)),
                                                  static_cast<int64_t>(sizeof(Tq))) + 2;
    return 2 * st + std::max(smem_path, reg_path) + 4;
  }
  const TsqrPlan<Tq> p = tsqr_plan<Tq>(n, m);
  const int64_t smem_path = (p.nleaf + ceil_div(p.nleaf, p.group) + 1) * m * m;
  const RegPlan r = reg_plan<Tq>(n, m);
  const int64_t reg_path = r.r_elems + ceil_div(r.n_ctr * static_cast<int64_t>(sizeof(int)),
                                                static_cast<int64_t>(sizeof(Tq))) + 2;
  return std::max(smem_path, reg_path);
}

// Whether some TSQR path handles an n x m block: the register TSQR, or the
// shared-memory leaf + tree (both the leaf tile and a node's stacked R
// factors must fit one CTA).  Wider blocks (m > ~110 fp64 / ~160 fp32) get
// their R from a Cholesky factor instead (solver.cpp tsqr_R).
template <typename Tin, typename Tq>
bool tsqr_fits(int64_t n, int64_t m) {
  const RegPlan rp = reg_plan<Tq>(n, m);
  if (rp.cfg.nw && reg_kernel<Tin, Tq>(rp.cfg)) return true;
  const TsqrPlan<Tq> p = tsqr_plan<Tq>(n, m);
  return p.ok && p.group * m * m * static_cast<int64_t>(sizeof(Tq)) <= 220 * 1024;
}
template bool tsqr_fits<double, double>(int64_t, int64_t);
template bool tsqr_fits<double, float>(int64_t, int64_t);
template bool tsqr_fits<float, float>(int64_t, int64_t);

template <typename Tin, typename Tq>
void tsqr_r(int64_t n, int64_t m, const Tin* W, int64_t ldw, Tq* R, int64_t ldr, Tq* work,
            int* status, cudaStream_t s, Tin* Rw_out, Tin* Rinv_out, int rank_check) {
  const int numeric = rank_check < 0 ? (sizeof(Tin) == sizeof(Tq) ? 1 : 0) : rank_check;
  const int mi = static_cast<int>(m);
  const std::vector<int64_t> passes = warpleaf_passes<Tq>(n, m);
  if (passes.size() > 1) {
    ProfScope prof("tsqr", s, double(sizeof(Tin)) * n * m, 2.0 * n * m * m);
    const int64_t st = passes[1] * m;
    Tq* stk[2] = {work, work + st};
    Tq* rest = work + 2 * st;
    const int wpc = warpleaf_warps<Tq>(m);
    const size_t smem = static_cast<size_t>(wpc) * 32 * kWarpLeafRPL * m * sizeof(Tq);
    const Tq* in_q = nullptr;
    for (size_t p = 0; p + 1 < passes.size(); ++p) {
      const int64_t rows = passes[p], nleaf = ceil_div(rows, 32 * kWarpLeafRPL);
      Tq* out = stk[p & 1];
      if (p == 0) {
        auto k = k_tsqr_warpleaf<Tin, Tq, kWarpLeafRPL>;
        MPB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k<<<static_cast<unsigned>(ceil_div(nleaf, wpc)), 32 * wpc, smem, s>>>(rows, mi, W, ldw,
                                                                                nleaf, out, status);
      } else {
        auto k = k_tsqr_warpleaf<Tq, Tq, kWarpLeafRPL>;
        MPB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k<<<static_cast<unsigned>(ceil_div(nleaf, wpc)), 32 * wpc, smem, s>>>(rows, mi, in_q, rows,
                                                                                nleaf, out, status);
      }
      MPB_LAUNCH_CHECK();
      in_q = out;
    }
    // the last stack: register TSQR with the original rank-check semantics;
    // R / R^-1 in the working precision formed after
    tsqr_r<Tq, Tq>(passes.back(), m, in_q, passes.back(), R, ldr, rest, status, s, nullptr,
                   nullptr, numeric);
    if (Rinv_out) tsqr_epilogue<Tin, Tq>(m, R, ldr, Rw_out, Rinv_out, status, s);
    return;
  }
  const RegPlan rp = reg_plan<Tq>(n, m);
  const RegKernel<Tin, Tq> rk = rp.cfg.nw ? reg_kernel<Tin, Tq>(rp.cfg) : nullptr;
  if (rk) {
    ProfScope prof("tsqr", s, double(sizeof(Tin)) * n * m, 2.0 * n * m * m);
    int* ctr = reinterpret_cast<int*>(work + rp.r_elems);
    const bool fuse = Rinv_out && m <= 16;
    rk<<<static_cast<unsigned>(rp.nleaf), rp.cfg.nw * 32, 0, s>>>(
        n, mi, W, ldw, work, ctr, rp.nleaf, static_cast<int>(rp.G), R, ldr, status, numeric,
        fuse ? Rw_out : nullptr, fuse ? Rinv_out : nullptr);
    MPB_LAUNCH_CHECK();
    if (Rinv_out && !fuse) tsqr_epilogue<Tin, Tq>(m, R, ldr, Rw_out, Rinv_out, status, s);
    return;
  }
  const TsqrPlan<Tq> p = tsqr_plan<Tq>(n, m);
  if (!p.ok) throw Error(MPEIG_E_CONFIG, "tsqr: block too wide for the shared-memory leaf");
  ProfScope prof("tsqr", s, double(sizeof(Tin)) * n * m, 2.0 * n * m * m);
  const size_t leaf_smem = static_cast<size_t>(p.leaf_rows * m * sizeof(Tq));
  MPB_CUDA(cudaFuncSetAttribute(k_tsqr_leaf<Tin, Tq>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(std::max<size_t>(leaf_smem, 48 * 1024))));
  Tq* bufA = work;
  Tq* bufB = work + p.nleaf * m * m;
  k_tsqr_leaf<Tin, Tq><<<static_cast<unsigned>(p.nleaf), kThreads, leaf_smem, s>>>(
      n, mi, W, ldw, static_cast<int>(p.leaf_rows), bufA, status);
  MPB_LAUNCH_CHECK();
  int64_t nR = p.nleaf;
  const size_t node_smem = static_cast<size_t>(p.group * m * m * sizeof(Tq));
  MPB_CUDA(cudaFuncSetAttribute(k_tsqr_node<Tq>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(std::max<size_t>(node_smem, 48 * 1024))));
  while (nR > 1) {
    const int64_t nout = ceil_div(nR, p.group);
    k_tsqr_node<Tq><<<static_cast<unsigned>(nout), kThreads, node_smem, s>>>(
        nR, mi, static_cast<int>(p.group), bufA, bufB);
    MPB_LAUNCH_CHECK();
    std::swap(bufA, bufB);
    nR = nout;
  }
  k_tsqr_finish<Tq><<<1, 256, 0, s>>>(mi, bufA, R, ldr, status, numeric);
  MPB_LAUNCH_CHECK();
  if (Rinv_out) tsqr_epilogue<Tin, Tq>(m, R, ldr, Rw_out, Rinv_out, status, s);
}

template int64_t tsqr_workspace_elems<double, double>(int64_t, int64_t);
template int64_t tsqr_workspace_elems<double, float>(int64_t, int64_t);
template int64_t tsqr_workspace_elems<float, float>(int64_t, int64_t);
template void tsqr_r<double, double>(int64_t, int64_t, const double*, int64_t, double*, int64_t,
                                     double*, int*, cudaStream_t, double*, double*, int);
template void tsqr_r<double, float>(int64_t, int64_t, const double*, int64_t, float*, int64_t,
                                    float*, int*, cudaStream_t, double*, double*, int);
template void tsqr_r<float, float>(int64_t, int64_t, const float*, int64_t, float*, int64_t,
                                   float*, int*, cudaStream_t, float*, float*, int);
template void tsqr_epilogue<double, double>(int64_t, const double*, int64_t, double*, double*, int*,
                                            cudaStream_t);
template void tsqr_epilogue<double, float>(int64_t, const float*, int64_t, double*, double*, int*,
                                           cudaStream_t);
template void tsqr_epilogue<float, float>(int64_t, const float*, int64_t, float*, float*, int*,
                                          cudaStream_t);

}  // namespace mpb
