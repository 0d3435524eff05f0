// ops.cu -- block operator apply A.X (K1): matrix-free stencils and CSR SpMM.
//
// Every output entry accumulates its row's entries in ascending column order
// starting from zero, each product and sum rounded separately, exactly like
// spmv_block (sparse_kernels.hpp:16-33) on the CSR form of the same matrix
// (csr_matrix.hpp:31-58 sorts columns).  The result is therefore bitwise
// identical to the reference operator, so A.X never contributes to
// trajectory drift.  Coefficients are exactly representable in fp32 as well
// (to_lower of -1, 4, 6), so the lower-precision apply follows the same code.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "rn.cuh"

namespace mpb {
namespace {

template <typename T>
__device__ __forceinline__ T acc_neg(T s, T x) {  // s += (-1) * x
  return add_rn(s, mul_rn(T(-1), x));
}

// One thread per (row, column); rows of a column are consecutive threads so
// every neighbour load of a warp is a contiguous 256-B segment (L1/L2 absorb
// the 7-fold reuse; HBM traffic stays ~ read X + write Y).
// Row-sharded z-slab: hlo / hhi are the neighbour ranks' adjacent planes
// (nx*ny per column, contiguous), nullptr at the domain boundary; the sum
// order is unchanged, so a sharded apply is bitwise the global one.
template <typename T>
__global__ void __launch_bounds__(256)
k_stencil7(int64_t nx, int64_t ny, int64_t nz, const T* __restrict__ X, int64_t ldx,
           T* __restrict__ Y, int64_t ldy, const T* __restrict__ hlo, const T* __restrict__ hhi,
           const T* __restrict__ dg, int64_t ldl, int64_t ldu) {
  MPB_PDL_WAIT();
  const int64_t n = nx * ny * nz;
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  const int64_t j = blockIdx.y;
  const T* x = X + j * ldx;
  const int64_t xi = p % nx;
  const int64_t yz = p / nx;
  const int64_t yi = yz % ny;
  const int64_t zi = yz / ny;
  const int64_t sy = nx, sz = nx * ny;
  T s = T(0);
  if (zi > 0)
    s = acc_neg(s, x[p - sz]);
  else if (hlo)
    s = acc_neg(s, hlo[p + j * ldl]);
  if (yi > 0) s = acc_neg(s, x[p - sy]);
  if (xi > 0) s = acc_neg(s, x[p - 1]);
  s = add_rn(s, mul_rn(dg ? dg[p] : T(6), x[p]));
  if (xi + 1 < nx) s = acc_neg(s, x[p + 1]);
  if (yi + 1 < ny) s = acc_neg(s, x[p + sy]);
  if (zi + 1 < nz)
    s = acc_neg(s, x[p + sz]);
  else if (hhi)
    s = acc_neg(s, hhi[p - (nz - 1) * sz + j * ldu]);
  Y[p + j * ldy] = s;
}

// Vectorised form (nx a multiple of V): a thread computes V consecutive x
// points with V-wide loads of its own, the y +- 1 and z +- 1 rows, plus the
// two scalar x neighbours -- 5 vector + 2 scalar loads for V points instead
// of 7 V scalar loads.  Per-point summation order unchanged (bitwise equal).
template <typename T, int V>
struct VecT;
template <>
struct VecT<double, 2> {
  using type = double2;
};
template <>
struct VecT<float, 4> {
  using type = float4;
};

template <typename T, int V>
__global__ void __launch_bounds__(256)
k_stencil7_vec(int64_t nx, int64_t ny, int64_t nz, const T* __restrict__ X, int64_t ldx,
               T* __restrict__ Y, int64_t ldy, const T* __restrict__ hlo, const T* __restrict__ hhi,
           const T* __restrict__ dg, int64_t ldl, int64_t ldu) {
  MPB_PDL_WAIT();
  using VT = typename VecT<T, V>::type;
  const int64_t nv = nx * ny * nz / V;
  const int64_t pv = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (pv >= nv) return;
  const int64_t j = blockIdx.y;
  const int64_t p = pv * V;
  const T* x = X + j * ldx;
  // grid coordinates: 32-bit division when the grid allows (a 64-bit
  // div / mod pair per point was the kernel's integer-pipe bottleneck)
  int64_t xi, yi, zi;
  if (nx * ny * nz <= 0xffffffffLL) {
    const uint32_t p32 = static_cast<uint32_t>(p), nx32 = static_cast<uint32_t>(nx),
                   ny32 = static_cast<uint32_t>(ny);
    const uint32_t yz32 = p32 / nx32;
    xi = p32 - yz32 * nx32;
    zi = yz32 / ny32;
    yi = yz32 - static_cast<uint32_t>(zi) * ny32;
  } else {
    const int64_t yz = p / nx;
    xi = p - yz * nx;
    yi = yz % ny;
    zi = yz / ny;
  }
  const int64_t sy = nx, sz = nx * ny;
  auto ldv = [](const T* a) {
    const VT v = *reinterpret_cast<const VT*>(a);
    return v;
  };
  const VT c = ldv(x + p);
  VT zm{}, ym{}, yp{}, zp{};
  const bool hz_m = zi > 0 || hlo, hz_p = zi + 1 < nz || hhi;
  if (zi > 0) zm = ldv(x + p - sz);
  else if (hlo) zm = ldv(hlo + p + j * ldl);
  if (yi > 0) ym = ldv(x + p - sy);
  if (yi + 1 < ny) yp = ldv(x + p + sy);
  if (zi + 1 < nz) zp = ldv(x + p + sz);
  else if (hhi) zp = ldv(hhi + p - (nz - 1) * sz + j * ldu);
  const T xl = xi > 0 ? x[p - 1] : T(0);
  const T xr = xi + V < nx ? x[p + V] : T(0);
  VT dd;
  if (dg) dd = ldv(dg + p);
  const T* dv = reinterpret_cast<const T*>(&dd);
  const T* cv = reinterpret_cast<const T*>(&c);
  const T* zmv = reinterpret_cast<const T*>(&zm);
  const T* ymv = reinterpret_cast<const T*>(&ym);
  const T* ypv = reinterpret_cast<const T*>(&yp);
  const T* zpv = reinterpret_cast<const T*>(&zp);
  VT out;
  T* o = reinterpret_cast<T*>(&out);
#pragma unroll
  for (int u = 0; u < V; ++u) {
    T s = T(0);
    if (hz_m) s = acc_neg(s, zmv[u]);
    if (yi > 0) s = acc_neg(s, ymv[u]);
    if (xi + u > 0) s = acc_neg(s, u == 0 ? xl : cv[u - 1]);
    s = add_rn(s, mul_rn(dg ? dv[u] : T(6), cv[u]));
    if (xi + u + 1 < nx) s = acc_neg(s, u + 1 == V ? xr : cv[u + 1]);
    if (yi + 1 < ny) s = acc_neg(s, ypv[u]);
    if (hz_p) s = acc_neg(s, zpv[u]);
    o[u] = s;
  }
  *reinterpret_cast<VT*>(Y + j * ldy + p) = out;
}

// Large grids: each thread marches V points of one (x, y) row position through
// ZC consecutive z-planes, so the z-1 / z+1 neighbours come from registers
// (the previous centre / the prefetched next plane) instead of two more L2
// reads per point; y +- 1 and x +- 1 hit L1 (the CTA covers whole rows).
// Same per-point summation order as k_stencil7_vec: bitwise equal.
template <typename T, int V, int ZC>
__global__ void __launch_bounds__(256)
k_stencil7_zm(int64_t nx, int64_t ny, int64_t nz, const T* __restrict__ X, int64_t ldx,
              T* __restrict__ Y, int64_t ldy, const T* __restrict__ hlo, const T* __restrict__ hhi,
           const T* __restrict__ dg, int64_t ldl, int64_t ldu) {
  MPB_PDL_WAIT();
  using VT = typename VecT<T, V>::type;
  const int64_t sz = nx * ny;
  const int64_t npv = sz / V;
  const int64_t pv = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (pv >= npv) return;
  const int64_t j = blockIdx.z;
  const int64_t q = pv * V;  // position within the plane
  const uint32_t q32 = static_cast<uint32_t>(q), nx32 = static_cast<uint32_t>(nx);
  const int64_t yi = q32 / nx32, xi = q32 - static_cast<uint32_t>(yi) * nx32;
  const int64_t sy = nx;
  const T* x = X + j * ldx;
  auto ldv = [](const T* a) { return *reinterpret_cast<const VT*>(a); };
  const int64_t z0 = static_cast<int64_t>(blockIdx.y) * ZC;
  const int64_t z1 = min(nz, z0 + ZC);
  if (z0 >= nz) return;
  VT zm{}, c = ldv(x + q + z0 * sz);
  if (z0 > 0) zm = ldv(x + q + (z0 - 1) * sz);
  else if (hlo) zm = ldv(hlo + q + j * ldl);
  for (int64_t zi = z0; zi < z1; ++zi) {
    const int64_t p = q + zi * sz;
    VT zp{}, ym{}, yp{};
    if (zi + 1 < nz) zp = ldv(x + p + sz);
    else if (hhi) zp = ldv(hhi + q + j * ldu);
    if (yi > 0) ym = ldv(x + p - sy);
    if (yi + 1 < ny) yp = ldv(x + p + sy);
    const T xl = xi > 0 ? x[p - 1] : T(0);
    const T xr = xi + V < nx ? x[p + V] : T(0);
    const bool hz_m = zi > 0 || hlo, hz_p = zi + 1 < nz || hhi;
    VT dd;
    if (dg) dd = ldv(dg + p);
    const T* dv = reinterpret_cast<const T*>(&dd);
    const T* cv = reinterpret_cast<const T*>(&c);
    const T* zmv = reinterpret_cast<const T*>(&zm);
    const T* ymv = reinterpret_cast<const T*>(&ym);
    const T* ypv = reinterpret_cast<const T*>(&yp);
    const T* zpv = reinterpret_cast<const T*>(&zp);
    VT out;
    T* o = reinterpret_cast<T*>(&out);
#pragma unroll
    for (int u = 0; u < V; ++u) {
      T s = T(0);
      if (hz_m) s = acc_neg(s, zmv[u]);
      if (yi > 0) s = acc_neg(s, ymv[u]);
      if (xi + u > 0) s = acc_neg(s, u == 0 ? xl : cv[u - 1]);
      s = add_rn(s, mul_rn(dg ? dv[u] : T(6), cv[u]));
      if (xi + u + 1 < nx) s = acc_neg(s, u + 1 == V ? xr : cv[u + 1]);
      if (yi + 1 < ny) s = acc_neg(s, ypv[u]);
      if (hz_p) s = acc_neg(s, zpv[u]);
      o[u] = s;
    }
    *reinterpret_cast<VT*>(Y + j * ldy + p) = out;
    zm = c;
    c = zp;
  }
}

// gen_laplace2d (generators.cpp:13-30): row p = i + nx*j, diag 4
template <typename T>
__global__ void __launch_bounds__(256)
k_stencil5(int64_t nx, int64_t ny, const T* __restrict__ X, int64_t ldx, T* __restrict__ Y,
           int64_t ldy) {
  MPB_PDL_WAIT();
  const int64_t n = nx * ny;
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n) return;
  const int64_t c = blockIdx.y;
  const T* x = X + c * ldx;
  const int64_t i = p % nx, j = p / nx;
  T s = T(0);
  if (j > 0) s = acc_neg(s, x[p - nx]);
  if (i > 0) s = acc_neg(s, x[p - 1]);
  s = add_rn(s, mul_rn(T(4), x[p]));
  if (i + 1 < nx) s = acc_neg(s, x[p + 1]);
  if (j + 1 < ny) s = acc_neg(s, x[p + nx]);
  Y[p + c * ldy] = s;
}

// Large 2-D grids: V points per thread marching through YC rows, the y - 1 /
// y + 1 neighbours from registers (previous centre / prefetched next row).
// Same per-point summation order as k_stencil5: bitwise equal.
template <typename T, int V, int YC>
__global__ void __launch_bounds__(256)
k_stencil5_ym(int64_t nx, int64_t ny, const T* __restrict__ X, int64_t ldx, T* __restrict__ Y,
              int64_t ldy) {
  MPB_PDL_WAIT();
  using VT = typename VecT<T, V>::type;
  const int64_t xv = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (xv * V >= nx) return;
  const int64_t i0 = xv * V;
  const int64_t c = blockIdx.z;
  const T* x = X + c * ldx;
  auto ldv = [](const T* a) { return *reinterpret_cast<const VT*>(a); };
  const int64_t y0 = static_cast<int64_t>(blockIdx.y) * YC;
  const int64_t y1 = min(ny, y0 + YC);
  if (y0 >= ny) return;
  VT ym{}, cur = ldv(x + i0 + y0 * nx);
  if (y0 > 0) ym = ldv(x + i0 + (y0 - 1) * nx);
  for (int64_t j = y0; j < y1; ++j) {
    const int64_t p = i0 + j * nx;
    VT yp{};
    if (j + 1 < ny) yp = ldv(x + p + nx);
    const T xl = i0 > 0 ? x[p - 1] : T(0);
    const T xr = i0 + V < nx ? x[p + V] : T(0);
    const T* cv = reinterpret_cast<const T*>(&cur);
    const T* ymv = reinterpret_cast<const T*>(&ym);
    const T* ypv = reinterpret_cast<const T*>(&yp);
    VT out;
    T* o = reinterpret_cast<T*>(&out);
#pragma unroll
    for (int u = 0; u < V; ++u) {
      T s = T(0);
      if (j > 0) s = acc_neg(s, ymv[u]);
      if (i0 + u > 0) s = acc_neg(s, u == 0 ? xl : cv[u - 1]);
      s = add_rn(s, mul_rn(T(4), cv[u]));
      if (i0 + u + 1 < nx) s = acc_neg(s, u + 1 == V ? xr : cv[u + 1]);
      if (j + 1 < ny) s = acc_neg(s, ypv[u]);
      o[u] = s;
    }
    *reinterpret_cast<VT*>(Y + c * ldy + p) = out;
    ym = cur;
    cur = yp;
  }
}

// CSR SpMM, Y = A X (spmv_block, sparse_kernels.hpp:16-33): a thread per row
// and CB block columns at once, so each row's entries (int32 column index +
// value) are read once per CB columns instead of once per column; the X
// gathers and Y stores are coalesced across the warp's consecutive rows.
// Every output entry sums its row's products in ascending column order with
// separately rounded multiplies and adds: bitwise the reference's sums.
template <typename T, int CB>
__global__ void __launch_bounds__(256)
k_csr_spmm(int n, const int* __restrict__ rp, const int* __restrict__ ci, const T* __restrict__ v,
           int c, const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy) {
  MPB_PDL_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c0 = blockIdx.y * CB;
  const int nc = min(CB, c - c0);
  const T* x = X + c0 * ldx;
  T acc[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) acc[u] = T(0);
  const int e = __ldg(rp + i + 1);
  for (int q = __ldg(rp + i); q < e; ++q) {
    const int col = __ldg(ci + q);
    const T a = __ldg(v + q);
#pragma unroll
    for (int u = 0; u < CB; ++u)
      if (u < nc) acc[u] = add_rn(acc[u], mul_rn(a, __ldg(x + u * ldx + col)));
  }
#pragma unroll
  for (int u = 0; u < CB; ++u)
    if (u < nc) Y[i + (c0 + u) * ldy] = acc[u];
}

// Row-sharded CSR: the rows of a list (rows == nullptr: 0 .. n-1), columns
// >= nown read from the ghost block G (ld ldg) -- the entries keep their
// global ascending order, so every row's sum is bitwise the global apply's.
template <typename T, int CB, bool kGhost>
__global__ void __launch_bounds__(256)
k_csr_spmm_rows(int nrows, const int* __restrict__ rows, const int* __restrict__ rp,
                const int* __restrict__ ci, const T* __restrict__ v, int c, const T* __restrict__ X,
                int64_t ldx, int nown, const T* __restrict__ G, int64_t ldg, T* __restrict__ Y,
                int64_t ldy) {
  MPB_PDL_WAIT();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int i = rows ? __ldg(rows + t) : t;
  const int c0 = blockIdx.y * CB;
  const int nc = min(CB, c - c0);
  const T* x = X + c0 * ldx;
  const T* g = kGhost ? G + c0 * ldg : nullptr;
  T acc[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) acc[u] = T(0);
  const int e = __ldg(rp + i + 1);
  for (int q = __ldg(rp + i); q < e; ++q) {
    const int col = __ldg(ci + q);
    const T a = __ldg(v + q);
    if (!kGhost || col < nown) {
#pragma unroll
      for (int u = 0; u < CB; ++u)
        if (u < nc) acc[u] = add_rn(acc[u], mul_rn(a, __ldg(x + u * ldx + col)));
    } else {
#pragma unroll
      for (int u = 0; u < CB; ++u)
        if (u < nc) acc[u] = add_rn(acc[u], mul_rn(a, __ldg(g + u * ldg + (col - nown))));
    }
  }
#pragma unroll
  for (int u = 0; u < CB; ++u)
    if (u < nc) Y[i + (c0 + u) * ldy] = acc[u];
}

// Y(k, j) = X(idx[k], j): the rows packed for one peer
template <typename T>
__global__ void k_gather_rows(int64_t nrows, const int* __restrict__ idx, int64_t c,
                              const T* __restrict__ X, int64_t ldx, T* __restrict__ Y, int64_t ldy) {
  MPB_PDL_WAIT();
  const int64_t total = nrows * c;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = e % nrows, j = e / nrows;
    Y[k + j * ldy] = X[__ldg(idx + k) + j * ldx];
  }
}

}  // namespace

template <typename T>
void csr_spmm_rows(int64_t nrows, const int* rows, const int* row_ptr, const int* col_idx,
                   const T* vals, int64_t c, const T* X, int64_t ldx, int64_t nown, const T* G,
                   int64_t ldg, T* Y, int64_t ldy, cudaStream_t s) {
  if (nrows <= 0 || c <= 0) return;
  auto go = [&](auto cb_tag) {
    constexpr int CB = decltype(cb_tag)::value;
    const dim3 grid(static_cast<unsigned>(ceil_div(nrows, 256)), static_cast<unsigned>(ceil_div(c, CB)));
    if (G)
      k_csr_spmm_rows<T, CB, true><<<grid, 256, 0, s>>>(static_cast<int>(nrows), rows, row_ptr, col_idx,
                                                        vals, static_cast<int>(c), X, ldx,
                                                        static_cast<int>(nown), G, ldg, Y, ldy);
    else
      k_csr_spmm_rows<T, CB, false><<<grid, 256, 0, s>>>(static_cast<int>(nrows), rows, row_ptr, col_idx,
                                                         vals, static_cast<int>(c), X, ldx,
                                                         static_cast<int>(nown), nullptr, 0, Y, ldy);
  };
  if constexpr (sizeof(T) == 8)
    go(std::integral_constant<int, 16>());
  else
    go(std::integral_constant<int, 4>());
  MPB_LAUNCH_CHECK();
}

template <typename T>
void gather_rows(int64_t nrows, const int* idx, int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy,
                 cudaStream_t s) {
  if (nrows <= 0 || c <= 0) return;
  const int64_t blocks = std::min<int64_t>(ceil_div(nrows * c, 256), 8 * kNumSMs);
  k_gather_rows<T><<<static_cast<unsigned>(blocks), 256, 0, s>>>(nrows, idx, c, X, ldx, Y, ldy);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void stencil7(int64_t nx, int64_t ny, int64_t nz, int64_t c, const T* X, int64_t ldx, T* Y,
              int64_t ldy, cudaStream_t s, const T* hlo, const T* hhi, const T* dg, int64_t ldl,
              int64_t ldu) {
  const int64_t n = nx * ny * nz;
  if (n <= 0 || c <= 0) return;
  if (ldl <= 0) ldl = nx * ny;  // halo planes packed per column
  if (ldu <= 0) ldu = nx * ny;
  // algorithmic bytes: X and Y once (+ the diagonal once per column block)
  ProfScope prof("stencil", s, (2.0 * c + (dg ? 1.0 : 0.0)) * sizeof(T) * n, 13.0 * n * c);
  constexpr int V = sizeof(T) == 8 ? 2 : 4;
  const bool aligned = nx % V == 0 && ldx % V == 0 && ldy % V == 0 &&
                       reinterpret_cast<uintptr_t>(X) % (V * sizeof(T)) == 0 &&
                       reinterpret_cast<uintptr_t>(Y) % (V * sizeof(T)) == 0 &&
                       reinterpret_cast<uintptr_t>(hlo) % (V * sizeof(T)) == 0 &&
                       reinterpret_cast<uintptr_t>(hhi) % (V * sizeof(T)) == 0 &&
                       reinterpret_cast<uintptr_t>(dg) % (V * sizeof(T)) == 0 && ldl % V == 0 && ldu % V == 0;
  constexpr int ZC = 16;
  if (aligned && n >= (int64_t(1) << 21) && nx * ny >= 256 * V && nx * ny <= 0xffffffffLL &&
      (nx * ny) % V == 0) {
    dim3 grid(static_cast<unsigned>(ceil_div(nx * ny / V, 256)),
              static_cast<unsigned>(ceil_div(nz, int64_t(ZC))), static_cast<unsigned>(c));
    k_stencil7_zm<T, V, ZC><<<grid, 256, 0, s>>>(nx, ny, nz, X, ldx, Y, ldy, hlo, hhi, dg, ldl, ldu);
    MPB_LAUNCH_CHECK();
    return;
  }
  if (aligned) {
    dim3 grid(static_cast<unsigned>(ceil_div(n / V, 256)), static_cast<unsigned>(c));
    k_stencil7_vec<T, V><<<grid, 256, 0, s>>>(nx, ny, nz, X, ldx, Y, ldy, hlo, hhi, dg, ldl, ldu);
    MPB_LAUNCH_CHECK();
    return;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(c));
  k_stencil7<T><<<grid, 256, 0, s>>>(nx, ny, nz, X, ldx, Y, ldy, hlo, hhi, dg, ldl, ldu);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void stencil5(int64_t nx, int64_t ny, int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy,
              cudaStream_t s) {
  const int64_t n = nx * ny;
  if (n <= 0 || c <= 0) return;
  ProfScope prof("stencil", s, 2.0 * sizeof(T) * n * c, 9.0 * n * c);
  constexpr int V = sizeof(T) == 8 ? 2 : 4, YC = 16;
  const bool aligned = nx % V == 0 && ldx % V == 0 && ldy % V == 0 &&
                       reinterpret_cast<uintptr_t>(X) % (V * sizeof(T)) == 0 &&
                       reinterpret_cast<uintptr_t>(Y) % (V * sizeof(T)) == 0;
  if (aligned && n >= (int64_t(1) << 20) && nx >= 64 * V) {
    dim3 grid(static_cast<unsigned>(ceil_div(nx / V, 256)),
              static_cast<unsigned>(ceil_div(ny, int64_t(YC))), static_cast<unsigned>(c));
    k_stencil5_ym<T, V, YC><<<grid, 256, 0, s>>>(nx, ny, X, ldx, Y, ldy);
    MPB_LAUNCH_CHECK();
    return;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(c));
  k_stencil5<T><<<grid, 256, 0, s>>>(nx, ny, X, ldx, Y, ldy);
  MPB_LAUNCH_CHECK();
}

template <typename T>
void csr_spmm(int64_t n, const int* row_ptr, const int* col_idx, const T* vals, int64_t nnz,
              int64_t c, const T* X, int64_t ldx, T* Y, int64_t ldy, cudaStream_t s) {
  if (n <= 0 || c <= 0) return;
  // algorithmic bytes: the matrix once (value + int32 index per entry, the
  // row pointers) and X, Y once each (SURVEY §8(d) K1 CSR)
  ProfScope prof("spmm", s, double(sizeof(T) + 4) * nnz + 4.0 * (n + 1) + 2.0 * sizeof(T) * n * c,
                 2.0 * nnz * c);
  // CB block columns per thread: each row's entries are read once per CB
  // columns.  Measured at 5-pt 1024^2 x 48 (scripts/spmm_bw.py): fp64 best at
  // 16 (the gathers' 8-B loads keep enough bytes in flight), fp32 at 4 (its
  // 4-B gathers need more threads in flight per byte)
  auto go = [&](auto cb_tag) {
    constexpr int CB = decltype(cb_tag)::value;
    const dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(ceil_div(c, CB)));
    k_csr_spmm<T, CB><<<grid, 256, 0, s>>>(static_cast<int>(n), row_ptr, col_idx, vals,
                                           static_cast<int>(c), X, ldx, Y, ldy);
  };
  if constexpr (sizeof(T) == 8)
    go(std::integral_constant<int, 16>());
  else
    go(std::integral_constant<int, 4>());
  MPB_LAUNCH_CHECK();
}

#define MPB_INST(T)                                                                          \
  template void stencil7<T>(int64_t, int64_t, int64_t, int64_t, const T*, int64_t, T*,       \
                            int64_t, cudaStream_t, const T*, const T*, const T*, int64_t,    \
                            int64_t);                      \
  template void stencil5<T>(int64_t, int64_t, int64_t, const T*, int64_t, T*, int64_t,       \
                            cudaStream_t);                                                   \
  template void csr_spmm<T>(int64_t, const int*, const int*, const T*, int64_t, int64_t,     \
                            const T*, int64_t, T*, int64_t, cudaStream_t);                   \
  template void csr_spmm_rows<T>(int64_t, const int*, const int*, const int*, const T*,      \
                                 int64_t, const T*, int64_t, int64_t, const T*, int64_t, T*, \
                                 int64_t, cudaStream_t);                                     \
  template void gather_rows<T>(int64_t, const int*, int64_t, const T*, int64_t, T*, int64_t, \
                               cudaStream_t);
MPB_INST(double)
MPB_INST(float)
#undef MPB_INST

}  // namespace mpb
