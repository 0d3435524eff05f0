// tc.cu -- the binary32 stage's Gram products and block updates on the
// 5th-generation tensor cores (tcgen05 / TMEM / TMA).
//
// G = A^T B (adjoint_matmul<float>, dense_kernels.hpp:36-52) and Y = beta Z +
// alpha A C (matmul<float>, :20-34) on B200's tcgen05 MMA.  tcgen05 has no
// fp32 multiplicand kind, so each binary32 operand is split exactly into three
// bfloat16 parts, x = hi + mid + lo (8 + 8 + 8 significand bits: every split
// is exact, bf16 has binary32's exponent range), and 8 part products (all but
// lo x lo, ~2^-32 relative) are accumulated in fp32 in tensor memory: hi x hi
// in one accumulator, the 7 smaller products in a second, summed once in the
// epilogue.  Each bf16 x bf16 product is exact in fp32, so the result carries
// only fp32 accumulation rounding -- the order of error of the reference's
// binary32 dot products, at tensor-core throughput.
//
// Kernels (newest first; the older ones remain as fallbacks):
//   * k_gemm_tma2: block update, C split once per call into its shared-memory
//     stage images (k_csplit), A streamed by TMA, warp roles (TMA, split, MMA,
//     epilogue, C bulk copy), double-buffered accumulator sets or a staged
//     TMA-store epilogue; in place when one column tile covers c.
//   * k_gram_tma: Gram chunk partials with TMA-fed 4-deep rings (reduced by
//     the deterministic combine of dense.cu).
//   * k_gemm_tma / k_gemm_tc / k_gram_tc: per-tile C split / cp.async loaders
//     (fallbacks: a call inside stream capture without scratch, no tensor-map
//     encoder).
// DESIGN.md §3.3-3.4 has the measurements and what bounds each kernel.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace mpb {
namespace {

constexpr int kTcM = 128;       // MMA M (output rows: columns of A)
constexpr int kTcThreads = 256;  // producer warps; + 1 MMA-issue warp
constexpr int kTcRing = 3;       // fp32 cp.async stages
constexpr int kTcProducts = 8;   // all part products but lo x lo (~2^-32 relative)

// Tile configuration: NMAX = widest B tile (MMA N), KC = rows of n per stage.
// <128, 32> for narrow products; <256, 16> keeps a 240-wide S^T AS in one tile
// (B read once per A tile) within shared memory.
template <int NMAX, int KC>
struct TcCfg {
  static constexpr int kHQ = KC / 16;                      // float4-quads per column
  static constexpr int kSlots = (kTcM + NMAX) / 8 * kHQ / (kTcThreads / 32);
  static constexpr int kSbo = (KC / 8) * 128;              // core-matrix group step along M/N
  static constexpr int kPartA = kTcM * KC * 2;             // one bf16 part of the A tile
  static constexpr int kBufBytes = 3 * (kTcM + NMAX) * KC * 2;
  static constexpr int kPitch = KC + 4;                    // fp32 ring column pitch (floats)
  static constexpr int kRingBytes = kTcRing * (kTcM + NMAX) * kPitch * 4;
  static constexpr int kSmem = 2 * kBufBytes + kRingBytes + 64;  // + 4 mbarriers, TMEM address
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8
// rows x 16 B; lbo = byte step between core matrices along K, sbo = along M/N
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm_100)
}

// instruction descriptor: kind::f16, A/B bf16 (K-major), D fp32, M = 128, N
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kTcM >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

// position in a ring of n slots: slot, phase parity, and whether the slot was
// used before (lap: wait for its release, parity phase ^ 1)
struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  bool lap = false;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
      lap = true;
    }
  }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
      smem_u32(bar)));
}

// x = hi + mid + lo exactly, each part a bfloat16 (its binary32 pattern has a
// zero low half): truncation splits, so every step is an exact subtraction
__device__ __forceinline__ void split3(float x, uint32_t& h, uint32_t& m, uint32_t& l) {
  h = __float_as_uint(x) & 0xFFFF0000u;
  const float r = x - __uint_as_float(h);
  m = __float_as_uint(r) & 0xFFFF0000u;
  l = __float_as_uint(r - __uint_as_float(m));
}
__device__ __forceinline__ uint32_t pack_hi(uint32_t a, uint32_t b) {  // bf16(a) | bf16(b) << 16
  return __byte_perm(a, b, 0x7632);
}

template <int NMAX, int KC>
__global__ void __launch_bounds__(kTcThreads + 32, 1)
k_gram_tc(int64_t n, int ka, int kb, const float* __restrict__ A, int64_t lda,
          const float* __restrict__ B, int64_t ldb, int64_t rows_per_chunk, int tiles_n, int ntile,
          float* __restrict__ part, int nprod, int do_store) {
  MPB_PDL_WAIT();
  using Cf = TcCfg<NMAX, KC>;
  constexpr int kTcSlots = Cf::kSlots, kTcSbo = Cf::kSbo, kTcPartA = Cf::kPartA;
  constexpr int kTcBufBytes = Cf::kBufBytes, kTcPitch = Cf::kPitch, kTcRingBytes = Cf::kRingBytes;
  constexpr int kTcNMax = NMAX, kTcKC = KC, kHQ = Cf::kHQ;
  constexpr uint32_t kAcc1 = NMAX;  // TMEM column of the small-products accumulator
  extern __shared__ __align__(1024) unsigned char tsm[];
  float* ring = reinterpret_cast<float*>(tsm + 2 * kTcBufBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + 2 * kTcBufBytes + kTcRingBytes);  // split stored
  uint64_t* empty = full + 2;                                             // stage MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 4);

  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * kTcM, j0 = tn * ntile;
  const int N = ntile;  // MMA N (multiple of 16)
  // Row blocks of kTcKC rows are dealt round-robin to the chunks (chunk c
  // takes blocks c, c + nchunk, ...): at any moment every SM streams the same
  // window of rows, so the operands' pages (one per column of a tall
  // column-major block) are shared GPU-wide instead of one set per chunk.
  const int64_t nchunk = gridDim.y;
  const int64_t r_end = n;
  (void)rows_per_chunk;
  auto stage_row = [&](int st) -> int64_t {
    return (static_cast<int64_t>(st) * nchunk + blockIdx.y) * kTcKC;
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kTcNMax));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&full[0], kTcThreads);
    mbar_init(&full[1], kTcThreads);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  // never-written columns (beyond ka / kb) of both split buffers stay zero
  for (int e = threadIdx.x; e < 2 * kTcBufBytes / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(tsm)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;

  // Work items: (8-column group g, row half hq) -> one warp instruction.  Lane
  // l: column g*8 + (l & 7), float4 index ch = (l >> 3) + 4 hq (rows 4ch..4ch+3
  // of the stage): a lane octet reads 64 contiguous bytes of one column, and
  // the 32 lanes' 8-byte bf16 stores land on 256 contiguous bytes of a core
  // matrix pair (conflict-free).
  const int ncols = kTcM + N;
  const int nitems = ncols / 8 * kHQ;
  const int cl = lane & 7, jl = lane >> 3;
  const float* src[kTcSlots];
  int soff[kTcSlots];  // byte offset of the 8-byte store inside one part
  int sprt[kTcSlots];  // part stride (bytes) of this column's operand
  int roff[kTcSlots];  // float offset of the item in one ring stage
  int rrow[kTcSlots];  // row of the item inside the stage (4 ch)
#pragma unroll
  for (int q = 0; q < kTcSlots; ++q) {
    const int it = warp + (kTcThreads / 32) * q;
    src[q] = nullptr;
    soff[q] = sprt[q] = roff[q] = rrow[q] = 0;
    if (it < nitems) {
      const int g = it / kHQ, hq = it % kHQ;
      const int col = g * 8 + cl, ch = jl + 4 * hq;
      const bool isa = col < kTcM;
      const int c = isa ? col : col - kTcM;
      const int gc = isa ? i0 + c : j0 + c;
      if (gc < (isa ? ka : kb))
        src[q] = isa ? A + static_cast<int64_t>(gc) * lda : B + static_cast<int64_t>(gc) * ldb;
      // A parts at 0, 1, 2 x kTcPartA; B parts after them, N * kTcKC * 2 apart
      soff[q] = (isa ? 0 : 3 * kTcPartA) + (c >> 3) * kTcSbo + (ch >> 1) * 128 + (c & 7) * 16 +
                (ch & 1) * 8;
      sprt[q] = isa ? kTcPartA : N * kTcKC * 2;
      roff[q] = col * kTcPitch + 4 * ch;
      rrow[q] = 4 * ch;
    }
  }
  // Each thread stages (cp.async) exactly the items it later splits, so the
  // ring needs no CTA barrier: cp.async.wait_group orders each thread's own data.
  auto fetch = [&](int slot, int64_t row0) {
    float* rs = ring + slot * (kTcM + kTcNMax) * kTcPitch;
#pragma unroll
    for (int q = 0; q < kTcSlots; ++q) {
      if (!src[q]) continue;
      const int64_t row = row0 + rrow[q];
      int bytes = 0;
      if (row < r_end) bytes = static_cast<int>(r_end - row < 4 ? r_end - row : 4) * 4;
      const float* p = bytes ? src[q] + row : src[q];
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(rs + roff[q])),
                   "l"(p), "r"(bytes));
    }
    asm volatile("cp.async.commit_group;\n");
  };
  auto store = [&](int slot, unsigned char* buf) {
    const float* rs = ring + slot * (kTcM + kTcNMax) * kTcPitch;
#pragma unroll
    for (int q = 0; q < kTcSlots; ++q) {
      if (!src[q]) continue;  // padding column: stays zero
      const float4 v = *reinterpret_cast<const float4*>(rs + roff[q]);
      uint32_t h0, m0, l0, h1, m1, l1, h2, m2, l2, h3, m3, l3;
      split3(v.x, h0, m0, l0);
      split3(v.y, h1, m1, l1);
      split3(v.z, h2, m2, l2);
      split3(v.w, h3, m3, l3);
      unsigned char* d = buf + soff[q];
      *reinterpret_cast<uint2*>(d) = make_uint2(pack_hi(h0, h1), pack_hi(h2, h3));
      *reinterpret_cast<uint2*>(d + sprt[q]) = make_uint2(pack_hi(m0, m1), pack_hi(m2, m3));
      *reinterpret_cast<uint2*>(d + 2 * sprt[q]) = make_uint2(pack_hi(l0, l1), pack_hi(l2, l3));
    }
  };

  const int64_t nblk = (n + kTcKC - 1) / kTcKC;
  static_assert(kTcKC % 16 == 0, "stage rows: whole MMA K-steps");
  const int nst = static_cast<int>(blockIdx.y < nblk ? (nblk - blockIdx.y + nchunk - 1) / nchunk : 0);
  const uint32_t idesc = idesc_bf16(N);
  const int part_b = N * kTcKC * 2;
  if (warp == kTcThreads / 32) {
    // MMA issue warp: one elected lane per stage, full -> MMAs -> commit(empty)
    if (lane == 0) {
      for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        mbar_wait(&full[buf], (st >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = smem_u32(tsm + buf * kTcBufBytes), b0 = a0 + 3 * kTcPartA;
        // part pairs (hi, mid, lo) x (hi, mid, lo) without lo x lo
        constexpr int pa_of[kTcProducts] = {0, 0, 1, 0, 1, 2, 1, 2};
        constexpr int pb_of[kTcProducts] = {0, 1, 0, 2, 1, 0, 2, 1};
#pragma unroll
        for (int pr = 0; pr < kTcProducts; ++pr)
#pragma unroll
          for (int kk = 0; kk < kTcKC / 16; ++kk) {
            if (pr >= nprod) continue;
            const uint64_t ad = umma_desc(a0 + pa_of[pr] * kTcPartA + kk * 256, 128, kTcSbo);
            const uint64_t bd = umma_desc(b0 + pb_of[pr] * part_b + kk * 256, 128, kTcSbo);
            // hi x hi into accumulator 0; the small part products into
            // accumulator 1, so the tensor core's accumulation rounding acts
            // on each sum at its own magnitude (summed once in the epilogue)
            if (pr == 0)
              mma_bf16(tmem, ad, bd, idesc, (st | kk) != 0);
            else
              mma_bf16(tmem + kAcc1, ad, bd, idesc, (st | (pr - 1) | kk) != 0);
          }
        mma_commit(&empty[buf]);
      }
    }
  } else {
    // producer warps: prefetch stage st+2 -> wait for stage st's data and for
    // the MMAs of stage st-2 (empty) -> split + store -> arrive(full)
    for (int q = 0; q < kTcRing - 1; ++q)
      if (q < nst) fetch(q, stage_row(q));
      else asm volatile("cp.async.commit_group;\n");
    for (int st = 0; st < nst; ++st) {
      const int buf = st & 1;
      if (st + kTcRing - 1 < nst)
        fetch((st + kTcRing - 1) % kTcRing, stage_row(st + kTcRing - 1));
      else
        asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kTcRing - 1));
      if (st >= 2) mbar_wait(&empty[buf], ((st >> 1) - 1) & 1);  // MMAs of stage st-2 done
      if (do_store) store(st % kTcRing, tsm + buf * kTcBufBytes);
      asm volatile("fence.proxy.async.shared::cta;\n");
      mbar_arrive(&full[buf]);
    }
    if (nst >= 1) mbar_wait(&empty[(nst - 1) & 1], ((nst - 1) >> 1) & 1);
    if (nst >= 2) mbar_wait(&empty[(nst - 2) & 1], ((nst - 2) >> 1) & 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  // epilogue (producer warps): TMEM lane = output row; warp w reads lane
  // quarter w % 4 and the column half w / 4 (8 columns per tcgen05.ld)
  if (warp < kTcThreads / 32) {
  float* out = part + static_cast<int64_t>(blockIdx.y) * ka * kb;
  const int quarter = warp & 3, half = warp >> 2;
  const int i = i0 + 32 * quarter + lane;
  const int cbeg = half * (N / 2), cend = cbeg + N / 2;
  for (int c0 = cbeg; c0 < cend; c0 += 8) {
    uint32_t v[8], w[8];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                   "=r"(w[6]), "=r"(w[7])
                 : "r"(taddr + kAcc1));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    if (i < ka) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + c0 + q;
        if (j < kb && c0 + q < N)
          out[i + static_cast<int64_t>(j) * ka] = __uint_as_float(v[q]) + __uint_as_float(w[q]);
      }
    }
  }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * kTcNMax));
}


// ---- the binary32 Gram with TMA-fed stages -----------------------------------
// Same MMA scheme as k_gram_tc, but the fp32 tiles of A and B are brought in by
// the Tensor Memory Accelerator: one elected lane of warp 0 issues the 2-D
// box loads (32 rows x <= 128 columns, 128-B swizzled: conflict-free splits)
// into a 4-deep ring of fp32 stages, completion tracked by mbarrier
// transaction counts.  No thread holds in-flight data, so the ring keeps up
// to four stages (128 KB per SM) in flight -- the register / cp.async
// loaders topped out near 2.7 TB/s for lack of bytes in flight.
// Warps 1..8 split a landed stage into the bf16 parts; warp 9 issues the MMAs.
constexpr int kTmN = 128, kTmKC = 32, kTmRing = 4;
constexpr int kTmStage = (kTcM + kTmN) * kTmKC * 4;            // fp32 bytes per ring stage
constexpr int kTmPartA = kTcM * kTmKC * 2, kTmPartB = kTmN * kTmKC * 2;
constexpr int kTmBuf = 3 * (kTmPartA + kTmPartB);
constexpr int kTmSmem = kTmRing * kTmStage + 2 * kTmBuf + 1024 + 128;  // + alignment, barriers
constexpr int kTmSplitThreads = 256;

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
}

__global__ void __launch_bounds__(kTmSplitThreads + 64, 1)
k_gram_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           int64_t n, int ka, int kb, int tiles_n, int ntile, float* __restrict__ part, int ablate) {
  MPB_PDL_WAIT();
  extern __shared__ unsigned char tsm_raw[];
  // 1024-B alignment for the 128-B swizzled TMA boxes
  unsigned char* tsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring = tsm;
  unsigned char* split = tsm + kTmRing * kTmStage;
  uint64_t* tfull = reinterpret_cast<uint64_t*>(split + 2 * kTmBuf);  // TMA landed
  uint64_t* tempty = tfull + kTmRing;                                 // stage split
  uint64_t* sfull = tempty + kTmRing;                                 // split stored
  uint64_t* sempty = sfull + 2;                                       // MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);
  constexpr uint32_t kAcc1 = kTmN;

  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int i0 = tm * kTcM, j0 = tn * ntile;
  const int N = ntile;
  const int64_t nchunk = gridDim.y;
  const int64_t nblk = (n + kTmKC - 1) / kTmKC;
  const int nst = static_cast<int>(blockIdx.y < nblk ? (nblk - blockIdx.y + nchunk - 1) / nchunk : 0);
  auto stage_row = [&](int st) -> int { return static_cast<int>((st * nchunk + blockIdx.y) * kTmKC); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kTmN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < kTmRing; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], kTmSplitThreads / 32);
    }
    mbar_init(&sfull[0], kTmSplitThreads / 32);
    mbar_init(&sfull[1], kTmSplitThreads / 32);
    mbar_init(&sempty[0], 1);
    mbar_init(&sempty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)));
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)));
  }
  for (int e = threadIdx.x; e < 2 * kTmBuf / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(split)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_bf16(N);

  if (warp == 0) {
    // ---- TMA producer
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>((kTcM + N) * kTmKC * 4);
      for (int st = 0; st < nst; ++st) {
        const int slot = st % kTmRing;
        if (st >= kTmRing) mbar_wait(&tempty[slot], ((st / kTmRing) - 1) & 1);
        if (ablate & 1) {  // diagnostics: no loads
          mbar_arrive(&tfull[slot]);
          continue;
        }
        mbar_expect_tx(&tfull[slot], bytes);
        const uint32_t dst = smem_u32(ring + slot * kTmStage);
        const uint32_t bar = smem_u32(&tfull[slot]);
        tma_load_2d(dst, &tmA, stage_row(st), i0, bar);
        tma_load_2d(dst + kTcM * kTmKC * 4, &tmB, stage_row(st), j0, bar);
      }
    }
  } else if (warp == 1 + kTmSplitThreads / 32) {
    // ---- MMA issuer
    if (lane == 0) {
      for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        mbar_wait(&sfull[buf], (st >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = smem_u32(split + buf * kTmBuf), b0 = a0 + 3 * kTmPartA;
        const uint64_t ad0 = umma_desc(a0, 128, 512), bd0 = umma_desc(b0, 128, 512);
        constexpr int pa_of[kTcProducts] = {0, 0, 1, 0, 1, 2, 1, 2};
        constexpr int pb_of[kTcProducts] = {0, 1, 0, 2, 1, 0, 2, 1};
        const uint32_t part_b = static_cast<uint32_t>(N * kTmKC * 2);
#pragma unroll
        for (int pr = 0; pr < kTcProducts; ++pr)
#pragma unroll
          for (int kk = 0; kk < kTmKC / 16; ++kk) {
            if ((ablate & 4) && pr > 0) continue;  // diagnostics: one product
            // descriptor = base + (byte offset >> 4): smem addresses stay below 2^18
            const uint64_t ad = ad0 + static_cast<uint64_t>((pa_of[pr] * kTmPartA + kk * 256) >> 4);
            const uint64_t bd = bd0 + static_cast<uint64_t>((pb_of[pr] * part_b + kk * 256) >> 4);
            if (pr == 0)
              mma_bf16(tmem, ad, bd, idesc, (st | kk) != 0);
            else
              mma_bf16(tmem + kAcc1, ad, bd, idesc, (st | (pr - 1) | kk) != 0);
          }
        mma_commit(&sempty[buf]);
      }
    }
  } else {
    // ---- split warps: item = (8-column group g, row half hq); lane (cl, jl)
    const int sw = warp - 1;  // 0..7
    const int cl = lane & 7, jl = lane >> 3;
    const int ncols = kTcM + N;
    const int nitems = ncols / 8 * 2;
    constexpr int kSlots = (kTcM + kTmN) / 8 * 2 / (kTmSplitThreads / 32);
    int roff[kSlots], soff[kSlots], sprt[kSlots];
    bool live[kSlots];
#pragma unroll
    for (int q = 0; q < kSlots; ++q) {
      const int it = sw + (kTmSplitThreads / 32) * q;
      const int g = it >> 1, hq = it & 1;
      const int col = g * 8 + cl, ch = jl + 4 * hq;
      const bool isa = col < kTcM;
      const int c = isa ? col : col - kTcM;
      live[q] = it < nitems && (isa ? i0 + c < ka : (c < N && j0 + c < kb));
      // the box row of column col is 128 B; its 16-B chunk ch sits at ch ^ (col & 7)
      roff[q] = col * 128 + ((ch ^ (col & 7)) << 4);
      soff[q] = (isa ? 0 : 3 * kTmPartA) + (c >> 3) * 512 + (ch >> 1) * 128 + (c & 7) * 16 + (ch & 1) * 8;
      sprt[q] = isa ? kTmPartA : N * kTmKC * 2;
    }
    for (int st = 0; st < nst; ++st) {
      const int slot = st % kTmRing, buf = st & 1;
      mbar_wait(&tfull[slot], (st / kTmRing) & 1);
      if (st >= 2) mbar_wait(&sempty[buf], ((st >> 1) - 1) & 1);
      const unsigned char* rs = ring + slot * kTmStage;
      unsigned char* bp = split + buf * kTmBuf;
#pragma unroll
      for (int q = 0; q < kSlots; ++q) {
        if (ablate & 2) break;  // diagnostics: no split
        if (!live[q]) continue;
        const float4 v = *reinterpret_cast<const float4*>(rs + roff[q]);
        uint32_t h0, m0, l0, h1, m1, l1, h2, m2, l2, h3, m3, l3;
        split3(v.x, h0, m0, l0);
        split3(v.y, h1, m1, l1);
        split3(v.z, h2, m2, l2);
        split3(v.w, h3, m3, l3);
        unsigned char* d = bp + soff[q];
        *reinterpret_cast<uint2*>(d) = make_uint2(pack_hi(h0, h1), pack_hi(h2, h3));
        *reinterpret_cast<uint2*>(d + sprt[q]) = make_uint2(pack_hi(m0, m1), pack_hi(m2, m3));
        *reinterpret_cast<uint2*>(d + 2 * sprt[q]) = make_uint2(pack_hi(l0, l1), pack_hi(l2, l3));
      }
      asm volatile("fence.proxy.async.shared::cta;\n");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sfull[buf]);
        mbar_arrive(&tempty[slot]);
      }
    }
    if (nst >= 1) mbar_wait(&sempty[(nst - 1) & 1], ((nst - 1) >> 1) & 1);
    if (nst >= 2) mbar_wait(&sempty[(nst - 2) & 1], ((nst - 2) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // epilogue: split warp w: TMEM lane quarter w % 4, column half w / 4
    float* out = part + static_cast<int64_t>(blockIdx.y) * ka * kb;
    const int quarter = warp & 3;  // the hardware lane quarter of this warp
    const int half = sw >> 2;
    const int i = i0 + 32 * quarter + lane;
    const int cbeg = half * (N / 2), cend = cbeg + N / 2;
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
      uint32_t v[8], w[8];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                     "=r"(v[6]), "=r"(v[7])
                   : "r"(taddr));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                     "=r"(w[6]), "=r"(w[7])
                   : "r"(taddr + kAcc1));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      if (i < ka) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + c0 + q;
          if (j < kb && c0 + q < N)
            out[i + static_cast<int64_t>(j) * ka] = __uint_as_float(v[q]) + __uint_as_float(w[q]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * kTmN));
}

// ---- Y = beta Z + alpha A C on tcgen05 ---------------------------------------
// CTA = 128 rows of Y (MMA M) x one N-wide column tile (N <= 128); K (= k,
// the columns of A) in stages of 32.  A's tile is M-contiguous in memory, so
// its bf16 parts go to the MN-major core-matrix layout (8 K-rows x 16 B of 8
// consecutive rows); C's columns are K-contiguous (K-major, as in the Gram).
constexpr int kGmN = 128, kGmKC = 32;
constexpr int kGmApitch = kTcM + 4;    // fp32 ring: A [k][128 rows]
constexpr int kGmCpitch = kGmKC + 4;   // fp32 ring: C [col][32 k]
constexpr int kGmRingStage = kGmKC * kGmApitch + kGmN * kGmCpitch;  // floats
constexpr int kGmPartA = kTcM * kGmKC * 2, kGmPartC = kGmN * kGmKC * 2;
constexpr int kGmBuf = 3 * (kGmPartA + kGmPartC);
constexpr int kGmSmem = 2 * kGmBuf + kTcRing * kGmRingStage * 4 + 64;
constexpr int kGmAItems = kGmKC * (kTcM / 4) / kTcThreads;  // float4 of A per thread per stage
constexpr int kGmCSlots = kGmN / 8 * 2 / (kTcThreads / 32);  // C items per thread (Gram mapping)
constexpr int kGmSplitA = kGmKC * (kTcM / 8) / kTcThreads;   // (k, 8-row group) items per thread

__global__ void __launch_bounds__(kTcThreads + 32, 1)
k_gemm_tc(int64_t n, int k, int c, int ntile, int tiles_n, int64_t ntiles, float alpha,
          const float* __restrict__ A, int64_t lda, const float* __restrict__ Cm, int64_t ldc,
          float beta, const float* Z, int64_t ldz, float* Y, int64_t ldy,
          const float* __restrict__ A2, float* Y2) {
  MPB_PDL_WAIT();
  if (blockIdx.z) {
    A = A2;
    Y = Y2;
  }
  extern __shared__ __align__(1024) unsigned char gsm[];
  float* ring = reinterpret_cast<float*>(gsm + 2 * kGmBuf);
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + 2 * kGmBuf + kTcRing * kGmRingStage * 4);
  uint64_t* empty = full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 4);
  const int N = ntile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kAcc1 = kGmN;  // TMEM column of the small-products accumulator

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kGmN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    mbar_init(&full[0], kTcThreads);
    mbar_init(&full[1], kTcThreads);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  for (int e = threadIdx.x; e < 2 * kGmBuf / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(gsm)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  const int nst = (k + kGmKC - 1) / kGmKC;
  // persistent: this CTA's tiles are blockIdx.x, + gridDim.x, ...; the stage
  // pipeline runs over the flattened (tile, K stage) sequence
  const int64_t my_tiles =
      blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = my_tiles * nst;
  // instruction descriptor: bf16 x bf16 -> f32, A MN-major (bit 15), B K-major
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                         (static_cast<uint32_t>(N >> 3) << 17) |
                         (static_cast<uint32_t>(kTcM >> 4) << 24);

  if (warp == kTcThreads / 32) {
    if (lane == 0) {
      for (int64_t g = 0; g < total; ++g) {
        const int buf = static_cast<int>(g & 1);
        const int st = static_cast<int>(g % nst);
        mbar_wait(&full[buf], static_cast<uint32_t>((g >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = smem_u32(gsm + buf * kGmBuf), c0 = a0 + 3 * kGmPartA;
        constexpr int pa_of[kTcProducts] = {0, 0, 1, 0, 1, 2, 1, 2};
        constexpr int pb_of[kTcProducts] = {0, 1, 0, 2, 1, 0, 2, 1};
#pragma unroll
        for (int pr = 0; pr < kTcProducts; ++pr)
#pragma unroll
          for (int kk = 0; kk < kGmKC / 16; ++kk) {
            // A: MN-major, k-groups (8 k) 128 B apart (lbo), row groups 512 B (sbo)
            const uint64_t ad = umma_desc(a0 + pa_of[pr] * kGmPartA + kk * 256, 128, 512);
            const uint64_t bd = umma_desc(c0 + pb_of[pr] * kGmPartC + kk * 256, 128, 512);
            // hi x hi into accumulator 0; the small part products into
            // accumulator 1, so the tensor core's accumulation rounding acts
            // on each sum at its own magnitude (summed once in the epilogue)
            if (pr == 0)
              mma_bf16(tmem, ad, bd, idesc, (st | kk) != 0);
            else
              mma_bf16(tmem + kAcc1, ad, bd, idesc, (st | (pr - 1) | kk) != 0);
          }
        mma_commit(&empty[buf]);
      }
    }
  } else {
    const int cl = lane & 7, jl = lane >> 3;
    // C items of this thread (the Gram's K-major mapping), per column tile
    int ccol[kGmCSlots], coff[kGmCSlots], croff[kGmCSlots], cch[kGmCSlots];
#pragma unroll
    for (int q = 0; q < kGmCSlots; ++q) {
      const int it = warp + (kTcThreads / 32) * q;
      const int g = it >> 1, hq = it & 1;
      const int col = 8 * g + cl, ch = jl + 4 * hq;
      ccol[q] = col;
      coff[q] = (col >> 3) * 512 + (ch >> 1) * 128 + (col & 7) * 16 + (ch & 1) * 8;
      croff[q] = kGmKC * kGmApitch + col * kGmCpitch + 4 * ch;
      cch[q] = 4 * ch;
    }
    auto tile_of = [&](int64_t g) { return blockIdx.x + (g / nst) * gridDim.x; };
    auto fetch = [&](int slot, int64_t g) {
      float* rs = ring + slot * kGmRingStage;
      const int64_t t = tile_of(g);
      const int64_t i0 = (t / tiles_n) * kTcM;
      const int j0 = static_cast<int>(t % tiles_n) * N;
      const int k0 = static_cast<int>(g % nst) * kGmKC;
#pragma unroll
      for (int q = 0; q < kGmAItems; ++q) {
        const int e = threadIdx.x + kTcThreads * q;
        const int kc = e / (kTcM / 4), ch = e % (kTcM / 4);
        const int64_t row = i0 + 4 * ch;
        int bytes = 0;
        if (k0 + kc < k && row < n) bytes = static_cast<int>(n - row < 4 ? n - row : 4) * 4;
        const float* p = bytes ? A + row + static_cast<int64_t>(k0 + kc) * lda : A;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                         smem_u32(rs + kc * kGmApitch + 4 * ch)),
                     "l"(p), "r"(bytes));
      }
#pragma unroll
      for (int q = 0; q < kGmCSlots; ++q) {
        if (ccol[q] >= N) continue;
        const int kr = k0 + cch[q];
        const int j = j0 + ccol[q];
        int bytes = 0;
        if (kr < k && j < c) bytes = (k - kr < 4 ? k - kr : 4) * 4;
        const float* p = bytes ? Cm + kr + static_cast<int64_t>(j) * ldc : Cm;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(rs + croff[q])),
                     "l"(p), "r"(bytes));
      }
      asm volatile("cp.async.commit_group;\n");
    };
    auto store = [&](int slot, unsigned char* buf) {
      const float* rs = ring + slot * kGmRingStage;
      // A -> MN-major: item (k, 8-row group gm): 8 consecutive rows of column k
#pragma unroll
      for (int q = 0; q < kGmSplitA; ++q) {
        const int e = threadIdx.x + kTcThreads * q;
        const int kc = e % kGmKC, gm = e / kGmKC;
        const float4 v0 = *reinterpret_cast<const float4*>(rs + kc * kGmApitch + 8 * gm);
        const float4 v1 = *reinterpret_cast<const float4*>(rs + kc * kGmApitch + 8 * gm + 4);
        const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t h[8], m[8], l[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) split3(f[t], h[t], m[t], l[t]);
        const int off = gm * 512 + (kc >> 3) * 128 + (kc & 7) * 16;
        *reinterpret_cast<uint4*>(buf + off) =
            make_uint4(pack_hi(h[0], h[1]), pack_hi(h[2], h[3]), pack_hi(h[4], h[5]), pack_hi(h[6], h[7]));
        *reinterpret_cast<uint4*>(buf + kGmPartA + off) =
            make_uint4(pack_hi(m[0], m[1]), pack_hi(m[2], m[3]), pack_hi(m[4], m[5]), pack_hi(m[6], m[7]));
        *reinterpret_cast<uint4*>(buf + 2 * kGmPartA + off) =
            make_uint4(pack_hi(l[0], l[1]), pack_hi(l[2], l[3]), pack_hi(l[4], l[5]), pack_hi(l[6], l[7]));
      }
      unsigned char* cb = buf + 3 * kGmPartA;
#pragma unroll
      for (int q = 0; q < kGmCSlots; ++q) {
        if (ccol[q] >= N) continue;
        const float4 v = *reinterpret_cast<const float4*>(rs + croff[q]);
        uint32_t h0, m0, l0, h1, m1, l1, h2, m2, l2, h3, m3, l3;
        split3(v.x, h0, m0, l0);
        split3(v.y, h1, m1, l1);
        split3(v.z, h2, m2, l2);
        split3(v.w, h3, m3, l3);
        unsigned char* d = cb + coff[q];
        *reinterpret_cast<uint2*>(d) = make_uint2(pack_hi(h0, h1), pack_hi(h2, h3));
        *reinterpret_cast<uint2*>(d + kGmPartC) = make_uint2(pack_hi(m0, m1), pack_hi(m2, m3));
        *reinterpret_cast<uint2*>(d + 2 * kGmPartC) = make_uint2(pack_hi(l0, l1), pack_hi(l2, l3));
      }
    };
    auto epilogue = [&](int64_t t) {
      const int64_t i0 = (t / tiles_n) * kTcM;
      const int j0 = static_cast<int>(t % tiles_n) * N;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      // TMEM lane = row of the tile; warp w: lane quarter w % 4, column half w / 4
      const int quarter = warp & 3, half = warp >> 2;
      const int64_t i = i0 + 32 * quarter + lane;
      const int cbeg = half * (N / 2), cend = cbeg + N / 2;
      for (int cc = cbeg; cc < cend; cc += 16) {
        // 16 columns: both TMEM loads and every Z load in flight before use
        uint32_t v[16];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + cc;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        if (cc + 8 < cend)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                       : "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                         "=r"(v[14]), "=r"(v[15])
                       : "r"(taddr + 8));
        uint32_t w[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                       "=r"(w[6]), "=r"(w[7])
                     : "r"(taddr + kAcc1));
        if (cc + 8 < cend)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                       : "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
                         "=r"(w[14]), "=r"(w[15])
                       : "r"(taddr + kAcc1 + 8));
        float z[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int j = j0 + cc + q;
          z[q] = (beta != 0.f && i < n && j < c && cc + q < cend) ? Z[i + static_cast<int64_t>(j) * ldz] : 0.f;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (i < n) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int j = j0 + cc + q;
            if (j < c && cc + q < cend) {
              float y = alpha * (__uint_as_float(v[q]) + __uint_as_float(w[q]));
              if (beta != 0.f) y = fmaf(beta, z[q], y);
              Y[i + static_cast<int64_t>(j) * ldy] = y;
            }
          }
        }
      }
      // the next tile's first MMA overwrites the accumulator: order these reads first
      asm volatile("tcgen05.fence::before_thread_sync;\n");
    };
    for (int q = 0; q < kTcRing - 1; ++q)
      if (q < total) fetch(q, q);
      else asm volatile("cp.async.commit_group;\n");
    for (int64_t g = 0; g < total; ++g) {
      const int buf = static_cast<int>(g & 1);
      if (g + kTcRing - 1 < total)
        fetch(static_cast<int>((g + kTcRing - 1) % kTcRing), g + kTcRing - 1);
      else
        asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kTcRing - 1));
      // the A tile is shared by all producers (row groups x k): a barrier
      // makes every thread's cp.async data visible before the split reads it
      asm volatile("bar.sync 1, %0;\n" ::"n"(kTcThreads));
      if (g >= 2) mbar_wait(&empty[buf], static_cast<uint32_t>(((g >> 1) - 1) & 1));
      store(static_cast<int>(g % kTcRing), gsm + buf * kGmBuf);
      asm volatile("fence.proxy.async.shared::cta;\n");
      mbar_arrive(&full[buf]);
      // the ring slot read here is refilled two stages later: order the reads
      asm volatile("bar.sync 1, %0;\n" ::"n"(kTcThreads));
      if (g % nst == nst - 1) {
        // last K stage of a tile: its MMAs done -> epilogue
        mbar_wait(&empty[buf], static_cast<uint32_t>((g >> 1) & 1));
        epilogue(tile_of(g));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * kGmN));
}


// ---- the binary32 block update with TMA-fed stages ----------------------------
// k_gemm_tc's scheme (persistent CTAs over 128-row tiles, K in stages of 32,
// two TMEM accumulators) with the fp32 tiles brought in by TMA: A's box is
// 128 rows x 32 columns (row-contiguous, unswizzled), C's 32 k-rows x N
// columns (128-B swizzled).  A's bf16 parts use the MN-major core-matrix
// layout with a 528-B group stride (16 B of padding per 8-row group), so the
// split's stores are conflict-free.
constexpr int kGtN = 128, kGtKC = 32, kGtRing = 4;
constexpr int kGtStageA = kGtKC * kTcM * 4;   // [k][128 rows] fp32
constexpr int kGtStage = kGtStageA + kGtN * kGtKC * 4;
constexpr int kGtSbo = 528;
constexpr int kGtPartA = (kTcM / 8) * kGtSbo, kGtPartC = kGtN * kGtKC * 2;
constexpr int kGtBuf = 3 * (kGtPartA + kGtPartC);
constexpr int kGtSmem = kGtRing * kGtStage + 2 * kGtBuf + 1024 + 128;
static_assert(kGtSmem <= 232448, "k_gemm_tma shared memory");

__global__ void __launch_bounds__(kTmSplitThreads + 64, 1)
k_gemm_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
           int64_t n, int k, int c, int ntile, int tiles_n, int64_t ntiles, float alpha, float beta,
           const float* Z, int64_t ldz, float* Y, int64_t ldy) {
  MPB_PDL_WAIT();
  extern __shared__ unsigned char gsm_raw[];
  unsigned char* gsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring = gsm;
  unsigned char* split = gsm + kGtRing * kGtStage;
  uint64_t* tfull = reinterpret_cast<uint64_t*>(split + 2 * kGtBuf);
  uint64_t* tempty = tfull + kGtRing;
  uint64_t* sfull = tempty + kGtRing;
  uint64_t* sempty = sfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);
  constexpr uint32_t kAcc1 = kGtN;
  const int N = ntile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * kGtN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < kGtRing; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], kTmSplitThreads);
    }
    mbar_init(&sfull[0], kTmSplitThreads);
    mbar_init(&sfull[1], kTmSplitThreads);
    mbar_init(&sempty[0], 1);
    mbar_init(&sempty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)));
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmC)));
  }
  for (int e = threadIdx.x; e < 2 * kGtBuf / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(split)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  const int nst = (k + kGtKC - 1) / kGtKC;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = my_tiles * nst;
  auto tile_of = [&](int64_t g) { return blockIdx.x + (g / nst) * gridDim.x; };
  // bf16 x bf16 -> f32, A MN-major (bit 15), B K-major
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                         (static_cast<uint32_t>(N >> 3) << 17) |
                         (static_cast<uint32_t>(kTcM >> 4) << 24);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(kGtStageA + N * kGtKC * 4);
      for (int64_t g = 0; g < total; ++g) {
        const int slot = static_cast<int>(g % kGtRing);
        if (g >= kGtRing) mbar_wait(&tempty[slot], static_cast<uint32_t>(((g / kGtRing) - 1) & 1));
        const int64_t t = tile_of(g);
        const int row0 = static_cast<int>((t / tiles_n) * kTcM);
        const int j0 = static_cast<int>(t % tiles_n) * N;
        const int k0 = static_cast<int>(g % nst) * kGtKC;
        mbar_expect_tx(&tfull[slot], bytes);
        const uint32_t dst = smem_u32(ring + slot * kGtStage);
        const uint32_t bar = smem_u32(&tfull[slot]);
        tma_load_2d(dst, &tmA, row0, k0, bar);
        tma_load_2d(dst + kGtStageA, &tmC, k0, j0, bar);
      }
    }
  } else if (warp == 1 + kTmSplitThreads / 32) {
    if (lane == 0) {
      for (int64_t g = 0; g < total; ++g) {
        const int buf = static_cast<int>(g & 1);
        const int st = static_cast<int>(g % nst);
        mbar_wait(&sfull[buf], static_cast<uint32_t>((g >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = smem_u32(split + buf * kGtBuf), c0 = a0 + 3 * kGtPartA;
        constexpr int pa_of[kTcProducts] = {0, 0, 1, 0, 1, 2, 1, 2};
        constexpr int pb_of[kTcProducts] = {0, 1, 0, 2, 1, 0, 2, 1};
#pragma unroll
        for (int pr = 0; pr < kTcProducts; ++pr)
#pragma unroll
          for (int kk = 0; kk < kGtKC / 16; ++kk) {
            const uint64_t ad = umma_desc(a0 + pa_of[pr] * kGtPartA + kk * 256, 128, kGtSbo);
            const uint64_t bd = umma_desc(c0 + pb_of[pr] * kGtPartC + kk * 256, 128, 512);
            if (pr == 0)
              mma_bf16(tmem, ad, bd, idesc, (st | kk) != 0);
            else
              mma_bf16(tmem + kAcc1, ad, bd, idesc, (st | (pr - 1) | kk) != 0);
          }
        mma_commit(&sempty[buf]);
      }
    }
  } else {
    const int sw = warp - 1;
    const int cl = lane & 7, jl = lane >> 3;
    // C items (K-major, the Gram's B mapping): column 8 g + cl, float4 ch
    constexpr int kCSlots = kGtN / 8 * 2 / (kTmSplitThreads / 32);
    int croff[kCSlots], csoff[kCSlots];
    bool clive[kCSlots];
#pragma unroll
    for (int q = 0; q < kCSlots; ++q) {
      const int it = sw + (kTmSplitThreads / 32) * q;
      const int g = it >> 1, hq = it & 1;
      const int col = 8 * g + cl, ch = jl + 4 * hq;
      clive[q] = col < N;
      croff[q] = kGtStageA + col * 128 + ((ch ^ (col & 7)) << 4);
      csoff[q] = 3 * kGtPartA + (col >> 3) * 512 + (ch >> 1) * 128 + (col & 7) * 16 + (ch & 1) * 8;
    }
    constexpr int kAItems = kGtKC * (kTcM / 8) / kTmSplitThreads;  // (k, 8-row group) items
    auto epilogue = [&](int64_t t) {
      const int64_t i0 = (t / tiles_n) * kTcM;
      const int j0 = static_cast<int>(t % tiles_n) * N;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int quarter = warp & 3, half = sw >> 2;
      const int64_t i = i0 + 32 * quarter + lane;
      const int cbeg = half * (N / 2), cend = cbeg + N / 2;
      for (int cc = cbeg; cc < cend; cc += 8) {
        uint32_t v[8], w[8];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * quarter) << 16) + cc;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                       "=r"(w[6]), "=r"(w[7])
                     : "r"(taddr + kAcc1));
        float z[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + cc + q;
          z[q] = (beta != 0.f && i < n && j < c && cc + q < cend) ? Z[i + static_cast<int64_t>(j) * ldz] : 0.f;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (i < n) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = j0 + cc + q;
            if (j < c && cc + q < cend) {
              float y = alpha * (__uint_as_float(v[q]) + __uint_as_float(w[q]));
              if (beta != 0.f) y = fmaf(beta, z[q], y);
              Y[i + static_cast<int64_t>(j) * ldy] = y;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
    };
    for (int64_t g = 0; g < total; ++g) {
      const int slot = static_cast<int>(g % kGtRing), buf = static_cast<int>(g & 1);
      mbar_wait(&tfull[slot], static_cast<uint32_t>((g / kGtRing) & 1));
      if (g >= 2) mbar_wait(&sempty[buf], static_cast<uint32_t>(((g >> 1) - 1) & 1));
      const unsigned char* rs = ring + slot * kGtStage;
      unsigned char* bp = split + buf * kGtBuf;
      // A -> MN-major: item (row group gm fastest, column kc): 8 rows of column kc
#pragma unroll
      for (int q = 0; q < kAItems; ++q) {
        const int e = (threadIdx.x - 32) + kTmSplitThreads * q;
        const int gm = e % (kTcM / 8), kc = e / (kTcM / 8);
        const float4 v0 = *reinterpret_cast<const float4*>(rs + kc * (kTcM * 4) + gm * 32);
        const float4 v1 = *reinterpret_cast<const float4*>(rs + kc * (kTcM * 4) + gm * 32 + 16);
        const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t h[8], m[8], l[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) split3(f[t], h[t], m[t], l[t]);
        const int off = gm * kGtSbo + (kc >> 3) * 128 + (kc & 7) * 16;
        *reinterpret_cast<uint4*>(bp + off) =
            make_uint4(pack_hi(h[0], h[1]), pack_hi(h[2], h[3]), pack_hi(h[4], h[5]), pack_hi(h[6], h[7]));
        *reinterpret_cast<uint4*>(bp + kGtPartA + off) =
            make_uint4(pack_hi(m[0], m[1]), pack_hi(m[2], m[3]), pack_hi(m[4], m[5]), pack_hi(m[6], m[7]));
        *reinterpret_cast<uint4*>(bp + 2 * kGtPartA + off) =
            make_uint4(pack_hi(l[0], l[1]), pack_hi(l[2], l[3]), pack_hi(l[4], l[5]), pack_hi(l[6], l[7]));
      }
#pragma unroll
      for (int q = 0; q < kCSlots; ++q) {
        if (!clive[q]) continue;
        const float4 v = *reinterpret_cast<const float4*>(rs + croff[q]);
        uint32_t h0, m0, l0, h1, m1, l1, h2, m2, l2, h3, m3, l3;
        split3(v.x, h0, m0, l0);
        split3(v.y, h1, m1, l1);
        split3(v.z, h2, m2, l2);
        split3(v.w, h3, m3, l3);
        unsigned char* d = bp + csoff[q];
        *reinterpret_cast<uint2*>(d) = make_uint2(pack_hi(h0, h1), pack_hi(h2, h3));
        *reinterpret_cast<uint2*>(d + kGtPartC) = make_uint2(pack_hi(m0, m1), pack_hi(m2, m3));
        *reinterpret_cast<uint2*>(d + 2 * kGtPartC) = make_uint2(pack_hi(l0, l1), pack_hi(l2, l3));
      }
      asm volatile("fence.proxy.async.shared::cta;\n");
      mbar_arrive(&sfull[buf]);
      mbar_arrive(&tempty[slot]);
      if (g % nst == nst - 1) {
        mbar_wait(&sempty[buf], static_cast<uint32_t>((g >> 1) & 1));
        epilogue(tile_of(g));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * kGtN));
}


// ---- the binary32 block update, C split once ----------------------------------
// Y = beta Z + alpha A C with C (k x c, the small coefficient block) split into
// its bf16 parts ONCE per call by k_csplit, straight into the shared-memory
// image the MMA reads (per 32-row K stage: 3 parts x N columns, K-major core
// matrices), so the persistent CTAs only split their A tiles; one column tile
// up to 256 wide (A is read and split once per row tile).  Roles:
//   warp 0       TMA producer of A (128 rows x 32 columns, 4-deep ring);
//   warps 1..8   split A into the MN-major bf16 parts (double-buffered);
//   warp 9       MMA issuer (8 part products x 2 K-steps per stage);
//   warps 10..17 epilogue: TMEM -> registers -> Y (two accumulator sets when
//                4 N <= 512 TMEM columns, so a tile drains while the next one
//                accumulates);
//   warp 18      bulk-copies the stage's C image (L2-resident) into a 2-deep
//                buffer behind the MMAs.
// Each CTA reads every K column of its rows before the epilogue writes them
// and one column tile covers all of c, so Y may alias A (in-place V U^-1).
constexpr int kG2KC = 32, kG2NMax = 256;
constexpr int kG2StageA = kG2KC * kTcM * 4;
constexpr int kG2Sbo = 528;
constexpr int kG2PartA = (kTcM / 8) * kG2Sbo, kG2BufA = 3 * kG2PartA;
constexpr int kG2Warps = 19, kG2Threads = 32 * kG2Warps;
constexpr int kG2SplitThreads = 256, kG2EpiThreads = 256;
__host__ __device__ constexpr int g2_cimg(int N) { return 3 * N * kG2KC * 2; }  // bytes per stage
// Ring depths (each 2..4) as shared memory allows: R fp32 A stages
// (TMA, HBM latency), S split A buffers (the split of stage g + S overlaps the
// MMAs of g + 1 .. g + S - 1), D C images (L2 latency of the bulk copies).
constexpr int kG2SmemMax = 232448 - 1024;  // less the static shared memory
struct G2Depth {
  int R, S, D;
};
__host__ __device__ constexpr int g2_smem(int N, G2Depth d) {
  return d.R * kG2StageA + d.S * kG2BufA + d.D * g2_cimg(N) + 1024 + 256;
}
inline G2Depth g2_depth(int N) {
  // (measured: deeper S and D past 2 change nothing at n = 2M, N = 80 .. 160)
  constexpr G2Depth pref[] = {{4, 2, 4}, {4, 2, 3}, {4, 2, 2}, {3, 2, 2}, {2, 2, 2}};
  for (const G2Depth& d : pref)
    if (g2_smem(N, d) <= kG2SmemMax) return d;
  return {2, 2, 2};
}
static_assert(g2_smem(kG2NMax, G2Depth{3, 3, 2}) <= kG2SmemMax, "k_gemm_tma2 shared memory");

// C image: [tn][st] stage images of 3 parts x N columns x 32 k (bf16), zero
// beyond k and c; thread = (column, 8-k chunk) of one stage
__global__ void k_csplit(int k, int c, int N, int nst, int tiles_n, const float* __restrict__ C,
                         int64_t ldc, unsigned char* __restrict__ img) {
  MPB_PDL_WAIT();
  const int64_t total = static_cast<int64_t>(tiles_n) * nst * N * (kG2KC / 8);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int kc = static_cast<int>(e % (kG2KC / 8));
    const int col = static_cast<int>((e / (kG2KC / 8)) % N);
    const int64_t ts = e / (kG2KC / 8) / N;  // tn * nst + st
    const int st = static_cast<int>(ts % nst), tn = static_cast<int>(ts / nst);
    const int j = tn * N + col;
    uint32_t h[8], m[8], l[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kk = st * kG2KC + kc * 8 + q;
      const float x = (kk < k && j < c && col < N) ? C[kk + static_cast<int64_t>(j) * ldc] : 0.f;
      split3(x, h[q], m[q], l[q]);
    }
    unsigned char* d = img + ts * g2_cimg(N) + (col >> 3) * 512 + kc * 128 + (col & 7) * 16;
    const int part = N * kG2KC * 2;
    *reinterpret_cast<uint4*>(d) =
        make_uint4(pack_hi(h[0], h[1]), pack_hi(h[2], h[3]), pack_hi(h[4], h[5]), pack_hi(h[6], h[7]));
    *reinterpret_cast<uint4*>(d + part) =
        make_uint4(pack_hi(m[0], m[1]), pack_hi(m[2], m[3]), pack_hi(m[4], m[5]), pack_hi(m[6], m[7]));
    *reinterpret_cast<uint4*>(d + 2 * part) =
        make_uint4(pack_hi(l[0], l[1]), pack_hi(l[2], l[3]), pack_hi(l[4], l[5]), pack_hi(l[6], l[7]));
  }
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(kG2Threads, 1)
k_gemm_tma2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmY,
            const unsigned char* __restrict__ cimg, int64_t n, int k, int c, int N, int tiles_n,
            int64_t rtiles, G2Depth dep, int stage_out, int two_acc, int nprod, int ablate,
            float alpha, float beta, const float* Z, int64_t ldz, float* Y, int64_t ldy) {
  MPB_PDL_WAIT();
  extern __shared__ unsigned char g2_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(g2_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int cbytes = g2_cimg(N);
  unsigned char* ring = sm;
  const int R = dep.R, S = dep.S, D = dep.D;
  unsigned char* abuf = ring + R * kG2StageA;
  unsigned char* cbuf = abuf + S * kG2BufA;
  // stage_out: the output tile (128 x N fp32, column-major) is staged in shared
  // memory and written by one TMA store, so the accumulators are released
  // as soon as they are read (one accumulator set: N > 128)
  float* stg = reinterpret_cast<float*>(cbuf + D * cbytes);
  uint64_t* afull = reinterpret_cast<uint64_t*>(cbuf + D * cbytes + (stage_out ? kTcM * N * 4 : 0));
  uint64_t* aempty = afull + 4;       // [4]: A stage split
  uint64_t* sfull = aempty + 4;       // [4]: split buffer stored
  uint64_t* cfull = sfull + 4;        // [4]: C image landed
  uint64_t* cdone = cfull + 4;        // [4]: MMAs of the image's stage done
  uint64_t* mdone = cdone + 4;        // [4]: MMAs of the split buffer's stage done
  uint64_t* accfull = mdone + 4;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto wait_ = [](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };
  // accumulator set = 1 or 2 TMEM accumulators of N columns (the second
  // collects the 7 smaller part products); two sets when they fit in 512
  const int set_cols = two_acc ? 2 * N : N;
  const int nacc = 2 * set_cols <= 512 ? 2 : 1;
  const uint32_t acc1_off = two_acc ? static_cast<uint32_t>(N) : 0u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) {
      mbar_init(&afull[q], 1);
      mbar_init(&aempty[q], kG2SplitThreads / 32);
      mbar_init(&cfull[q], 1);
      mbar_init(&cdone[q], 1);
      mbar_init(&sfull[q], kG2SplitThreads / 32);
      mbar_init(&mdone[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&accfull[q], 1);
      mbar_init(&accempty[q], kG2EpiThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)));
  }
  for (int e = threadIdx.x; e < S * kG2BufA / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(abuf)[e] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tmem_slot;
  const int nst = (k + kG2KC - 1) / kG2KC;
  // local tile tl: row tile blockIdx.x + (tl / tiles_n) * gridDim.x, column
  // tile tl % tiles_n (a row tile's column tiles back to back: A from L2)
  const int64_t my_rows = blockIdx.x < rtiles ? (rtiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t my_tiles = my_rows * tiles_n;
  const int64_t total = my_tiles * nst;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) |
                         (static_cast<uint32_t>(N >> 3) << 17) |
                         (static_cast<uint32_t>(kTcM >> 4) << 24);

  // loop state advanced incrementally: no 64-bit divisions on the hand-off path
  // (a runtime int64 div / mod is a ~100-instruction call; several per stage
  // per role cost ~1 us per stage)
  if (warp == 0) {
    if (lane == 0) {
      RingPos rp;
      int st = 0, ct = 0;
      int64_t rt = blockIdx.x;
      for (int64_t g = 0; g < total; ++g) {
        if (rp.lap) wait_(&aempty[rp.slot], rp.phase ^ 1u);
        if (ablate & 8) {  // diagnostics: no A loads
          mbar_arrive(&afull[rp.slot]);
        } else {
          mbar_expect_tx(&afull[rp.slot], kG2StageA);
          tma_load_2d(smem_u32(ring + rp.slot * kG2StageA), &tmA, static_cast<int>(rt * kTcM),
                      st * kG2KC, smem_u32(&afull[rp.slot]));
        }
        rp.next(R);
        if (++st == nst) {
          st = 0;
          if (++ct == tiles_n) {
            ct = 0;
            rt += gridDim.x;
          }
        }
      }
    }
  } else if (warp == kG2Warps - 1) {
    if (lane == 0) {
      RingPos cp;
      int st = 0, ct = 0;
      for (int64_t g = 0; g < total; ++g) {
        if (cp.lap) wait_(&cdone[cp.slot], cp.phase ^ 1u);
        if ((ablate & 1) && g >= D) {  // diagnostics: no C reloads
          mbar_arrive(&cfull[cp.slot]);
        } else {
          mbar_expect_tx(&cfull[cp.slot], static_cast<uint32_t>(cbytes));
          bulk_load(smem_u32(cbuf + cp.slot * cbytes),
                    cimg + static_cast<int64_t>(ct * nst + st) * cbytes, static_cast<uint32_t>(cbytes),
                    smem_u32(&cfull[cp.slot]));
        }
        cp.next(D);
        if (++st == nst) {
          st = 0;
          if (++ct == tiles_n) ct = 0;
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      const uint32_t part_c = static_cast<uint32_t>(N * kG2KC * 2);
      RingPos sp, cp, ap;
      int st = 0;
      for (int64_t g = 0; g < total; ++g) {
        if (st == 0 && ap.lap) wait_(&accempty[ap.slot], ap.phase ^ 1u);
        wait_(&sfull[sp.slot], sp.phase);
        wait_(&cfull[cp.slot], cp.phase);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t a0 = smem_u32(abuf + sp.slot * kG2BufA), c0 = smem_u32(cbuf + cp.slot * cbytes);
        // descriptor = base + (byte offset >> 4): smem addresses stay below 2^18
        const uint64_t ad0 = umma_desc(a0, 128, kG2Sbo), bd0 = umma_desc(c0, 128, 512);
        const uint32_t acc = tmem + static_cast<uint32_t>(ap.slot * set_cols);
        constexpr int pa_of[kTcProducts] = {0, 0, 1, 0, 1, 2, 1, 2};
        constexpr int pb_of[kTcProducts] = {0, 1, 0, 2, 1, 0, 2, 1};
#pragma unroll
        for (int pr = 0; pr < kTcProducts; ++pr)
#pragma unroll
          for (int kk = 0; kk < kG2KC / 16; ++kk) {
            if (pr >= nprod) continue;
            const uint64_t ad = ad0 + static_cast<uint64_t>((pa_of[pr] * kG2PartA + kk * 256) >> 4);
            const uint64_t bd = bd0 + static_cast<uint64_t>((pb_of[pr] * part_c + kk * 256) >> 4);
            if (pr == 0)
              mma_bf16(acc, ad, bd, idesc, (st | kk) != 0);
            else
              mma_bf16(acc + acc1_off, ad, bd, idesc, two_acc ? ((st | (pr - 1) | kk) != 0) : 1u);
          }
        mma_commit(&mdone[sp.slot]);
        mma_commit(&cdone[cp.slot]);
        sp.next(S);
        cp.next(D);
        if (++st == nst) {
          mma_commit(&accfull[ap.slot]);
          ap.next(nacc);
          st = 0;
        }
      }
    }
  } else if (warp <= 8) {
    // ---- split A: item (8-row group gm fastest, column kc)
    constexpr int kAItems = kG2KC * (kTcM / 8) / kG2SplitThreads;
    const int tid = threadIdx.x - 32;
    RingPos rp, sp;
    for (int64_t g = 0; g < total; ++g) {
      const int slot = rp.slot, buf = sp.slot;
      wait_(&afull[slot], rp.phase);
      if (sp.lap) wait_(&mdone[buf], sp.phase ^ 1u);
      rp.next(R);
      sp.next(S);
      const unsigned char* rs = ring + slot * kG2StageA;
      unsigned char* bp = abuf + buf * kG2BufA;
#pragma unroll
      for (int q = 0; q < kAItems; ++q) {
        if (ablate & 2) break;  // diagnostics: no split
        const int e = tid + kG2SplitThreads * q;
        const int gm = e % (kTcM / 8), kc = e / (kTcM / 8);
        const float4 v0 = *reinterpret_cast<const float4*>(rs + kc * (kTcM * 4) + gm * 32);
        const float4 v1 = *reinterpret_cast<const float4*>(rs + kc * (kTcM * 4) + gm * 32 + 16);
        const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t h[8], m[8], l[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) split3(f[t], h[t], m[t], l[t]);
        const int off = gm * kG2Sbo + (kc >> 3) * 128 + (kc & 7) * 16;
        *reinterpret_cast<uint4*>(bp + off) =
            make_uint4(pack_hi(h[0], h[1]), pack_hi(h[2], h[3]), pack_hi(h[4], h[5]), pack_hi(h[6], h[7]));
        *reinterpret_cast<uint4*>(bp + kG2PartA + off) =
            make_uint4(pack_hi(m[0], m[1]), pack_hi(m[2], m[3]), pack_hi(m[4], m[5]), pack_hi(m[6], m[7]));
        *reinterpret_cast<uint4*>(bp + 2 * kG2PartA + off) =
            make_uint4(pack_hi(l[0], l[1]), pack_hi(l[2], l[3]), pack_hi(l[4], l[5]), pack_hi(l[6], l[7]));
      }
      if (!(ablate & 32)) {  // 32: no proxy fence (diagnostics); 64: one per warp
        if (!(ablate & 64)) {
          asm volatile("fence.proxy.async.shared::cta;\n");
        } else {
          __syncwarp();
          if (lane == 0) asm volatile("fence.proxy.async.shared::cta;\n");
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sfull[buf]);
        mbar_arrive(&aempty[slot]);
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lane quarter w % 4, column half
    const int quarter = warp & 3, half = (warp - 10) >> 2;
    const int cbeg = half * (N / 2), cend = cbeg + N / 2;
    RingPos ap;
    int ct = 0;
    int64_t rt = blockIdx.x;
    for (int64_t tl = 0; tl < my_tiles; ++tl) {
      const int a = ap.slot;
      wait_(&accfull[a], ap.phase);
      ap.next(nacc);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int64_t row0 = rt * kTcM, i = row0 + 32 * quarter + lane;
      const int j0 = ct * N;
      if (++ct == tiles_n) {
        ct = 0;
        rt += gridDim.x;
      }
      const uint32_t acc = tmem + static_cast<uint32_t>(a * set_cols) + (static_cast<uint32_t>(32 * quarter) << 16);
      for (int cc = cbeg; cc < cend; cc += 8) {
        if (ablate & 16) break;  // diagnostics: no TMEM drain
        uint32_t v[8], w[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(acc + cc));
        if (two_acc) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                       : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                         "=r"(w[6]), "=r"(w[7])
                       : "r"(acc + N + cc));
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = 0u;
        }
        float z[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = j0 + cc + q;
          z[q] = (beta != 0.f && i < n && j < c) ? Z[i + static_cast<int64_t>(j) * ldz] : 0.f;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (stage_out) {
          float* col = stg + static_cast<int64_t>(cc) * kTcM + 32 * quarter + lane;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float y = alpha * (__uint_as_float(v[q]) + __uint_as_float(w[q]));
            if (beta != 0.f) y = fmaf(beta, z[q], y);
            col[q * kTcM] = y;
          }
        } else if (i < n && !(ablate & 4)) {  // ablate 4 (diagnostics): no stores
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = j0 + cc + q;
            if (j < c) {
              float y = alpha * (__uint_as_float(v[q]) + __uint_as_float(w[q]));
              if (beta != 0.f) y = fmaf(beta, z[q], y);
              Y[i + static_cast<int64_t>(j) * ldy] = y;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[a]);
      if (stage_out) {
        // all epilogue threads' staging stores -> the async proxy; one TMA
        // store of the tile (rows >= n and columns >= c are clipped by the
        // map); the staging buffer is reused once the store has read it
        asm volatile("fence.proxy.async.shared::cta;\n");
        __syncwarp();
        asm volatile("bar.sync 1, %0;\n" ::"r"(kG2EpiThreads));
        if (warp == 10 && lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                  reinterpret_cast<uint64_t>(&tmY)),
              "r"(static_cast<int>(row0)), "r"(j0), "r"(smem_u32(stg))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;\n");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
        __syncwarp();  // bar.sync counts whole warps: reconverge lane 0 first
        asm volatile("bar.sync 1, %0;\n" ::"r"(kG2EpiThreads));
      }
    }
    if (stage_out && warp == 10 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

}  // namespace

int g_gram_tc = 1, g_gemm_tc = 1;
int g_tc_nprod = kTcProducts, g_tc_store = 1;  // experiment knobs

bool gram_tc_eligible(int64_t n, int64_t ka, int64_t kb, int64_t lda, int64_t ldb, const float* A,
                      const float* B) {
  return n >= 32 && (lda % 4 == 0) && (ldb % 4 == 0) &&
         (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
         ka >= 1 && kb >= 1;
}

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// 2-D map of a column-major rows x cols fp32 block (ld elements between
// columns), boxes of 32 rows x box_cols columns, 128-B swizzle
// general: boxes of box_rows x box_cols, 128-B swizzle or none
bool make_map_rows(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld,
                   int box_rows, int box_cols, bool swizzle) {
  EncodeTiled enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_cols)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld,
              int box_cols) {
  EncodeTiled enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTmKC), static_cast<cuuint32_t>(box_cols)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int g_gram_tma = 1;

// Chunk partials of G = A^T B (ka x kb each, column-major, ld ka) into part,
// nchunk row chunks; returns nchunk (the caller's deterministic combine sums them).
int64_t gram_tc_f32(int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb, const float* B,
                    int64_t ldb, int64_t max_chunks, float* part, cudaStream_t s) {
  auto go = [&](auto nmax_tag, auto kc_tag) -> int64_t {
    constexpr int NMAX = decltype(nmax_tag)::value, KC = decltype(kc_tag)::value;
    const int64_t tiles_m = ceil_div(ka, kTcM);
    const int64_t tiles_n = ceil_div(kb, NMAX);
    const int64_t ntile = round_up(ceil_div(kb, tiles_n), 16);  // MMA N: multiple of 16
    const int64_t tiles = tiles_m * tiles_n;
    int64_t nchunk = std::max<int64_t>(1, kNumSMs / tiles);
    nchunk = std::min(nchunk, std::max<int64_t>(1, max_chunks));
    nchunk = std::min(nchunk, ceil_div(n, KC));
    constexpr int smem = TcCfg<NMAX, KC>::kSmem;
    smem_opt_in(reinterpret_cast<const void*>(k_gram_tc<NMAX, KC>), smem);
    const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nchunk));
    k_gram_tc<NMAX, KC><<<grid, kTcThreads + 32, smem, s>>>(
        n, static_cast<int>(ka), static_cast<int>(kb), A, lda, B, ldb, 0, static_cast<int>(tiles_n),
        static_cast<int>(ntile), part, g_tc_nprod, g_tc_store);
    MPB_LAUNCH_CHECK();
    return nchunk;
  };
  if (g_gram_tma && n < (int64_t(1) << 31)) {
    // TMA-fed stages: B tiles up to 128 wide (240 = 2 x 120)
    const int64_t tiles_m = ceil_div(ka, kTcM), tiles_n = ceil_div(kb, kTmN);
    const int64_t ntile = round_up(ceil_div(kb, tiles_n), 16);
    CUtensorMap ma, mb;
    if (make_map(&ma, A, n, ka, lda, kTcM) && make_map(&mb, B, n, kb, ldb, static_cast<int>(ntile))) {
      const int64_t tiles = tiles_m * tiles_n;
      int64_t nchunk = std::max<int64_t>(1, kNumSMs / tiles);
      nchunk = std::min(nchunk, std::max<int64_t>(1, max_chunks));
      nchunk = std::min(nchunk, ceil_div(n, kTmKC));
      smem_opt_in(reinterpret_cast<const void*>(k_gram_tma), kTmSmem);
      const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nchunk));
      k_gram_tma<<<grid, kTmSplitThreads + 64, kTmSmem, s>>>(ma, mb, n, static_cast<int>(ka),
                                                           static_cast<int>(kb), static_cast<int>(tiles_n),
                                                           static_cast<int>(ntile), part, g_tc_ablate);
      MPB_LAUNCH_CHECK();
      return nchunk;
    }
  }
  if (kb <= 128) return go(std::integral_constant<int, 128>(), std::integral_constant<int, 32>());
  return go(std::integral_constant<int, 256>(), std::integral_constant<int, 16>());
}

bool gemm_tc_eligible(int64_t n, int64_t k, int64_t c, int64_t lda, int64_t ldc, const float* A,
                      const float* C) {
  return n >= kTcM && k >= 1 && c >= 1 && (lda % 4 == 0) && (ldc % 4 == 0) &&
         (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
}

namespace {
// Per (device, stream) scratch for the split C images; grown outside stream
// capture only (a captured call that needs more falls back to k_gemm_tma).
// Outgrown buffers stay allocated (a captured graph may still use them) until
// the owning context releases its stream (tc_scratch_release).
struct TcScratch {
  void* cur = nullptr;
  size_t cap = 0;
  std::vector<void*> old;
};
std::mutex& tc_scratch_mu() {
  static std::mutex mu;
  return mu;
}
std::map<std::pair<int, cudaStream_t>, TcScratch>& tc_scratch_map() {
  static std::map<std::pair<int, cudaStream_t>, TcScratch> m;
  return m;
}
unsigned char* tc_scratch(size_t bytes, cudaStream_t s) {
  int dev = 0;
  MPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(tc_scratch_mu());
  TcScratch& b = tc_scratch_map()[{dev, s}];
  if (b.cap >= bytes) return static_cast<unsigned char*>(b.cur);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  MPB_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return nullptr;
  const size_t want = std::max<size_t>({bytes, 2 * b.cap, size_t(4) << 20});
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (b.cur) b.old.push_back(b.cur);
  b.cur = p;
  b.cap = want;
  return static_cast<unsigned char*>(p);
}
}  // namespace

// the scratch of a stream the caller is about to destroy (its work finished)
void tc_scratch_release(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(tc_scratch_mu());
  auto& m = tc_scratch_map();
  for (auto it = m.begin(); it != m.end();) {
    if (it->first.second == s) {
      cudaFree(it->second.cur);
      for (void* p : it->second.old) cudaFree(p);
      it = m.erase(it);
    } else {
      ++it;
    }
  }
}

int g_gemm_tma2 = 1, g_tc_twoacc = 1, g_tc_ablate = 0, g_g2_depth = 0, g_tc_stage = 1;

bool gemm_tc_inplace_ok(int64_t c) { return g_gemm_tma2 && c <= kG2NMax; }

bool gemm_tc_f32(int64_t n, int64_t k, int64_t c, float alpha, const float* A, int64_t lda,
                 const float* C, int64_t ldc, float beta, const float* Z, int64_t ldz, float* Y,
                 int64_t ldy, const float* A2, float* Y2, bool inplace, cudaStream_t s) {
  if (g_gemm_tma2 && n < (int64_t(1) << 31) && k < (int64_t(1) << 31)) {
    // C split once into its shared-memory stage images; A streamed by TMA
    // c > 128: one column tile (one accumulator set) or two column tiles of
    // <= 128 (double-buffered accumulators, A re-read from L2); in place: one
    const int64_t tiles_n = ceil_div(c, (g_gemm_tma2 == 2 && !inplace) ? kGtN : kG2NMax);
    const int N = static_cast<int>(round_up(ceil_div(c, tiles_n), 16));
    const int nst = static_cast<int>(ceil_div(k, kG2KC));
    const size_t img = static_cast<size_t>(tiles_n) * nst * g2_cimg(N);
    unsigned char* cimg = tc_scratch(img, s);
    if (cimg) {
      const int64_t items = tiles_n * nst * N * (kG2KC / 8);
      k_csplit<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(items, 256), 4 * kNumSMs)), 256, 0, s>>>(
          static_cast<int>(k), static_cast<int>(c), N, nst, static_cast<int>(tiles_n), C, ldc, cimg);
      MPB_LAUNCH_CHECK();
      const int64_t rtiles = ceil_div(n, kTcM);
      G2Depth dep = g2_depth(N);
      // one accumulator set (two accumulators of N > 128 columns): stage the
      // output for a TMA store when the smem allows (ring depths 2)
      const bool one_set = 2 * (g_tc_twoacc ? 2 * N : N) > 512;
      const auto aligned16 = [](const float* p, int64_t ld) {
        return p && reinterpret_cast<uintptr_t>(p) % 16 == 0 && ld % 4 == 0;
      };
      int stage_out = one_set && g_tc_stage && aligned16(Y, ldy) && (!A2 || aligned16(Y2, ldy)) &&
                      g2_smem(N, G2Depth{2, 2, 2}) + kTcM * N * 4 <= kG2SmemMax;
      if (stage_out) dep = G2Depth{2, 2, 2};
      if (g_g2_depth) {  // diagnostics: forced ring depths RSD (e.g. 423)
        const G2Depth f{g_g2_depth / 100, g_g2_depth / 10 % 10, g_g2_depth % 10};
        if (f.R >= 2 && f.R <= 4 && f.S >= 2 && f.S <= 4 && f.D >= 2 && f.D <= 4 &&
            g2_smem(N, f) + (stage_out ? kTcM * N * 4 : 0) <= kG2SmemMax)
          dep = f;
      }
      CUtensorMap ma[2], my[2];
      bool ok = make_map_rows(&ma[0], A, n, k, lda, kTcM, kG2KC, false) &&
                (!A2 || make_map_rows(&ma[1], A2, n, k, lda, kTcM, kG2KC, false));
      if (ok && stage_out)
        stage_out = make_map_rows(&my[0], Y, n, c, ldy, kTcM, N, false) &&
                    (!A2 || make_map_rows(&my[1], Y2, n, c, ldy, kTcM, N, false));
      if (!stage_out) my[0] = my[1] = ma[0];  // unused
      const int smem = g2_smem(N, dep) + (stage_out ? kTcM * N * 4 : 0);
      for (int z = 0; ok && z < (A2 ? 2 : 1); ++z) {
        smem_opt_in(reinterpret_cast<const void*>(k_gemm_tma2), kG2SmemMax);
        int64_t ctas = std::min<int64_t>(rtiles, kNumSMs);
        if (g_tc_ablate >> 16) ctas = std::min<int64_t>(ctas, g_tc_ablate >> 16);  // diagnostics
        k_gemm_tma2<<<static_cast<unsigned>(ctas), kG2Threads, smem, s>>>(
            ma[z], my[z], cimg, n, static_cast<int>(k), static_cast<int>(c), N,
            static_cast<int>(tiles_n), rtiles, dep, stage_out, g_tc_twoacc, g_tc_nprod, g_tc_ablate,
            alpha, beta, Z, ldz, z ? Y2 : Y, ldy);
        MPB_LAUNCH_CHECK();
      }
      if (ok) return true;
    }
  }
  // the kernels below cover c in column tiles of <= 128: in place only up to 128
  if (inplace && c > kGtN) return false;
  if (g_gram_tma && n < (int64_t(1) << 31) && k < (int64_t(1) << 31)) {
    // TMA-fed stages; the paired product (A2 C -> Y2) as a second launch
    const int64_t tiles_n = ceil_div(c, kGtN);
    const int64_t ntile = round_up(ceil_div(c, tiles_n), 16);
    const int64_t tiles = ceil_div(n, kTcM) * tiles_n;
    CUtensorMap mc;
    bool ok = make_map_rows(&mc, C, k, c, ldc, kGtKC, static_cast<int>(ntile), true);
    for (int z = 0; ok && z < (A2 ? 2 : 1); ++z) {
      CUtensorMap ma;
      if (!make_map_rows(&ma, z ? A2 : A, n, k, lda, kTcM, kGtKC, false)) {
        ok = false;
        break;
      }
      smem_opt_in(reinterpret_cast<const void*>(k_gemm_tma), kGtSmem);
      const int64_t ctas = std::min<int64_t>(tiles, kNumSMs);
      k_gemm_tma<<<static_cast<unsigned>(ctas), kTmSplitThreads + 64, kGtSmem, s>>>(
          ma, mc, n, static_cast<int>(k), static_cast<int>(c), static_cast<int>(ntile),
          static_cast<int>(tiles_n), tiles, alpha, beta, Z, ldz, z ? Y2 : Y, ldy);
      MPB_LAUNCH_CHECK();
    }
    if (ok) return true;
  }
  if (inplace && c > kGmN) return false;
  const int64_t tiles_n = ceil_div(c, kGmN);
  const int64_t ntile = round_up(ceil_div(c, tiles_n), 16);
  const int64_t tiles = ceil_div(n, kTcM) * tiles_n;
  smem_opt_in(reinterpret_cast<const void*>(k_gemm_tc), kGmSmem);
  // persistent: one CTA per SM (per product of the pair)
  const int64_t ctas = std::min<int64_t>(tiles, A2 ? kNumSMs / 2 : kNumSMs);
  const dim3 grid(static_cast<unsigned>(ctas), 1, A2 ? 2u : 1u);
  k_gemm_tc<<<grid, kTcThreads + 32, kGmSmem, s>>>(n, static_cast<int>(k), static_cast<int>(c),
                                                   static_cast<int>(ntile), static_cast<int>(tiles_n),
                                                   tiles, alpha, A, lda, C, ldc, beta, Z, ldz, Y, ldy,
                                                   A2, Y2);
  MPB_LAUNCH_CHECK();
  return true;
}

}  // namespace mpb
