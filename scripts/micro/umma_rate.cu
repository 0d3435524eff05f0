// tcgen05.mma (kind::f16, bf16 -> fp32, cta_group::1, M = 128) issue rate per
// SM for the shared-memory operand layouts the tc.cu kernels use:
//   layout 0: A, B K-major, no swizzle (core matrices 8 rows x 16 B)
//   layout 1: A MN-major no swizzle (k_gemm_tma*), B K-major no swizzle
//   layout 2: A, B K-major, 128-B swizzle
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |
         (static_cast<uint64_t>(layout) << 61);
}

// bounded wait: false after ~2^31 cycles (a faulting MMA never arrives)
__device__ bool wait_bar(uint64_t* bar, uint32_t phase) {
  const long long t0 = clock64();
  while (true) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase));
    if (ok) return true;
    if (clock64() - t0 > (1ll << 31)) return false;
  }
}

__global__ void __launch_bounds__(128, 1) k_rate(int N, int layout, int iters, long long* cyc, int mode) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(8) uint64_t bar2[2];
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar[1])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar2[0])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar2[1])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sm), b0 = a0 + 48 * 1024;
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
    if (layout == 1) idesc |= 1u << 15;
    uint64_t ad[2], bd[2];
    for (int kk = 0; kk < 2; ++kk) {
      if (layout == 0) {
        ad[kk] = desc(a0 + kk * 256, 128, 512, 0);
        bd[kk] = desc(b0 + kk * 256, 128, 512, 0);
      } else if (layout == 1) {
        ad[kk] = desc(a0 + kk * 256, 128, 528, 0);
        bd[kk] = desc(b0 + kk * 256, 128, 512, 0);
      } else {
        ad[kk] = desc(a0 + kk * 32, 16, 1024, 2);
        bd[kk] = desc(b0 + kk * 32, 16, 1024, 2);
      }
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      if (mode >= 4 && it >= 1) {  // the MMA warp waits on an already completed barrier + fence
        wait_bar(&bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
      }
      if (mode >= 2) asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // mode 0: alternate two accumulators; mode >= 1: 2 MMAs to acc 0 then 14 to acc 1
        const uint32_t acc = mode == 0 ? (j & 1) * 256 : (j < 2 ? 0 : 256);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + acc),
                     "l"(ad[j & 1]), "l"(bd[j & 1]), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar[it & 1])));
      if (mode >= 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar2[it & 1])));
      if (it >= 1) {  // keep at most two batches in flight (one barrier each)
        const int p = it - 1;
        if (!wait_bar(&bar[p & 1], (p >> 1) & 1)) { cyc[blockIdx.x] = -1; break; }
      }
    }
    if (!wait_bar(&bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1)) cyc[blockIdx.x] = -1;
    long long t1 = clock64();
    if (cyc[blockIdx.x] >= 0) cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode)
    for (int N : {80, 160}) {
      const int layout = 1;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaMemset(d, 0, 148 * sizeof(long long));
        cudaEventRecord(e0);
        k_rate<<<148, 128, smem>>>(N, layout, iters, d, mode);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        if (err != cudaSuccess || h[0] < 0) { printf("mode %d N %d: %s / timeout\n", mode, N, cudaGetErrorString(err)); return 1; }
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        if (rep)
          printf("mode %d N %3d: %7.1f clk/MMA (floor %5.1f)\n", mode, N, avg / (iters * 16.0), 128.0 * N / 256);
      }
    }
  return 0;
}
