// microbench.cu -- device peaks and per-kernel throughput of the hot-path kernels.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2302_12528_b200/csrc \
//        scripts/microbench.cu -L paper_2302_12528_b200 -lmpeig_b200 -lcublas -lcusolver -o build/microbench
//
// Prints one line per measurement: name, time per launch, algorithmic GB/s and GFLOP/s.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#include "kernels.cuh"

using namespace mpb;

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)


static double time_ms(std::function<void()> f, int reps, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) f();
  CK(cudaStreamSynchronize(s));
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b, s);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

static void report(const char* name, double ms, double bytes, double flops) {
  printf("%-44s %10.4f ms  %9.1f GB/s  %9.1f GFLOP/s\n", name, ms, bytes / ms / 1e6, flops / ms / 1e6);
  fflush(stdout);
}

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5) out[0] = 1;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  if (s == 1234.5) out[0] = 1;
}

__global__ void k_dmma16(double* out, int iters) {
  double a[8], b[4];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-9 + q;
  for (int q = 0; q < 4; ++q) b[q] = 1.0 + q;
  double c[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int q = 0; q < 2; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 1234.5) out[0] = 1;
}

// single-thread dependent-chain latencies (cycles per op)
__global__ void k_lat(double* out, long long* cyc, double x0) {
  double x = x0, y = x0 * 0.5 + 1.0;
  float xf = static_cast<float>(x0);
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) x = rsqrt(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) x = 1.0 / (x + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) x = sqrt(x + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) xf = fmaf(xf, 0.999999f, 1e-7f);
  long long t5 = clock64();
  for (int i = 0; i < 256; ++i) y = y * x + 0.5;
  long long t6 = clock64();
  out[0] = x + y + xf;
  cyc[0] = (t1 - t0) / 256;
  cyc[1] = (t2 - t1) / 256;
  cyc[2] = (t3 - t2) / 256;
  cyc[3] = (t4 - t3) / 256;
  cyc[4] = (t5 - t4) / 256;
  cyc[5] = (t6 - t5) / 256;
}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main(int argc, char** argv) {
  const bool quick = argc > 1;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  double* dummy;
  CK(cudaMalloc(&dummy, 64));
  {
    long long* cyc;
    CK(cudaMalloc(&cyc, 64));
    k_lat<<<1, 1, 0, s>>>(dummy, cyc, 0.5);
    CK(cudaStreamSynchronize(s));
    long long h[6];
    CK(cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost));
    printf("latency (cycles/op): dfma %lld  drsqrt %lld  ddiv %lld  dsqrt %lld  ffma %lld  dmul+dadd %lld\n", h[0],
           h[1] - 1, h[2] - 1, h[3] - 1, h[4], h[5]);
  }
  // ---- peaks
  {
    const int iters = 4096;
    const int blocks = 148 * 8, threads = 256;
    double ms = time_ms([&] { k_dfma<<<blocks, threads, 0, s>>>(dummy, iters); }, 5, s);
    report("peak DFMA (8 chains/thread)", ms, 0, 2.0 * 8 * iters * blocks * threads);
    ms = time_ms([&] { k_dmma<<<blocks, threads, 0, s>>>(dummy, iters); }, 5, s);
    report("peak DMMA m8n8k4", ms, 0, 2.0 * 8 * 8 * 4 * 4 * iters * (blocks * threads / 32));
    ms = time_ms([&] { k_dmma16<<<blocks, threads, 0, s>>>(dummy, iters / 4); }, 5, s);
    report("peak DMMA m16n8k16", ms, 0, 2.0 * 16 * 8 * 16 * 2 * (iters / 4) * (blocks * threads / 32));
  }
  {
    const size_t n = size_t(1) << 28;  // 2 GiB
    double *a, *b;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    CK(cudaMemset(a, 0, n * 8));
    double ms = time_ms([&] { k_copy<<<148 * 16, 256, 0, s>>>((double4*)a, (double4*)b, n / 4); }, 5, s);
    report("HBM copy (read+write)", ms, 2.0 * n * 8, 0);
    CK(cudaFree(a));
    CK(cudaFree(b));
  }
  {
    cublasHandle_t h;
    cublasCreate(&h);
    cublasSetStream(h, s);
    const int N = 8192;
    double *A, *B, *C;
    CK(cudaMalloc(&A, (size_t)N * N * 8));
    CK(cudaMalloc(&B, (size_t)N * N * 8));
    CK(cudaMalloc(&C, (size_t)N * N * 8));
    CK(cudaMemset(A, 0, (size_t)N * N * 8));
    CK(cudaMemset(B, 0, (size_t)N * N * 8));
    const double one = 1, zero = 0;
    double ms = time_ms([&] { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N); }, 3, s);
    report("cuBLAS DGEMM 8192^3", ms, 0, 2.0 * N * N * (double)N);
    // tall-skinny Gram via cuBLAS for comparison: n=1M, 144x144
    const int n = 1 << 20, k = 144;
    double *X, *G;
    CK(cudaMalloc(&X, (size_t)n * k * 8));
    CK(cudaMalloc(&G, (size_t)k * k * 8));
    CK(cudaMemset(X, 0, (size_t)n * k * 8));
    ms = time_ms([&] { cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, k, k, n, &one, X, n, X, n, &zero, G, k); }, 5, s);
    report("cuBLAS DGEMM^T gram n=1M 144x144", ms, 2.0 * n * k * 8, 2.0 * n * k * (double)k);
    CK(cudaFree(A));
    CK(cudaFree(B));
    CK(cudaFree(C));
    CK(cudaFree(X));
    CK(cudaFree(G));
    cublasDestroy(h);
  }
  // ---- small eig options
  {
    cusolverDnHandle_t h;
    cusolverDnCreate(&h);
    cusolverDnSetStream(h, s);
    for (int sdim : {18, 48, 96, 144, 240, 576}) {
      std::vector<double> Mh((size_t)sdim * sdim);
      for (int j = 0; j < sdim; ++j)
        for (int i = 0; i < sdim; ++i) Mh[i + (size_t)j * sdim] = (i == j) ? 1.0 + i : 1.0 / (1 + i + j);
      double *M, *Mw, *W, *work;
      int* info;
      CK(cudaMalloc(&M, Mh.size() * 8));
      CK(cudaMalloc(&Mw, Mh.size() * 8));
      CK(cudaMalloc(&W, sdim * 8));
      CK(cudaMalloc(&info, 4));
      CK(cudaMemcpy(M, Mh.data(), Mh.size() * 8, cudaMemcpyHostToDevice));
      int lw = 0;
      cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, Mw, sdim, W, &lw);
      CK(cudaMalloc(&work, (size_t)lw * 8));
      char name[64];
      double ms = time_ms([&] {
        cudaMemcpyAsync(Mw, M, Mh.size() * 8, cudaMemcpyDeviceToDevice, s);
        cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, Mw, sdim, W, work, lw, info);
      }, 10, s);
      snprintf(name, sizeof name, "syevd s=%d", sdim);
      report(name, ms, 0, 0);
      CK(cudaFree(work));
      syevjInfo_t jp;
      cusolverDnCreateSyevjInfo(&jp);
      cusolverDnXsyevjSetTolerance(jp, 1e-15);
      cusolverDnXsyevjSetMaxSweeps(jp, 100);
      cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, Mw, sdim, W, &lw, jp);
      CK(cudaMalloc(&work, (size_t)lw * 8));
      ms = time_ms([&] {
        cudaMemcpyAsync(Mw, M, Mh.size() * 8, cudaMemcpyDeviceToDevice, s);
        cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, Mw, sdim, W, work, lw, info, jp);
      }, 10, s);
      snprintf(name, sizeof name, "syevj s=%d", sdim);
      report(name, ms, 0, 0);
      CK(cudaFree(work));
      cusolverDnParams_t prm;
      cusolverDnCreateParams(&prm);
      size_t dws = 0, hws = 0;
      cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, CUDA_R_64F, Mw,
                                        sdim, CUDA_R_64F, W, CUDA_R_64F, &dws, &hws, 1);
      void* dw;
      CK(cudaMalloc(&dw, dws + 8));
      std::vector<char> hw(hws + 8);
      ms = time_ms([&] {
        cudaMemcpyAsync(Mw, M, Mh.size() * 8, cudaMemcpyDeviceToDevice, s);
        cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, sdim, CUDA_R_64F, Mw, sdim,
                               CUDA_R_64F, W, CUDA_R_64F, dw, dws, hw.data(), hws, info, 1);
      }, 10, s);
      snprintf(name, sizeof name, "XsyevBatched(1) s=%d", sdim);
      report(name, ms, 0, 0);
      if (small_syev_supported<double>(sdim)) {
        ms = time_ms([&] {
          cudaMemcpyAsync(Mw, M, Mh.size() * 8, cudaMemcpyDeviceToDevice, s);
          small_syev<double>(sdim, Mw, sdim, W, info, s);
        }, 10, s);
        long long* dprof;
        CK(cudaMalloc(&dprof, 64));
        CK(cudaMemset(dprof, 0, 64));
        cudaMemcpyAsync(Mw, M, Mh.size() * 8, cudaMemcpyDeviceToDevice, s);
        small_syev_prof<double>(sdim, Mw, sdim, W, info, dprof, s);
        long long hp[8];
        CK(cudaMemcpy(hp, dprof, sizeof hp, cudaMemcpyDeviceToHost));
        snprintf(name, sizeof name, "mpb small_syev<double> s=%d", sdim);
        report(name, ms, 0, 0);
        printf("  phases (cycles): tridiag %lld [norm %lld mv %lld upd %lld]  QL %lld  sort %lld  sweeps %lld  chain %lld\n",
               hp[0], hp[5], hp[6], hp[7], hp[1], hp[2], hp[3], hp[4]);
        cudaFree(dprof);
        {  // correctness of both precisions on the same matrix
          std::vector<double> V((size_t)sdim * sdim), lam(sdim);
          CK(cudaMemcpy(V.data(), Mw, V.size() * 8, cudaMemcpyDeviceToHost));
          CK(cudaMemcpy(lam.data(), W, sdim * 8, cudaMemcpyDeviceToHost));
          double orth = 0, res = 0;
          for (int a = 0; a < sdim; ++a)
            for (int b = 0; b < sdim; ++b) {
              double o = 0, r = 0;
              for (int i = 0; i < sdim; ++i) {
                o += V[i + (size_t)a * sdim] * V[i + (size_t)b * sdim];
                r += Mh[a + (size_t)i * sdim] * V[i + (size_t)b * sdim];
              }
              orth = std::max(orth, std::fabs(o - (a == b)));
              res = std::max(res, std::fabs(r - lam[b] * V[a + (size_t)b * sdim]));
            }
          printf("  f64 check s=%d: orth %.2e resid %.2e\n", sdim, orth, res);
          std::vector<float> Mf(Mh.begin(), Mh.end());
          float *Mfd, *Wf;
          CK(cudaMalloc(&Mfd, Mf.size() * 4));
          CK(cudaMalloc(&Wf, sdim * 4));
          CK(cudaMemcpy(Mfd, Mf.data(), Mf.size() * 4, cudaMemcpyHostToDevice));
          small_syev<float>(sdim, Mfd, sdim, Wf, info, s);
          std::vector<float> Vf((size_t)sdim * sdim), lf(sdim);
          CK(cudaMemcpy(Vf.data(), Mfd, Vf.size() * 4, cudaMemcpyDeviceToHost));
          CK(cudaMemcpy(lf.data(), Wf, sdim * 4, cudaMemcpyDeviceToHost));
          orth = res = 0;
          int nan = 0;
          for (int a = 0; a < sdim; ++a)
            for (int b = 0; b < sdim; ++b) {
              double o = 0, r = 0;
              for (int i = 0; i < sdim; ++i) {
                o += (double)Vf[i + (size_t)a * sdim] * Vf[i + (size_t)b * sdim];
                r += (double)Mf[a + (size_t)i * sdim] * Vf[i + (size_t)b * sdim];
              }
              if (std::isnan(o) || std::isnan(r)) ++nan;
              orth = std::max(orth, std::fabs(o - (a == b)));
              res = std::max(res, std::fabs(r - lf[b] * Vf[a + (size_t)b * sdim]));
            }
          printf("  f32 check s=%d: orth %.2e resid %.2e nan %d lam0 %g\n", sdim, orth, res, nan, lf[0]);
          {
            float* Mfw;
            CK(cudaMalloc(&Mfw, Mf.size() * 4));
            CK(cudaMemcpy(Mfd, Mf.data(), Mf.size() * 4, cudaMemcpyHostToDevice));
            const double msf = time_ms([&] {
              cudaMemcpyAsync(Mfw, Mfd, Mf.size() * 4, cudaMemcpyDeviceToDevice, s);
              small_syev<float>(sdim, Mfw, sdim, Wf, info, s);
            }, 10, s);
            snprintf(name, sizeof name, "mpb small_syev<float> s=%d", sdim);
            report(name, msf, 0, 0);
            long long* dpf;
            CK(cudaMalloc(&dpf, 64));
            CK(cudaMemset(dpf, 0, 64));
            cudaMemcpyAsync(Mfw, Mfd, Mf.size() * 4, cudaMemcpyDeviceToDevice, s);
            small_syev_prof<float>(sdim, Mfw, sdim, Wf, info, dpf, s);
            long long hpf[5];
            CK(cudaMemcpy(hpf, dpf, sizeof hpf, cudaMemcpyDeviceToHost));
            printf("  f32 phases (cycles): tridiag %lld  QL %lld  sort %lld  sweeps %lld  chain %lld\n", hpf[0],
                   hpf[1], hpf[2], hpf[3], hpf[4]);
            cudaFree(dpf);
            cudaFree(Mfw);
          }
          cudaFree(Mfd);
          cudaFree(Wf);
        }
      }
      CK(cudaFree(dw));
      CK(cudaFree(M));
      CK(cudaFree(Mw));
      CK(cudaFree(W));
      CK(cudaFree(info));
    }
    cusolverDnDestroy(h);
  }
  if (quick) return 0;
  // ---- hot-path kernels
  {
    struct Shape {
      int64_t n, k;
      const char* tag;
    } shapes[] = {{32768, 48, "cfg1 n=32768 s=48"}, {1 << 20, 144, "cfg2 n=1M s=144"},
                  {2097152, 240, "cfg4@8 n=2M s=240"}};
    for (auto sh : shapes) {
      const int64_t n = sh.n, k = sh.k, m = k / 3;
      double *S, *AS, *G, *Y, *work;
      CK(cudaMalloc(&S, n * k * 8));
      CK(cudaMalloc(&AS, n * k * 8));
      CK(cudaMalloc(&Y, n * k * 8));
      CK(cudaMalloc(&G, k * k * 8));
      CK(cudaMemset(S, 0, n * k * 8));
      CK(cudaMemset(AS, 0, n * k * 8));
      const int64_t gw = gram_workspace_elems<double>(n, k, k);
      CK(cudaMalloc(&work, gw * 8 + 64));
      CK(cudaMemset(work, 0, gw * 8 + 64));
      char name[96];
      double ms = time_ms([&] { gram<double>(n, k, S, n, k, AS, n, G, k, 1, work, s); }, 5, s);
      snprintf(name, sizeof name, "gram S^T AS %s", sh.tag);
      report(name, ms, 2.0 * n * k * 8, 2.0 * n * k * k);
      ms = time_ms([&] { gram<double>(n, 2 * m, S, n, m, S + 2 * m * n, n, G, 2 * m, 0, work, s); }, 5, s);
      snprintf(name, sizeof name, "gram B^T W (2m x m) %s", sh.tag);
      report(name, ms, 3.0 * n * m * 8, 2.0 * n * 2 * m * m);
      {
        float* wf;
        const int64_t gwf = gram_workspace_elems<float>(n, k, k);
        CK(cudaMalloc(&wf, gwf * 4 + 64));
        CK(cudaMemset(wf, 0, gwf * 4 + 64));
        const float* Sf = reinterpret_cast<const float*>(S);
        const float* ASf = reinterpret_cast<const float*>(AS);
        ms = time_ms([&] { gram<float>(n, k, Sf, n, k, ASf, n, reinterpret_cast<float*>(G), k, 1, wf, s); }, 5, s);
        snprintf(name, sizeof name, "gram<float> S^T AS %s", sh.tag);
        report(name, ms, 2.0 * n * k * 4, 2.0 * n * k * k);
        CK(cudaFree(wf));
      }
      ms = time_ms([&] { gemm_tn<double>(n, k, 2 * m, 1.0, S, n, G, k, 0.0, nullptr, 0, Y, n, s); }, 5, s);
      snprintf(name, sizeof name, "gemm S C (s -> 2m) %s", sh.tag);
      report(name, ms, (double)(n * k + n * 2 * m) * 8, 2.0 * n * k * 2 * m);
      ms = time_ms([&] { gemm_tn<double>(n, 2 * m, m, -1.0, S, n, G, 2 * m, 1.0, Y, n, Y, n, s); }, 5, s);
      snprintf(name, sizeof name, "gemm W -= B G %s", sh.tag);
      report(name, ms, (double)(n * 2 * m + 2 * n * m) * 8, 2.0 * n * 2 * m * m);
      {
        const float* Sf = reinterpret_cast<const float*>(S);
        const float* Gf = reinterpret_cast<const float*>(G);
        float* Yf = reinterpret_cast<float*>(Y);
        ms = time_ms([&] { gemm_tn<float>(n, k, 2 * m, 1.f, Sf, n, Gf, k, 0.f, nullptr, 0, Yf, n, s); }, 5, s);
        snprintf(name, sizeof name, "gemm<float> S C (s -> 2m) %s", sh.tag);
        report(name, ms, (double)(n * k + n * 2 * m) * 4, 2.0 * n * k * 2 * m);
      }
      double* Rt;
      CK(cudaMalloc(&Rt, m * m * 8));
      int* st;
      CK(cudaMalloc(&st, 64));
      CK(cudaMemset(st, 0, 64));
      // tsqr on a well-conditioned block: fill with something non-degenerate
      std::vector<double> hcol(n);
      for (int64_t i = 0; i < n; ++i) hcol[i] = 1.0 / (1 + (i * 7919) % 1000);
      for (int64_t j = 0; j < m; ++j) {
        for (int64_t i = 0; i < n; ++i) hcol[i] = ((i * (j + 3) * 2654435761ULL) % 1000003) * 1e-6 - 0.5;
        CK(cudaMemcpy(S + j * n, hcol.data(), n * 8, cudaMemcpyHostToDevice));
      }
      float* tw;
      const int64_t tws = tsqr_workspace_elems<double, float>(n, m);
      CK(cudaMalloc(&tw, tws * 4 + 64));
      CK(cudaMemset(tw, 0, tws * 4 + 64));
      float* Rf;
      CK(cudaMalloc(&Rf, m * m * 4));
      ms = time_ms([&] { tsqr_r<double, float>(n, m, S, n, Rf, m, tw, st, s); }, 5, s);
      snprintf(name, sizeof name, "tsqr fp32(R) from fp64 W %s", sh.tag);
      report(name, ms, (double)n * m * 8, 2.0 * n * m * m);
      double* tw64;
      const int64_t tws64 = tsqr_workspace_elems<double, double>(n, m);
      CK(cudaMalloc(&tw64, tws64 * 8 + 64));
      CK(cudaMemset(tw64, 0, tws64 * 8 + 64));
      ms = time_ms([&] { tsqr_r<double, double>(n, m, S, n, Rt, m, tw64, st, s); }, 5, s);
      snprintf(name, sizeof name, "tsqr fp64 %s", sh.tag);
      report(name, ms, (double)n * m * 8, 2.0 * n * m * m);
      double* rw;
      CK(cudaMalloc(&rw, (resid_workspace_elems(n, m) + 4 * m) * 8));
      ms = time_ms([&] {
        residual_precond<double>(kResidPlain, n, m, S, n, AS, n, G, nullptr, Y, n, rw, rw + 2 * m, st, rw + 4 * m, s);
      }, 5, s);
      snprintf(name, sizeof name, "residual+norms %s", sh.tag);
      report(name, ms, 3.0 * n * m * 8, 4.0 * n * m);
      CK(cudaFree(S));
      CK(cudaFree(AS));
      CK(cudaFree(Y));
      CK(cudaFree(G));
      CK(cudaFree(work));
      CK(cudaFree(Rt));
      CK(cudaFree(st));
      CK(cudaFree(tw));
      CK(cudaFree(Rf));
      CK(cudaFree(tw64));
      CK(cudaFree(rw));
    }
    // stencils
    {
      const int64_t N = 256, n = N * N * N, c = 16;
      double *X, *Y;
      CK(cudaMalloc(&X, n * c * 8));
      CK(cudaMalloc(&Y, n * c * 8));
      CK(cudaMemset(X, 0, n * c * 8));
      double ms = time_ms([&] { stencil7<double>(N, N, N, c, X, n, Y, n, s); }, 5, s);
      report("stencil7 256^3 x16 fp64", ms, 2.0 * n * c * 8, 13.0 * n * c);
      ms = time_ms([&] { stencil7<float>(N, N, N, c, (float*)X, n, (float*)Y, n, s); }, 5, s);
      report("stencil7 256^3 x16 fp32", ms, 2.0 * n * c * 4, 13.0 * n * c);
      const int64_t M2 = 1024, n2 = M2 * M2, c2 = 48;
      ms = time_ms([&] { stencil5<double>(M2, M2, c2, X, n2, Y, n2, s); }, 5, s);
      report("stencil5 1024^2 x48 fp64", ms, 2.0 * n2 * c2 * 8, 9.0 * n2 * c2);
      CK(cudaFree(X));
      CK(cudaFree(Y));
    }
  }
  return 0;
}
