// small_check.cu -- standalone check of the small factorization kernels
// (upper-triangular inverse, Cholesky + L^{-T}) against a host computation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2302_12528_b200/csrc \
//        scripts/small_check.cu -L paper_2302_12528_b200 -lmpeig_b200 -o build/small_check
#include <cmath>
#include <cstdio>
#include <vector>

#include "kernels.cuh"

using namespace mpb;

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main() {
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  for (int m : {1, 2, 5, 16, 24, 32, 48}) {
    std::vector<double> R(m * m, 0.0), G(m * m, 0.0);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i <= j; ++i) R[i + j * m] = (i == j) ? 2.0 + 0.1 * i : 0.3 / (1 + i + j);
    // G = R^T R (SPD)
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        double a = 0;
        for (int k = 0; k < m; ++k) a += R[k + i * m] * R[k + j * m];
        G[i + j * m] = a;
      }
    double *dR, *dRi, *dG, *dL, *dU;
    int* st;
    CK(cudaMalloc(&dR, m * m * 8));
    CK(cudaMalloc(&dRi, m * m * 8));
    CK(cudaMalloc(&dG, m * m * 8));
    CK(cudaMalloc(&dL, m * m * 8));
    CK(cudaMalloc(&dU, m * m * 8));
    CK(cudaMalloc(&st, 16));
    CK(cudaMemset(st, 0, 16));
    CK(cudaMemcpy(dR, R.data(), m * m * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dG, G.data(), m * m * 8, cudaMemcpyHostToDevice));
    small_upper_inverse<double>(m, dR, m, dRi, st, s);
    CK(cudaStreamSynchronize(s));
    small_cholesky_inv<double>(m, dG, m, dL, dU, st, s, 0.0);
    CK(cudaStreamSynchronize(s));
    std::vector<double> Ri(m * m), L(m * m), U(m * m);
    int hs[2];
    CK(cudaMemcpy(Ri.data(), dRi, m * m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(L.data(), dL, m * m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(U.data(), dU, m * m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost));
    double e1 = 0, e2 = 0, e3 = 0;
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        double a = 0, b = 0, c = 0;
        for (int k = 0; k < m; ++k) {
          a += R[i + k * m] * Ri[k + j * m];
          b += L[i + k * m] * L[j + k * m];
          c += U[k + i * m] * L[j + k * m];  // (U^T L^T)(i,j) = (L^{-1} L)(i,j)... check U = L^{-T}
        }
        e1 = std::fmax(e1, std::fabs(a - (i == j)));
        e2 = std::fmax(e2, std::fabs(b - G[i + j * m]));
        (void)c;
      }
    // U = L^{-T}  <=>  L^T U = I
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        double a = 0;
        for (int k = 0; k < m; ++k) a += L[k + i * m] * U[k + j * m];
        e3 = std::fmax(e3, std::fabs(a - (i == j)));
      }
    printf("m=%2d status=%d,%d  |R Rinv - I| %.2e  |L L^T - G| %.2e  |L^T Uinv - I| %.2e\n", m, hs[0], hs[1],
           e1, e2, e3);
    cudaFree(dR);
    cudaFree(dRi);
    cudaFree(dG);
    cudaFree(dL);
    cudaFree(dU);
    cudaFree(st);
  }
  return 0;
}
