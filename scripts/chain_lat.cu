// chain_lat.cu -- cycles per Givens step of the implicit-QL rotation chain
// (k_small_ql2's serial producer) under a few formulations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/chain_lat.cu -o build/chain_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k_chain(double* dd, double* ee, double* rr, int n, int reps, long long* out) {
  __shared__ double d[64], e[64], r[128];
  if (threadIdx.x < 64) {
    d[threadIdx.x] = dd[threadIdx.x];
    e[threadIdx.x] = ee[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < reps; ++rep) {
    double g = d[n - 1] - d[0] + 0.25, sn = 1, cs = 1, pp = 0;
    double ei = e[n - 2], di = d[n - 2], di1 = d[n - 1];
    int nrot = 0;
    for (int i1 = n - 2; i1 >= 0; --i1) {
      const double ei_next = i1 > 0 ? e[i1 - 1] : 0.0;
      const double di_next = i1 > 0 ? d[i1 - 1] : 0.0;
      const double f = sn * ei;
      const double bb = cs * ei;
      const double r2 = fma(f, f, g * g);
      if (V == 0) {
        if (r2 == 0.0) break;
        const double gg = di1 - pp;
        const double u = fma(di - gg, f, 2.0 * g * bb);
        const double rinv = rsqrt(r2);
        e[i1 + 1] = r2 * rinv;
        sn = f * rinv;
        cs = g * rinv;
        const double rq = u * rinv;
        pp = sn * rq;
        d[i1 + 1] = gg + pp;
        g = fma(cs, rq, -bb);
        r[2 * nrot] = cs;
        r[2 * nrot + 1] = sn;
      } else if (V == 1) {  // no zero test, no stores
        const double gg = di1 - pp;
        const double u = fma(di - gg, f, 2.0 * g * bb);
        const double rinv = rsqrt(r2);
        acc += r2 * rinv;
        sn = f * rinv;
        cs = g * rinv;
        const double rq = u * rinv;
        pp = sn * rq;
        acc += gg + pp;
        g = fma(cs, rq, -bb);
      } else if (V == 2) {  // float-seeded Newton rsqrt
        const double gg = di1 - pp;
        const double u = fma(di - gg, f, 2.0 * g * bb);
        double y = static_cast<double>(rsqrtf(static_cast<float>(r2)));
        const double h = 0.5 * r2;
        y = y * fma(-h, y * y, 1.5);
        y = y * fma(-h, y * y, 1.5);
        const double rinv = y;
        e[i1 + 1] = r2 * rinv;
        sn = f * rinv;
        cs = g * rinv;
        const double rq = u * rinv;
        pp = sn * rq;
        d[i1 + 1] = gg + pp;
        g = fma(cs, rq, -bb);
        r[2 * nrot] = cs;
        r[2 * nrot + 1] = sn;
      } else if (V == 3) {  // stores kept, zero test deferred to after the chain
        const double gg = di1 - pp;
        const double u = fma(di - gg, f, 2.0 * g * bb);
        const double rinv = rsqrt(r2);
        e[i1 + 1] = r2 * rinv;
        sn = f * rinv;
        cs = g * rinv;
        const double rq = u * rinv;
        pp = sn * rq;
        d[i1 + 1] = gg + pp;
        g = fma(cs, rq, -bb);
        r[2 * nrot] = cs;
        r[2 * nrot + 1] = sn;
      } else if (V == 5 || V == 6) {  // MUFU seed + one 3rd-order Newton step, no range branch
        const double gg = di1 - pp;
        const double u = fma(di - gg, f, 2.0 * g * bb);
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
        const double t = fma(-r2 * y, y, 1.0);
        const double rinv = fma(y * t, fma(0.375, t, 0.5), y);
        if (V == 5) e[i1 + 1] = r2 * rinv; else acc += r2 * rinv;
        sn = f * rinv;
        cs = g * rinv;
        const double rq = u * rinv;
        pp = sn * rq;
        if (V == 5) d[i1 + 1] = gg + pp; else acc += gg + pp;
        g = fma(cs, rq, -bb);
        if (V == 5) {
          r[2 * nrot] = cs;
          r[2 * nrot + 1] = sn;
        }
      } else if (V == 4) {  // sqrt + two divides (reference formulation)
        const double rr2 = sqrt(r2);
        if (rr2 == 0.0) break;
        e[i1 + 1] = rr2;
        sn = f / rr2;
        cs = g / rr2;
        const double gg = di1 - pp;
        const double rq = (di - gg) * sn + 2.0 * cs * bb;
        pp = sn * rq;
        d[i1 + 1] = gg + pp;
        g = cs * rq - bb;
        r[2 * nrot] = cs;
        r[2 * nrot + 1] = sn;
      }
      ++nrot;
      ei = ei_next;
      di1 = di;
      di = di_next;
    }
    acc += g + pp + r[nrot] + e[1];
    d[0] = d[0] * 0.5 + 1.0;
  }
  long long t1 = clock64();
  out[V] = t1 - t0;
  if (acc == 12345.0) out[7] = 1;
  (void)rr;
}

int main() {
  double hd[64], he[64];
  for (int i = 0; i < 64; ++i) {
    hd[i] = 1.0 + i * 0.37;
    he[i] = 0.3 + 0.01 * i;
  }
  double *dd, *ee, *rr;
  long long* out;
  cudaMalloc(&dd, 512);
  cudaMalloc(&ee, 512);
  cudaMalloc(&rr, 1024);
  cudaMalloc(&out, 64);
  cudaMemcpy(dd, hd, 512, cudaMemcpyHostToDevice);
  cudaMemcpy(ee, he, 512, cudaMemcpyHostToDevice);
  const int n = 48, reps = 200;
  k_chain<0><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<1><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<2><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<3><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<4><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<5><<<1, 64>>>(dd, ee, rr, n, reps, out);
  k_chain<6><<<1, 64>>>(dd, ee, rr, n, reps, out);
  long long h[8];
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
  const char* names[] = {"current (zero test, smem stores)", "no test, no stores", "f32-seeded newton",
                         "no zero test, stores", "sqrt + 2 div (reference form)",
                         "approx seed + 1 Newton, stores", "approx seed + 1 Newton, no stores"};
  for (int v = 0; v < 7; ++v)
    printf("chain variant %d %-36s %.1f cycles/step\n", v, names[v], double(h[v]) / (reps * (n - 1)));
  return 0;
}
