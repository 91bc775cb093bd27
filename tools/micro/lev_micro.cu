// Micro-benchmark of the one-warp Schur-Levinson variants used by the N<=256
// solver path: register-resident (toeplitz_factor_regs) vs shared-memory
// (toeplitz_factor_warp).  One warp per problem, B problems, R repeats.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda
//        -Iinclude -Ipaper_1705_06073_b200/csrc tools/micro/lev_micro.cu -o /tmp/lev_micro
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "slse_toeplitz.cuh"

using namespace slse;

template <int V>
__global__ void __launch_bounds__(32, 16) lev_kernel(const cplx* cols, int n, int reps, cplx* rho_out, double* logdet) {
  __shared__ double red[64];
  __shared__ cplx E[512];
  __shared__ double dt[256];
  Blk b{(int)threadIdx.x, 32, red, 0};
  const cplx* c = cols + (size_t)blockIdx.x * n;
  cplx* rho = rho_out + (size_t)blockIdx.x * n;
  double ld = 0.0;
  for (int r = 0; r < reps; ++r) {
    Factor F = V == 0 ? toeplitz_factor_regs<8>(c, n, nullptr, dt, rho, b)
                      : toeplitz_factor_warp<8>(c, n, E, nullptr, dt, rho, b);
    ld += F.logdet + F.status;
  }
  if (threadIdx.x == 0) logdet[blockIdx.x] = ld;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int B = argc > 2 ? atoi(argv[2]) : 4736;
  const int reps = argc > 3 ? atoi(argv[3]) : 8;
  std::vector<cplx> h((size_t)B * n);
  srand(1);
  for (int p = 0; p < B; ++p) {
    // c_m = beta [m==0] + sum_k g_k e^{j 2 pi m th_k}
    for (int m = 0; m < n; ++m) h[(size_t)p * n + m] = mk(m == 0 ? 0.05 : 0.0, 0.0);
    for (int k = 0; k < 16; ++k) {
      const double th = rand() / (double)RAND_MAX, g = 0.5 + rand() / (double)RAND_MAX;
      for (int m = 0; m < n; ++m) {
        h[(size_t)p * n + m].re += g * cos(2 * M_PI * m * th);
        h[(size_t)p * n + m].im += g * sin(2 * M_PI * m * th);
      }
    }
    h[(size_t)p * n].im = 0.0;
  }
  cplx *dc, *r0, *r1;
  double *l0, *l1;
  cudaMalloc(&dc, h.size() * sizeof(cplx));
  cudaMalloc(&r0, h.size() * sizeof(cplx));
  cudaMalloc(&r1, h.size() * sizeof(cplx));
  cudaMalloc(&l0, B * sizeof(double));
  cudaMalloc(&l1, B * sizeof(double));
  cudaMemcpy(dc, h.data(), h.size() * sizeof(cplx), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms[2];
  for (int v = 0; v < 2; ++v) {
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(e0);
      if (v == 0) lev_kernel<0><<<B, 32>>>(dc, n, reps, r0, l0);
      else lev_kernel<1><<<B, 32>>>(dc, n, reps, r1, l1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[v], e0, e1);
    }
  }
  std::vector<cplx> a(h.size()), c(h.size());
  std::vector<double> la(B), lb(B);
  cudaMemcpy(a.data(), r0, h.size() * sizeof(cplx), cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), r1, h.size() * sizeof(cplx), cudaMemcpyDeviceToHost);
  cudaMemcpy(la.data(), l0, B * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(lb.data(), l1, B * sizeof(double), cudaMemcpyDeviceToHost);
  double md = 0, mx = 0, ldd = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    md = fmax(md, fabs(a[i].re - c[i].re) + fabs(a[i].im - c[i].im));
    mx = fmax(mx, fabs(c[i].re) + fabs(c[i].im));
  }
  for (int p = 0; p < B; ++p) ldd = fmax(ldd, fabs(la[p] - lb[p]) / fmax(1.0, fabs(lb[p])));
  const double builds = (double)B * reps;
  printf("n=%d B=%d reps=%d  regs: %.3f ms (%.2f us/build-slot, %.0f builds/s)  smem: %.3f ms (%.0f builds/s)  "
         "max|drho|/max|rho| = %.2e  logdet rel = %.2e  err=%s\n",
         n, B, reps, ms[0], 1e3 * ms[0] / builds, builds / ms[0] * 1e3, ms[1], builds / ms[1] * 1e3, md / mx, ldd,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
