// Micro-benchmark of the one-warp GS apply (gs_apply_warp) and the compact
// register Levinson, each alone on the GPU: W warps per CTA (each an
// independent problem), 148*16/W CTAs, R repeats per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --extended-lambda
//        -Iinclude -Ipaper_1705_06073_b200/csrc tools/micro/gs_micro.cu -o tools/micro/gs_micro
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "slse_toeplitz.cuh"

using namespace slse;

constexpr int kRegion = 12288;

template <int OP>
__global__ void __launch_bounds__(512, 1) micro_kernel(const cplx* rho_all, const cplx* y_all, const cplx* xh_all,
                                                      cplx* work, int n, int reps, const cplx* tw, int twlog,
                                                      double* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int prob = blockIdx.x * (blockDim.x >> 5) + warp;
  cplx* S = (cplx*)(sm + warp * kRegion);
  double* dt = (double*)(S + 600);
  const int nf = 1 << ilog2(2 * n);
  const cplx* rho = rho_all + (size_t)prob * n;
  const cplx* y = y_all + (size_t)prob * n;
  const cplx* xh = xh_all + (size_t)prob * nf;
  cplx* P = work + (size_t)prob * 5 * nf;
  cplx* U = P + nf;
  cplx* V = U + nf;
  cplx* w = V + nf;
  double acc = 0.0;
  Blk b{lane, 32, (double*)(S + 700), 0};
  for (int r = 0; r < reps; ++r) {
    if (OP == 0) {
      acc += gs_apply_warp(rho, n, ilog2(2 * n), 1.0, y, xh, P, U, V, w, S, tw, twlog, lane);
    } else {
      Factor F = toeplitz_factor_regs_c<8>(y, n, nullptr, dt, w, b);
      acc += F.logdet;
    }
  }
  if (lane == 0) out[prob] = acc;
}

// level-major table (slse_fft.cuh tw_index), T = tw_entries(twlog) entries
__global__ void tw_fill(cplx* tw, int T) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > 0 && i < T) {
    const int l = 31 - __clz(i), k = i - (1 << l);
    double s, c;
    sincospi(-2.0 * k / (double)(1 << l), &s, &c);
    tw[i] = mk(c, s);
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int W = argc > 2 ? atoi(argv[2]) : 16;
  const int reps = argc > 3 ? atoi(argv[3]) : 8;
  const int ctas = 148 * 16 / W, B = ctas * W;
  const int nf = 1 << ilog2(2 * n);
  const int twlog = 10, T = (int)tw_entries(twlog);
  std::vector<cplx> h((size_t)B * nf);
  srand(1);
  for (auto& v : h) v = mk(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  // Toeplitz-like PD columns for the Levinson leg: c0 large
  std::vector<cplx> c((size_t)B * n);
  for (int p = 0; p < B; ++p)
    for (int m = 0; m < n; ++m) c[(size_t)p * n + m] = m == 0 ? mk(2.0, 0.0) : mk(0.5 * cos(0.3 * m) / (1 + m), 0.2 * sin(0.7 * m) / (1 + m));
  cplx *drho, *dy, *dxh, *dwork, *dtw;
  double* dout;
  cudaMalloc(&drho, (size_t)B * n * sizeof(cplx));
  cudaMalloc(&dy, (size_t)B * n * sizeof(cplx));
  cudaMalloc(&dxh, (size_t)B * nf * sizeof(cplx));
  cudaMalloc(&dwork, (size_t)B * 5 * nf * sizeof(cplx));
  cudaMalloc(&dtw, T * sizeof(cplx));
  cudaMalloc(&dout, B * sizeof(double));
  cudaMemcpy(drho, h.data(), (size_t)B * n * sizeof(cplx), cudaMemcpyHostToDevice);
  cudaMemcpy(dy, c.data(), (size_t)B * n * sizeof(cplx), cudaMemcpyHostToDevice);
  cudaMemcpy(dxh, h.data(), (size_t)B * nf * sizeof(cplx), cudaMemcpyHostToDevice);
  tw_fill<<<(T + 255) / 256, 256>>>(dtw, T);
  const size_t smem = (size_t)W * kRegion;
  cudaFuncSetAttribute(micro_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(micro_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int op = 0; op < 2; ++op) {
    float ms = 0;
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(e0);
      if (op == 0) micro_kernel<0><<<ctas, 32 * W, smem>>>(drho, dy, dxh, dwork, n, reps, dtw, twlog, dout);
      else micro_kernel<1><<<ctas, 32 * W, smem>>>(drho, dy, dxh, dwork, n, reps, dtw, twlog, dout);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("%s n=%d W=%d warps=%d reps=%d: %.3f ms  %.2f M calls/s  err=%s\n", op == 0 ? "gs_apply_warp" : "levinson_c",
           n, W, B, reps, ms, (double)B * reps / ms * 1e-3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
