// Per-step cost of a CTA-barrier recursion (the superfast leaf / block
// Schur-Levinson pattern): thread 1 publishes a value, barrier, everyone
// reads it and runs a short dependent FP64 chain.  Prints cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAIN>
__global__ void bar_kernel(int steps, double* out, long long* cyc) {
  __shared__ double kb[2];
  double x = threadIdx.x * 1e-3, k = 0.5;
  if (threadIdx.x == 0) kb[0] = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int t = 0; t < steps; ++t) {
    k = kb[t & 1];
#pragma unroll
    for (int c = 0; c < CHAIN; ++c) x = fma(x, k, 0.25);
    if (threadIdx.x == 1) kb[(t + 1) & 1] = x * 1e-9 + 0.5;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
template <int CHAIN>
void run(int nt) {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int steps = 4096;
  bar_kernel<CHAIN><<<148, nt>>>(steps, out, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("nt=%4d chain=%2d: %.1f cycles/step\n", nt, CHAIN, (double)h / steps);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int nt : {32, 64, 256, 512, 1024}) { run<0>(nt); run<4>(nt); run<16>(nt); }
  return 0;
}
