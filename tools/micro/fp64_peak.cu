// FP64 DFMA throughput probe (the FP64 roofline denominator):
// every thread runs 8 independent DFMA chains; 148 x 8 CTAs x 256 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/fp64_peak.cu -o tools/micro/fp64_peak
#include <cstdio>

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int ctas = sms * 8, threads = 256, iters = 20000;
  dfma_loop<<<ctas, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<ctas, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * (double)iters * ctas * threads;
  printf("{\"fp64_dfma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n", flops / best * 1e-9, sms, best,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
