// slse_solve_sf.cu -- the semifast (Woodbury) solver instantiation
// (SLSE_SEMIFAST: Solver bundles from slse_semifast.cuh) and its per-call
// bundle kernel; model_core.py:316-409, estimator.py:117-275.
#include "slse_kernels.cuh"

#ifndef SLSE_SEMIFAST
#error "compile with -DSLSE_SEMIFAST"
#endif

cudaError_t slse_solve_sf_occupancy(size_t smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(slse_k::solve_sf_kernel<kSfThreads>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, slse_k::solve_sf_kernel<kSfThreads>, kSfThreads, smem);
}

cudaError_t slse_solve_sf_launch(int grid, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                 const slse::cplx* ys, const int* idx, const slse::cplx* sc, int pstride, int B,
                                 const slse_outputs& out, char* ws, size_t slab, int* queue, const slse::cplx* tw,
                                 int twlog, int fft_cap) {
  cudaError_t e = cudaFuncSetAttribute(slse_k::solve_sf_kernel<kSfThreads>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  slse_k::solve_sf_kernel<kSfThreads><<<grid, kSfThreads, smem, st>>>(P, ys, idx, sc, pstride, B, out, ws, slab,
                                                                      queue, tw, twlog, fft_cap);
  return cudaGetLastError();
}

cudaError_t slse_sf_bundle_launch(size_t smem, cudaStream_t st, const slse::SolveParams& P, const double* theta,
                                  const double* gamma, const int* kcount, int kstride, const double* beta,
                                  const slse::cplx* ys, const int* idx, const slse::cplx* sc, int pstride, int B,
                                  char* ws, size_t slab, const slse::cplx* tw, int twlog, int fft_cap,
                                  double* data_term, slse::cplx* e, slse::cplx* q, slse::cplx* r, slse::cplx* u,
                                  double* s, slse::cplx* t, slse::cplx* v, double* x, slse::cplx* q_grid,
                                  double* s_grid, int* status) {
  cudaError_t err = cudaFuncSetAttribute(slse_k::sf_bundle_kernel<kSfThreads>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  slse_k::sf_bundle_kernel<kSfThreads><<<B, kSfThreads, smem, st>>>(
      P, theta, gamma, kcount, kstride, beta, ys, idx, sc, pstride, ws, slab, tw, twlog, fft_cap, data_term, e, q, r,
      u, s, t, v, x, q_grid, s_grid, status);
  return cudaGetLastError();
}
