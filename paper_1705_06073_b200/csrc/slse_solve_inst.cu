// slse_solve_inst.cu -- one solver instantiation per block size; compiled
// once per SLSE_NT (128, 256, 512, 1024) so the four builds run in parallel.
#include "slse_kernels.cuh"

#ifndef SLSE_NT
#error "compile with -DSLSE_NT=<threads per block>"
#endif

#define SLSE_CAT2(a, b) a##b
#define SLSE_CAT(a, b) SLSE_CAT2(a, b)

cudaError_t SLSE_CAT(slse_solve_occupancy_, SLSE_NT)(size_t smem, int* occ) {
  cudaError_t e = cudaFuncSetAttribute(slse_k::solve_kernel<SLSE_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, slse_k::solve_kernel<SLSE_NT>, SLSE_NT, smem);
}

cudaError_t SLSE_CAT(slse_solve_launch_, SLSE_NT)(int grid, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                                  const slse::CfTable& cft, const slse::cplx* ys, int B,
                                                  const slse_outputs& out, char* ws, size_t slab, int* queue,
                                                  const slse::cplx* tw, int twlog, int fft_cap, int rec_smem) {
  cudaError_t e = cudaFuncSetAttribute(slse_k::solve_kernel<SLSE_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  slse_k::solve_kernel<SLSE_NT><<<grid, SLSE_NT, smem, st>>>(P, cft, ys, B, out, ws, slab, queue, tw, twlog, fft_cap,
                                                             rec_smem);
  return cudaGetLastError();
}

#if SLSE_NT == 512
// one problem per 2-CTA cluster (slse_split.cuh)
cudaError_t slse_solve_pair_launch_512(int clusters, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                       const slse::CfTable& cft, const slse::cplx* ys, int B,
                                       const slse_outputs& out, char* ws, size_t slab, int* queue,
                                       const slse::cplx* tw, int twlog, int fft_cap, slse::SplitJob* jobs) {
  auto kern = slse_k::solve_kernel_pair<512>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(512, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, P, cft, ys, B, out, ws, slab, queue, tw, twlog, fft_cap, jobs);
}
#endif

#ifdef SLSE_SOLVER_PROF
// Read (and optionally reset) the solver phase-cycle accumulators of this
// instantiation (see slse_solver.cuh, SLSE_SOLVER_PROF).
extern "C" int SLSE_CAT(slse_solver_prof_, SLSE_NT)(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, slse::slse_prof_cycles, sizeof(unsigned long long) * 16);
  if (e == cudaSuccess && reset) {
    const unsigned long long z[16] = {};
    e = cudaMemcpyToSymbol(slse::slse_prof_cycles, z, sizeof(z));
  }
  return (int)e;
}
#endif
