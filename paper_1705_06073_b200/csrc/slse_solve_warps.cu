// slse_solve_warps.cu -- warp-mode solver: W independent one-warp solvers
// per CTA with a CTA-wide rendezvous per heavy operation (see
// Solver::build).  Compiled with -DSLSE_WARP_MODE, which turns every group
// barrier of the shared device code into a warp barrier.
#ifndef SLSE_WARP_MODE
#error "compile with -DSLSE_WARP_MODE"
#endif
#include "slse_kernels.cuh"

cudaError_t slse_solve_warps_launch(int W, int ctas, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                    const slse::CfTable& cft, const slse::cplx* ys, int B, const slse_outputs& out,
                                    char* ws, size_t slab, int* queue, const slse::cplx* tw, int twlog, int fft_cap,
                                    int rec_smem, int warp_smem) {
  cudaError_t e;
  switch (W) {
    case 16:
      e = cudaFuncSetAttribute(slse_k::solve_kernel_warps<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      slse_k::solve_kernel_warps<16><<<ctas, 32 * 16, smem, st>>>(P, cft, ys, B, out, ws, slab, queue, tw, twlog,
                                                                    fft_cap, rec_smem, warp_smem);
      break;
    case 8:
      e = cudaFuncSetAttribute(slse_k::solve_kernel_warps<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      slse_k::solve_kernel_warps<8><<<ctas, 32 * 8, smem, st>>>(P, cft, ys, B, out, ws, slab, queue, tw, twlog,
                                                                  fft_cap, rec_smem, warp_smem);
      break;
    case 4:
      e = cudaFuncSetAttribute(slse_k::solve_kernel_warps<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      slse_k::solve_kernel_warps<4><<<ctas, 32 * 4, smem, st>>>(P, cft, ys, B, out, ws, slab, queue, tw, twlog,
                                                                  fft_cap, rec_smem, warp_smem);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

#ifdef SLSE_SOLVER_PROF
extern "C" int slse_solver_prof_warps(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, slse::slse_prof_cycles, sizeof(unsigned long long) * 16);
  if (e == cudaSuccess && reset) {
    const unsigned long long z[16] = {};
    e = cudaMemcpyToSymbol(slse::slse_prof_cycles, z, sizeof(z));
  }
  return (int)e;
}
#endif
