// slse_split.cuh -- one problem on a CTA pair (thread-block cluster of 2).
//
// When a batch has at most half as many problems as SMs (cfg5: 64 problems
// of N = 16384 on 148 SMs) one CTA per problem leaves most SMs idle and the
// batch time is its slowest problem.  solve_kernel_pair runs each problem on
// a 2-CTA cluster: rank 0 executes the estimator state machine exactly as
// solve_kernel does; rank 1 is a helper that executes the other half of the
// data-parallel operations rank 0 posts as jobs:
//   * the covariance column / Psi mu steering sums (steer_forward),
//   * the component statistics (component_stats, one warp per frequency),
//   * the superfast factor's batched node transforms (dnc_split: the 4 / 2
//     transforms of an FFT node are shared between the two CTAs),
//   * the activation grid's residue batches (grid_gain_fused: even / odd r),
//   * the GS apply's two independent transform chains (gs_chain on U / V).
// Every job is the same device function on this CTA's share of the work
// (alternate output chunks, alternate frequencies, half of a node's
// transforms), so each output is computed by the same source arithmetic as
// on one CTA (the separately compiled kernel can still round differently
// where the compiler contracts products into FMAs: cfg5 estimates agree
// with the one-CTA kernel to ~1e-9 relative, far inside the parity bars, and
// the parity tests run the pair).  A job is one descriptor in global memory and two
// cluster barriers (barrier.cluster arrive.release / wait.acquire): rank 0
// writes the descriptor, both arrive (the helper was waiting), both run
// their half, both arrive again (results visible to rank 0).  The
// sequential parts (Schur leaves, control code) stay on rank 0.
#pragma once
#include <string.h>

#include "slse_port.cuh"

namespace slse {

// The pair kernel exists only in the 512-thread solver unit; every other
// instantiation compiles the split branches away.
#if defined(SLSE_NT) && SLSE_NT == 512 && !defined(SLSE_HOST_EMU)
#define SLSE_PAIR 1
#else
#define SLSE_PAIR 0
#endif

enum SplitKind : int { kJobQuit = 0, kJobSteer = 1, kJobStats = 2, kJobDncFft = 3, kJobGrid = 4, kJobGsChain = 5 };

struct SplitJob {
  int kind;
  alignas(16) unsigned char args[176];  // the job's argument struct (memcpy'd)
  template <class A>
  SLSE_D void set(int k, const A& a) {
    static_assert(sizeof(A) <= sizeof(args), "split job arguments too large");
    kind = k;
    memcpy(args, &a, sizeof(A));
  }
  template <class A>
  SLSE_D A get() const {
    A a;
    memcpy(&a, args, sizeof(A));
    return a;
  }
};

// cluster barrier: every thread of both CTAs (release / acquire at cluster scope)
SLSE_D void cluster_sync_all() {
#ifndef SLSE_HOST_EMU
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
#endif
}

struct GsChainArgs {
  void* Y;
  int n, nf;
};

struct Split {
  SplitJob* job;  // this cluster's descriptor slot (global memory)
  int rank;       // 0 = solver CTA, 1 = helper CTA
  // virtual block of the pair: this CTA's threads as half of 2 nt
  SLSE_D Blk half(const Blk& b) const {
    Blk v = b;
    v.tid = b.tid + rank * b.nt;
    v.nt = 2 * b.nt;
    return v;
  }
  // rank 0: publish a job (thread 0) and release the helper
  SLSE_D void post(const SplitJob& j, const Blk& b) {
    if (b.tid == 0) *job = j;
    cluster_sync_all();
  }
  SLSE_D void done() { cluster_sync_all(); }
};

}  // namespace slse
