// slse_kernels.cuh -- kernel templates and launch configuration shared by
// the C-ABI translation unit (slse_capi.cu) and the per-block-size solver
// instantiations (slse_solve_inst.cu, compiled once per NT in parallel).
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>

#include "superlse_b200.h"
#include "slse_solver.cuh"

using namespace slse;

// min resident CTAs per SM for the one-warp solver (caps registers)
#ifndef SLSE_SOLVER_MINB_WIDE
#define SLSE_SOLVER_MINB_WIDE (NT == 256 ? 2 : 1)  // NT = 256 runs two CTAs per SM (solver_paired)
#endif
#ifndef SLSE_SOLVER_MINB32
#define SLSE_SOLVER_MINB32 16
#endif


namespace slse_k {

// ---------------------------------------------------------- configuration
// shared-memory head: Blk reduction scratch (2 banks x nwarps x 16 doubles)
// followed by the cf table; the FFT / recursion region starts at head_bytes
SLSE_HD constexpr size_t red_bytes(int nt) { return (2 * ((nt + 31) / 32) * 16 * sizeof(double) + 255) & ~(size_t)255; }
SLSE_HD constexpr size_t head_bytes(int nt) { return red_bytes(nt) + ((sizeof(CfTable) + 255) & ~(size_t)255); }
constexpr size_t kRedBytes = red_bytes(1024);
constexpr size_t kCfBytes = (sizeof(CfTable) + 255) & ~(size_t)255;
constexpr size_t kHeadBytes = head_bytes(1024);
constexpr size_t kRegionBudget = 200 * 1024;

// Experiment overrides used by tools/ (environment variables) exist only in
// builds compiled with -DSLSE_DEBUG_KNOBS; the product library reads no
// environment.
inline const char* slse_knob(const char* name) {
#ifdef SLSE_DEBUG_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

inline int block_threads(int n) {
  if (n <= 128) return 128;
  if (n <= 512) return 256;
  if (n <= 2048) return 512;
  return 1024;
}

struct SmemPlan {
  int rec_in_smem;
  int fft_cap;
  size_t bytes;
};

inline SmemPlan smem_plan(int n, int L, int nt, bool dnc = false, size_t region_budget = 0) {
  SmemPlan p;
  // one-warp solvers: keep the region small so more problems stay resident
  // (only the recursion and the 2N-point transforms are staged; the grid's
  // L-point transforms then run from L1/L2); paired 256-thread solvers get
  // half an SM (region_budget)
  size_t budget = region_budget ? region_budget : kRegionBudget;
  if (nt <= 32 && !dnc) {
    const char* env = slse_knob("SLSE_WARP_REGION_KB");
    budget = env ? (size_t)atoi(env) * 1024 : 48 * (size_t)n;
    if (budget < 48 * (size_t)n) budget = 48 * (size_t)n;
  }
  if (const char* env = slse_knob("SLSE_REGION_KB")) {  // experiment override
    const size_t v = (size_t)atoi(env) * 1024;
    if (dnc || v >= 48 * (size_t)n) budget = v;
  }
  const size_t rec = dnc ? 0 : 48 * (size_t)n;
  p.rec_in_smem = (!dnc && rec <= budget) ? 1 : 0;
  const int fftmax = L > 2 * n ? L : (1 << ilog2(2 * n));
  size_t cap_bytes = p.rec_in_smem ? rec : 0;
  // staging capacity in complex elements: the largest power-of-two transform
  // that fits, in the skewed layout (sk_len)
  int F = 1;
  if (16 * (size_t)sk_len(fftmax) <= budget) {
    F = fftmax;
  } else {
    const size_t lim = cap_bytes > 0 ? cap_bytes : budget;
    while (16 * (size_t)sk_len(F * 2) <= lim) F *= 2;
  }
  p.fft_cap = sk_len(F);
  size_t region = 16 * (size_t)p.fft_cap;
  if (p.rec_in_smem && rec > region) region = rec;
  p.fft_cap = (int)(region / 16);  // staging capacity = the whole region (recursion and FFTs alternate)
  p.bytes = head_bytes(nt) + region;
  return p;
}



// ------------------------------------------------------------------ kernels
struct OutPtrs {
  slse_outputs o;
};

// output views of problem p
SLSE_D ProbOut prob_out(const slse_outputs& out, const SolveParams& P, int p) {
  const size_t K = (size_t)P.kmax;
  ProbOut o;
  o.khat = out.k_hat + p;
  o.status = out.status + p;
  o.iters = out.iterations + p;
  o.flags = out.flags + p;
  o.beta = out.beta + p;
  o.zeta = out.zeta + p;
  o.theta = out.theta + p * K;
  o.gamma = out.gamma + p * K;
  o.alpha = (cplx*)out.alpha + (size_t)p * K * P.g;  // [B, G, kmax]
  o.slot = out.slot + p * K;
  o.trace = out.trace + (size_t)p * P.tcap;
  o.stage = out.stage + (size_t)p * P.tcap;
  o.trace_k = out.trace_k + (size_t)p * P.tcap;
  o.ntrace = out.n_trace + p;
  o.events = out.events + (size_t)p * P.ecap * 3;
  o.nevents = out.n_events + p;
  o.counters = (long long*)out.counters + (size_t)p * 4;
  o.stage_s = out.stage_seconds + (size_t)p * 6;
  o.iter_s = out.iter_seconds ? out.iter_seconds + (size_t)p * P.max_outer : nullptr;
  return o;
}

template <int NT>
__global__ void __launch_bounds__(NT, (NT <= 32 ? SLSE_SOLVER_MINB32 : SLSE_SOLVER_MINB_WIDE)) solve_kernel(SolveParams P, CfTable cft, const cplx* __restrict__ ys,
                                                   int B, slse_outputs out, char* ws, size_t slab_bytes,
                                                   int* queue, const cplx* tw, int twlog, int fft_cap,
                                                   int rec_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* red = (double*)smem_raw;
  CfTable* cf = (CfTable*)(smem_raw + red_bytes(NT));
  cplx* region = (cplx*)(smem_raw + head_bytes(NT));
  __shared__ int s_prob;
  if (threadIdx.x == 0) *cf = cft;
  Blk b;
  b.tid = threadIdx.x;
  b.nt = NT;
  b.red = red;
  b.bank = 0;
  FftCtx f;
  f.tw = tw;
  f.twlog = twlog;
  f.smem = region;
  f.smem_cap = fft_cap;
  char* slab = ws + (size_t)blockIdx.x * slab_bytes;
  const Layout lay = make_layout(P.n, P.L, P.kmax, P.lbfgs_mem, rec_smem != 0, P.dnc != 0, P.g);
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_prob = atomicAdd(queue, 1);
    __syncthreads();
    const int p = s_prob;
    __syncthreads();
    if (p >= B) break;
    const ProbOut o = prob_out(out, P, p);
    Solver S(b, P, cf, ys + (size_t)p * P.n * P.g, o, slab, lay, rec_smem ? region : nullptr, f);
    S.run();
    b.bank = S.b.bank;
    __syncthreads();
  }
}

// One problem per 2-CTA cluster (slse_split.cuh): rank 0 runs the solver
// (problems from the atomic queue), rank 1 executes the jobs rank 0 posts
// until it posts kJobQuit.  Launched with cluster dimension 2.
template <int NT>
__global__ void __launch_bounds__(NT, 1) solve_kernel_pair(SolveParams P, CfTable cft, const cplx* __restrict__ ys,
                                                            int B, slse_outputs out, char* ws, size_t slab_bytes,
                                                            int* queue, const cplx* tw, int twlog, int fft_cap,
                                                            SplitJob* jobs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* red = (double*)smem_raw;
  CfTable* cf = (CfTable*)(smem_raw + red_bytes(NT));
  cplx* region = (cplx*)(smem_raw + head_bytes(NT));
  __shared__ int s_prob;
  if (threadIdx.x == 0) *cf = cft;
  Blk b;
  b.tid = threadIdx.x;
  b.nt = NT;
  b.red = red;
  b.bank = 0;
  FftCtx f;
  f.tw = tw;
  f.twlog = twlog;
  f.smem = region;
  f.smem_cap = fft_cap;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cid = blockIdx.x >> 1;
  Split sp;
  sp.job = jobs + cid;
  sp.rank = (int)rank;
  __syncthreads();
  if (rank != 0) {  // helper
    for (;;) {
      cluster_sync_all();  // rank 0 posted a job
      const SplitJob j = *sp.job;  // visible: the barrier acquired it
      if (j.kind == kJobQuit) break;
      run_split_job(j, 1, cf, f, b);
      cluster_sync_all();  // both halves done
    }
    return;
  }
  char* slab = ws + (size_t)cid * slab_bytes;
  const Layout lay = make_layout(P.n, P.L, P.kmax, P.lbfgs_mem, false, P.dnc != 0, P.g);
  for (;;) {
    if (threadIdx.x == 0) s_prob = atomicAdd(queue, 1);
    __syncthreads();
    const int p = s_prob;
    __syncthreads();
    if (p >= B) break;
    const ProbOut o = prob_out(out, P, p);
    Solver S(b, P, cf, ys + (size_t)p * P.n * P.g, o, slab, lay, nullptr, f);
    S.sp = &sp;
    S.run();
    b.bank = S.b.bank;
    __syncthreads();
  }
  SplitJob q;
  q.kind = kJobQuit;
  sp.post(q, b);
}

#ifdef SLSE_WARP_MODE
// W independent one-warp solvers per CTA (one CTA per SM), meeting at a
// CTA-wide rendezvous for every heavy operation (Solver::build / stats /
// grid_curve in warp mode).  Shared memory: the cf table, then per warp its
// reduction scratch and its FFT / recursion region (warp_smem bytes).
template <int W>
__global__ void __launch_bounds__(32 * W, 16 / W) solve_kernel_warps(SolveParams P, CfTable cft, const cplx* __restrict__ ys,
                                                                    int B, slse_outputs out, char* ws, size_t slab_bytes,
                                                                    int* queue, const cplx* tw, int twlog, int fft_cap,
                                                                    int rec_smem, int warp_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CfTable* cf = (CfTable*)smem_raw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* mine = smem_raw + kCfBytes + (size_t)warp * warp_smem;
  if (threadIdx.x == 0) *cf = cft;
  __syncthreads();
  Blk b;
  b.tid = lane;
  b.nt = 32;
  b.red = (double*)mine;
  b.bank = 0;
  FftCtx f;
  f.tw = tw;
  f.twlog = twlog;
  f.smem = (cplx*)(mine + red_bytes(32));
  f.smem_cap = fft_cap;
  cplx* region = f.smem;
  char* slab = ws + ((size_t)blockIdx.x * W + warp) * slab_bytes;
  const Layout lay = make_layout(P.n, P.L, P.kmax, P.lbfgs_mem, rec_smem != 0, P.dnc != 0, P.g);
  for (;;) {
    int p = 0;
    if (lane == 0) p = atomicAdd(queue, 1);
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p >= B) break;
    const ProbOut o = prob_out(out, P, p);
    Solver S(b, P, cf, ys + (size_t)p * P.n * P.g, o, slab, lay, rec_smem ? region : nullptr, f);
    S.run();
    b.bank = S.b.bank;
    __syncwarp();
  }
  // no problem left: answer the other warps' rendezvous until all are idle
  while (!rv_arrive(1)) rv_depart();
}
#endif

template <int NT>
__global__ void __launch_bounds__(NT) cov_kernel(const double* theta, const double* gamma, const int* kcount,
                                                 int kstride, const double* beta, int n, cplx* c) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  steer_forward(c + (size_t)p * n, n, theta + (size_t)p * kstride, gamma + (size_t)p * kstride, nullptr,
                kcount[p], beta[p], true, b);
}

template <int NT>
__global__ void __launch_bounds__(NT) factor_kernel(const cplx* c, int n, cplx* rho, double* delta,
                                                    double* logdet, int* status, cplx* scratch, double* dscratch,
                                                    int rec_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  cplx* e;
  if (rec_smem) {
    e = (cplx*)(smem_raw + kHeadBytes);
  } else {
    e = scratch + (size_t)p * 3 * n;
  }
  Factor F = toeplitz_factor(c + (size_t)p * n, n, e, e + n, e + 2 * n, delta ? delta + (size_t)p * n : nullptr,
                             dscratch + (size_t)p * n, rho + (size_t)p * n, b);
  if (threadIdx.x == 0) {
    logdet[p] = F.logdet;
    status[p] = F.status;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) apply_kernel(const cplx* rho, const double* delta_last, const cplx* y, int n,
                                                   cplx* w, double* quad, cplx* scratch, const cplx* tw, int twlog,
                                                   int fft_cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  FftCtx f{tw, twlog, (cplx*)(smem_raw + kHeadBytes), fft_cap};
  const int p = blockIdx.x;
  const int nf = 1 << ilog2(2 * n);
  cplx* yh = scratch + (size_t)p * 4 * nf;
  const cplx* yp = y + (size_t)p * n;
  fft(yh, nf, -1.0, [=](int i) { return i < n ? yp[i] : mk(0.0, 0.0); }, [=](int i, cplx v) { yh[i] = v; }, f, b);
  double qd = gs_apply(rho + (size_t)p * n, n, delta_last[p], yp, yh, yh + nf, yh + 2 * nf, yh + 3 * nf,
                       w + (size_t)p * n, f, b);
  if (quad && threadIdx.x == 0) quad[p] = qd;
}

// Row 7: the four diagonal-sum vectors omega_kind(i), i = -(N-1)..N-1
// (toeplitz.py:415-432) from the same cf table as the product-form stats:
//   omega_kind(i) = scale / delta  sum_ab cf[kind][a][b] R_ab(i),
//   R_ab(i) = sum_q q^a rho_q (q+i)^b conj(rho_{q+i})
//           = IFFT( P_a . Y_b )(i) / nf,  P_a = sum_q q^a rho_q e^{+j..},
//             Y_b = FFT(q^b conj(rho)),  nf >= 2N - 1  (no wrap),
// so 4 + 4 + 4 transforms of nf per problem; s and x are symmetrised as
// the reference does (:428-430).  Scratch: 9 nf complex per problem.
template <int NT>
__global__ void __launch_bounds__(NT) omegas_kernel(CfTable cft, const cplx* rho, const double* delta_last, int n,
                                                    cplx* om_s, cplx* om_t, cplx* om_v, cplx* om_x, cplx* scratch,
                                                    const cplx* tw, int twlog, int fft_cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  FftCtx f{tw, twlog, (cplx*)(smem_raw + kHeadBytes), fft_cap};
  const int p = blockIdx.x;
  const int lg = ilog2(2 * n - 1);
  const int nf = 1 << lg;
  cplx* P = scratch + (size_t)p * 9 * nf;
  cplx* Y = P + 4 * (size_t)nf;
  cplx* W = Y + 4 * (size_t)nf;
  const cplx* rp = rho + (size_t)p * n;
  const cplx z = mk(0.0, 0.0);
  for (int a = 0; a < 4; ++a) {
    cplx* Pa = P + (size_t)a * nf;
    fft(W, nf, 1.0, [=](int i) { return i < n ? cscale(rp[i], a == 0 ? 1.0 : pow((double)i, (double)a)) : z; },
        [=](int i, cplx v) { Pa[i] = v; }, f, b);
    cplx* Yb = Y + (size_t)a * nf;
    fft(W, nf, -1.0, [=](int i) { return i < n ? cscale(conjg(rp[i]), a == 0 ? 1.0 : pow((double)i, (double)a)) : z; },
        [=](int i, cplx v) { Yb[i] = v; }, f, b);
  }
  const double dl = delta_last[p];
  const double scales[4] = {1.0, 2.0 * kPi, 4.0 * kPi * kPi, 4.0 * kPi * kPi};
  cplx* outs[4] = {om_s, om_t, om_v, om_x};
  const int len = 2 * n - 1;
  for (int kind = 0; kind < 4; ++kind) {
    cplx* om = outs[kind] + (size_t)p * len;
    const double sc = scales[kind] / (dl * (double)nf);
    const CfTable T = cft;
    const cplx* Pc = P;
    const cplx* Yc = Y;
    fft(W, nf, 1.0,
        [=](int fi) {
          cplx acc = z;
          for (int a = 0; a < 4; ++a)
            for (int bb = 0; bb < 4; ++bb) {
              const double c = T.cf[kind][a][bb];
              if (c != 0.0) acc = cadd(acc, cscale(cmul(Pc[(size_t)a * nf + fi], Yc[(size_t)bb * nf + fi]), c));
            }
          return acc;
        },
        [=](int i, cplx v) {
          int d = -1;
          if (i <= n - 1) d = i + n - 1;             // lag i >= 0
          else if (i >= nf - (n - 1)) d = i - nf + n - 1;  // lag i - nf < 0
          if (d >= 0) om[d] = cscale(v, sc);
        },
        f, b);
    if (kind == 0 || kind == 3) {  // Hermitian symmetrisation (s, x)
      b.sync();
      for (int d = threadIdx.x; d < n - 1; d += NT) om[d] = conjg(om[len - 1 - d]);
      if (threadIdx.x == 0) om[n - 1].im = 0.0;
      b.sync();
    }
  }
}

// Row 10: Delta-L curve over the grid and its argmin (lowest index on ties),
// one CTA per problem.  gbar, zeta per problem; zeta is clamped as the
// prior does (prior_zeta).
template <int NT>
__global__ void __launch_bounds__(NT) act_curve_kernel(const cplx* q_grid, const double* s_grid, const double* gbar,
                                                       const double* zeta, int kmax, int L, double* curve,
                                                       int* argmin_idx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  const double gb = gbar[p];
  const double ze = prior_zeta(zeta[p], kmax);
  const double lr = log((1.0 - ze) / ze);
  double bv = 0.0;
  int bi = -1;
  for (int l = threadIdx.x; l < L; l += NT) {
    const double dv = gain(cabs2(q_grid[(size_t)p * L + l]), s_grid[(size_t)p * L + l], gb, lr);
    if (curve) curve[(size_t)p * L + l] = dv;
    if (Blk::better(dv, l, bv, bi)) { bv = dv; bi = l; }
  }
  b.argmin(bv, bi);
  if (threadIdx.x == 0) argmin_idx[p] = bi;
}

// Row 11: deactivation margins of the kcount[p] components (smlr.py:174-200)
// and their argmin (lowest index on ties).
template <int NT>
__global__ void __launch_bounds__(NT) deact_kernel(const cplx* q, const double* s, const double* gamma,
                                                   const int* kcount, int kstride, const double* zeta, int kmax,
                                                   double* margin, int* argmin_idx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  const int k = kcount[p];
  const double ze = prior_zeta(zeta[p], kmax);
  const double rhs = log((1.0 - ze) / ze);
  double bv = 0.0;
  int bi = -1;
  for (int i = threadIdx.x; i < k; i += NT) {
    const size_t o = (size_t)p * kstride + i;
    const double mg = deact_margin(gamma[o], s[o], cabs2(q[o]), rhs);
    if (margin) margin[o] = mg;
    if (Blk::better(mg, i, bv, bi)) { bv = mg; bi = i; }
  }
  b.argmin(bv, bi);
  if (threadIdx.x == 0) argmin_idx[p] = bi;
}

// Row 12: gradient and diagonal Hessian (model_core.py:497-536), one thread
// per component; g and d are [B, 2 kstride] (theta block, then gamma block).
static __global__ void grad_kernel(const cplx* q, const cplx* r, const cplx* u, const double* s, const cplx* t, const cplx* v,
                            const double* x, const double* gamma, const int* kcount, int kstride, int B, int n,
                            double* g, double* d) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * kstride) return;
  const int p = (int)(idx / kstride), i = (int)(idx - (long long)p * kstride);
  if (i >= kcount[p]) return;
  const int k = kcount[p];
  double gth, gga, dth, dga;
  grad_diag_comp(gamma[idx], q + idx, r + idx, u + idx, 0, 1, s[idx], t[idx], v[idx], x[idx], n, &gth, &gga, &dth,
                 &dga);
  double* gp = g + (size_t)p * 2 * kstride;
  double* dp = d + (size_t)p * 2 * kstride;
  gp[i] = gth;
  gp[k + i] = gga;
  dp[i] = dth;
  dp[k + i] = dga;
}

template <int NT>
__global__ void __launch_bounds__(NT) stats_kernel(CfTable cft, const double* theta, const int* kcount, int kstride,
                                                   const cplx* rho, const double* delta_last, const cplx* w, int n,
                                                   cplx* q, cplx* r, cplx* u, double* s, cplx* t, cplx* v,
                                                   double* x) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CfTable* cf = (CfTable*)(smem_raw + kRedBytes);
  if (threadIdx.x == 0) *cf = cft;
  __syncthreads();
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  const size_t o = (size_t)p * kstride;
  component_stats(theta + o, kcount[p], rho + (size_t)p * n, w + (size_t)p * n, n, delta_last[p], cf, q + o, r + o,
                  u + o, s + o, t + o, v + o, x + o, b);
}

// Row 9 standalone (the roofline kernel): all three length-L transforms in
// shared memory when 48 L bytes fit, one pass over HBM in and out.
template <int NT>
__global__ void __launch_bounds__(NT) grid_kernel(const cplx* __restrict__ rho, const double* __restrict__ delta_last,
                                                  const cplx* __restrict__ w, int n, int L, cplx* __restrict__ q_grid,
                                                  double* __restrict__ s_grid, cplx* scratch, const cplx* tw,
                                                  int twlog, int fused) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  const int p = blockIdx.x;
  const cplx* rp = rho + (size_t)p * n;
  const cplx* wp = w + (size_t)p * n;
  cplx* qg = q_grid + (size_t)p * L;
  double* sgp = s_grid + (size_t)p * L;
  const double inv_d = 1.0 / delta_last[p];
  const double c2n = 2.0 - (double)n;
  if (fused) {
    cplx* X0 = (cplx*)(smem_raw + kHeadBytes);
    cplx* X1 = X0 + L;
    cplx* X2 = X1 + L;
    FftCtx f{tw, twlog, X0, 0};
    const int lg = ilog2(L);
    for (int i = threadIdx.x; i < L; i += NT) {
      const unsigned j = brev_bits((unsigned)i, lg);
      cplx a = mk(0.0, 0.0), rr = mk(0.0, 0.0);
      if (i < n) { a = wp[i]; rr = rp[i]; }
      X0[j] = a;
      X1[j] = rr;
      X2[j] = cscale(rr, (double)i);
    }
    __syncthreads();
    fft_passes(X0, L, -1.0, f, b);
    fft_passes(X1, L, -1.0, f, b);
    fft_passes(X2, L, -1.0, f, b);
    for (int l = threadIdx.x; l < L; l += NT) {
      const cplx a0 = X1[l], a1 = X2[l];
      qg[l] = X0[l];
      sgp[l] = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
    }
  } else {
    FftCtx f{tw, twlog, (cplx*)(smem_raw + kHeadBytes), 0};
    cplx* G1 = scratch + (size_t)p * 2 * L;
    grid_eval(rp, wp, n, delta_last[p], L, qg, G1, G1 + L, sgp, f, b);
  }
}



template <int NT>
__global__ void __launch_bounds__(NT) factor_dnc_kernel(const cplx* c, int n, cplx* rho, double* delta, double* logdet,
                                                        int* status, cplx* scratch, size_t per_problem,
                                                        double* dscratch, const cplx* tw, int twlog, int fft_cap,
                                                        int direct_max, long long* prof) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b{(int)threadIdx.x, NT, (double*)smem_raw, 0};
  FftCtx f{tw, twlog, (cplx*)(smem_raw + kHeadBytes), fft_cap};
  const int p = blockIdx.x;
  cplx* T = scratch + (size_t)p * per_problem;
  Factor F = toeplitz_factor_dnc(c + (size_t)p * n, n, T, T + 4 * (size_t)n, delta ? delta + (size_t)p * n : nullptr,
                                 dscratch + (size_t)p * n, rho + (size_t)p * n, f, b, 0, direct_max,
                                 (prof && p == 0) ? prof : nullptr);
  if (threadIdx.x == 0) {
    logdet[p] = F.logdet;
    status[p] = F.status;
  }
}

// Row 9 standalone, register-Stockham variant: the three length-L transforms
// (w, rho, n*rho) live in shared memory; only their nonzero heads (the
// first L/2^Q points, n <= L/2^Q) are loaded, the first radix-16 pass is
// pruned accordingly, and the combine writes q^G and s^G once.
template <int NT, int LG, int Q>
__global__ void __launch_bounds__(NT, (NT <= 192 ? 3 : (NT <= 256 ? 2 : 1))) grid_stockham_kernel(
    const cplx* __restrict__ rho, const double* __restrict__ delta_last, const cplx* __restrict__ w, int n,
    cplx* __restrict__ q_grid, double* __restrict__ s_grid, const cplx* tw, int twlog) {
  constexpr int L = 1 << LG;
  constexpr int LS = L + (L >> 4);
  constexpr int H = L >> Q;  // loaded head (>= n)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int p = blockIdx.x;
  const cplx* rp = rho + (size_t)p * n;
  const cplx* wp = w + (size_t)p * n;
  cplx* X = (cplx*)(smem_raw + head_bytes(NT));
  for (int i = threadIdx.x; i < H; i += NT) {
    cplx a = mk(0.0, 0.0), rr = mk(0.0, 0.0);
    if (i < n) { a = wp[i]; rr = rp[i]; }
    const int si = sk(i);
    X[si] = a;
    X[LS + si] = rr;
    X[2 * LS + si] = cscale(rr, (double)i);
  }
  __syncthreads();
  fft_fixed_pruned<LG, Q>(X, 3, -1.0, tw, twlog, threadIdx.x, NT);
  const double inv_d = 1.0 / delta_last[p];
  const double c2n = 2.0 - (double)n;
  cplx* qg = q_grid + (size_t)p * L;
  double* sgp = s_grid + (size_t)p * L;
  for (int l = threadIdx.x; l < L; l += NT) {
    const int sl = sk(l);
    const cplx a0 = X[LS + sl], a1 = X[2 * LS + sl];
    qg[l] = X[sl];
    sgp[l] = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
  }
}



#ifndef SLSE_GRID_MINB
#define SLSE_GRID_MINB 3
#endif
// Row 9 standalone, v3: pass 1 (pruned radix-16) reads w / rho straight from
// HBM (no staging copy), the middle passes run in skewed shared memory, and
// the last radix-RL pass is fused with the product-form combine: thread j
// transforms item j of all three buffers and writes q^G and s^G at
// l = j + r L/RL directly (coalesced), so the final spectra never touch
// shared memory.  Requires RL = 2^(LG - 4 - 4k) in {2, 4, 8}.
template <int NT, int LG, int Q>
__global__ void __launch_bounds__(NT, (NT <= 256 ? SLSE_GRID_MINB : 1)) grid_fused_kernel(
    const cplx* __restrict__ rho, const double* __restrict__ delta_last, const cplx* __restrict__ w, int n,
    cplx* __restrict__ q_grid, double* __restrict__ s_grid, const cplx* tw, int twlog) {
  constexpr int L = 1 << LG;
  constexpr int LS = L + (L >> 4);
  constexpr int LGRL = (LG - 4) % 4;  // last radix (1 <= LGRL <= 3)
  constexpr int RL = 1 << LGRL;
  constexpr int PER = L / RL;         // last-pass items per buffer (== NT)
  constexpr int NZ = 16 >> Q;
  constexpr int P1 = L / 16;          // first-pass items per buffer
  static_assert(LGRL >= 1 && PER == NT, "grid_fused_kernel: plan needs NT = L / RL");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int p = blockIdx.x;
  const int tid = threadIdx.x;
  const cplx* rp = rho + (size_t)p * n;
  const cplx* wp = w + (size_t)p * n;
  cplx* X = (cplx*)(smem_raw + head_bytes(NT));
  // ---- pass 1: pruned radix-16 straight from global
  for (int it = tid; it < 3 * P1; it += NT) {
    const int c = it / P1, j = it - c * P1;
    cplx v[16];
#pragma unroll
    for (int r = 0; r < NZ; ++r) {
      const int i = j + r * P1;
      cplx x = mk(0.0, 0.0);
      if (i < n) {
        if (c == 0) x = wp[i];
        else if (c == 1) x = rp[i];
        else x = cscale(rp[i], (double)i);
      }
      v[r] = x;
    }
    DifPrunedStage<16, NZ, 8>::run(v, -1.0);
    cplx* xc = X + (size_t)c * LS;
#pragma unroll
    for (int r = 0; r < 16; ++r) xc[sk(j * 16 + r)] = v[brev_const(r, 16)];
  }
  __syncthreads();
  // ---- middle radix-16 passes
  FixedPlanMid<LG, 4, LG - LGRL, (3 * (L / 16) + NT - 1) / NT>::run(X, 3, -1.0, tw, twlog, tid, NT);
  // ---- last pass fused with the combine (q^G first, then the (A0, A1)
  // pair, keeping at most 2 RL complex values live)
  const int j = tid;
  constexpr int NS = L / RL;
  cplx* qg = q_grid + (size_t)p * L;
  double* sgp = s_grid + (size_t)p * L;
  {
    cplx v0[RL];
#pragma unroll
    for (int r = 0; r < RL; ++r) v0[r] = X[sk(j + r * PER)];
#pragma unroll
    for (int r = 1; r < RL; ++r) v0[r] = cmul(v0[r], twid_tab(tw, twlog, j * r, LG, -1.0));
    dft_dif<RL>(v0, -1.0);
#pragma unroll
    for (int r = 0; r < RL; ++r) qg[j + r * NS] = v0[brev_const(r, RL)];
  }
  const double inv_d = 1.0 / delta_last[p];
  const double c2n = 2.0 - (double)n;
  cplx v1[RL], v2[RL];
#pragma unroll
  for (int r = 0; r < RL; ++r) {
    v1[r] = X[LS + sk(j + r * PER)];
    v2[r] = X[2 * LS + sk(j + r * PER)];
  }
#pragma unroll
  for (int r = 1; r < RL; ++r) {
    const cplx t = twid_tab(tw, twlog, j * r, LG, -1.0);
    v1[r] = cmul(v1[r], t);
    v2[r] = cmul(v2[r], t);
  }
  dft_dif<RL>(v1, -1.0);
  dft_dif<RL>(v2, -1.0);
#pragma unroll
  for (int r = 0; r < RL; ++r) {
    const cplx a0 = v1[brev_const(r, RL)], a1 = v2[brev_const(r, RL)];
    sgp[j + r * NS] = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
  }
}

#ifdef SLSE_SEMIFAST
// Semifast solver (slse_solve_sf.cu): the same persistent estimate() loop
// with semifast bundles on an observation pattern (model_core.py:316-409);
// y rows hold G x M observed samples, the pattern (idx, scales) is shared
// by the batch (pstride 0) or given per problem (pstride M).
#ifndef SLSE_SF_MINB
#define SLSE_SF_MINB 6  // 80 registers: cfg2-shape semifast 149 -> 94 ms per 4096 problems (2 -> 6 CTAs per SM)
#endif
template <int NT>
__global__ void __launch_bounds__(NT, SLSE_SF_MINB) solve_sf_kernel(SolveParams P, const cplx* __restrict__ ys,
                                                      const int* __restrict__ pidx, const cplx* __restrict__ psc,
                                                      int pstride, int B, slse_outputs out, char* ws,
                                                      size_t slab_bytes, int* queue, const cplx* tw, int twlog,
                                                      int fft_cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* red = (double*)smem_raw;
  cplx* region = (cplx*)(smem_raw + red_bytes(NT));
  __shared__ int s_prob;
  Blk b;
  b.tid = threadIdx.x;
  b.nt = NT;
  b.red = red;
  b.bank = 0;
  FftCtx f;
  f.tw = tw;
  f.twlog = twlog;
  f.smem = region;
  f.smem_cap = fft_cap;
  char* slab = ws + (size_t)blockIdx.x * slab_bytes;
  const Layout lay = make_layout(P.n, P.L, P.kmax, P.lbfgs_mem, false, false, P.g, 1, P.m, P.kcap);
  for (;;) {
    if (threadIdx.x == 0) s_prob = atomicAdd(queue, 1);
    __syncthreads();
    const int p = s_prob;
    __syncthreads();
    if (p >= B) break;
    const ProbOut o = prob_out(out, P, p);
    Solver S(b, P, nullptr, ys + (size_t)p * P.m * P.g, o, slab, lay, nullptr, f);
    S.obs.idx = pidx + (size_t)p * pstride;
    S.obs.sc = psc ? psc + (size_t)p * pstride : nullptr;
    S.run();
    b.bank = S.b.bank;
    __syncthreads();
  }
}

// Per-call semifast bundle (the parity tests' view of one bundle): one CTA
// per problem builds the bundle of (theta, gamma, beta) and writes its data
// term, e = Phi^H C^{-1} y, the component statistics and the grid.
template <int NT>
__global__ void __launch_bounds__(NT) sf_bundle_kernel(SolveParams P, const double* theta, const double* gamma,
                                                       const int* kcount, int kstride, const double* beta,
                                                       const cplx* __restrict__ ys, const int* __restrict__ pidx,
                                                       const cplx* __restrict__ psc, int pstride, char* ws,
                                                       size_t slab_bytes, const cplx* tw, int twlog, int fft_cap,
                                                       double* data_term, cplx* e, cplx* q, cplx* r, cplx* u,
                                                       double* s, cplx* t, cplx* v, double* x, cplx* q_grid,
                                                       double* s_grid, int* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Blk b;
  b.tid = threadIdx.x;
  b.nt = NT;
  b.red = (double*)smem_raw;
  b.bank = 0;
  FftCtx f;
  f.tw = tw;
  f.twlog = twlog;
  f.smem = (cplx*)(smem_raw + red_bytes(NT));
  f.smem_cap = fft_cap;
  const int p = blockIdx.x;
  char* slab = ws + (size_t)p * slab_bytes;
  const Layout lay = make_layout(P.n, P.L, P.kmax, P.lbfgs_mem, false, false, P.g, 1, P.m, P.kcap);
  ProbOut o = {};
  Solver S(b, P, nullptr, ys + (size_t)p * P.m * P.g, o, slab, lay, nullptr, f);
  S.obs.idx = pidx + (size_t)p * pstride;
  S.obs.sc = psc ? psc + (size_t)p * pstride : nullptr;
  const int kk = kcount[p];
  for (int i = threadIdx.x; i < kk; i += NT) {
    S.act_theta[i] = theta[(size_t)p * kstride + i];
    S.act_gamma[i] = gamma[(size_t)p * kstride + i];
  }
  __syncthreads();
  S.k = kk;
  Bundle& B = S.bun[0];
  const int st = S.sf_build(B, S.act_theta, S.act_gamma, kk, beta[p]);
  if (threadIdx.x == 0) status[p] = st;
  if (st != kOk) return;
  if (threadIdx.x == 0) data_term[p] = B.data_term;
  for (int i = threadIdx.x; i < P.n * P.g; i += NT) e[(size_t)p * P.n * P.g + i] = B.w[i];
  if (kk) {
    S.sf_stats(B, S.act_theta, kk);
    for (int i = threadIdx.x; i < kk; i += NT) {
      for (int g = 0; g < P.g; ++g) {
        const size_t o_ = ((size_t)p * P.g + g) * kstride + i;
        q[o_] = B.q[(size_t)g * P.kmax + i];
        r[o_] = B.r[(size_t)g * P.kmax + i];
        u[o_] = B.u[(size_t)g * P.kmax + i];
      }
      s[(size_t)p * kstride + i] = B.s[i];
      t[(size_t)p * kstride + i] = B.t[i];
      v[(size_t)p * kstride + i] = B.v[i];
      x[(size_t)p * kstride + i] = B.x[i];
    }
  }
  S.cur = 0;
  S.sf_grid(B, 1.0, 0.0, q_grid + (size_t)p * P.g * P.L);
  for (int l = threadIdx.x; l < P.L; l += NT) s_grid[(size_t)p * P.L + l] = S.sg[l];
}
#endif

SLSE_D cplx ldg_c(const cplx* p) {
  const double2 d = __ldg((const double2*)p);
  return mk(d.x, d.y);
}

}  // namespace slse_k

// per-NT solver entry points (slse_solve_inst.cu)
#define SLSE_DECL_SOLVE(NT)                                                                            \
  cudaError_t slse_solve_occupancy_##NT(size_t smem, int* occ);                                       \
  cudaError_t slse_solve_launch_##NT(int grid, size_t smem, cudaStream_t st, const slse::SolveParams& P, \
                                     const slse::CfTable& cft, const slse::cplx* ys, int B,            \
                                     const slse_outputs& out, char* ws, size_t slab, int* queue,       \
                                     const slse::cplx* tw, int twlog, int fft_cap, int rec_smem);
SLSE_DECL_SOLVE(32)
SLSE_DECL_SOLVE(64)
SLSE_DECL_SOLVE(128)
SLSE_DECL_SOLVE(256)
SLSE_DECL_SOLVE(512)
SLSE_DECL_SOLVE(1024)

// semifast solver (slse_solve_sf.cu, 128 threads per problem)
constexpr int kSfThreads = 128;
cudaError_t slse_solve_sf_occupancy(size_t smem, int* occ);
cudaError_t slse_solve_sf_launch(int grid, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                 const slse::cplx* ys, const int* idx, const slse::cplx* sc, int pstride, int B,
                                 const slse_outputs& out, char* ws, size_t slab, int* queue, const slse::cplx* tw,
                                 int twlog, int fft_cap);
cudaError_t slse_sf_bundle_launch(size_t smem, cudaStream_t st, const slse::SolveParams& P, const double* theta,
                                  const double* gamma, const int* kcount, int kstride, const double* beta,
                                  const slse::cplx* ys, const int* idx, const slse::cplx* sc, int pstride, int B,
                                  char* ws, size_t slab, const slse::cplx* tw, int twlog, int fft_cap,
                                  double* data_term, slse::cplx* e, slse::cplx* q, slse::cplx* r, slse::cplx* u,
                                  double* s, slse::cplx* t, slse::cplx* v, double* x, slse::cplx* q_grid,
                                  double* s_grid, int* status);

// CTA-pair solver (slse_solve_inst.cu): one problem per 2-CTA cluster
cudaError_t slse_solve_pair_launch_512(int clusters, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                       const slse::CfTable& cft, const slse::cplx* ys, int B,
                                       const slse_outputs& out, char* ws, size_t slab, int* queue,
                                       const slse::cplx* tw, int twlog, int fft_cap, slse::SplitJob* jobs);

// warp-mode solver (slse_solve_warps.cu): W one-warp solvers per CTA
cudaError_t slse_solve_warps_launch(int W, int ctas, size_t smem, cudaStream_t st, const slse::SolveParams& P,
                                    const slse::CfTable& cft, const slse::cplx* ys, int B, const slse_outputs& out,
                                    char* ws, size_t slab, int* queue, const slse::cplx* tw, int twlog, int fft_cap,
                                    int rec_smem, int warp_smem);
