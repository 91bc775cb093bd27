// slse_solver.cuh -- the whole Superfast-LSE estimate() for ONE problem,
// executed by one CTA (persistent; problems are pulled from a work queue).
//
// Mirrors estimator.estimate (estimator.py:117-275) for complete data and a
// single snapshot (G = 1): warm-up, initial activation sweeps
// (smlr.py:125-171), greedy activations (smlr.py:107-122), zeta and beta
// block updates (estimator.py:69-90,184-203), L-BFGS refinement
// (lbfgs.py:63-136) with deactivation (smlr.py:174-225) and the stopping
// rules.  Every scalar decision is computed redundantly by all threads from
// block reductions that return identical bits, so control flow is uniform.
#pragma once
#include "slse_stats.cuh"
#include "slse_dnc.cuh"
#include "slse_semifast.cuh"
#include "superlse_b200.h"

#ifdef SLSE_HOST_EMU
#include <chrono>
#endif

namespace slse {

constexpr double kEpsObjective = 2.220446049250313e-16;  // smlr.py:31
constexpr double kSweepWithin = 5.0;                     // smlr.py:35
constexpr double kSweepSpacing = 0.05;                   // smlr.py:36
constexpr double kGammaBarKInit = 4.0;                   // smlr.py:40
constexpr double kArmijoC1 = 1e-4;                       // lbfgs.py:21
constexpr double kBacktrack = 0.5;                       // lbfgs.py:22
constexpr int kMaxBacktracks = 30;                       // lbfgs.py:23
constexpr double kCurvEps = 1e-12;                       // lbfgs.py:26
constexpr double kInitialZeta = 0.2;                     // estimator.py:30
constexpr double kInitialBetaFrac = 0.01;                // estimator.py:31
constexpr double kBetaFloorScale = 1e-12;                // model_core.py:36
constexpr double kTiny = 2.2250738585072014e-308;        // np.finfo(float64).tiny

enum Stage : int { kStInit = 0, kStBeta = 1, kStActivate = 2, kStZeta = 3, kStRefine = 4, kStDeactivate = 5 };
enum EvKind : int { kEvSweep = 0, kEvActivate = 1, kEvDeactivate = 2, kEvEnd = -1 };
enum Flags : int { kFlConverged = 1, kFlKmaxCap = 2, kFlTraceFull = 4, kFlEventsFull = 8 };
enum Timer : int { kTmActivate = 0, kTmObjective = 1, kTmBeta = 2, kTmRefine = 3, kTmDeactivate = 4, kTmTotal = 5 };

// Optional per-phase cycle profile of the solver (build with
// -DSLSE_SOLVER_PROF; tools/solver_prof.py).  Leader-thread clock64 deltas,
// accumulated per problem and added to slse_prof_cycles at finish():
// 0 covariance column, 1 factor, 2 GS apply, 3 stats, 4 grid, 5 whole run,
// 6 waiting to enter an operation window, 7 waiting for it to close (warp mode),
// control code (exclusive of the operations inside): 8 sweep, 9 try_activate,
// 10 deactivate, 11 lbfgs_step, 12 record, 13 beta EM (residual_value);
// inside lbfgs_step: 14 the accepted point's stats call (inclusive),
// 15 gradient + memory push + slot update.
#ifdef SLSE_SOLVER_PROF
__device__ unsigned long long slse_prof_cycles[16];
#define SLSE_PROF_T0(v) const long long v = clock64()
#define SLSE_PROF_ADD(i, v) (prof_acc[i] += clock64() - (v))
// control-code slots: time inside the function minus the operations it ran
#define SLSE_PROF_C0(v) const long long v##_t = clock64(), v##_o = prof_ops()
#define SLSE_PROF_CADD(i, v) (prof_acc[i] += (clock64() - v##_t) - (prof_ops() - v##_o))
#else
#define SLSE_PROF_T0(v)
#define SLSE_PROF_ADD(i, v)
#define SLSE_PROF_C0(v)
#define SLSE_PROF_CADD(i, v)
#endif

// Control-code loops (thread-strided over k, dim, L): kept rolled -- the
// solver's control code is executed rarely per instruction but its size
// sets the instruction-cache footprint (SLSE_CTRL_UNROLL=1 restores the
// compiler's unrolling).
#ifdef SLSE_CTRL_UNROLL
#define SLSE_CTRL_LOOP
#else
#define SLSE_CTRL_LOOP _Pragma("unroll 1")
#endif

struct SolveParams {
  int n, L, kmax;
  int g;  // snapshots sharing the frequencies (MMV, estimator.py:278-283); 1 = single snapshot
  int max_outer, inner_max, sweep_iters, lbfgs_mem;
  int tcap, ecap;
  double tau, conv_tol_scale, dec_tol_scale;
  int dnc;  // 1: superfast divide-and-conquer Schur (slse_dnc.cuh), 0: Schur-Levinson
  int dnc_stockham;  // product transforms with the register Stockham passes
  int grid_fused;    // activation grid via the zero-padding-aware R x M decomposition
  int dnc_direct;    // superfast nodes up to this many steps use direct products
  int m;             // observed samples per snapshot (Observation.m; = n for complete data)
  int semifast;      // 1: semifast (Woodbury) bundles, slse_semifast.cuh (SLSE_SEMIFAST builds)
  int kcap;          // semifast: K x K matrices sized kcap (active sets beyond it stop, status 3)
};

// Superfast divide-and-conquer factorisation: decomp_method 2 ("schur",
// toeplitz.generalized_schur), or "auto" from kDncMinN up (the measured
// crossover of the two device factorisations; the reference's own auto
// switches at N > 256, toeplitz.py:36,263-276 -- both agree to ~1e-12).
constexpr int kDncMinN = 4096;
SLSE_HD bool use_dnc(int n, int decomp_method) {
  return decomp_method == 2 || (decomp_method == 0 && n >= kDncMinN);
}

// Launch-uniform parameters from the C-ABI options (estimator.py:34-50).
SLSE_HD SolveParams make_params(int n, const slse_options& o) {
  SolveParams P;
  P.n = n;
  P.g = 1;
  int target = 2 * n > o.grid_factor * n ? 2 * n : o.grid_factor * n;
  int L = 1;
  while (L < target) L <<= 1;  // model_core.py:224-227
  P.L = L;
  P.kmax = o.k_max > 0 ? o.k_max : n;
  P.max_outer = o.max_outer_iterations;
  P.inner_max = o.lbfgs_inner_max;
  P.sweep_iters = o.initial_sweep_iterations;
  P.lbfgs_mem = o.lbfgs_memory;
  P.tcap = o.trace_capacity > 0 ? o.trace_capacity : 2 + 13 * o.max_outer_iterations;
  P.ecap = o.event_capacity > 0 ? o.event_capacity : 4 * P.kmax + 64;
  P.tau = o.tau;
  P.conv_tol_scale = o.convergence_tol_scale;
  P.dec_tol_scale = o.newton_decrement_tol_scale;
  P.dnc = use_dnc(n, o.decomp_method) ? 1 : 0;
  P.dnc_stockham = 0;
  P.grid_fused = 1;
  P.dnc_direct = SLSE_DNC_DIRECT;
  P.m = n;
  P.semifast = 0;
  P.kcap = 0;
  return P;
}

// Per-CTA workspace layout (offsets in bytes from the CTA's slab).
struct Layout {
  size_t yhat, c, e, bg, a, dT, darena, rho[2], w[2], P, U, V, G0, G1, G2;
  size_t st_q[2], st_r[2], st_u[2], st_t[2], st_v[2], mu;
  size_t dtmp, dl, q2, sg, theta, gamma, act_theta, act_gamma, st_s[2], st_x[2];
  size_t lbS, lbY, lbR, diag, g0, gnew, dir, pt, cand, cth, cga, marg, cflist_d;
  size_t z, act_slot, cidx, csort;
  // semifast bundles (model_core.py:316-409): per bundle the Gram matrices,
  // the Cholesky factor (kcap x kcap) and the positive-variance list; shared
  // phases (m x kcap), solve scratch, A^H y and the grid's b(l) rows
  size_t sfG0[2], sfG1[2], sfG2[2], sfL[2], sfLd[2], sfP[2], sfE, sfX, sfAhy, sfBb;
  size_t total;
};

SLSE_HD size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

SLSE_HD Layout make_layout(int n, int L, int kmax, int lbfgs_mem, bool recursion_in_smem, bool dnc = false,
                           int g = 1, int semifast = 0, int m = 0, int kcap = 0) {
  Layout l;
  size_t o = 0;
  const size_t C = 16, D = 8, I = 4;
  const int nf = 1 << ilog2(2 * n);
  const size_t K = (size_t)kmax, K2 = 2 * (size_t)kmax;
  const size_t G = (size_t)g;
  l.yhat = o; o = al(o + C * nf * G);
  l.c = o; o = al(o + C * n);
  l.dT = l.darena = 0;
  if (dnc) {
    l.e = l.bg = l.a = 0;
    l.dT = o; o = al(o + C * 4 * (size_t)n);
    l.darena = o; o = al(o + C * (dnc_arena_elems(n - 1) + 16));
  } else if (recursion_in_smem) {
    l.e = l.bg = l.a = 0;
  } else {
    l.e = o; o = al(o + C * n);
    l.bg = o; o = al(o + C * n);
    l.a = o; o = al(o + C * n);
  }
  for (int i = 0; i < 2; ++i) { l.rho[i] = o; o = al(o + C * n); l.w[i] = o; o = al(o + C * n * G); }
  l.P = o; o = al(o + C * nf);
  l.U = o; o = al(o + C * nf);
  l.V = o; o = al(o + C * nf);
  l.G0 = o; o = al(o + C * L);
  l.G1 = o; o = al(o + C * L);
  l.G2 = o; o = al(o + C * L);
  for (int i = 0; i < 2; ++i) {
    l.st_q[i] = o; o = al(o + C * K * G);  // row g at g * kmax
    l.st_r[i] = o; o = al(o + C * K * G);
    l.st_u[i] = o; o = al(o + C * K * G);
    l.st_t[i] = o; o = al(o + C * K);
    l.st_v[i] = o; o = al(o + C * K);
    l.st_s[i] = o; o = al(o + D * K);
    l.st_x[i] = o; o = al(o + D * K);
  }
  l.mu = o; o = al(o + C * K * G);
  l.dtmp = o; o = al(o + D * n);
  l.dl = o; o = al(o + D * L);
  l.q2 = o; o = al(o + D * L);
  l.sg = o; o = al(o + D * L);
  l.theta = o; o = al(o + D * K);
  l.gamma = o; o = al(o + D * K);
  l.act_theta = o; o = al(o + D * K);
  l.act_gamma = o; o = al(o + D * K);
  l.lbS = o; o = al(o + D * K2 * lbfgs_mem);
  l.lbY = o; o = al(o + D * K2 * lbfgs_mem);
  l.lbR = o; o = al(o + D * (lbfgs_mem + 1));
  l.diag = o; o = al(o + D * K2);
  l.g0 = o; o = al(o + D * K2);
  l.gnew = o; o = al(o + D * K2);
  l.dir = o; o = al(o + D * K2);
  l.pt = o; o = al(o + D * K2);
  l.cand = o; o = al(o + D * K2);
  l.cth = o; o = al(o + D * K);
  l.cga = o; o = al(o + D * K);
  l.marg = o; o = al(o + D * K);
  l.cflist_d = o; o = al(o + D * L);
  l.z = o; o = al(o + I * K);
  l.act_slot = o; o = al(o + I * K);
  l.cidx = o; o = al(o + I * L);
  l.csort = o; o = al(o + I * L);
  for (int i = 0; i < 2; ++i) l.sfG0[i] = l.sfG1[i] = l.sfG2[i] = l.sfL[i] = l.sfLd[i] = l.sfP[i] = 0;
  l.sfE = l.sfX = l.sfAhy = l.sfBb = 0;
  if (semifast) {
    const size_t KC = (size_t)kcap, K2c = KC * KC;
    for (int i = 0; i < 2; ++i) {
      l.sfG0[i] = o; o = al(o + C * K2c);
      l.sfG1[i] = o; o = al(o + C * K2c);
      l.sfG2[i] = o; o = al(o + C * K2c);
      l.sfL[i] = o; o = al(o + C * K2c);
      l.sfLd[i] = o; o = al(o + D * KC);
      l.sfP[i] = o; o = al(o + I * KC);
    }
    l.sfE = o; o = al(o + C * (size_t)m * KC);
    l.sfX = o; o = al(o + C * KC * (KC > G ? KC : G));
    l.sfAhy = o; o = al(o + C * KC * G);
    l.sfBb = o; o = al(o + C * KC * (size_t)L);
  }
  l.total = o;
  return l;
}

// Outputs of one problem (pointers already offset to the problem).
struct ProbOut {
  int* khat;
  int* status;
  int* iters;
  int* flags;
  double* beta;
  double* zeta;
  double* theta;   // [kmax] active, slot order
  double* gamma;   // [kmax]
  cplx* alpha;     // [kmax]
  int* slot;       // [kmax]
  double* trace;   // [tcap]
  int* stage;      // [tcap]
  int* trace_k;    // [tcap]
  int* ntrace;
  int* events;     // [ecap][3]
  int* nevents;
  long long* counters;  // [4] builds, grids, stats, backtracks
  double* stage_s;      // [6] seconds per stage (estimator.py:106-114 buckets)
  double* iter_s;       // [max_outer] seconds per outer iteration (estimator.py:165,247), or nullptr
};

SLSE_D double prior_zeta(double zeta, int kmax) {  // model_core.py:230-234
  double z = fmax(zeta, 0.5 / (double)kmax);
  return z < 0.5 ? z : 0.5;
}

// Row 11: one deactivation margin (smlr.py:174-200); rhs = ln((1-ze)/ze).
// qq = sum over snapshots of |q_g|^2; G snapshots (the log1p term carries G).
SLSE_HD double deact_margin(double ga, double s, double qq, double rhs, int G = 1) {
  const double den = 1.0 - ga * s;
  if (ga <= 0.0) return rhs > 0.0 ? -INFINITY : 0.0;
  if (den <= 0.0) return INFINITY;
  const double q2dd = qq / (den * den);
  const double sdd = s / den;
  const double lg = log1p(ga * sdd);
  return (q2dd / (1.0 / ga + sdd) - (G == 1 ? lg : (double)G * lg)) - rhs;
}

// Row 12: gradient and diagonal Hessian of one component
// (model_core.py:497-536).  q, r, u point at snapshot 0 of this component,
// rows `stride` apart; G snapshots (sums over g, G factors as the reference).
SLSE_HD void grad_diag_comp(double ga, const cplx* q, const cplx* r, const cplx* u, size_t stride, int G, double s,
                            cplx t, cplx v, double x, int n, double* gth, double* gga, double* dth, double* dga) {
  cplx cross = cmul(conjg(q[0]), r[0]);
  double qq = cabs2(q[0]), rr = cabs2(r[0]);
  cplx rqc = cmul(r[0], conjg(q[0]));
  cplx uqc = cmul(u[0], conjg(q[0]));
  for (int g = 1; g < G; ++g) {
    const cplx qg = q[g * stride], rg = r[g * stride], ug = u[g * stride];
    cross = cadd(cross, cmul(conjg(qg), rg));
    qq += cabs2(qg);
    rr += cabs2(rg);
    rqc = cadd(rqc, cmul(rg, conjg(qg)));
    uqc = cadd(uqc, cmul(ug, conjg(qg)));
  }
  const double Gd = (double)G;
  *gth = 2.0 * ga * ((G == 1 ? t.im : Gd * t.im) - cross.im);
  *gga = (G == 1 ? s : Gd * s) - qq;
  // core = G (x - v) + ga G (t^2 - x s) + ga (x q2 + s r2 - 2 t rqc) + uqc - r2
  const cplx t2 = cmul(t, t);
  cplx c1 = mk(x - v.re, -v.im);
  cplx c2 = cscale(mk(t2.re - x * s, t2.im), ga);
  if (G != 1) {
    c1 = cscale(c1, Gd);
    c2 = cscale(mk(t2.re - x * s, t2.im), ga * Gd);
  }
  const cplx trq = cmul(mk(2.0 * t.re, 2.0 * t.im), rqc);
  const cplx c3 = cscale(mk(x * qq + s * rr - trq.re, -trq.im), ga);
  cplx core = cadd(cadd(c1, c2), c3);
  core = cadd(core, uqc);
  core.re -= rr;
  double d2t = 2.0 * ga * core.re;
  double d2g = 2.0 * s * qq - (G == 1 ? s * s : Gd * (s * s));
  if (d2t <= 0.0) d2t = (double)(50 * n) * (double)(50 * n);
  if (d2g <= 0.0) {
    const double sg_ = ga > 0.0 ? ga : 1.0 / (50.0 * (double)n);
    d2g = 1.0 / (sg_ * sg_);
  }
  *dth = d2t;
  *dga = d2g;
}


SLSE_D double prior_term(int k, double zeta, int kmax) {  // model_core.py:237-239
  const double ze = prior_zeta(zeta, kmax);
  return -((double)k * log(ze) + (double)(kmax - k) * log1p(-ze));
}

SLSE_D double np_mod1(double x) {  // numpy float mod by 1.0 (npy_divmod)
  double m = fmod(x, 1.0);
  if (m != 0.0) {
    if (m < 0.0) m += 1.0;
  } else {
    m = 0.0;
  }
  return m;
}

SLSE_D double wrap_dist(double x, double y) {  // simdata.py:50-53
  double d = np_mod1(fabs(x - y));
  double e = 1.0 - d;
  return d < e ? d : e;
}

SLSE_D unsigned long long now_ns() {
#ifdef SLSE_HOST_EMU
  return (unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
#else
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
#endif
}

// ---- CTA-pair jobs (slse_split.cuh) ----
struct SteerArgs {
  cplx* out;
  const double *th, *cre, *cim;
  int n, k, column;
  double beta0;
};
struct StatsArgs {
  const double* th;
  const cplx *rho, *w;
  cplx *q, *r, *u, *t, *v;
  double *s, *x;
  int K, n;
  double delta_last;
};

struct GridArgs {
  const cplx *rho, *w;
  double *dl, *q2, *sg;
  int n, L;
  double delta_last, gb, lr;
};

// One half (rank) of a job: the same device function as the single-CTA
// path, on this CTA's share of the work.
SLSE_D void run_split_job(const SplitJob& j, int rank, const CfTable* cf, const FftCtx& f, Blk& b) {
  if (j.kind == kJobSteer) {
    const SteerArgs a = j.get<SteerArgs>();
    steer_forward(a.out, a.n, a.th, a.cre, a.cim, a.k, a.beta0, a.column != 0, b, rank, 2);
  } else if (j.kind == kJobStats) {
    const StatsArgs a = j.get<StatsArgs>();
    Blk v = b;
    v.tid = b.tid + rank * b.nt;  // one warp per frequency: warps of both CTAs
    v.nt = 2 * b.nt;
    component_stats(a.th, a.K, a.rho, a.w, a.n, a.delta_last, cf, a.q, a.r, a.u, a.s, a.t, a.v, a.x, v);
  } else if (j.kind == kJobGsChain) {
    const GsChainArgs a = j.get<GsChainArgs>();
    gs_chain((cplx*)a.Y, a.n, a.nf, f, b);
  } else if (j.kind == kJobGrid) {
    const GridArgs a = j.get<GridArgs>();
    grid_gain_fused(a.rho, a.w, a.n, a.delta_last, a.L, a.gb, a.lr, a.dl, a.q2, a.sg, f, b, rank, 2);
  } else if (j.kind == kJobDncFft) {
    const DncFftArgs a = j.get<DncFftArgs>();
    const int cnt = dnc_fft_count(a.site);
    dnc_fft_site(a, rank ? cnt / 2 : 0, rank ? cnt : cnt / 2, f, b);
  }
}

struct Bundle {
  cplx* rho;
  cplx* w;  // C^{-1} y (superfast); e = Phi^H C^{-1} y (semifast), G rows of n
  cplx *q, *r, *u, *t, *v;
  double *s, *x;
  double data_term, delta_last, logdet;
  int stats_valid;
#ifdef SLSE_SEMIFAST
  // semifast (model_core.py:316-409): Gram matrices, Cholesky factor of
  // Sigma^{-1} (strict lower part + real diagonal sLd), positive list sP
  cplx *sG0, *sG1, *sG2, *sL;
  double* sLd;
  int* sP;
  int kp;
  double sbeta;
#endif
};

struct Solver {
  Blk& b;
  FftCtx f;
  const SolveParams& P;
  const CfTable* cf;
  const cplx* y;
  ProbOut o;
  // workspace
  cplx *yhat, *c, *e, *bg, *a, *dT, *darena, *PP, *U, *V, *G0, *G1, *G2, *mu;
  double *dtmp, *dl, *q2, *sg, *theta, *gamma, *act_theta, *act_gamma;
  double *lbS, *lbY, *lbR, *diag, *g0, *gnew, *dir, *pt, *cand, *cth, *cga, *marg;
  int *z, *act_slot, *cidx, *csort;
  Bundle bun[2];
  int cur;
  int cur_valid;
  // scalar state (identical in every thread)
  int n, L, kmax, k;
  Split* sp = nullptr;  // CTA pair (solve_kernel_pair): data-parallel jobs shared with the helper CTA
  int m;  // observed samples per snapshot (P.m): y holds G rows of m
#ifdef SLSE_SEMIFAST
  SfObs obs;
  cplx *sfE, *sfX, *sfAhy, *sfBb;
  const Bundle* sfE_of = nullptr;  // the bundle whose (theta, kk) the steering matrix sfE currently holds
  int sfE_kk = 0;
  int kcap;
#endif
  int G;  // snapshots (P.g): y, yhat and w hold G rows of n / nf; q, r, u, mu G rows of kmax
  double beta, zeta, energy, floor_beta;
  int status;
  int ntrace, nevents, flags;
  int mem_valid, mem_dim, mem_count, mem_head;
  long long n_builds, n_grids, n_stats, n_backtracks;
#ifdef SLSE_SOLVER_PROF
  long long prof_acc[16], prof_run0;
  SLSE_D long long prof_ops() const {
    return prof_acc[0] + prof_acc[1] + prof_acc[2] + prof_acc[3] + prof_acc[4] + prof_acc[6] + prof_acc[7];
  }
#endif
  unsigned long long t_mark, t_start;
  double tm[6];
  int free_hint;

  SLSE_D Solver(Blk& blk, const SolveParams& p, const CfTable* cf_, const cplx* y_, ProbOut out,
                char* slab, const Layout& lay, cplx* rec_smem, const FftCtx& fc)
      : b(blk), f(fc), P(p), cf(cf_), y(y_), o(out) {
    n = p.n; L = p.L; kmax = p.kmax; G = p.g;
    m = p.m;
#ifdef SLSE_SEMIFAST
    kcap = p.kcap;
    obs.idx = nullptr;
    obs.sc = nullptr;
    obs.m = m;
    sfE = (cplx*)(slab + lay.sfE); sfX = (cplx*)(slab + lay.sfX);
    sfAhy = (cplx*)(slab + lay.sfAhy); sfBb = (cplx*)(slab + lay.sfBb);
#endif
    yhat = (cplx*)(slab + lay.yhat);
    c = (cplx*)(slab + lay.c);
    if (rec_smem) {
      e = rec_smem; bg = rec_smem + n; a = rec_smem + 2 * n;
    } else {
      e = (cplx*)(slab + lay.e); bg = (cplx*)(slab + lay.bg); a = (cplx*)(slab + lay.a);
    }
    dT = (cplx*)(slab + lay.dT);
    darena = (cplx*)(slab + lay.darena);
    for (int i = 0; i < 2; ++i) {
      bun[i].rho = (cplx*)(slab + lay.rho[i]);
      bun[i].w = (cplx*)(slab + lay.w[i]);
      bun[i].q = (cplx*)(slab + lay.st_q[i]);
      bun[i].r = (cplx*)(slab + lay.st_r[i]);
      bun[i].u = (cplx*)(slab + lay.st_u[i]);
      bun[i].t = (cplx*)(slab + lay.st_t[i]);
      bun[i].v = (cplx*)(slab + lay.st_v[i]);
      bun[i].s = (double*)(slab + lay.st_s[i]);
      bun[i].x = (double*)(slab + lay.st_x[i]);
      bun[i].stats_valid = 0;
      bun[i].data_term = bun[i].delta_last = bun[i].logdet = 0.0;
#ifdef SLSE_SEMIFAST
      bun[i].sG0 = (cplx*)(slab + lay.sfG0[i]);
      bun[i].sG1 = (cplx*)(slab + lay.sfG1[i]);
      bun[i].sG2 = (cplx*)(slab + lay.sfG2[i]);
      bun[i].sL = (cplx*)(slab + lay.sfL[i]);
      bun[i].sLd = (double*)(slab + lay.sfLd[i]);
      bun[i].sP = (int*)(slab + lay.sfP[i]);
      bun[i].kp = 0;
      bun[i].sbeta = 0.0;
#endif
    }
    PP = (cplx*)(slab + lay.P); U = (cplx*)(slab + lay.U); V = (cplx*)(slab + lay.V);
    G0 = (cplx*)(slab + lay.G0); G1 = (cplx*)(slab + lay.G1); G2 = (cplx*)(slab + lay.G2);
    mu = (cplx*)(slab + lay.mu);
    dtmp = (double*)(slab + lay.dtmp);
    dl = (double*)(slab + lay.dl); q2 = (double*)(slab + lay.q2); sg = (double*)(slab + lay.sg);
    theta = (double*)(slab + lay.theta); gamma = (double*)(slab + lay.gamma);
    act_theta = (double*)(slab + lay.act_theta); act_gamma = (double*)(slab + lay.act_gamma);
    lbS = (double*)(slab + lay.lbS); lbY = (double*)(slab + lay.lbY); lbR = (double*)(slab + lay.lbR);
    diag = (double*)(slab + lay.diag); g0 = (double*)(slab + lay.g0); gnew = (double*)(slab + lay.gnew);
    dir = (double*)(slab + lay.dir); pt = (double*)(slab + lay.pt); cand = (double*)(slab + lay.cand);
    cth = (double*)(slab + lay.cth); cga = (double*)(slab + lay.cga); marg = (double*)(slab + lay.marg);
    z = (int*)(slab + lay.z); act_slot = (int*)(slab + lay.act_slot);
    cidx = (int*)(slab + lay.cidx); csort = (int*)(slab + lay.csort);
    cur = 0; cur_valid = 0; status = kOk; ntrace = 0; nevents = 0; flags = 0;
    mem_valid = 0; mem_dim = 0; mem_count = 0; mem_head = 0;
    n_builds = n_grids = n_stats = n_backtracks = 0;
#ifdef SLSE_SOLVER_PROF
    for (int i = 0; i < 16; ++i) prof_acc[i] = 0;
#endif
    for (int i = 0; i < 6; ++i) tm[i] = 0.0;
    free_hint = 0;
    k = 0;
  }

  // ---- timers (estimator.py:106-114) ----
  SLSE_D void lap(int which) {
    unsigned long long t = now_ns();
    tm[which] += (double)(t - t_mark) * 1e-9;
    t_mark = t;
  }

  // ---- active set bookkeeping ----
  // rebuild act_slot / act_theta / act_gamma from the slot arrays (slot order)
  SLSE_NIM void compact() {
    const int tid_ = b.tid, nt_ = b.nt;
    const int chunk = (kmax + nt_ - 1) / nt_;
    const int lo = tid_ * chunk;
    const int hi = lo + chunk < kmax ? lo + chunk : kmax;
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += z[i];
    int total = 0;
    int off = b.exscan(cnt, total);
    for (int i = lo; i < hi; ++i) {
      if (z[i]) {
        act_slot[off] = i;
        act_theta[off] = theta[i];
        act_gamma[off] = gamma[i];
        ++off;
      }
    }
    k = total;
    b.sync();
  }

  // lowest free slot (smlr.py:99-104); leader only
  SLSE_D int lowest_free() {
    int s = free_hint;
    while (s < kmax && z[s]) ++s;
    free_hint = s + 1;
    return s;
  }

  SLSE_D void push_event(int kind, int slot, int idx) {
    if (b.leader()) {
      if (nevents < P.ecap) {
        o.events[3 * nevents] = kind;
        o.events[3 * nevents + 1] = slot;
        o.events[3 * nevents + 2] = idx;
      }
    }
    if (nevents < P.ecap) ++nevents; else flags |= kFlEventsFull;
  }

  // steer_forward on this CTA, or split with the helper CTA of a pair
  SLSE_D void steer(cplx* out, const double* th, const double* cre, const double* cim, int kk, double be,
                      bool column) {
    if (SLSE_PAIR && sp) {
      SteerArgs a{out, th, cre, cim, n, kk, column ? 1 : 0, be};
      SplitJob j;
      j.set(kJobSteer, a);
      sp->post(j, b);
      steer_forward(out, n, th, cre, cim, kk, be, column, b, 0, 2);
      sp->done();
    } else {
      steer_forward(out, n, th, cre, cim, kk, be, column, b);
    }
  }

  // ---- model evaluation ----
  // Bundle for (th[0..kk), ga[0..kk), beta): model_core.py:257-274
  // Warp mode (several one-warp solvers per CTA, SLSE_WARP_MODE): every heavy
  // operation runs inside a CTA-wide operation window (rv_arrive ..
  // rv_depart, slse_port.cuh) and all control code between operations in
  // the complementary control window, so the SM never interleaves the
  // solver's large control code with the operations' hot loops
  // (instruction-cache locality; measured no-instruction stalls drop from
  // ~45 % of samples to ~1 %).  Long operations yield at rv_slice points.
  // A warp with no problem left keeps answering with an idle vote until the
  // whole CTA is idle (solve_kernel_warps).

  SLSE_NIM int build(Bundle& B, const double* th, const double* ga, int kk, double be) {
    ++n_builds;
#ifdef SLSE_SEMIFAST
    return sf_build(B, th, ga, kk, be);
#endif
    if (kk == 0) return build_white(B, be);
#ifdef SLSE_WARP_MODE
    SLSE_PROF_T0(w0);
    rv_arrive(0);
    SLSE_PROF_ADD(6, w0);
    const int st = build_impl(B, th, ga, kk, be);
    SLSE_PROF_T0(w1);
    rv_depart();
    SLSE_PROF_ADD(7, w1);
    return st;
#else
    return build_impl(B, th, ga, kk, be);
#endif
  }

  SLSE_NIM int build_impl(Bundle& B, const double* th, const double* ga, int kk, double be) {
    SLSE_PROF_T0(t0);
#ifndef SLSE_HOST_EMU
    if (b.nt == 32 && n <= 512) steer_forward_warp(c, n, th, ga, nullptr, kk, be, true, b.tid);
    else
#endif
      steer(c, th, ga, nullptr, kk, be, true);
    SLSE_PROF_ADD(0, t0);
    SLSE_PROF_T0(t1);
    Factor F = P.dnc ? toeplitz_factor_dnc(c, n, dT, darena, nullptr, dtmp, B.rho, f, b, P.dnc_stockham, P.dnc_direct,
                                           nullptr, sp)
                     : toeplitz_factor(c, n, e, bg, a, nullptr, dtmp, B.rho, b);
    SLSE_PROF_ADD(1, t1);
    if (F.status != kOk) return F.status;
    B.delta_last = F.delta_last;
    B.logdet = F.logdet;
    SLSE_PROF_T0(t2);
    const int nf = 1 << ilog2(2 * n);
    double quad = gs_apply_any(B.rho, n, F.delta_last, y, yhat, PP, U, V, B.w, f, b, sp);
    for (int g = 1; g < G; ++g)  // MMV: one C^{-1} y_g per snapshot (model_core.py:267-269)
      quad += gs_apply_any(B.rho, n, F.delta_last, y + (size_t)g * n, yhat + (size_t)g * nf, PP, U, V,
                           B.w + (size_t)g * n, f, b, sp);
    SLSE_PROF_ADD(2, t2);
    B.data_term = (G == 1 ? F.logdet : (double)G * F.logdet) + quad;
    B.stats_valid = 0;
    return kOk;
  }

  // Empty active set: C = beta I.  The recursion's reflection coefficients
  // are all exactly zero, so rho = e_{N-1}, every pivot is beta and
  // C^{-1} y = y / beta (exact; the reference's LD produces the same rho and
  // pivots bit for bit, toeplitz.py:135-142).
  SLSE_NIM int build_white(Bundle& B, double be) {
    if (!(be > 0.0)) return kBadColumn;  // c_0 must be real positive (toeplitz.py:55-57)
    const int tid_ = b.tid, nt_ = b.nt;
    const double inv = 1.0 / be;
    double qp = 0.0;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < n; i += nt_) B.rho[i] = mk(i == n - 1 ? 1.0 : 0.0, 0.0);
    SLSE_CTRL_LOOP
    for (int i = tid_; i < n * G; i += nt_) {
      const cplx wi = cscale(y[i], inv);
      B.w[i] = wi;
      qp += y[i].re * wi.re + y[i].im * wi.im;
    }
    const double quad = b.sum(qp);
    B.delta_last = be;
    B.logdet = (double)n * log(be);
    B.data_term = (G == 1 ? B.logdet : (double)G * B.logdet) + quad;
    B.stats_valid = 0;
    return kOk;
  }

  SLSE_NIM void stats(Bundle& B, const double* th, int kk) {
    if (B.stats_valid) return;
    ++n_stats;
#ifdef SLSE_SEMIFAST
    sf_stats(B, th, kk);
    return;
#endif
#if defined(SLSE_WARP_MODE) && defined(SLSE_STATS_RV)
    SLSE_PROF_T0(w0);
    rv_arrive(0);
    SLSE_PROF_ADD(6, w0);
    stats_impl(B, th, kk);
    SLSE_PROF_T0(w1);
    rv_depart();
    SLSE_PROF_ADD(7, w1);
#else
    stats_impl(B, th, kk);
#endif
  }

  SLSE_NIM void stats_impl(Bundle& B, const double* th, int kk) {
    SLSE_PROF_T0(t0);
    for (int g = 0; g < G; ++g) {  // s, t, v, x do not depend on g (recomputed identically)
      const cplx* wg = B.w + (size_t)g * n;
      cplx *qg = B.q + (size_t)g * kmax, *rg = B.r + (size_t)g * kmax, *ug = B.u + (size_t)g * kmax;
#ifndef SLSE_HOST_EMU
      if (b.nt == 32 && n <= 512)
        component_stats_warp(th, kk, B.rho, wg, n, B.delta_last, cf, qg, rg, ug, B.s, B.t, B.v, B.x, b.tid);
      else
#endif
      {
        if (SLSE_PAIR && sp) {
          StatsArgs a{th, B.rho, wg, qg, rg, ug, B.t, B.v, B.s, B.x, kk, n, B.delta_last};
          SplitJob j;
          j.set(kJobStats, a);
          sp->post(j, b);
          run_split_job(j, 0, cf, f, b);
          sp->done();
        } else {
          component_stats(th, kk, B.rho, wg, n, B.delta_last, cf, qg, rg, ug, B.s, B.t, B.v, B.x, b);
        }
      }
    }
    SLSE_PROF_ADD(3, t0);
    B.stats_valid = 1;
  }

  SLSE_D double objective(const Bundle& B) const { return B.data_term + prior_term(k, zeta, kmax); }

  SLSE_NIM int ensure_cur() {
    if (cur_valid) return kOk;
    int st = build(bun[cur], act_theta, act_gamma, k, beta);
    if (st == kOk) cur_valid = 1;
    return st;
  }

  SLSE_NIM void record(int stage) {
    SLSE_PROF_C0(pc);
    record_body(stage);
    SLSE_PROF_CADD(12, pc);
  }

  SLSE_NIM void record_body(int stage) {
    const double val = objective(bun[cur]);
    if (b.leader() && ntrace < P.tcap) {
      o.trace[ntrace] = val;
      o.stage[ntrace] = stage;
      o.trace_k[ntrace] = k;
    }
    if (ntrace < P.tcap) ++ntrace; else flags |= kFlTraceFull;
    last_trace = val;
  }
  double last_trace;

#ifdef SLSE_SEMIFAST
  // ---- semifast bundle (model_core._SemifastBundle :316-409) ----
  // Bundle for (th[0..kk), ga[0..kk), be) on the observation pattern `obs`:
  // Gram matrices, Cholesky of Sigma^{-1} over the positive-variance
  // components, ln|C|, y^H C^{-1} y and e = Phi^H C^{-1} y (:320-363).
  SLSE_NIM int sf_build(Bundle& B, const double* th, const double* ga, int kk, double be) {
    const int tid_ = b.tid, nt_ = b.nt;
    if (!(be > 0.0)) return kBadColumn;
    if (kk > kcap) return kCapacity;
    int kp = 0;
    SLSE_CTRL_LOOP
    for (int p = 0; p < kk; ++p) kp += ga[p] > 0.0 ? 1 : 0;  // self.pos (:325)
    if (tid_ == 0) {
      int j = 0;
      for (int p = 0; p < kk; ++p)
        if (ga[p] > 0.0) B.sP[j++] = p;
    }
    B.kp = kp;
    B.sbeta = be;
    // y^H y over the pattern, and A^H Phi^H y (steer_adjoint of scatter(y), :338)
    double yy = 0.0;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < m * G; i += nt_) yy += cabs2(y[i]);
    const double quad_y = b.sum(yy);
    double ln_c = (double)m * log(be);  // :339
    double quad = quad_y / be;
    if (kk) {
      sf_phases(sfE, m, obs, th, kk, b);
      sfE_of = &B;
      sfE_kk = kk;
      sf_gram(B.sG0, B.sG1, B.sG2, kcap, sfE, m, obs, kk, b, th, n);
      {
        // one (component, snapshot) item per group of lanes, the positions split over the group
        const int items = kk * G, nch = sf_chunks(items, nt_, 32), tot = items * nch;
        SLSE_CTRL_LOOP
        for (int base = 0; base < tot; base += nt_) {
          const int t = base + tid_;
          const bool act = t < tot;
          const int it = act ? t / nch : 0, ch = t - (t / nch) * nch;
          const int p = it / G, g = it - p * G;
          const cplx* yg = y + (size_t)g * m;
          const cplx* Ep = sfE + (size_t)p * m;
          cplx acc = mk(0.0, 0.0);
          if (act) {
#pragma unroll 4
            for (int i = ch; i < m; i += nch) {
              const cplx ys = cmulc(yg[i], sf_scale(obs, i));           // scatter: conj(a_i) y_i
              const cplx e = Ep[i];
              acc = mk(acc.re + e.re * ys.re + e.im * ys.im, acc.im + e.re * ys.im - e.im * ys.re);  // conj(E_ip) ys
            }
          }
          acc = sf_group_sum(acc, nch);
          if (act && ch == 0) sfAhy[it] = acc;
        }
      }
      b.sync();
    }
    if (kp) {
      const int st = sf_cholesky(B.sL, B.sLd, kcap, B.sG0, kcap, B.sP, ga, kp, be, b);  // :342-343
      if (st != kOk) return st;
      double lg = 0.0, ll = 0.0;
      SLSE_CTRL_LOOP
      for (int j = 0; j < kp; ++j) {
        lg += log(ga[B.sP[j]]);
        ll += log(B.sLd[j]);
      }
      ln_c += lg;         // :344
      ln_c += 2.0 * ll;   // :345
      // wp = Sigma A_P^H y (:346), kp x G
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * G; t += nt_) {
        const int j = t / G, g = t - j * G;
        sfX[t] = sfAhy[B.sP[j] * G + g];
      }
      b.sync();
      sf_cho_solve(B.sL, B.sLd, kcap, kp, sfX, G, G, b);
      double cr = 0.0;
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * G; t += nt_) {
        const int j = t / G, g = t - j * G;
        const cplx a = sfAhy[B.sP[j] * G + g], w = sfX[t];
        cr += a.re * w.re + a.im * w.im;  // Re(conj(A^H y) wp)
      }
      const double corr = b.sum(cr);
      quad = quad_y / be - corr / (be * be);  // :347-349
    }
    // e = scatter(y / beta - sample(A_P wp) / beta^2) (:350-351, :358)
    SLSE_CTRL_LOOP
    for (int i = tid_; i < n * G; i += nt_) B.w[i] = mk(0.0, 0.0);
    b.sync();
    SLSE_CTRL_LOOP
    for (int t = tid_; t < m * G; t += nt_) {
      const int g = t / m, i = t - g * m;
      const cplx a = sf_scale(obs, i);
      cplx cy = mk(y[t].re / be, y[t].im / be);
      if (kp) {
        cplx zs = mk(0.0, 0.0);
        SLSE_CTRL_LOOP
        for (int j = 0; j < kp; ++j) zs = cadd(zs, cmul(sfE[(size_t)B.sP[j] * m + i], sfX[j * G + g]));
        const cplx az = cmul(a, zs);
        const double b2 = be * be;
        cy = csub(cy, mk(az.re / b2, az.im / b2));
      }
      B.w[(size_t)g * n + obs.idx[i]] = cmulc(cy, a);  // conj(a_i) (C^{-1} y)_i
    }
    b.sync();
    B.data_term = (G == 1 ? ln_c : (double)G * ln_c) + quad;  // :355
    B.stats_valid = 0;
    return kOk;
  }

  // stats (:368-390): q, r, u = Psi^H [e, D e, D^2 e]; s, t, v, x from the
  // Gram diagonals minus the Woodbury terms diag(G_a[:,P] Sigma G_b[P,:])
  SLSE_NIM void sf_stats(Bundle& B, const double* th, int kk) {
    const int tid_ = b.tid, nt_ = b.nt;
    const double be = B.sbeta, b2 = be * be;
    // (a bundle's statistics and grid use the theta it was built from: its steering matrix is still
    // in sfE unless another bundle was built since)
    if (sfE_of != &B || sfE_kk != kk) {
      sf_phases(sfE, m, obs, th, kk, b);
      sfE_of = &B;
      sfE_kk = kk;
    }
    {
      const int items = kk * G, nch = sf_chunks(items, nt_, 32), tot = items * nch;
      SLSE_CTRL_LOOP
      for (int base = 0; base < tot; base += nt_) {
        const int t = base + tid_;
        const bool act = t < tot;
        const int it = act ? t / nch : 0, ch = t - (t / nch) * nch;
        const int g = it / kk, p = it - g * kk;
        const cplx* eg = B.w + (size_t)g * n;
        const cplx* Ep = sfE + (size_t)p * m;
        cplx aq = mk(0.0, 0.0), ar = aq, au = aq;
        if (act) {
#pragma unroll 4
          for (int i = ch; i < m; i += nch) {
            const int ni = obs.idx[i];
            const double d = 2.0 * kPi * (double)ni;
            const cplx ph = conjg(Ep[i]);
            const cplx e0 = eg[ni];
            aq = cadd(aq, cmul(ph, e0));
            ar = cadd(ar, cmul(ph, cscale(e0, d)));
            au = cadd(au, cmul(ph, cscale(e0, d * d)));
          }
        }
        aq = sf_group_sum(aq, nch);
        ar = sf_group_sum(ar, nch);
        au = sf_group_sum(au, nch);
        if (act && ch == 0) {
          B.q[(size_t)g * kmax + p] = aq;
          B.r[(size_t)g * kmax + p] = ar;
          B.u[(size_t)g * kmax + p] = au;
        }
      }
    }
    SLSE_CTRL_LOOP
    for (int p = tid_; p < kk; p += nt_) {
      B.s[p] = B.sG0[p * kcap + p].re / be;
      B.t[p] = mk(B.sG1[p * kcap + p].re / be, B.sG1[p * kcap + p].im / be);
      B.v[p] = mk(B.sG2[p * kcap + p].re / be, B.sG2[p * kcap + p].im / be);
      B.x[p] = B.sG2[p * kcap + p].re / be;
    }
    b.sync();
    const int kp = B.kp;
    if (kp) {
      // W00 = Sigma G0[P, :] (:381)
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * kk; t += nt_) {
        const int j = t / kk, c = t - j * kk;
        sfX[t] = B.sG0[B.sP[j] * kcap + c];
      }
      b.sync();
      sf_cho_solve(B.sL, B.sLd, kcap, kp, sfX, kk, kk, b);
      SLSE_CTRL_LOOP
      for (int c = tid_; c < kk; c += nt_) {
        double as = 0.0;
        cplx at = mk(0.0, 0.0), av = at;
        SLSE_CTRL_LOOP
        for (int j = 0; j < kp; ++j) {
          const cplx w = sfX[j * kk + c];
          const int pj = B.sP[j];
          const cplx g0 = B.sG0[c * kcap + pj], g1 = B.sG1[c * kcap + pj], g2 = B.sG2[c * kcap + pj];
          as += g0.re * w.re - g0.im * w.im;
          at = cadd(at, cmul(g1, w));
          av = cadd(av, cmul(g2, w));
        }
        B.s[c] -= as / b2;                                    // :382
        B.t[c] = csub(B.t[c], mk(at.re / b2, at.im / b2));   // :383
        B.v[c] = csub(B.v[c], mk(av.re / b2, av.im / b2));   // :384
      }
      b.sync();
      // W11 = Sigma G1[:, P]^H (:385), G1 Hermitian: rows G1[P, :]
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * kk; t += nt_) {
        const int j = t / kk, c = t - j * kk;
        sfX[t] = conjg(B.sG1[c * kcap + B.sP[j]]);
      }
      b.sync();
      sf_cho_solve(B.sL, B.sLd, kcap, kp, sfX, kk, kk, b);
      SLSE_CTRL_LOOP
      for (int c = tid_; c < kk; c += nt_) {
        double ax = 0.0;
        SLSE_CTRL_LOOP
        for (int j = 0; j < kp; ++j) {
          const cplx w = sfX[j * kk + c], g1 = B.sG1[c * kcap + B.sP[j]];
          ax += g1.re * w.re - g1.im * w.im;
        }
        B.x[c] -= ax / b2;  // :386
      }
      b.sync();
    }
    B.stats_valid = 1;
  }

  // grid (:392-409): q2 = sum_g |FFT_L(e_g)|^2, s^G = sum w0 / beta -
  // |L^{-1} b(l)|^2 / beta^2 with b_p = L IFFT_L(scatter(w0 e^{-j 2 pi n theta_p}))
  SLSE_NIM void sf_grid(Bundle& B, double gb, double lr, cplx* qg_out = nullptr) {
    const int tid_ = b.tid, nt_ = b.nt;
    const double be = B.sbeta, b2 = be * be;
    for (int g = 0; g < G; ++g) {
      const cplx* eg = B.w + (size_t)g * n;
      const int nn = n;
      double* q2_ = q2;
      const int first = g == 0;
      cplx* qo = qg_out ? qg_out + (size_t)g * L : nullptr;
      fft(G0, L, -1.0, [=](int i) { return i < nn ? eg[i] : mk(0.0, 0.0); },
          [=](int l, cplx v) {
            q2_[l] = (first ? 0.0 : q2_[l]) + cabs2(v);
            if (qo) qo[l] = v;
          }, f, b);
    }
    double w0s = 0.0;
    SLSE_CTRL_LOOP
    for (int i = 0; i < m; ++i) w0s += sf_w0(obs, i);
    const double base = w0s / be;  // :397
    const int kp = B.kp;
    if (kp) {
      if (sfE_of != &B || sfE_kk != k) {
        sf_phases(sfE, m, obs, act_theta, k, b);
        sfE_of = &B;
        sfE_kk = k;
      }
      // b_p(l), p in P (:400-403): scatter every row, then one batched
      // inverse transform of the kp rows (in place)
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * L; t += nt_) sfBb[t] = mk(0.0, 0.0);
      b.sync();
      SLSE_CTRL_LOOP
      for (int t = tid_; t < kp * m; t += nt_) {
        const int j = t / m, i = t - j * m;
        sfBb[(size_t)j * L + obs.idx[i]] = cscale(conjg(sfE[(size_t)B.sP[j] * m + i]), sf_w0(obs, i));
      }
      b.sync();
      {
        cplx* bb = sfBb;
        const int LL = L;
        fft_multi(G1, kp, L, +1.0, [=](int c, int i) { return bb[(size_t)c * LL + i]; },
                  [=](int c, int l, cplx v) { bb[(size_t)c * LL + l] = v; }, f, b);
      }
      // |L^{-1} b(l)|^2 per grid point (b^H Sigma b, :404-405), in place
      SLSE_CTRL_LOOP
      for (int l = tid_; l < L; l += nt_) {
        double acc = 0.0;
        SLSE_CTRL_LOOP
        for (int j = 0; j < kp; ++j) {
          cplx a = sfBb[(size_t)j * L + l];
          const cplx* Lj = B.sL + j * kcap;
          const cplx* bl = sfBb + l;
#pragma unroll 4
          for (int c = 0; c < j; ++c) {  // (the solved entries a_c are final: independent loads)
            const cplx lc = Lj[c], ac = bl[(size_t)c * L];
            a = mk(fma(lc.im, ac.im, fma(-lc.re, ac.re, a.re)), fma(-lc.im, ac.re, fma(-lc.re, ac.im, a.im)));
          }
          const double inv = 1.0 / B.sLd[j];  // uniform: one reciprocal per pivot, not two divisions per point
          a = mk(a.re * inv, a.im * inv);
          sfBb[(size_t)j * L + l] = a;
          acc += cabs2(a);
        }
        sg[l] = base - acc / b2;
      }
    } else {
      SLSE_CTRL_LOOP
      for (int l = tid_; l < L; l += nt_) sg[l] = base;
    }
    SLSE_CTRL_LOOP
    for (int l = tid_; l < L; l += nt_) dl[l] = gain_g(q2[l], sg[l], gb, lr, G);
    b.sync();
  }
#endif

  // ---- activation (smlr.py:53-171) ----
  SLSE_NIM double gamma_bar() {
    const int tid_ = b.tid, nt_ = b.nt;  // smlr.py:53-59
    if (k) {
      double part = 0.0;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < k; i += nt_) part += act_gamma[i];
      double bar = b.sum(part) / (double)k;
      if (bar > 0.0) return bar;
    }
    double g = energy / ((double)m * kGammaBarKInit);  // obs.m (smlr.py:59)
    return g > kTiny ? g : kTiny;
  }

  SLSE_NIM void grid_curve(double gb, double ze) {
    ++n_grids;
#if defined(SLSE_WARP_MODE) && defined(SLSE_GRID_RV)
    SLSE_PROF_T0(w0);
    rv_arrive(0);
    SLSE_PROF_ADD(6, w0);
    grid_impl(gb, ze);
    SLSE_PROF_T0(w1);
    rv_depart();
    SLSE_PROF_ADD(7, w1);
#else
    grid_impl(gb, ze);
#endif
  }

  SLSE_NIM void grid_impl(double gb, double ze) {
    const int tid_ = b.tid, nt_ = b.nt;
    Bundle& B = bun[cur];
    const double lr = log((1.0 - ze) / ze);
#ifdef SLSE_SEMIFAST
    sf_grid(B, gb, lr);
    return;
#endif
    SLSE_PROF_T0(t0);
    if (SLSE_PAIR && sp && G == 1 && P.grid_fused) {
      GridArgs a{B.rho, B.w, dl, q2, sg, n, L, B.delta_last, gb, lr};
      SplitJob j;
      j.set(kJobGrid, a);
      sp->post(j, b);
      const bool ok = grid_gain_fused(B.rho, B.w, n, B.delta_last, L, gb, lr, dl, q2, sg, f, b, 0, 2);
      sp->done();
      if (ok) {
        SLSE_PROF_ADD(4, t0);
        return;
      }
    } else if (G == 1 && P.grid_fused && grid_gain_fused(B.rho, B.w, n, B.delta_last, L, gb, lr, dl, q2, sg, f, b)) {
      SLSE_PROF_ADD(4, t0);
      return;
    }
    // q2 = sum_g |q^G_g|^2, gain with the G log1p term (smlr.py:62-70)
    for (int g = 0; g < G; ++g) {
      grid_eval(B.rho, B.w + (size_t)g * n, n, B.delta_last, L, G0, G1, G2, sg, f, b);
      SLSE_CTRL_LOOP
      for (int l = tid_; l < L; l += nt_) q2[l] = (g == 0 ? 0.0 : q2[l]) + cabs2(G0[l]);
      b.sync();
    }
    SLSE_CTRL_LOOP
    for (int l = tid_; l < L; l += nt_) dl[l] = gain_g(q2[l], sg[l], gb, lr, G);
    b.sync();
  }

  SLSE_D static double gamma_estimate(double kappa, double s) {  // smlr.py:73-76
    return kappa > 1.0 ? (kappa * s - s) / (s * s) : 0.0;
  }

  SLSE_D static bool snr_ok(double kappa, double s, double gb, double ze, double tau) {  // smlr.py:79-81
    const double rhs = (1.0 + 1.0 / (gb * s)) * log((1.0 + gb * s) * (1.0 - ze) / ze);
    return kappa > rhs + tau;
  }

  // returns 1 if a component was activated (smlr.py:107-122)
  SLSE_NIM int try_activate() {
    SLSE_PROF_C0(pc);
    const int rv_ = try_activate_body();
    SLSE_PROF_CADD(9, pc);
    return rv_;
  }

  SLSE_NIM int try_activate_body() {
    const int tid_ = b.tid, nt_ = b.nt;
    if (k >= kmax) return 0;
    const double gb = gamma_bar();
    const double ze = prior_zeta(zeta, kmax);
    grid_curve(gb, ze);
    double best = 0.0;
    int bi = -1;
    SLSE_CTRL_LOOP
    for (int l = tid_; l < L; l += nt_) {
      const double d = dl[l];
      if (Blk::better(d, l, best, bi)) { best = d; bi = l; }
    }
    b.argmin(best, bi);
    if (bi < 0) return 0;
    const double s = sg[bi];
    const double kappa = (G == 1 ? q2[bi] : q2[bi] / (double)G) / s;
    const double gam = gamma_estimate(kappa, s);
    if (best >= -kEpsObjective || gam <= 0.0) return 0;
    if (!snr_ok(kappa, s, gb, ze, P.tau)) return 0;
    int slot = 0;
    if (b.leader()) {
      slot = lowest_free();
      z[slot] = 1;
      theta[slot] = (double)bi / (double)L;
      gamma[slot] = gam;
    }
    slot = b.bcast_i(slot);
    free_hint = slot + 1;
    push_event(kEvActivate, slot, bi);
    push_event(kEvEnd, -1, -1);
    compact();
    cur_valid = 0;
    return 1;
  }

  // initial multi-activation sweep (smlr.py:125-171); returns #added
  SLSE_NIM int sweep() {
    SLSE_PROF_C0(pc);
    const int rv_ = sweep_body();
    SLSE_PROF_CADD(8, pc);
    return rv_;
  }

  SLSE_NIM int sweep_body() {
    const int tid_ = b.tid, nt_ = b.nt;
    const double gb = gamma_bar();
    const double ze = prior_zeta(zeta, kmax);
    grid_curve(gb, ze);
    // circular local minima and their minimum
    double mn = 0.0;
    int mi = -1;
    SLSE_CTRL_LOOP
    for (int l = tid_; l < L; l += nt_) {
      const double d = dl[l];
      const double dp = dl[(l + L - 1) & (L - 1)], dn = dl[(l + 1) & (L - 1)];
      if (d <= dp && d <= dn) {
        if (Blk::better(d, l, mn, mi)) { mn = d; mi = l; }
      }
    }
    b.argmin(mn, mi);
    if (mi < 0) return 0;
    const double dmin = mn;
    if (dmin >= -kEpsObjective) return 0;
    const double thr = dmin / kSweepWithin;
    // compact qualifying minima in index order
    const int chunk = (L + nt_ - 1) / nt_;
    const int lo = tid_ * chunk;
    const int hi = lo + chunk < L ? lo + chunk : L;
    int cnt = 0;
    for (int l = lo; l < hi; ++l) {
      const double d = dl[l];
      const double dp = dl[(l + L - 1) & (L - 1)], dn = dl[(l + 1) & (L - 1)];
      if (d <= dp && d <= dn && d < -kEpsObjective && !(d > thr)) ++cnt;
    }
    int m = 0;
    int off = b.exscan(cnt, m);
    for (int l = lo; l < hi; ++l) {
      const double d = dl[l];
      const double dp = dl[(l + L - 1) & (L - 1)], dn = dl[(l + 1) & (L - 1)];
      if (d <= dp && d <= dn && d < -kEpsObjective && !(d > thr)) cidx[off++] = l;
    }
    b.sync();
    // stable sort by (delta, index): rank = #{j: (d_j, j) < (d_i, i)}
    SLSE_CTRL_LOOP
    for (int i = tid_; i < m; i += nt_) {
      const int li = cidx[i];
      const double di = dl[li];
      int rank = 0;
      for (int j = 0; j < m; ++j) {
        const int lj = cidx[j];
        const double dj = dl[lj];
        rank += (dj < di || (dj == di && lj < li)) ? 1 : 0;
      }
      csort[rank] = li;
    }
    b.sync();
    // serial pass in sorted order (leader), activating as in the reference
    int added = 0;
    if (b.leader()) {
      const double spacing = kSweepSpacing / (double)n;
      int kk = k;
      for (int i = 0; i < m; ++i) {
        if (kk >= kmax) break;
        const int l = csort[i];
        const double s = sg[l];
        const double kappa = (G == 1 ? q2[l] : q2[l] / (double)G) / s;
        const double gnew_ = gamma_estimate(kappa, s);
        if (gnew_ <= 0.0) continue;
        const double tau_eff = (kk == 0) ? P.tau : 0.0;
        if (!snr_ok(kappa, s, gb, ze, tau_eff)) continue;
        const double th = (double)l / (double)L;
        if (kk) {
          double dmn = 2.0;
          for (int j = 0; j < k; ++j) { double dd = wrap_dist(th, act_theta[j]); dmn = dd < dmn ? dd : dmn; }
          for (int j = 0; j < added; ++j) { double dd = wrap_dist(th, cth[j]); dmn = dd < dmn ? dd : dmn; }
          if (dmn < spacing) continue;
        }
        const int slot = lowest_free();
        z[slot] = 1;
        theta[slot] = th;
        gamma[slot] = gnew_;
        cth[added] = th;
        marg[added] = (double)slot;  // scratch: remember slot order of additions
        cidx[added] = l;             // cidx no longer needed; reuse for grid index
        ++added;
        ++kk;
      }
    }
    added = b.bcast_i(added);
    if (added) {
      for (int i = 0; i < added; ++i) push_event(kEvSweep, (int)marg[i], cidx[i]);
      push_event(kEvEnd, -1, -1);
      compact();
      cur_valid = 0;
    } else {
      b.sync();
    }
    return added;
  }

  // ---- deactivation (smlr.py:174-225) ----
  // on return: number removed; cur is valid for the new state (stats too if k>0)
  SLSE_NIM int deactivate(int* st) {
    SLSE_PROF_C0(pc);
    const int rv_ = deactivate_body(st);
    SLSE_PROF_CADD(10, pc);
    return rv_;
  }

  SLSE_NIM int deactivate_body(int* st) {
    const int tid_ = b.tid, nt_ = b.nt;
    int removed = 0;
    *st = kOk;
    while (k) {
      Bundle& B = bun[cur];
      const double ze = prior_zeta(zeta, kmax);
      const double rhs = log((1.0 - ze) / ze);
      double wv = 0.0;
      int wi = -1;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < k; i += nt_) {
        double qq = cabs2(B.q[i]);
        for (int g = 1; g < G; ++g) qq += cabs2(B.q[(size_t)g * kmax + i]);
        const double mgn = deact_margin(act_gamma[i], B.s[i], qq, rhs, G);
        if (Blk::better(mgn, i, wv, wi)) { wv = mgn; wi = i; }
      }
      b.argmin(wv, wi);
      if (wi < 0 || !(wv < 0.0)) break;
      const int slot = act_slot[wi];
      if (b.leader()) {
        z[slot] = 0;
        gamma[slot] = 0.0;
      }
      if (slot < free_hint) free_hint = slot;
      b.sync();
      push_event(kEvDeactivate, slot, -1);
      ++removed;
      compact();
      cur_valid = 0;
      if (k == 0) break;
      *st = ensure_cur();
      if (*st != kOk) return removed;
      stats(bun[cur], act_theta, k);
    }
    if (removed) push_event(kEvEnd, -1, -1);
    return removed;
  }

  // ---- gradient / diag Hessian (model_core.py:497-536) ----
  SLSE_NIM void gradient(const Bundle& B, const double* ga, double* g) {
    const int tid_ = b.tid, nt_ = b.nt;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < k; i += nt_) {
      double dth, dga;
      grad_diag_comp(ga[i], B.q + i, B.r + i, B.u + i, (size_t)kmax, G, B.s[i], B.t[i], B.v[i], B.x[i], n, &g[i],
                     &g[k + i], &dth, &dga);
    }
  }

  SLSE_NIM void diag_hessian(const Bundle& B, const double* ga_, double* d) {
    const int tid_ = b.tid, nt_ = b.nt;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < k; i += nt_) {
      double gth, gga;
      grad_diag_comp(ga_[i], B.q + i, B.r + i, B.u + i, (size_t)kmax, G, B.s[i], B.t[i], B.v[i], B.x[i], n, &gth,
                     &gga, &d[i], &d[k + i]);
    }
  }

  // ---- L-BFGS (lbfgs.py) ----
  SLSE_D double dot(const double* p, const double* q, int dim) {
    const int tid_ = b.tid, nt_ = b.nt;
    double part = 0.0;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) part += p[i] * q[i];
    return b.sum(part);
  }

  // two-loop recursion into dir (lbfgs.py:63-76); uses gnew as q scratch
#ifndef SLSE_HOST_EMU
  // One-warp two-loop recursion for dim <= 64 (two entries per lane): q and
  // the direction stay in registers, the memory pairs are read once, the
  // dot products are warp xor-sums (the same bits as Blk::sum for one warp),
  // and the loop over pairs is unrolled with predicates so the alphas stay in
  // registers.  Same arithmetic as two_loop.
  SLSE_NIM void two_loop_warp(int dim) {
    const int lane = b.tid;
    const bool in0 = lane < dim, in1 = lane + 32 < dim;
    double q0 = in0 ? g0[lane] : 0.0, q1 = in1 ? g0[lane + 32] : 0.0;
    const int K2 = 2 * kmax;
    const int mc = mem_count;
    double alphas[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {  // jj = mc - 1 - t, descending
      alphas[t] = 0.0;
      if (t < mc) {
        const int slot = (mem_head + (mc - 1 - t)) % P.lbfgs_mem;
        const double* S = lbS + (size_t)slot * K2;
        const double* Y = lbY + (size_t)slot * K2;
        double part = 0.0;
        if (in0) part += S[lane] * q0;
        if (in1) part += S[lane + 32] * q1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const double al_ = lbR[slot] * part;
        alphas[t] = al_;
        if (in0) q0 -= al_ * Y[lane];
        if (in1) q1 -= al_ * Y[lane + 32];
      }
    }
    double d0 = in0 ? q0 / diag[lane] : 0.0, d1 = in1 ? q1 / diag[lane + 32] : 0.0;
#pragma unroll
    for (int t = 15; t >= 0; --t) {  // jj = mc - 1 - t, ascending
      if (t < mc) {
        const int slot = (mem_head + (mc - 1 - t)) % P.lbfgs_mem;
        const double* S = lbS + (size_t)slot * K2;
        const double* Y = lbY + (size_t)slot * K2;
        double part = 0.0;
        if (in0) part += Y[lane] * d0;
        if (in1) part += Y[lane + 32] * d1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const double be = lbR[slot] * part;
        const double coef = alphas[t] - be;
        if (in0) d0 += S[lane] * coef;
        if (in1) d1 += S[lane + 32] * coef;
      }
    }
    if (in0) dir[lane] = -d0;
    if (in1) dir[lane + 32] = -d1;
    __syncwarp();
  }
#endif

  SLSE_NIM void two_loop(int dim) {
#ifndef SLSE_HOST_EMU
    if (b.nt == 32 && dim <= 64 && P.lbfgs_mem <= 16) {
      two_loop_warp(dim);
      return;
    }
#endif
    const int tid_ = b.tid, nt_ = b.nt;
    double alphas[16];
    double* qv = gnew;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) qv[i] = g0[i];
    const int K2 = 2 * kmax;
    for (int jj = mem_count - 1; jj >= 0; --jj) {
      const int slot = (mem_head + jj) % P.lbfgs_mem;
      const double* S = lbS + (size_t)slot * K2;
      const double* Y = lbY + (size_t)slot * K2;
      const double al_ = lbR[slot] * dot(S, qv, dim);
      alphas[jj] = al_;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < dim; i += nt_) qv[i] -= al_ * Y[i];
    }
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) dir[i] = qv[i] / diag[i];
    for (int jj = 0; jj < mem_count; ++jj) {
      const int slot = (mem_head + jj) % P.lbfgs_mem;
      const double* S = lbS + (size_t)slot * K2;
      const double* Y = lbY + (size_t)slot * K2;
      const double be = lbR[slot] * dot(Y, dir, dim);
      const double coef = alphas[jj] - be;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < dim; i += nt_) dir[i] += S[i] * coef;
    }
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) dir[i] = -dir[i];
  }

  // memory.push(alpha*dir, gnew - g0) (lbfgs.py:47-53)
  SLSE_NIM void push_pair(double alpha, int dim) {
    const int tid_ = b.tid, nt_ = b.nt;
    const int K2 = 2 * kmax;
    const int slot = (mem_count < P.lbfgs_mem) ? (mem_head + mem_count) % P.lbfgs_mem : mem_head;
    double* S = lbS + (size_t)slot * K2;
    double* Y = lbY + (size_t)slot * K2;
    double pv[3] = {0.0, 0.0, 0.0};
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) {
      const double s = alpha * dir[i];
      const double yv = gnew[i] - g0[i];
      S[i] = s;
      Y[i] = yv;
      pv[0] += s * yv;
      pv[1] += s * s;
      pv[2] += yv * yv;
    }
    b.sumv(pv, 3);
    const double curv = pv[0];
    if (curv <= kCurvEps * sqrt(pv[1]) * sqrt(pv[2])) return;
    if (b.leader()) lbR[slot] = 1.0 / curv;
    if (mem_count < P.lbfgs_mem) {
      ++mem_count;
    } else {
      mem_head = (mem_head + 1) % P.lbfgs_mem;
    }
    b.sync();
  }

  // One lbfgs_step (lbfgs.py:100-136).  Returns 0 accepted, 1 line-search
  // failure, or a negative model status.  On acceptance the new point is in
  // the slot arrays, cur is the accepted bundle (stats valid), *dec set.
  SLSE_NIM int lbfgs_step(double f0, double* dec) {
    SLSE_PROF_C0(pc);
    const int rv_ = lbfgs_step_body(f0, dec);
    SLSE_PROF_CADD(11, pc);
    return rv_;
  }

  SLSE_NIM int lbfgs_step_body(double f0, double* dec) {
    const int tid_ = b.tid, nt_ = b.nt;
    const int dim = 2 * k;
    // any(g0)?
    double nz = 0.0;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < dim; i += nt_) nz += (g0[i] != 0.0) ? 1.0 : 0.0;
    if (b.sum(nz) == 0.0) {
      *dec = 0.0;
      return 0;  // point unchanged
    }
    two_loop(dim);
    double slope = dot(g0, dir, dim);
    if (slope >= 0.0) {
      SLSE_CTRL_LOOP
      for (int i = tid_; i < dim; i += nt_) dir[i] = -g0[i] / diag[i];
      slope = dot(g0, dir, dim);
    }
    *dec = -slope;
    // gamma step cap (lbfgs.py:84-90)
    double capv = INFINITY;
    SLSE_CTRL_LOOP
    for (int i = tid_; i < k; i += nt_) {
      const double dg = dir[k + i];
      if (dg < 0.0) {
        const double r = pt[k + i] / -dg;
        capv = r < capv ? r : capv;
      }
    }
    capv = b.minv(capv);
    double alpha = capv < 1.0 ? capv : 1.0;
    if (alpha <= 0.0) return 1;
    Bundle& T = bun[cur ^ 1];
    SLSE_PROF_C0(pl);
    for (int bt = 0; bt < kMaxBacktracks; ++bt) {
      ++n_backtracks;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < k; i += nt_) {
        cth[i] = np_mod1(pt[i] + alpha * dir[i]);
        cga[i] = pt[k + i] + alpha * dir[k + i];
        cand[i] = cth[i];
        cand[k + i] = cga[i];
      }
      b.sync();
      int st = build(T, cth, cga, k, beta);
      if (st != kOk) return -st;
      const double fn = T.data_term + prior_term(k, zeta, kmax);
      if (fn <= f0 + kArmijoC1 * alpha * slope) {
        SLSE_PROF_T0(ps);
        stats(T, cth, k);
        SLSE_PROF_ADD(14, ps);
        SLSE_PROF_T0(pa);
        gradient(T, cga, gnew);
        b.sync();
        push_pair(alpha, dim);
        // accept: write the point into the slots; swap bundles
        SLSE_CTRL_LOOP
        for (int i = tid_; i < k; i += nt_) {
          const int s = act_slot[i];
          theta[s] = cth[i];
          gamma[s] = cga[i];
          act_theta[i] = cth[i];
          act_gamma[i] = cga[i];
        }
        b.sync();
        cur ^= 1;
        cur_valid = 1;
        SLSE_PROF_ADD(15, pa);
        return 0;
      }
      alpha *= kBacktrack;
    }
    return 1;
  }

  // ---- the outer loop (estimator.py:117-275) ----
  SLSE_NIM void run() {
    t_start = now_ns();
#ifdef SLSE_SOLVER_PROF
    prof_run0 = clock64();
#endif
    t_mark = t_start;
    // energy, floor, beta0 (model_core.py:125-130; estimator.py:135-137)
    double part = 0.0;
    for (int i = b.tid; i < m * G; i += b.nt) {
      part += cabs2(y[i]);
    }
    energy = b.sum(part);
    if (G != 1) energy /= (double)G;  // mean per-snapshot energy (model_core.py:125-127)
    floor_beta = kBetaFloorScale * energy / (double)m;
    const double b0 = kInitialBetaFrac * energy / (double)m;
    beta = b0 > floor_beta ? b0 : floor_beta;
    zeta = kInitialZeta;
    for (int i = b.tid; i < kmax; i += b.nt) { z[i] = 0; theta[i] = 0.0; gamma[i] = 0.0; }
    k = 0;
    // cached spectrum of y for every GS apply (superfast)
#ifndef SLSE_SEMIFAST
    for (int g = 0; g < G; ++g) {
      const cplx* yg = y + (size_t)g * n;
      cplx* yh = yhat + ((size_t)g << ilog2(2 * n));
      fft(yh, 1 << ilog2(2 * n), -1.0, [=](int i) { return i < n ? yg[i] : mk(0.0, 0.0); },
          [=](int i, cplx v) { yh[i] = v; }, f, b);
    }
#endif
    status = ensure_cur();
    if (status != kOk) { finish(0, 0); return; }
    record(kStInit);
    {  // warm-up beta (estimator.py:153)
      const double v = energy / (double)m;
      beta = floor_beta > v ? floor_beta : v;
      cur_valid = 0;
    }
    status = ensure_cur();
    if (status != kOk) { finish(0, 0); return; }
    record(kStBeta);
    lap(kTmObjective);
    double previous = last_trace;
    int z_dirty = 1;
    int converged = 0;
    int iterations = 0;
    for (int it = 1; it <= P.max_outer; ++it) {
      iterations = it;
      const unsigned long long t_iter = now_ns();
      // 1) activation
      if (it <= P.sweep_iters) {
        status = ensure_cur();
        if (status != kOk) break;
        if (sweep()) z_dirty = 1;
      } else {
        int hit_cap = 1;
        for (int rep = 0; rep < kmax; ++rep) {
          status = ensure_cur();
          if (status != kOk) break;
          if (!try_activate()) { hit_cap = 0; break; }
          z_dirty = 1;
        }
        if (status != kOk) break;
        if (hit_cap) flags |= kFlKmaxCap;
      }
      lap(kTmActivate);
      status = ensure_cur();
      if (status != kOk) break;
      record(kStActivate);
      lap(kTmObjective);
      // 2) zeta (estimator.py:69-74)
      {
        const double zz = (double)k / (double)kmax;
        zeta = zz < 0.5 ? zz : 0.5;
      }
      record(kStZeta);
      // 3) beta EM step (estimator.py:184-203)
      double value;
      if (k) {
        Bundle& B = bun[cur];
        stats(B, act_theta, k);
        double tr_part = 0.0;
        for (int i = b.tid; i < k; i += b.nt) {
          for (int g = 0; g < G; ++g) mu[(size_t)g * kmax + i] = cscale(B.q[(size_t)g * kmax + i], act_gamma[i]);
          tr_part += B.s[i] * act_gamma[i];
        }
        const double tr = beta * b.sum(tr_part);
        value = residual_value(tr);
      } else {
        value = energy / (double)m;
      }
      const double bc = floor_beta > value ? floor_beta : value;
      {
        Bundle& T = bun[cur ^ 1];
        status = build(T, act_theta, act_gamma, k, bc);
        if (status != kOk) break;
        const double fc = T.data_term + prior_term(k, zeta, kmax);
        if (fc <= last_trace) {
          beta = bc;
          cur ^= 1;
          cur_valid = 1;
        }
      }
      lap(kTmBeta);
      record(kStBeta);
      lap(kTmObjective);
      // 4) refinement (estimator.py:206-245)
      if (k) {
        for (int inner = 0; inner < P.inner_max; ++inner) {
          Bundle& B = bun[cur];
          stats(B, act_theta, k);
          if (z_dirty || !mem_valid || mem_dim != 2 * k) {
            diag_hessian(B, act_gamma, diag);
            mem_valid = 1;
            mem_dim = 2 * k;
            mem_count = 0;
            mem_head = 0;
            z_dirty = 0;
          }
          gradient(B, act_gamma, g0);
          for (int i = b.tid; i < k; i += b.nt) { pt[i] = act_theta[i]; pt[k + i] = act_gamma[i]; }
          b.sync();
          const double f0 = objective(B);
          double dec = 0.0;
          int rs = lbfgs_step(f0, &dec);
          if (rs < 0) { status = -rs; break; }
          if (rs == 1) break;
          lap(kTmRefine);
          record(kStRefine);
          lap(kTmObjective);
          int st = kOk;
          stats(bun[cur], act_theta, k);
          int removed = deactivate(&st);
          if (st != kOk) { status = st; break; }
          if (removed) {
            z_dirty = 1;
            lap(kTmDeactivate);
            status = ensure_cur();
            if (status != kOk) break;
            record(kStDeactivate);
            lap(kTmObjective);
            if (k == 0) break;
          }
          if (dec < (double)m * P.dec_tol_scale) break;
        }
        if (status != kOk) break;
      }
      lap(kTmRefine);
      if (o.iter_s && b.leader()) o.iter_s[it - 1] = (double)(now_ns() - t_iter) * 1e-9;  // estimator.py:247
      const double current = last_trace;
      if (fabs(previous - current) < (double)m * P.conv_tol_scale) {
        converged = 1;
        break;
      }
      previous = current;
    }
    finish(iterations, converged);
  }

  // beta EM value (tr + ||y - Psi(theta) mu||^2) / M  (estimator.py:86-88)
  SLSE_NIM double residual_value(double tr) {
    SLSE_PROF_C0(pc);
    const double rv_ = residual_value_body(tr);
    SLSE_PROF_CADD(13, pc);
    return rv_;
  }

  SLSE_NIM double residual_value_body(double tr) {
    const int tid_ = b.tid, nt_ = b.nt;
    double* mre = marg;  // scratch (length >= k)
    double* mim = dtmp;  // scratch (length n >= k), free outside build()
    double part = 0.0;
    for (int g = 0; g < G; ++g) {  // sum_g ||y_g - Psi mu_g||^2 (estimator.py:86-88)
      const cplx* mg = mu + (size_t)g * kmax;
      SLSE_CTRL_LOOP
      for (int i = tid_; i < k; i += nt_) { mre[i] = mg[i].re; mim[i] = mg[i].im; }
      b.sync();
#ifndef SLSE_HOST_EMU
      if (b.nt == 32 && n <= 512) steer_forward_warp(c, n, act_theta, mre, mim, k, 0.0, false, b.tid);
      else
#endif
        steer(c, act_theta, mre, mim, k, 0.0, false);
      const cplx* yg = y + (size_t)g * m;
#ifdef SLSE_SEMIFAST
      // y - Phi Psi mu over the observed samples (estimator.py:86-87, Observation.sample)
      SLSE_CTRL_LOOP
      for (int i = tid_; i < m; i += nt_) part += cabs2(csub(yg[i], cmul(sf_scale(obs, i), c[obs.idx[i]])));
#else
      SLSE_CTRL_LOOP
      for (int i = tid_; i < n; i += nt_) part += cabs2(csub(yg[i], c[i]));
#endif
      b.sync();
    }
    const double resid = b.sum(part);
    return (tr + (G == 1 ? resid : resid / (double)G)) / (double)m;
  }

  SLSE_NIM void finish(int iterations, int converged) {
    const int tid_ = b.tid, nt_ = b.nt;
    // posterior mean alpha = gamma * q (model_core.py:539-547)
    if (status == kOk && k) {
      int st = ensure_cur();
      if (st == kOk) {
        stats(bun[cur], act_theta, k);
        SLSE_CTRL_LOOP
        for (int i = tid_; i < k; i += nt_) {
          for (int g = 0; g < G; ++g)  // alpha_hat (G, k): gamma * q_g (model_core.py:539-547)
            o.alpha[(size_t)g * kmax + i] = cscale(bun[cur].q[(size_t)g * kmax + i], act_gamma[i]);
          o.theta[i] = act_theta[i];
          o.gamma[i] = act_gamma[i];
          o.slot[i] = act_slot[i];
        }
      } else {
        status = st;
      }
    }
    tm[kTmTotal] = (double)(now_ns() - t_start) * 1e-9;
#ifdef SLSE_SOLVER_PROF
    prof_acc[5] = clock64() - prof_run0;
    if (b.leader())
      for (int i = 0; i < 16; ++i) atomicAdd(&slse_prof_cycles[i], (unsigned long long)prof_acc[i]);
#endif
    if (converged) flags |= kFlConverged;
    if (b.leader()) {
      *o.khat = k;
      *o.status = status;
      *o.iters = iterations;
      *o.flags = flags;
      *o.beta = beta;
      *o.zeta = zeta;
      *o.ntrace = ntrace;
      *o.nevents = nevents;
      o.counters[0] = n_builds;
      o.counters[1] = n_grids;
      o.counters[2] = n_stats;
      o.counters[3] = n_backtracks;
      for (int i = 0; i < 6; ++i) o.stage_s[i] = tm[i];
    }
    b.sync();
  }
};

}  // namespace slse
