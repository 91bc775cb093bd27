// TEST-ONLY host emulation of the per-problem device program.
//
// Compiles the product's device headers (paper_1705_06073_b200/csrc/*.cuh)
// with g++ -DSLSE_HOST_EMU, where a "block" is one serial thread.  It lets
// the CPU test suite exercise the estimator state machine (sweeps,
// activations, L-BFGS, deactivation, trace/event recording) against the
// oracle without a GPU.  It is never loaded by the package: the product path
// is the nvcc-built libsuperlse_b200.so and fails loudly without it.
#define SLSE_HOST_EMU 1
#include <cmath>
#include <cstdlib>
#include <vector>

#include "slse_solver.cuh"
#include "slse_dnc.cuh"

using namespace slse;

// level-major layout, as the device table (slse_fft.cuh tw_index)
static std::vector<cplx> make_twiddles(int lg) {
  std::vector<cplx> tw(tw_entries(lg), mk(1.0, 0.0));
  for (int l = 0; l <= lg; ++l)
    for (int k = 0; k < (1 << l); ++k) {
      double s, c;
      sincos2pi((double)k / (double)(1 << l), &s, &c);
      tw[tw_index(k, l)] = mk(c, -s);
    }
  return tw;
}

extern "C" int emu_estimate_batch(const double* y, int N, int B, const slse_options* opts, const slse_outputs* out) {
  SolveParams P = make_params(N, *opts);  // P.dnc from opts->decomp_method
  const int fmax = P.L > 2 * N ? P.L : 2 * N;
  std::vector<cplx> tw = make_twiddles(ilog2(fmax));
  CfTable cf;
  cf_build(cf, N);
  Layout lay = make_layout(N, P.L, P.kmax, P.lbfgs_mem, false, P.dnc != 0);
  std::vector<char> slab(lay.total + 256);
  char* base = (char*)(((uintptr_t)slab.data() + 255) & ~(uintptr_t)255);
  std::vector<double> red(2 * 32 * 16);
  std::vector<cplx> region(fmax);
  FftCtx f{tw.data(), ilog2(fmax), region.data(), fmax};
  const size_t K = (size_t)P.kmax;
  for (int p = 0; p < B; ++p) {
    Blk b{0, 1, red.data(), 0};
    ProbOut o;
    o.khat = out->k_hat + p;
    o.status = out->status + p;
    o.iters = out->iterations + p;
    o.flags = out->flags + p;
    o.beta = out->beta + p;
    o.zeta = out->zeta + p;
    o.theta = out->theta + p * K;
    o.gamma = out->gamma + p * K;
    o.alpha = (cplx*)out->alpha + p * K;
    o.slot = out->slot + p * K;
    o.trace = out->trace + (size_t)p * P.tcap;
    o.stage = out->stage + (size_t)p * P.tcap;
    o.trace_k = out->trace_k + (size_t)p * P.tcap;
    o.ntrace = out->n_trace + p;
    o.events = out->events + (size_t)p * P.ecap * 3;
    o.nevents = out->n_events + p;
    o.counters = (long long*)out->counters + (size_t)p * 4;
    o.stage_s = out->stage_seconds + (size_t)p * 6;
    o.iter_s = out->iter_seconds ? out->iter_seconds + (size_t)p * P.max_outer : nullptr;
    Solver S(b, P, &cf, (const cplx*)y + (size_t)p * N, o, base, lay, nullptr, f);
    S.run();
  }
  return 0;
}

// per-call operators on host arrays (one problem)
extern "C" int emu_bundle(const double* y, int N, const double* th, const double* ga, int k, double beta, int L,
                          double* c, double* rho, double* w, double* scal /* logdet, delta_last, data_term */,
                          double* qg, double* sg, double* st /* q r u t v (complex k each), s x (k each) */) {
  const int fmax = L > 2 * N ? L : 2 * N;
  std::vector<cplx> tw = make_twiddles(ilog2(fmax));
  std::vector<cplx> region(fmax);
  FftCtx f{tw.data(), ilog2(fmax), region.data(), fmax};
  std::vector<double> red(2 * 32 * 16);
  Blk b{0, 1, red.data(), 0};
  std::vector<cplx> e(N), bg(N), a(N), yh(2 * N), P(2 * N), U(2 * N), V(2 * N), G1(L), G2(L);
  std::vector<double> dt(N);
  steer_forward((cplx*)c, N, th, ga, nullptr, k, beta, true, b);
  Factor F = toeplitz_factor((const cplx*)c, N, e.data(), bg.data(), a.data(), nullptr, dt.data(), (cplx*)rho, b);
  if (F.status) return F.status;
  const cplx* yy = (const cplx*)y;
  fft(yh.data(), 2 * N, -1.0, [&](int i) { return i < N ? yy[i] : mk(0, 0); }, [&](int i, cplx v) { yh[i] = v; }, f, b);
  double quad = gs_apply((const cplx*)rho, N, F.delta_last, yy, yh.data(), P.data(), U.data(), V.data(), (cplx*)w, f, b);
  scal[0] = F.logdet;
  scal[1] = F.delta_last;
  scal[2] = F.logdet + quad;
  grid_eval((const cplx*)rho, (const cplx*)w, N, F.delta_last, L, (cplx*)qg, G1.data(), G2.data(), sg, f, b);
  if (k) {
    CfTable cf;
    cf_build(cf, N);
    cplx* q = (cplx*)st;
    cplx* r = q + k;
    cplx* u = r + k;
    cplx* t = u + k;
    cplx* v = t + k;
    double* s = (double*)(v + k);
    double* x = s + k;
    component_stats(th, k, (const cplx*)rho, (const cplx*)w, N, F.delta_last, &cf, q, r, u, s, t, v, x, b);
  }
  return 0;
}

// Stockham register FFT (count buffers of n, in place)
extern "C" int emu_fft_stockham(double* x, int count, int n, int sign) {
  const int lg = ilog2(n) > 4 ? ilog2(n) : 4;
  std::vector<cplx> tw = make_twiddles(lg);
  std::vector<double> red(64);
  Blk b{0, 1, red.data(), 0};
  FftCtx f{tw.data(), lg, nullptr, 0};
  std::vector<cplx> sx((size_t)count * sk_len(n));
  cplx* xx = (cplx*)x;
  for (int c = 0; c < count; ++c)
    for (int i = 0; i < n; ++i) sx[(size_t)c * sk_len(n) + sk(i)] = xx[(size_t)c * n + i];
  fft_stockham(sx.data(), count, n, (double)sign, f, b);
  for (int c = 0; c < count; ++c)
    for (int i = 0; i < n; ++i) xx[(size_t)c * n + i] = sx[(size_t)c * sk_len(n) + sk(i)];
  return 0;
}

// radix-4 DIT reference path
extern "C" int emu_fft_dit(double* x, int n, int sign) {
  const int lg = ilog2(n) > 4 ? ilog2(n) : 4;
  std::vector<cplx> tw = make_twiddles(lg);
  std::vector<double> red(64);
  std::vector<cplx> sm(n);
  Blk b{0, 1, red.data(), 0};
  FftCtx f{tw.data(), lg, sm.data(), n};
  fft_inplace((cplx*)x, n, (double)sign, f, b);
  return 0;
}

// grid kernel pipeline (load head, pruned Stockham over 3 buffers, combine)
template <int LG, int Q>
static void grid_pruned_t(const cplx* w, const cplx* rho, int n, double dl, cplx* qg, double* sg) {
  constexpr int L = 1 << LG;
  const int LS = sk_len(L);
  std::vector<cplx> tw = make_twiddles(LG);
  std::vector<cplx> X(3 * LS, mk(0, 0));
  for (int i = 0; i < (L >> Q); ++i) {
    cplx a = mk(0, 0), r = mk(0, 0);
    if (i < n) { a = w[i]; r = rho[i]; }
    X[sk(i)] = a; X[LS + sk(i)] = r; X[2 * LS + sk(i)] = cscale(r, (double)i);
  }
  fft_fixed_pruned<LG, Q>(X.data(), 3, -1.0, tw.data(), LG, 0, 1);
  for (int l = 0; l < L; ++l) {
    const cplx a0 = X[LS + sk(l)], a1 = X[2 * LS + sk(l)];
    qg[l] = X[sk(l)];
    sg[l] = ((2.0 - n) * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) / dl;
  }
}

extern "C" int emu_grid_pruned(const double* w, const double* rho, int n, double dl, int L, double* qg, double* sg) {
  int q = 0;
  while (q < 3 && (n << (q + 1)) <= L) ++q;
  const cplx* W = (const cplx*)w;
  const cplx* R = (const cplx*)rho;
#define C(LGV) \
  if (L == (1 << LGV)) { \
    if (q == 0) grid_pruned_t<LGV, 0>(W, R, n, dl, (cplx*)qg, sg); \
    if (q == 1) grid_pruned_t<LGV, 1>(W, R, n, dl, (cplx*)qg, sg); \
    if (q == 2) grid_pruned_t<LGV, 2>(W, R, n, dl, (cplx*)qg, sg); \
    if (q == 3) grid_pruned_t<LGV, 3>(W, R, n, dl, (cplx*)qg, sg); \
    return q; }
  C(6) C(7) C(8) C(9) C(10) C(11) C(12)
#undef C
  return -1;
}

#include "slse_dnc.cuh"
// superfast D&C factorisation
extern "C" int emu_factor_dnc(const double* c, int n, double* rho, double* delta, double* logdet) {
  const int F = 1 << ilog2(2 * n);
  std::vector<cplx> tw = make_twiddles(ilog2(F) > 4 ? ilog2(F) : 4);
  std::vector<cplx> region(sk_len(F));
  std::vector<double> red(64);
  Blk b{0, 1, red.data(), 0};
  FftCtx f{tw.data(), ilog2(F) > 4 ? ilog2(F) : 4, region.data(), (int)region.size()};
  std::vector<cplx> T(4 * (size_t)n + 4), arena(dnc_arena_elems(n - 1) + 16);
  std::vector<double> dt(n);
  Factor Fa = toeplitz_factor_dnc((const cplx*)c, n, T.data(), arena.data(), delta, dt.data(), (cplx*)rho, f, b);
  *logdet = Fa.logdet;
  return Fa.status;
}

// batched transform through fft_multi with a small staging cap (exercises the four-step path)
extern "C" int emu_fft_multi(double* x, int count, int n, int sign, int cap) {
  const int lg = ilog2(n) > 4 ? ilog2(n) : 4;
  std::vector<cplx> tw = make_twiddles(lg);
  std::vector<double> red(64);
  std::vector<cplx> sm(cap > 0 ? cap : 1), work((size_t)count * n), out((size_t)count * n);
  Blk b{0, 1, red.data(), 0};
  FftCtx f{tw.data(), lg, sm.data(), cap};
  cplx* xx = (cplx*)x;
  fft_multi(work.data(), count, n, (double)sign, [=](int c, int i) { return xx[(size_t)c * n + i]; },
            [&](int c, int i, cplx v) { out[(size_t)c * n + i] = v; }, f, b);
  for (size_t i = 0; i < out.size(); ++i) xx[i] = out[i];
  return 0;
}
