// slse_stats.cuh -- per-component statistics (q, r, u, s, t, v, x) at the
// active frequencies and the activation grid (q^G, s^G) with the fused
// activation-gain curve.
//
// Reference: model_core.py:281-313 (_SuperfastBundle.stats / grid),
// toeplitz.py:317-432 (omega diagonal sums), nufft.py:147-181 (adjoint and
// two-sided sums), smlr.py:62-70 (gain curve).
//
// Product form (no omega sums): with A_a(th) = sum_q q^a rho_q e^{-j2pi q th},
//   kind(th) = scale_kind / delta * sum_{(a,b)} cf^{kind}_{ab} A_a conj(A_b)
// where cf are the reference's cross-correlation-basis coefficients
// (toeplitz.py:317-365): R_ab(i) = sum_q q^a rho_q (q+i)^b conj(rho_{q+i})
// and sum_i R_ab(i) e^{j2pi i th} = A_a conj(A_b) exactly.
#pragma once
#include "slse_toeplitz.cuh"

namespace slse {

constexpr double kPi = 3.14159265358979323846;

// cf[kind][a][b], kind = s,t,v,x ; mirrors toeplitz.py:317-365.
struct CfTable {
  double cf[4][4][4];
};

SLSE_HD void cf_add(CfTable& T, int kind, int a, int b, double c) {
  // q^a i^b with i = m - q  ->  sum_j C(b,j) m^j (-q)^{b-j}
  const int binom[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 2, 1, 0}, {1, 3, 3, 1}};
  for (int j = 0; j <= b; ++j) {
    const double sgn = ((b - j) & 1) ? -1.0 : 1.0;
    T.cf[kind][a + b - j][j] += c * (double)binom[b][j] * sgn;
  }
}

SLSE_HD void cf_build(CfTable& T, int n_) {
  const double n = (double)n_;
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) T.cf[k][a][b] = 0.0;
  const double n3 = (double)((long long)n_ * n_ * n_);
  // s
  cf_add(T, 0, 0, 0, 2.0 - n);
  cf_add(T, 0, 0, 1, 1.0);
  cf_add(T, 0, 1, 0, 2.0);
  // t
  cf_add(T, 1, 1, 1, -1.0);
  cf_add(T, 1, 0, 1, n - 1.5);
  cf_add(T, 1, 0, 2, -0.5);
  cf_add(T, 1, 1, 0, n - 1.0);
  cf_add(T, 1, 0, 0, -(n - 1.0) * (n - 2.0) / 2.0);
  // v
  cf_add(T, 2, 3, 0, 2.0 / 3.0);
  cf_add(T, 2, 2, 1, 1.0);
  cf_add(T, 2, 1, 2, 1.0);
  cf_add(T, 2, 2, 0, 2.0 - n);
  cf_add(T, 2, 1, 1, 3.0 - 2.0 * n);
  cf_add(T, 2, 1, 0, n * n - 3.0 * n + 7.0 / 3.0);
  cf_add(T, 2, 0, 3, 1.0 / 3.0);
  cf_add(T, 2, 0, 2, 1.5 - n);
  cf_add(T, 2, 0, 1, n * n - 3.0 * n + 13.0 / 6.0);
  cf_add(T, 2, 0, 0, 1.5 * n * n - n3 / 3.0 - 13.0 * n / 6.0 + 1.0);
  // x
  cf_add(T, 3, 3, 0, 2.0 / 3.0);
  cf_add(T, 3, 2, 1, 1.0);
  cf_add(T, 3, 2, 0, 2.0 - n);
  cf_add(T, 3, 1, 1, 2.0 - n);
  cf_add(T, 3, 1, 0, n * n - 3.0 * n + 7.0 / 3.0);
  cf_add(T, 3, 0, 3, -1.0 / 6.0);
  cf_add(T, 3, 0, 1, (3.0 * n * n - 9.0 * n + 7.0) / 6.0);
  cf_add(T, 3, 0, 0, -n3 / 3.0 + 1.5 * n * n - 13.0 * n / 6.0 + 1.0);
}

// Statistics for K frequencies.  One warp per frequency; lanes stride the
// sample axis with a phasor recurrence re-anchored (exact sincospi) every
// 32 steps.  Outputs (length K): q, r, u, t, v complex; s, x real.
// `cf` must be visible to the whole block (shared memory or global).
SLSE_NI void component_stats(const double* SLSE_RESTRICT thetas, int K, const cplx* SLSE_RESTRICT rho,
                            const cplx* SLSE_RESTRICT w, int n, double delta_last, const CfTable* cf,
                            cplx* q, cplx* r, cplx* u, double* s, cplx* t, cplx* v, double* x,
                            Blk& b) {
  const int tid_ = b.tid, nt_ = b.nt;
  const double inv_d = 1.0 / delta_last;
  const double two_pi = 2.0 * kPi;
#ifdef SLSE_HOST_EMU
  const int lanes = 1, lane = 0, warp = 0, nwarp = 1;
#else
  const int lanes = 32, lane = tid_ & 31, warp = tid_ >> 5, nwarp = nt_ >> 5;
#endif
  // Two frequencies per warp pass: two independent phasor chains per lane
  // share the sample loads (the recurrence is the latency chain).  Every
  // frequency's sums are formed exactly as with one chain.
  const auto finish = [&](double* acc, int kk) {
#ifndef SLSE_HOST_EMU
    // Transposed warp reduction: 16 shuffles for the 14 sums (vs 70), sum v
    // ends in lanes 2v, 2v+1.
    acc[14] = acc[15] = 0.0;
    const double red = warp_tsum<16>(acc, lane);
    const auto from = [&](int v) { return __shfl_sync(0xffffffffu, red, 2 * v); };
    // Lanes 0..15 each form one product A_a conj(A_b) (a = lane/4, b = lane%4)
    // and its four cf-weighted terms; a second transposed reduction over the
    // 16 lanes leaves s, t, v, x in lanes 0, 2..4, 6..8, 10.
    const int pa = (lane >> 2) & 3, pb = lane & 3;
    const cplx Aa = mk(from(2 * pa), from(2 * pa + 1));
    const cplx Ab = mk(from(2 * pb), from(2 * pb + 1));
    const cplx P = cmulc(Aa, Ab);
    double term[8];
    const double* c = &cf->cf[0][pa][pb];
    const double c0 = lane < 16 ? c[0] : 0.0, c1 = lane < 16 ? c[16] : 0.0;
    const double c2 = lane < 16 ? c[32] : 0.0, c3 = lane < 16 ? c[48] : 0.0;
    term[0] = c0 * P.re;
    term[1] = c1 * P.re; term[2] = c1 * P.im;
    term[3] = c2 * P.re; term[4] = c2 * P.im;
    term[5] = c3 * P.re;
    term[6] = term[7] = 0.0;
    const double tot = warp_tsum<8>(term, lane);
    const double sc_tv = two_pi * inv_d, sc_vx = 4.0 * kPi * kPi * inv_d;
    double* qd = (double*)&q[kk];
    double* rd = (double*)&r[kk];
    double* ud = (double*)&u[kk];
    double* td = (double*)&t[kk];
    double* vd = (double*)&v[kk];
    switch (lane) {
      case 0: s[kk] = tot * inv_d; break;
      case 2: td[0] = tot * sc_tv; break;
      case 4: td[1] = tot * sc_tv; break;
      case 6: vd[0] = tot * sc_vx; break;
      case 8: vd[1] = tot * sc_vx; break;
      case 10: x[kk] = tot * sc_vx; break;
      case 16: qd[0] = red; break;
      case 18: qd[1] = red; break;
      case 20: rd[0] = red; break;
      case 22: rd[1] = red; break;
      case 24: ud[0] = red; break;
      case 26: ud[1] = red; break;
      default: break;
    }
#else
    if (lane == 0) {
      cplx A[4];
      for (int a = 0; a < 4; ++a) A[a] = mk(acc[2 * a], acc[2 * a + 1]);
      q[kk] = mk(acc[8], acc[9]);
      r[kk] = mk(acc[10], acc[11]);
      u[kk] = mk(acc[12], acc[13]);
      cplx sum[4];
      for (int kind = 0; kind < 4; ++kind) {
        cplx tot = mk(0.0, 0.0);
        for (int a = 0; a < 4; ++a)
          for (int bb = 0; bb < 4; ++bb) {
            const double c = cf->cf[kind][a][bb];
            if (c != 0.0) tot = cadd(tot, cscale(cmulc(A[a], A[bb]), c));
          }
        sum[kind] = tot;
      }
      const double sc_tv = two_pi * inv_d, sc_vx = 4.0 * kPi * kPi * inv_d;
      s[kk] = sum[0].re * inv_d;
      t[kk] = cscale(sum[1], sc_tv);
      v[kk] = cscale(sum[2], sc_vx);
      x[kk] = sum[3].re * sc_vx;
    }
#endif
  };
  for (int kk0 = warp; kk0 < K; kk0 += 2 * nwarp) {
    const int kk1 = kk0 + nwarp;
    const bool two = kk1 < K;  // warp-uniform
    const double th0 = thetas[kk0], th1 = two ? thetas[kk1] : th0;
    double acc0[16], acc1[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc0[i] = acc1[i] = 0.0;
    const cplx step0 = expj2pi((double)lanes, th0, -1.0), step1 = expj2pi((double)lanes, th1, -1.0);
    cplx e0 = mk(1.0, 0.0), e1 = e0;
    int since = 1 << 30;
    for (int m = lane; m < n; m += lanes) {
      if (since >= 32) {
        e0 = expj2pi((double)m, th0, -1.0);
        e1 = expj2pi((double)m, th1, -1.0);
        since = 0;
      }
      const double dm = (double)m;
      const cplx rm = rho[m], wm = w[m];
      const double m2 = dm * dm, m3 = m2 * dm;
      const double d1 = two_pi * dm;
      const double d2 = d1 * d1;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double* acc = c ? acc1 : acc0;
        const cplx e = c ? e1 : e0;
        const cplx p = cmul(rm, e);
        const cplx qq = cmul(wm, e);
        acc[0] += p.re;       acc[1] += p.im;
        acc[2] += dm * p.re;  acc[3] += dm * p.im;
        acc[4] += m2 * p.re;  acc[5] += m2 * p.im;
        acc[6] += m3 * p.re;  acc[7] += m3 * p.im;
        acc[8] += qq.re;       acc[9] += qq.im;
        acc[10] += d1 * qq.re; acc[11] += d1 * qq.im;
        acc[12] += d2 * qq.re; acc[13] += d2 * qq.im;
      }
      e0 = cmul(e0, step0);
      e1 = cmul(e1, step1);
      ++since;
    }
    finish(acc0, kk0);
    if (two) finish(acc1, kk1);
  }
  b.sync();
}

#ifndef SLSE_HOST_EMU
// One-warp form of component_stats (N <= 512 solver path): same sums and
// epilogue, rolled loops, one phasor recurrence per frequency.
static __device__ __noinline__ void component_stats_warp(const double* SLSE_RESTRICT thetas, int K,
                                                         const cplx* SLSE_RESTRICT rho, const cplx* SLSE_RESTRICT w,
                                                         int n, double delta_last, const CfTable* cf, cplx* q,
                                                         cplx* r, cplx* u, double* s, cplx* t, cplx* v, double* x,
                                                         int lane) {
  const double inv_d = 1.0 / delta_last;
  const double two_pi = 2.0 * kPi;
  const double sc_tv = two_pi * inv_d, sc_vx = 4.0 * kPi * kPi * inv_d;
  const int pa = (lane >> 2) & 3, pb = lane & 3;
  const double* cfp = &cf->cf[0][pa][pb];
  const double c0 = lane < 16 ? cfp[0] : 0.0, c1 = lane < 16 ? cfp[16] : 0.0;
  const double c2 = lane < 16 ? cfp[32] : 0.0, c3 = lane < 16 ? cfp[48] : 0.0;
#pragma unroll 1
  for (int kk = 0; kk < K; ++kk) {
    const double th = thetas[kk];
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    cplx e = expj2pi((double)lane, th, -1.0);
    const cplx step = expj2pi(32.0, th, -1.0);
#pragma unroll 1
    for (int m = lane; m < n; m += 32) {
      const double dm = (double)m;
      const cplx p = cmul(rho[m], e);
      const cplx qq = cmul(w[m], e);
      const double m2 = dm * dm, m3 = m2 * dm;
      acc[0] += p.re;       acc[1] += p.im;
      acc[2] += dm * p.re;  acc[3] += dm * p.im;
      acc[4] += m2 * p.re;  acc[5] += m2 * p.im;
      acc[6] += m3 * p.re;  acc[7] += m3 * p.im;
      const double d1 = two_pi * dm;
      const double d2 = d1 * d1;
      acc[8] += qq.re;       acc[9] += qq.im;
      acc[10] += d1 * qq.re; acc[11] += d1 * qq.im;
      acc[12] += d2 * qq.re; acc[13] += d2 * qq.im;
      e = cmul(e, step);
    }
    const double red = warp_tsum<16>(acc, lane);  // sum v in lanes 2v, 2v+1
    const double a_re = __shfl_sync(0xffffffffu, red, 4 * pa), a_im = __shfl_sync(0xffffffffu, red, 4 * pa + 2);
    const double b_re = __shfl_sync(0xffffffffu, red, 4 * pb), b_im = __shfl_sync(0xffffffffu, red, 4 * pb + 2);
    const cplx P = cmulc(mk(a_re, a_im), mk(b_re, b_im));
    double term[8];
    term[0] = c0 * P.re;
    term[1] = c1 * P.re; term[2] = c1 * P.im;
    term[3] = c2 * P.re; term[4] = c2 * P.im;
    term[5] = c3 * P.re;
    term[6] = term[7] = 0.0;
    const double tot = warp_tsum<8>(term, lane);
    // lane -> output: 0 s, 2/4 t, 6/8 v, 10 x (from tot); 16..26 q, r, u (from red)
    double* dst = nullptr;
    double val = 0.0;
    if (lane < 12 && !(lane & 1)) {
      const int o = lane >> 1;
      val = tot * (o == 0 ? inv_d : (o <= 2 ? sc_tv : sc_vx));
      dst = o == 0 ? &s[kk] : (o <= 2 ? (double*)&t[kk] + (o - 1) : (o <= 4 ? (double*)&v[kk] + (o - 3) : &x[kk]));
    } else if (lane >= 16 && lane < 28 && !(lane & 1)) {
      const int o = (lane - 16) >> 1;
      val = red;
      cplx* arr = o < 2 ? q : (o < 4 ? r : u);
      dst = (double*)&arr[kk] + (o & 1);
    }
    if (dst) *dst = val;
  }
  __syncwarp();
}
#endif

// Activation grid (model_core.py:303-313) in product form:
//   q^G = FFT_L(w),  s^G = delta^{-1} [(2-N)|A0|^2 + 2 Re(A1 conj A0)],
//   A0 = FFT_L(rho), A1 = FFT_L(n rho_n).
// Results land in G0 (q^G), and sg (s^G, real).  G1/G2 are scratch.
SLSE_NI void grid_eval(const cplx* SLSE_RESTRICT rho, const cplx* SLSE_RESTRICT w, int n, double delta_last,
                      int L, cplx* G0, cplx* G1, cplx* G2, double* sg, const FftCtx& f, Blk& b) {
  const int tid_ = b.tid, nt_ = b.nt;
  const cplx z = mk(0.0, 0.0);
  fft(G0, L, -1.0, [=](int i) { return i < n ? w[i] : z; }, [=](int i, cplx v) { G0[i] = v; }, f, b);
  fft(G1, L, -1.0, [=](int i) { return i < n ? rho[i] : z; }, [=](int i, cplx v) { G1[i] = v; }, f, b);
  fft(G2, L, -1.0, [=](int i) { return i < n ? cscale(rho[i], (double)i) : z; },
      [=](int i, cplx v) { G2[i] = v; }, f, b);
  const double c2n = 2.0 - (double)n;
  const double inv_d = 1.0 / delta_last;
  for (int l = tid_; l < L; l += nt_) {
    const cplx a0 = G1[l], a1 = G2[l];
    sg[l] = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
  }
  b.sync();
}

// Activation grid fused with the gain curve, exploiting the zero padding:
// with M = 2^ceil(log2 N) and R = L / M, grid point l = m R + r is
//   X[m R + r] = sum_{i<N} (x_i W_L^{i r}) W_M^{i m},
// so the three length-L transforms (w, rho, i rho) become R batches of three
// length-M transforms -- no work on the zero tail, each batch staged in
// shared memory (needs 3 M <= f.smem_cap) -- and every output is combined
// straight into s^G, |q^G|^2 and the gain curve (no L-sized complex
// buffers).  When 3 M does not fit the staging (large N) M is capped and the
// input folded: X[m R + r] = sum_{i<M} (sum_j x_{i+jM} W_L^{(i+jM) r}) W_M^{i m}.
// Residues r0, r0 + rstep, ... only (a CTA pair splits them).  Returns false
// when not even a 64-point batch fits (caller falls back to grid_eval).
SLSE_NI bool grid_gain_fused(const cplx* SLSE_RESTRICT rho, const cplx* SLSE_RESTRICT w, int n, double delta_last,
                             int L, double gb, double log_ratio, double* dl, double* q2, double* sg,
                             const FftCtx& f, Blk& b, int r0 = 0, int rstep = 1) {
  int M = 1 << ilog2(n);
  while (M > 64 && 3 * M > f.smem_cap) M >>= 1;
  if (3 * M > f.smem_cap || M > L) return false;
  const int tid = b.tid, nt = b.nt;
  const int R = L / M;
  const int lgL = ilog2(L), p = ilog2(M);
  const double c2n = 2.0 - (double)n;
  const double inv_d = 1.0 / delta_last;
  cplx* x = f.smem;
#ifndef SLSE_HOST_EMU
  // shared staging in the swizzled layout (fswz): the bit-reversed scatter
  // is otherwise a 32-way bank conflict, and the first radix-4 passes 2-way
  __builtin_assume(__isShared(x));
  const auto gz = [p](int i) { return fswz(i, p); };
#else
  const auto gz = [](int i) { return i; };
#endif
  for (int r = r0; r < R; r += rstep) {
    for (int t = tid; t < 3 * M; t += nt) {
      const int c = t >> p, i0 = t & (M - 1);
      cplx v = mk(0.0, 0.0);
      for (int i = i0; i < n; i += M) {  // one term unless the input is folded
        const cplx tw = twid_tab(f.tw, f.twlog, (int)(((long long)i * r) & (L - 1)), lgL, -1.0);
        const cplx src = c == 0 ? w[i] : (c == 1 ? rho[i] : cscale(rho[i], (double)i));
        v = cadd(v, r ? cmul(src, tw) : src);
      }
      x[(size_t)c * M + gz(brev_bits((unsigned)i0, p))] = v;
    }
    fft_barrier();
#ifndef SLSE_HOST_EMU
    fft_passes_multi_swz(x, 3, M, -1.0, f.tw, f.twlog, tid, nt);
#else
    fft_passes_multi(x, 3, M, -1.0, f.tw, f.twlog, tid, nt);
#endif
    for (int m = tid; m < M; m += nt) {
      const int l = m * R + r;
      const int ms = gz(m);
      const cplx q = x[ms], a0 = x[M + ms], a1 = x[2 * M + ms];
      const double s = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
      const double qq = cabs2(q);
      sg[l] = s;
      q2[l] = qq;
      dl[l] = (log1p(gb * s) + log_ratio) - qq / (1.0 / gb + s);
    }
    fft_barrier();
  }
  return true;
}

// Activation gain (smlr.py:62-70, G = 1):
//   Delta = log1p(gb s) + log((1-ze)/ze) - |q|^2 / (1/gb + s)
SLSE_D double gain(double q2, double s, double gb, double log_ratio) {
  return (log1p(gb * s) + log_ratio) - q2 / (1.0 / gb + s);
}

// G snapshots: q2 = sum_g |q^G_g|^2 and the log1p term carries G (smlr.py:66-69)
SLSE_D double gain_g(double q2, double s, double gb, double log_ratio, int G) {
  const double lg = log1p(gb * s);
  return ((G == 1 ? lg : (double)G * lg) + log_ratio) - q2 / (1.0 / gb + s);
}

}  // namespace slse
