// slse_dnc.cuh -- superfast (divide-and-conquer, FFT-doubling) generalized
// Schur factorisation of a Hermitian PD Toeplitz matrix.
//
// Reference: toeplitz.generalized_schur / _schur_split / _schur_base /
// _theta_matmul (pkg/src/superlse/toeplitz.py:148-260), O(N log^2 N).
//
// Formulation (own; unnormalised steps).  With generator polynomials
// e(z) = sum e_j z^j, b(z) = sum b_j z^j (e = b = c initially) one Schur
// step with reflection coefficient k = -e_{m+1} / delta_m is
//     [e; b] <- M_k [e; b],   M_k = [[1, k z], [conj(k), z]],
// delta_{m+1} = delta_m (1 - |k|^2), and the Levinson predictor pair
// (a, conj-reversed a) obeys the same recursion from [1; 1], so after all
// N-1 steps  a = Theta_11 + Theta_12  for Theta = M_{N-2} ... M_0.
//
// split(E, Bw, s): transfer matrix Theta of s steps from the generator
// window E[j] = e_{m0+j} (j <= s), Bw[j] = b_{m0+j} (j < s):
//   s <= 32 : leaf -- one warp runs the classical recursion in registers
//             (shuffles, no block barriers) and accumulates Theta;
//   else    : Theta1 = split(left half h = s/2); the right half's window is
//             the middle product [h, s] of Theta1 with (E, Bw); Theta2 =
//             split(right half); Theta = Theta2 Theta1.  Every product is
//             a cyclic convolution of length F = 2^ceil(log2(s+1)), done
//             with the block FFT (shared-memory staged when it fits).
#pragma once
#include "slse_split.cuh"
#include "slse_toeplitz.cuh"

namespace slse {

constexpr int kDncLeaf = 32;
#ifndef SLSE_DNC_LEAF2
#define SLSE_DNC_LEAF2 1  // block leaves take two Schur steps per barrier (dnc_leaf_block2)
#endif
#ifndef SLSE_DNC_BLOCK_LEAF
#define SLSE_DNC_BLOCK_LEAF 256  // CTA-wide leaves up to this many steps (0 / 32: one-warp leaves only)
#endif
// nodes up to this many steps multiply their polynomials directly (one
// output coefficient per thread, two barriers per node) instead of through
// batched FFTs, whose fixed barrier cost dominates at small sizes
#ifndef SLSE_DNC_DIRECT
#define SLSE_DNC_DIRECT 256
#endif

struct DncCtx {
  FftCtx f;
  cplx* arena;        // global scratch (bump allocated along the recursion)
  double* delta_tmp;  // pivots delta_0..delta_{N-1}
  double floor_;      // PD floor = PD_EPS * c0
  double d;           // current pivot (identical in every thread)
  int step;           // steps done
  int status;
  int direct_max;     // nodes with s <= direct_max use direct products
  int leaf_max;       // subtrees with s <= leaf_max run as one leaf (dnc_leaf_block above 32)
  long long* prof;    // optional: clock64 per phase (leaf, direct1, direct2, fft1, fft2, total)
  Split* sp;          // CTA pair (slse_split.cuh): node transforms shared with the helper CTA, or null
};

// Node transforms of one FFT node site, transforms [qlo, qhi) of the site's
// batch (dnc_split below; the helper CTA of a pair runs the other half).
// site 0: forward T11, T12, E, Bw -> S[0..1], SE, SB      (phase 1)
// site 1: inverse of the E2 / B2 window products           (phase 1)
// site 2: forward rows of T2 -> A                           (phase 2)
// site 3: inverse of row 1 of T2 T1 -> T                    (phase 2)
struct DncFftArgs {
  int site, F, h, s, l1, l2, ld;
  double invF;
  const cplx *T1, *E, *Bw, *T2;
  cplx *S, *SE, *SB, *E2, *B2, *A, *T, *work;
};
SLSE_HD constexpr int dnc_fft_count(int site) { return site == 0 ? 4 : 2; }
// transforms of at least this size are shared by the two CTAs of a pair
constexpr int kDncSplitMinF = 1024;

SLSE_D void dnc_fft_site(const DncFftArgs& a, int qlo, int qhi, const FftCtx& f, Blk& b) {
  const int F = a.F, h = a.h, s = a.s, l1 = a.l1, l2 = a.l2, ld = a.ld;
  const double invF = a.invF;
  const int cnt = qhi - qlo;
  if (cnt <= 0) return;
  cplx* work = a.work + (size_t)qlo * F;
  if (a.site == 0) {
    const cplx *T1 = a.T1, *E = a.E, *Bw = a.Bw;
    cplx *S = a.S, *SEw = a.SE;
    fft_multi(work, cnt, F, -1.0,
              [=](int q, int i) {
                q += qlo;
                if (q < 2) return i < l1 ? T1[q * l1 + i] : mk(0.0, 0.0);
                if (q == 2) return i <= s ? E[i] : mk(0.0, 0.0);
                return i < s ? Bw[i] : mk(0.0, 0.0);
              },
              [=](int q, int i, cplx v) {
                q += qlo;
                (q < 2 ? S + (size_t)q * F : SEw + (size_t)(q - 2) * F)[i] = v;
              },
              f, b);
  } else if (a.site == 1) {
    const cplx *S = a.S, *SE = a.SE, *SB = a.SB;
    cplx *E2 = a.E2, *B2 = a.B2;
    fft_multi(work, cnt, F, 1.0,
              [=](int q, int k) {
                q += qlo;
                return q == 0 ? cadd(cmul(S[k], SE[k]), cmul(S[F + k], SB[k]))
                              : cadd(cmul(S[2 * F + k], SE[k]), cmul(S[3 * F + k], SB[k]));
              },
              [=](int q, int i, cplx v) {
                q += qlo;
                if (q == 0) {
                  if (i >= h && i <= s) E2[i - h] = cscale(v, invF);
                } else if (i >= h && i < s) {
                  B2[i - h] = cscale(v, invF);
                }
              },
              f, b);
  } else if (a.site == 2) {
    const cplx* T2 = a.T2;
    cplx* A = a.A;
    fft_multi(work, cnt, F, -1.0, [=](int q, int i) { q += qlo; return i < l2 ? T2[q * l2 + i] : mk(0.0, 0.0); },
              [=](int q, int i, cplx v) { q += qlo; A[(size_t)q * F + i] = v; }, f, b);
  } else {
    const cplx *A = a.A, *S = a.S;
    cplx* T = a.T;
    // T_rc = A_r1 S_1c + A_r2 S_2c ; output q = 2 r + c
    fft_multi(work, cnt, F, 1.0,
              [=](int q, int k) {
                q += qlo;
                const int r = q >> 1, c = q & 1;
                return cadd(cmul(A[(size_t)(2 * r) * F + k], S[(size_t)c * F + k]),
                            cmul(A[(size_t)(2 * r + 1) * F + k], S[(size_t)(2 + c) * F + k]));
              },
              [=](int q, int i, cplx v) { q += qlo; if (i < ld) T[q * ld + i] = cscale(v, invF); }, f, b);
  }
}

// All transforms of a site: shared with the helper CTA when the pair is
// active and the transforms are large enough, else on this CTA alone.
SLSE_D void dnc_fft_run(DncCtx& X, const DncFftArgs& a, Blk& b) {
  const int cnt = dnc_fft_count(a.site);
  if (SLSE_PAIR && X.sp && a.F >= kDncSplitMinF) {
    SplitJob j;
    j.set(kJobDncFft, a);
    X.sp->post(j, b);
    dnc_fft_site(a, 0, cnt / 2, X.f, b);
    X.sp->done();
  } else {
    dnc_fft_site(a, 0, cnt, X.f, b);
  }
}

SLSE_D long long dnc_clock() {
#ifdef SLSE_HOST_EMU
  return 0;
#else
  return clock64();
#endif
}

#ifndef SLSE_HOST_EMU
SLSE_D cplx shfl_c(cplx v, int src) {
  return mk(__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src));
}
SLSE_D cplx shfl_down_c(cplx v, int d) {
  return mk(__shfl_down_sync(0xffffffffu, v.re, d), __shfl_down_sync(0xffffffffu, v.im, d));
}
SLSE_D cplx shfl_up_c(cplx v, int d) {
  return mk(__shfl_up_sync(0xffffffffu, v.re, d), __shfl_up_sync(0xffffffffu, v.im, d));
}
#endif

// Leaf: s <= 32 steps.  E1[j] = e_{m0+1+j}, Bw[j] = b_{m0+j} (j < s).
// Writes Theta (4 polys of s+1 coefficients, row-major T11 T12 T21 T22 at
// stride s+1), pivots, and updates X.d / X.step / X.status (uniform).
SLSE_NI void dnc_leaf(DncCtx& X, const cplx* E1, const cplx* Bw, int s, cplx* T, Blk& b) {
  const int ld = s + 1;
#ifdef SLSE_HOST_EMU
  std::vector<cplx> e(E1, E1 + s), bb(Bw, Bw + s);
  std::vector<cplx> t11(ld + 1, mk(0, 0)), t12(ld + 1, mk(0, 0)), t21(ld + 1, mk(0, 0)), t22(ld + 1, mk(0, 0));
  t11[0] = mk(1, 0);
  t22[0] = mk(1, 0);
  double d = X.d;
  int st = 0;
  for (int t = 0; t < s; ++t) {
    const double inv = 1.0 / d;
    const cplx k = mk(-e[t].re * inv, -e[t].im * inv), kc = conjg(k);
    for (int j = 0; j < s - t; ++j) {
      const cplx ej = e[t + j], bj = bb[j];
      e[t + j] = cadd(ej, cmul(k, bj));
      bb[j] = cadd(bj, cmul(kc, ej));
    }
    for (int i = t + 1; i >= 0; --i) {  // degree grows by one per step
      const cplx a11 = t11[i], a12 = t12[i];
      const cplx p21 = i ? t21[i - 1] : mk(0, 0), p22 = i ? t22[i - 1] : mk(0, 0);
      t11[i] = cadd(a11, cmul(k, p21));
      t12[i] = cadd(a12, cmul(k, p22));
      t21[i] = cadd(cmul(kc, a11), p21);
      t22[i] = cadd(cmul(kc, a12), p22);
    }
    d = d * (1.0 - (k.re * k.re + k.im * k.im));
    X.delta_tmp[X.step + t + 1] = d;
    if (!(d > X.floor_)) { st = kNotPD; break; }
  }
  for (int i = 0; i < ld; ++i) {
    T[i] = t11[i];
    T[ld + i] = t12[i];
    T[2 * ld + i] = t21[i];
    T[3 * ld + i] = t22[i];
  }
  X.d = d;
  X.step += s;
  if (st) X.status = st;
  (void)b;
#else
  __shared__ double s_out[2];
  if (b.tid < 32) {
    const int lane = b.tid;
    // generator pairs in the shifted frame: lane j holds (e_{m0+t+1+j}, b_{m0+t+j})
    cplx ej = lane < s ? E1[lane] : mk(0.0, 0.0);
    cplx bj = lane < s ? Bw[lane] : mk(0.0, 0.0);
    // Theta coefficients i = lane (and i = 32 kept redundantly in x*)
    cplx t11 = mk(lane == 0 ? 1.0 : 0.0, 0.0), t12 = mk(0.0, 0.0), t21 = mk(0.0, 0.0);
    cplx t22 = mk(lane == 0 ? 1.0 : 0.0, 0.0);
    cplx x11 = mk(0.0, 0.0), x12 = mk(0.0, 0.0), x21 = mk(0.0, 0.0), x22 = mk(0.0, 0.0);
    double d = X.d;
    double* dtmp = X.delta_tmp + X.step;
    const double floor_ = X.floor_;
    int st = 0;
    cplx k;
    {
      const cplx e0 = shfl_c(ej, 0);
      const double inv = 1.0 / d;
      k = mk(-e0.re * inv, -e0.im * inv);
    }
    for (int t = 0; t < s; ++t) {
      // next coefficient straight from lane 1's pre-update pair: off the
      // shift/broadcast path, so one step costs ~ a reciprocal, not shuffles
      const cplx ej1 = shfl_c(ej, 1), bj1 = shfl_c(bj, 1);
      const cplx kc = conjg(k);
      const double dn = d * (1.0 - (k.re * k.re + k.im * k.im));
      const double invn = rcp_pos(dn);
      const cplx enext = cadd(ej1, cmul(k, bj1));
      const cplx knext = mk(-enext.re * invn, -enext.im * invn);
      const cplx en = cadd(ej, cmul(k, bj));
      const cplx bn = cadd(bj, cmul(kc, ej));
      ej = shfl_down_c(en, 1);
      bj = bn;
      // Theta <- M_k Theta : T1x[i] += k T2x[i-1] ; T2x[i] = conj(k) T1x[i] + T2x[i-1]
      if (t == 31) {  // coefficient 32 (x*) is zero until the 32nd step: only then does 31 feed it
        const cplx l21 = shfl_c(t21, 31), l22 = shfl_c(t22, 31);
        const cplx m11 = cadd(x11, cmul(k, l21)), m12 = cadd(x12, cmul(k, l22));
        const cplx m21 = cadd(cmul(kc, x11), l21), m22 = cadd(cmul(kc, x12), l22);
        x11 = m11; x12 = m12; x21 = m21; x22 = m22;
      }
      const cplx p21 = shfl_up_c(t21, 1), p22 = shfl_up_c(t22, 1);
      const cplx q21 = lane ? p21 : mk(0.0, 0.0), q22 = lane ? p22 : mk(0.0, 0.0);
      const cplx n11 = cadd(t11, cmul(k, q21)), n12 = cadd(t12, cmul(k, q22));
      const cplx n21 = cadd(cmul(kc, t11), q21), n22 = cadd(cmul(kc, t12), q22);
      t11 = n11; t12 = n12; t21 = n21; t22 = n22;
      d = dn;
      if (lane == 0) dtmp[t + 1] = d;
      if (!(d > floor_)) { st = kNotPD; break; }
      k = knext;
    }
    if (lane < ld) {
      T[lane] = t11;
      T[ld + lane] = t12;
      T[2 * ld + lane] = t21;
      T[3 * ld + lane] = t22;
    }
    if (lane == 31 && ld > 32) {
      T[32] = x11;
      T[ld + 32] = x12;
      T[2 * ld + 32] = x21;
      T[3 * ld + 32] = x22;
    }
    if (lane == 0) {
      s_out[0] = d;
      s_out[1] = (double)st;
    }
  }
  b.sync();
  X.d = s_out[0];
  X.step += s;
  if (s_out[1] != 0.0) X.status = (int)s_out[1];
  b.sync();
#endif
}

// Block leaf: s <= nt - 2 steps with the whole CTA, one barrier per step.
// The same recursion as dnc_leaf, laid out in the shared staging region:
// thread j < s - t updates the generator pair (e_{t+j}, b_j) in place and
// thread 1 forms the next reflection coefficient from its fresh e_{t+1};
// thread nt-1-i updates Theta coefficient i <= t + 1 (Theta_11 / Theta_12
// in place, Theta_21 / Theta_22 ping-pong because coefficient i reads
// i - 1).  Replaces the 32-step one-warp leaves and the small product nodes
// above them, whose per-node latency (barriers, global round trips)
// dominated the superfast factorisation.
SLSE_NI void dnc_leaf_block(DncCtx& X, const cplx* E1, const cplx* Bw, int s, cplx* T, Blk& b) {
#ifdef SLSE_HOST_EMU
  dnc_leaf(X, E1, Bw, s, T, b);
#else
  const int tid = b.tid, nt = b.nt;
  const int ld = s + 1, lp = s + 2;  // Theta_2x ping-pong rows: offset i + 1 holds coefficient i
  __builtin_assume(__isShared(X.f.smem));  // shared-memory instructions, not generic LD / ST
  cplx* e = X.f.smem;                 // s
  cplx* bb = e + s;                   // s
  cplx* t1 = bb + s;                  // Theta_11 | Theta_12 : 2 ld
  cplx* t2 = t1 + 2 * ld;             // [2][Theta_21 | Theta_22] : 4 lp
  cplx* kb = t2 + 4 * lp;             // [2] reflection coefficients (double-buffered)
  const cplx z = mk(0.0, 0.0);
  for (int i = tid; i < s; i += nt) {
    e[i] = E1[i];
    bb[i] = Bw[i];
  }
  for (int i = tid; i < 2 * ld; i += nt) t1[i] = (i == 0) ? mk(1.0, 0.0) : z;
  for (int i = tid; i < 4 * lp; i += nt) t2[i] = (i == lp + 1) ? mk(1.0, 0.0) : z;  // buffer 0: Theta_22[0] = 1
  b.sync();
  double d = X.d;
  double* dtmp = X.delta_tmp + X.step;
  const double floor_ = X.floor_;
  if (tid == 0) {
    const double inv = 1.0 / d;
    kb[0] = mk(-e[0].re * inv, -e[0].im * inv);
  }
  b.sync();
  int st = 0;
  const int ci = nt - 1 - tid;  // Theta coefficient of this thread
  for (int t = 0; t < s; ++t) {
    const cplx k = kb[t & 1], kc = conjg(k);
    const double dn = d * (1.0 - (k.re * k.re + k.im * k.im));
    if (tid < s - t) {
      const cplx ej = e[t + tid], bj = bb[tid];
      const cplx en = cadd(ej, cmul(k, bj));
      e[t + tid] = en;
      bb[tid] = cadd(bj, cmul(kc, ej));
      if (tid == 1) {
        const double invn = rcp_pos(dn);
        kb[(t + 1) & 1] = mk(-en.re * invn, -en.im * invn);
      }
    }
    if (ci <= t + 1) {
      const cplx* r2 = t2 + (t & 1) * 2 * lp;
      cplx* w2 = t2 + ((t + 1) & 1) * 2 * lp;
      const cplx a11 = t1[ci], a12 = t1[ld + ci];
      const cplx p21 = r2[ci], p22 = r2[lp + ci];  // coefficient ci - 1 (zero slot for ci = 0)
      t1[ci] = cadd(a11, cmul(k, p21));
      t1[ld + ci] = cadd(a12, cmul(k, p22));
      w2[ci + 1] = cadd(cmul(kc, a11), p21);
      w2[lp + ci + 1] = cadd(cmul(kc, a12), p22);
    }
    d = dn;
    if (tid == 0) dtmp[t + 1] = d;
    if (!(d > floor_)) {  // uniform: every thread holds the same d
      st = kNotPD;
      break;
    }
    b.sync();
  }
  b.sync();
  if (!st) {
    const cplx* r2 = t2 + (s & 1) * 2 * lp;
    for (int i = tid; i < ld; i += nt) {
      T[i] = t1[i];
      T[ld + i] = t1[ld + i];
      T[2 * ld + i] = r2[i + 1];
      T[3 * ld + i] = r2[lp + i + 1];
    }
  }
  b.sync();
  X.d = d;
  X.step += s;
  if (st) X.status = st;
#endif
}

// c + a * b.  SLSE_LEAF_CFMA = 1: four fused multiply-adds (two levels deep)
// instead of multiply, fused multiply-add and add (three levels, six
// instructions); 0 keeps the arithmetic of dnc_leaf / dnc_leaf_block bit for bit.
#ifndef SLSE_LEAF_CFMA
#define SLSE_LEAF_CFMA 1
#endif
SLSE_D cplx lf_fma(cplx a, cplx b, cplx c) {
#if SLSE_LEAF_CFMA
  return mk(fma(-a.im, b.im, fma(a.re, b.re, c.re)), fma(a.im, b.re, fma(a.re, b.im, c.im)));
#else
  return cadd(c, cmul(a, b));
#endif
}
template <class P>
SLSE_D void lf_swap(P& a, P& b) {
  const P t = a;
  a = b;
  b = t;
}

// Block leaf, two Schur steps per barrier.  The same recursion as
// dnc_leaf_block (identical arithmetic), but each item also computes the
// step-t value of its right-hand neighbour (generator slot j + 1, or Theta
// coefficient i - 1 of row 2) from the pre-pair state, so it can apply step
// t + 1 without waiting for that neighbour.  All state is ping-ponged
// between two buffers per pair.  The next pair's coefficients k_{t+2},
// k_{t+3} (slots 1..3 of the pre-pair state, two reciprocals: the longest
// dependent chain of the pair) are formed by a dedicated "chain warp" before
// its own items, not by item 1 after its update: as item 1's divergent tail
// the chain ran after warp 0's generator work and every other warp waited
// at the barrier for it.  Needs s <= nt (a few threads then also hold the
// top Theta coefficients, s + 3 > nt).
SLSE_NI void dnc_leaf_block2(DncCtx& X, const cplx* E1, const cplx* Bw, int s, cplx* T, Blk& b) {
#ifdef SLSE_HOST_EMU
  dnc_leaf(X, E1, Bw, s, T, b);
#else
  const int tid = b.tid, nt = b.nt;
  const int ld = s + 1;
  const int le = s + 4, l1 = ld + 2, l2 = ld + 3;  // row strides (zero prefixes: 1 for row 1, 2 for row 2)
  __builtin_assume(__isShared(X.f.smem));
  cplx* eb = X.f.smem;        // [2][le]
  cplx* bbuf = eb + 2 * le;   // [2][le]
  cplx* r1 = bbuf + 2 * le;   // [2][Theta_11 | Theta_12][l1], coefficient i at i + 1
  cplx* r2 = r1 + 4 * l1;     // [2][Theta_21 | Theta_22][l2], coefficient i at i + 2
  cplx* kb = r2 + 4 * l2;     // [2][2] (k_t, k_{t+1}) of the pair
  const cplx z = mk(0.0, 0.0);
  for (int i = tid; i < 2 * le; i += nt) {
    const int q = i % le;
    eb[i] = (i < le && q < s) ? E1[q] : z;
    bbuf[i] = (i < le && q < s) ? Bw[q] : z;
  }
  for (int i = tid; i < 4 * l1; i += nt) r1[i] = (i == 1) ? mk(1.0, 0.0) : z;           // Theta_11[0] = 1
  for (int i = tid; i < 4 * l2; i += nt) r2[i] = (i == l2 + 2) ? mk(1.0, 0.0) : z;      // Theta_22[0] = 1
  double d = X.d;
  double* dtmp = X.delta_tmp + X.step;
  const double floor_ = X.floor_;
  double* dsh = (double*)(kb + 4);  // the chain warp's running prediction error (read after the loop)
  if (tid == 0) {  // k_0, and k_1 from the pre-update pair (e_1, b_1)
    const double inv = 1.0 / d;
    const cplx e0 = E1[0];
    const cplx k0 = mk(-e0.re * inv, -e0.im * inv);
    kb[0] = k0;
    dsh[0] = d;
    if (s > 1) {
      const double d1 = d * (1.0 - (k0.re * k0.re + k0.im * k0.im));
      const cplx en = cadd(E1[1], cmul(k0, Bw[1]));
      const double inv1 = rcp_pos(d1);
      kb[1] = mk(-en.re * inv1, -en.im * inv1);
    }
  }
  b.sync();
  int st = 0;
  const int ci = nt - 1 - tid;  // Theta coefficient of this thread
  const int cw = nt >> 6;       // chain warp: a middle warp (the fewest own items over the leaf)
  const bool chain = (tid >> 5) == cw;
  // current / next buffers of the pair, swapped after every pair
  cplx *ec = eb, *en_ = eb + le, *bc = bbuf, *bn_ = bbuf + le;
  cplx *r1c = r1, *r1n = r1 + 2 * l1, *r2c = r2, *r2n = r2 + 2 * l2;
  cplx *kc_ = kb, *kn_ = kb + 2;
  int t = 0;
  for (; t + 1 < s; t += 2) {
    const cplx ka = kc_[0], kk = kc_[1];
    if (ka.re != ka.re) {  // uniform: the chain warp's not-positive-definite marker
      st = kNotPD;
      break;
    }
    const cplx kac = conjg(ka), kkc = conjg(kk);
    if (chain) {
      // Chain warp: the prediction errors of this pair, the check that they
      // stay above the floor, and the next pair's coefficients from slots
      // 1..3 of the pre-pair state, all before this warp's own items (every
      // lane computes them, lane 0 publishes).  The other warps only read
      // (k_t, k_{t+1}); a failed check reaches them as a NaN coefficient.
      const double d1 = d * (1.0 - (ka.re * ka.re + ka.im * ka.im));
      const double d2 = d1 * (1.0 - (kk.re * kk.re + kk.im * kk.im));
      const bool ok = (d1 > floor_) && (d2 > floor_);
      cplx kn0 = mk(0.0, 0.0), kn1 = kn0;
      if (t + 2 < s) {
        const cplx e1s = ec[t + 1], e2s = ec[t + 2], e3s = ec[t + 3];
        const cplx b1s = bc[1], b2s = bc[2], b3s = bc[3];
        const cplx b1 = lf_fma(kac, e1s, b1s);
        const cplx e1h = lf_fma(ka, b2s, e2s);
        const cplx e2 = lf_fma(kk, b1, e1h);        // e^{(t+2)}_{t+2}
        const cplx b2 = lf_fma(kkc, e1h, b1);
        const cplx b1_2 = lf_fma(kac, e2s, b2s);
        const cplx e1h_3 = lf_fma(ka, b3s, e3s);
        const cplx e2_2 = lf_fma(kk, b1_2, e1h_3);  // e^{(t+2)}_{t+3}
        const double inv2 = rcp_pos(d2);
        kn0 = mk(-e2.re * inv2, -e2.im * inv2);
        const double d3 = d2 * (1.0 - (kn0.re * kn0.re + kn0.im * kn0.im));
        const cplx e3n = lf_fma(kn0, b2, e2_2);     // e^{(t+3)}_{t+3}
        const double inv3 = rcp_pos(d3);
        kn1 = mk(-e3n.re * inv3, -e3n.im * inv3);
      }
      if (!ok) kn0.re = __longlong_as_double(0x7ff8000000000000LL);
      if ((tid & 31) == 0) {
        kn_[0] = kn0;
        kn_[1] = kn1;
        dsh[0] = d2;
        dtmp[t + 1] = d1;
        dtmp[t + 2] = d2;
      }
      d = d2;
    }
    const int j = tid;
    if (j < s - t - 1) {
      const cplx ej = ec[t + j], bj = bc[j];
      const cplx ej1 = ec[t + 1 + j], bj1 = bc[j + 1];
      const cplx b1 = lf_fma(kac, ej, bj);        // step t, own slot
      const cplx e1h = lf_fma(ka, bj1, ej1);      // step t, slot j + 1 (index t + 1 + j)
      en_[t + 1 + j] = lf_fma(kk, b1, e1h);       // step t + 1, own slot
      bn_[j] = lf_fma(kkc, e1h, b1);
    }
    // Theta coefficient ci (and ci + nt when s >= nt: only the top one)
    for (int cq = ci; cq <= t + 2; cq += nt) {
      const cplx a11 = r1c[cq + 1], a12 = r1c[l1 + cq + 1];
      const cplx h11 = r1c[cq], h12 = r1c[l1 + cq];            // coefficient cq - 1, row 1
      const cplx p21 = r2c[cq + 1], p22 = r2c[l2 + cq + 1];    // coefficient cq - 1, row 2
      const cplx q21 = r2c[cq], q22 = r2c[l2 + cq];            // coefficient cq - 2, row 2
      const cplx A1 = lf_fma(ka, p21, a11), A2 = lf_fma(ka, p22, a12);
      const cplx H1 = lf_fma(kac, h11, q21), H2 = lf_fma(kac, h12, q22);
      r1n[cq + 1] = lf_fma(kk, H1, A1);
      r1n[l1 + cq + 1] = lf_fma(kk, H2, A2);
      r2n[cq + 2] = lf_fma(kkc, A1, H1);
      r2n[l2 + cq + 2] = lf_fma(kkc, A2, H2);
    }
    b.sync();
    lf_swap(ec, en_);
    lf_swap(bc, bn_);
    lf_swap(r1c, r1n);
    lf_swap(r2c, r2n);
    lf_swap(kc_, kn_);
  }
  // every thread: the chain warp's prediction error, and a failure in the last pair
  d = dsh[0];
  if (!st && kc_[0].re != kc_[0].re) st = kNotPD;
  if (!st && t < s) {  // odd s: one last single step with k_{s-1}
    const cplx ka = kc_[0], kac = conjg(ka);
    const double d1 = d * (1.0 - (ka.re * ka.re + ka.im * ka.im));
    for (int cq = ci; cq <= t + 1; cq += nt) {
      const cplx a11 = r1c[cq + 1], a12 = r1c[l1 + cq + 1];
      const cplx p21 = r2c[cq + 1], p22 = r2c[l2 + cq + 1];
      r1n[cq + 1] = lf_fma(ka, p21, a11);
      r1n[l1 + cq + 1] = lf_fma(ka, p22, a12);
      r2n[cq + 2] = lf_fma(kac, a11, p21);
      r2n[l2 + cq + 2] = lf_fma(kac, a12, p22);
    }
    if (tid == 0) dtmp[t + 1] = d1;
    d = d1;
    if (!(d1 > floor_)) st = kNotPD;
    lf_swap(r1c, r1n);
    lf_swap(r2c, r2n);
  }
  b.sync();
  if (!st) {
    for (int i = tid; i < ld; i += nt) {
      T[i] = r1c[i + 1];
      T[ld + i] = r1c[l1 + i + 1];
      T[2 * ld + i] = r2c[i + 2];
      T[3 * ld + i] = r2c[l2 + i + 2];
    }
  }
  b.sync();
  X.d = d;
  X.step += s;
  if (st) X.status = st;
#endif
}

// forward transform of src[0..len) zero padded to F -> dst[0..F)
SLSE_D void dnc_fwd(cplx* dst, const cplx* src, int len, int F, cplx* work, const FftCtx& f, Blk& b) {
  fft(work, F, -1.0, [=](int i) { return i < len ? src[i] : mk(0.0, 0.0); },
      [=](int i, cplx v) { dst[i] = v; }, f, b);
}

// One internal node's buffers, all carved from `base` (see dnc_arena_elems);
// the product stage uses 8 F above them.
struct DncNode {
  int h, F;
  cplx *T1, *S, *SE, *SB, *work_multi, *E2, *B2, *T2, *above;
};

SLSE_D DncNode dnc_node(cplx* base, int s) {
  DncNode d;
  d.h = s / 2;
  d.F = 1 << ilog2(s + 1);
  d.T1 = base;                         // 4 (h+1)
  d.S = d.T1 + 4 * (d.h + 1);          // 4 F : spectra of T1 (kept for the product)
  d.SE = d.S + 4 * (size_t)d.F;        // F
  d.SB = d.SE + d.F;                   // F
  d.work_multi = d.SB + d.F;           // 6 F (global fallback buffer of the batched FFTs)
  d.E2 = d.work_multi + 6 * (size_t)d.F;  // s - h + 1
  d.B2 = d.E2 + (s - d.h + 1);         // s - h
  d.T2 = d.B2 + (s - d.h);             // 4 (s - h + 1)
  d.above = d.T2 + 4 * (s - d.h + 1);  // children / product scratch start here
  return d;
}

// Theta is J-para-unitary: every factor M_k = [[1, k z], [conj(k), z]]
// satisfies Theta_21 = Theta_12^# and Theta_22 = Theta_11^#, where
// p^#(z) = z^s conj(p(1 / conj z)) reverses and conjugates the s + 1
// coefficients (s steps, degree s).  So only row 1 of a product is
// computed; row 2 is this O(s) reversal (and, for spectra, W^{s k} conj).
SLSE_D void dnc_fill_row2(cplx* T, int s, Blk& b) {
  const int ld = s + 1;
  for (int i = b.tid; i < ld; i += b.nt) {
    T[2 * ld + i] = conjg(T[ld + (s - i)]);
    T[3 * ld + i] = conjg(T[s - i]);
  }
  fft_barrier();
}

struct DncFrame {
  const cplx* E;
  const cplx* Bw;
  cplx* T;
  cplx* base;
  int s;
  int phase;
  int row1;  // only Theta_11, Theta_12 are needed (the root and its right spine)
};

// Transfer matrix of s steps (iterative post-order traversal; an explicit
// frame stack instead of device recursion keeps the stack statically sized).
SLSE_NI void dnc_split(DncCtx& X, const cplx* E0, const cplx* Bw0, int s0, cplx* T0, Blk& b) {
  DncFrame fr[40];
  int sp = 0;
  fr[sp++] = DncFrame{E0, Bw0, T0, X.arena, s0, 0, 1};
  const bool prof = X.prof != nullptr && b.tid == 0;
  const long long tstart = dnc_clock();
  while (sp > 0 && !X.status) {
    DncFrame& cf = fr[sp - 1];
    const int s = cf.s;
    const long long t0 = prof ? dnc_clock() : 0;
    if (s <= X.leaf_max) {
      if (s <= kDncLeaf && X.leaf_max <= kDncLeaf) dnc_leaf(X, cf.E + 1, cf.Bw, s, cf.T, b);
#if SLSE_DNC_LEAF2
      else if (s <= b.nt && 12 * s + 50 <= X.f.smem_cap) dnc_leaf_block2(X, cf.E + 1, cf.Bw, s, cf.T, b);
#endif
      else dnc_leaf_block(X, cf.E + 1, cf.Bw, s, cf.T, b);
      if (prof) X.prof[0] += dnc_clock() - t0;
      --sp;
      continue;
    }
    const DncNode d = dnc_node(cf.base, s);
    const int h = d.h, F = d.F;
    const double invF = 1.0 / (double)F;
    if (cf.phase == 0) {  // descend into the left half
      cf.phase = 1;
      fr[sp++] = DncFrame{cf.E, cf.Bw, d.T1, d.above, h, 0, 0};
      continue;
    }
    if (s <= X.direct_max) {  // small node: direct products
      const int tid = b.tid, nt = b.nt;
      const int l1 = h + 1;
      const cplx* T1 = d.T1;
      if (cf.phase == 1) {
        const cplx* E = cf.E;
        const cplx* Bw = cf.Bw;
        cplx* E2 = d.E2;
        cplx* B2 = d.B2;
        const int ne = s - h + 1, nb = s - h;
        if (4 * l1 + 2 * s + 2 <= X.f.smem_cap) {  // operands to shared memory (latency)
          cplx* sT = X.f.smem;
          cplx* sE = sT + 4 * l1;
          cplx* sB = sE + (s + 1);
          for (int i = tid; i < 4 * l1; i += nt) sT[i] = T1[i];
          for (int i = tid; i <= s; i += nt) sE[i] = E[i];
          for (int i = tid; i <= s; i += nt) sB[i] = i < s ? Bw[i] : mk(0.0, 0.0);  // b_s := 0 (no bound test)
          fft_barrier();
          // four interleaved partial sums: the FMA chain is a quarter as deep
          for (int t = tid; t < ne + nb; t += nt) {
            const bool isE = t < ne;
            const int j = isE ? t : t - ne;
            const cplx* A = sT + (isE ? 0 : 2 * l1);  // T11,T12 or T21,T22
            const cplx* Ek = sE + h + j;              // Ek[-i] = e_{h+j-i}
            const cplx* Bk = sB + h + j;
            cplx acc[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
            int i = 0;
            for (; i + 4 <= l1; i += 4) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                acc[u] = cadd(acc[u], cmul(A[i + u], Ek[-(i + u)]));
                acc[u] = cadd(acc[u], cmul(A[l1 + i + u], Bk[-(i + u)]));
              }
            }
            for (; i < l1; ++i) {
              acc[0] = cadd(acc[0], cmul(A[i], Ek[-i]));
              acc[0] = cadd(acc[0], cmul(A[l1 + i], Bk[-i]));
            }
            const cplx r = cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3]));
            if (isE) E2[j] = r; else B2[j] = r;
          }
        } else {
          for (int t = tid; t < ne + nb; t += nt) {
            const bool isE = t < ne;
            const int j = isE ? t : t - ne;
            const cplx* A = T1 + (isE ? 0 : 2 * l1);  // T11,T12 or T21,T22
            cplx acc = mk(0.0, 0.0);
            for (int i = 0; i < l1; ++i) {
              const int k = h + j - i;  // 0 <= k <= s
              acc = cadd(acc, cmul(A[i], E[k]));
              if (k < s) acc = cadd(acc, cmul(A[l1 + i], Bw[k]));
            }
            if (isE) E2[j] = acc; else B2[j] = acc;
          }
        }
        fft_barrier();
        if (prof) X.prof[1] += dnc_clock() - t0;
        cf.phase = 2;
        fr[sp++] = DncFrame{d.E2, d.B2, d.T2, d.above, s - h, 0, cf.row1};
        continue;
      }
      // Theta = T2 T1 ; T_rc[k] = sum_i T2_r1[i] T1_1c[k-i] + T2_r2[i] T1_2c[k-i]
      const int l2 = s - h + 1, ld = s + 1;
      const cplx* T2 = d.T2;
      cplx* T = cf.T;
      if (4 * (l1 + l2) <= X.f.smem_cap) {
        cplx* s1 = X.f.smem;
        cplx* s2 = s1 + 4 * l1;
        for (int i = tid; i < 4 * l1; i += nt) s1[i] = T1[i];
        for (int i = tid; i < 4 * l2; i += nt) s2[i] = T2[i];
        fft_barrier();
        T1 = s1;
        T2 = s2;
      }
      const int nrow = 2;  // row 1 only; row 2 by dnc_fill_row2 (not needed on the right spine)
      for (int t = tid; t < nrow * ld; t += nt) {
        const int q = t / ld, k = t - q * ld;
        const int r = q >> 1, c = q & 1;
        const cplx* A1 = T2 + (2 * r) * l2;
        const cplx* A2 = T2 + (2 * r + 1) * l2;
        const cplx* B1 = T1 + c * l1;
        const cplx* B2p = T1 + (2 + c) * l1;
        const int lo = k - h > 0 ? k - h : 0;
        const int hi = k < l2 - 1 ? k : l2 - 1;
        cplx acc4[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
        int i = lo;
        for (; i + 4 <= hi + 1; i += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc4[u] = cadd(acc4[u], cmul(A1[i + u], B1[k - i - u]));
            acc4[u] = cadd(acc4[u], cmul(A2[i + u], B2p[k - i - u]));
          }
        }
        for (; i <= hi; ++i) {
          acc4[0] = cadd(acc4[0], cmul(A1[i], B1[k - i]));
          acc4[0] = cadd(acc4[0], cmul(A2[i], B2p[k - i]));
        }
        const cplx acc = cadd(cadd(acc4[0], acc4[1]), cadd(acc4[2], acc4[3]));
        T[t] = acc;
      }
      fft_barrier();
      if (!cf.row1) dnc_fill_row2(T, s, b);
      if (prof) X.prof[2] += dnc_clock() - t0;
      --sp;
      continue;
    }
    if (cf.phase == 1) {  // left done: middle products give the right window
      const int l1 = h + 1;
      const cplx* T1 = d.T1;
      const cplx* E = cf.E;
      const cplx* Bw = cf.Bw;
      cplx* S = d.S;  // S[0..3] = spectra of T1, S[4] = E, S[5] = Bw (contiguous: S, SE, SB)
      // four forward transforms in one batch (T11, T12, E, Bw); the spectra
      // of T21 = T12^#, T22 = T11^# (degree h) follow as W^{h k} conj(.)
      DncFftArgs fa{};
      fa.F = F; fa.h = h; fa.s = s; fa.l1 = l1; fa.invF = invF;
      fa.T1 = T1; fa.E = E; fa.Bw = Bw;
      fa.S = S; fa.SE = d.SE; fa.SB = d.SB; fa.E2 = d.E2; fa.B2 = d.B2;
      fa.work = d.work_multi;
      fa.site = 0;
      dnc_fft_run(X, fa, b);
      {
        const int lgF = ilog2(F);
        for (int k = b.tid; k < F; k += b.nt) {
          const cplx wk = twid_tab(X.f.tw, X.f.twlog, (int)(((long long)h * k) & (F - 1)), lgF, -1.0);
          S[2 * (size_t)F + k] = cmul(wk, conjg(S[(size_t)F + k]));
          S[3 * (size_t)F + k] = cmul(wk, conjg(S[k]));
        }
        fft_barrier();
      }
      // E2 = (T11 E + T12 Bw)[h..s], B2 = (T21 E + T22 Bw)[h..s-1]
      fa.site = 1;
      dnc_fft_run(X, fa, b);
      if (prof) {
        const long long dt = dnc_clock() - t0;
        X.prof[3] += dt;
        const int lv = ilog2(F) - 9;
        if (lv >= 0 && lv < 8) X.prof[8 + lv] += dt;
      }
      cf.phase = 2;
      fr[sp++] = DncFrame{d.E2, d.B2, d.T2, d.above, s - h, 0, cf.row1};
      continue;
    }
    // phase 2: Theta = T2 T1 (degree s; F >= s + 1 so no wrap)
    {
      const int l2 = s - h + 1;
      const cplx* T2 = d.T2;
      cplx* A = d.above;            // 4 F : spectra of T2
      cplx* wk = d.above + 4 * (size_t)F;  // 4 F global work
      // only row 1 of the product is transformed (2 + 2 transforms instead
      // of 4 + 4); row 2 follows by symmetry, skipped on the right spine
      // (row 1 of T2 and of the product; row 2 by dnc_fill_row2)
      cplx* T = cf.T;
      DncFftArgs fa{};
      fa.F = F; fa.h = h; fa.s = s; fa.l2 = l2; fa.ld = s + 1; fa.invF = invF;
      fa.T2 = T2; fa.A = A; fa.S = d.S; fa.T = T; fa.work = wk;
      fa.site = 2;
      dnc_fft_run(X, fa, b);
      fa.site = 3;
      dnc_fft_run(X, fa, b);
      if (!cf.row1) dnc_fill_row2(T, s, b);
      if (prof) {
        const long long dt = dnc_clock() - t0;
        X.prof[4] += dt;
        const int lv = ilog2(F) - 9;
        if (lv >= 0 && lv < 8) X.prof[8 + lv] += dt;
      }
      --sp;
    }
  }
  if (prof) X.prof[5] += dnc_clock() - tstart;
}

// arena size (complex elements) needed by dnc_split for s steps: own
// buffers plus the larger of the (right, i.e. larger) child's need and the
// product stage's 2F; iterative along the chain of larger children.
SLSE_HD size_t dnc_arena_elems(int s) {
  int chain[48];
  int cnt = 0;
  for (int t = s; t > kDncLeaf && cnt < 48; t -= t / 2) chain[cnt++] = t;
  size_t below = 0;
  for (int i = cnt - 1; i >= 0; --i) {
    const int t = chain[i];
    const int h = t / 2;
    const size_t F = (size_t)1 << ilog2(t + 1);
    const size_t own = 4 * (size_t)(h + 1) + 12 * F + 2 * (size_t)(t - h) + 1 + 4 * (size_t)(t - h + 1);
    below = own + (below > 8 * F ? below : 8 * F);
  }
  return below;
}

// Superfast factorisation: same outputs as toeplitz_factor.  T is the root
// transfer matrix storage (4 N complex), arena from dnc_arena_elems(N-1).
SLSE_NI Factor toeplitz_factor_dnc(const cplx* SLSE_RESTRICT c, int n, cplx* T, cplx* arena, double* delta_out,
                                   double* delta_tmp, cplx* SLSE_RESTRICT rho, const FftCtx& f, Blk& b,
                                   int dnc_stockham = 0, int direct_max = SLSE_DNC_DIRECT,
                                   long long* prof = nullptr, Split* sp = nullptr) {
  Factor F;
  F.logdet = 0.0;
  F.status = kOk;
  const cplx c0c = c[0];
  F.c0 = c0c.re;
  F.delta_last = c0c.re;
  if (fabs(c0c.im) > 1e-10 * fmax(fabs(c0c.re), 1.0) || !(c0c.re > 0.0)) {
    F.status = kBadColumn;
    return F;
  }
  const double c0 = c0c.re;
  if (b.tid == 0) delta_tmp[0] = c0;
  DncCtx X;
  X.f = f;
  X.f.stockham = dnc_stockham;  // register Stockham passes for the product transforms
  X.arena = arena;
  X.delta_tmp = delta_tmp;
  X.floor_ = kPdEps * c0;
  X.d = c0;
  X.step = 0;
  X.status = 0;
  X.direct_max = direct_max;
  // block leaves need s + 2 <= nt threads and 8 s + 14 staging elements
  X.leaf_max = kDncLeaf;
#ifndef SLSE_HOST_EMU
  {
    int lm = SLSE_DNC_BLOCK_LEAF;
#if SLSE_DNC_LEAF2
    while (lm > kDncLeaf && (lm > b.nt || 12 * lm + 48 > f.smem_cap)) lm >>= 1;
#else
    while (lm > kDncLeaf && (lm + 2 > b.nt || 8 * lm + 14 > f.smem_cap)) lm >>= 1;
#endif
    if (lm > kDncLeaf) X.leaf_max = lm;
  }
#endif
  X.prof = prof;
  X.sp = sp;
  b.sync();
  // the root window is the column itself: e = b = c (c_0 forced real)
  // (E[0] and Bw[0] are c_0; E[j] = Bw[j] = c_j)
  if (n > 1) dnc_split(X, c, c, n - 1, T, b);
  b.sync();
  if (X.status) {
    F.status = X.status;
    return F;
  }
  F.delta_last = X.d;
  // a = Theta_11 + Theta_12 (first n coefficients), rho_i = conj(a_{n-1-i}) / conj(a_0)
  const int ld = n;  // root Theta has s + 1 = n coefficients
  const cplx a0 = cadd(T[0], T[ld]);
  double part = 0.0;
  for (int j = b.tid; j < n; j += b.nt) {
    const cplx aj = cadd(T[n - 1 - j], T[ld + n - 1 - j]);
    // conj(aj) / conj(a0)
    const double den = cabs2(a0);
    const cplx num = cmul(conjg(aj), a0);
    rho[j] = (n == 1) ? mk(1.0, 0.0) : mk(num.re / den, num.im / den);
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
  }
  F.logdet = b.sum(part);
  return F;
}

}  // namespace slse
