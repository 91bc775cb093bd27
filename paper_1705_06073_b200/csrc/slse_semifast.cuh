// slse_semifast.cuh -- the semifast (Woodbury) bundle: complete OR incomplete
// data.
//
// Reference: _SemifastBundle (pkg/src/superlse/model_core.py:316-409), the
// engine it serves (SemifastEngine :456-460, make_engine "auto" :466-472),
// nufft.gram (nufft.py:184-210, direct evaluation) and the observation
// operator Phi of Observation (model_core.py:43-130: scatter :109-117,
// sample :119-123).
//
// With P the components of positive variance, E_ip = e^{j 2 pi n_i theta_p}
// at the M observed positions n_i (scales a_i, weights w0_i = |a_i|^2,
// d_i = 2 pi n_i):
//   G_j        = E^H diag(w0 d^j) E                  (K x K, j = 0, 1, 2)
//   Sigma^{-1} = G_0[P,P] / beta + diag(1 / gamma_P) = L L^H   (Cholesky)
//   ln|C|      = M ln beta + sum_P ln gamma + 2 sum ln L_jj
//   C^{-1} y   = y / beta - a . (E_P Sigma E_P^H Phi^H y) / beta^2
//   e          = Phi^H C^{-1} y  (length N, zero off the pattern)
//   stats      q, r, u = Psi^H [e, D e, D^2 e];  s, t, v, x = diag(G) / beta
//              minus the Woodbury corrections (G Sigma G)_kk / beta^2
//   grid       q^G = FFT_L(e);  s^G_l = sum w0 / beta - |L^{-1} b(l)|^2 / beta^2,
//              b_p(l) = sum_i w0_i e^{-j 2 pi n_i theta_p} e^{+j 2 pi n_i l / L}
// Everything is CTA-cooperative (Blk) on K x K matrices of leading dimension
// kcap stored in the solver's workspace slab.
#pragma once
#include "slse_stats.cuh"

#define SLSE_CTRL_LOOP_SF _Pragma("unroll 1")
#ifndef SLSE_SF_GRAM_CLOSED
#define SLSE_SF_GRAM_CLOSED 1  // complete data: closed-form Gram sums (sf_gram_complete)
#endif

namespace slse {

// Observation pattern of one problem (model_core.Observation): M observed
// 0-based positions (sorted, < N) and their complex scales (nullptr = ones).
struct SfObs {
  const int* idx;
  const cplx* sc;
  int m;
};

SLSE_D cplx sf_scale(const SfObs& o, int i) { return o.sc ? o.sc[i] : mk(1.0, 0.0); }
SLSE_D double sf_w0(const SfObs& o, int i) { return o.sc ? cabs2(o.sc[i]) : 1.0; }

// Sums over the observed positions are split over groups of `nch` adjacent
// lanes (chunk ch of an item takes i = ch, ch + nch, ...) and combined by
// shuffles, so every thread of the CTA works on them (K items alone would
// occupy K of the 128 threads).  Every lane of a warp must call sf_group_sum.
// lane groups need whole warps (and do not exist in the serial host emulation)
SLSE_D bool sf_lanes_ok(int nt) {
#ifdef SLSE_HOST_EMU
  (void)nt;
  return false;
#else
  return (nt & 31) == 0;
#endif
}
// lanes per item: the smallest power of two that gives every thread a chunk (at most cap <= 32)
SLSE_D int sf_chunks(int items, int nt, int cap) {
  if (!sf_lanes_ok(nt)) return 1;
  int nch = 1;
  while (nch < cap && items * nch < nt) nch *= 2;
  return nch;
}
SLSE_D double sf_group_sum(double v, int nch) {
#ifndef SLSE_HOST_EMU
  for (int o = nch >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
#else
  (void)nch;
#endif
  return v;
}
SLSE_D cplx sf_group_sum(cplx v, int nch) { return mk(sf_group_sum(v.re, nch), sf_group_sum(v.im, nch)); }

// E[p * ld + i] = e^{j 2 pi n_i theta_p}, i < m, p < kk (exactly reduced
// phases), component-major: the sums over i below read consecutive
// addresses, per thread and across the lanes of a group.
SLSE_D void sf_phases(cplx* E, int ld, const SfObs& o, const double* th, int kk, Blk& b) {
  const int tot = o.m * kk;
  SLSE_CTRL_LOOP_SF
  for (int t = b.tid; t < tot; t += b.nt) {
    const int p = t / o.m, i = t - p * o.m;
    E[(size_t)p * ld + i] = expj2pi((double)o.idx[i], th[p], 1.0);
  }
  b.sync();
}

// Weighted steering Gram matrices (nufft.gram, direct; model_core.py:331-333)
// G_j[r, c] = sum_i w0_i d_i^j conj(E_ir) E_ic, Hermitian by construction
// (the reference symmetrises, _hermitize :412-413: real diagonal).  One
// (r <= c) pair per group of 8 lanes.
SLSE_D void sf_gram_complete(cplx* G0, cplx* G1, cplx* G2, int ld, const cplx* E, int lde, const double* th, int n,
                             int kk, Blk& b);
SLSE_D void sf_gram(cplx* G0, cplx* G1, cplx* G2, int ld, const cplx* E, int lde, const SfObs& o, int kk, Blk& b,
                    const double* th = nullptr, int n = 0) {
  if (SLSE_SF_GRAM_CLOSED && th && o.sc == nullptr && o.m == n) {  // complete data: idx = 0 .. n-1, unit scales
    sf_gram_complete(G0, G1, G2, ld, E, lde, th, n, kk, b);
    return;
  }
  const int npairs = kk * (kk + 1) / 2;
  const int nch = sf_lanes_ok(b.nt) ? 8 : 1;  // 8 lanes per pair on the device
  const int tot = npairs * nch;
  SLSE_CTRL_LOOP_SF
  for (int base = 0; base < tot; base += b.nt) {
    const int t = base + b.tid;
    const bool act = t < tot;
    const int q = act ? t / nch : 0, ch = t - (t / nch) * nch;
    int c = 0;  // pair q -> (r, c), r <= c, column-major over the upper triangle
    while ((c + 1) * (c + 2) / 2 <= q) ++c;
    const int r = q - c * (c + 1) / 2;
    cplx a0 = mk(0.0, 0.0), a1 = a0, a2 = a0;
    if (act) {
      const cplx* Ec = E + (size_t)c * lde;
      const cplx* Er = E + (size_t)r * lde;
#pragma unroll 4
      for (int i = ch; i < o.m; i += nch) {
        const cplx e = cmulc(Ec[i], Er[i]);  // E_ic conj(E_ir)
        const double w0 = sf_w0(o, i);
        const double d = 2.0 * kPi * (double)o.idx[i];
        const double wd = w0 * d, wd2 = w0 * (d * d);
        a0 = mk(fma(w0, e.re, a0.re), fma(w0, e.im, a0.im));
        a1 = mk(fma(wd, e.re, a1.re), fma(wd, e.im, a1.im));
        a2 = mk(fma(wd2, e.re, a2.re), fma(wd2, e.im, a2.im));
      }
    }
    a0 = sf_group_sum(a0, nch);
    a1 = sf_group_sum(a1, nch);
    a2 = sf_group_sum(a2, nch);
    if (act && ch == 0) {
      if (r == c) {
        a0.im = 0.0;
        a1.im = 0.0;
        a2.im = 0.0;
      }
      G0[r * ld + c] = a0;
      G1[r * ld + c] = a1;
      G2[r * ld + c] = a2;
      G0[c * ld + r] = conjg(a0);
      G1[c * ld + r] = conjg(a1);
      G2[c * ld + r] = conjg(a2);
    }
  }
  b.sync();
}

// Complete data (positions 0 .. N-1, unit scales): the Gram entries are the
// geometric sums S_j(x) = sum_{i<N} i^j z^i, z = e^{j 2 pi x}, x = theta_c - theta_r
// (wrapped to [-1/2, 1/2)), in closed form -- O(K^2) per bundle instead of
// O(K^2 N):
//   S_0 = (1 - z^N) / (1 - z)
//   S_1 = (z - N z^N + (N-1) z^{N+1}) / (1 - z)^2
//   S_2 = z (1 + z - N^2 z^{N-1} + (2N^2 - 2N - 1) z^N - (N-1)^2 z^{N+1}) / (1 - z)^3
// with 1 - z = 2 sin(pi x) (sin(pi x) - j cos(pi x)) (no cancellation) and
// z^N from the exactly reduced phase N x.  The numerators cancel like
// 1 / (N |x|)^{j+1}: within ~1e-12 of the direct sums for N |x| >= 1/2
// (checked against them up to N = 500); closer pairs take the direct sums.
SLSE_D void sf_gram_complete(cplx* G0, cplx* G1, cplx* G2, int ld, const cplx* E, int lde, const double* th, int n,
                             int kk, Blk& b) {
  const int npairs = kk * (kk + 1) / 2;
  const double N = (double)n;
  const double tp = 2.0 * kPi;
  SLSE_CTRL_LOOP_SF
  for (int q = b.tid; q < npairs; q += b.nt) {
    int c = 0;
    while ((c + 1) * (c + 2) / 2 <= q) ++c;
    const int r = q - c * (c + 1) / 2;
    cplx a0, a1, a2;
    double x = th[c] - th[r];
    x -= floor(x + 0.5);
    if (r == c) {
      a0 = mk(N, 0.0);
      a1 = mk(tp * (0.5 * N * (N - 1.0)), 0.0);
      a2 = mk(tp * tp * ((N - 1.0) * N * (2.0 * N - 1.0) / 6.0), 0.0);
    } else if (fabs(x) * N < 0.5) {
      a0 = a1 = a2 = mk(0.0, 0.0);
      const cplx* Ec = E + (size_t)c * lde;
      const cplx* Er = E + (size_t)r * lde;
      SLSE_CTRL_LOOP_SF
      for (int i = 0; i < n; ++i) {
        const cplx e = cmulc(Ec[i], Er[i]);
        const double d = tp * (double)i;
        a0 = cadd(a0, e);
        a1 = mk(fma(d, e.re, a1.re), fma(d, e.im, a1.im));
        a2 = mk(fma(d * d, e.re, a2.re), fma(d * d, e.im, a2.im));
      }
    } else {
      double sn, cs;
      sincos2pi(0.5 * x, &sn, &cs);  // sin / cos (pi x)
      const cplx omz = mk(2.0 * sn * sn, -2.0 * sn * cs);  // 1 - z
      const cplx z = mk(1.0 - omz.re, -omz.im);
      const cplx zN = expj2pi(N, x, 1.0);                  // z^N, phase N x reduced exactly
      const cplx zNm1 = cmulc(zN, z), zNp1 = cmul(zN, z);
      const double i2 = 1.0 / cabs2(omz);
      const cplx inv = mk(omz.re * i2, -omz.im * i2);      // 1 / (1 - z)
      const cplx inv2 = cmul(inv, inv), inv3 = cmul(inv2, inv);
      const cplx n0 = mk(1.0 - zN.re, -zN.im);
      const cplx n1 = mk(z.re - N * zN.re + (N - 1.0) * zNp1.re, z.im - N * zN.im + (N - 1.0) * zNp1.im);
      const double k1 = N * N, k2 = 2.0 * N * N - 2.0 * N - 1.0, k3 = (N - 1.0) * (N - 1.0);
      const cplx n2 = cmul(z, mk(1.0 + z.re - k1 * zNm1.re + k2 * zN.re - k3 * zNp1.re,
                                 z.im - k1 * zNm1.im + k2 * zN.im - k3 * zNp1.im));
      a0 = cmul(n0, inv);
      a1 = cscale(cmul(n1, inv2), tp);
      a2 = cscale(cmul(n2, inv3), tp * tp);
    }
    G0[r * ld + c] = a0;
    G1[r * ld + c] = a1;
    G2[r * ld + c] = a2;
    G0[c * ld + r] = conjg(a0);
    G1[c * ld + r] = conjg(a1);
    G2[c * ld + r] = conjg(a2);
  }
  b.sync();
}

// Cholesky (lower, scipy cho_factor(lower=True) role) of
// A = G0[P,P] / beta + diag(1 / gamma_P) into Lc (strict lower part; the
// diagonal of Lc keeps A_jj) and the real diagonal ld_[j] = L_jj.
// Returns kNotPD if a pivot is not positive (scipy raises LinAlgError).
SLSE_D int sf_cholesky(cplx* Lc, double* ldg, int ld, const cplx* G0, int ldg0, const int* P, const double* ga,
                       int kp, double be, Blk& b) {
  const int tot = kp * kp;
  SLSE_CTRL_LOOP_SF
  for (int t = b.tid; t < tot; t += b.nt) {
    const int i = t / kp, j = t - i * kp;
    if (j > i) continue;
    const cplx g = G0[P[i] * ldg0 + P[j]];
    Lc[i * ld + j] = i == j ? mk(g.re / be + 1.0 / ga[P[i]], 0.0) : mk(g.re / be, g.im / be);
  }
  b.sync();
  SLSE_CTRL_LOOP_SF
  for (int j = 0; j < kp; ++j) {
    // every thread forms the pivot itself (identical bits, no broadcast)
    double d = Lc[j * ld + j].re;
    SLSE_CTRL_LOOP_SF
    for (int k = 0; k < j; ++k) d -= cabs2(Lc[j * ld + k]);
    if (!(d > 0.0)) return kNotPD;
    const double ljj = sqrt(d);
    const double rjj = 1.0 / ljj;
    if (b.tid == 0) ldg[j] = ljj;
    SLSE_CTRL_LOOP_SF
    for (int i = j + 1 + b.tid; i < kp; i += b.nt) {
      cplx a = Lc[i * ld + j];
      SLSE_CTRL_LOOP_SF
      for (int k = 0; k < j; ++k) a = csub(a, cmulc(Lc[i * ld + k], Lc[j * ld + k]));  // L_ik conj(L_jk)
      Lc[i * ld + j] = mk(a.re * rjj, a.im * rjj);
    }
    b.sync();
  }
  return kOk;
}

// X <- (L L^H)^{-1} X in place (scipy cho_solve), X: kp rows of nrhs
// (row stride ldx).  Column-oriented substitutions, one barrier per pivot.
SLSE_D void sf_cho_solve(const cplx* Lc, const double* ldg, int ld, int kp, cplx* X, int ldx, int nrhs, Blk& b) {
  // forward: L z = x
  SLSE_CTRL_LOOP_SF
  for (int j = 0; j < kp; ++j) {
    const double inv = 1.0 / ldg[j];
    const int tot = (kp - j - 1) * nrhs;
    SLSE_CTRL_LOOP_SF
    for (int t = b.tid; t < tot; t += b.nt) {
      const int i = j + 1 + t / nrhs, c = t % nrhs;
      const cplx xj = cscale(X[j * ldx + c], inv);
      X[i * ldx + c] = csub(X[i * ldx + c], cmul(Lc[i * ld + j], xj));
    }
    b.sync();
  }
  SLSE_CTRL_LOOP_SF
  for (int t = b.tid; t < kp * nrhs; t += b.nt) {
    const int i = t / nrhs, c = t % nrhs;
    X[i * ldx + c] = cscale(X[i * ldx + c], 1.0 / ldg[i]);
  }
  b.sync();
  // backward: L^H x = z
  SLSE_CTRL_LOOP_SF
  for (int j = kp - 1; j >= 0; --j) {
    const double inv = 1.0 / ldg[j];
    const int tot = j * nrhs;
    SLSE_CTRL_LOOP_SF
    for (int t = b.tid; t < tot; t += b.nt) {
      const int i = t / nrhs, c = t % nrhs;
      const cplx xj = cscale(X[j * ldx + c], inv);
      X[i * ldx + c] = csub(X[i * ldx + c], cmul(conjg(Lc[j * ld + i]), xj));  // conj(L_ji) x_j
    }
    b.sync();
  }
  SLSE_CTRL_LOOP_SF
  for (int t = b.tid; t < kp * nrhs; t += b.nt) {
    const int i = t / nrhs, c = t % nrhs;
    X[i * ldx + c] = cscale(X[i * ldx + c], 1.0 / ldg[i]);
  }
  b.sync();
}

}  // namespace slse
