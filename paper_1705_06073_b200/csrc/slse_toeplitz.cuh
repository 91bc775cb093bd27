// slse_toeplitz.cuh -- Hermitian-Toeplitz column, Gohberg-Semencul factor,
// GS apply (C^{-1} y) and the objective's data term.
//
// Reference: toeplitz.py (HermitianToeplitz :44-64, levinson_durbin
// :121-145, generalized_schur :230-260, apply_inverse :279-309,
// log_det :312-314); model_core.py:242-249, 256-274.
#pragma once
#include "slse_fft.cuh"
#include "slse_split.cuh"

namespace slse {

constexpr double kPdEps = 1e-13;  // toeplitz.py:32

enum Status : int {
  kOk = 0,
  kNotPD = 1,          // NotPositiveDefinite (toeplitz.py:55-57, 141-142, 191-192, 249-252)
  kBadColumn = 2,      // c_0 not real-positive (toeplitz.py:55-57)
  kCapacity = 3,       // trace / event buffer too small (results truncated)
};

// ---------------------------------------------------------------------------
// Row 1: y_m = beta*[m==0] + sum_k coef_k e^{+j 2 pi m theta_k}, m = 0..n-1
// (nufft.py:126-144 direct branch; model_core.py:264-265).  Thread t owns
// m = t, t+nt, ...; e^{j2pi m theta} advances by the phasor e^{j2pi nt theta}
// and is re-anchored with an exact sincospi every 16 steps.
// coef_re/coef_im: coefficient k (coef_im may be null for real gammas).
// column=true: covariance-column convention, c_0 <- Re(c_0) + beta0.
SLSE_NI void steer_forward(cplx* SLSE_RESTRICT out, int n, const double* SLSE_RESTRICT thetas,
                          const double* SLSE_RESTRICT coef_re, const double* SLSE_RESTRICT coef_im,
                          int k, double beta0, bool column, Blk& b, int chunk0 = 0, int chunks = 1) {
  const int tid_ = b.tid, nt_ = b.nt;
  // accumulate in registers chunk-wise: each thread handles up to 16 owned m
  // values per sweep over k.  (chunk0, chunks): this block computes chunks
  // chunk0, chunk0 + chunks, ... of 16 nt outputs (a CTA pair splits the
  // chunks; every output's arithmetic is the same either way)
  for (int m0 = tid_ + chunk0 * 16 * nt_; m0 < n; m0 += chunks * 16 * nt_) {
    const int J = (n - m0 + nt_ - 1) / nt_;  // owned values in this chunk (<= 16 used)
    cplx acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = mk(0.0, 0.0);
    // frequencies in pairs: two independent phasor chains (the recurrence
    // is the latency chain); acc[j] still adds them in slot order
    int kk = 0;
    for (; kk + 1 < k; kk += 2) {
      const double tha = thetas[kk], thb = thetas[kk + 1];
      const double cra = coef_re[kk], crb = coef_re[kk + 1];
      const double cia = coef_im ? coef_im[kk] : 0.0, cib = coef_im ? coef_im[kk + 1] : 0.0;
      cplx ea = expj2pi((double)m0, tha, 1.0), eb = expj2pi((double)m0, thb, 1.0);
      const cplx sa = expj2pi((double)nt_, tha, 1.0), sb = expj2pi((double)nt_, thb, 1.0);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < J) {
          acc[j].re += ea.re * cra - ea.im * cia;
          acc[j].im += ea.re * cia + ea.im * cra;
          acc[j].re += eb.re * crb - eb.im * cib;
          acc[j].im += eb.re * cib + eb.im * crb;
          ea = cmul(ea, sa);
          eb = cmul(eb, sb);
        }
      }
    }
    for (; kk < k; ++kk) {
      const double th = thetas[kk];
      const double cr = coef_re[kk];
      const double ci = coef_im ? coef_im[kk] : 0.0;
      cplx e = expj2pi((double)m0, th, 1.0);
      cplx step = expj2pi((double)nt_, th, 1.0);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < J) {
          // coef * basis, summed over k in slot order
          acc[j].re += e.re * cr - e.im * ci;
          acc[j].im += e.re * ci + e.im * cr;
          e = cmul(e, step);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = m0 + j * nt_;
      if (m < n) {
        cplx v = acc[j];
        if (column && m == 0) v = mk(v.re + beta0, 0.0);  // c_0 forced real (toeplitz.py:58-59)
        out[m] = v;
      }
    }
  }
  b.sync();
}

#ifndef SLSE_HOST_EMU
// One-warp form of steer_forward (N <= 512 solver path): lane owns
// m = lane + 32 j in chunks of 8, phasor recurrence anchored by an exact
// sincospi per chunk; small rolled body (instruction-cache footprint).
static __device__ __noinline__ void steer_forward_warp(cplx* SLSE_RESTRICT out, int n,
                                                       const double* SLSE_RESTRICT thetas,
                                                       const double* SLSE_RESTRICT coef_re,
                                                       const double* SLSE_RESTRICT coef_im, int k, double beta0,
                                                       bool column, int lane) {
#pragma unroll 1
  for (int m0 = lane; m0 < n; m0 += 256) {
    cplx acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = mk(0.0, 0.0);
#pragma unroll 1
    for (int kk = 0; kk < k; ++kk) {
      const double th = thetas[kk];
      const double cr = coef_re[kk];
      const double ci = coef_im ? coef_im[kk] : 0.0;
      cplx e = expj2pi((double)m0, th, 1.0);
      const cplx step = expj2pi(32.0, th, 1.0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[j].re += e.re * cr - e.im * ci;
        acc[j].im += e.re * ci + e.im * cr;
        e = cmul(e, step);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int m = m0 + 32 * j;
      if (m < n) out[m] = (column && m == 0) ? mk(acc[j].re + beta0, 0.0) : acc[j];
    }
  }
  __syncwarp();
}
#endif

// ---------------------------------------------------------------------------
// Rows 2-4: Gohberg-Semencul parameters (rho, delta) by the Schur-Levinson
// recursion.  Reflection coefficients come from the Schur generators
// (no inner products: one barrier per step), the predictor a follows the
// Levinson update a <- a + k z conj(rev a) (toeplitz.py:135-142); with
// e_j^{(m)} = sum_i a_i c_{j-i} and B_j^{(m)} = b_{j+m}^{(m)} the backward
// residual in a shifted frame:
//   k      = -e_{m+1} / delta_m
//   e_{j+m+1} += k B_j ,  B_j += conj(k) e_{j+m+1}      (j = 0..N-2-m)
//   delta_{m+1} = delta_m (1 - |k|^2)
// Numerically equivalent to the reference's LD / generalized Schur within
// ~1e-13.  Work arrays e, B, a hold n complex each (shared
// memory when they fit, else global).  Output rho_i = conj(a_{N-1-i})
// (rho_{N-1} = 1), delta (optional array), sum log delta, delta_{N-1}.
struct Factor {
  double logdet;
  double delta_last;
  double c0;
  int status;
};

template <bool SH>
SLSE_D Factor toeplitz_factor_impl(const cplx* SLSE_RESTRICT c, int n, cplx* e, cplx* B, cplx* a,
                                   double* delta_out, double* delta_tmp, cplx* SLSE_RESTRICT rho,
                                   Blk& b) {
  const int tid_ = b.tid, nt_ = b.nt;
  Factor F;
  F.logdet = 0.0;
  F.status = kOk;
  const cplx c0c = c[0];
  F.c0 = c0c.re;
  F.delta_last = c0c.re;
  // HermitianToeplitz validation (toeplitz.py:55-57)
  if (fabs(c0c.im) > 1e-10 * fmax(fabs(c0c.re), 1.0) || !(c0c.re > 0.0)) {
    F.status = kBadColumn;
    return F;
  }
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
#ifndef SLSE_HOST_EMU
  if (SH) {  // work arrays in shared memory: let the compiler emit LDS/STS
    __builtin_assume(__isShared(e));
    __builtin_assume(__isShared(B));
    __builtin_assume(__isShared(a));
  }
#endif
  for (int j = tid_; j < n; j += nt_) {
    cplx cj = (j == 0) ? mk(c0, 0.0) : c[j];
    e[j] = cj;
    B[j] = cj;
    a[j] = mk(j == 0 ? 1.0 : 0.0, 0.0);
    delta_tmp[j] = 0.0;
  }
  if (tid_ == 0) delta_tmp[0] = c0;
  b.sync();
  double delta = c0;
  int fail = 0;
  // Reflection coefficient of step 0.  Every step uses one reciprocal of
  // delta (instead of two divisions); a single-warp block also computes the
  // NEXT coefficient from the pre-update values e_{m+2}, B_1 before its bulk
  // update (lookahead), taking the reciprocal off the critical path.
  const bool look = nt_ <= 32;
  cplx k = mk(0.0, 0.0);
  if (n > 1) {
    const cplx e1 = e[1];
    const double inv = 1.0 / delta;
    k = mk(-e1.re * inv, -e1.im * inv);
  }
  for (int m = 0; m + 1 < n; ++m) {
    const cplx kc = conjg(k);
    const double dnext = delta * (1.0 - (k.re * k.re + k.im * k.im));
    // 1 / delta_{m+1}, formed before the step's updates so the next
    // coefficient after the barrier is a load and a multiply
    const double inv_next = rcp_pos(dnext);
    cplx knext = mk(0.0, 0.0);
    if (look && m + 2 < n) {
      const cplx e2 = e[m + 2], b1 = B[1];
      const cplx emn = cadd(e2, cmul(k, b1));
      const double invn = 1.0 / dnext;
      knext = mk(-emn.re * invn, -emn.im * invn);
      b.sync();  // every lane has read e_{m+2}, B_1 before any write below
    }
    const int cnt = n - 1 - m;  // pairs j = 0..cnt-1
    for (int j = tid_; j < cnt; j += nt_) {
      const cplx ej = e[j + m + 1];
      const cplx bj = B[j];
      if (j > 0) e[j + m + 1] = cadd(ej, cmul(k, bj));
      B[j] = cadd(bj, cmul(kc, ej));
    }
    // predictor: a_i' = a_i + k conj(a_{m+1-i}), i = 1..m+1 (a_{m+1} = 0 before)
    const int top = m + 1;
    const int npair = (top + 1) / 2;
    for (int i = tid_; i <= npair; i += nt_) {
      if (i == 0) {
        a[top] = cmul(k, conjg(a[0]));
      } else {
        const int jj = top - i;
        if (i < jj) {
          const cplx ai = a[i], aj = a[jj];
          a[i] = cadd(ai, cmul(k, conjg(aj)));
          a[jj] = cadd(aj, cmul(k, conjg(ai)));
        } else if (i == jj) {
          const cplx ai = a[i];
          a[i] = cadd(ai, cmul(k, conjg(ai)));
        }
      }
    }
    if (tid_ == 0) delta_tmp[m + 1] = dnext;
    b.sync();
    delta = dnext;
    if (!(delta > floor_)) { fail = 1; break; }
    if (m + 2 < n) {
      if (look) {
        k = knext;
      } else {
        const cplx em = e[m + 2];
        k = mk(-em.re * inv_next, -em.im * inv_next);
      }
    }
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
  F.delta_last = delta;
  double part = 0.0;
  for (int j = tid_; j < n; j += nt_) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
    rho[j] = conjg(a[n - 1 - j]);
  }
  F.logdet = b.sum(part);
  return F;
}

#ifndef SLSE_HOST_EMU
// One-warp Schur-Levinson (the N <= 512 solver path).  Register slot
// r = lane + 32 q holds, in a shifted frame where it never changes lanes,
// either the backward generator B_r (r < n-1-m at step m) or the backward
// predictor coefficient b_m[r - n + 1 + m] (r >= n-1-m).  The two ranges tile
// [0, n) exactly, and both updates read and write E[r + m + 1], where
// E[0, n) is the forward generator e and E[n-1+j] the forward predictor a_j:
//   E <- E + k B,   B <- B + conj(k) E,
// so each step is one uniform pass over the Q register slots (no separate
// predictor loop).  The slot that retires from the generator range at step
// m becomes the new predictor coefficient b_{m+1}[0] = conj(k).  Needs E of
// 2n elements (e and the adjacent generator buffer); warp barriers only.
template <int Q>
SLSE_D Factor toeplitz_factor_warp(const cplx* SLSE_RESTRICT c, int n, cplx* E, double* delta_out,
                                   double* delta_tmp, cplx* SLSE_RESTRICT rho, Blk& b) {
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
  __builtin_assume(__isShared(E));
  const int lane = b.tid;
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
  cplx Breg[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = lane + 32 * q;
    cplx cj = mk(0.0, 0.0);
    if (j < n) cj = (j == 0) ? mk(c0, 0.0) : c[j];
    Breg[q] = (j == n - 1) ? mk(1.0, 0.0) : cj;  // b_0 = 1 sits in slot n-1
    if (j < n) {
      E[j] = cj;
      E[n + j] = mk(0.0, 0.0);
      delta_tmp[j] = 0.0;
    }
  }
  if (lane == 0) delta_tmp[0] = c0;
  __syncwarp();
  double delta = c0;
  int fail = 0;
  cplx k = mk(0.0, 0.0);
  if (n > 1) {
    const cplx e1 = E[1];
    const double inv = 1.0 / delta;
    k = mk(-e1.re * inv, -e1.im * inv);
  }
  for (int m = 0; m + 1 < n; ++m) {
    const cplx kc = conjg(k);
    const double dnext = delta * (1.0 - (k.re * k.re + k.im * k.im));
    // 1 / delta_{m+1}, formed before the step's updates so the next
    // coefficient after the barrier is a load and a multiply
    const double inv_next = rcp_pos(dnext);
    cplx knext = mk(0.0, 0.0);
    if (m + 2 < n) {  // lookahead from pre-update values
      const cplx e2 = E[m + 2];
      const cplx b1 = mk(__shfl_sync(0xffffffffu, Breg[0].re, 1), __shfl_sync(0xffffffffu, Breg[0].im, 1));
      const cplx emn = cadd(e2, cmul(k, b1));
      const double invn = 1.0 / dnext;
      knext = mk(-emn.re * invn, -emn.im * invn);
      __syncwarp();
    }
    const int top = n - 2 - m;  // generator slot retiring at this step
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int r = lane + 32 * q;
      if (r < n) {
        const cplx ej = E[r + m + 1];
        const cplx bj = Breg[q];
        if (r > 0) E[r + m + 1] = cadd(ej, cmul(k, bj));
        Breg[q] = (r == top) ? kc : cadd(bj, cmul(kc, ej));
      }
    }
    if (lane == 0) delta_tmp[m + 1] = dnext;
    __syncwarp();
    delta = dnext;
    if (!(delta > floor_)) { fail = 1; break; }
    k = knext;
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
  F.delta_last = delta;
  double part = 0.0;
  for (int j = lane; j < n; j += 32) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
    rho[j] = (j == n - 1) ? mk(1.0, 0.0) : conjg(E[2 * n - 2 - j]);  // conj(a_{n-1-j}), a_0 = 1
  }
  F.logdet = b.sum(part);
  return F;
}
#endif

#ifndef SLSE_HOST_EMU
// Register-resident one-warp Schur-Levinson for N <= 32 Q.  Same slot scheme
// as toeplitz_factor_warp, but lane L owns the CONTIGUOUS slots
// r = Q L + i and keeps both E[r + m + 1] and B_r in registers: after each
// step E moves down one slot, which is a static register rotation (the m
// loop is unrolled Q times) plus one shuffle from lane L+1.  No shared
// memory traffic; lane 0 owns slot 1, so it forms the next reflection
// coefficient from its own update and broadcasts it.  Slots r >= n hold
// zeros and stay zero.
//
// The n-1 steps are aligned so that they END on a block boundary: the first
// block starts at sub-step t0 = (-(n-1)) mod Q.  Then at sub-step t the
// retiring generator slot n-2-m always sits in register Q-1-t (only its
// lane varies), and the final rotation is the identity.
template <int Q, int T>
SLSE_D void lev_regs_step(cplx (&Er)[Q], cplx (&Br)[Q], cplx& k, double& delta, int m, int n, int lane,
                          double* delta_tmp) {
  const double kr = k.re, ki = k.im;
  const double dnext = delta * (1.0 - (kr * kr + ki * ki));
  const double inv = rcp_pos(dnext);
  const int top = n - 2 - m;
  const bool mine = (top - (Q - 1 - T)) == Q * lane;  // this lane owns the retiring slot
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int p = (i + T) % Q;  // physical E register of logical slot i (B does not move)
    const cplx ej = Er[p], bj = Br[i];
    // E <- E + k B ;  B <- B + conj(k) E
    Er[p] = mk(fma(kr, bj.re, fma(-ki, bj.im, ej.re)), fma(kr, bj.im, fma(ki, bj.re, ej.im)));
    cplx bn = mk(fma(kr, ej.re, fma(ki, ej.im, bj.re)), fma(kr, ej.im, fma(-ki, ej.re, bj.im)));
    if (i == Q - 1 - T) bn = mine ? mk(kr, -ki) : bn;  // b_{m+1}[0] = conj(k)
    Br[i] = bn;
  }
  // lane 0 holds slot 1, i.e. the updated e_{m+2}: the next pivot
  const cplx e2 = Er[(1 + T) % Q];
  const double nr = __shfl_sync(0xffffffffu, -e2.re * inv, 0);
  const double ni = __shfl_sync(0xffffffffu, -e2.im * inv, 0);
  // shift E down one slot: logical slot 0 of lane L+1 becomes logical slot
  // Q-1 of lane L (the same physical register under the rotation)
  constexpr int p0 = T % Q;
  const double sr = __shfl_down_sync(0xffffffffu, Er[p0].re, 1);
  const double si = __shfl_down_sync(0xffffffffu, Er[p0].im, 1);
  Er[p0] = (lane == 31) ? mk(0.0, 0.0) : mk(sr, si);
  if (lane == 0) delta_tmp[m + 1] = dnext;
  delta = dnext;
  k = mk(nr, ni);
}

template <int Q, int T>
SLSE_D void lev_regs_block(cplx (&Er)[Q], cplx (&Br)[Q], cplx& k, double& delta, int& m, int n, int lane,
                           double* delta_tmp, int t0) {
  if constexpr (T < Q) {
    if (T >= t0) {
      lev_regs_step<Q, T>(Er, Br, k, delta, m, n, lane, delta_tmp);
      ++m;
    }
    lev_regs_block<Q, T + 1>(Er, Br, k, delta, m, n, lane, delta_tmp, t0);
  }
}

template <int Q, int T>
SLSE_D void lev_regs_full(cplx (&Er)[Q], cplx (&Br)[Q], cplx& k, double& delta, int m, int n, int lane,
                          double* delta_tmp) {
  if constexpr (T < Q) {
    lev_regs_step<Q, T>(Er, Br, k, delta, m + T, n, lane, delta_tmp);
    lev_regs_full<Q, T + 1>(Er, Br, k, delta, m, n, lane, delta_tmp);
  }
}

template <int Q>
SLSE_D Factor toeplitz_factor_regs(const cplx* SLSE_RESTRICT c, int n, double* delta_out, double* delta_tmp,
                                   cplx* SLSE_RESTRICT rho, Blk& b) {
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
  const int lane = b.tid;
  const int base = Q * lane;
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
  const int t0 = (Q - (n - 1) % Q) % Q;  // first block runs sub-steps t0..Q-1
  cplx Er[Q], Br[Q];
#pragma unroll
  for (int p = 0; p < Q; ++p) {
    const int i = (p - t0 + Q) % Q;  // logical slot held by physical register p at the start
    const int r = base + i;
    Er[p] = (r + 1 < n) ? c[r + 1] : mk(0.0, 0.0);
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int r = base + i;
    Br[i] = (r + 1 < n) ? (r == 0 ? mk(c0, 0.0) : c[r]) : mk(r == n - 1 ? 1.0 : 0.0, 0.0);
    if (r < n) delta_tmp[r] = 0.0;
  }
  __syncwarp();
  if (lane == 0) delta_tmp[0] = c0;
  double delta = c0;
  cplx k = mk(0.0, 0.0);
  if (n > 1) {
    const double e1r = __shfl_sync(0xffffffffu, c[1].re, 0), e1i = __shfl_sync(0xffffffffu, c[1].im, 0);
    const double inv = 1.0 / delta;
    k = mk(-e1r * inv, -e1i * inv);
  }
  int fail = 0;
  if (n > 1) {
    int m = 0;
    lev_regs_block<Q, 0>(Er, Br, k, delta, m, n, lane, delta_tmp, t0);
    fail = !(delta > floor_);
    for (; m + 1 < n && !fail; m += Q) {
      lev_regs_full<Q, 0>(Er, Br, k, delta, m, n, lane, delta_tmp);
      fail = !(delta > floor_);
    }
  }
  __syncwarp();
  if (!fail) {  // a pivot below the floor anywhere inside a block
    for (int j = lane + 1; j < n; j += 32) fail |= !(delta_tmp[j] > floor_);
    fail = __any_sync(0xffffffffu, fail);
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
  // after n-1 steps (rotation back to identity) logical slot i of lane L
  // holds a_{QL+i+1}; rho_j = conj(a_{n-1-j})
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int j = base + i + 1;
    if (j <= n - 1) rho[n - 1 - j] = conjg(Er[i]);
  }
  if (lane == 0) rho[n - 1] = mk(1.0, 0.0);
  F.delta_last = delta;
  double part = 0.0;
  for (int j = lane; j < n; j += 32) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
  }
  F.logdet = b.sum(part);
  return F;
}
#endif

#ifndef SLSE_HOST_EMU
// Compact form of toeplitz_factor_regs (the default): the same register
// slots, but a rolled step loop -- E moves down one slot by register moves
// and the retiring slot is found by compare -- so the whole recursion is a
// ~2.5 KB loop body instead of a 30 KB unrolled one.  The persistent solver
// interleaves every phase on an SM, so instruction-cache footprint matters
// more than the ~40 % extra ALU instructions (measured on B200).
#ifndef SLSE_LEV_SLICE
#define SLSE_LEV_SLICE 0  // warp mode: yield the operation window every this many steps (0: never)
#endif
template <int Q>
SLSE_D Factor toeplitz_factor_regs_c(const cplx* SLSE_RESTRICT c, int n, double* delta_out, double* delta_tmp,
                                     cplx* SLSE_RESTRICT rho, Blk& b) {
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
  const int lane = b.tid;
  const int base = Q * lane;
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
  cplx Er[Q], Br[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int r = base + i;
    Er[i] = (r + 1 < n) ? c[r + 1] : mk(0.0, 0.0);
    Br[i] = (r + 1 < n) ? (r == 0 ? mk(c0, 0.0) : c[r]) : mk(r == n - 1 ? 1.0 : 0.0, 0.0);
    if (r < n) delta_tmp[r] = 0.0;
  }
  __syncwarp();
  if (lane == 0) delta_tmp[0] = c0;
  double delta = c0;
  double kr = 0.0, ki = 0.0;
  if (n > 1) {
    const double e1r = __shfl_sync(0xffffffffu, Er[0].re, 0), e1i = __shfl_sync(0xffffffffu, Er[0].im, 0);
    const double inv = 1.0 / delta;
    kr = -e1r * inv;
    ki = -e1i * inv;
  }
  int fail = 0;
#pragma unroll 1
  for (int m = 0; m + 1 < n; ++m) {
    const double dnext = delta * (1.0 - (kr * kr + ki * ki));
    const double inv = rcp_pos(dnext);
    const int toff = n - 2 - m - base;  // retiring generator slot, if this lane owns it
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const cplx ej = Er[i], bj = Br[i];
      Er[i] = mk(fma(kr, bj.re, fma(-ki, bj.im, ej.re)), fma(kr, bj.im, fma(ki, bj.re, ej.im)));
      const cplx bn = mk(fma(kr, ej.re, fma(ki, ej.im, bj.re)), fma(kr, ej.im, fma(-ki, ej.re, bj.im)));
      Br[i] = (i == toff) ? mk(kr, -ki) : bn;  // b_{m+1}[0] = conj(k)
    }
    // lane 0 holds slot 1 = the updated e_{m+2}: the next pivot
    const double nr = __shfl_sync(0xffffffffu, -Er[1].re * inv, 0);
    const double ni = __shfl_sync(0xffffffffu, -Er[1].im * inv, 0);
    const double sr = __shfl_down_sync(0xffffffffu, Er[0].re, 1);
    const double si = __shfl_down_sync(0xffffffffu, Er[0].im, 1);
#pragma unroll
    for (int i = 0; i + 1 < Q; ++i) Er[i] = Er[i + 1];
    Er[Q - 1] = (lane == 31) ? mk(0.0, 0.0) : mk(sr, si);
    if (lane == 0) delta_tmp[m + 1] = dnext;
    delta = dnext;
    if (!(delta > floor_)) { fail = 1; break; }
    kr = nr;
    ki = ni;
#if SLSE_LEV_SLICE > 0
    if ((m & (SLSE_LEV_SLICE - 1)) == SLSE_LEV_SLICE - 1) SLSE_RV_SLICE();
#endif
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int j = base + i + 1;
    if (j <= n - 1) rho[n - 1 - j] = conjg(Er[i]);
  }
  if (lane == 0) rho[n - 1] = mk(1.0, 0.0);
  F.delta_last = delta;
  __syncwarp();
  double part = 0.0;
  for (int j = lane; j < n; j += 32) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
  }
  F.logdet = b.sum(part);
  return F;
}
#endif

#ifndef SLSE_HOST_EMU
// Block form of toeplitz_factor_regs_c: the same register slots across a
// whole CTA -- slot r = Q tid + i holds (E_r, B_r) -- so a step touches no
// shared memory except the next reflection coefficient (thread 0 forms it
// from its own update) and one boundary value per warp for the one-slot
// shift of E (lane 31 takes warp w+1's first slot); both double-buffered,
// one barrier per step.  Replaces the shared-memory Schur-Levinson loops
// (LDS -> FMA -> STS chains per item) for 512 < N <= Q nt.
template <int Q>
SLSE_D Factor toeplitz_factor_regs_blk(const cplx* SLSE_RESTRICT c, int n, cplx* scratch, double* delta_out,
                                       double* delta_tmp, cplx* SLSE_RESTRICT rho, Blk& b) {
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
  const int tid = b.tid, nt = b.nt;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int base = Q * tid;
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
  cplx* kbuf = scratch;     // [2] next reflection coefficient
  cplx* bnd = scratch + 2;  // [2][nw] first E slot of each warp (post-update)
  cplx Er[Q], Br[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int r = base + i;
    Er[i] = (r + 1 < n) ? c[r + 1] : mk(0.0, 0.0);
    Br[i] = (r + 1 < n) ? (r == 0 ? mk(c0, 0.0) : c[r]) : mk(r == n - 1 ? 1.0 : 0.0, 0.0);
    if (r < n) delta_tmp[r] = 0.0;
  }
  b.sync();
  if (tid == 0) delta_tmp[0] = c0;
  double delta = c0;
  double kr = 0.0, ki = 0.0;
  if (n > 1) {
    const cplx e1 = c[1];
    const double inv = 1.0 / delta;
    kr = -e1.re * inv;
    ki = -e1.im * inv;
  }
  int fail = 0;
#pragma unroll 1
  for (int m = 0; m + 1 < n; ++m) {
    const double dnext = delta * (1.0 - (kr * kr + ki * ki));
    const double inv = rcp_pos(dnext);
    const int toff = n - 2 - m - base;  // retiring generator slot, if this thread owns it
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const cplx ej = Er[i], bj = Br[i];
      Er[i] = mk(fma(kr, bj.re, fma(-ki, bj.im, ej.re)), fma(kr, bj.im, fma(ki, bj.re, ej.im)));
      const cplx bn = mk(fma(kr, ej.re, fma(ki, ej.im, bj.re)), fma(kr, ej.im, fma(-ki, ej.re, bj.im)));
      Br[i] = (i == toff) ? mk(kr, -ki) : bn;  // b_{m+1}[0] = conj(k)
    }
    // thread 0 holds slot 1 = the updated e_{m+2}: the next pivot
    if (tid == 0) kbuf[(m + 1) & 1] = Er[1];  // raw: scaled by 1/delta after the barrier
    if (lane == 0 && warp > 0) bnd[(m & 1) * nw + warp] = Er[0];
    const double sr = __shfl_down_sync(0xffffffffu, Er[0].re, 1);
    const double si = __shfl_down_sync(0xffffffffu, Er[0].im, 1);
    b.sync();
    cplx nx = mk(sr, si);
    if (lane == 31) nx = (warp + 1 < nw) ? bnd[(m & 1) * nw + warp + 1] : mk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i + 1 < Q; ++i) Er[i] = Er[i + 1];
    Er[Q - 1] = nx;
    if (tid == 0) delta_tmp[m + 1] = dnext;
    delta = dnext;
    if (!(delta > floor_)) { fail = 1; break; }  // uniform
    const cplx kn = kbuf[(m + 1) & 1];
    kr = -kn.re * inv;
    ki = -kn.im * inv;
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int j = base + i + 1;
    if (j <= n - 1) rho[n - 1 - j] = conjg(Er[i]);
  }
  if (tid == 0) rho[n - 1] = mk(1.0, 0.0);
  F.delta_last = delta;
  b.sync();
  double part = 0.0;
  for (int j = tid; j < n; j += nt) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
  }
  F.logdet = b.sum(part);
  return F;
}
#endif

#ifndef SLSE_HOST_EMU
// Unrolled form of toeplitz_factor_regs_blk (static register renaming, as
// toeplitz_factor_regs does for one warp): Q sub-steps per loop iteration,
// E's one-slot shift is a renaming, and only the one register that can hold
// the retiring slot carries a select -- no per-slot moves or selects.
template <int Q, int T>
SLSE_D void lev_blk_step(cplx (&Er)[Q], cplx (&Br)[Q], double& kr, double& ki, double& delta, int m, int n, int tid,
                         int lane, int warp, int nw, cplx* kbuf, cplx* bnd, double* delta_tmp, Blk& b) {
  const double dnext = delta * (1.0 - (kr * kr + ki * ki));
  const double inv = rcp_pos(dnext);
  const int top = n - 2 - m;
  const bool mine = (top - (Q - 1 - T)) == Q * tid;  // this thread owns the retiring slot
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int p = (i + T) % Q;  // physical E register of logical slot i (B does not move)
    const cplx ej = Er[p], bj = Br[i];
    Er[p] = mk(fma(kr, bj.re, fma(-ki, bj.im, ej.re)), fma(kr, bj.im, fma(ki, bj.re, ej.im)));
    cplx bn = mk(fma(kr, ej.re, fma(ki, ej.im, bj.re)), fma(kr, ej.im, fma(-ki, ej.re, bj.im)));
    if (i == Q - 1 - T) bn = mine ? mk(kr, -ki) : bn;  // b_{m+1}[0] = conj(k)
    Br[i] = bn;
  }
  if (tid == 0) {  // slot 1 = the updated e_{m+2}: the next pivot
    const cplx e2 = Er[(1 + T) % Q];
    kbuf[(m + 1) & 1] = e2;  // raw: every thread scales it by its own 1/delta after the barrier
  }
  constexpr int p0 = T % Q;
  if (lane == 0 && warp > 0) bnd[(m & 1) * nw + warp] = Er[p0];
  const double sr = __shfl_down_sync(0xffffffffu, Er[p0].re, 1);
  const double si = __shfl_down_sync(0xffffffffu, Er[p0].im, 1);
  if (tid == 0) delta_tmp[m + 1] = dnext;
  b.sync();
  Er[p0] = (lane == 31) ? ((warp + 1 < nw) ? bnd[(m & 1) * nw + warp + 1] : mk(0.0, 0.0)) : mk(sr, si);
  delta = dnext;
  const cplx kn = kbuf[(m + 1) & 1];
  kr = -kn.re * inv;
  ki = -kn.im * inv;
}

template <int Q, int T>
SLSE_D void lev_blk_block(cplx (&Er)[Q], cplx (&Br)[Q], double& kr, double& ki, double& delta, int& m, int n, int tid,
                          int lane, int warp, int nw, cplx* kbuf, cplx* bnd, double* delta_tmp, Blk& b, int t0) {
  if constexpr (T < Q) {
    if (T >= t0) {
      lev_blk_step<Q, T>(Er, Br, kr, ki, delta, m, n, tid, lane, warp, nw, kbuf, bnd, delta_tmp, b);
      ++m;
    }
    lev_blk_block<Q, T + 1>(Er, Br, kr, ki, delta, m, n, tid, lane, warp, nw, kbuf, bnd, delta_tmp, b, t0);
  }
}

template <int Q>
SLSE_D Factor toeplitz_factor_regs_blk_u(const cplx* SLSE_RESTRICT c, int n, cplx* scratch, double* delta_out,
                                         double* delta_tmp, cplx* SLSE_RESTRICT rho, Blk& b) {
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
  const int tid = b.tid, nt = b.nt;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int base = Q * tid;
  const double c0 = c0c.re;
  const double floor_ = kPdEps * c0;
  cplx* kbuf = scratch;
  cplx* bnd = scratch + 2;
  const int t0 = (Q - (n - 1) % Q) % Q;  // first block runs sub-steps t0..Q-1 (steps end on a block boundary)
  cplx Er[Q], Br[Q];
#pragma unroll
  for (int p = 0; p < Q; ++p) {
    const int i = (p - t0 + Q) % Q;  // logical slot held by physical register p at the start
    const int r = base + i;
    Er[p] = (r + 1 < n) ? c[r + 1] : mk(0.0, 0.0);
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int r = base + i;
    Br[i] = (r + 1 < n) ? (r == 0 ? mk(c0, 0.0) : c[r]) : mk(r == n - 1 ? 1.0 : 0.0, 0.0);
    if (r < n) delta_tmp[r] = 0.0;
  }
  b.sync();
  if (tid == 0) delta_tmp[0] = c0;
  double delta = c0;
  double kr = 0.0, ki = 0.0;
  if (n > 1) {
    const cplx e1 = c[1];
    const double inv = 1.0 / delta;
    kr = -e1.re * inv;
    ki = -e1.im * inv;
  }
  int fail = 0;
  if (n > 1) {
    int m = 0;
    lev_blk_block<Q, 0>(Er, Br, kr, ki, delta, m, n, tid, lane, warp, nw, kbuf, bnd, delta_tmp, b, t0);
    fail = !(delta > floor_);
#pragma unroll 1
    for (; m + 1 < n && !fail; m += Q) {
      lev_blk_block<Q, 0>(Er, Br, kr, ki, delta, m, n, tid, lane, warp, nw, kbuf, bnd, delta_tmp, b, 0);
      m -= Q;  // (lev_blk_block advanced m by Q)
      fail = !(delta > floor_);
    }
  }
  b.sync();
  if (!fail) {  // a pivot below the floor anywhere inside a block
    int bad = 0;
    for (int j = tid + 1; j < n; j += nt) bad |= !(delta_tmp[j] > floor_);
    fail = b.sumi(bad) != 0;
  }
  if (fail) {
    F.status = kNotPD;
    return F;
  }
  // after n-1 steps (rotation back to identity) logical slot i holds a_{Q tid + i + 1}
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int j = base + i + 1;
    if (j <= n - 1) rho[n - 1 - j] = conjg(Er[i]);
  }
  if (tid == 0) rho[n - 1] = mk(1.0, 0.0);
  F.delta_last = delta;
  b.sync();
  double part = 0.0;
  for (int j = tid; j < n; j += nt) {
    part += log(delta_tmp[j]);
    if (delta_out) delta_out[j] = delta_tmp[j];
  }
  F.logdet = b.sum(part);
  return F;
}
#endif

#ifndef SLSE_LEV_BLK_UNROLL
#define SLSE_LEV_BLK_UNROLL 1
#endif

#ifndef SLSE_HOST_EMU
// Out-of-line entry points: each variant gets its own register allocation,
// so the unrolled bodies (which need the 128-register budget) do not push
// the 1024-thread instantiations of toeplitz_factor into spills.
template <int Q, bool U>
SLSE_NI Factor factor_regs_blk_ni(const cplx* SLSE_RESTRICT c, int n, cplx* scratch, double* delta_out,
                                  double* delta_tmp, cplx* SLSE_RESTRICT rho, Blk& b) {
  if constexpr (U) return toeplitz_factor_regs_blk_u<Q>(c, n, scratch, delta_out, delta_tmp, rho, b);
  else return toeplitz_factor_regs_blk<Q>(c, n, scratch, delta_out, delta_tmp, rho, b);
}
#endif

#ifndef SLSE_LEV_BLK
#define SLSE_LEV_BLK 1  // register block Schur-Levinson for wide CTAs
#endif

SLSE_NI Factor toeplitz_factor(const cplx* SLSE_RESTRICT c, int n, cplx* e, cplx* B, cplx* a,
                              double* delta_out, double* delta_tmp, cplx* SLSE_RESTRICT rho, Blk& b) {
#ifndef SLSE_HOST_EMU
#ifndef SLSE_LEV_SMEM
#ifdef SLSE_LEV_UNROLLED
  if (b.nt == 32 && n <= 256) return toeplitz_factor_regs<8>(c, n, delta_out, delta_tmp, rho, b);
#else
  if (b.nt == 32 && n <= 256) return toeplitz_factor_regs_c<8>(c, n, delta_out, delta_tmp, rho, b);
#endif
#endif
  if (b.nt == 32 && __isShared(e) && __isShared(a)) {
    // e and B are adjacent (B == e + n) in every caller's shared-memory plan
    if (B == e + n && n <= 256) return toeplitz_factor_warp<8>(c, n, e, delta_out, delta_tmp, rho, b);
    if (B == e + n && n <= 512) return toeplitz_factor_warp<16>(c, n, e, delta_out, delta_tmp, rho, b);
  }
#if SLSE_LEV_BLK
  if (b.nt >= 64 && (b.nt & 31) == 0 && n >= 64) {  // (scratch: 2 + 2 nt / 32 elements of e)
    // the unrolled body needs the 128-register budget: not at 1024 threads
    const bool u = SLSE_LEV_BLK_UNROLL && b.nt <= 512;
    if (n <= 4 * b.nt) return u ? factor_regs_blk_ni<4, true>(c, n, e, delta_out, delta_tmp, rho, b)
                                : factor_regs_blk_ni<4, false>(c, n, e, delta_out, delta_tmp, rho, b);
    if (n <= 8 * b.nt) return u ? factor_regs_blk_ni<8, true>(c, n, e, delta_out, delta_tmp, rho, b)
                                : factor_regs_blk_ni<8, false>(c, n, e, delta_out, delta_tmp, rho, b);
  }
#endif
  if (__isShared(e)) return toeplitz_factor_impl<true>(c, n, e, B, a, delta_out, delta_tmp, rho, b);
#endif
  return toeplitz_factor_impl<false>(c, n, e, B, a, delta_out, delta_tmp, rho, b);
}

// ---------------------------------------------------------------------------
// Row 5: w = C^{-1} x = delta^{-1} (T1^H T1 x - T0 T0^H x) via FFTs of length
// nf = 2^ceil(log2 2N) (toeplitz.py:279-309).  All four kernel spectra derive from
// P1 = FFT(rho): with W = e^{-2 pi i/nf},
//   FFT(conj(rev rho))_k = W^{(N-1)k} conj(P1_k)
//   P0_k  = FFT(v0)_k    = W^k (P1_k - rho_{N-1} W^{(N-1)k}),  v0 = [0, rho_0..rho_{N-2}]
//   P0h_k = FFT(conj(rev v0))_k = W^{(N-1)k} conj(P0_k).
// Xhat = FFT_nf(x) is cached by the caller (x = y is fixed per problem).
// Buffers P, U, V: nf complex each (global).
#ifndef SLSE_GS_CHAIN2
#define SLSE_GS_CHAIN2 1
#endif
// One of GS apply's two independent chains: Y <- FFT(shift_{N-1}(IFFT(Y)) / nf)
// (U and V below; a CTA pair runs one each, slse_split.cuh).
SLSE_NI void gs_chain(cplx* Y, int n, int nf, const FftCtx& f, Blk& b) {
  const int tid_ = b.tid, nt_ = b.nt;
  const double inv = 1.0 / (double)nf;
  fft_inplace(Y, nf, 1.0, f, b);
  // shift down by N-1 through registers (barrier between read and write)
  for (int i0 = 0; i0 < nf; i0 += nt_) {
    const int i = i0 + tid_;
    cplx u = mk(0.0, 0.0);
    if (i < n) u = cscale(Y[n - 1 + i], inv);
    b.sync();
    if (i < nf) Y[i] = u;
    b.sync();
  }
  fft_inplace(Y, nf, -1.0, f, b);
}

// Both chains at once: the transforms of U and V batched (one barrier
// sequence for two transforms in flight).
SLSE_NI void gs_chain2(cplx* U, cplx* V, cplx* work, int n, int nf, const FftCtx& f, Blk& b) {
  const int tid_ = b.tid, nt_ = b.nt;
  const double inv = 1.0 / (double)nf;
  fft_multi(work, 2, nf, 1.0, [=](int c, int i) { return c ? V[i] : U[i]; },
            [=](int c, int i, cplx v) { (c ? V : U)[i] = v; }, f, b);
  for (int i0 = 0; i0 < nf; i0 += nt_) {
    const int i = i0 + tid_;
    cplx u = mk(0.0, 0.0), v = mk(0.0, 0.0);
    if (i < n) { u = cscale(U[n - 1 + i], inv); v = cscale(V[n - 1 + i], inv); }
    b.sync();
    if (i < nf) { U[i] = u; V[i] = v; }
    b.sync();
  }
  fft_multi(work, 2, nf, -1.0, [=](int c, int i) { return c ? V[i] : U[i]; },
            [=](int c, int i, cplx v) { (c ? V : U)[i] = v; }, f, b);
}

SLSE_NI double gs_apply(const cplx* SLSE_RESTRICT rho, int n, double delta_last,
                       const cplx* SLSE_RESTRICT x, const cplx* SLSE_RESTRICT Xhat, cplx* P, cplx* U,
                       cplx* V, cplx* SLSE_RESTRICT w, const FftCtx& f, Blk& b, Split* sp = nullptr) {
  const int tid_ = b.tid, nt_ = b.nt;
  const int lg = ilog2(2 * n);  // nf = next power of two >= 2N
  const int nf = 1 << lg;
  const cplx rlast = rho[n - 1];
  // P = FFT(rho zero-padded)
  fft(P, nf, -1.0,
      [=](int i) { return i < n ? rho[i] : mk(0.0, 0.0); },
      [=](int i, cplx v) { P[i] = v; }, f, b);
  // U = Xhat * P1 ; V = Xhat * P0h
  for (int k = tid_; k < nf; k += nt_) {
    const cplx p1 = P[k];
    const cplx wk = twid(f, k, lg, -1.0);
    const cplx wn1 = twid(f, (int)(((long long)(n - 1) * k) & (nf - 1)), lg, -1.0);
    const cplx p0 = cmul(wk, csub(p1, cmul(rlast, wn1)));
    const cplx p0h = cmul(wn1, conjg(p0));
    const cplx xk = Xhat[k];
    U[k] = cmul(xk, p1);
    V[k] = cmul(xk, p0h);
  }
  b.sync();
  const double inv = 1.0 / (double)nf;
  // t1x = IFFT(U)[N-1 : 2N-1] and t0hx = IFFT(V)[N-1 : 2N-1], zero padded,
  // transformed back: two independent chains
  if (SLSE_PAIR && sp) {
    GsChainArgs a{V, n, nf};
    SplitJob j;
    j.set(kJobGsChain, a);
    sp->post(j, b);
    gs_chain(U, n, nf, f, b);
    sp->done();
  } else if (SLSE_GS_CHAIN2 && 2 * nf <= f.smem_cap) {
    gs_chain2(U, V, nullptr, n, nf, f, b);
  } else {
    gs_chain(U, n, nf, f, b);
    gs_chain(V, n, nf, f, b);
  }
  // Z = F1 * P1h - F0 * P0  -> U
  for (int k = tid_; k < nf; k += nt_) {
    const cplx p1 = P[k];
    const cplx wk = twid(f, k, lg, -1.0);
    const cplx wn1 = twid(f, (int)(((long long)(n - 1) * k) & (nf - 1)), lg, -1.0);
    const cplx p1h = cmul(wn1, conjg(p1));
    const cplx p0 = cmul(wk, csub(p1, cmul(rlast, wn1)));
    U[k] = csub(cmul(U[k], p1h), cmul(V[k], p0));
  }
  b.sync();
  const double sc = inv / delta_last;
  double quad = 0.0;
  fft_inplace(U, nf, 1.0, f, b);
  for (int i = tid_; i < n; i += nt_) {
    const cplx wi = cscale(U[i], sc);
    w[i] = wi;
    quad += x[i].re * wi.re + x[i].im * wi.im;  // Re(conj(x) w)
  }
  return b.sum(quad);
}

#ifndef SLSE_WARP_FFT_R8
#define SLSE_WARP_FFT_R8 1  // radix-8 passes (cfg2 36.5 -> 32.2 ms: the warp-mode FFTs are shared-memory bound)
#endif
#ifndef SLSE_HOST_EMU
// Runtime-size one-warp Stockham pass of radix R over 2^lg <= 512 points
// (MAXI = 16 / R groups per lane held across the warp barrier, in place).
template <int R>
SLSE_D void warp_pass_rt(cplx* S, int lg, int lgns, double sign, const cplx* __restrict__ tw, int twlog,
                         unsigned lane) {
  constexpr int MAXI = 16 / R;
  const unsigned per = (1u << lg) / R, NS = 1u << lgns;
  const int lgt = lgns + ilog2(R);
  cplx v[MAXI][R];
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const unsigned j = lane + 32u * i;
    if (j < per) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = S[sk(j + r * per)];
      if (NS > 1) {
        const unsigned kk = j & (NS - 1);
        const cplx w1 = twid_tab(tw, twlog, kk, lgt, sign);
        v[i][1] = cmul(v[i][1], w1);
        if constexpr (R >= 4) {
          const cplx w2 = cmul(w1, w1);
          v[i][2] = cmul(v[i][2], w2);
          const cplx w3 = cmul(w2, w1);
          v[i][3] = cmul(v[i][3], w3);
          if constexpr (R == 8) {
            const cplx w4 = cmul(w2, w2);
            v[i][4] = cmul(v[i][4], w4);
            v[i][5] = cmul(v[i][5], cmul(w4, w1));
            v[i][6] = cmul(v[i][6], cmul(w4, w2));
            v[i][7] = cmul(v[i][7], cmul(w4, w3));
          }
        }
      }
      dft_dif<R>(v[i], sign);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const unsigned j = lane + 32u * i;
    if (j < per) {
      const unsigned kk = j & (NS - 1);
      const unsigned base = (j - kk) * R + kk;
#pragma unroll
      for (int r = 0; r < R; ++r) S[sk(base + r * NS)] = v[i][brev_const(r, R)];
    }
  }
  __syncwarp();
}

// One-warp in-place transform of 2^lg (<= 512) points on the skewed shared
// buffer S: radix-8 passes, then radix-4 / radix-2 for the remainder.  One
// compact out-of-line body for every size and direction.  In warp mode the
// sixteen warps of an SM run their transforms together, so the passes are
// bound by shared-memory bandwidth (every pass moves every point twice):
// 3 radix-8 passes for 512 points beat 5 radix-4 ones (cfg2 36.5 -> 32.2 ms,
// tools/r8_exp.sh), although the body is larger (the free-running solver
// once measured the opposite, from instruction fetch).
static __device__ __noinline__ void warp_fft_rt(cplx* S, int lg, double sign, const cplx* __restrict__ tw, int twlog,
                                         int lane_) {
  __builtin_assume(__isShared(S));
  const unsigned lane = (unsigned)lane_ & 31u;
  int lgns = 0;
#if SLSE_WARP_FFT_R8
  // radix-8 passes first: 3 shared-memory round trips for 512 points instead of 5
#pragma unroll 1
  for (; lg - lgns >= 3; lgns += 3) warp_pass_rt<8>(S, lg, lgns, sign, tw, twlog, lane);
#endif
#pragma unroll 1
  for (; lg - lgns >= 2; lgns += 2) warp_pass_rt<4>(S, lg, lgns, sign, tw, twlog, lane);
  if (lg - lgns == 1) warp_pass_rt<2>(S, lg, lgns, sign, tw, twlog, lane);
}

// IFFT, keep [N-1, 2N-1) scaled by 1/nf, zero pad, FFT (the middle of a GS
// product), in place on S.
static __device__ __noinline__ void warp_gs_middle(cplx* S, int n, int lg, const cplx* __restrict__ tw, int twlog,
                                            int lane) {
  __builtin_assume(__isShared(S));
  const int nf = 1 << lg;
  warp_fft_rt(S, lg, 1.0, tw, twlog, lane);
  const double inv = 1.0 / (double)nf;
  cplx hold[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int i = lane + 32 * t;
    hold[t] = i < n ? cscale(S[sk(n - 1 + i)], inv) : mk(0.0, 0.0);
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int i = lane + 32 * t;
    if (i < nf) S[sk(i)] = hold[t];
  }
  __syncwarp();
  warp_fft_rt(S, lg, -1.0, tw, twlog, lane);
}

// One-warp GS apply (N <= 256 solver path): the same six transforms as
// gs_apply, each an in-place warp Stockham on ONE skewed shared-memory
// buffer S; the spectra that must survive a transform (P = FFT(rho), the
// V chain input, the partial Z) go to the global work arrays P, V, U in
// coalesced passes.
static __device__ __noinline__ double gs_apply_warp(const cplx* SLSE_RESTRICT rho, int n, int lg, double delta_last,
                                             const cplx* SLSE_RESTRICT x, const cplx* SLSE_RESTRICT Xhat,
                                             cplx* SLSE_RESTRICT P, cplx* SLSE_RESTRICT U, cplx* SLSE_RESTRICT V,
                                             cplx* SLSE_RESTRICT w, cplx* S, const cplx* __restrict__ tw, int twlog,
                                             int lane) {
  const int nf = 1 << lg;
  __builtin_assume(__isShared(S));
  const cplx z = mk(0.0, 0.0);
  const cplx rlast = rho[n - 1];
  // P = FFT(rho zero-padded)
#pragma unroll 1
  for (int i = lane; i < nf; i += 32) S[sk(i)] = i < n ? rho[i] : z;
  __syncwarp();
  warp_fft_rt(S, lg, -1.0, tw, twlog, lane);
  // P -> global; U = Xhat P1 -> S; V = Xhat P0h -> global
#pragma unroll 1
  for (int k = lane; k < nf; k += 32) {
    const cplx p1 = S[sk(k)];
    const cplx wk = twid_tab(tw, twlog, k, lg, -1.0);
    const cplx wn1 = twid_tab(tw, twlog, (int)(((long long)(n - 1) * k) & (nf - 1)), lg, -1.0);
    const cplx p0 = cmul(wk, csub(p1, cmul(rlast, wn1)));
    const cplx p0h = cmul(wn1, conjg(p0));
    const cplx xk = Xhat[k];
    P[k] = p1;
    S[sk(k)] = cmul(xk, p1);
    V[k] = cmul(xk, p0h);
  }
  __syncwarp();
  // U chain; Z = U'' P1h -> global U; V -> S
  warp_gs_middle(S, n, lg, tw, twlog, lane);
#pragma unroll 1
  for (int k = lane; k < nf; k += 32) {
    const cplx wn1 = twid_tab(tw, twlog, (int)(((long long)(n - 1) * k) & (nf - 1)), lg, -1.0);
    const cplx p1h = cmul(wn1, conjg(P[k]));
    U[k] = cmul(S[sk(k)], p1h);
    S[sk(k)] = V[k];
  }
  __syncwarp();
  // V chain, then Z = U'' P1h - V'' P0 -> S, IFFT
  warp_gs_middle(S, n, lg, tw, twlog, lane);
#pragma unroll 1
  for (int k = lane; k < nf; k += 32) {
    const cplx p1 = P[k];
    const cplx wk = twid_tab(tw, twlog, k, lg, -1.0);
    const cplx wn1 = twid_tab(tw, twlog, (int)(((long long)(n - 1) * k) & (nf - 1)), lg, -1.0);
    const cplx p0 = cmul(wk, csub(p1, cmul(rlast, wn1)));
    S[sk(k)] = csub(U[k], cmul(S[sk(k)], p0));
  }
  __syncwarp();
  warp_fft_rt(S, lg, 1.0, tw, twlog, lane);
  const double sc = 1.0 / ((double)nf * delta_last);
  double quad = 0.0;
#pragma unroll 1
  for (int i = lane; i < n; i += 32) {
    const cplx wi = cscale(S[sk(i)], sc);
    w[i] = wi;
    quad += x[i].re * wi.re + x[i].im * wi.im;  // Re(conj(x) w)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) quad += __shfl_xor_sync(0xffffffffu, quad, o);
  __syncwarp();
  return quad;
}
#endif

// GS apply dispatch: the one-warp shared-memory version for 2N in [64, 512]
// when the staging fits, else the general block version.
SLSE_NI double gs_apply_any(const cplx* SLSE_RESTRICT rho, int n, double delta_last, const cplx* SLSE_RESTRICT x,
                           const cplx* SLSE_RESTRICT Xhat, cplx* P, cplx* U, cplx* V, cplx* SLSE_RESTRICT w,
                           const FftCtx& f, Blk& b, Split* sp = nullptr) {
#if !defined(SLSE_HOST_EMU) && !defined(SLSE_GS_BLOCK)
  if (b.nt == 32 && __isShared(f.smem)) {
    const int lg = ilog2(2 * n);
    if (sk_len(1 << lg) <= f.smem_cap) {
      if (lg >= 5 && lg <= 9) return gs_apply_warp(rho, n, lg, delta_last, x, Xhat, P, U, V, w, f.smem, f.tw, f.twlog, b.tid);
    }
  }
#endif
  return gs_apply(rho, n, delta_last, x, Xhat, P, U, V, w, f, b, sp);
}

}  // namespace slse
