// slse_grid3.cuh -- Row 9 coefficient form for the large grids (L >= 4096,
// N <= L / 4: BASELINE cfg3 / cfg4 / cfg5 shapes): register transforms of
// 4096 points, three DFT16 passes, two in-place shared-memory exchanges.
//
// Reference: _SuperfastBundle.grid (pkg/src/superlse/model_core.py:303-313):
//   q^G = FFT_L(w),  s^G = L IFFT_L(buf).real,  buf[i mod L] = om_s(i);
// with d_0 = om_s(0), d_k = 2 om_s(k):  s^G = Re FFT_L(conj d)  (slse_grid.cuh).
//
// With L = R M (M = 4096) and l = r + R m the L-point transform of an
// N <= L / 4 point signal is R independent M-point transforms
//   X[r + R m] = sum_{i<M} z_r(i) W_M^{i m},
//   z_r(i)     = W_L^{i r} sum_{j : i + j M < N} x_{i + j M} W_R^{j r}.
// One task = (problem, signal, residue); tasks are problem-major so the R
// residue tasks that interleave into one problem's output rows run at the
// same time on neighbouring CTAs and their partial sectors merge in L2.
//   R = 1  (cfg3, N <= 1024): z = x, zero past M / 4: the first pass is four
//          radix-4 butterflies per thread (pruned DFT16);
//   R = 4  (cfg4, N <= 4096): z_r(i) = W_L^{i r} x_i, no fold;
//   R = 16 (cfg5, N <= 16384): four folds.
//
// The M-point transform, i = n0 + 16 n1 + 256 n2, m = k0 + 16 k1 + 256 k2:
//   pass A  thread (n0, n1): DFT16 over n2            -> A(n0, n1, k0)
//   pass B  thread (n0, k0): W256^{n1 k0}, DFT16 over n1 -> B(n0, k0, k1)
//   pass C  thread (k0, k1): W4096^{n0 (k0 + 16 k1)}, DFT16 over n0 -> X[tid + 256 k2]
// so the loads (i = tid + 256 n2) and the stores (m = tid + 256 k2) are
// coalesced, 16 bytes per lane.  256 threads; every thread holds 16 points.
//
// Exchanges are in place in ONE 4368-complex buffer (69.9 KB: three CTAs per
// SM), slot (p, q, x) = p sP + q sQ + x:
//   A writes (k0, n0, n1);  B reads (k0, n0, *) and overwrites its own 16
//   slots with its outputs (k0, n0, k1);  C reads (k0, *, k1);
// the NEXT task's pass A of the same thread then writes exactly the slots
// its pass C read, if the next task swaps sP and sQ.  Two barriers per task
// (after the A stores, after the B stores), none between tasks.  sP, sQ are
// 273 and 17, both = 1 mod 8, so every quarter-warp
// (8 lanes, consecutive n0 or k0) touches 8 different 16-byte bank groups in
// all six access patterns.
#pragma once
#include "slse_grid.cuh"

namespace slse_k {

constexpr int kR3Threads = 256;
constexpr int kR3StrideHi = 273, kR3StrideLo = 17;
constexpr int kR3Buf = 16 * kR3StrideHi;  // 4368 complex
SLSE_HD constexpr size_t r3_smem_bytes() { return 16 * (size_t)kR3Buf; }
#ifndef SLSE_R3_MINB
#define SLSE_R3_MINB 3
#endif

// pruned DFT16: inputs x0..x3 at n2 = 0..3, zero beyond; A[r + 4 k] for the
// residue R16 = r: one radix-4 of the inputs pre-twiddled by W16^{n2 r}
template <int R16>
SLSE_D void r3_pruned4(const cplx* x, cplx* v) {
  cplx a = x[0], b = x[1], c = x[2], d = x[3];
  g5_r4<4 * R16, 8 * R16, 12 * R16>(a, b, c, d);
  v[R16] = a;
  v[R16 + 4] = b;
  v[R16 + 8] = c;
  v[R16 + 12] = d;
}

// v[t] *= base * step^t, t = 0..15 (two interleaved chains)
SLSE_D void r3_chain_twiddles(cplx* v, cplx base, cplx step) {
  const cplx step2 = cmul(step, step);
  cplx pe = base, po = cmul(base, step);
  v[0] = cmul(v[0], pe);
  v[1] = cmul(v[1], po);
#pragma unroll
  for (int t = 2; t < 16; t += 2) {
    pe = cmul(pe, step2);
    po = cmul(po, step2);
    v[t] = cmul(v[t], pe);
    v[t + 1] = cmul(v[t + 1], po);
  }
}

// MODE 0: R = 1 pruned (N <= 1024);  MODE 1: R >= 4, J = R / 4 folds
template <int MODE>
__global__ void __launch_bounds__(kR3Threads, SLSE_R3_MINB) grid_r3_kernel(const cplx* __restrict__ w,
                                                                          const cplx* __restrict__ om_s, int n,
                                                                          int lgL, int B, cplx* __restrict__ q_grid,
                                                                          double* __restrict__ s_grid,
                                                                          const cplx* __restrict__ tw) {
  constexpr int M = 4096;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* X = (cplx*)smem_raw;
  const int tid = threadIdx.x;
  const int a = tid & 15, b = tid >> 4;
  const int lgR = lgL - 12;
  const int R = 1 << lgR;
  const size_t L = (size_t)1 << lgL;
  const long long T = ((long long)B * 2) << lgR;
  const size_t om_stride = 2 * (size_t)n - 1;
  const int J = (n + M - 1) >> 12;
  // fixed per thread: pass B twiddle step W256^{b}, pass C step W4096^{tid}
  const cplx* twb = tw + tw_index(b, 8);
  const cplx* twc = tw + tw_index(tid, 12);
  int sP = kR3StrideHi, sQ = kR3StrideLo;

  for (long long task = blockIdx.x; task < T; task += gridDim.x) {
    const int r = (int)(task & (R - 1));
    const int sig = (int)(task >> lgR) & 1;
    const int p = (int)(task >> (lgR + 1));
    const cplx* src = sig ? om_s + (size_t)p * om_stride + (n - 1) : w + (size_t)p * n;
    cplx v[16];
    // ---- pass A
    // signal 1 is conj d, d_0 = om_s(0), d_m = 2 om_s(m)
    const auto ld = [&](int m) {
      cplx xv = m < n ? ldg_c(src + m) : mk(0.0, 0.0);
      if (sig) {
        const double f = m ? 2.0 : 1.0;
        xv = mk(f * xv.re, -f * xv.im);
      }
      return xv;
    };
    if (MODE == 0) {
      cplx x[4];
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2) x[n2] = ld(tid + 256 * n2);
      r3_pruned4<0>(x, v);
      r3_pruned4<1>(x, v);
      r3_pruned4<2>(x, v);
      r3_pruned4<3>(x, v);
      // v[k0] = A(k0)
#pragma unroll
      for (int k0 = 0; k0 < 16; ++k0) X[k0 * sP + a * sQ + b] = v[k0];
    } else {
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) v[n2] = ld(tid + 256 * n2);
      for (int j = 1; j < J; ++j) {
        const cplx t = ldg_c(tw + tw_index((j * r) & (R - 1), lgR));  // W_R^{j r}
#pragma unroll
        for (int n2 = 0; n2 < 16; ++n2) v[n2] = cadd(v[n2], cmul(ld(tid + 256 * n2 + (j << 12)), t));
      }
      if (r) {
        // W_L^{(tid + 256 n2) r} = W_L^{tid r} (W_{L/256}^{r})^{n2}
        const cplx base = ldg_c(tw + tw_index(tid * r, lgL));
        const cplx step = ldg_c(tw + tw_index(r, lgL - 8));
        r3_chain_twiddles(v, base, step);
      }
      dft16_t<0>(v);
#pragma unroll
      for (int k0 = 0; k0 < 16; ++k0) X[k0 * sP + a * sQ + b] = v[g5_pos(k0)];
    }
    __syncthreads();
    // ---- pass B: thread (n0 = a, k0 = b)
    {
      cplx* row = X + b * sP + a * sQ;
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = row[n1];
      g5_outer_twiddles(v, twb, b);
      dft16_t<0>(v);
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) row[k1] = v[g5_pos(k1)];
    }
    __syncthreads();
    // ---- pass C: thread (k0 = a, k1 = b)
    {
      const cplx* col = X + a * sP + b;
#pragma unroll
      for (int n0 = 0; n0 < 16; ++n0) v[n0] = col[n0 * sQ];
    }
    g5_outer_twiddles(v, twc, tid);
    dft16_t<0>(v);
    if (sig == 0) {
      double2* qg = (double2*)(q_grid + (size_t)p * L) + r + ((size_t)tid << lgR);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const cplx o = v[g5_pos(k2)];
        __stcs(&qg[(size_t)(256 * k2) << lgR], make_double2(o.re, o.im));
      }
    } else {
      double* sg = s_grid + (size_t)p * L + r + ((size_t)tid << lgR);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) __stcs(&sg[(size_t)(256 * k2) << lgR], v[g5_pos(k2)].re);
    }
    const int tmp = sP;
    sP = sQ;
    sQ = tmp;
  }
}

}  // namespace slse_k
