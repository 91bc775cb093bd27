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
// Three kernels share the transform below:
//   grid_r3c_kernel  L = 4096, N <= 1024 (cfg3): R = 1, z = x, zero past
//                    M / 4: the first pass is four radix-4 butterflies per
//                    thread (pruned DFT16); s^G of TWO problems per transform;
//   grid_r3s_kernel  L >= 16384, N <= L / 4 (cfg4, cfg5): tasks are residue
//                    PAIRS stored as whole 32-byte sectors, s^G at half length;
//   grid_r3_kernel   every other L >= 4096 shape: one (problem, signal,
//                    residue) per task, dense input, J = ceil(N / M) folds.
//
// The M-point transform, i = n0 + 16 n1 + 256 n2, m = k0 + 16 k1 + 256 k2:
//   pass A  thread (n0, n1): DFT16 over n2            -> A(n0, n1, k0)
//   pass B  thread (n0, k0): W256^{n1 k0}, DFT16 over n1 -> B(n0, k0, k1)
//   pass C  thread (k0, k1): W4096^{n0 (k0 + 16 k1)}, DFT16 over n0 -> X[tid + 256 k2]
// so the loads (i = tid + 256 n2) and the stores (m = tid + 256 k2) are
// coalesced, 16 bytes per lane.  256 threads; every thread holds 16 points.
//
// Exchanges are in place in ONE 4368-complex buffer (69.9 KB), slot (p, q, x) = p sP + q sQ + x:
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
#define SLSE_R3_MINB 2  // 128 registers: 3 CTAs at 80 registers spill (cfg3 shape 0.48 vs 0.585 of HBM)
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

// v[t] *= w^t, t = 1..15, from w and w^2 (two interleaved chains)
SLSE_D void r3_pow_twiddles(cplx* v, cplx wa, cplx wa2) {
  cplx pe = wa2, po = wa;
  v[1] = cmul(v[1], wa);
#pragma unroll
  for (int tt = 2; tt < 16; tt += 2) {
    if (tt > 2) pe = cmul(pe, wa2);
    po = cmul(po, wa2);
    v[tt] = cmul(v[tt], pe);
    v[tt + 1] = cmul(v[tt + 1], po);
  }
}

// Residue pre-twiddle W_Le^{i r}, i = n0 + 16 n1 + 256 n2, folded into the
// three passes at no per-element cost:
//   n2: (W_{Le/256}^r)^{n2} is W64^{n2 e}, e = 16384 r / Le, whenever that is
//       an integer below 4 (every cfg4 task, a quarter of cfg5's): dft16_t<e>
//       carries it in its compile-time twiddles; otherwise a chain;
//   n1: (W_{Le/16}^r)^{n1} joins pass B's chain: its step W256^{k0} is
//       multiplied by W_{Le/16}^r once;
//   n0: (W_Le^r)^{n0} joins pass C's chain the same way.
SLSE_D void r3_pass_a_dft(cplx* v, int r, int lgLe, const cplx* __restrict__ tw) {
  const int num = r << 14;
  const int e = num >> lgLe;
  if ((num & ((1 << lgLe) - 1)) == 0 && e < 4) {
    switch (e) {
      case 0: dft16_t<0>(v); break;
      case 1: dft16_t<1>(v); break;
      case 2: dft16_t<2>(v); break;
      default: dft16_t<3>(v); break;
    }
  } else {
    const cplx step = ldg_c(tw + tw_index(r, lgLe - 8));
    r3_pow_twiddles(v, step, cmul(step, step));
    dft16_t<0>(v);
  }
}

// Streaming (evict-first) stores only when a task writes whole lines (R = 1):
// with R > 1 a line is completed by the R residue tasks of its problem, and
// an evict-first partial line leaves L2 before they arrive.
template <typename V>
SLSE_D void r3_store(V* p, V x, int lgR) {
  if (lgR == 0) __stcs(p, x);
  else *p = x;
}

// Dense single-residue tasks: any N <= L, L >= 4096 (the shapes the pruned
// and the pair kernels below do not take: N > L / 4, or L = 4096 / 8192 with
// N > 1024).  J = ceil(N / 4096) folds.  Two CTAs per SM at 128 registers
// (three at 80 registers spill).  The two table entries of each pass's
// twiddle chain are loaded before the barrier that precedes the pass.
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
  // fixed per thread: pass B twiddles (W256^{b})^t, pass C twiddles (W4096^{tid})^t
  const cplx* twb = tw + tw_index(b, 8);
  const cplx* twc = tw + tw_index(tid, 12);
  int sP = kR3StrideHi, sQ = kR3StrideLo;

  for (long long task = blockIdx.x; task < T; task += gridDim.x) {
    const int r = (int)(task & (R - 1));
    const int sig = (int)(task >> lgR) & 1;
    const int p = (int)(task >> (lgR + 1));
    const cplx* src = sig ? om_s + (size_t)p * om_stride + (n - 1) : w + (size_t)p * n;
    cplx v[16];
    // ---- pass A; signal 1 is conj d, d_0 = om_s(0), d_m = 2 om_s(m)
    const auto ld = [&](int m) {
      cplx xv = m < n ? ldg_c(src + m) : mk(0.0, 0.0);
      if (sig) {
        const double f = m ? 2.0 : 1.0;
        xv = mk(f * xv.re, -f * xv.im);
      }
      return xv;
    };
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = ld(tid + 256 * n2);
    for (int j = 1; j < J; ++j) {
      const cplx t = ldg_c(tw + tw_index((j * r) & (R - 1), lgR));  // W_R^{j r}
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) v[n2] = cadd(v[n2], cmul(ld(tid + 256 * n2 + (j << 12)), t));
    }
    r3_pass_a_dft(v, r, lgL, tw);
#pragma unroll
    for (int k0 = 0; k0 < 16; ++k0) X[k0 * sP + a * sQ + b] = v[g5_pos(k0)];
    cplx wb1 = ldg_c(twb), wb2 = ldg_c(twb + b);
    if (r) {  // the residue pre-twiddle's n1 part (r3_pass_a_dft)
      wb1 = cmul(wb1, ldg_c(tw + tw_index(r, lgL - 4)));
      wb2 = cmul(wb1, wb1);
    }
    __syncthreads();
    // ---- pass B: thread (n0 = a, k0 = b)
    {
      cplx* row = X + b * sP + a * sQ;
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = row[n1];
      r3_pow_twiddles(v, wb1, wb2);
      dft16_t<0>(v);
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) row[k1] = v[g5_pos(k1)];
    }
    cplx wc1 = ldg_c(twc), wc2 = ldg_c(twc + tid);
    if (r) {
      wc1 = cmul(wc1, ldg_c(tw + tw_index(r, lgL)));
      wc2 = cmul(wc1, wc1);
    }
    __syncthreads();
    // ---- pass C: thread (k0 = a, k1 = b)
    {
      const cplx* col = X + a * sP + b;
#pragma unroll
      for (int n0 = 0; n0 < 16; ++n0) v[n0] = col[n0 * sQ];
    }
    r3_pow_twiddles(v, wc1, wc2);
    dft16_t<0>(v);
    if (sig == 0) {
      double2* qg = (double2*)(q_grid + (size_t)p * L) + r + ((size_t)tid << lgR);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const cplx o = v[g5_pos(k2)];
        r3_store(&qg[(size_t)(256 * k2) << lgR], make_double2(o.re, o.im), lgR);
      }
    } else {
      double* sg = s_grid + (size_t)p * L + r + ((size_t)tid << lgR);
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) r3_store(&sg[(size_t)(256 * k2) << lgR], v[g5_pos(k2)].re, lgR);
    }
    const int tmp = sP;
    sP = sQ;
    sQ = tmp;
  }
}

// L2 prefetch of `bytes` (multiple of 16) at a 16-byte aligned address
SLSE_D void r3_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// ---------------------------------------------------------------------------
// cfg3 shape (L = 4096, N <= 1024), s^G of TWO problems in one transform.
// With h_k = conj om_s(k) for all |k| < N (om_s Hermitian), s^G = FFT_L(h) is
// real, so for problems p0, p1
//   FFT_L(h^{p0} + i h^{p1})[l] = s^{p0}_l + i s^{p1}_l :
// three tasks per problem pair (q^G of p0, q^G of p1, the shared s^G) instead
// of four.  The input c = h^{p0} + i h^{p1} is two-sided: c[k] = conj om^{p0}(k)
// + i conj om^{p1}(k) for 0 <= k < N and c[L - k] = om^{p0}(k) + i om^{p1}(k)
// for 0 < k < N, i.e. i = tid + 256 n2 is non-zero for n2 in {0..3} and
// {12..15} = {n2a - 4}: the pruned pass A folds the second group in with the
// trivial factor W16^{-4 k0} = i^{k0} before its radix-4 butterflies.
// The q^G tasks are grid_r3_kernel<0>'s (inputs prefetched into registers).
__global__ void __launch_bounds__(kR3Threads, 2) grid_r3c_kernel(const cplx* __restrict__ w,
                                                                 const cplx* __restrict__ om_s, int n, int B,
                                                                 cplx* __restrict__ q_grid, double* __restrict__ s_grid,
                                                                 const cplx* __restrict__ tw) {
  constexpr int L = 4096;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* X = (cplx*)smem_raw;
  const int tid = threadIdx.x;
  const int a = tid & 15, b = tid >> 4;
  const int T = 3 * ((B + 1) >> 1);
  const size_t om_stride = 2 * (size_t)n - 1;
  const cplx* twb = tw + tw_index(b, 8);
  const cplx* twc = tw + tw_index(tid, 12);
  const cplx wb1 = ldg_c(twb), wb2 = ldg_c(twb + b), wc1 = ldg_c(twc), wc2 = ldg_c(twc + tid);
  int sP = kR3StrideHi, sQ = kR3StrideLo;
  cplx xn[4];  // the next q^G task's inputs
  const auto prefetch = [&](int task) {
    const int role = task % 3, p = 2 * (task / 3) + role;
    if (task < T && role < 2 && p < B) {
      const cplx* src = w + (size_t)p * n;
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2) xn[n2] = tid + 256 * n2 < n ? ldg_c(src + tid + 256 * n2) : mk(0.0, 0.0);
    } else if (task < T && role == 2 && tid < 2 && p - 2 + tid < B) {
      // the s^G task's two om_s half rows towards L2 (its 16 loads per thread are not prefetched)
      r3_prefetch_l2(om_s + (size_t)(p - 2 + tid) * om_stride + (n - 1), 16u * (unsigned)n);
    }
  };
  prefetch(blockIdx.x);

  for (int task = blockIdx.x; task < T; task += gridDim.x) {
    const int role = task % 3, p0 = 2 * (task / 3);
    const int p = role < 2 ? p0 + role : p0;
    if (p >= B) {  // odd batch: the last pair has no second q^G task
      prefetch(task + gridDim.x);
      continue;
    }
    cplx v[16];
    if (role < 2) {
      r3_pruned4<0>(xn, v);
      r3_pruned4<1>(xn, v);
      r3_pruned4<2>(xn, v);
      r3_pruned4<3>(xn, v);
    } else {
      const bool two = p0 + 1 < B;
      const cplx* o0 = om_s + (size_t)p0 * om_stride + (n - 1);
      const cplx* o1 = o0 + (two ? om_stride : 0);
      const double f1 = two ? 1.0 : 0.0;
      cplx xp[4], xm[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kp = tid + 256 * j;        // i = kp            (n2 = j)
        const int km = 256 * (4 - j) - tid;  // i = L - km        (n2 = 12 + j)
        const cplx a0 = kp < n ? ldg_c(o0 + kp) : mk(0.0, 0.0), a1 = kp < n ? ldg_c(o1 + kp) : mk(0.0, 0.0);
        const cplx b0 = km < n ? ldg_c(o0 + km) : mk(0.0, 0.0), b1 = km < n ? ldg_c(o1 + km) : mk(0.0, 0.0);
        xp[j] = mk(a0.re + f1 * a1.im, f1 * a1.re - a0.im);  // conj a0 + i conj a1
        xm[j] = mk(b0.re - f1 * b1.im, b0.im + f1 * b1.re);  // b0 + i b1
      }
      cplx y[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = cadd(xp[j], xm[j]);
      r3_pruned4<0>(y, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = mk(xp[j].re - xm[j].im, xp[j].im + xm[j].re);  // + i xm
      r3_pruned4<1>(y, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = csub(xp[j], xm[j]);
      r3_pruned4<2>(y, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = mk(xp[j].re + xm[j].im, xp[j].im - xm[j].re);  // - i xm
      r3_pruned4<3>(y, v);
    }
#pragma unroll
    for (int k0 = 0; k0 < 16; ++k0) X[k0 * sP + a * sQ + b] = v[k0];
    prefetch(task + gridDim.x);
    __syncthreads();
    {
      cplx* row = X + b * sP + a * sQ;
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = row[n1];
      r3_pow_twiddles(v, wb1, wb2);
      dft16_t<0>(v);
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) row[k1] = v[g5_pos(k1)];
    }
    __syncthreads();
    {
      const cplx* col = X + a * sP + b;
#pragma unroll
      for (int n0 = 0; n0 < 16; ++n0) v[n0] = col[n0 * sQ];
    }
    r3_pow_twiddles(v, wc1, wc2);
    dft16_t<0>(v);
    if (role < 2) {
      double2* qg = (double2*)(q_grid + (size_t)p * L) + tid;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const cplx o = v[g5_pos(k2)];
        __stcs(&qg[256 * k2], make_double2(o.re, o.im));
      }
    } else {
      double* s0 = s_grid + (size_t)p0 * L + tid;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) __stcs(&s0[256 * k2], v[g5_pos(k2)].re);
      if (p0 + 1 < B) {
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) __stcs(&s0[L + 256 * k2], v[g5_pos(k2)].im);
      }
    }
    const int tmp = sP;
    sP = sQ;
    sQ = tmp;
  }
}

// ---------------------------------------------------------------------------
// Residue PAIRS for L >= 16384, N <= L / 4 (cfg4 / cfg5 shapes).  A residue
// task above writes 16-byte (q^G) or 8-byte (s^G) pieces at stride 16 R
// bytes: partial 32-byte sectors.  Every partial piece costs a whole sector
// on the SM -> L2 path and a sector operation in L2, and L2 completes evicted
// partial sectors by read-modify-write against DRAM (ncu at the cfg4 shape:
// DRAM reads 4.3x, writes 1.7x the algorithmic bytes).  Here one task is a
// PAIR of residues r = 2 pair, r + 1 of a problem, and every store is one
// whole 32-byte sector (bins r, r + 1 of one m; STG.256).
//
// s^G additionally runs at HALF length: with h_k = conj om_s(k) (all |k| < N)
//   s_l = sum_k h_k W_L^{k l},   z_m = s_{2m} + i s_{2m+1} = FFT_{L/2}(g)[m],
//   g[k mod L/2] = h_k (1 + i W_L^k),
// (2N - 1 <= L / 2, no aliasing), a complex transform of L / 2 points whose
// output IS the s^G row (re, im interleaved = consecutive doubles): R / 4
// pair tasks instead of R / 2, their 32-byte pieces at stride 16 R bytes
// like q^G's pairs (contiguous rows at cfg4, where R / 2 = 2).
//
// The pair runs SEQUENTIALLY in one 256-thread CTA: residue r, whose 16
// outputs per thread are parked (10 in shared memory, 6 in registers), then
// residue r + 1, then the stores.  Two CTAs per SM (110.8 KB each) overlap
// each other's barriers and loads.  (A lock-step variant -- 512 threads,
// lanes 0-15 / 16-31 of every warp on the two residues, outputs paired by
// shuffle -- measured the same 0.28 of HBM at the cfg4 shape as this one
// before the 32-byte stores, with one CTA per SM and nothing to overlap its
// load latency; removed.)
// one 32-byte store (sm_100: STG.256), p 32-byte aligned
SLSE_D void r3_store32(double2* p, cplx lo, cplx hi) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(lo.re), "d"(lo.im), "d"(hi.re), "d"(hi.im)
               : "memory");
}
#ifndef SLSE_R3_L2PF
#define SLSE_R3_L2PF 1
#endif
#ifndef SLSE_R3_SAVE_SMEM
#define SLSE_R3_SAVE_SMEM 10
#endif
constexpr int kR3SaveSmem = SLSE_R3_SAVE_SMEM;  // outputs per thread parked in shared memory
SLSE_HD constexpr size_t r3s_smem_bytes() { return 16 * ((size_t)kR3Buf + kR3SaveSmem * kR3Threads); }

__global__ void __launch_bounds__(kR3Threads, 2) grid_r3s_kernel(const cplx* __restrict__ w,
                                                                 const cplx* __restrict__ om_s, int n, int lgL, int B,
                                                                 cplx* __restrict__ q_grid, double* __restrict__ s_grid,
                                                                 const cplx* __restrict__ tw) {
  constexpr int M = 4096;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* X = (cplx*)smem_raw;
  cplx* S = X + kR3Buf;
  const int tid = threadIdx.x;
  const int a = tid & 15, b = tid >> 4;
  const int lgR = lgL - 12;
  const int R = 1 << lgR;
  const size_t L = (size_t)1 << lgL;
  const int TPq = R >> 1, TP = TPq + (R >> 2);
  const long long T = (long long)B * TP;
  const size_t om_stride = 2 * (size_t)n - 1;
  const int Jq = (n + M - 1) >> 12;
  const cplx* twb = tw + tw_index(b, 8);
  const cplx* twc = tw + tw_index(tid, 12);
  const cplx* twL = tw + tw_index(0, lgL);
  const cplx wg = ldg_c(twL + tid);  // W_L^{tid}
  const cplx w256 = ldg_c(twL + 256);
  int sP = kR3StrideHi, sQ = kR3StrideLo;
  int p = (int)(blockIdx.x / TP), t = (int)(blockIdx.x - (long long)p * TP);
  const int dp = (int)(gridDim.x / TP), dt = (int)(gridDim.x - (long long)dp * TP);

  for (long long task = blockIdx.x; task < T; task += gridDim.x) {
    const int sig = t >= TPq;
    const int pair = sig ? t - TPq : t;
    const int lgLe = lgL - sig, lgRe = lgLe - 12;
    const int Re = 1 << lgRe;
    const int Le = 1 << lgLe;
    const cplx* src = sig ? om_s + (size_t)p * om_stride + (n - 1) : w + (size_t)p * n;
    const int J = sig ? Re : Jq;
    if (SLSE_R3_L2PF && task + gridDim.x < T) {
      // the next task's input row towards L2 (16 KB pieces, one per thread)
      int pn = p + dp, tn = t + dt;
      if (tn >= TP) tn -= TP, ++pn;
      const cplx* nsrc = tn >= TPq ? om_s + (size_t)pn * om_stride + (n - 1) : w + (size_t)pn * n;
      const int piece = tid << 10;
      if (piece < n) r3_prefetch_l2(nsrc + piece, 16u * (unsigned)(n - piece < 1024 ? n - piece : 1024));
    }
    // fold j of the length-Le input at i = tid + 256 n2, n2 = 8 h8 .. 8 h8 + 7:
    // w (zero past n), or g.  A fold of g lies wholly on one side (Le / 2 is
    // a multiple of M): kap = i + j M < n (k = kap) or k = Le - kap.  Eight
    // loads are issued before the arithmetic; W_L^k runs as a chain from
    // W_L^{tid} (wg) times a uniform table entry, step W_L^{+-256}.
    const auto load_fold = [&](int j, int h8, cplx* x) {
      const int kap0 = tid + 2048 * h8 + (j << 12);
      if (!sig) {
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = kap0 + 256 * u < n ? ldg_c(src + kap0 + 256 * u) : mk(0.0, 0.0);
        return;
      }
      const bool pos = (j << 12) < n;
      const int k0 = pos ? kap0 : Le - kap0, dk = pos ? 256 : -256;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + dk * u;
        x[u] = ldg_c(src + (k < n ? k : 0));
      }
      const double sg = pos ? 1.0 : -1.0;
      // W_L^{k0} = W_L^{k0 -+ tid} (W_L^{tid})^{+-1}
      cplx W = cmul(ldg_c(twL + (pos ? kap0 - tid : k0 + tid)), mk(wg.re, sg * wg.im));
      const cplx st = mk(w256.re, sg * w256.im);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // k = kap: conj(om) (1 + i W);  k = Le - kap: om (1 + i conj W)
        const double ur = 1.0 - sg * W.im, oi = -sg * x[u].im, orr = x[u].re;
        x[u] = k0 + dk * u < n ? mk(orr * ur - oi * W.re, orr * W.re + oi * ur) : mk(0.0, 0.0);
        W = cmul(W, st);
      }
    };
    // (Both residues' pass A from ONE pass over the input -- the second one's
    // outputs parked in S / sv until the first one's pass C has read the
    // buffer -- measured no faster: 550 vs 542 us at the cfg4 shape, 1100 vs
    // 1016 us at cfg5; its two accumulators spill.)
    cplx sv[16 - kR3SaveSmem];
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int r = 2 * pair + h;
      cplx v[16];
      load_fold(0, 0, v);
      load_fold(0, 1, v + 8);
      for (int j = 1; j < J; ++j) {
        const cplx tj = ldg_c(tw + tw_index((j * r) & (Re - 1), lgRe));  // W_Re^{j r}
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8) {
          cplx x[8];
          load_fold(j, h8, x);
#pragma unroll
          for (int u = 0; u < 8; ++u) v[8 * h8 + u] = cadd(v[8 * h8 + u], cmul(x[u], tj));
        }
      }
      r3_pass_a_dft(v, r, lgLe, tw);
#pragma unroll
      for (int k0 = 0; k0 < 16; ++k0) X[k0 * sP + a * sQ + b] = v[g5_pos(k0)];
      cplx wb1 = ldg_c(twb), wb2 = ldg_c(twb + b);
      if (r) {
        wb1 = cmul(wb1, ldg_c(tw + tw_index(r, lgLe - 4)));
        wb2 = cmul(wb1, wb1);
      }
      __syncthreads();
      {
        cplx* row = X + b * sP + a * sQ;
#pragma unroll
        for (int n1 = 0; n1 < 16; ++n1) v[n1] = row[n1];
        r3_pow_twiddles(v, wb1, wb2);
        dft16_t<0>(v);
#pragma unroll
        for (int k1 = 0; k1 < 16; ++k1) row[k1] = v[g5_pos(k1)];
      }
      cplx wc1 = ldg_c(twc), wc2 = ldg_c(twc + tid);
      if (r) {
        wc1 = cmul(wc1, ldg_c(tw + tw_index(r, lgLe)));
        wc2 = cmul(wc1, wc1);
      }
      __syncthreads();
      {
        const cplx* col = X + a * sP + b;
#pragma unroll
        for (int n0 = 0; n0 < 16; ++n0) v[n0] = col[n0 * sQ];
      }
      r3_pow_twiddles(v, wc1, wc2);
      dft16_t<0>(v);
      if (h == 0) {
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
          if (k2 < kR3SaveSmem) S[k2 * kR3Threads + tid] = v[g5_pos(k2)];
          else sv[k2 - kR3SaveSmem] = v[g5_pos(k2)];
        }
      } else {
        // bins l = 2 pair + {0, 1} + Re m, m = tid + 256 k2, in 16-byte units
        double2* out = sig ? (double2*)(s_grid + (size_t)p * L) : (double2*)(q_grid + (size_t)p * L);
        out += 2 * pair + ((size_t)tid << lgRe);
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) {
          const cplx lo = k2 < kR3SaveSmem ? S[k2 * kR3Threads + tid] : sv[k2 < kR3SaveSmem ? 0 : k2 - kR3SaveSmem];
          const cplx hi = v[g5_pos(k2)];
          r3_store32(out + ((size_t)(256 * k2) << lgRe), lo, hi);
        }
      }
      const int tmp = sP;
      sP = sQ;
      sQ = tmp;
    }
    p += dp;
    t += dt;
    if (t >= TP) {
      t -= TP;
      ++p;
    }
  }
}

// ---------------------------------------------------------------------------
// cfg1 shape (L = 256, N <= 64): one warp per problem, no CTA barrier.
// i = t + 16 n1 (n1 < 4 non-zero), l = k0 + 16 k1:
//   pass A  lane t:  pruned DFT16 over n1                      -> A(t, k0)
//   pass B  lane k0: W256^{t k0}, DFT16 over t                 -> X[k0 + 16 k1]
// lanes 0-15 run q^G = FFT_L(w), lanes 16-31 s^G = Re FFT_L(conj d); the
// exchange is a 16 x 17 complex tile per half-warp (__syncwarp only); the two
// table entries of the twiddle chain stay in registers and the next
// problem's four inputs are loaded before the exchange.
constexpr int kC1Warps = 4;
#ifndef SLSE_C1_MINB
#define SLSE_C1_MINB 4  // 128 registers, 16 warps per SM: 0.83 of HBM (5: 96 registers spill, 0.74; 6: 0.46)
#endif
SLSE_HD constexpr size_t c1_smem_bytes() { return 16 * (size_t)kC1Warps * 2 * 16 * 17; }

__global__ void __launch_bounds__(32 * kC1Warps, SLSE_C1_MINB) grid_c1_kernel(const cplx* __restrict__ w,
                                                                const cplx* __restrict__ om_s, int n, int B,
                                                                cplx* __restrict__ q_grid, double* __restrict__ s_grid,
                                                                const cplx* __restrict__ tw) {
  constexpr int L = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane >> 4, t = lane & 15;
  cplx* X = (cplx*)smem_raw + (warp * 2 + h) * (16 * 17);
  const size_t om_stride = 2 * (size_t)n - 1;
  const cplx w1 = ldg_c(tw + tw_index(t, 8)), w2 = ldg_c(tw + tw_index(2 * t, 8));  // W256^{t}, W256^{2t}
  const int stride = gridDim.x * kC1Warps;
  const auto load = [&](int p, cplx* x) {
    if (p >= B) return;
    const cplx* src = h ? om_s + (size_t)p * om_stride + (n - 1) : w + (size_t)p * n;
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) x[n1] = t + 16 * n1 < n ? ldg_c(src + t + 16 * n1) : mk(0.0, 0.0);
  };
  int p = blockIdx.x * kC1Warps + warp;
  cplx xn[4];
  load(p, xn);
  for (; p < B; p += stride) {
    cplx x[4], v[16];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      // signal 1 is conj d, d_0 = om_s(0), d_m = 2 om_s(m)
      const double f = (t + 16 * n1) ? 2.0 : 1.0;
      x[n1] = h ? mk(f * xn[n1].re, -f * xn[n1].im) : xn[n1];
    }
    r3_pruned4<0>(x, v);
    r3_pruned4<1>(x, v);
    r3_pruned4<2>(x, v);
    r3_pruned4<3>(x, v);
#pragma unroll
    for (int k0 = 0; k0 < 16; ++k0) X[k0 * 17 + t] = v[k0];
    load(p + stride, xn);
    __syncwarp();
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = X[t * 17 + tt];
    __syncwarp();
    r3_pow_twiddles(v, w1, w2);  // lane k0 = t: input tt times W256^{tt k0}
    dft16_t<0>(v);
    if (h == 0) {
      double2* qg = (double2*)(q_grid + (size_t)p * L) + t;
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) {
        const cplx o = v[g5_pos(k1)];
        __stcs(&qg[16 * k1], make_double2(o.re, o.im));
      }
    } else {
      double* sg = s_grid + (size_t)p * L + t;
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) __stcs(&sg[16 * k1], v[g5_pos(k1)].re);
    }
  }
}

}  // namespace slse_k
