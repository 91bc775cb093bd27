// slse_fft.cuh -- block-cooperative complex128 FFT of power-of-two length.
//
// Replaces numpy.fft (pocketfft) at the reference call sites
// toeplitz.py:104-111,298-305 and model_core.py:306,311.
//
// Layout: the input is gathered through a Load functor straight into
// bit-reversed order (zero padding / weighting fused into the gather), the
// decimation-in-time passes run as radix-4 (two radix-2 stages held in
// registers) plus one radix-2 pass when log2(n) is odd, and the result
// leaves through a Store functor (pointwise epilogues fused into the
// write-back).  When 16*n bytes fit in the CTA's shared-memory scratch the
// passes run there; otherwise they run in place in a global work buffer
// (L2-resident at these sizes).
//
// Twiddles come from a level-major device table (tw_index below), filled
// once per device with sincospi (exact at the quarter points).
#pragma once
#include "slse_port.cuh"

namespace slse {

struct FftCtx {
  const cplx* tw;   // full-circle table, TW entries
  int twlog;        // log2(TW)
  cplx* smem;       // shared scratch for staging
  int smem_cap;     // capacity in complex elements
  int stockham = 0; // 1: prefer the register Stockham passes when they fit
};

SLSE_HD int ilog2(int n) {  // ceil(log2 n), n >= 1
#if defined(__CUDA_ARCH__)
  return n <= 1 ? 0 : 32 - __clz(n - 1);
#else
  int p = 0;
  while ((1 << p) < n) ++p;
  return p;
#endif
}

SLSE_D unsigned brev_bits(unsigned i, int p) {
  if (p == 0) return 0;
#ifdef SLSE_HOST_EMU
  unsigned r = 0;
  for (int b = 0; b < p; ++b) r |= ((i >> b) & 1u) << (p - 1 - b);
  return r;
#else
  return __brev(i) >> (32 - p);
#endif
}

// Level-major twiddle table (levels lg = 0..twlog, 2^(twlog+1) entries):
// entry 2^lg + k holds exp(-2 pi i k / 2^lg), k < 2^lg.  The twiddles of one
// transform size are contiguous, so a pass's lookups stay within a few L1
// lines (a single full-circle table at stride 2^(twlog - lg) puts every
// twiddle of a large pass in its own line).
SLSE_HD size_t tw_index(int k, int lg) { return ((size_t)1 << lg) + (size_t)k; }
SLSE_HD size_t tw_entries(int twlog) { return (size_t)2 << twlog; }

// twiddle exp(sign * 2 pi i k / 2^lg), k < 2^lg <= 2^twlog
SLSE_D cplx twid_tab(const cplx* __restrict__ tw, int twlog, int k, int lg, double sign) {
  (void)twlog;
  cplx t = tw[tw_index(k, lg)];
  if (sign > 0) t.im = -t.im;
  return t;
}

SLSE_D cplx twid(const FftCtx& f, int k, int lg, double sign) {
  cplx t = f.tw[tw_index(k, lg)];
  if (sign > 0) t.im = -t.im;
  return t;
}

// In-place DIT passes on bit-reversed data x[0..n).
SLSE_D void fft_barrier() { SLSE_GROUP_SYNC(); }

// DIT passes over `count` contiguous bit-reversed buffers of n points
// (one barrier per pass for all of them).
// Swizzled staging layout (fft_multi's staged path): point idx of a 2^p
// buffer lives at idx ^ ((bits 2..4) ^ (top 3 bits)), so the bit-reversed
// scatter of 8 consecutive points lands in 8 different 16-byte bank groups
// instead of one (a 32-way serialisation otherwise).
// The XOR also takes bits 2..4, which spreads the strided
// accesses of the first radix-4 passes (half-spans 1 and 4) too; the map
// stays a bijection because only bits >= 2 feed the low three.
SLSE_HD int fswz(int idx, int p) {
  // (below 2^6 points the top bits overlap the low three: no swizzle)
  return p >= 6 ? (idx ^ (((idx >> 2) ^ (idx >> (p - 3))) & 7)) : idx;
}

// SWZ: 0 natural, 1 fswz within each buffer, 2 XOR with the buffer index
// (the four-step path's column groups, whose scatter strides by a buffer)
template <bool SH, int SWZ = 0>
SLSE_D void fft_passes_multi_impl(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                                  int tid, int nt) {
#ifndef SLSE_HOST_EMU
  if constexpr (SH) __builtin_assume(__isShared(x));  // LDS / STS instead of generic LD / ST
#endif
  const int p = ilog2(n);
  int cur_c = 0;
  const auto at = [p, &cur_c](int i) {
    if (SWZ == 1) return fswz(i, p);
    if (SWZ == 2) return p >= 3 ? (i ^ (cur_c & 7)) : i;
    if (SWZ == 3) return p >= 3 ? (fswz(i, p) ^ (cur_c & 7)) : i;
    return i;
  };
  int lgh = 0;  // log2 of current half-span
  if (p & 1) {
    const int per = n >> 1;
    for (int t = tid; t < count * per; t += nt) {
      const int c = t >> (p - 1), u = t & (per - 1);
      cplx* xc = x + (size_t)c * n;
      cur_c = c;
      const int i0 = at(2 * u), i1 = at(2 * u + 1);
      cplx x0 = xc[i0], x1 = xc[i1];
      xc[i0] = cadd(x0, x1);
      xc[i1] = csub(x0, x1);
    }
    fft_barrier();
    lgh = 1;
  }
  const int per = n >> 2;
  for (; lgh + 2 <= p; lgh += 2) {
    const int h = 1 << lgh;
    for (int t = tid; t < count * per; t += nt) {
      const int c = t >> (p - 2), u = t & (per - 1);
      cplx* xc = x + (size_t)c * n;
      cur_c = c;
      const int pos = u & (h - 1);
      const int base = ((u >> lgh) << (lgh + 2)) + pos;
      const int j0 = at(base), j1 = at(base + h), j2 = at(base + 2 * h), j3 = at(base + 3 * h);
      cplx x0 = xc[j0], x1 = xc[j1], x2 = xc[j2], x3 = xc[j3];
      // stage span 2h
      // one table load per butterfly: W_{4h}^{pos}, and W_{2h}^{pos} as its square
      // (the tables of large passes do not stay in the small L1 beside a big
      // shared-memory carve-out)
      cplx w2 = twid_tab(tw, twlog, pos, lgh + 2, sign);
      cplx w1 = cmul(w2, w2);
      cplx t1 = cmul(w1, x1);
      cplx a0 = cadd(x0, t1), a1 = csub(x0, t1);
      cplx t3 = cmul(w1, x3);
      cplx a2 = cadd(x2, t3), a3 = csub(x2, t3);
      // stage span 4h: W^{pos} and W^{pos+h} = (-+ i) W^{pos}
      cplx u2 = cmul(w2, a2);
      cplx u3 = cmul(w2, a3);
      u3 = (sign < 0) ? mk(u3.im, -u3.re) : mk(-u3.im, u3.re);
      xc[j0] = cadd(a0, u2);
      xc[j2] = csub(a0, u2);
      xc[j1] = cadd(a1, u3);
      xc[j3] = csub(a1, u3);
    }
    fft_barrier();
  }
}

// x is either the shared staging area or a global work buffer: dispatch so
// the staged case compiles to shared-memory instructions
SLSE_NI void fft_passes_multi(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                              int tid, int nt) {
#ifndef SLSE_HOST_EMU
  if (__isShared(x)) {
    fft_passes_multi_impl<true>(x, count, n, sign, tw, twlog, tid, nt);
    return;
  }
#endif
  fft_passes_multi_impl<false>(x, count, n, sign, tw, twlog, tid, nt);
}

#ifndef SLSE_HOST_EMU
// passes over shared staging in the swizzled layout (fswz)
SLSE_NI void fft_passes_multi_swz(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                                  int tid, int nt) {
  fft_passes_multi_impl<true, 1>(x, count, n, sign, tw, twlog, tid, nt);
}
// both: fswz within the buffer, then XOR by (c & 7) (the four-step rows)
SLSE_NI void fft_passes_multi_rswz(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                                   int tid, int nt) {
  fft_passes_multi_impl<true, 3>(x, count, n, sign, tw, twlog, tid, nt);
}
// passes over shared staging with buffer c's points XORed by (c & 7) (n >= 8)
SLSE_NI void fft_passes_multi_bswz(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                                   int tid, int nt) {
  fft_passes_multi_impl<true, 2>(x, count, n, sign, tw, twlog, tid, nt);
}
#endif

SLSE_D void fft_passes_v(cplx* x, int n, double sign, const cplx* __restrict__ tw, int twlog, int tid, int nt) {
  fft_passes_multi(x, 1, n, sign, tw, twlog, tid, nt);
}

SLSE_D void fft_passes(cplx* x, int n, double sign, const FftCtx& f, Blk& b) {
  fft_passes_v(x, n, sign, f.tw, f.twlog, b.tid, b.nt);
}

// out = FFT_n(load) ; store(i, out_i).  `work` (global, n elements) is used
// when the transform does not fit the shared scratch; the loader must then
// NOT read `work` (use fft_inplace for that) and the store may write work[i]
// only at its own index i.  sign -1: numpy fft
// convention; sign +1: unscaled inverse (caller applies 1/n).
template <class Load, class Store>
SLSE_D void fft_dit(cplx* work, int n, double sign, Load ld, Store st, const FftCtx& f, Blk& b) {
  const int p = ilog2(n);
  cplx* x = (n <= f.smem_cap) ? f.smem : work;
  for (int i = b.tid; i < n; i += b.nt) x[brev_bits((unsigned)i, p)] = ld(i);
  b.sync();
  fft_passes(x, n, sign, f, b);
  for (int i = b.tid; i < n; i += b.nt) st(i, x[i]);
  b.sync();
}

// In-place transform of data[0..n) (global).  Post-processing is the
// caller's business (one more loop).
SLSE_NI void fft_inplace_dit(cplx* data, int n, double sign, const FftCtx& f, Blk& b) {
  const int p = ilog2(n);
  if (n <= f.smem_cap) {
    cplx* x = f.smem;
    for (int i = b.tid; i < n; i += b.nt) x[brev_bits((unsigned)i, p)] = data[i];
    b.sync();
    fft_passes(x, n, sign, f, b);
    for (int i = b.tid; i < n; i += b.nt) data[i] = x[i];
    b.sync();
  } else {
    for (int i = b.tid; i < n; i += b.nt) {
      const int j = (int)brev_bits((unsigned)i, p);
      if (i < j) {
        cplx t = data[i];
        data[i] = data[j];
        data[j] = t;
      }
    }
    b.sync();
    fft_passes_v(data, n, sign, f.tw, f.twlog, b.tid, b.nt);
  }
}

// ===========================================================================
// Register-resident Stockham autosort FFT (radix 16/8/4/2 passes).
//
// Each pass: a thread loads R points of one sub-transform (stride n/R),
// applies the pass twiddles W_{Ns R}^{(j mod Ns) r}, runs a radix-R DFT in
// registers (compile-time constants, trivial rotations folded) and, after a
// barrier, stores them to their autosorted positions -- in place, natural
// order in and out, no bit reversal.  Requires that every pass's items fit
// the block's registers (count * n / R <= MAXI(R) * nt).
namespace fftc {
// cos / sin of 2 pi k / 16, k = 0..4 (other octants by symmetry)
SLSE_HD constexpr double c16q(int k) {  // cos(2 pi k / 16), k in [0, 4]
  return k == 0 ? 1.0
                : (k == 1 ? 0.92387953251128673848
                          : (k == 2 ? 0.70710678118654752440 : (k == 3 ? 0.38268343236508978178 : 0.0)));
}
SLSE_HD constexpr double cos16(int k) {  // cos(2 pi k / 16), k in [0, 16)
  return k <= 4 ? c16q(k) : (k <= 8 ? -c16q(8 - k) : (k <= 12 ? -c16q(k - 8) : c16q(16 - k)));
}
SLSE_HD constexpr double sin16(int k) { return cos16((k + 12) & 15); }  // sin x = cos(x - pi/2)
}  // namespace fftc

// Runtime-indexed constant rotation: with every loop unrolled k16 is a
// compile-time constant and the branches fold (trivial rotations free).
SLSE_D cplx rot16(cplx v, int k16, double sign) {
  if (k16 == 0) return v;
  if (k16 == 4) return sign < 0 ? mk(v.im, -v.re) : mk(-v.im, v.re);
  if (k16 == 8) return mk(-v.re, -v.im);
  if (k16 == 12) return sign < 0 ? mk(-v.im, v.re) : mk(v.im, -v.re);
  const double c = fftc::cos16(k16), ss = sign * fftc::sin16(k16);
  return mk(v.re * c - v.im * ss, v.re * ss + v.im * c);
}

SLSE_HD constexpr int brev_const(int r, int R) {
  int out = 0;
  for (int m = R >> 1, q = 1; m >= 1; m >>= 1, q <<= 1)
    if (r & q) out |= m;
  return out;
}

// In-place radix-2 DIF DFT of R = 2..16 register points: natural order in,
// bit-reversed order out (X[k] = v[brev(k)]); no temporaries.  Stages are
// template-recursive so every index is a compile-time constant.
template <int R, int SPAN>
struct DifStage {
  SLSE_D static void run(cplx* v, double sign) {
#pragma unroll
    for (int g = 0; g < R; g += 2 * SPAN) {
#pragma unroll
      for (int p = 0; p < SPAN; ++p) {
        const cplx a = v[g + p], c = v[g + p + SPAN];
        v[g + p] = cadd(a, c);
        v[g + p + SPAN] = rot16(csub(a, c), p * (16 / (2 * SPAN)), sign);
      }
    }
    DifStage<R, SPAN / 2>::run(v, sign);
  }
};
template <int R>
struct DifStage<R, 0> {
  SLSE_D static void run(cplx*, double) {}
};

template <int R>
SLSE_D void dft_dif(cplx* v, double sign) {
  DifStage<R, R / 2>::run(v, sign);
}

// shared-memory skew: one pad slot per 16 points, so the stride-R stores of
// a pass (and stride-16 anything) spread over all banks
SLSE_HD int sk(int i) { return i + (i >> 4); }
SLSE_HD int sk_len(int n) { return n + (n >> 4); }

SLSE_D void block_barrier() { SLSE_GROUP_SYNC(); }

template <int R, int MAXI>
SLSE_D void stockham_pass_inl(cplx* x, int count, int n, int Ns, double sign, const cplx* __restrict__ tw, int twlog,
                           int tid, int nt) {
  const int per = n / R;
  const int total = count * per;
  const int lg = ilog2(Ns * R);
#ifdef SLSE_HOST_EMU
  // serial emulation: hold every item of the pass (the device holds MAXI per thread)
  std::vector<std::array<cplx, R>> vv(total);
  for (int it = 0; it < total; ++it) {
    const int c = it / per, j = it - c * per;
    const cplx* xc = x + (size_t)c * sk_len(n);
    for (int r = 0; r < R; ++r) vv[it][r] = xc[sk(j + r * per)];
    if (Ns > 1) {
      const int kk = j & (Ns - 1);
      for (int r = 1; r < R; ++r) vv[it][r] = cmul(vv[it][r], twid_tab(tw, twlog, kk * r, lg, sign));
    }
    dft_dif<R>(vv[it].data(), sign);
  }
  for (int it = 0; it < total; ++it) {
    const int c = it / per, j = it - c * per;
    cplx* xc = x + (size_t)c * sk_len(n);
    const int kk = j & (Ns - 1);
    const int base = (j - kk) * R + kk;
    for (int r = 0; r < R; ++r) xc[sk(base + r * Ns)] = vv[it][brev_const(r, R)];
  }
  (void)tid; (void)nt;
  return;
#endif
  cplx v[MAXI][R];
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int it = tid + i * nt;
    if (it < total) {
      const int c = it / per, j = it - c * per;
      const cplx* xc = x + (size_t)c * sk_len(n);
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = xc[sk(j + r * per)];
      if (Ns > 1) {
        const int kk = j & (Ns - 1);
        if constexpr (R >= 8) {
          // two table loads (W^kk, W^4kk); the rest by short products
          const cplx w1 = twid_tab(tw, twlog, kk, lg, sign);
          const cplx w4 = twid_tab(tw, twlog, 4 * kk, lg, sign);
          const cplx w2 = cmul(w1, w1), w3 = cmul(w2, w1);
          cplx wq = w4;
#pragma unroll
          for (int q = 0; q < R / 4; ++q) {
            if (q >= 2) wq = cmul(wq, w4);
            if (q == 0) {
              v[i][1] = cmul(v[i][1], w1);
              v[i][2] = cmul(v[i][2], w2);
              v[i][3] = cmul(v[i][3], w3);
            } else {
              v[i][4 * q] = cmul(v[i][4 * q], wq);
              v[i][4 * q + 1] = cmul(v[i][4 * q + 1], cmul(wq, w1));
              v[i][4 * q + 2] = cmul(v[i][4 * q + 2], cmul(wq, w2));
              v[i][4 * q + 3] = cmul(v[i][4 * q + 3], cmul(wq, w3));
            }
          }
        } else {
#pragma unroll
          for (int r = 1; r < R; ++r) v[i][r] = cmul(v[i][r], twid_tab(tw, twlog, kk * r, lg, sign));
        }
      }
      dft_dif<R>(v[i], sign);
    }
  }
  block_barrier();
#pragma unroll
  for (int i = 0; i < MAXI; ++i) {
    const int it = tid + i * nt;
    if (it < total) {
      const int c = it / per, j = it - c * per;
      cplx* xc = x + (size_t)c * sk_len(n);
      const int kk = j & (Ns - 1);
      const int base = (j - kk) * R + kk;
#pragma unroll
      for (int r = 0; r < R; ++r) xc[sk(base + r * Ns)] = v[i][brev_const(r, R)];
    }
  }
  block_barrier();
}

template <int R, int MAXI>
SLSE_NI void stockham_pass(cplx* x, int count, int n, int Ns, double sign, const cplx* __restrict__ tw, int twlog,
                           int tid, int nt) {
  stockham_pass_inl<R, MAXI>(x, count, n, Ns, sign, tw, twlog, tid, nt);
}

// Compile-time pass schedule for a transform of 2^LG points (radix 16 while
// at least 16 points per sub-transform remain, then the remainder): fully
// inlined so the register allocator sees straight-line passes.
template <int LG, int LGNS>
struct FixedPlan {
  SLSE_D static void run(cplx* x, int count, double sign, const cplx* __restrict__ tw, int twlog, int tid, int nt) {
    constexpr int rem = LG - LGNS;
    constexpr int lr = rem >= 4 ? 4 : rem;
    constexpr int R = 1 << lr;
    constexpr int MAXI = 16 / R;
    stockham_pass_inl<R, MAXI>(x, count, 1 << LG, 1 << LGNS, sign, tw, twlog, tid, nt);
    FixedPlan<LG, LGNS + lr>::run(x, count, sign, tw, twlog, tid, nt);
  }
};
template <int LG>
struct FixedPlan<LG, LG> {
  SLSE_D static void run(cplx*, int, double, const cplx* __restrict__, int, int, int) {}
};


// Fixed-schedule radix-16 passes from log2(Ns) = LGNS up to LGEND (the
// caller runs the remaining pass itself).  MAXI: radix-16 items per thread,
// ceil(count * 2^LG / 16 / nt) -- every item of every buffer must be covered.
template <int LG, int LGNS, int LGEND, int MAXI = 1>
struct FixedPlanMid {
  SLSE_D static void run(cplx* x, int count, double sign, const cplx* __restrict__ tw, int twlog, int tid, int nt) {
    if constexpr (LGNS + 4 <= LGEND) {
      stockham_pass_inl<16, MAXI>(x, count, 1 << LG, 1 << LGNS, sign, tw, twlog, tid, nt);
      FixedPlanMid<LG, LGNS + 4, LGEND, MAXI>::run(x, count, sign, tw, twlog, tid, nt);
    }
  }
};

// radix for the pass with `rem` = n / Ns points per sub-transform left
SLSE_D int stockham_radix(int rem, int count, int n, int nt) {
#ifdef SLSE_HOST_EMU
  nt = 1 << 24;  // no register cap in the serial emulation
#endif
  const int caps[4][2] = {{16, 1}, {8, 2}, {4, 4}, {2, 8}};
  for (int q = 0; q < 4; ++q) {
    const int R = caps[q][0];
    if (R <= rem && count * (n / R) <= caps[q][1] * nt) return R;
  }
  return 0;
}

// true if the register Stockham applies to (count, n) with nt threads
SLSE_D bool stockham_ok(int count, int n, int nt) {
  for (int Ns = 1; Ns < n;) {
    const int R = stockham_radix(n / Ns, count, n, nt);
    if (R == 0) return false;
    Ns *= R;
  }
  return true;
}

// in-place forward/backward transform of `count` buffers of n points held
// in the skewed layout (buffer c at x + c * sk_len(n), point i at sk(i))
SLSE_D void fft_stockham_inl(cplx* x, int count, int n, double sign, const cplx* __restrict__ tw, int twlog,
                             Blk& b) {
  for (int Ns = 1; Ns < n;) {
    const int R = stockham_radix(n / Ns, count, n, b.nt);
    switch (R) {
      case 16: stockham_pass<16, 1>(x, count, n, Ns, sign, tw, twlog, b.tid, b.nt); break;
      case 8: stockham_pass<8, 2>(x, count, n, Ns, sign, tw, twlog, b.tid, b.nt); break;
      case 4: stockham_pass<4, 4>(x, count, n, Ns, sign, tw, twlog, b.tid, b.nt); break;
      default: stockham_pass<2, 8>(x, count, n, Ns, sign, tw, twlog, b.tid, b.nt); break;
    }
    Ns *= R;
  }
}

SLSE_NI void fft_stockham(cplx* x, int count, int n, double sign, const FftCtx& f, Blk& b) {
  Blk bb = b;
  fft_stockham_inl(x, count, n, sign, f.tw, f.twlog, bb);
  b.bank = bb.bank;
}


// ---------------------------------------------------------------------------
// Dispatch: the register Stockham when the transform fits the shared
// staging area and the block's register caps, else radix-4 DIT.
#ifndef SLSE_SOLVER_STOCKHAM
#define SLSE_SOLVER_STOCKHAM 0
#endif
// Stockham (by value: table, thread index/count) on skewed shared staging
SLSE_NI void fft_stockham_v(cplx* x, int n, double sign, const cplx* __restrict__ tw, int twlog, int tid, int nt) {
#ifndef SLSE_HOST_EMU
  __builtin_assume(__isShared(x));  // always the shared staging area
#endif
  for (int Ns = 1; Ns < n;) {
    const int R = stockham_radix(n / Ns, 1, n, nt);
    switch (R) {
      case 16: stockham_pass_inl<16, 1>(x, 1, n, Ns, sign, tw, twlog, tid, nt); break;
      case 8: stockham_pass_inl<8, 2>(x, 1, n, Ns, sign, tw, twlog, tid, nt); break;
      case 4: stockham_pass_inl<4, 4>(x, 1, n, Ns, sign, tw, twlog, tid, nt); break;
      default: stockham_pass_inl<2, 8>(x, 1, n, Ns, sign, tw, twlog, tid, nt); break;
    }
    Ns *= R;
  }
}

// Stockham wins for wide blocks (cfg3: 187 vs 195 ms), DIT for one-warp
// solvers (cfg2: 49 vs 69 ms), measured on B200.
SLSE_D bool use_stockham(const FftCtx& f, int n, int nt) {
  return (SLSE_SOLVER_STOCKHAM || f.stockham || nt >= 256) && n >= 4 && sk_len(n) <= f.smem_cap &&
         stockham_ok(1, n, nt);
}

template <class Load, class Store>
SLSE_D void fft(cplx* work, int n, double sign, Load ld, Store st, const FftCtx& f, Blk& b) {
  const int tid = b.tid, nt = b.nt;
  if (use_stockham(f, n, nt)) {
    cplx* x = f.smem;
#ifndef SLSE_HOST_EMU
    __builtin_assume(__isShared(x));  // the staging area: LDS / STS
#endif
    for (int i = tid; i < n; i += nt) x[sk(i)] = ld(i);
    fft_barrier();
    fft_stockham_v(x, n, sign, f.tw, f.twlog, tid, nt);
    for (int i = tid; i < n; i += nt) st(i, x[sk(i)]);
    fft_barrier();
  } else {
    const int p = ilog2(n);
    cplx* x = (n <= f.smem_cap) ? f.smem : work;
    for (int i = tid; i < n; i += nt) x[brev_bits((unsigned)i, p)] = ld(i);
    fft_barrier();
    fft_passes_v(x, n, sign, f.tw, f.twlog, tid, nt);
    for (int i = tid; i < n; i += nt) st(i, x[i]);
    fft_barrier();
  }
}

#ifndef SLSE_MULTI_SWZ
#define SLSE_MULTI_SWZ 1
#endif
// `count` transforms of n points at once: ld(c, i) -> FFT -> st(c, i, v).
// Staged in shared memory when count*n fits, else in `work` (count*n,
// global; the loader must not read `work`).
template <class Load, class Store>
SLSE_D void fft_multi(cplx* work, int count, int n, double sign, Load ld, Store st, const FftCtx& f, Blk& b) {
  const int tid = b.tid, nt = b.nt;
  const int p = ilog2(n);
  // as many buffers per group as the shared staging holds (all of them in
  // one group when possible); only a transform larger than the staging
  // runs in the global work buffer
  if (n > f.smem_cap && n >= 64 && (1 << (p - (p >> 1))) <= f.smem_cap) {
    // four-step: n = n1 n2, column transforms of n1 then rows of n2, both
    // staged in shared memory in groups; `work` holds the intermediate.
    const int p1 = p >> 1, p2 = p - p1;
    const int n1 = 1 << p1, n2 = 1 << p2;
    int G = 1;
    while (2 * G * (n1 > n2 ? n1 : n2) <= f.smem_cap && 2 * G <= n2 && 2 * G <= n1) G *= 2;
    cplx* x = f.smem;
    for (int c = 0; c < count; ++c) {
      cplx* wc = work + (size_t)c * n;
      for (int j0 = 0; j0 < n2; j0 += G) {  // columns j2 = j0 .. j0+G-1
        // column g's points XORed by (g & 7): the strided scatter / gather
        // over consecutive g then spreads over the shared-memory banks
#ifndef SLSE_HOST_EMU
        const auto bx = [](int g, int i) { return i ^ (g & 7); };
#else
        const auto bx = [](int, int i) { return i; };  // (the emulation's passes are unswizzled)
#endif
        for (int t = tid; t < G * n1; t += nt) {
          const int j1 = t / G, g = t - j1 * G;  // consecutive threads -> consecutive j2 (coalesced)
          x[(size_t)g * n1 + bx(g, (int)brev_bits((unsigned)j1, p1))] = ld(c, (j0 + g) + n2 * j1);
        }
        fft_barrier();
#ifndef SLSE_HOST_EMU
        fft_passes_multi_bswz(x, G, n1, sign, f.tw, f.twlog, tid, nt);
#else
        fft_passes_multi(x, G, n1, sign, f.tw, f.twlog, tid, nt);
#endif
        for (int t = tid; t < G * n1; t += nt) {
          const int k1 = t / G, g = t - k1 * G;
          const int j2 = j0 + g;
          const cplx v = cmul(x[(size_t)g * n1 + bx(g, k1)], twid_tab(f.tw, f.twlog, (j2 * k1) & (n - 1), p, sign));
          wc[(size_t)k1 * n2 + j2] = v;
        }
        fft_barrier();
      }
      for (int k0 = 0; k0 < n1; k0 += G) {  // rows k1 = k0 .. k0+G-1
#ifndef SLSE_HOST_EMU
        const auto rx = [p2](int g, int i) { return p2 >= 3 ? (fswz(i, p2) ^ (g & 7)) : i; };
#else
        const auto rx = [](int, int i) { return i; };
#endif
        for (int t = tid; t < G * n2; t += nt) {
          const int g = t >> p2, j2 = t & (n2 - 1);
          x[(size_t)g * n2 + rx(g, (int)brev_bits((unsigned)j2, p2))] = wc[(size_t)(k0 + g) * n2 + j2];
        }
        fft_barrier();
#ifndef SLSE_HOST_EMU
        fft_passes_multi_rswz(x, G, n2, sign, f.tw, f.twlog, tid, nt);
#else
        fft_passes_multi(x, G, n2, sign, f.tw, f.twlog, tid, nt);
#endif
        for (int t = tid; t < G * n2; t += nt) {
          const int k2 = t / G, g = t - k2 * G;  // consecutive threads -> consecutive k1 (coalesced)
          st(c, (k0 + g) + n1 * k2, x[(size_t)g * n2 + rx(g, k2)]);
        }
        fft_barrier();
      }
    }
    return;
  }
  const int g = n <= f.smem_cap ? (f.smem_cap / n < count ? f.smem_cap / n : count) : count;
#if SLSE_MULTI_SWZ && !defined(SLSE_HOST_EMU)
  const bool swz = n <= f.smem_cap;  // staged in shared memory: swizzled layout
#else
  const bool swz = false;
#endif
  cplx* x = n <= f.smem_cap ? f.smem : work;
  for (int c0 = 0; c0 < count; c0 += g) {
    const int gc = count - c0 < g ? count - c0 : g;
    for (int t = tid; t < gc * n; t += nt) {
      const int c = t >> p, i = t & (n - 1);
      const int j = (int)brev_bits((unsigned)i, p);
      x[(size_t)c * n + (swz ? fswz(j, p) : j)] = ld(c0 + c, i);
    }
    fft_barrier();
#if SLSE_MULTI_SWZ && !defined(SLSE_HOST_EMU)
    if (swz) fft_passes_multi_swz(x, gc, n, sign, f.tw, f.twlog, tid, nt);
    else
#endif
    fft_passes_multi(x, gc, n, sign, f.tw, f.twlog, tid, nt);
    for (int t = tid; t < gc * n; t += nt) {
      const int c = t >> p, i = t & (n - 1);
      st(c0 + c, i, x[(size_t)c * n + (swz ? fswz(i, p) : i)]);
    }
    fft_barrier();
  }
}

SLSE_D void fft_inplace(cplx* data, int n, double sign, const FftCtx& f, Blk& b) {
  const int tid = b.tid, nt = b.nt;
  if (use_stockham(f, n, nt)) {
    cplx* x = f.smem;
#ifndef SLSE_HOST_EMU
    __builtin_assume(__isShared(x));
#endif
    for (int i = tid; i < n; i += nt) x[sk(i)] = data[i];
    fft_barrier();
    fft_stockham_v(x, n, sign, f.tw, f.twlog, tid, nt);
    for (int i = tid; i < n; i += nt) data[i] = x[sk(i)];
    fft_barrier();
  } else {
    fft_inplace_dit(data, n, sign, f, b);
  }
}

// ---------------------------------------------------------------------------
// Pruned first pass for zero-padded inputs: only the first NZ of the R
// points of every radix-R sub-transform are nonzero (input support
// [0, n*NZ/R)).  The DIF stages with span >= NZ reduce to rotations of the
// nonzero half (no additions), and the zero inputs are never loaded.
template <int R, int NZ, int SPAN>
struct DifPrunedStage {
  SLSE_D static void run(cplx* v, double sign) {
    if constexpr (SPAN >= NZ) {
#pragma unroll
      for (int g = 0; g < R; g += 2 * SPAN) {
#pragma unroll
        for (int p = 0; p < NZ; ++p) v[g + p + SPAN] = rot16(v[g + p], p * (16 / (2 * SPAN)), sign);
      }
    } else {
#pragma unroll
      for (int g = 0; g < R; g += 2 * SPAN) {
#pragma unroll
        for (int p = 0; p < SPAN; ++p) {
          const cplx a = v[g + p], c = v[g + p + SPAN];
          v[g + p] = cadd(a, c);
          v[g + p + SPAN] = rot16(csub(a, c), p * (16 / (2 * SPAN)), sign);
        }
      }
    }
    DifPrunedStage<R, NZ, SPAN / 2>::run(v, sign);
  }
};
template <int R, int NZ>
struct DifPrunedStage<R, NZ, 0> {
  SLSE_D static void run(cplx*, double) {}
};

template <int R, int NZ>
SLSE_D void stockham_first_pruned(cplx* x, int count, int n, double sign, int tid, int nt) {
  const int per = n / R;
  const int total = count * per;
#ifdef SLSE_HOST_EMU
  std::vector<std::array<cplx, R>> vv(total);
  for (int it = 0; it < total; ++it) {
    const int c = it / per, j = it - c * per;
    const cplx* xc = x + (size_t)c * sk_len(n);
    for (int r = 0; r < NZ; ++r) vv[it][r] = xc[sk(j + r * per)];
    DifPrunedStage<R, NZ, R / 2>::run(vv[it].data(), sign);
  }
  for (int it = 0; it < total; ++it) {
    const int c = it / per, j = it - c * per;
    cplx* xc = x + (size_t)c * sk_len(n);
    for (int r = 0; r < R; ++r) xc[sk(j * R + r)] = vv[it][brev_const(r, R)];
  }
  (void)tid; (void)nt;
  return;
#endif
  cplx v[R];
  const int it = tid;
  const bool act = it < total;
  int c = 0, j = 0;
  if (act) {
    c = it / per;
    j = it - c * per;
    const cplx* xc = x + (size_t)c * sk_len(n);
#pragma unroll
    for (int r = 0; r < NZ; ++r) v[r] = xc[sk(j + r * per)];
    DifPrunedStage<R, NZ, R / 2>::run(v, sign);
  }
  block_barrier();
  if (act) {
    cplx* xc = x + (size_t)c * sk_len(n);
#pragma unroll
    for (int r = 0; r < R; ++r) xc[sk(j * R + r)] = v[brev_const(r, R)];
  }
  block_barrier();
}

// Whole transform for inputs supported on the first 2^-Q of each buffer:
// pruned radix-16 first pass, then the fixed schedule.  Needs count*n/16 <= nt.
template <int LG, int Q>
SLSE_D void fft_fixed_pruned(cplx* x, int count, double sign, const cplx* __restrict__ tw, int twlog, int tid, int nt) {
  static_assert(LG >= 4 && Q >= 0 && Q <= 3, "pruned plan: L >= 16, support >= L/8");
  stockham_first_pruned<16, (16 >> Q)>(x, count, 1 << LG, sign, tid, nt);
  FixedPlan<LG, 4>::run(x, count, sign, tw, twlog, tid, nt);
}

}  // namespace slse
