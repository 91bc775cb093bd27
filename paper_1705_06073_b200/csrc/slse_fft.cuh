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
// Twiddles come from a device table tw[k] = exp(-2 pi i k / TW), TW = 2^twlog,
// filled once per launch with sincospi (exact at the quarter points).
#pragma once
#include "slse_port.cuh"

namespace slse {

struct FftCtx {
  const cplx* tw;   // full-circle table, TW entries
  int twlog;        // log2(TW)
  cplx* smem;       // shared scratch for staging
  int smem_cap;     // capacity in complex elements
};

SLSE_HD int ilog2(int n) {
  int p = 0;
  while ((1 << p) < n) ++p;
  return p;
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

// twiddle exp(sign * 2 pi i k / 2^lg)
SLSE_D cplx twid(const FftCtx& f, int k, int lg, double sign) {
  cplx t = f.tw[(size_t)k << (f.twlog - lg)];
  if (sign > 0) t.im = -t.im;
  return t;
}

// In-place DIT passes on bit-reversed data x[0..n).
SLSE_NI void fft_passes(cplx* x, int n, double sign, const FftCtx& f, Blk& b) {
  const int p = ilog2(n);
  int lgh = 0;  // log2 of current half-span
  if (p & 1) {
    for (int t = b.tid; t < (n >> 1); t += b.nt) {
      cplx x0 = x[2 * t], x1 = x[2 * t + 1];
      x[2 * t] = cadd(x0, x1);
      x[2 * t + 1] = csub(x0, x1);
    }
    b.sync();
    lgh = 1;
  }
  for (; lgh + 2 <= p; lgh += 2) {
    const int h = 1 << lgh;
    for (int t = b.tid; t < (n >> 2); t += b.nt) {
      const int pos = t & (h - 1);
      const int base = ((t >> lgh) << (lgh + 2)) + pos;
      cplx x0 = x[base], x1 = x[base + h], x2 = x[base + 2 * h], x3 = x[base + 3 * h];
      // stage span 2h
      cplx w1 = twid(f, pos, lgh + 1, sign);
      cplx t1 = cmul(w1, x1);
      cplx a0 = cadd(x0, t1), a1 = csub(x0, t1);
      cplx t3 = cmul(w1, x3);
      cplx a2 = cadd(x2, t3), a3 = csub(x2, t3);
      // stage span 4h: W^{pos} and W^{pos+h} = (-+ i) W^{pos}
      cplx w2 = twid(f, pos, lgh + 2, sign);
      cplx u2 = cmul(w2, a2);
      cplx u3 = cmul(w2, a3);
      u3 = (sign < 0) ? mk(u3.im, -u3.re) : mk(-u3.im, u3.re);
      x[base] = cadd(a0, u2);
      x[base + 2 * h] = csub(a0, u2);
      x[base + h] = cadd(a1, u3);
      x[base + 3 * h] = csub(a1, u3);
    }
    b.sync();
  }
}

// out = FFT_n(load) ; store(i, out_i).  `work` (global, n elements) is used
// when the transform does not fit the shared scratch; the loader must then
// NOT read `work` (use fft_inplace for that) and the store may write work[i]
// only at its own index i.  sign -1: numpy fft
// convention; sign +1: unscaled inverse (caller applies 1/n).
template <class Load, class Store>
SLSE_D void fft(cplx* work, int n, double sign, Load ld, Store st, const FftCtx& f, Blk& b) {
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
SLSE_NI void fft_inplace(cplx* data, int n, double sign, const FftCtx& f, Blk& b) {
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
    fft_passes(data, n, sign, f, b);
  }
}

}  // namespace slse
