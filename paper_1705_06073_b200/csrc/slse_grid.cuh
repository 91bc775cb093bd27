// slse_grid.cuh -- Row 9 standalone activation grid, v5 ("two-pass, TMA in").
//
// Reference: _SuperfastBundle.grid (pkg/src/superlse/model_core.py:303-313):
//   q^G = FFT_L(w),  s^G = delta^-1 [(2 - N)|A0|^2 + 2 Re(A1 conj A0)],
//   A0 = FFT_L(rho), A1 = FFT_L(n rho_n)   (product form).
//
// Shape this kernel serves: L = 1024, 128 < N <= 256 (BASELINE cfg2).  The
// three zero-padded 1024-point transforms run as ONE shared-memory exchange:
//   n = t + 16 s  (t < 16, s < 64, nonzero only for s < 16 since N <= 256)
//   l = a + 64 b  (a < 64, b < 16)
//   X[a + 64 b] = sum_t W16^{t b} W1024^{t a} Y(t, a),
//   Y(t, a)     = sum_{s<16} x_{t+16s} W64^{s a}.
// With a = r + 4 a' the inner sum is a 16-point DFT over s of the
// pre-twiddled x_{t+16s} W64^{s r} (r = 0..3 residues), so
//   inner pass: thread (signal c, t, r) -> one DFT16, 16 values Y(t, r+4a');
//   exchange:   Y to shared memory at [a][t] (row stride 17: conflict-free);
//   outer pass: thread (c, a) -> W1024^{t a} twiddles, one DFT16 over t,
//               bins l = a + 64 b, b = 0..15 -> consecutive lanes write
//               consecutive l: q^G and s^G leave coalesced from registers.
// vs v3 (pruned radix-16, radix-16, radix-4 through two exchanges): half the
// shared-memory round trips, the only traffic that competes with FP64.
//
// Inputs arrive by TMA bulk copy (cp.async.bulk + mbarrier complete_tx):
// the CTA is persistent, and one thread issues the copy of its NEXT problem's
// (w, rho) rows as soon as every warp has pulled the current ones into
// registers, so HBM reads overlap the whole transform.  192 threads:
//   inner: warps 0-3 -> residue r = warp of w (lanes 0-15) and rho (lanes 16-31),
//          warps 4-5 -> n rho at r = 2 (warp - 4) + lane / 16
//   outer: warps 4-5 -> q^G for a = tid - 128; warps 0-3 -> (a, e) pairs, e = 0: A0,
//          e = 1: A1; the pair swaps half of its bins by shuffle and each
//          lane finishes s^G for 8 bins.
#pragma once
#include "slse_fft.cuh"

namespace slse_k {
using namespace slse;

// ------------------------------------------------------------ TMA / mbarrier
SLSE_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
SLSE_D void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SLSE_D void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
SLSE_D void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
SLSE_D void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0)
SLSE_D void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

#ifndef SLSE_G5_MAXREG
#define SLSE_G5_MAXREG 96
#endif
#define SLSE_G5_BOUNDS __maxnreg__(SLSE_G5_MAXREG)

// cos(2 pi k / 64), k = 0..16 (correctly rounded); other k by symmetry
SLSE_HD constexpr double g5_c64q(int k) {
  constexpr double c[17] = {1.0, 0.9951847266721969, 0.9807852804032304, 0.9569403357322088, 0.9238795325112867,
                            0.881921264348355, 0.8314696123025452, 0.773010453362737, 0.7071067811865476,
                            0.6343932841636455, 0.5555702330196022, 0.47139673682599764, 0.3826834323650898,
                            0.2902846772544624, 0.19509032201612828, 0.0980171403295606, 0.0};
  return c[k];
}
SLSE_HD constexpr double g5_cos64(int k) {
  k &= 63;
  return k <= 16 ? g5_c64q(k) : (k <= 32 ? -g5_c64q(32 - k) : (k <= 48 ? -g5_c64q(k - 32) : g5_c64q(64 - k)));
}
SLSE_HD constexpr double g5_sin64(int k) { return g5_cos64(k + 48); }  // sin x = cos(x - pi/2)

// v[s] *= W64^{s r}, r = 2 RP + h: the two candidate twiddles are
// compile-time constants, picked per half-warp by selects (no table loads)
template <int RP>
SLSE_D void g5_pretwiddle(cplx* v, int h) {
#pragma unroll
  for (int s = 1; s < 16; ++s) {
    const int k0 = (s * 2 * RP) & 63, k1 = (s * (2 * RP + 1)) & 63;
    const double cr = h ? g5_cos64(k1) : g5_cos64(k0);
    const double ci = h ? -g5_sin64(k1) : -g5_sin64(k0);
    v[s] = cmul(v[s], mk(cr, ci));
  }
}

// ---------------------------------------------------------------------------
// DFT16 as radix-4 x radix-4 with the twiddles in "scaled" form, so a
// twiddled butterfly input costs one FMA per component instead of a full
// complex multiply (the tangent method):
//   W64^e z = sigma * q,  tangent:   sigma = cos, q = (x + T y, y - T x), T = tan
//                         cotangent: sigma = sin, q = (K x + y, K y - x), K = cot
// (whichever keeps |T|, |K| <= 1), exact swaps for e = 16, 32, 48.  A radix-4
// butterfly with scaled inputs b, c, d then folds the scales into its FMAs:
// 22 ops for three general twiddles vs 28 (3 cmul + 16 adds).
// dft16_t<R>: X[k] = sum_s x[s] W64^{s R} W16^{s k}, i.e. a DFT16 of the
// input pre-twiddled by W64^{s R}; the pre-twiddle splits as W64^{4 n2 R}
// (stage-1 twiddles) times W64^{n1 R}, which merges into the stage-2
// twiddles W64^{n1 (4 k2 + R)} at no cost (s = n1 + 4 n2, k = 4 k1 + k2).
enum { G5_ID = 0, G5_ROT = 1, G5_TAN = 2, G5_COT = 3 };
SLSE_HD constexpr double g5_abs(double x) { return x < 0 ? -x : x; }
SLSE_HD constexpr int g5_kind(int e) {
  return (e & 63) == 0 ? G5_ID
                       : ((e & 15) == 0 ? G5_ROT : (g5_abs(g5_cos64(e)) >= g5_abs(g5_sin64(e)) ? G5_TAN : G5_COT));
}
SLSE_HD constexpr double g5_sigma(int e) {
  return g5_kind(e) == G5_TAN ? g5_cos64(e) : (g5_kind(e) == G5_COT ? g5_sin64(e) : 1.0);
}
template <int E>
SLSE_D cplx g5_q(cplx z) {
  constexpr int k = g5_kind(E);
  if constexpr (k == G5_ID) {
    return z;
  } else if constexpr (k == G5_ROT) {
    constexpr int e = E & 63;
    if constexpr (e == 16) return mk(z.im, -z.re);    // -i z
    else if constexpr (e == 32) return mk(-z.re, -z.im);
    else return mk(-z.im, z.re);                      // +i z
  } else if constexpr (k == G5_TAN) {
    constexpr double T = g5_sin64(E) / g5_cos64(E);
    return mk(fma(T, z.im, z.re), fma(-T, z.re, z.im));
  } else {
    constexpr double K = g5_cos64(E) / g5_sin64(E);
    return mk(fma(K, z.re, z.im), fma(K, z.im, -z.re));
  }
}
// k * x + y, folding k = +-1 to an add / subtract
SLSE_D cplx g5_fmac(double k, cplx x, cplx y) {
  if (k == 1.0) return cadd(y, x);
  if (k == -1.0) return csub(y, x);
  return mk(fma(k, x.re, y.re), fma(k, x.im, y.im));
}
SLSE_D double g5_fmar(double k, double x, double y) {
  if (k == 1.0) return y + x;
  if (k == -1.0) return y - x;
  return fma(k, x, y);
}
// radix-4 (forward) of (a, W^EB b, W^EC c, W^ED d); results y0..y3 in a..d
template <int EB, int EC, int ED>
SLSE_D void g5_r4(cplx& a, cplx& b, cplx& c, cplx& d) {
  constexpr double sb = g5_sigma(EB), sc = g5_sigma(EC), sd = g5_sigma(ED);
  constexpr double rr = sd / sb;
  const cplx qb = g5_q<EB>(b), qc = g5_q<EC>(c), qd = g5_q<ED>(d);
  const cplx s0 = g5_fmac(sc, qc, a), d0 = g5_fmac(-sc, qc, a);
  const cplx s1 = g5_fmac(rr, qd, qb), d1 = g5_fmac(-rr, qd, qb);
  a = g5_fmac(sb, s1, s0);
  c = g5_fmac(-sb, s1, s0);
  b = mk(g5_fmar(sb, d1.im, d0.re), g5_fmar(-sb, d1.re, d0.im));  // d0 - i sb d1
  d = mk(g5_fmar(-sb, d1.im, d0.re), g5_fmar(sb, d1.re, d0.im));  // d0 + i sb d1
}
template <int R>
SLSE_D void dft16_t(cplx* v) {
  // stage 1: radix-4 over n2 for each n1 (inputs v[n1 + 4 n2]), twiddles W64^{4 n2 R}
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) g5_r4<4 * R, 8 * R, 12 * R>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
  // now v[n1 + 4 k2] = Z[n1][k2]; stage 2: radix-4 over n1 for each k2
  g5_r4<1 * (0 + R), 2 * (0 + R), 3 * (0 + R)>(v[0], v[1], v[2], v[3]);
  g5_r4<1 * (4 + R), 2 * (4 + R), 3 * (4 + R)>(v[4], v[5], v[6], v[7]);
  g5_r4<1 * (8 + R), 2 * (8 + R), 3 * (8 + R)>(v[8], v[9], v[10], v[11]);
  g5_r4<1 * (12 + R), 2 * (12 + R), 3 * (12 + R)>(v[12], v[13], v[14], v[15]);
  // v[4 k2 + k1] = X[4 k1 + k2]
}
// output index of bin k after dft16_t
SLSE_HD constexpr int g5_pos(int k) { return 4 * (k & 3) + (k >> 2); }

constexpr int kG5Threads = 192;
constexpr int kG5Warps = kG5Threads / 32;
constexpr int kG5Row = 17;                    // exchange row stride (complex) per a
constexpr int kG5Buf = 64 * kG5Row + 4;       // one signal's exchange buffer (+4: A0 / A1 rows of one a land in different bank groups)
constexpr int kG5Rows = 256;  // stage row length: rows are zero past n, so the inner loads need no bounds select
SLSE_HD constexpr size_t g5_smem_bytes() {
  // mbarriers (128 B) | 2 stages of (w, rho) (2 x 2 x 256 cplx) | X (3 buffers)
  return 128 + 2 * 2 * 16 * (size_t)kG5Rows + 3 * 16 * (size_t)kG5Buf;
}

// v[t] *= W1024^{t a}, t = 1..15, by two interleaved chains (even / odd t)
// from the table entries W^a, W^2a (twa = &W^a, level 10).  (A depth-2 tree
// from W^a, W^2a, W^4a, W^8a -- 11 products instead of 14 -- measured no
// faster: 126.9 vs 122.1 us per 10752-problem launch.)
SLSE_D void g5_outer_twiddles(cplx* v, const cplx* twa, int a) {
  const cplx wa = ldg_c(twa), wa2 = ldg_c(twa + a);
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

SLSE_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Synchronisation per problem k (stage k & 1):
//   full[k & 1]   TMA complete_tx: (w, rho) of problem k landed;
//   __syncthreads every warp stored its inner spectra to X (the one true
//                 barrier); it also proves stage k & 1 fully read, so thread
//                 0 then refills it with problem k + 2;
//   xfree         one arrival per warp once it has pulled its outer inputs
//                 from X; a warp waits on it (previous phase) only right
//                 before its next inner stores, long after everyone arrived.
__global__ void SLSE_G5_BOUNDS grid_tma_kernel(
    const cplx* __restrict__ rho, const double* __restrict__ delta_last, const cplx* __restrict__ w, int n, int B,
    cplx* __restrict__ q_grid, double* __restrict__ s_grid, const cplx* __restrict__ tw, int twlog) {
  constexpr int L = 1024;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* full = (uint64_t*)smem_raw;  // [2]
  uint64_t* xfree = full + 2;
  cplx* stage = (cplx*)(smem_raw + 128);  // [2][w | rho], kG5Rows each (zero past n)
  cplx* X = stage + 4 * kG5Rows;          // 3 exchange buffers
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned row_bytes = 16u * (unsigned)n;
  const int G = gridDim.x;

  const auto issue = [&](int prob, int st) {
    mbar_expect_tx(&full[st], 2 * row_bytes);
    tma_load_1d(stage + st * 2 * kG5Rows, w + (size_t)prob * n, row_bytes, &full[st]);
    tma_load_1d(stage + st * 2 * kG5Rows + kG5Rows, rho + (size_t)prob * n, row_bytes, &full[st]);
  };
  for (int i = tid; i < 4 * kG5Rows; i += kG5Threads)  // zero tails (the copies never touch them)
    if ((i & (kG5Rows - 1)) >= n) stage[i] = mk(0.0, 0.0);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(xfree, kG5Warps);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    if ((int)blockIdx.x < B) issue(blockIdx.x, 0);
    if ((int)blockIdx.x + G < B) issue(blockIdx.x + G, 1);
  }
  // inner-pass role (fixed for the kernel's lifetime): warps 0-3 run residue
  // r = warp for w (lanes 0-15) and rho (lanes 16-31), warp-uniform so the
  // pre-twiddles fold into the DFT's compile-time twiddles; warps 4-5 run
  // n rho with r = 2 (warp - 4) + lane / 16 (selected constants)
  const bool ia1 = warp >= 4;
  const int h = lane >> 4, t = lane & 15;
  const int r = ia1 ? 2 * (warp - 4) + h : warp;
  const int ic = ia1 ? 2 : h;                        // 0: w, 1: rho (A0), 2: n rho (A1)
  cplx* Xi = X + ic * kG5Buf;
  const double dt = (double)t;
  // outer-pass role
  // (q^G goes to warps 4-5, whose inner pass is the heaviest: balances the
  // per-problem work of the six warps between barriers to within ~3 %)
  const bool oq = warp >= 4;
  const int oa = oq ? tid - 128 : tid >> 1;           // a = 0..63
  const int oe = oq ? 0 : (tid & 1);                  // A-pair member: 0 -> A0, 1 -> A1
  const cplx* Xo = X + (oq ? 0 : 1 + oe) * kG5Buf + oa * kG5Row;
  // middle twiddles W1024^{t a}, t = 0..15: fixed per thread, recomputed per
  // problem from two table entries (keeps registers for the transform)
  // (W1024^a, W1024^2a are re-read from the L1-resident table every problem
  // rather than held in registers across the loop: 96 registers, no spills)
  const cplx* twa = tw + tw_index(oa, 10);

  int p = blockIdx.x;
  for (unsigned k = 0; p < B; ++k, p += G) {
    const unsigned st = k & 1;
    const double dl = oq ? 1.0 : delta_last[p];  // issued early, used by the outer pass
    mbar_wait(&full[st], (k >> 1) & 1);
    // ---- inner pass: load x_{t + 16 s}, s < 16 (zero beyond n)
    const cplx* src = stage + st * 2 * kG5Rows + (ic == 0 ? 0 : kG5Rows);
    cplx v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = src[t + 16 * s];
    if (ia1) {
#pragma unroll
      for (int s = 0; s < 16; ++s) v[s] = cscale(v[s], dt + (double)(16 * s));
      if (warp == 4) g5_pretwiddle<0>(v, h);
      else g5_pretwiddle<1>(v, h);
      dft16_t<0>(v);
    } else {
      switch (warp) {  // Y(t, r + 4 a') = v[g5_pos(a')]
        case 0: dft16_t<0>(v); break;
        case 1: dft16_t<1>(v); break;
        case 2: dft16_t<2>(v); break;
        default: dft16_t<3>(v); break;
      }
    }
    if (k) mbar_wait(xfree, (k - 1) & 1);  // everyone has read problem k-1's X
#pragma unroll
    for (int a2 = 0; a2 < 16; ++a2) Xi[(r + 4 * a2) * kG5Row + t] = v[g5_pos(a2)];
    __syncthreads();
    if (tid == 0 && p + 2 * G < B) issue(p + 2 * G, st);
    // ---- outer pass: Y(t, a) W1024^{t a}, DFT16 over t
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = Xo[tt];
    __syncwarp();
    if (lane == 0) mbar_arrive(xfree);
    g5_outer_twiddles(v, twa, oa);
    dft16_t<0>(v);  // bin l = a + 64 b is v[g5_pos(b)]
    if (oq) {
      double2* qg = (double2*)(q_grid + (size_t)p * L);
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const cplx o = v[g5_pos(b)];
        __stcs(&qg[oa + 64 * b], make_double2(o.re, o.im));
      }
    } else {
      // lane pair (e = 0: A0, e = 1: A1): e keeps bins b in [8e, 8e + 8) and
      // receives the partner's spectrum there
      const double inv_d = 1.0 / dl;
      double* sg = s_grid + (size_t)p * L;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const cplx lo = v[g5_pos(j)], hi = v[g5_pos(j + 8)];
        const cplx mine = oe ? hi : lo, give = oe ? lo : hi;
        cplx got;
        got.re = __shfl_xor_sync(0xffffffffu, give.re, 1);
        got.im = __shfl_xor_sync(0xffffffffu, give.im, 1);
        const cplx a0 = oe ? got : mine, a1 = oe ? mine : got;
        const double sv = ((2.0 - (double)n) * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
        __stcs(&sg[oa + 64 * (j + 8 * oe)], sv);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Coefficient form, the reference's own grid() (model_core.py:303-313):
//   q^G = FFT_L(w),   s^G = L IFFT_L(buf).real,  buf[i mod L] = om_s(i), |i| < N,
// with om_s = all_diagonal_sums()["s"] (toeplitz.py:415-432), Hermitian by
// construction (toeplitz.py:428-430).  So with d_0 = om_s(0), d_k = 2 om_s(k):
//   s^G_l = Re sum_{k<N} d_k e^{+j 2 pi k l / L} = Re FFT_L(conj d)[l],
// one forward N-point-supported transform per output, the real part kept
// (the last radix-4 stage's imaginary halves are dead code).  Inputs: the
// w row and the non-negative half of the om_s row (16 N bytes each, the same
// algorithmic bytes as the (w, rho) form); 2 transforms instead of 3.
//
// L = 1024, 128 < N <= 256 (cfg2).  Same two-pass exchange as grid_tma_kernel,
// 128 threads per CTA, every role warp-uniform:
//   inner: warp r = residue, lanes 0-15 w, 16-31 conj d (t = lane & 15): the
//          W64^{s r} pre-twiddles are compile-time for the whole warp;
//   outer: warps 0-1 q^G (a = tid), warps 2-3 s^G (a = tid - 64).
// Inputs by TMA bulk copy into NS stages; persistent CTAs; one barrier per
// problem, plus the xfree mbarrier guarding the exchange buffer.
constexpr int kGCThreads = 128;
constexpr int kGCWarps = kGCThreads / 32;
#ifndef SLSE_GC_STAGES
#define SLSE_GC_STAGES 2  // measured at B = 43008: 2 stages 250 us, 3: 261 us, 4: 262 us (4 vs 3 CTAs per SM)
#endif
constexpr int kGCStages = SLSE_GC_STAGES;
SLSE_HD constexpr size_t gc_smem_bytes() {
  // mbarriers (128 B) | NS stages of (w, om) rows | X (2 exchange buffers)
  return 128 + (size_t)kGCStages * 2 * 16 * kG5Rows + 2 * 16 * (size_t)kG5Buf;
}

__global__ void __launch_bounds__(kGCThreads) grid_coef_kernel(const cplx* __restrict__ w,
                                                                 const cplx* __restrict__ om_s, int n, int B,
                                                                 cplx* __restrict__ q_grid,
                                                                 double* __restrict__ s_grid,
                                                                 const cplx* __restrict__ tw) {
  constexpr int L = 1024;
  constexpr int NS = kGCStages;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* full = (uint64_t*)smem_raw;  // [NS]
  uint64_t* xfree = full + NS;
  cplx* stage = (cplx*)(smem_raw + 128);  // [NS][w | om], kG5Rows each (zero past n)
  cplx* X = stage + NS * 2 * kG5Rows;     // 2 exchange buffers
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const unsigned row_bytes = 16u * (unsigned)n;
  const int G = gridDim.x;
  const size_t om_stride = 2 * (size_t)n - 1;

  const auto issue = [&](int prob, int st) {
    mbar_expect_tx(&full[st], 2 * row_bytes);
    tma_load_1d(stage + st * 2 * kG5Rows, w + (size_t)prob * n, row_bytes, &full[st]);
    tma_load_1d(stage + st * 2 * kG5Rows + kG5Rows, om_s + (size_t)prob * om_stride + (n - 1), row_bytes,
                &full[st]);
  };
  for (int i = tid; i < NS * 2 * kG5Rows; i += kGCThreads)  // zero tails (the copies never touch them)
    if ((i & (kG5Rows - 1)) >= n) stage[i] = mk(0.0, 0.0);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    mbar_init(xfree, kGCWarps);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if ((int)blockIdx.x + s * G < B) issue(blockIdx.x + s * G, s);
  }
  const int h = lane >> 4, t = lane & 15;
  cplx* Xi = X + h * kG5Buf;
  const bool oq = warp < 2;
  const int oa = tid & 63;
  const cplx* Xo = X + (oq ? 0 : 1) * kG5Buf + oa * kG5Row;
  const cplx* twa = tw + tw_index(oa, 10);
  // om half: conj, doubled except om_s(0)
  const double sc0 = (h && t) ? 2.0 : 1.0;

  int p = blockIdx.x;
  unsigned st = 0, ph = 0;
  for (unsigned k = 0; p < B; ++k, p += G) {
    mbar_wait(&full[st], ph);
    const cplx* src = stage + st * 2 * kG5Rows + h * kG5Rows;
    cplx v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = src[t + 16 * s];
    if (h) {
      v[0] = mk(sc0 * v[0].re, -sc0 * v[0].im);
#pragma unroll
      for (int s = 1; s < 16; ++s) v[s] = mk(2.0 * v[s].re, -2.0 * v[s].im);
    }
    switch (warp) {  // Y(t, r + 4 a') = v[g5_pos(a')], r = warp
      case 0: dft16_t<0>(v); break;
      case 1: dft16_t<1>(v); break;
      case 2: dft16_t<2>(v); break;
      default: dft16_t<3>(v); break;
    }
    if (k) mbar_wait(xfree, (k - 1) & 1);  // everyone has read problem k-1's X
#pragma unroll
    for (int a2 = 0; a2 < 16; ++a2) Xi[(warp + 4 * a2) * kG5Row + t] = v[g5_pos(a2)];
    __syncthreads();
    if (tid == 0 && p + NS * G < B) issue(p + NS * G, st);
    if (++st == NS) { st = 0; ph ^= 1u; }
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) v[tt] = Xo[tt];
    __syncwarp();
    if (lane == 0) mbar_arrive(xfree);
    g5_outer_twiddles(v, twa, oa);
    dft16_t<0>(v);  // bin l = a + 64 b is v[g5_pos(b)]
    if (oq) {
      double2* qg = (double2*)(q_grid + (size_t)p * L);
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const cplx o = v[g5_pos(b)];
        __stcs(&qg[oa + 64 * b], make_double2(o.re, o.im));
      }
    } else {
      double* sg = s_grid + (size_t)p * L;
#pragma unroll
      for (int b = 0; b < 16; ++b) __stcs(&sg[oa + 64 * b], v[g5_pos(b)].re);
    }
  }
}

// Coefficient form for tiny grids (L < 16): one thread per (problem, bin),
// direct sums with the table's exact twiddles W_L^{(m l) mod L}.
__global__ void grid_coef_direct_kernel(const cplx* __restrict__ w, const cplx* __restrict__ om_s, int n, int lgL,
                                        int B, cplx* __restrict__ q_grid, double* __restrict__ s_grid,
                                        const cplx* __restrict__ tw) {
  const int L = 1 << lgL;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * L) return;
  const int p = (int)(i >> lgL), l = (int)(i & (L - 1));
  const cplx* wp = w + (size_t)p * n;
  const cplx* op = om_s + (size_t)p * (2 * (size_t)n - 1) + (n - 1);
  cplx q = mk(0.0, 0.0);
  double s = 0.0;
  for (int m = 0; m < n; ++m) {
    const cplx e = tw[tw_index((m * l) & (L - 1), lgL)];  // e^{-j 2 pi m l / L}
    q = cadd(q, cmul(wp[m], e));
    const double f = m ? 2.0 : 1.0;
    s += f * (op[m].re * e.re + op[m].im * e.im);  // Re(om conj(e))
  }
  q_grid[i] = q;
  s_grid[i] = s;
}

// ---------------------------------------------------------------------------
// Residue-decomposed grid for the other large shapes (L >= 2048): with
// L = R M and l = r + R m,
//   X[r + R m] = sum_{i<M} z_r(i) W_M^{i m},
//   z_r(i)     = W_L^{i r} sum_{j : i + j M < n} x_{i + j M} W_R^{j r}
// (W_L^{j M r} = W_R^{j r}), i.e. R independent M-point transforms of
// folded, twiddled inputs, M <= 2048 so the three of one residue (w, rho,
// n rho) stay in shared memory together and run the compile-time Stockham
// schedule of the cfg1/cfg3 kernels.  One task = (problem, residue); tasks
// are problem-major, so the R residue tasks that fill one problem's output
// lines run together and their interleaved writes merge in L2.  Persistent
// CTAs, one barrier between tasks.
#ifndef SLSE_GRES_MINB
#define SLSE_GRES_MINB 2
#endif
#ifndef SLSE_GRES_U
#define SLSE_GRES_U 2
#endif
//
// OMEGA = true: the coefficient form (grid_coef_kernel above): `rho` is the
// om_s array ([B, 2N-1], row p's om_s(0) at p (2N-1) + N-1) and the second
// signal is conj d (d_0 = om_s(0), d_k = 2 om_s(k)); two transforms per
// residue, s^G = Re of the second; `delta_last` is unused.
template <int NT, int LGM, bool OMEGA = false>
__global__ void __launch_bounds__(NT, (NT <= 192 ? 3 : SLSE_GRES_MINB)) grid_res_kernel(
    const cplx* __restrict__ rho, const double* __restrict__ delta_last, const cplx* __restrict__ w, int n, int lgL,
    int B, cplx* __restrict__ q_grid, double* __restrict__ s_grid, const cplx* __restrict__ tw, int twlog) {
  constexpr int M = 1 << LGM;
  constexpr int MS = M + (M >> 4);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* X = (cplx*)smem_raw;
  const int L = 1 << lgL;
  const int lgR = lgL - LGM;
  const int T = B << lgR;
  const int J = (n + M - 1) >> LGM;  // folds
  const double c2n = 2.0 - (double)n;
  for (int task = blockIdx.x; task < T; task += gridDim.x) {
    const int r = task & ((1 << lgR) - 1);
    const int p = task >> lgR;
    const cplx* wp = w + (size_t)p * n;
    const cplx* rp = OMEGA ? rho + (size_t)p * (2 * (size_t)n - 1) + (n - 1) : rho + (size_t)p * n;
    // U items per thread per round, their loads issued together (the fold
    // reads L2: one load round trip per fold step instead of per item)
    constexpr int U = SLSE_GRES_U;
    for (int i0 = threadIdx.x; i0 < M; i0 += U * NT) {
      cplx z0[U], z1[U], z2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) z0[u] = z1[u] = z2[u] = mk(0.0, 0.0);
      for (int j = 0; j < J; ++j) {
        cplx a[U], bb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int m = i0 + u * NT + (j << LGM);
          const bool ok = i0 + u * NT < M && m < n;
          a[u] = ok ? wp[m] : mk(0.0, 0.0);
          bb[u] = ok ? rp[m] : mk(0.0, 0.0);
          if (OMEGA) {
            const double f = m ? 2.0 : 1.0;
            bb[u] = mk(f * bb[u].re, -f * bb[u].im);
          }
        }
        const cplx t = (j == 0 || r == 0) ? mk(1.0, 0.0) : tw[tw_index((j * r) & ((1 << lgR) - 1), lgR)];  // W_R^{j r}
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int m = i0 + u * NT + (j << LGM);
          const cplx bm = cscale(bb[u], (double)m);
          if (j == 0 || r == 0) {
            z0[u] = cadd(z0[u], a[u]);
            z1[u] = cadd(z1[u], bb[u]);
            if (!OMEGA) z2[u] = cadd(z2[u], bm);
          } else {
            z0[u] = cadd(z0[u], cmul(a[u], t));
            z1[u] = cadd(z1[u], cmul(bb[u], t));
            if (!OMEGA) z2[u] = cadd(z2[u], cmul(bm, t));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * NT;
        if (i >= M) break;
        cplx y0 = z0[u], y1 = z1[u], y2 = z2[u];
        if (r) {
          const cplx t = tw[tw_index(i * r, lgL)];  // W_L^{i r}, i r < M R = L
          y0 = cmul(y0, t);
          y1 = cmul(y1, t);
          if (!OMEGA) y2 = cmul(y2, t);
        }
        const int si = sk(i);
        X[si] = y0;
        X[MS + si] = y1;
        if (!OMEGA) X[2 * MS + si] = y2;
      }
    }
    __syncthreads();
    // (the signal count stays a run-time value: a compile-time 2 made nvcc
    // unroll the plan's count loops into a 656-byte stack frame)
    fft_fixed_pruned<LGM, 0>(X, OMEGA ? 2 + (lgL < 0) : 3, -1.0, tw, twlog, threadIdx.x, NT);
    if (OMEGA) {
      cplx* qg = q_grid + (size_t)p * L + r;
      double* sg = s_grid + (size_t)p * L + r;
      for (int k = threadIdx.x; k < M; k += NT) {
        const int sk_ = sk(k);
        qg[(size_t)k << lgR] = X[sk_];
        sg[(size_t)k << lgR] = X[MS + sk_].re;
      }
      __syncthreads();
      continue;
    }
    const double inv_d = 1.0 / delta_last[p];
    cplx* qg = q_grid + (size_t)p * L + r;
    double* sg = s_grid + (size_t)p * L + r;
    for (int k = threadIdx.x; k < M; k += NT) {
      const int sk_ = sk(k);
      const cplx a0 = X[MS + sk_], a1 = X[2 * MS + sk_];
      qg[(size_t)k << lgR] = X[sk_];
      sg[(size_t)k << lgR] = (c2n * cabs2(a0) + 2.0 * (a1.re * a0.re + a1.im * a0.im)) * inv_d;
    }
    __syncthreads();
  }
}

}  // namespace slse_k
