// slse_port.cuh -- complex type, block context and deterministic block
// reductions shared by every Superfast-LSE kernel.
//
// The same headers compile two ways:
//   * nvcc (the product): SLSE_D = __device__, a Blk is one CTA, reductions
//     use warp shuffles + one shared-memory exchange;
//   * g++ -DSLSE_HOST_EMU (tests/ only, a logic debugger for the per-problem
//     program): a Blk is ONE serial thread (tid = 0, nt = 1) and every
//     reduction is the identity.  Nothing in the shipped package loads it.
#pragma once
#include <stdint.h>

#ifdef SLSE_HOST_EMU
#include <algorithm>
#include <array>
#include <cmath>
#include <vector>
#include <cstring>
#define SLSE_D inline
#define SLSE_NI inline
#define SLSE_NIM inline
#define SLSE_HD inline
#define SLSE_RESTRICT
#else
#define SLSE_D __device__ __forceinline__
#define SLSE_NI static __device__ __noinline__
#define SLSE_NIM __device__ __noinline__
#define SLSE_HD __host__ __device__ __forceinline__
#define SLSE_RESTRICT __restrict__
#endif

namespace slse {

struct alignas(16) cplx {
  double re, im;
};

SLSE_HD cplx mk(double r, double i) { cplx c; c.re = r; c.im = i; return c; }
SLSE_HD cplx cadd(cplx a, cplx b) { return mk(a.re + b.re, a.im + b.im); }
SLSE_HD cplx csub(cplx a, cplx b) { return mk(a.re - b.re, a.im - b.im); }
// numpy's complex multiply: (ar*br - ai*bi, ar*bi + ai*br)
SLSE_HD cplx cmul(cplx a, cplx b) { return mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
SLSE_HD cplx cmulc(cplx a, cplx b) {  // a * conj(b)
  return mk(a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im);
}
SLSE_HD cplx conjg(cplx a) { return mk(a.re, -a.im); }
SLSE_HD cplx cscale(cplx a, double s) { return mk(a.re * s, a.im * s); }
SLSE_HD double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }
// correctly rounded reciprocal (== 1.0 / x on both sides); unused on the hot paths now
SLSE_HD double rcp_rn(double x) {
#if defined(__CUDA_ARCH__)
  return __drcp_rn(x);
#else
  return 1.0 / x;
#endif
}
// Reciprocal of a positive normal double (the prediction errors d > floor):
// MUFU.RCP64H seed plus one cubic Newton step, within 1 ulp, branch-free, so
// the scheduler interleaves it with the surrounding chain (__drcp_rn adds two
// more dependent DFMAs and a special-case branch for correct rounding).
SLSE_HD double rcp_pos(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
#else
  return 1.0 / x;
#endif
}
// a / b for complex b (Smith-free plain formula is fine: |b| ~ pivot scale)
SLSE_HD cplx cdiv_real(cplx a, double b) { return mk(a.re / b, a.im / b); }

// e^{j 2 pi phi} for phi given as (integer n) * theta reduced EXACTLY mod 1:
// p = n*theta rounded, e = fma(n, theta, -p) exact residual, frac(p) + e.
SLSE_HD double frac_mul(double n, double theta) {
  double p = n * theta;
#ifdef SLSE_HOST_EMU
  double e = std::fma(n, theta, -p);
  double f = p - std::floor(p);
#else
  double e = fma(n, theta, -p);
  double f = p - floor(p);
#endif
  return f + e;
}

SLSE_HD void sincos2pi(double phi, double* s, double* c) {
#ifdef SLSE_HOST_EMU
  const double kPi = 3.14159265358979323846;
  double x = 2.0 * phi;
  // reduce to [-1, 1] before the libm call
  x = x - 2.0 * std::floor(0.5 * x + 0.5);
  *s = std::sin(kPi * x);
  *c = std::cos(kPi * x);
#else
  sincospi(2.0 * phi, s, c);
#endif
}

// e^{sign * j 2 pi n theta}
SLSE_HD cplx expj2pi(double n, double theta, double sign) {
  double s, c;
  sincos2pi(frac_mul(n, theta), &s, &c);
  return mk(c, sign * s);
}

#ifdef SLSE_HOST_EMU
using std::fabs; using std::floor; using std::fma; using std::fmod; using std::log; using std::log1p;
using std::sqrt; using std::isnan;
#endif

#ifndef SLSE_HOST_EMU
// Transposed warp sum of V (power of two, <= 16) per-lane values over groups
// of 2V lanes: each xor stage sends half of the remaining values and keeps
// the other half, so it takes V shuffles instead of 5 V.  Sum v ends in lanes
// 2v and 2v+1 of each group (value bit i <-> lane bit i+1).  Clobbers v.
template <int V>
SLSE_D double warp_tsum(double* v, int lane) {
#pragma unroll
  for (int h = V / 2; h >= 1; h >>= 1) {
    const bool up = (lane & (2 * h)) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
#endif

// Barrier of one cooperative group ("block").  In warp mode
// (SLSE_WARP_MODE: several independent one-warp solvers share a CTA) a
// group is one warp, so every group barrier is a warp barrier.
#ifdef SLSE_HOST_EMU
#define SLSE_GROUP_SYNC()
#elif defined(SLSE_WARP_MODE)
#define SLSE_GROUP_SYNC() __syncwarp()
#else
#define SLSE_GROUP_SYNC() __syncthreads()
#endif

#if defined(SLSE_WARP_MODE) && !defined(SLSE_HOST_EMU)
// CTA-wide rendezvous of the warp-mode solver (see Solver::build).  Heavy
// operations run between rv_arrive (barrier 0, with an all-idle vote) and
// rv_depart (barrier 1); control code runs between rv_depart and the next
// rv_arrive.  A long operation yields at rv_slice points, ending the current
// operation window and waiting out the control window, so short operations
// of the other warps do not wait for it to finish.
#ifndef SLSE_RV_GROUPS
#define SLSE_RV_GROUPS 4  // rendezvous groups per CTA: warps w with equal w % GROUPS (one per SM sub-partition)
#endif
SLSE_D bool rv_arrive(int idle) {
#if SLSE_RV_GROUPS == 1
  return __syncthreads_and(idle) != 0;
#else
  const unsigned g = (threadIdx.x >> 5) % SLSE_RV_GROUPS, cnt = blockDim.x / SLSE_RV_GROUPS;
  unsigned r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.and.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((unsigned)idle), "r"(1 + g), "r"(cnt)
      : "memory");
  return r != 0;
#endif
}
SLSE_D void rv_depart() {
#if SLSE_RV_GROUPS == 1
  asm volatile("bar.sync 1;" ::: "memory");
#else
  const unsigned g = (threadIdx.x >> 5) % SLSE_RV_GROUPS, cnt = blockDim.x / SLSE_RV_GROUPS;
  asm volatile("bar.sync %0, %1;" ::"r"(1 + SLSE_RV_GROUPS + g), "r"(cnt) : "memory");
#endif
}
SLSE_D void rv_slice() {
  rv_depart();
  (void)rv_arrive(0);
}
#define SLSE_RV_SLICE() rv_slice()
#else
#define SLSE_RV_SLICE()
#endif

// ---------------------------------------------------------------------------
// Block context.  All reductions return the SAME bits to every thread (warp
// xor-butterflies are symmetric; the cross-warp stage is a fixed sequential
// order), so scalar control flow derived from them stays uniform.
// Block reductions are out of line on the device: one shared copy instead of
// an inlined shuffle tree (plus the compiler's divergent fallback) at every
// call site of the control code -- instruction-cache footprint.
#ifdef SLSE_HOST_EMU
#define SLSE_BLK_NI SLSE_D
#else
#define SLSE_BLK_NI __device__ __noinline__
#endif

struct Blk {
  int tid;
  int nt;
  double* red;  // shared scratch: 2 banks x nwarps x 16 doubles
  int bank;     // alternates so one barrier per reduction suffices

  SLSE_D void sync() { SLSE_GROUP_SYNC(); }
  SLSE_D bool leader() const { return tid == 0; }

#ifdef SLSE_HOST_EMU
  SLSE_D double sum(double v) { return v; }
  SLSE_D cplx sum(cplx v) { return v; }
  SLSE_D void sumv(double* v, int k) { (void)v; (void)k; }
  SLSE_D double minv(double v) { return v; }
  SLSE_D double maxv(double v) { return v; }
  SLSE_D int sumi(int v) { return v; }
  // argmin with lowest index on ties; idx < 0 means "no candidate"
  SLSE_D void argmin(double& v, int& idx) { (void)v; (void)idx; }
  SLSE_D int bcast_i(int v) { return v; }
  SLSE_D double bcast_d(double v) { return v; }
  SLSE_D int exscan(int v, int& total) { total = v; return 0; }
#else
  SLSE_D int nwarps() const { return (nt + 31) >> 5; }
  // k <= 16 doubles reduced at once
  SLSE_BLK_NI void sumv(double* v, int k) {
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < k) {
        double x = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        v[i] = x;
      }
    }
    double* r = red + bank * (nwarps() * 16);
    if (lane == 0) {
      for (int i = 0; i < k; ++i) r[w * 16 + i] = v[i];
    }
    SLSE_GROUP_SYNC();
    const int nw = nwarps();
    for (int i = 0; i < k; ++i) {
      double acc = r[i];
      for (int j = 1; j < nw; ++j) acc += r[j * 16 + i];
      v[i] = acc;
    }
    bank ^= 1;
  }
  SLSE_D double sum(double x) { double v[1] = {x}; sumv(v, 1); return v[0]; }
  SLSE_D cplx sum(cplx x) { double v[2] = {x.re, x.im}; sumv(v, 2); return mk(v[0], v[1]); }
  SLSE_D int sumi(int x) { return (int)sum((double)x); }
  SLSE_BLK_NI double minv(double x) {
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    double* r = red + bank * (nwarps() * 16);
    if (lane == 0) r[w * 16] = x;
    SLSE_GROUP_SYNC();
    double acc = r[0];
    for (int j = 1; j < nwarps(); ++j) acc = fmin(acc, r[j * 16]);
    bank ^= 1;
    return acc;
  }
  SLSE_D double maxv(double x) { return -minv(-x); }
  SLSE_BLK_NI void argmin(double& v, int& idx) {
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, v, o);
      int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
    }
    double* r = red + bank * (nwarps() * 16);
    if (lane == 0) { r[w * 16] = v; r[w * 16 + 1] = (double)idx; }
    SLSE_GROUP_SYNC();
    v = r[0]; idx = (int)r[1];
    for (int j = 1; j < nwarps(); ++j) {
      double ov = r[j * 16]; int oi = (int)r[j * 16 + 1];
      if (better(ov, oi, v, idx)) { v = ov; idx = oi; }
    }
    bank ^= 1;
  }
  SLSE_BLK_NI int bcast_i(int x) {  // value of thread 0
    double* r = red + bank * (nwarps() * 16);
    if (tid == 0) r[0] = (double)x;
    SLSE_GROUP_SYNC();
    int out = (int)r[0];
    bank ^= 1;
    return out;
  }
  SLSE_BLK_NI double bcast_d(double x) {
    double* r = red + bank * (nwarps() * 16);
    if (tid == 0) r[0] = x;
    SLSE_GROUP_SYNC();
    double out = r[0];
    bank ^= 1;
    return out;
  }
  // exclusive prefix sum over threads in tid order; total to everyone
  SLSE_BLK_NI int exscan(int x, int& total) {
    const int lane = tid & 31, w = tid >> 5;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    double* r = red + bank * (nwarps() * 16);
    if (lane == 31) r[w * 16] = (double)inc;
    SLSE_GROUP_SYNC();
    int before = 0, tot = 0;
    for (int j = 0; j < nwarps(); ++j) {
      int c = (int)r[j * 16];
      if (j < w) before += c;
      tot += c;
    }
    bank ^= 1;
    total = tot;
    return before + inc - x;
  }
#endif
  // (ov, oi) beats (v, i): smaller value, lowest index on ties; idx < 0 = empty
  SLSE_HD static bool better(double ov, int oi, double v, int i) {
    if (oi < 0) return false;
    if (i < 0) return true;
    if (ov < v) return true;
    if (ov == v && oi < i) return true;
    return false;
  }
};

#ifdef SLSE_HOST_EMU
SLSE_D void host_argmin_combine(double& v, int& idx, double ov, int oi) {
  if (Blk::better(ov, oi, v, idx)) { v = ov; idx = oi; }
}
#endif

}  // namespace slse
