// slse_sim.cu -- on-device synthetic scenes and evaluation metrics
// (reference pkg/src/superlse/simdata.py).
//
// sim_generate_kernel (one CTA per trial) draws a scene with the reference
// generator's laws (simdata.generate :109-122):
//   * observation pattern: first and last sample always observed, M - 2 of
//     the inner N - 2 uniformly without replacement (:78-86);
//   * frequencies by sequential rejection with wrap-around separation
//     > min_sep, at most 100000 draws each (:61-73, :25);
//   * coefficients a = CN(0, 0.8^2) + 0.2 e^{j arg a} per snapshot (:56-58);
//   * noise variance beta = mean_g ||Phi Psi alpha_g||^2 / (M snr) and
//     y = Phi Psi alpha + sqrt(beta/2) (n1 + j n2) (:89-102);
// from a counter-based Philox-4x32-10 stream keyed by (seed, point) with
// counter (trial, stream, draw) -- every trial is independent and
// reproducible, whatever the batch split.  (The host generator in
// simdata.py reproduces the reference's numpy streams bit for bit; this one
// is the throughput path for Monte-Carlo sweeps: same laws, its own stream.)
//
// sim_metrics_kernel (one CTA per trial) evaluates the reference metrics on
// the device: NMSE of the full-length reconstruction (:160-169) and the
// component success ratio (:196-205); block success needs the Hungarian
// assignment (:172-193), which stays on the host (scipy), fed by the
// per-trial nearest-distance data computed here.
#include <cuda_runtime.h>

#include "slse_port.cuh"
#include "superlse_b200.h"

namespace {
using namespace slse;

constexpr int kSimThreads = 128;
constexpr int kMaxRejections = 100000;  // simdata.py:25
constexpr double kCoeffStd = 0.8;       // simdata.py:23
constexpr double kCoeffOffset = 0.2;    // simdata.py:22

// ---- Philox-4x32-10 (Salmon et al., SC'11), counter-based ----
struct U4 {
  unsigned x, y, z, w;
};
__device__ __forceinline__ U4 philox(U4 c, unsigned k0, unsigned k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
struct Stream {
  unsigned k0, k1, trial, sid;
  // two uniforms in [0, 1) with 53 random bits each, draw index i
  __device__ __forceinline__ void uniform2(unsigned i, double* a, double* b) const {
    const U4 r = philox(U4{i, 0u, trial, sid}, k0, k1);
    const unsigned long long u0 = ((unsigned long long)r.x << 32 | r.y) >> 11;
    const unsigned long long u1 = ((unsigned long long)r.z << 32 | r.w) >> 11;
    *a = (double)u0 * 0x1.0p-53;
    *b = (double)u1 * 0x1.0p-53;
  }
  // two independent standard normals (Box-Muller), draw index i
  __device__ __forceinline__ void normal2(unsigned i, double* a, double* b) const {
    double u, v;
    uniform2(i, &u, &v);
    const double r = sqrt(-2.0 * log(1.0 - u));  // 1 - u in (0, 1]
    double s, c;
    sincospi(2.0 * v, &s, &c);
    *a = r * c;
    *b = r * s;
  }
};
enum { kStTheta = 0, kStPattern = 1, kStCoeff = 2, kStNoise = 3 };

__device__ double wrap_d(double x, double y) {  // simdata.py:50-53
  double d = fabs(x - y);
  d = d - floor(d);
  return d < 1.0 - d ? d : 1.0 - d;
}

// Per-CTA reduction of one double (fixed order: deterministic).
__device__ double cta_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double acc = 0.0;
  for (int j = 0; j < nw; ++j) acc += red[j];
  __syncthreads();
  return acc;
}

// smem: [n] observed flags (int), reduction scratch
__global__ void __launch_bounds__(kSimThreads) sim_generate_kernel(
    unsigned long long seed, unsigned point, int n, int m, int k, int G, double snr_db, double min_sep,
    int pairs, double intra_sep, cplx* __restrict__ y, int* __restrict__ idx, double* __restrict__ theta,
    cplx* __restrict__ alpha, double* __restrict__ beta, int* __restrict__ status, unsigned char* scratch) {
  extern __shared__ double red[];
  const int t = blockIdx.x;
  const unsigned k0 = (unsigned)seed ^ (point * 0x85EBCA6Bu), k1 = (unsigned)(seed >> 32) + point;
  const Stream sth{k0, k1, (unsigned)t, kStTheta}, spa{k0, k1, (unsigned)t, kStPattern},
      sco{k0, k1, (unsigned)t, kStCoeff}, sno{k0, k1, (unsigned)t, kStNoise};
  int* flag = (int*)(scratch + (size_t)t * n * sizeof(int));
  int* ti = idx + (size_t)t * m;
  double* th = theta + (size_t)t * k;
  cplx* al = alpha + (size_t)t * G * k;
  cplx* yt = y + (size_t)t * G * m;
  __shared__ int s_ok;
  // ---- pattern (simdata.py:78-86): Floyd's sampling of M - 2 of the inner
  // positions 2..N-1 (1-based) on a flag map, then an ordered compaction
  for (int i = threadIdx.x; i < n; i += blockDim.x) flag[i] = (m == n) ? 1 : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_ok = 1;
    if (m < n) {
      flag[0] = 1;
      flag[n - 1] = 1;
      const int pop = n - 2, draw = m - 2;
      for (int j = pop - draw, d = 0; j < pop; ++j, ++d) {  // Floyd: a uniform subset of size draw
        double u, v;
        spa.uniform2((unsigned)d, &u, &v);
        int r = (int)(u * (double)(j + 1));
        if (r > j) r = j;
        if (flag[1 + r]) r = j;
        flag[1 + r] = 1;
      }
    }
    // ---- frequencies by sequential rejection (simdata.py:61-73); pairs mode
    // (generate_pairs :125-149): base and base + intra_sep, the others > min_sep away
    unsigned d = 0;
    const int units = pairs ? k / 2 : k;
    for (int c = 0; c < units && s_ok; ++c) {
      int placed = 0;
      for (int tries = 0; tries < kMaxRejections; ++tries) {
        double u, v;
        sth.uniform2(d++, &u, &v);
        if (!pairs) {
          bool ok = true;
          for (int j = 0; j < c; ++j)
            if (!(wrap_d(u, th[j]) > min_sep)) { ok = false; break; }
          if (ok) { th[c] = u; placed = 1; break; }
        } else {
          double second = u + intra_sep;
          second -= floor(second);
          bool ok = true;
          for (int j = 0; j < 2 * c && ok; ++j)
            if (!(wrap_d(u, th[j]) > min_sep) || !(wrap_d(second, th[j]) > min_sep)) ok = false;
          if (ok) { th[2 * c] = u; th[2 * c + 1] = second; placed = 1; break; }
        }
      }
      if (!placed) s_ok = 0;
    }
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) status[t] = 1;  // InfeasibleSeparation (simdata.py:70-73)
    return;
  }
  // ordered compaction of the observed positions (0-based)
  if (threadIdx.x == 0) {
    int c = 0;
    for (int i = 0; i < n; ++i)
      if (flag[i]) ti[c++] = i;
  }
  __syncthreads();
  // ---- coefficients (simdata.py:56-58): a = CN(0, 0.8^2) + 0.2 e^{j arg a}
  for (int e = threadIdx.x; e < G * k; e += blockDim.x) {
    double a, b;
    sco.normal2((unsigned)e, &a, &b);
    const double sd = kCoeffStd / sqrt(2.0);
    a *= sd;
    b *= sd;
    const double r = hypot(a, b);
    al[e] = r > 0.0 ? mk(a + kCoeffOffset * a / r, b + kCoeffOffset * b / r) : mk(kCoeffOffset, 0.0);
  }
  __syncthreads();
  // ---- clean samples y_g(i) = sum_k alpha_gk e^{j 2 pi n_i theta_k}, energy
  double part = 0.0;
  for (int e = threadIdx.x; e < G * m; e += blockDim.x) {
    const int g = e / m, i = e - g * m;
    const double ni = (double)ti[i];
    cplx acc = mk(0.0, 0.0);
    for (int c = 0; c < k; ++c) acc = cadd(acc, cmul(al[g * k + c], expj2pi(ni, th[c], 1.0)));
    yt[e] = acc;
    part += cabs2(acc);
  }
  const double energy = cta_sum(part, red) / (double)G;
  const double b_ = energy / ((double)m * pow(10.0, snr_db / 10.0));  // simdata.py:96-97
  const double sc = sqrt(b_ / 2.0);
  for (int e = threadIdx.x; e < G * m; e += blockDim.x) {
    double a, b;
    sno.normal2((unsigned)e, &a, &b);
    yt[e] = cadd(yt[e], mk(sc * a, sc * b));
  }
  if (threadIdx.x == 0) {
    beta[t] = b_;
    status[t] = 0;
  }
}

// NMSE (simdata.py:160-169) and CSR (:196-205) per trial; mind[t, j] = the
// wrap distance from true component j to its nearest estimate (host BSR).
__global__ void __launch_bounds__(kSimThreads) sim_metrics_kernel(
    int n, int G, const double* __restrict__ th_true, const cplx* __restrict__ al_true, int k,
    const double* __restrict__ th_est, const cplx* __restrict__ al_est, const int* __restrict__ khat,
    int kstride, double* __restrict__ nmse, double* __restrict__ csr, double* __restrict__ mind) {
  extern __shared__ double red[];
  const int t = blockIdx.x;
  const int kh = khat[t];
  const double* tt = th_true + (size_t)t * k;
  const cplx* at = al_true + (size_t)t * G * k;
  const double* te = th_est + (size_t)t * kstride;
  const cplx* ae = al_est + (size_t)t * G * kstride;
  double num = 0.0, den = 0.0;
  for (int e = threadIdx.x; e < G * n; e += blockDim.x) {
    const int g = e / n;
    const double ni = (double)(e - g * n);
    cplx c = mk(0.0, 0.0), s = mk(0.0, 0.0);
    for (int j = 0; j < k; ++j) c = cadd(c, cmul(at[g * k + j], expj2pi(ni, tt[j], 1.0)));
    for (int j = 0; j < kh; ++j) s = cadd(s, cmul(ae[g * kstride + j], expj2pi(ni, te[j], 1.0)));
    num += cabs2(csub(s, c));
    den += cabs2(c);
  }
  num = cta_sum(num, red);
  den = cta_sum(den, red);
  const double radius = 0.5 / (double)n;  // simdata.py:21
  double hits = 0.0;
  for (int j = threadIdx.x; j < k + kh; j += blockDim.x) {
    const bool est = j >= k;
    const double x = est ? te[j - k] : tt[j];
    double best = 1.0;
    const int other = est ? k : kh;
    for (int q = 0; q < other; ++q) {
      const double d = wrap_d(x, est ? tt[q] : te[q]);
      best = d < best ? d : best;
    }
    if (other > 0 && best < radius) hits += 1.0;
    if (!est) mind[(size_t)t * k + j] = other > 0 ? best : 1.0;
  }
  hits = cta_sum(hits, red);
  if (threadIdx.x == 0) {
    nmse[t] = num / den;
    csr[t] = (k + kh) ? hits / (double)(k + kh) : 0.0;
  }
}

int sim_fail(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e - 1000; }
}  // namespace

extern "C" {

size_t slse_sim_workspace_bytes(int n, int trials) { return (size_t)trials * n * sizeof(int); }

int slse_sim_generate(unsigned long long seed, unsigned point, int trials, int n, int m, int k, int G, double snr_db,
                      double min_sep, int pairs, double intra_sep, double* y, int32_t* idx, double* theta,
                      double* alpha, double* beta, int32_t* status, void* workspace, void* stream) {
  if (trials < 0 || n < 2 || m < 2 || m > n || k < 0 || G < 1 || (pairs && (k & 1))) return -1;
  if (trials == 0) return 0;
  sim_generate_kernel<<<trials, kSimThreads, (kSimThreads / 32) * sizeof(double), (cudaStream_t)stream>>>(
      seed, point, n, m, k, G, snr_db, min_sep, pairs, intra_sep, (cplx*)y, idx, theta, (cplx*)alpha, beta, status,
      (unsigned char*)workspace);
  return sim_fail(cudaGetLastError());
}

int slse_sim_metrics(int trials, int n, int G, const double* theta_true, const double* alpha_true, int k,
                     const double* theta_est, const double* alpha_est, const int32_t* k_hat, int kstride,
                     double* nmse, double* csr, double* mind, void* stream) {
  if (trials < 0 || n < 1 || G < 1 || k < 0 || kstride < 1) return -1;
  if (trials == 0) return 0;
  sim_metrics_kernel<<<trials, kSimThreads, (kSimThreads / 32) * sizeof(double), (cudaStream_t)stream>>>(
      n, G, theta_true, (const cplx*)alpha_true, k, theta_est, (const cplx*)alpha_est, k_hat, kstride, nmse, csr,
      mind);
  return sim_fail(cudaGetLastError());
}

}  // extern "C"
