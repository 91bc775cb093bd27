// slse_capi.cu -- sm_100a kernels and the extern "C" boundary declared in
// include/superlse_b200.h.
//
// Kernels:
//   solve_kernel<NT>      persistent: each CTA pulls problems from an atomic
//                         work queue and runs the whole estimate() for one
//                         problem (slse_solver.cuh); per-CTA workspace slab.
//   cov_kernel / factor_kernel / apply_kernel / stats_kernel / grid_kernel
//                         one CTA per problem; the per-call operators the
//                         parity tests check against the oracle.
//   tw_fill_kernel        twiddle table exp(-2 pi i k / TW).
#include "slse_kernels.cuh"
#include "slse_grid.cuh"
#include "slse_grid3.cuh"
#ifndef SLSE_R3S_MAXLG
#define SLSE_R3S_MAXLG 30
#endif

#include <cstdlib>

thread_local char g_err[512] = "";

using namespace slse_k;

namespace {


int fail(const char* what, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
  return -(int)e - 1000;
}

int fail_arg(const char* what) {
  snprintf(g_err, sizeof(g_err), "%s", what);
  return -1;
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// ---------------------------------------------------------------- twiddles
// level-major table (slse_fft.cuh tw_index): entry 2^l + k = exp(-2 pi i k / 2^l)
__global__ void tw_fill_kernel(cplx* tw, int lg) {
  const int n = (int)tw_entries(lg);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i == 0) {
      tw[0] = mk(1.0, 0.0);  // unused slot
      continue;
    }
    const int l = 31 - __clz(i);
    const int k = i - (1 << l);
    double s, c;
    // k / 2^l exact (power of two)
    sincospi(2.0 * ((double)k / (double)(1 << l)), &s, &c);
    tw[i] = mk(c, -s);
  }
}

struct TwEntry {
  cplx* ptr = nullptr;
  int lg = 0;
};
std::mutex g_tw_mu;
TwEntry g_tw[64];

constexpr int kMinTwLog = 17;  // 131072 entries (2 MiB) covers L = 4N up to N = 32768

int twiddles(int need_lg, cudaStream_t st, const cplx** out, int* out_lg) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail("cudaGetDevice", e);
  std::lock_guard<std::mutex> lk(g_tw_mu);
  TwEntry& t = g_tw[dev & 63];
  if (t.ptr == nullptr || t.lg < need_lg) {
    const int lg = need_lg > kMinTwLog ? need_lg : kMinTwLog;
    cplx* p = nullptr;
    e = cudaMalloc(&p, sizeof(cplx) * tw_entries(lg));
    if (e != cudaSuccess) return fail("cudaMalloc(twiddles)", e);
    tw_fill_kernel<<<256, 256, 0, st>>>(p, lg);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail("tw_fill_kernel", e);
    // the table is shared by every later caller, whatever stream it uses: wait
    // for the fill once before publishing it (a one-time cost per device/size)
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail("tw_fill_kernel (sync)", e);
    // older tables stay allocated: in-flight kernels may still read them
    t.ptr = p;
    t.lg = lg;
  }
  *out = t.ptr;
  *out_lg = t.lg;
  return 0;
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}


#define SLSE_DISPATCH_NT(nt, ...) \
  switch (nt) {                    \
    case 32: { constexpr int NTC = 32; __VA_ARGS__; } break; \
    case 64: { constexpr int NTC = 64; __VA_ARGS__; } break; \
    case 128: { constexpr int NTC = 128; __VA_ARGS__; } break; \
    case 256: { constexpr int NTC = 256; __VA_ARGS__; } break; \
    case 512: { constexpr int NTC = 512; __VA_ARGS__; } break; \
    default: { constexpr int NTC = 1024; __VA_ARGS__; } break; \
  }

template <class KernelT>
cudaError_t set_smem(KernelT kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

namespace {
// threads per solver CTA: small N run one warp per problem (no block-wide
// barriers; many problems resident per SM); SLSE_SOLVER_NT overrides.
// Two 256-thread solver CTAs per SM ("paired") when the batch has more
// problems than SMs and the per-problem shared region fits in half an SM:
// measured on B200 (tools/occ_exp.sh) cfg3 181 -> 130 ms, cfg4 1.00 -> 0.82 s;
// with B <= SMs (cfg5) one 512-thread CTA per problem stays faster.
constexpr size_t kPairRegion = 100 * 1024;
constexpr int kWideMaxPerSM = 5;       // N <= 512: 128-thread CTA per problem up to 5 problems per SM
constexpr int kWarpModeMinPerSM = 10;  // N <= 512: warp mode from 10 problems per SM
bool solver_paired(int n, int B, bool dnc) {
  if (slse_knob("SLSE_NO_PAIR")) return false;
  if (n <= 512 || B <= sm_count()) return false;
  return dnc || 48 * (size_t)n <= kPairRegion;
}

int solver_threads(int n, int B, bool dnc) {
  const char* env = slse_knob("SLSE_SOLVER_NT");
  if (env) {
    int v = atoi(env);
    if (v == 32 || v == 64 || v == 128 || v == 256 || v == 512 || v == 1024) return v;
  }
  // N <= 512: by batch size (measured, N = 256, tools/small_batch.sh): up to
  // 5 problems per SM one 128-thread CTA per problem is fastest (B = 148:
  // 4.4 ms vs 14.3 ms in warp mode, which packs 16 problems on 10 SMs);
  // one-warp CTAs (classic, several per SM) up to 10 per SM; warp mode
  // (16 one-warp solvers per CTA, operation windows) from there (B = 4096:
  // 30.9 ms vs 68 ms classic)
  if (n <= 512) return B <= kWideMaxPerSM * sm_count() ? 128 : 32;
  if (solver_paired(n, B, dnc)) return 256;
  if (n <= 2048) return 256;  // cfg3: 167 ms (256) vs 205 (128) / 236 (512) per 1024 x N=1024
  return 512;                 // cfg4/5 with B <= SMs (superfast): 8.8 s (512) vs 13.1 (1024) / 12 (128) at cfg5
}

// Warp mode: the one-warp solvers run W per CTA (one CTA per SM) with a
// CTA-wide rendezvous per heavy operation (slse_solve_warps.cu).  Returns
// W (16, 8 or 4 -- as many as the per-warp shared memory allows), or 0 when
// the classic one-problem-per-CTA kernel is used (nt > 32, SLSE_NO_WARPS).
int warps_per_cta(int nt, bool dnc, const SmemPlan& plan, int* warp_smem, int B) {
  if (nt != 32 || dnc || slse_knob("SLSE_NO_WARPS")) return 0;  // (the superfast factor keeps CTA-static scratch)
  if (B < kWarpModeMinPerSM * sm_count()) return 0;  // classic one-warp CTAs (see solver_threads)
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t ws = red_bytes(32) + (plan.bytes - head_bytes(32));
  *warp_smem = (int)ws;
  for (int W = 16; W >= 4; W >>= 1)
    if (kCfBytes + (size_t)W * ws <= (size_t)optin) return W;
  return 0;
}

// One problem per 2-CTA cluster (slse_split.cuh) when the superfast batch
// leaves at least half the SMs idle (cfg5: 64 problems on 148 SMs).
bool solver_pair(int n, int B, bool dnc) {
  if (slse_knob("SLSE_NO_CTA_PAIR")) return false;
  return dnc && solver_threads(n, B, dnc) == 512 && 2 * B <= sm_count();
}

int grid_size_for_solver(int n, int G, int B, const slse_options& o, size_t* slab_out, SmemPlan* plan_out) {
  SolveParams P = make_params(n, o);
  const bool dnc = P.dnc != 0;
  const int nt = solver_threads(n, B, dnc);
  if (solver_pair(n, B, dnc)) {  // B clusters, one slab each (+ one job slot, see slse_estimate_batch_mmv)
    SmemPlan plan = smem_plan(n, P.L, nt, dnc, 0);
    Layout lay = make_layout(n, P.L, P.kmax, P.lbfgs_mem, false, true, G);
    *slab_out = lay.total + sizeof(SplitJob);
    if (plan_out) *plan_out = plan;
    return B < 1 ? 1 : B;
  }
  SmemPlan plan = smem_plan(n, P.L, nt, dnc, (nt == 256 && solver_paired(n, B, dnc)) ? kPairRegion : 0);
  int wsm = 0;
  if (const int W = warps_per_cta(nt, P.dnc != 0, plan, &wsm, B)) {  // one slab per warp of every CTA
    int ctas = (B + W - 1) / W;
    if (ctas > sm_count()) ctas = sm_count();
    if (ctas < 1) ctas = 1;
    Layout lay = make_layout(n, P.L, P.kmax, P.lbfgs_mem, plan.rec_in_smem != 0, P.dnc != 0, G);
    *slab_out = lay.total;
    if (plan_out) *plan_out = plan;
    return ctas * W;
  }
  int occ = 1;
  cudaError_t e = cudaSuccess;
  switch (nt) {
    case 32: e = slse_solve_occupancy_32(plan.bytes, &occ); break;
    case 64: e = slse_solve_occupancy_64(plan.bytes, &occ); break;
    case 128: e = slse_solve_occupancy_128(plan.bytes, &occ); break;
    case 256: e = slse_solve_occupancy_256(plan.bytes, &occ); break;
    case 512: e = slse_solve_occupancy_512(plan.bytes, &occ); break;
    default: e = slse_solve_occupancy_1024(plan.bytes, &occ); break;
  }
  if (e != cudaSuccess) return fail("solver occupancy", e);
  if (occ < 1) occ = 1;
  int g = sm_count() * occ;
  if (g > B) g = B;
  if (g < 1) g = 1;
  Layout lay = make_layout(n, P.L, P.kmax, P.lbfgs_mem, plan.rec_in_smem != 0, P.dnc != 0, G);
  *slab_out = lay.total;
  if (plan_out) *plan_out = plan;
  return g;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int slse_abi_version(void) { return SLSE_ABI_VERSION; }

const char* slse_last_error(void) { return g_err; }

int slse_device_info(int* sms, int* smem_optin, int* major, int* minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail("cudaGetDevice", e);
  if (sms) cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
  if (smem_optin) cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (major) cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  if (minor) cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  return 0;
}

void slse_default_options(slse_options* o) {
  o->grid_factor = 8;
  o->tau = 5.0;
  o->max_outer_iterations = 200;
  o->convergence_tol_scale = 1e-7;
  o->lbfgs_inner_max = 5;
  o->newton_decrement_tol_scale = 1e-8;
  o->initial_sweep_iterations = 3;
  o->lbfgs_memory = 10;
  o->k_max = 0;
  o->trace_capacity = 0;
  o->event_capacity = 0;
  o->decomp_method = 0;
  o->k_cap = 0;
}

int slse_cov_column(const double* theta, const double* gamma, const int32_t* kcount, int kstride, const double* beta,
                    int N, int B, double* c, void* stream) {
  if (N < 1 || B < 0 || kstride < 0) return fail_arg("slse_cov_column: bad sizes");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int nt = block_threads(N);
  SLSE_DISPATCH_NT(nt, { cov_kernel<NTC><<<B, NTC, kRedBytes, st>>>(theta, gamma, kcount, kstride, beta, N, (cplx*)c); });
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail("cov_kernel", e);
}

int slse_toeplitz_factor(const double* c, int N, int B, double* rho, double* delta, double* logdet, int32_t* status,
                         void* stream) {
  return slse_toeplitz_factor_ex(c, N, B, rho, delta, logdet, status, 0, stream);
}

int slse_toeplitz_factor_ex(const double* c, int N, int B, double* rho, double* delta, double* logdet,
                            int32_t* status, int method, void* stream) {
  if (N < 1 || B < 0 || method < 0 || method > 2) return fail_arg("slse_toeplitz_factor: bad arguments");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (use_dnc(N, method)) {
    const cplx* tw;
    int twlog;
    const int F = 1 << ilog2(N);
    int rc = twiddles(ilog2(F > 16 ? F : 16), st, &tw, &twlog);
    if (rc) return rc;
    const int nt = N <= 2048 ? 256 : 512;  // 1024 threads cap registers at 64 and the leaves spill
    int cap = 1;
    while (16 * (size_t)sk_len(cap * 2) <= kRegionBudget) cap *= 2;
    if (cap > F) cap = F;
    cap = sk_len(cap);  // staging capacity in the skewed layout
    const size_t smem = kHeadBytes + 16 * (size_t)cap;
    const size_t per = 4 * (size_t)N + dnc_arena_elems(N - 1) + 16;
    cplx* scratch = nullptr;
    double* dscr = nullptr;
    cudaError_t e = cudaMallocAsync(&scratch, sizeof(cplx) * per * B, st);
    if (e != cudaSuccess) return fail("cudaMallocAsync", e);
    e = cudaMallocAsync(&dscr, sizeof(double) * (size_t)N * B, st);
    if (e != cudaSuccess) return fail("cudaMallocAsync", e);
    SLSE_DISPATCH_NT(nt, {
      e = set_smem(factor_dnc_kernel<NTC>, smem);
      if (e == cudaSuccess) {
        const char* dd = slse_knob("SLSE_DNC_DIRECT_MAX");
        long long* prof = nullptr;
        if (slse_knob("SLSE_DNC_PROF")) {  // debug: phase clocks of problem 0, printed to stderr
          cudaMalloc(&prof, 16 * sizeof(long long));
          cudaMemsetAsync(prof, 0, 16 * sizeof(long long), st);
        }
        factor_dnc_kernel<NTC><<<B, NTC, smem, st>>>((const cplx*)c, N, (cplx*)rho, delta, logdet, status, scratch, per,
                                                    dscr, tw, twlog, cap, dd ? atoi(dd) : SLSE_DNC_DIRECT, prof);
        if (prof) {
          long long h[16];
          cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          fprintf(stderr, "[dnc prof N=%d] leaf %lld direct1 %lld direct2 %lld fft1 %lld fft2 %lld total %lld cycles;"
                          " fft by F=512..: %lld %lld %lld %lld %lld %lld\n",
                  N, h[0], h[1], h[2], h[3], h[4], h[5], h[8], h[9], h[10], h[11], h[12], h[13]);
          cudaFree(prof);
        }
        e = cudaGetLastError();
      }
    });
    cudaFreeAsync(scratch, st);
    cudaFreeAsync(dscr, st);
    return e == cudaSuccess ? 0 : fail("factor_dnc_kernel", e);
  }
  const int nt = block_threads(N);
  const size_t rec = 48 * (size_t)N;
  const int rec_smem = rec <= kRegionBudget ? 1 : 0;
  const size_t smem = kHeadBytes + (rec_smem ? rec : 0);
  cplx* scratch = nullptr;
  double* dscr = nullptr;
  cudaError_t e = cudaMallocAsync(&dscr, sizeof(double) * (size_t)N * B, st);
  if (e != cudaSuccess) return fail("cudaMallocAsync", e);
  if (!rec_smem) {
    e = cudaMallocAsync(&scratch, sizeof(cplx) * 3 * (size_t)N * B, st);
    if (e != cudaSuccess) return fail("cudaMallocAsync", e);
  }
  SLSE_DISPATCH_NT(nt, {
    e = set_smem(factor_kernel<NTC>, smem);
    if (e == cudaSuccess) {
      factor_kernel<NTC><<<B, NTC, smem, st>>>((const cplx*)c, N, (cplx*)rho, delta, logdet, status, scratch, dscr,
                                              rec_smem);
      e = cudaGetLastError();
    }
  });
  if (scratch) cudaFreeAsync(scratch, st);
  cudaFreeAsync(dscr, st);
  return e == cudaSuccess ? 0 : fail("factor_kernel", e);
}

int slse_gs_apply(const double* rho, const double* delta_last, const double* y, int N, int B, double* w, double* quad,
                  void* stream) {
  if (N < 1 || B < 0) return fail_arg("slse_gs_apply: bad sizes");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* tw;
  int twlog;
  const int nf = 1 << ilog2(2 * N);
  int rc = twiddles(ilog2(nf), st, &tw, &twlog);
  if (rc) return rc;
  const int nt = block_threads(N);
  int cap = 16 * (size_t)nf <= kRegionBudget ? nf : 0;
  const size_t smem = kHeadBytes + 16 * (size_t)cap;
  cplx* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(cplx) * 4 * (size_t)nf * B, st);
  if (e != cudaSuccess) return fail("cudaMallocAsync", e);
  SLSE_DISPATCH_NT(nt, {
    e = set_smem(apply_kernel<NTC>, smem);
    if (e == cudaSuccess) {
      apply_kernel<NTC><<<B, NTC, smem, st>>>((const cplx*)rho, delta_last, (const cplx*)y, N, (cplx*)w, quad, scratch,
                                             tw, twlog, cap);
      e = cudaGetLastError();
    }
  });
  cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? 0 : fail("apply_kernel", e);
}

int slse_omegas(const double* rho, const double* delta_last, int N, int B, double* om_s, double* om_t, double* om_v,
                double* om_x, void* stream) {
  if (N < 2 || B < 0) return fail_arg("slse_omegas: need N >= 2");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int nf = 1 << ilog2(2 * N - 1);
  const cplx* tw;
  int twlog;
  int rc = twiddles(ilog2(nf), st, &tw, &twlog);
  if (rc) return rc;
  CfTable cft;
  cf_build(cft, N);
  const int nt = block_threads(N);
  const int cap = 16 * (size_t)sk_len(nf) <= kRegionBudget ? sk_len(nf) : 0;
  const size_t smem = kHeadBytes + 16 * (size_t)cap;
  cplx* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(cplx) * 9 * (size_t)nf * B, st);
  if (e != cudaSuccess) return fail("cudaMallocAsync", e);
  SLSE_DISPATCH_NT(nt, {
    e = set_smem(omegas_kernel<NTC>, smem);
    if (e == cudaSuccess) {
      omegas_kernel<NTC><<<B, NTC, smem, st>>>(cft, (const cplx*)rho, delta_last, N, (cplx*)om_s, (cplx*)om_t,
                                              (cplx*)om_v, (cplx*)om_x, scratch, tw, twlog, cap);
      e = cudaGetLastError();
    }
  });
  cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? 0 : fail("omegas_kernel", e);
}

int slse_activation_curve(const double* q_grid, const double* s_grid, const double* gamma_bar, const double* zeta,
                          int kmax, int L, int B, double* curve, int32_t* argmin, void* stream) {
  if (L < 1 || B < 0 || kmax < 1 || argmin == nullptr) return fail_arg("slse_activation_curve: bad arguments");
  if (B == 0) return 0;
  act_curve_kernel<256><<<B, 256, kHeadBytes, (cudaStream_t)stream>>>((const cplx*)q_grid, s_grid, gamma_bar, zeta,
                                                                       kmax, L, curve, argmin);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail("act_curve_kernel", e);
}

int slse_deactivation_margins(const double* q, const double* s, const double* gamma, const int32_t* kcount,
                              int kstride, const double* zeta, int kmax, int B, double* margin, int32_t* argmin,
                              void* stream) {
  if (kstride < 1 || B < 0 || kmax < 1 || argmin == nullptr) return fail_arg("slse_deactivation_margins: bad arguments");
  if (B == 0) return 0;
  deact_kernel<128><<<B, 128, kHeadBytes, (cudaStream_t)stream>>>((const cplx*)q, s, gamma, kcount, kstride, zeta,
                                                                  kmax, margin, argmin);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail("deact_kernel", e);
}

int slse_gradient_hessian(const double* q, const double* r, const double* u, const double* s, const double* t,
                          const double* v, const double* x, const double* gamma, const int32_t* kcount, int kstride,
                          int N, int B, double* g, double* d, void* stream) {
  if (kstride < 1 || B < 0 || N < 1) return fail_arg("slse_gradient_hessian: bad arguments");
  if (B == 0) return 0;
  const long long tot = (long long)B * kstride;
  grad_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const cplx*)q, (const cplx*)r, (const cplx*)u, s, (const cplx*)t, (const cplx*)v, x, gamma, kcount, kstride, B,
      N, g, d);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail("grad_kernel", e);
}

int slse_component_stats(const double* theta, const int32_t* kcount, int kstride, const double* rho,
                         const double* delta_last, const double* w, int N, int B, double* q, double* r, double* u,
                         double* s, double* t, double* v, double* x, void* stream) {
  if (N < 1 || B < 0) return fail_arg("slse_component_stats: bad sizes");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  CfTable cft;
  cf_build(cft, N);
  // at most 512 threads: the two-chain sums (component_stats) need ~100
  // registers, which 1024-thread blocks cannot give (measured 10x slower)
  const int nt = block_threads(N) < 512 ? block_threads(N) : 512;
  cudaError_t e = cudaSuccess;
  SLSE_DISPATCH_NT(nt, {
    stats_kernel<NTC><<<B, NTC, kHeadBytes, st>>>(cft, theta, kcount, kstride, (const cplx*)rho, delta_last,
                                                 (const cplx*)w, N, (cplx*)q, (cplx*)r, (cplx*)u, s, (cplx*)t,
                                                 (cplx*)v, x);
    e = cudaGetLastError();
  });
  return e == cudaSuccess ? 0 : fail("stats_kernel", e);
}

int slse_grid_eval(const double* rho, const double* delta_last, const double* w, int N, int L, int B, double* q_grid,
                   double* s_grid, void* stream) {
  if (N < 1 || !pow2(L) || L < N || B < 0) return fail_arg("slse_grid_eval: L must be a power of two >= N");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* tw;
  int twlog;
  int rc = twiddles(ilog2(L), st, &tw, &twlog);
  if (rc) return rc;
  cudaError_t e = cudaSuccess;
  // L = 1024, 128 < N <= 256 (cfg2): v5 (slse_grid.cuh), two-pass transform,
  // TMA bulk input prefetch, persistent CTAs
  if (L == 1024 && N > 128 && N <= 256) {
    const size_t smem = g5_smem_bytes();
    e = set_smem(grid_tma_kernel, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_tma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_tma_kernel, kG5Threads, smem);
    if (e == cudaSuccess && occ > 0) {
      int g = sm_count() * occ;
      if (g > B) g = B;
      grid_tma_kernel<<<g, kG5Threads, smem, st>>>((const cplx*)rho, delta_last, (const cplx*)w, N, B, (cplx*)q_grid,
                                                  s_grid, tw, twlog);
      e = cudaGetLastError();
      return e == cudaSuccess ? 0 : fail("grid_tma_kernel", e);
    }
    if (e != cudaSuccess) return fail("grid_tma_kernel setup", e);
  }
  const char* gmin = slse_knob("SLSE_GRES_MIN_L");  // experiment override of the residue-kernel threshold
  if (L >= (gmin ? atoi(gmin) : 8192) && N >= 64 && !slse_knob("SLSE_GRID_OLD")) {
    // residue decomposition (slse_grid.cuh): R transforms of M <= 2048 points
    // per signal, three per task staged in shared memory.  Measured at the
    // cfg4 / cfg5 shapes (batches > 2x L2): 374 us (14.4 % of HBM) vs 2208 us
    // for the generic passes through global scratch, 608 vs 4076 us; at
    // L = 4096 (cfg3) the register-Stockham kernel below stays faster (243 vs 283 us)
    const int lgM = ilog2(N) < 11 ? ilog2(N) : 11;
#define SLSE_GRID_RES(NTV, LGMV)                                                                            \
  case LGMV: {                                                                                              \
    const size_t smem = 3 * 16 * (size_t)sk_len(1 << LGMV);                                                 \
    e = set_smem(grid_res_kernel<NTV, LGMV>, smem);                                                         \
    int occ = 0;                                                                                            \
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_res_kernel<NTV, LGMV>, NTV, smem); \
    if (e != cudaSuccess || occ < 1) return fail("grid_res_kernel setup", e);                               \
    long long g = (long long)sm_count() * occ;                                                              \
    const long long tasks = (long long)B << (ilog2(L) - LGMV);                                              \
    if (g > tasks) g = tasks;                                                                               \
    grid_res_kernel<NTV, LGMV><<<(int)g, NTV, smem, st>>>((const cplx*)rho, delta_last, (const cplx*)w, N,   \
                                                          ilog2(L), B, (cplx*)q_grid, s_grid, tw, twlog);   \
    e = cudaGetLastError();                                                                                 \
    return e == cudaSuccess ? 0 : fail("grid_res_kernel", e);                                               \
  }
    switch (lgM) {
      SLSE_GRID_RES(128, 6)
      SLSE_GRID_RES(128, 7)
      SLSE_GRID_RES(128, 8)
      SLSE_GRID_RES(128, 9)
      SLSE_GRID_RES(192, 10)
      SLSE_GRID_RES(384, 11)
      default: break;
    }
#undef SLSE_GRID_RES
  }
  {
    const int lg = ilog2(L);
    int q = 0;
    while (q < 3 && (N << (q + 1)) <= L) ++q;  // input support n <= L / 2^q
    // v3 (fused last pass) for the other L = 2^10 shapes
    if (lg == 10) {
#define SLSE_GRID3_Q(NTV, LGV, QV)                                                                         \
  case QV: {                                                                                               \
    const size_t ssmem = head_bytes(NTV) + 48 * (size_t)sk_len(1 << LGV);                                  \
    e = set_smem(grid_fused_kernel<NTV, LGV, QV>, ssmem);                                                  \
    if (e == cudaSuccess) {                                                                                \
      grid_fused_kernel<NTV, LGV, QV><<<B, NTV, ssmem, st>>>((const cplx*)rho, delta_last, (const cplx*)w, N,   \
                                                            (cplx*)q_grid, s_grid, tw, twlog);             \
      e = cudaGetLastError();                                                                              \
    }                                                                                                      \
    return e == cudaSuccess ? 0 : fail("grid_fused_kernel", e);                                            \
  }
      switch (q) { SLSE_GRID3_Q(256, 10, 0) SLSE_GRID3_Q(256, 10, 1) SLSE_GRID3_Q(256, 10, 2) SLSE_GRID3_Q(256, 10, 3) }
#undef SLSE_GRID3_Q
    }
    // register-Stockham kernel: 3 L-point transforms resident in shared
    // memory, compile-time pass schedules for L = 2^6 .. 2^12, pruned first pass
#define SLSE_GRID_Q(NTV, LGV, QV)                                                                          \
  case QV: {                                                                                               \
    const size_t ssmem = head_bytes(NTV) + 48 * (size_t)sk_len(1 << LGV);                                  \
    e = set_smem(grid_stockham_kernel<NTV, LGV, QV>, ssmem);                                               \
    if (e == cudaSuccess) {                                                                                \
      grid_stockham_kernel<NTV, LGV, QV><<<B, NTV, ssmem, st>>>((const cplx*)rho, delta_last, (const cplx*)w, N, \
                                                               (cplx*)q_grid, s_grid, tw, twlog);          \
      e = cudaGetLastError();                                                                              \
    }                                                                                                      \
    return e == cudaSuccess ? 0 : fail("grid_stockham_kernel", e);                                         \
  }
#define SLSE_GRID_CASE(LGV, NTV)                                                \
  case LGV:                                                                     \
    switch (q) {                                                                \
      SLSE_GRID_Q(NTV, LGV, 0) SLSE_GRID_Q(NTV, LGV, 1) SLSE_GRID_Q(NTV, LGV, 2) SLSE_GRID_Q(NTV, LGV, 3) \
    }                                                                           \
    break;
    switch (lg) {
      SLSE_GRID_CASE(6, 32)
      SLSE_GRID_CASE(7, 32)
      SLSE_GRID_CASE(8, 64)
      SLSE_GRID_CASE(9, 96)
      SLSE_GRID_CASE(11, 384)
      SLSE_GRID_CASE(12, 768)
      default: break;
    }
#undef SLSE_GRID_CASE
#undef SLSE_GRID_Q
  }
  // L > 4096 (and L < 64): one CTA per problem, radix-2/4 passes over the
  // three transforms in shared memory when they fit, else through global scratch
  const int nt = block_threads(N);
  const int fused = 48 * (size_t)L <= kRegionBudget ? 1 : 0;
  const size_t smem = kHeadBytes + (fused ? 48 * (size_t)L : 0);
  cplx* scratch = nullptr;
  if (!fused) {
    e = cudaMallocAsync(&scratch, sizeof(cplx) * 2 * (size_t)L * B, st);
    if (e != cudaSuccess) return fail("cudaMallocAsync", e);
  }
  SLSE_DISPATCH_NT(nt, {
    e = set_smem(grid_kernel<NTC>, smem);
    if (e == cudaSuccess) {
      grid_kernel<NTC><<<B, NTC, smem, st>>>((const cplx*)rho, delta_last, (const cplx*)w, N, L, (cplx*)q_grid, s_grid,
                                            scratch, tw, twlog, fused);
      e = cudaGetLastError();
    }
  });
  if (scratch) cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? 0 : fail("grid_kernel", e);
}

int slse_grid_eval_omega(const double* w, const double* om_s, int N, int L, int B, double* q_grid, double* s_grid,
                         void* stream) {
  // the reference's grid length is a power of two >= 2N (model_core.py:224-227);
  // below 2N - 1 its buffer placement would alias om_s(i) and om_s(i - L)
  if (N < 1 || !pow2(L) || L < 2 * N - 1 || B < 0)
    return fail_arg("slse_grid_eval_omega: L must be a power of two >= 2N - 1");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* tw;
  int twlog;
  int rc = twiddles(ilog2(L), st, &tw, &twlog);
  if (rc) return rc;
  cudaError_t e = cudaSuccess;
  if (L == 1024 && N > 128 && N <= 256) {
    // cfg2 shape: two-pass exchange, TMA bulk input stages, persistent CTAs
    const size_t smem = gc_smem_bytes();
    e = set_smem(grid_coef_kernel, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_coef_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_coef_kernel, kGCThreads, smem);
    if (e != cudaSuccess || occ < 1) return fail("grid_coef_kernel setup", e);
    int g = sm_count() * occ;
    if (g > B) g = B;
    grid_coef_kernel<<<g, kGCThreads, smem, st>>>((const cplx*)w, (const cplx*)om_s, N, B, (cplx*)q_grid, s_grid, tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_coef_kernel", e);
  }
  const int lgL = ilog2(L);
  if (lgL >= 14 && lgL <= SLSE_R3S_MAXLG && 4LL * N <= L && !slse_knob("SLSE_GRID_NO_R3P")) {
    // residue pairs (whole-sector stores), s^G at half length (slse_grid3.cuh).  From L = 65536 the
    // folds (4 for q^G, 8 for the half-length s^G, re-read per residue) outweigh the store savings:
    // cfg5 shape 1.82 ms here vs 1.40 ms on the single-residue tasks below.
    const long long tasks = (long long)B * (3 << (lgL - 14));
    const size_t smem = r3s_smem_bytes();
    e = set_smem(grid_r3s_kernel, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_r3s_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_r3s_kernel, kR3Threads, smem);
    if (e != cudaSuccess || occ < 1) return fail("grid_r3s_kernel setup", e);
    long long g = (long long)sm_count() * occ;
    if (g > tasks) g = tasks;
    grid_r3s_kernel<<<(int)g, kR3Threads, smem, st>>>((const cplx*)w, (const cplx*)om_s, N, lgL, B, (cplx*)q_grid,
                                                      s_grid, tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_r3s_kernel", e);
  }
  if (L == 256 && N <= 64 && !slse_knob("SLSE_GRID_NO_C1")) {
    // cfg1 shape: one warp per problem, two DFT16 passes through a warp-local exchange
    const size_t smem = c1_smem_bytes();
    e = set_smem(grid_c1_kernel, smem);
    int occ = 0;
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_c1_kernel, 32 * kC1Warps, smem);
    if (e != cudaSuccess || occ < 1) return fail("grid_c1_kernel setup", e);
    long long g = (long long)sm_count() * occ;
    const long long ctas = ((long long)B + kC1Warps - 1) / kC1Warps;
    if (g > ctas) g = ctas;
    grid_c1_kernel<<<(int)g, 32 * kC1Warps, smem, st>>>((const cplx*)w, (const cplx*)om_s, N, B, (cplx*)q_grid, s_grid,
                                                        tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_c1_kernel", e);
  }
  if (lgL == 12 && N <= 1024 && !slse_knob("SLSE_GRID_NO_R3C")) {
    // cfg3 shape: pruned 4096-point register transforms, s^G of two problems per transform
    const size_t smem = r3_smem_bytes();
    e = set_smem(grid_r3c_kernel, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_r3c_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_r3c_kernel, kR3Threads, smem);
    if (e != cudaSuccess || occ < 1) return fail("grid_r3c_kernel setup", e);
    long long g = (long long)sm_count() * occ;
    const long long tasks = 3LL * ((B + 1) / 2);
    if (g > tasks) g = tasks;
    grid_r3c_kernel<<<(int)g, kR3Threads, smem, st>>>((const cplx*)w, (const cplx*)om_s, N, B, (cplx*)q_grid, s_grid,
                                                      tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_r3c_kernel", e);
  }
  if (lgL >= 12 && !slse_knob("SLSE_GRID_NO_R3")) {
    // dense 4096-point register transforms per (problem, signal, residue) task (slse_grid3.cuh)
    const size_t smem = r3_smem_bytes();
    e = set_smem(grid_r3_kernel, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_r3_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_r3_kernel, kR3Threads, smem);
    if (e != cudaSuccess || occ < 1) return fail("grid_r3_kernel setup", e);
    long long g = (long long)sm_count() * occ;
    const long long tasks = ((long long)B * 2) << (lgL - 12);
    if (g > tasks) g = tasks;
    grid_r3_kernel<<<(int)g, kR3Threads, smem, st>>>((const cplx*)w, (const cplx*)om_s, N, lgL, B, (cplx*)q_grid,
                                                     s_grid, tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_r3_kernel", e);
  }
  if (L < 16) {
    const long long items = (long long)B * L;
    grid_coef_direct_kernel<<<(unsigned)((items + 127) / 128), 128, 0, st>>>((const cplx*)w, (const cplx*)om_s, N, lgL,
                                                                            B, (cplx*)q_grid, s_grid, tw);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : fail("grid_coef_direct_kernel", e);
  }
  // residue decomposition with two transforms per (problem, residue)
  int lgM = ilog2(N);
  if (lgM < 4) lgM = 4;
  if (lgM > 11) lgM = 11;
#define SLSE_GRID_RES_OM(NTV, LGMV)                                                                         \
  case LGMV: {                                                                                              \
    const size_t smem = 2 * 16 * (size_t)sk_len(1 << LGMV);                                                 \
    e = set_smem(grid_res_kernel<NTV, LGMV, true>, smem);                                                   \
    int occ = 0;                                                                                            \
    if (e == cudaSuccess)                                                                                   \
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_res_kernel<NTV, LGMV, true>, NTV, smem); \
    if (e != cudaSuccess || occ < 1) return fail("grid_res_kernel (omega) setup", e);                       \
    long long g = (long long)sm_count() * occ;                                                              \
    const long long tasks = (long long)B << (lgL - LGMV);                                                   \
    if (g > tasks) g = tasks;                                                                               \
    grid_res_kernel<NTV, LGMV, true><<<(int)g, NTV, smem, st>>>((const cplx*)om_s, nullptr, (const cplx*)w, N, \
                                                                lgL, B, (cplx*)q_grid, s_grid, tw, twlog);  \
    e = cudaGetLastError();                                                                                 \
    return e == cudaSuccess ? 0 : fail("grid_res_kernel (omega)", e);                                       \
  }
  switch (lgM) {
    SLSE_GRID_RES_OM(64, 4)
    SLSE_GRID_RES_OM(64, 5)
    SLSE_GRID_RES_OM(128, 6)
    SLSE_GRID_RES_OM(128, 7)
    SLSE_GRID_RES_OM(128, 8)
    SLSE_GRID_RES_OM(128, 9)
    SLSE_GRID_RES_OM(192, 10)
    SLSE_GRID_RES_OM(384, 11)
    default: break;
  }
#undef SLSE_GRID_RES_OM
  return fail_arg("slse_grid_eval_omega: unsupported shape");
}

size_t slse_estimate_workspace_bytes_mmv(int N, int G, int B, const slse_options* opts) {
  slse_options o;
  if (opts) o = *opts; else slse_default_options(&o);
  if (G < 1) return 0;
  size_t slab = 0;
  int g = grid_size_for_solver(N, G, B, o, &slab, nullptr);
  if (g < 0) return 0;
  return 256 + (size_t)g * slab;
}

size_t slse_estimate_workspace_bytes(int N, int B, const slse_options* opts) {
  return slse_estimate_workspace_bytes_mmv(N, 1, B, opts);
}

int slse_estimate_batch(const double* y, int N, int B, const slse_options* opts, const slse_outputs* out,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return slse_estimate_batch_mmv(y, N, 1, B, opts, out, workspace, workspace_bytes, stream);
}

int slse_estimate_batch_mmv(const double* y, int N, int G, int B, const slse_options* opts, const slse_outputs* out,
                            void* workspace, size_t workspace_bytes, void* stream) {
  slse_options o;
  if (opts) o = *opts; else slse_default_options(&o);
  if (N < 2) return fail_arg("slse_estimate_batch: need at least two observed samples");
  if (G < 1) return fail_arg("slse_estimate_batch_mmv: need at least one snapshot");
  if (o.lbfgs_memory < 1 || o.lbfgs_memory > 16) return fail_arg("slse_estimate_batch: lbfgs_memory must be 1..16");
  if (B < 0 || out == nullptr) return fail_arg("slse_estimate_batch: bad arguments");
  if (B == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  size_t slab = 0;
  SmemPlan plan;
  int g = grid_size_for_solver(N, G, B, o, &slab, &plan);
  if (g < 0) return g;
  const size_t need = 256 + (size_t)g * slab;
  if (workspace_bytes < need) {
    snprintf(g_err, sizeof(g_err), "slse_estimate_batch: workspace %zu < required %zu bytes", workspace_bytes, need);
    return -2;
  }
  SolveParams P = make_params(N, o);
  P.g = G;
  P.dnc_stockham = slse_knob("SLSE_DNC_STOCKHAM") ? 1 : 0;
  P.grid_fused = slse_knob("SLSE_GRID_UNFUSED") ? 0 : 1;
  if (const char* dd = slse_knob("SLSE_DNC_DIRECT_MAX")) P.dnc_direct = atoi(dd);
  const cplx* tw;
  int twlog;
  const int fmax = P.L > 2 * N ? P.L : (1 << ilog2(2 * N));
  int rc = twiddles(ilog2(fmax), st, &tw, &twlog);
  if (rc) return rc;
  CfTable cft;
  cf_build(cft, N);
  int* queue = (int*)workspace;
  cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(int), st);
  if (e != cudaSuccess) return fail("cudaMemsetAsync", e);
  char* ws = (char*)workspace + 256;
  const int nt = solver_threads(N, B, P.dnc != 0);
  if (solver_pair(N, B, P.dnc != 0)) {
    // g clusters; the job slots follow the slabs (slab includes one slot's bytes)
    const size_t lay_total = slab - sizeof(SplitJob);
    SplitJob* jobs = (SplitJob*)(ws + (size_t)g * lay_total);
    e = slse_solve_pair_launch_512(g, plan.bytes, st, P, cft, (const cplx*)y, B, *out, ws, lay_total, queue, tw,
                                   twlog, plan.fft_cap, jobs);
    return e == cudaSuccess ? 0 : fail("solve_kernel_pair", e);
  }
  int wsm = 0;
  if (const int W = warps_per_cta(nt, P.dnc != 0, plan, &wsm, B)) {
    const size_t smem = kCfBytes + (size_t)W * wsm;
    e = slse_solve_warps_launch(W, g / W, smem, st, P, cft, (const cplx*)y, B, *out, ws, slab, queue, tw, twlog,
                                plan.fft_cap, plan.rec_in_smem, wsm);
    return e == cudaSuccess ? 0 : fail("solve_kernel_warps", e);
  }
#define SLSE_SOLVE_ARGS g, plan.bytes, st, P, cft, (const cplx*)y, B, *out, ws, slab, queue, tw, twlog, plan.fft_cap, \
                        plan.rec_in_smem
  switch (nt) {
    case 32: e = slse_solve_launch_32(SLSE_SOLVE_ARGS); break;
    case 64: e = slse_solve_launch_64(SLSE_SOLVE_ARGS); break;
    case 128: e = slse_solve_launch_128(SLSE_SOLVE_ARGS); break;
    case 256: e = slse_solve_launch_256(SLSE_SOLVE_ARGS); break;
    case 512: e = slse_solve_launch_512(SLSE_SOLVE_ARGS); break;
    default: e = slse_solve_launch_1024(SLSE_SOLVE_ARGS); break;
  }
#undef SLSE_SOLVE_ARGS
  return e == cudaSuccess ? 0 : fail("solve_kernel", e);
}

// ------------------------------------------------------------ semifast
}  // extern "C"

namespace {
// Launch geometry of the semifast solver (slse_solve_sf.cu).
struct SfSetup {
  SolveParams P;
  size_t slab, smem;
  int fft_cap, grid;
};

int sf_setup(int N, int M, int G, int B, const slse_options& o, SfSetup* S) {
  if (N < 1 || M < 2 || M > N || G < 1 || B < 0) return fail_arg("semifast: need 2 <= M <= N, G >= 1, B >= 0");
  SolveParams P = make_params(N, o);
  P.g = G;
  P.m = M;
  P.semifast = 1;
  P.dnc = 0;
  P.kmax = o.k_max > 0 ? o.k_max : M;  // EstimationState K_max = M (estimator.py:126)
  if (o.event_capacity <= 0) P.ecap = 4 * P.kmax + 64;
  const int cap = o.k_cap > 0 ? o.k_cap : 64;
  P.kcap = cap < P.kmax ? cap : P.kmax;
  if (P.kcap < 1) P.kcap = 1;
  SmemPlan plan = smem_plan(N, P.L, kSfThreads, false);
  S->fft_cap = plan.fft_cap;
  S->smem = red_bytes(kSfThreads) + 16 * (size_t)plan.fft_cap;
  S->slab = make_layout(N, P.L, P.kmax, P.lbfgs_mem, false, false, G, 1, M, P.kcap).total;
  int occ = 1;
  cudaError_t e = slse_solve_sf_occupancy(S->smem, &occ);
  if (e != cudaSuccess) return fail("semifast occupancy", e);
  if (occ < 1) occ = 1;
  int g = sm_count() * occ;
  if (g > B) g = B;
  if (g < 1) g = 1;
  S->grid = g;
  S->P = P;
  return 0;
}
}  // namespace

extern "C" {

size_t slse_estimate_workspace_bytes_semifast(int N, int M, int G, int B, const slse_options* opts) {
  slse_options o;
  if (opts) o = *opts; else slse_default_options(&o);
  SfSetup S;
  if (sf_setup(N, M, G, B, o, &S)) return 0;
  return 256 + (size_t)S.grid * S.slab;
}

int slse_estimate_batch_semifast(const double* y, int N, int M, int G, int B, const int32_t* idx,
                                 const double* scales, int pattern_stride, const slse_options* opts,
                                 const slse_outputs* out, void* workspace, size_t workspace_bytes, void* stream) {
  slse_options o;
  if (opts) o = *opts; else slse_default_options(&o);
  if (o.lbfgs_memory < 1 || o.lbfgs_memory > 16) return fail_arg("semifast: lbfgs_memory must be 1..16");
  if (out == nullptr || idx == nullptr || (pattern_stride != 0 && pattern_stride != M))
    return fail_arg("semifast: bad pattern arguments (pattern_stride must be 0 or M)");
  if (B == 0) return 0;
  SfSetup S;
  int rc = sf_setup(N, M, G, B, o, &S);
  if (rc) return rc;
  const size_t need = 256 + (size_t)S.grid * S.slab;
  if (workspace_bytes < need) {
    snprintf(g_err, sizeof(g_err), "semifast: workspace %zu < required %zu bytes", workspace_bytes, need);
    return -2;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* tw;
  int twlog;
  rc = twiddles(ilog2(S.P.L), st, &tw, &twlog);
  if (rc) return rc;
  int* queue = (int*)workspace;
  cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(int), st);
  if (e != cudaSuccess) return fail("cudaMemsetAsync", e);
  e = slse_solve_sf_launch(S.grid, S.smem, st, S.P, (const cplx*)y, idx, (const cplx*)scales, pattern_stride, B,
                           *out, (char*)workspace + 256, S.slab, queue, tw, twlog, S.fft_cap);
  return e == cudaSuccess ? 0 : fail("solve_sf_kernel", e);
}

size_t slse_semifast_bundle_workspace_bytes(int N, int M, int G, int B, int L, int kstride) {
  if (!pow2(L) || L < N || kstride < 1) return 0;
  slse_options o;
  slse_default_options(&o);
  o.k_max = kstride;
  o.k_cap = kstride;
  SfSetup S;
  if (sf_setup(N, M, G, 1, o, &S)) return 0;
  SolveParams P = S.P;
  P.L = L;
  return (size_t)B * make_layout(N, L, P.kmax, P.lbfgs_mem, false, false, G, 1, M, P.kcap).total;
}

int slse_semifast_bundle(const double* theta, const double* gamma, const int32_t* kcount, int kstride,
                         const double* beta, const double* y, int N, int M, int G, int B, const int32_t* idx,
                         const double* scales, int pattern_stride, int L, double* data_term, double* e, double* q,
                         double* r, double* u, double* s, double* t, double* v, double* x, double* q_grid,
                         double* s_grid, int32_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  if (!pow2(L) || L < N || kstride < 1 || idx == nullptr || (pattern_stride != 0 && pattern_stride != M))
    return fail_arg("slse_semifast_bundle: L must be a power of two >= N, kstride >= 1, pattern_stride 0 or M");
  if (B == 0) return 0;
  slse_options o;
  slse_default_options(&o);
  o.k_max = kstride;
  o.k_cap = kstride;
  SfSetup S;
  int rc = sf_setup(N, M, G, 1, o, &S);
  if (rc) return rc;
  SolveParams P = S.P;
  P.L = L;
  SmemPlan plan = smem_plan(N, L, kSfThreads, false);
  const size_t smem = red_bytes(kSfThreads) + 16 * (size_t)plan.fft_cap;
  const size_t slab = make_layout(N, L, P.kmax, P.lbfgs_mem, false, false, G, 1, M, P.kcap).total;
  if (workspace_bytes < (size_t)B * slab) return fail_arg("slse_semifast_bundle: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const cplx* tw;
  int twlog;
  rc = twiddles(ilog2(L), st, &tw, &twlog);
  if (rc) return rc;
  cudaError_t err = slse_sf_bundle_launch(
      smem, st, P, theta, gamma, kcount, kstride, beta, (const cplx*)y, idx, (const cplx*)scales, pattern_stride, B,
      (char*)workspace, slab, tw, twlog, plan.fft_cap, data_term, (cplx*)e, (cplx*)q, (cplx*)r, (cplx*)u, s, (cplx*)t,
      (cplx*)v, x, (cplx*)q_grid, s_grid, status);
  return err == cudaSuccess ? 0 : fail("sf_bundle_kernel", err);
}

}  // extern "C"
