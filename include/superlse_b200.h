/*
 * superlse_b200.h -- C ABI of the B200-native Superfast LSE inner loop.
 *
 * Plain pointers and sizes only.  Every array argument is a DEVICE pointer
 * (cudaMalloc / torch CUDA storage) unless stated; complex128 arrays are
 * interleaved (re, im) doubles.  Calls are stream-ordered on `stream`
 * (a cudaStream_t passed as void*; NULL = legacy default stream) and never
 * synchronise.  Batched entry points process B independent problems; a
 * problem's slice of a (B, X) array starts at b * X.
 *
 * Return codes: 0 = launched; < 0 = launch/argument error (message in
 * slse_last_error()).  Per-problem numerical outcomes are int32 status
 * codes: 0 ok, 1 not positive definite (superlse.errors.NotPositiveDefinite,
 * toeplitz.py:141-142,191-192,249-252), 2 invalid diagonal (toeplitz.py:55-57).
 *
 * Reference interfaces replaced (paths relative to the reference package
 * pkg/src/superlse/):
 *   slse_cov_column        <- model_core.covariance_first_column :242-249
 *                             and nufft.steer_forward :126-144
 *   slse_toeplitz_factor   <- toeplitz.decompose :263-276
 *                             (levinson_durbin :121-145, generalized_schur :230-260)
 *   slse_gs_apply          <- toeplitz.apply_inverse :279-309 (+ quad, model_core.py:268-269)
 *   slse_omegas            <- toeplitz.all_diagonal_sums :415-432 (model_core.omegas :276-279)
 *   slse_component_stats   <- model_core._SuperfastBundle.stats :281-301
 *   slse_grid_eval         <- model_core._SuperfastBundle.grid :303-313
 *   slse_activation_curve  <- smlr._delta_objective_curve :62-70 + best_candidate argmin :84-96
 *   slse_deactivation_margins <- smlr.deactivation_margins :174-200 (+ try_deactivate argmin :203-225)
 *   slse_gradient_hessian  <- model_core.gradient :497-505, diag_hessian :508-536
 *   slse_estimate_batch    <- estimator.estimate :117-275 (complete data, G = 1,
 *                             backend "superfast"), one problem per batch row
 *   slse_estimate_batch_mmv <- estimator.estimate_mmv :278-283 (G >= 1 snapshots)
 *   slse_estimate_batch_semifast <- estimator.estimate :117-275 with backend "semifast"
 *                             (SemifastEngine, model_core.py:456-460; complete or
 *                             incomplete data, Observation :43-130)
 *   slse_semifast_bundle   <- model_core._SemifastBundle :316-409 (data_term, stats, grid)
 *                             with nufft.gram :184-210
 *   slse_sim_generate      <- simdata.generate :109-122 / generate_pairs :125-149 (on-device
 *                             scenes, counter-based Philox stream)
 *   slse_sim_metrics       <- simdata.nmse :160-169, csr :196-205 (+ nearest distances for
 *                             bsr_trial :185-193, whose Hungarian assignment stays on the host)
 */
#ifndef SUPERLSE_B200_H
#define SUPERLSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLSE_ABI_VERSION 3

/* EstimatorOptions (estimator.py:34-50), superfast fields. */
typedef struct slse_options {
  int grid_factor;               /* 8 */
  double tau;                    /* 5.0 (smlr.DEFAULT_TAU) */
  int max_outer_iterations;      /* 200 */
  double convergence_tol_scale;  /* 1e-7 */
  int lbfgs_inner_max;           /* 5 */
  double newton_decrement_tol_scale; /* 1e-8 */
  int initial_sweep_iterations;  /* 3 */
  int lbfgs_memory;              /* 10 (<= 16) */
  int k_max;                     /* <= 0: M */
  int trace_capacity;            /* <= 0: 2 + 13 * max_outer_iterations */
  int event_capacity;            /* <= 0: 4 * k_max + 64 */
  int decomp_method;             /* EstimatorOptions.decomp_method (toeplitz.decompose :263-276):
                                    0 "auto" (superfast from N >= 4096), 1 "levinson"
                                    (Schur-Levinson, O(N^2)), 2 "schur" (superfast
                                    divide-and-conquer generalized Schur, O(N log^2 N)) */
  int k_cap;                     /* semifast backend only: K x K matrices are sized k_cap
                                    (<= 0: min(k_max, 64)); a problem whose active set
                                    outgrows it stops with status 3 (rerun it with a
                                    larger k_cap; estimator.py does so automatically) */
} slse_options;

/* Outputs of slse_estimate_batch (device pointers, per problem b at offset
 * b * stride).  K = k_max, T = trace_capacity, E = event_capacity. */
typedef struct slse_outputs {
  int32_t* k_hat;        /* [B] */
  int32_t* status;       /* [B] 0 ok, 1 not PD, 2 invalid diagonal, 3 semifast
                                  active set outgrew k_cap */
  int32_t* iterations;   /* [B] */
  int32_t* flags;        /* [B] bit0 converged, bit1 K_max-cap warning,
                                  bit2 trace truncated, bit3 events truncated */
  double* beta;          /* [B] */
  double* zeta;          /* [B] */
  double* theta;         /* [B, K] active frequencies, slot order */
  double* gamma;         /* [B, K] */
  double* alpha;         /* [B, K] complex (posterior means) */
  int32_t* slot;         /* [B, K] slot index of each active component */
  double* trace;         /* [B, T] objective trace */
  int32_t* stage;        /* [B, T] 0 init 1 beta 2 activate 3 zeta 4 refine 5 deactivate */
  int32_t* trace_k;      /* [B, T] model order at each record */
  int32_t* n_trace;      /* [B] */
  int32_t* events;       /* [B, E, 3] (kind, slot, grid index); kind 0 sweep,
                            1 activate, 2 deactivate, -1 end-of-event */
  int32_t* n_events;     /* [B] */
  int64_t* counters;     /* [B, 4] builds, grid evals, stats evals, line-search trials */
  double* stage_seconds; /* [B, 6] activate objective beta refine deactivate total */
  double* iter_seconds;  /* [B, max_outer_iterations] wall seconds of each outer iteration
                            (LseResult.wall_time_per_stage["per_iteration"], estimator.py:165,247);
                            may be NULL */
} slse_outputs;

int slse_abi_version(void);
const char* slse_last_error(void);
/* SM count and opt-in shared memory per block of the current device. */
int slse_device_info(int* sm_count, int* smem_optin_bytes, int* cc_major, int* cc_minor);

/* default options (host struct) */
void slse_default_options(slse_options* opts);

/* Row 1: c[b, m] = beta[b] [m == 0] + sum_{k < kcount[b]} gamma[b,k] e^{j2 pi m theta[b,k]},
 * c_0 forced real.  theta/gamma rows have stride kstride. c: [B, N] complex. */
int slse_cov_column(const double* theta, const double* gamma, const int32_t* kcount, int kstride,
                    const double* beta, int N, int B, double* c, void* stream);

/* Rows 2-4: Gohberg-Semencul parameters.  c: [B, N] complex -> rho [B, N]
 * complex, delta [B, N] (may be NULL), logdet [B], status [B]. */
int slse_toeplitz_factor(const double* c, int N, int B, double* rho, double* delta, double* logdet,
                         int32_t* status, void* stream);

/* Same with an explicit algorithm: 0 auto (superfast from N >= 4096),
 * 1 Schur-Levinson O(N^2) (toeplitz.levinson_durbin role),
 * 2 superfast divide-and-conquer Schur O(N log^2 N) (toeplitz.generalized_schur). */
int slse_toeplitz_factor_ex(const double* c, int N, int B, double* rho, double* delta, double* logdet,
                            int32_t* status, int method, void* stream);

/* Row 5: w = C^{-1} y from (rho, delta_{N-1}); quad[b] = Re(y^H w) (may be NULL). */
int slse_gs_apply(const double* rho, const double* delta_last, const double* y, int N, int B,
                  double* w, double* quad, void* stream);

/* Row 7: diagonal sums omega_kind(i), i = -(N-1)..N-1 (index i + N - 1) for
 * kind = s, t, v, x; each [B, 2N-1] complex (s and x Hermitian-symmetrised
 * as toeplitz.py:428-430). */
int slse_omegas(const double* rho, const double* delta_last, int N, int B, double* om_s, double* om_t,
                double* om_v, double* om_x, void* stream);

/* Row 8: statistics at kcount[b] frequencies (rows of stride kstride).
 * q, r, u, t, v: [B, kstride] complex; s, x: [B, kstride] real. */
int slse_component_stats(const double* theta, const int32_t* kcount, int kstride, const double* rho,
                         const double* delta_last, const double* w, int N, int B, double* q,
                         double* r, double* u, double* s, double* t, double* v, double* x,
                         void* stream);

/* Row 9: activation grid.  q_grid [B, L] complex (FFT_L(w)), s_grid [B, L] real. */
int slse_grid_eval(const double* rho, const double* delta_last, const double* w, int N, int L, int B,
                   double* q_grid, double* s_grid, void* stream);

/* Row 9, the reference's own form (model_core._SuperfastBundle.grid :303-313
 * literally): q_grid = FFT_L(w), s_grid = L IFFT_L(buf).real with
 * buf[i mod L] = om_s(i), |i| < N.  om_s: [B, 2N-1] complex, index i + N - 1
 * (the slse_omegas "s" output; Hermitian, toeplitz.py:428-430, so only its
 * i >= 0 half is read).  Same outputs as slse_grid_eval.  Kernels by shape
 * (DESIGN.md 4): L = 256 / 1024 / 4096 with N <= L / 4 and every L >= 16384
 * have register-transform kernels (cfg1-cfg5 shapes), other shapes the
 * residue kernel. */
int slse_grid_eval_omega(const double* w, const double* om_s, int N, int L, int B, double* q_grid, double* s_grid,
                         void* stream);

/* Row 10: activation curve Delta L_l = log1p(gbar s_l) + ln((1-ze)/ze)
 * - |q_l|^2 / (1/gbar + s_l) over the grid (G = 1; ze = clamp(zeta[b],
 * 1/(2 kmax), 1/2)) and its argmin, lowest index on ties.  curve [B, L]
 * (may be NULL), argmin [B]. */
int slse_activation_curve(const double* q_grid, const double* s_grid, const double* gamma_bar,
                          const double* zeta, int kmax, int L, int B, double* curve, int32_t* argmin,
                          void* stream);

/* Row 11: deactivation margins of the kcount[b] active components (rows of
 * stride kstride: q complex, s and gamma real) and their argmin (lowest
 * index on ties; -1 when kcount[b] = 0).  margin [B, kstride] (may be NULL). */
int slse_deactivation_margins(const double* q, const double* s, const double* gamma, const int32_t* kcount,
                              int kstride, const double* zeta, int kmax, int B, double* margin,
                              int32_t* argmin, void* stream);

/* Row 12: gradient and diagonal Hessian in (theta, gamma) of the kcount[b]
 * components from their statistics (layout of slse_component_stats) and
 * gamma [B, kstride].  g, d: [B, 2 kstride]; row b holds the theta block
 * in [0, k) and the gamma block in [k, 2k), k = kcount[b]. */
int slse_gradient_hessian(const double* q, const double* r, const double* u, const double* s,
                          const double* t, const double* v, const double* x, const double* gamma,
                          const int32_t* kcount, int kstride, int N, int B, double* g, double* d,
                          void* stream);

/* Rows 10-15: the whole estimate() per problem.  y: [B, N] complex.
 * workspace: device buffer of slse_estimate_workspace_bytes() bytes. */
size_t slse_estimate_workspace_bytes(int N, int B, const slse_options* opts);
int slse_estimate_batch(const double* y, int N, int B, const slse_options* opts,
                        const slse_outputs* out, void* workspace, size_t workspace_bytes,
                        void* stream);

/* MMV (G >= 1 snapshots sharing the frequencies; estimator.estimate_mmv
 * :278-283, all data sums over snapshots): y is [B, G, N] complex, and the
 * outputs' alpha is [B, G, kmax] (row g = snapshot g); every other output as
 * slse_estimate_batch.  G = 1 is slse_estimate_batch. */
size_t slse_estimate_workspace_bytes_mmv(int N, int G, int B, const slse_options* opts);
int slse_estimate_batch_mmv(const double* y, int N, int G, int B, const slse_options* opts,
                            const slse_outputs* out, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Semifast (Woodbury) backend, complete or incomplete data: the whole
 * estimate() per problem with _SemifastBundle (model_core.py:316-409).
 * y: [B, G, M] complex observed samples; the observation pattern is
 * idx[M] (0-based positions, sorted, unique, < N) and scales[M] complex
 * (NULL = ones), shared by the batch (pattern_stride 0) or given per problem
 * (pattern_stride M: idx [B, M], scales [B, M]).  Outputs as slse_estimate_batch
 * with K = k_max (default M). */
size_t slse_estimate_workspace_bytes_semifast(int N, int M, int G, int B, const slse_options* opts);
int slse_estimate_batch_semifast(const double* y, int N, int M, int G, int B, const int32_t* idx,
                                 const double* scales, int pattern_stride, const slse_options* opts,
                                 const slse_outputs* out, void* workspace, size_t workspace_bytes, void* stream);

/* One semifast bundle per problem at (theta, gamma)[b, :kcount[b]] (rows of
 * stride kstride) and beta[b] on the pattern above (grid length L): data_term
 * [B] (G ln|C| + sum_g y_g^H C^-1 y_g), e [B, G, N] complex (Phi^H C^-1 y),
 * q, r, u [B, G, kstride] complex, s, x [B, kstride], t, v [B, kstride] complex,
 * q_grid [B, G, L] complex, s_grid [B, L], status [B]; workspace from
 * slse_semifast_bundle_workspace_bytes. */
size_t slse_semifast_bundle_workspace_bytes(int N, int M, int G, int B, int L, int kstride);
int slse_semifast_bundle(const double* theta, const double* gamma, const int32_t* kcount, int kstride,
                         const double* beta, const double* y, int N, int M, int G, int B, const int32_t* idx,
                         const double* scales, int pattern_stride, int L, double* data_term, double* e, double* q,
                         double* r, double* u, double* s, double* t, double* v, double* x, double* q_grid,
                         double* s_grid, int32_t* status, void* workspace, size_t workspace_bytes, void* stream);

/* On-device synthetic scenes (simdata.generate laws): trials independent
 * scenes of n samples, m observed (first and last always; m = n: complete),
 * k frequencies (pairs != 0: k / 2 pairs at intra_sep, generate_pairs), G
 * snapshots, SNR snr_db, from the Philox stream keyed by (seed, point) with
 * the trial index as counter.  Outputs: y [trials, G, m] complex, idx
 * [trials, m] 0-based observed positions, theta [trials, k], alpha
 * [trials, G, k] complex, beta [trials], status [trials] (0 ok, 1 infeasible
 * separation).  workspace: slse_sim_workspace_bytes(n, trials). */
size_t slse_sim_workspace_bytes(int n, int trials);
int slse_sim_generate(unsigned long long seed, unsigned point, int trials, int n, int m, int k, int G, double snr_db,
                      double min_sep, int pairs, double intra_sep, double* y, int32_t* idx, double* theta,
                      double* alpha, double* beta, int32_t* status, void* workspace, void* stream);

/* Metrics per trial (simdata.nmse, csr): nmse [trials], csr [trials] and
 * mind [trials, k] (wrap distance of each true frequency to its nearest
 * estimate, for the host's block-success check).  theta_est/alpha_est rows
 * of stride kstride with k_hat[t] valid entries; alpha_est [trials, G, kstride]. */
int slse_sim_metrics(int trials, int n, int G, const double* theta_true, const double* alpha_true, int k,
                     const double* theta_est, const double* alpha_est, const int32_t* k_hat, int kstride,
                     double* nmse, double* csr, double* mind, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SUPERLSE_B200_H */
