"""CPU oracle for the Superfast LSE inner loop -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`superlse`, /root/reference/pkg/src/superlse): the superfast bundle
(complete data) and the semifast (Woodbury) bundle (complete or incomplete
data), G >= 1 snapshots, and the estimator loop.  It exists for three
purposes only:

* the checker in ``tests/`` (parity of the CUDA path against it),
* ``__graft_entry__.smoke()`` (one small check on cuda:0),
* the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.

The product path (``paper_1705_06073_b200``) never imports it.

Pinning: the oracle is checked against golden vectors produced by the real
reference (``tests/golden/make_golden.py`` imports /root/reference in the
build container and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Algorithm choices (each equivalent within ~1e-13 to the reference's own
``auto`` dispatch, as measured in SURVEY.md section 8(c)):

* Toeplitz factor: Levinson-Durbin at every N (reference: LD for N <= 256,
  divide-and-conquer Schur above; toeplitz.py:263-276).  LD is also the
  faster of the two in numpy.
* Off-grid Fourier sums: direct O(NK) sums at every N (reference: direct
  below N = 512, Gaussian-gridding NUFFT above; nufft.py:118-123).

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from math import comb

import numpy as np

# --- constants (reference values) -------------------------------------------
PD_EPS = 1e-13                       # toeplitz.py:32
BETA_FLOOR_SCALE = 1e-12             # model_core.py:36
DEFAULT_TAU = 5.0                    # smlr.py:28
EPS_OBJECTIVE = float(np.finfo(np.float64).eps)  # smlr.py:31
SWEEP_WITHIN_FACTOR = 5.0            # smlr.py:35
SWEEP_MIN_SPACING_SCALE = 0.05       # smlr.py:36
GAMMA_BAR_K_INIT = 4                 # smlr.py:40
MAX_PAIRS = 10                       # lbfgs.py:19
ARMIJO_C1 = 1e-4                     # lbfgs.py:21
BACKTRACK_FACTOR = 0.5               # lbfgs.py:22
MAX_BACKTRACKS = 30                  # lbfgs.py:23
CURVATURE_EPS = 1e-12                # lbfgs.py:26
INITIAL_ZETA = 0.2                   # estimator.py:30
INITIAL_BETA_ENERGY_FRACTION = 0.01  # estimator.py:31

STAGES = ("init", "beta", "activate", "zeta", "refine", "deactivate")


class OracleNotPD(Exception):
    """Mirror of superlse.errors.NotPositiveDefinite (errors.py:8)."""


class OracleLineSearchFailed(Exception):
    """Mirror of superlse.errors.LineSearchFailed (errors.py:28)."""


# --- grid size / prior --------------------------------------------------------
def default_grid_size(n, grid_factor=8):
    """model_core.py:224-227."""
    target = max(2 * n, grid_factor * n)
    return 1 << int(np.ceil(np.log2(target)))


def prior_zeta(zeta, k_max):
    """model_core.py:230-234."""
    return float(min(max(zeta, 0.5 / k_max), 0.5))


def prior_term(k_hat, zeta, k_max):
    """model_core.py:237-239."""
    ze = prior_zeta(zeta, k_max)
    return -(k_hat * np.log(ze) + (k_max - k_hat) * np.log1p(-ze))


def wrap_distance(x, y):
    """simdata.py:50-53."""
    d = np.abs(np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)) % 1.0
    return np.minimum(d, 1.0 - d)


# --- Row 1: Toeplitz column ---------------------------------------------------
def steer_forward(thetas, coeffs, n):
    """sum_k coeffs_k e^{j 2 pi m theta_k}, m = 0..n-1 (nufft.py:126-144, direct
    branch :139-141)."""
    thetas = np.asarray(thetas, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.complex128)
    if thetas.size == 0:
        return np.zeros(n, dtype=np.complex128)
    basis = _phase_basis(thetas, np.arange(n), 1.0).T
    return basis @ coeffs


# Exactly reduced phases (test-only accuracy reference): the reference's
# direct sums form 2 pi m theta in double, whose rounding grows like m eps,
# ~1e-8 relative on cancelling sums at N = 4096 (the reference's own NUFFT /
# direct switch differs by up to 5e-10).  EXACT_PHASE = True
# reduces m theta mod 1 in extended precision first, which is what the CUDA
# path does with FMA residuals; the per-call size sweep uses it at large N.
EXACT_PHASE = False


def _phase_basis(thetas, m, sign):
    if not EXACT_PHASE:
        return np.exp(sign * 2j * np.pi * np.outer(thetas, m))
    ph = np.outer(np.asarray(thetas, dtype=np.longdouble), np.asarray(m, dtype=np.longdouble)) % 1
    ang = sign * 2 * np.longdouble(np.pi) * ph
    return (np.cos(ang) + 1j * np.sin(ang)).astype(np.complex128)


def steer_adjoint(thetas, x):
    """sum_m x_m e^{-j 2 pi m theta_k} (nufft.py:147-159, direct :156-158)."""
    thetas = np.asarray(thetas, dtype=np.float64)
    x = np.asarray(x, dtype=np.complex128)
    n = x.shape[0]
    if thetas.size == 0:
        return np.zeros((0,) + x.shape[1:], dtype=np.complex128)
    basis = _phase_basis(thetas, np.arange(n), -1.0)
    return basis @ x


def fourier_sum_two_sided(thetas, omega):
    """sum_{i=-(N-1)}^{N-1} omega(i) e^{j 2 pi i theta} (nufft.py:162-181)."""
    omega = np.asarray(omega, dtype=np.complex128)
    vec = omega.ndim == 1
    if vec:
        omega = omega[:, None]
    n = (omega.shape[0] + 1) // 2
    pos = omega[n - 1:]
    neg = np.zeros_like(pos)
    neg[1:] = omega[n - 2::-1]
    out = np.conj(steer_adjoint(thetas, np.conj(pos))) + steer_adjoint(thetas, neg)
    return out[:, 0] if vec else out


def cov_column(thetas, gammas, beta, n):
    """c_m = beta [m == 0] + sum_k gamma_k e^{j2 pi m theta_k}
    (model_core.py:242-249 and :264-265; toeplitz.py:55-59 forces c_0 real)."""
    c = steer_forward(thetas, np.asarray(gammas, dtype=np.complex128), n)
    c[0] = c[0].real + beta
    return c


def check_column(c):
    """HermitianToeplitz validation, toeplitz.py:44-64."""
    c0 = c[0]
    if abs(c0.imag) > 1e-10 * max(abs(c0.real), 1.0) or c0.real <= 0.0:
        raise OracleNotPD("diagonal entry c_0 must be real and positive")
    c = c.copy()
    c[0] = c0.real
    return c


# --- Row 3: Levinson-Durbin -------------------------------------------------------
def levinson(c):
    """Levinson-Durbin recursion giving the Gohberg-Semencul parameters
    (rho, delta); toeplitz.py:121-145."""
    c = check_column(np.asarray(c, dtype=np.complex128))
    n = c.size
    c0 = c[0].real
    delta = np.empty(n)
    delta[0] = c0
    a = np.zeros(n, dtype=np.complex128)
    a[0] = 1.0
    floor = PD_EPS * c0
    for m in range(1, n):
        acc = c[m] + np.dot(a[1:m], c[m - 1:0:-1])
        k = -acc / delta[m - 1]
        a[1:m + 1] = a[1:m + 1] + k * np.conj(a[m - 1::-1])
        delta[m] = delta[m - 1] * (1.0 - (k * np.conj(k)).real)
        if not delta[m] > floor:
            raise OracleNotPD(f"pivot delta_{m} = {delta[m]:.3e} <= {floor:.3e}")
    rho = np.conj(a)[::-1]
    rho = rho / rho[-1]
    return rho, delta


# --- Row 5: GS apply ------------------------------------------------------------
def _pow2_at_least(n):
    return 1 << int(np.ceil(np.log2(max(n, 1))))


def gs_apply(rho, delta_last, x):
    """C^{-1} x = delta_{N-1}^{-1} (T1^H T1 x - T0 T0^H x) through four FFT
    convolutions (toeplitz.py:279-309, plan :93-112).  nfft is any length
    >= 2N-1 (reference: next_fast_len; the result does not depend on it
    beyond roundoff)."""
    n = rho.size
    x = np.asarray(x, dtype=np.complex128)
    if n == 1:
        return x / delta_last
    nfft = _pow2_at_least(2 * n - 1)
    v0 = np.concatenate(([0.0], rho[:-1]))
    f_t1 = np.fft.fft(rho, nfft)
    f_t1h = np.fft.fft(np.conj(rho)[::-1], nfft)
    f_t0h = np.fft.fft(np.conj(v0)[::-1], nfft)
    f_t0 = np.fft.fft(v0, nfft)
    fx = np.fft.fft(x, nfft)
    t1x = np.fft.ifft(fx * f_t1)[n - 1:2 * n - 1]
    t0hx = np.fft.ifft(fx * f_t0h)[n - 1:2 * n - 1]
    y1 = np.fft.ifft(np.fft.fft(t1x, nfft) * f_t1h)[:n]
    y0 = np.fft.ifft(np.fft.fft(t0hx, nfft) * f_t0)[:n]
    return (y1 - y0) / delta_last


# --- Row 7: omega diagonal sums -----------------------------------------------------
def weight_coefficients(kind, n):
    """Diagonal weights in powers q^a i^b (toeplitz.py:317-354)."""
    if kind == "s":
        return {(0, 0): 2.0 - n, (0, 1): 1.0, (1, 0): 2.0}
    if kind == "t":
        return {(1, 1): -1.0, (0, 1): n - 1.5, (0, 2): -0.5, (1, 0): n - 1.0,
                (0, 0): -(n - 1.0) * (n - 2.0) / 2.0}
    if kind == "v":
        return {(3, 0): 2.0 / 3.0, (2, 1): 1.0, (1, 2): 1.0, (2, 0): 2.0 - n,
                (1, 1): 3.0 - 2.0 * n, (1, 0): n * n - 3.0 * n + 7.0 / 3.0,
                (0, 3): 1.0 / 3.0, (0, 2): 1.5 - n,
                (0, 1): n * n - 3.0 * n + 13.0 / 6.0,
                (0, 0): 1.5 * n * n - n ** 3 / 3.0 - 13.0 * n / 6.0 + 1.0}
    if kind == "x":
        return {(3, 0): 2.0 / 3.0, (2, 1): 1.0, (2, 0): 2.0 - n, (1, 1): 2.0 - n,
                (1, 0): n * n - 3.0 * n + 7.0 / 3.0, (0, 3): -1.0 / 6.0,
                (0, 1): (3.0 * n * n - 9.0 * n + 7.0) / 6.0,
                (0, 0): -(n ** 3) / 3.0 + 1.5 * n * n - 13.0 * n / 6.0 + 1.0}
    raise ValueError(kind)


def crosscorr_basis(coeffs):
    """(q, i) -> (q, m = q + i) change of basis (toeplitz.py:357-365)."""
    out = {}
    for (a, b), cf in coeffs.items():
        for j in range(b + 1):
            key = (a + b - j, j)
            out[key] = out.get(key, 0.0) + cf * comb(b, j) * (-1.0) ** (b - j)
    return out


OMEGA_SCALE = {"s": 1.0, "t": 2.0 * np.pi, "v": 4.0 * np.pi ** 2, "x": 4.0 * np.pi ** 2}


def _fftconv(a, b):
    nfft = _pow2_at_least(a.size + b.size - 1)
    return np.fft.ifft(np.fft.fft(a, nfft) * np.fft.fft(b, nfft))[: a.size + b.size - 1]


def omegas(rho, delta_last):
    """All four diagonal-sum vectors over lags -(N-1)..N-1
    (toeplitz.py:368-432; s and x symmetrised as at :428-430)."""
    n = rho.size
    q = np.arange(n, dtype=np.float64)
    sets = {k: crosscorr_basis(weight_coefficients(k, n)) for k in "stvx"}
    pairs = sorted({key for cs in sets.values() for key in cs})
    corr = {}
    for a, b in pairs:
        corr[(a, b)] = _fftconv((q ** b) * np.conj(rho), ((q ** a) * rho)[::-1])
    mid = n - 1
    out = {}
    for kind, cs in sets.items():
        om = np.zeros(2 * n - 1, dtype=np.complex128)
        for key, cf in cs.items():
            om += cf * corr[key]
        om *= OMEGA_SCALE[kind] / delta_last
        if kind in ("s", "x"):
            om[:mid] = np.conj(om[mid + 1:][::-1])
            om[mid] = om[mid].real
        out[kind] = om
    return out


# --- Bundle: rows 1, 3, 5, 6 (+7, 8, 9 lazily) ------------------------------------------
class Bundle:
    """One evaluation of the model at (theta, gamma, beta):
    _SuperfastBundle, model_core.py:256-313."""

    def __init__(self, y, thetas, gammas, beta):
        # y: (N,) for one snapshot or (G, N) for G snapshots (model_core.py:266-270)
        y2 = np.atleast_2d(y)
        n = y2.shape[1]
        self.y = y
        self.g = y2.shape[0]
        self.thetas = np.asarray(thetas, dtype=np.float64)
        self.gammas = np.asarray(gammas, dtype=np.float64)
        self.beta = beta
        self.c = cov_column(self.thetas, self.gammas, beta, n)
        self.rho, self.delta = levinson(self.c)
        w2 = np.stack([gs_apply(self.rho, self.delta[-1], yg) for yg in y2])
        self.w = w2 if y.ndim == 2 else w2[0]
        quad = float(np.sum(np.conj(y2) * w2).real)
        self.logdet = float(np.sum(np.log(self.delta)))
        self.data_term = self.g * self.logdet + quad
        self._om = None
        self._stats = None
        self._grid = {}

    def omegas(self):
        if self._om is None:
            self._om = omegas(self.rho, self.delta[-1])
        return self._om

    def stats(self):
        """model_core.py:281-301 (direct sums); q, r, u are (G, K) for a
        (G, N) observation, (K,) for a single snapshot."""
        if self._stats is None:
            w2 = np.atleast_2d(self.w)
            n = w2.shape[1]
            d = 2.0 * np.pi * np.arange(n)
            qs, rs, us = [], [], []
            for wg in w2:
                stack = np.stack((wg, d * wg, d ** 2 * wg), axis=1)
                adj = steer_adjoint(self.thetas, stack)
                qs.append(adj[:, 0].copy())
                rs.append(adj[:, 1].copy())
                us.append(adj[:, 2].copy())
            om = self.omegas()
            omstack = np.stack([om["s"], om["t"], om["v"], om["x"]], axis=1)
            stvx = fourier_sum_two_sided(self.thetas, omstack)
            one = np.ndim(self.w) == 1
            pick = (lambda a: a[0]) if one else np.stack
            self._stats = dict(q=pick(qs), r=pick(rs), u=pick(us),
                               s=stvx[:, 0].real.copy(), t=stvx[:, 1].copy(),
                               v=stvx[:, 2].copy(), x=stvx[:, 3].real.copy())
        return self._stats

    def grid(self, length):
        """model_core.py:303-313; q_grid is (G, L) for a (G, N) observation."""
        if length not in self._grid:
            n = self.rho.size
            q_grid = np.fft.fft(self.w, n=length, axis=-1)
            buf = np.zeros(length, dtype=np.complex128)
            buf[np.arange(-(n - 1), n) % length] = self.omegas()["s"]
            s_grid = (length * np.fft.ifft(buf)).real
            self._grid[length] = (q_grid, s_grid)
        return self._grid[length]


# --- semifast bundle ----------------------------------------
def gram(t_rows, t_cols, weights, idx):
    """nufft.gram direct branch (nufft.py:184-210): entry (i, k) =
    sum_m w_m e^{j 2 pi (I(m) - 1)(theta_k - theta_i)}, I 1-based."""
    er = np.exp(2j * np.pi * np.outer(idx - 1, t_rows))
    ec = np.exp(2j * np.pi * np.outer(idx - 1, t_cols))
    return (np.conj(er) * weights[:, None]).T @ ec


def _chol_solve(lower, rhs):
    """scipy cho_solve(lower=True): (L L^H)^{-1} rhs by two triangular solves."""
    z = np.linalg.solve(lower, rhs)
    return np.linalg.solve(np.conj(lower).T, z)


class SemifastBundle:
    """_SemifastBundle (model_core.py:316-409): Woodbury form of C on an
    observation pattern (Observation, model_core.py:43-130; scatter :109-117,
    sample :119-123).  y is (G, M) observed samples, idx 1-based positions,
    scales complex (ones for complete data)."""

    def __init__(self, y, n, idx, scales, thetas, gammas, beta):
        y2 = np.atleast_2d(np.asarray(y, dtype=np.complex128))
        self.y, self.n, self.idx, self.sc = y2, n, np.asarray(idx), np.asarray(scales, dtype=np.complex128)
        self.g, m = y2.shape
        self.thetas = np.asarray(thetas, dtype=np.float64)
        self.gammas = np.asarray(gammas, dtype=np.float64)
        self.beta = beta
        self.pos = self.gammas > 0.0  # :325
        w0 = np.abs(self.sc) ** 2
        d1 = 2.0 * np.pi * (self.idx - 1)
        self.w0 = w0
        herm = lambda a: 0.5 * (a + np.conj(a).T)  # _hermitize :412-413
        self.g0 = herm(gram(self.thetas, self.thetas, w0, self.idx))
        self.g1 = herm(gram(self.thetas, self.thetas, w0 * d1, self.idx))
        self.g2 = herm(gram(self.thetas, self.thetas, w0 * d1 ** 2, self.idx))
        pos = self.pos
        kp = int(np.count_nonzero(pos))
        ycols = y2.T  # (M, G)
        ys = self._scatter(ycols)
        self.ahy = steer_adjoint(self.thetas, ys) if self.thetas.size else np.zeros((0, self.g), complex)
        ln_c = m * np.log(beta)
        if kp:
            sigma_inv = self.g0[np.ix_(pos, pos)] / beta + np.diag(1.0 / self.gammas[pos])
            self.chol = np.linalg.cholesky(sigma_inv)
            ln_c += float(np.sum(np.log(self.gammas[pos])))
            ln_c += 2.0 * float(np.sum(np.log(np.diag(self.chol).real)))
            wp = _chol_solve(self.chol, self.ahy[pos])
            quad = float(np.sum(np.abs(ycols) ** 2)) / beta - float(
                np.sum(np.conj(self.ahy[pos]) * wp).real) / beta ** 2
            z1 = steer_forward(self.thetas[pos], wp, n)
            cinv_y = ycols / beta - self._sample(z1) / beta ** 2
        else:
            self.chol = None
            quad = float(np.sum(np.abs(ycols) ** 2)) / beta
            cinv_y = ycols / beta
        self.ln_c = ln_c
        self.data_term = self.g * ln_c + quad
        self.e = self._scatter(cinv_y)  # (N, G)
        self.w = self.e.T if self.g > 1 else self.e[:, 0]
        self._stats = None
        self._grid = {}

    def _scatter(self, w):
        out = np.zeros((self.n,) + w.shape[1:], dtype=np.complex128)
        out[self.idx - 1] = np.conj(self.sc).reshape((-1,) + (1,) * (w.ndim - 1)) * w
        return out

    def _sample(self, z):
        return self.sc.reshape((-1,) + (1,) * (z.ndim - 1)) * z[self.idx - 1]

    def stats(self):
        """:368-390."""
        if self._stats is None:
            beta = self.beta
            d = 2.0 * np.pi * np.arange(self.n)
            stack = np.concatenate((self.e, d[:, None] * self.e, (d ** 2)[:, None] * self.e), axis=1)
            adj = steer_adjoint(self.thetas, stack)
            g = self.g
            q, r, u = adj[:, :g].T, adj[:, g:2 * g].T, adj[:, 2 * g:].T
            pos = self.pos
            s = np.diag(self.g0).real / beta
            t = np.diag(self.g1).astype(np.complex128) / beta
            v = np.diag(self.g2).astype(np.complex128) / beta
            x = np.diag(self.g2).real / beta
            if self.chol is not None:
                w00 = _chol_solve(self.chol, self.g0[pos])
                s = s - np.einsum("kp,pk->k", self.g0[:, pos], w00).real / beta ** 2
                t = t - np.einsum("kp,pk->k", self.g1[:, pos], w00) / beta ** 2
                v = v - np.einsum("kp,pk->k", self.g2[:, pos], w00) / beta ** 2
                w11 = _chol_solve(self.chol, np.conj(self.g1[:, pos]).T)
                x = x - np.einsum("kp,pk->k", self.g1[:, pos], w11).real / beta ** 2
            one = g == 1
            self._stats = dict(q=q[0] if one else q, r=r[0] if one else r, u=u[0] if one else u,
                               s=s, t=t, v=v, x=x)
        return self._stats

    def grid(self, length):
        """:392-409; q_grid is (G, L) for G > 1 snapshots."""
        if length not in self._grid:
            beta = self.beta
            q_grid = np.fft.fft(self.e, n=length, axis=0).T
            s_grid = np.full(length, float(np.sum(self.w0)) / beta)
            pos = self.pos
            if self.chol is not None and np.any(pos):
                phases = np.exp(-2j * np.pi * np.outer(self.idx - 1, self.thetas[pos]))
                scat = np.zeros((length, int(np.count_nonzero(pos))), dtype=np.complex128)
                np.add.at(scat, self.idx - 1, self.w0[:, None] * phases)
                b = (length * np.fft.ifft(scat, axis=0)).T
                wb = _chol_solve(self.chol, b)
                s_grid = s_grid - np.einsum("pl,pl->l", np.conj(b), wb).real / beta ** 2
            self._grid[length] = (q_grid[0] if self.g == 1 else q_grid, s_grid)
        return self._grid[length]


# --- Row 10: activation -----------------------------------------------------------
def gamma_bar(active_gamma, energy, m):
    """smlr.py:53-59."""
    if active_gamma.size:
        bar = float(np.mean(active_gamma))
        if bar > 0.0:
            return bar
    return max(energy / (m * GAMMA_BAR_K_INIT), np.finfo(np.float64).tiny)


def delta_curve(q_grid, s_grid, gbar, zeta_eff):
    """smlr.py:62-70; q_grid (L,) or (G, L).  Returns (delta, mean_g |q|^2)."""
    q2 = np.atleast_2d(q_grid)
    g = q2.shape[0]
    sum_q2 = np.sum(np.abs(q2) ** 2, axis=0)
    log_ratio = np.log((1.0 - zeta_eff) / zeta_eff)
    delta = g * np.log1p(gbar * s_grid) + log_ratio - sum_q2 / (1.0 / gbar + s_grid)
    return delta, sum_q2 / g


def gamma_estimate(kappa, s):
    """smlr.py:73-76."""
    return (kappa * s - s) / s ** 2 if kappa > 1.0 else 0.0


def snr_criterion(kappa, s, gbar, zeta_eff, tau):
    """smlr.py:79-81."""
    rhs = (1.0 + 1.0 / (gbar * s)) * np.log((1.0 + gbar * s) * (1.0 - zeta_eff) / zeta_eff)
    return kappa > rhs + tau


# --- Row 12: gradient / diag Hessian -------------------------------------------------
def gradient(gammas, st):
    """model_core.py:497-505 (sums over snapshots; q, r may be (G, K))."""
    q, r = np.atleast_2d(st["q"]), np.atleast_2d(st["r"])
    g = q.shape[0]
    cross = np.sum(np.conj(q) * r, axis=0)
    d_theta = 2.0 * gammas * (g * st["t"] - cross).imag
    d_gamma = g * st["s"] - np.sum(np.abs(q) ** 2, axis=0)
    return np.concatenate((d_theta, d_gamma))


def diag_hessian(gammas, st, n):
    """model_core.py:508-536 (fallback on; q, r, u may be (G, K))."""
    ga = gammas
    q, r, u = np.atleast_2d(st["q"]), np.atleast_2d(st["r"]), np.atleast_2d(st["u"])
    g = q.shape[0]
    q2 = np.sum(np.abs(q) ** 2, axis=0)
    r2 = np.sum(np.abs(r) ** 2, axis=0)
    rqc = np.sum(r * np.conj(q), axis=0)
    uqc = np.sum(u * np.conj(q), axis=0)
    s, t, v, x = st["s"], st["t"], st["v"], st["x"]
    core = g * (x - v) + ga * g * (t ** 2 - x * s) + ga * (x * q2 + s * r2 - 2.0 * t * rqc) + uqc - r2
    d2_theta = 2.0 * ga * core.real
    d2_gamma = 2.0 * s * q2 - g * s ** 2
    d2_theta = np.where(d2_theta <= 0.0, float(50 * n) ** 2, d2_theta)
    safe = np.where(ga > 0.0, ga, 1.0 / (50.0 * n))
    d2_gamma = np.where(d2_gamma <= 0.0, safe ** -2, d2_gamma)
    return np.concatenate((d2_theta, d2_gamma))


# --- Row 13: L-BFGS ---------------------------------------------------------------
@dataclass
class Memory:
    """lbfgs.py:29-53."""
    diag: np.ndarray
    pairs: list = field(default_factory=list)
    max_pairs: int = MAX_PAIRS

    @property
    def dim(self):
        return self.diag.size

    def push(self, step, gdiff):
        curv = float(np.dot(step, gdiff))
        if curv <= CURVATURE_EPS * np.linalg.norm(step) * np.linalg.norm(gdiff):
            return
        self.pairs.append((step, gdiff, 1.0 / curv))
        if len(self.pairs) > self.max_pairs:
            self.pairs.pop(0)


def two_loop(mem, g):
    """lbfgs.py:63-76."""
    q = g.copy()
    alphas = []
    for s, y, r in reversed(mem.pairs):
        a = r * np.dot(s, q)
        alphas.append(a)
        q -= a * y
    r_ = q / mem.diag
    for (s, y, r), a in zip(mem.pairs, reversed(alphas)):
        b = r * np.dot(y, r_)
        r_ += s * (a - b)
    return -r_


_MARGINS = None  # list receiving (kind, normalised margin, trace length) while estimate() runs
_TRACE = None    # the running estimate()'s objective trace (for the decision's position)


def _margin(kind, lhs, rhs, scale):
    """Record how far a decision lhs <= rhs (or lhs < rhs) was from flipping,
    in units of `scale` (the decision's roundoff noise), and the length of
    the objective trace when it was taken (the trace entry it first affects)."""
    if _MARGINS is not None:
        _MARGINS.append((kind, abs(lhs - rhs) / scale, len(_TRACE) if _TRACE is not None else -1))


def lbfgs_step(mem, point, f0, g0, objective_fn, gradient_fn):
    """lbfgs.py:100-136."""
    if not np.any(g0):
        return point, f0, g0, 0.0, 0
    d = two_loop(mem, g0)
    slope = float(np.dot(g0, d))
    dec = -slope
    if slope >= 0.0:
        d = -g0 / mem.diag
        slope = float(np.dot(g0, d))
        dec = -slope
    k = point.size // 2
    dg = d[k:]
    shrink = dg < 0.0
    cap = float(np.min(point[k:][shrink] / -dg[shrink])) if np.any(shrink) else np.inf
    alpha = min(1.0, cap)
    if alpha <= 0.0:
        raise OracleLineSearchFailed("pinned")
    for trial in range(MAX_BACKTRACKS):
        cand = point + alpha * d
        cand[:k] = np.mod(cand[:k], 1.0)
        f_new = objective_fn(cand)
        _margin("armijo", f_new, f0 + ARMIJO_C1 * alpha * slope, 1e-12 * max(1.0, abs(f0)))
        if f_new <= f0 + ARMIJO_C1 * alpha * slope:
            g_new = gradient_fn(cand)
            mem.push(alpha * d, g_new - g0)
            return cand, f_new, g_new, dec, trial + 1
        alpha *= BACKTRACK_FACTOR
    raise OracleLineSearchFailed("no sufficient decrease")


# --- Row 15: the loop -----------------------------------------------------------
@dataclass
class OracleOptions:
    """estimator.py:34-50 (fields used on the superfast path)."""
    grid_factor: int = 8
    tau: float = DEFAULT_TAU
    max_outer_iterations: int = 200
    convergence_tol_scale: float = 1e-7
    lbfgs_inner_max: int = 5
    newton_decrement_tol_scale: float = 1e-8
    initial_sweep_iterations: int = 3
    lbfgs_memory: int = 10
    k_max: int = None
    backend: str = "superfast"  # or "semifast" (model_core.py:456-472)


class _State:
    def __init__(self, k_max, beta, zeta):
        self.z = np.zeros(k_max, dtype=bool)
        self.theta = np.zeros(k_max)
        self.gamma = np.zeros(k_max)
        self.beta = float(beta)
        self.zeta = float(zeta)

    def copy(self):
        o = _State.__new__(_State)
        o.z, o.theta, o.gamma = self.z.copy(), self.theta.copy(), self.gamma.copy()
        o.beta, o.zeta = self.beta, self.zeta
        return o

    @property
    def k_max(self):
        return self.z.size

    @property
    def k_hat(self):
        return int(np.count_nonzero(self.z))

    @property
    def act(self):
        return np.flatnonzero(self.z)


class _Engine:
    """LRU(4) bundle cache keyed on the exact state bytes (model_core.py:416-444)."""

    def __init__(self, y, grid_size, pattern=None):
        self.y = y
        self.grid_size = grid_size
        self.pattern = pattern  # None: superfast bundles; (n, idx 1-based, scales): semifast
        self._b = {}
        self._order = []
        self.builds = 0

    def bundle(self, st):
        th = st.theta[st.z]
        ga = st.gamma[st.z]
        key = (th.tobytes(), ga.tobytes(), float(st.beta))
        hit = self._b.get(key)
        if hit is not None:
            return hit
        if self.pattern is None:
            b = Bundle(self.y, th, ga, float(st.beta))
        else:
            b = SemifastBundle(self.y, *self.pattern, th, ga, float(st.beta))
        self.builds += 1
        self._b[key] = b
        self._order.append(key)
        if len(self._order) > 4:
            self._b.pop(self._order.pop(0), None)
        return b

    def objective(self, st):
        return self.bundle(st).data_term + prior_term(st.k_hat, st.zeta, st.k_max)


def _activate_slot(st, theta, gamma):
    """smlr.py:99-104: the lowest free slot."""
    slot = int(np.flatnonzero(~st.z)[0])
    st.z[slot] = True
    st.theta[slot] = theta
    st.gamma[slot] = gamma
    return slot


def try_activate(st, energy, m, q_grid, s_grid, tau):
    """smlr.py:84-122. Returns (new_state, slot, grid_index) or None."""
    if st.k_hat >= st.k_max:
        return None
    gbar = gamma_bar(st.gamma[st.z], energy, m)
    ze = prior_zeta(st.zeta, st.k_max)
    delta, q2 = delta_curve(q_grid, s_grid, gbar, ze)
    best = int(np.argmin(delta))
    kappa = float(q2[best] / s_grid[best])
    gam = gamma_estimate(kappa, float(s_grid[best]))
    if float(delta[best]) >= -EPS_OBJECTIVE or gam <= 0.0:
        return None
    if not snr_criterion(kappa, float(s_grid[best]), gbar, ze, tau):
        return None
    out = st.copy()
    slot = _activate_slot(out, best / s_grid.size, gam)
    return out, slot, best


def initial_sweep(st, energy, m, n, q_grid, s_grid, tau):
    """smlr.py:125-171.  Returns (state, [(slot, grid_index), ...])."""
    gbar = gamma_bar(st.gamma[st.z], energy, m)
    ze = prior_zeta(st.zeta, st.k_max)
    delta, q2 = delta_curve(q_grid, s_grid, gbar, ze)
    length = s_grid.size
    local_min = (delta <= np.roll(delta, 1)) & (delta <= np.roll(delta, -1))
    cands = np.flatnonzero(local_min)
    if cands.size == 0:
        return st, []
    cands = cands[np.argsort(delta[cands], kind="stable")]
    dmin = float(delta[cands[0]])
    if dmin >= -EPS_OBJECTIVE:
        return st, []
    out = st.copy()
    spacing = SWEEP_MIN_SPACING_SCALE / n
    added = []
    for idx in cands:
        if out.k_hat >= out.k_max:
            break
        d = float(delta[idx])
        if d >= -EPS_OBJECTIVE or d > dmin / SWEEP_WITHIN_FACTOR:
            continue
        kappa = float(q2[idx] / s_grid[idx])
        gnew = gamma_estimate(kappa, float(s_grid[idx]))
        if gnew <= 0.0:
            continue
        tau_eff = tau if out.k_hat == 0 else 0.0
        if not snr_criterion(kappa, float(s_grid[idx]), gbar, ze, tau_eff):
            continue
        th = idx / length
        if out.k_hat and np.min(wrap_distance(th, out.theta[out.z])) < spacing:
            continue
        added.append((_activate_slot(out, th, gnew), int(idx)))
    return out, added


def deactivation_margins(st, stt):
    """smlr.py:174-200 (q may be (G, K))."""
    gamma = st.gamma[st.z]
    ze = prior_zeta(st.zeta, st.k_max)
    rhs = np.log((1.0 - ze) / ze)
    denom = 1.0 - gamma * stt["s"]
    qa = np.atleast_2d(stt["q"])
    g = qa.shape[0]
    q2 = np.sum(np.abs(qa) ** 2, axis=0)
    out = np.empty(gamma.size)
    for i in range(gamma.size):
        if gamma[i] <= 0.0:
            out[i] = -np.inf if rhs > 0.0 else 0.0
            continue
        if denom[i] <= 0.0:
            out[i] = np.inf
            continue
        q2dd = q2[i] / denom[i] ** 2
        sdd = stt["s"][i] / denom[i]
        out[i] = q2dd / (1.0 / gamma[i] + sdd) - g * np.log1p(gamma[i] * sdd) - rhs
    return out


def try_deactivate(st, stt, recompute):
    """smlr.py:203-225."""
    removed = []
    cur = st
    while cur.k_hat:
        mg = deactivation_margins(cur, stt)
        worst = int(np.argmin(mg))
        if not mg[worst] < 0.0:
            break
        slot = int(cur.act[worst])
        cur = cur.copy() if cur is st else cur
        cur.z[slot] = False
        cur.gamma[slot] = 0.0
        removed.append(slot)
        if cur.k_hat == 0:
            break
        stt = recompute(cur)
    return cur, removed


@dataclass
class OracleResult:
    k_hat: int
    theta_hat: np.ndarray
    alpha_hat: np.ndarray
    beta_hat: float
    gamma_hat: np.ndarray
    zeta_hat: float
    objective_trace: np.ndarray
    trace_stages: list
    trace_khat: list
    iterations: int
    converged: bool
    warnings: list
    events: list
    slots: np.ndarray
    builds: int = 0
    wall_time: float = 0.0
    min_margin: float = float("inf")  # smallest decision margin in roundoff units
    margins: list = None  # every decision: (kind, margin, trace position)


def estimate(y, opts: OracleOptions = None, n=None, observed_indices=None, scales=None) -> OracleResult:
    """estimator.py:117-275; y is one snapshot (M,) or G snapshots (G, M)
    sharing the frequencies (MMV).  opts.backend "superfast" (complete data)
    or "semifast" (complete, or incomplete with n, 1-based observed_indices
    and complex scales: Observation.incomplete, model_core.py:43-130).

    `events` is the active-set history: ("sweep", [(slot, idx)...]),
    ("activate", slot, idx), ("deactivate", [slots]) in order."""
    global _MARGINS, _TRACE
    t_start = time.perf_counter()
    opts = opts or OracleOptions()
    _MARGINS = []
    y = np.asarray(y, dtype=np.complex128)
    if y.ndim != 2:
        y = y.ravel()
    g = 1 if y.ndim == 1 else y.shape[0]
    m = y.shape[-1]
    if observed_indices is None:
        n = m
        obs_idx, obs_sc = np.arange(1, m + 1), np.ones(m, dtype=np.complex128)
    else:
        obs_idx = np.asarray(observed_indices, dtype=np.int64)
        obs_sc = np.ones(m, dtype=np.complex128) if scales is None else np.asarray(scales, dtype=np.complex128)
    if m < 2:
        raise ValueError("need at least two observed samples")
    k_max = opts.k_max if opts.k_max is not None else m
    L = default_grid_size(n, opts.grid_factor)
    semifast = opts.backend == "semifast"
    if not semifast and observed_indices is not None:
        raise ValueError("superfast backend requires the complete observation pattern")
    eng = _Engine(y, L, (n, obs_idx, obs_sc) if semifast else None)
    energy = float(np.mean(np.sum(np.abs(np.atleast_2d(y)) ** 2, axis=1)))
    floor = BETA_FLOOR_SCALE * energy / m
    beta0 = max(INITIAL_BETA_ENERGY_FRACTION * energy / m, floor)
    st = _State(k_max, beta0, INITIAL_ZETA)
    trace, stages, khat, events, warns = [], [], [], [], []
    _TRACE = trace

    def record(stage):
        trace.append(eng.objective(st))
        stages.append(stage)
        khat.append(st.k_hat)

    record("init")
    st = st.copy()
    st.beta = max(floor, energy / m)
    record("beta")
    previous = trace[-1]
    mem = None
    z_dirty = True
    converged = False
    iterations = 0

    def stats_of(s):
        return eng.bundle(s).stats()

    for it in range(1, opts.max_outer_iterations + 1):
        iterations = it
        if it <= opts.initial_sweep_iterations:
            qg, sg = eng.bundle(st).grid(L)
            new, added = initial_sweep(st, energy, m, n, qg, sg, opts.tau)
            if new.k_hat != st.k_hat:
                st, z_dirty = new, True
                events.append(("sweep", added))
        else:
            for _ in range(k_max):
                qg, sg = eng.bundle(st).grid(L)
                res = try_activate(st, energy, m, qg, sg, opts.tau)
                if res is None:
                    break
                st, slot, idx = res
                z_dirty = True
                events.append(("activate", slot, idx))
            else:
                warns.append(f"iteration {it}: activation loop hit the K_max cap")
        record("activate")
        st = st.copy()
        st.zeta = min(0.5, st.k_hat / st.k_max)
        record("zeta")
        cand = st.copy()
        if st.k_hat:
            stt = stats_of(st)
            ga = st.gamma[st.z]
            mu = ga * stt["q"]  # (K,) or (G, K)
            tr = float(st.beta * np.sum(stt["s"] * ga))
            fitted = steer_forward(st.theta[st.z], mu if g == 1 else mu.T, n)
            if semifast:  # y - sample(fitted) (estimator.py:86-87)
                fitted = (obs_sc[:, None] * fitted[obs_idx - 1]) if g > 1 else obs_sc * fitted[obs_idx - 1]
            resid = y - fitted if g == 1 else y.T - fitted
            value = (tr + float(np.sum(np.abs(resid) ** 2)) / g) / m
        else:
            value = energy / m
        cand.beta = max(floor, value)
        _margin("beta", eng.objective(cand), trace[-1], 1e-12 * max(1.0, abs(trace[-1])))
        if eng.objective(cand) <= trace[-1]:
            st = cand
        record("beta")
        if st.k_hat:
            for _ in range(opts.lbfgs_inner_max):
                stt = stats_of(st)
                if z_dirty or mem is None or mem.dim != 2 * st.k_hat:
                    mem = Memory(diag=diag_hessian(st.gamma[st.z], stt, n), max_pairs=opts.lbfgs_memory)
                    z_dirty = False
                g0 = gradient(st.gamma[st.z], stt)
                f0 = eng.objective(st)
                base = st

                def with_point(p, base=base):
                    o = base.copy()
                    a = o.act
                    k = a.size
                    o.theta[a] = p[:k]
                    o.gamma[a] = p[k:]
                    return o

                point = np.concatenate((st.theta[st.z], st.gamma[st.z]))
                def grad_at(p):
                    trial = with_point(p)
                    return gradient(trial.gamma[trial.z], stats_of(trial))

                try:
                    newp, _, _, dec, _ = lbfgs_step(
                        mem, point, f0, g0, lambda p: eng.objective(with_point(p)), grad_at)
                except OracleLineSearchFailed:
                    break
                st = with_point(newp)
                record("refine")
                new, removed = try_deactivate(st, stats_of(st), stats_of)
                if removed:
                    st, z_dirty = new, True
                    events.append(("deactivate", removed))
                    record("deactivate")
                    if st.k_hat == 0:
                        break
                _margin("decrement", dec, m * opts.newton_decrement_tol_scale,
                        1e-9 * m * opts.newton_decrement_tol_scale + 1e-12 * max(1.0, abs(trace[-1])))
                if dec < m * opts.newton_decrement_tol_scale:
                    break
        current = trace[-1]
        _margin("converge", abs(previous - current), m * opts.convergence_tol_scale,
                1e-12 * max(1.0, abs(current)))
        if abs(previous - current) < m * opts.convergence_tol_scale:
            converged = True
            break
        previous = current

    if st.k_hat:
        alpha = np.atleast_2d(st.gamma[st.z] * stats_of(st)["q"])
    else:
        alpha = np.zeros((1, 0), dtype=np.complex128)
    return OracleResult(
        k_hat=st.k_hat, theta_hat=st.theta[st.z].copy(), alpha_hat=alpha, beta_hat=st.beta,
        gamma_hat=st.gamma[st.z].copy(), zeta_hat=st.zeta, objective_trace=np.array(trace),
        trace_stages=stages, trace_khat=khat, iterations=iterations, converged=converged,
        warnings=warns, events=events, slots=st.act.copy(), builds=eng.builds,
        wall_time=time.perf_counter() - t_start,
        min_margin=min((mg for _, mg, _ in _MARGINS), default=float("inf")),
        margins=list(_MARGINS),
    )


# --- seeded config generator -----------------------------
CONFIGS = {
    # cfg: (B, N, K, min_sep_scale, amplitude law, snr_db)
    1: (1, 64, 4, 2.0, "unit", 20.0),
    2: (4096, 256, 16, 1.5, "cn", 15.0),
    3: (1024, 1024, 64, 2.0, "uniform", 20.0),
    4: (256, 4096, 256, 2.0, "cn", 20.0),
    5: (64, 16384, 512, 1.0, "loguniform", 10.0),
}


def generate_problem(seed, cfg, b, n=None, k=None):
    """One seeded problem y (complex128[N]) plus its truth, drawn with
    rng = default_rng([seed, cfg, b]) (simdata.py:12-14 stream contract).
    Frequencies: sequential rejection sampling (simdata.py:61-73); noise
    variance from the paper SNR definition (simdata.py:96-99)."""
    _, n0, k0, sep, law, snr = CONFIGS[cfg]
    n = n or n0
    k = k or k0
    rng = np.random.default_rng([seed, cfg, b])
    min_sep = sep / n
    thetas = []
    while len(thetas) < k:
        cand = rng.random()
        if not thetas or np.min(wrap_distance(cand, np.array(thetas))) > min_sep:
            thetas.append(cand)
    thetas = np.array(thetas)
    phase = np.exp(2j * np.pi * rng.random(k))
    if law == "unit":
        mag = np.ones(k)
    elif law == "cn":
        a = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
        mag, phase = np.abs(a), np.exp(1j * np.angle(a))
    elif law == "uniform":
        mag = rng.uniform(0.5, 1.5, k)
    elif law == "loguniform":
        # 20 dB power range: |alpha|^2 in [0.01, 1]
        mag = 10.0 ** rng.uniform(-1.0, 0.0, k)
    else:
        raise ValueError(law)
    alpha = mag * phase
    clean = steer_forward(thetas, alpha, n)
    beta = float(np.sum(np.abs(clean) ** 2)) / (n * 10.0 ** (snr / 10.0))
    noise = np.sqrt(beta / 2.0) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return clean + noise, dict(thetas=thetas, alphas=alpha, beta=beta)


def generate_batch(seed, cfg, count, n=None, k=None, start=0):
    ys = [generate_problem(seed, cfg, start + b, n=n, k=k)[0] for b in range(count)]
    return np.stack(ys)


def generate_problem_mmv(seed, cfg, b, g, n=None, k=None):
    """G snapshots sharing the frequencies (MMV, estimator.py:278-283):
    y (G, N).  rng = default_rng([seed, cfg, 1000 + g, b]); frequencies as
    generate_problem; amplitudes drawn per snapshot with the config's law;
    one noise variance from the mean clean power and the config's SNR."""
    _, n0, k0, sep, law, snr = CONFIGS[cfg]
    n = n or n0
    k = k or k0
    rng = np.random.default_rng([seed, cfg, 1000 + g, b])
    min_sep = sep / n
    thetas = []
    while len(thetas) < k:
        cand = rng.random()
        if not thetas or np.min(wrap_distance(cand, np.array(thetas))) > min_sep:
            thetas.append(cand)
    thetas = np.array(thetas)
    alphas = np.empty((g, k), dtype=np.complex128)
    for gi in range(g):
        phase = np.exp(2j * np.pi * rng.random(k))
        if law == "unit":
            mag = np.ones(k)
        elif law == "cn":
            a = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
            mag, phase = np.abs(a), np.exp(1j * np.angle(a))
        elif law == "uniform":
            mag = rng.uniform(0.5, 1.5, k)
        else:
            mag = 10.0 ** rng.uniform(-1.0, 0.0, k)
        alphas[gi] = mag * phase
    clean = np.stack([steer_forward(thetas, alphas[gi], n) for gi in range(g)])
    beta = float(np.mean(np.sum(np.abs(clean) ** 2, axis=1))) / (n * 10.0 ** (snr / 10.0))
    noise = np.sqrt(beta / 2.0) * (rng.standard_normal((g, n)) + 1j * rng.standard_normal((g, n)))
    return clean + noise, dict(thetas=thetas, alphas=alphas, beta=beta)
