"""Synthetic scenes and evaluation metrics (reference
pkg/src/superlse/simdata.py).

Three layers:

* ``CONFIGS`` / ``problem`` / ``batch`` -- the seeded BASELINE.json config
  generator of SURVEY.md 8(d) used by bench.py (per problem
  ``default_rng([seed, cfg, b])``; frequencies by sequential rejection,
  amplitude law per config, noise from the paper's SNR definition).
* The reference's public generator and metrics with its semantics:
  ``generate`` / ``generate_pairs`` draw from the caller's numpy Generator
  in the reference's order (pattern, frequencies, coefficients, noise), so a
  reference user's seeded streams give the same scenes; ``nmse``,
  ``assign`` (Hungarian, scipy), ``bsr_trial`` and ``csr``.
* The device path for Monte-Carlo throughput: ``generate_device`` draws
  whole batches of scenes on the GPU (csrc/slse_sim.cu: the same laws from a
  counter-based Philox stream per trial), ``metrics_device`` evaluates NMSE
  and CSR there (block success keeps its Hungarian assignment on the host),
  and ``montecarlo`` chains generation -> estimate_batch -> metrics.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import InfeasibleSeparation
from .model_core import Observation

# cfg: (B, N, K, min_sep_scale, amplitude law, snr_db)   (BASELINE.json configs)
CONFIGS = {
    1: (1, 64, 4, 2.0, "unit", 20.0),
    2: (4096, 256, 16, 1.5, "cn", 15.0),
    3: (1024, 1024, 64, 2.0, "uniform", 20.0),
    4: (256, 4096, 256, 2.0, "cn", 20.0),
    5: (64, 16384, 512, 1.0, "loguniform", 10.0),
}

# reference constants (simdata.py:19-25)
MIN_SEP_SCALE = 2.0        # default separation 2/N
SUCCESS_RADIUS = 0.5       # recovered within 0.5/N
COEFF_OFFSET = 0.2         # |alpha| pushed out by 0.2 along its phase
COEFF_STD = 0.8            # std of the complex Gaussian part
MAX_DRAWS = 100_000        # rejection attempts per frequency


def wrap_distance(x, y):
    """Distance on the unit circle, min(|x - y|, 1 - |x - y|) mod 1 (broadcasts)."""
    d = np.abs(np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)) % 1.0
    return np.minimum(d, 1.0 - d)


# ------------------------------------------------------------ bench configs
def problem(seed: int, cfg: int, b: int):
    """(y complex128[N], truth dict) for problem b of config cfg."""
    _, n, k, sep, law, snr = CONFIGS[cfg]
    rng = np.random.default_rng([seed, cfg, b])
    min_sep = sep / n
    th = []
    while len(th) < k:
        cand = rng.random()
        if not th or np.min(wrap_distance(cand, np.array(th))) > min_sep:
            th.append(cand)
    th = np.array(th)
    phase = np.exp(2j * np.pi * rng.random(k))
    if law == "unit":
        mag = np.ones(k)
    elif law == "cn":
        a = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) / np.sqrt(2.0)
        mag, phase = np.abs(a), np.exp(1j * np.angle(a))
    elif law == "uniform":
        mag = rng.uniform(0.5, 1.5, k)
    else:  # log-uniform over a 20 dB power range: |alpha|^2 in [0.01, 1]
        mag = 10.0 ** rng.uniform(-1.0, 0.0, k)
    alpha = mag * phase
    clean = np.exp(2j * np.pi * np.outer(np.arange(n), th)) @ alpha
    beta = float(np.sum(np.abs(clean) ** 2)) / (n * 10.0 ** (snr / 10.0))
    noise = np.sqrt(beta / 2.0) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return clean + noise, dict(thetas=th, alphas=alpha, beta=beta)


def batch(seed: int, cfg: int, count: int = None, start: int = 0) -> np.ndarray:
    """(count, N) complex128 stack of problems start..start+count-1."""
    count = CONFIGS[cfg][0] if count is None else count
    return np.stack([problem(seed, cfg, start + b)[0] for b in range(count)])


# ------------------------------------------------------------ reference API
@dataclass
class GroundTruth:
    """simdata.GroundTruth (:33-47): k, thetas (K,), alphas (G, K), beta_true, snr_db."""

    k: int
    thetas: np.ndarray
    alphas: np.ndarray
    beta_true: float
    snr_db: float

    def __post_init__(self):
        self.thetas = np.asarray(self.thetas, dtype=np.float64)
        self.alphas = np.atleast_2d(np.asarray(self.alphas, dtype=np.complex128))


def _pattern(rng, n, m):
    """1-based sorted positions: 1 and n always, M - 2 of 2..n-1 without
    replacement (simdata.py:78-86); None for complete data."""
    if m is None or m == n:
        return None
    if m < 2 or m > n:
        raise ValueError("m must satisfy 2 <= m <= n")
    inner = rng.choice(np.arange(2, n), size=m - 2, replace=False)
    return np.sort(np.concatenate(([1], inner, [n])))


def _frequencies(rng, k, min_sep):
    """Sequential rejection (simdata.py:61-73)."""
    out = np.empty(0)
    for _ in range(k):
        for _ in range(MAX_DRAWS):
            cand = rng.random()
            if out.size == 0 or np.min(wrap_distance(cand, out)) > min_sep:
                out = np.append(out, cand)
                break
        else:
            raise InfeasibleSeparation(f"could not place {k} frequencies with separation {min_sep:.4g}")
    return out


def _coefficients(rng, g, k):
    """CN(0, 0.8^2) pushed out by 0.2 along its phase (simdata.py:56-58)."""
    z = (rng.standard_normal((g, k)) + 1j * rng.standard_normal((g, k))) * (COEFF_STD / np.sqrt(2.0))
    return z + COEFF_OFFSET * np.exp(1j * np.angle(z))


def _steer(thetas, coeffs, n):
    """sum_k coeffs_k e^{j 2 pi m theta_k}, m < n; coeffs (K,) or (K, G)."""
    return np.exp(2j * np.pi * np.outer(np.arange(n), thetas)) @ coeffs


def _scene(rng, n, idx, thetas, alphas, snr_db):
    """y = Phi Psi alpha + noise with beta = mean ||Phi Psi alpha||^2 / (M snr)
    (simdata.py:89-106)."""
    g, k = alphas.shape
    full = _steer(thetas, alphas.T, n).T  # (G, N)
    clean = full if idx is None else full[:, idx - 1]
    m = clean.shape[1]
    beta = float(np.mean(np.sum(np.abs(clean) ** 2, axis=1))) / (m * 10.0 ** (snr_db / 10.0))
    y = clean + np.sqrt(beta / 2.0) * (rng.standard_normal((g, m)) + 1j * rng.standard_normal((g, m)))
    obs = Observation.complete(y) if idx is None else Observation.incomplete(y, n, idx)
    return obs, GroundTruth(k=k, thetas=thetas, alphas=alphas, beta_true=beta, snr_db=snr_db)


def generate(n, m_pattern, k, snr_db, rng, min_sep=None, snapshots=1):
    """Random scene with k separated components (simdata.generate :109-122):
    (Observation, GroundTruth).  m_pattern None or n: complete data."""
    min_sep = MIN_SEP_SCALE / n if min_sep is None else min_sep
    if k * min_sep >= 1.0:
        raise InfeasibleSeparation(f"{k} frequencies with separation {min_sep:.4g} cannot fit in [0,1)")
    idx = _pattern(rng, n, m_pattern)
    thetas = _frequencies(rng, k, min_sep)
    alphas = _coefficients(rng, snapshots, k)
    return _scene(rng, n, idx, thetas, alphas, snr_db)


def generate_pairs(n, num_pairs, intra_sep, snr_db, rng, snapshots=1, m_pattern=None):
    """num_pairs pairs at intra_sep, pairs 2/N apart (simdata.generate_pairs :125-149)."""
    min_sep = MIN_SEP_SCALE / n
    if num_pairs * (intra_sep + 2 * min_sep) >= 1.0:
        raise InfeasibleSeparation(f"{num_pairs} pairs of width {intra_sep:.4g} cannot fit in [0,1)")
    th = []
    for _ in range(num_pairs):
        for _ in range(MAX_DRAWS):
            base = rng.random()
            pair = np.array([base, (base + intra_sep) % 1.0])
            if not th or all(np.min(wrap_distance(f, np.array(th))) > min_sep for f in pair):
                th.extend(pair)
                break
        else:
            raise InfeasibleSeparation("could not place well-separated pairs")
    idx = _pattern(rng, n, m_pattern)
    alphas = _coefficients(rng, snapshots, 2 * num_pairs)
    return _scene(rng, n, idx, np.array(th), alphas, snr_db)


def _synth(thetas, alphas, n):
    if len(thetas) == 0:
        g = alphas.shape[0] if alphas is not None and np.ndim(alphas) == 2 else 1
        return np.zeros((g, n), dtype=np.complex128)
    return _steer(np.asarray(thetas), np.atleast_2d(alphas).T, n).T


def nmse(truth: GroundTruth, result, n) -> float:
    """Full-grid reconstruction error ||Psi a_hat - Psi a||^2 / ||Psi a||^2,
    snapshots pooled (simdata.nmse :160-169)."""
    ref = _synth(truth.thetas, truth.alphas, n)
    est = _synth(result.theta_hat, result.alpha_hat, n)
    if est.shape[0] != ref.shape[0]:
        raise ValueError("snapshot counts of truth and estimate differ")
    return float(np.sum(np.abs(est - ref) ** 2) / np.sum(np.abs(ref) ** 2))


def assign(truth_thetas, est_thetas):
    """Hungarian matching under squared wrap distance (simdata.assign :172-181)."""
    from scipy.optimize import linear_sum_assignment

    a = np.atleast_1d(np.asarray(truth_thetas, dtype=np.float64))
    b = np.atleast_1d(np.asarray(est_thetas, dtype=np.float64))
    if a.size == 0 or b.size == 0:
        raise ValueError("assign requires nonempty frequency sets")
    return linear_sum_assignment(wrap_distance(a[:, None], b[None, :]) ** 2)


def bsr_trial(truth: GroundTruth, result, n) -> bool:
    """Exact model order and every matched frequency within 0.5/N
    (simdata.bsr_trial :184-193)."""
    if result.k_hat != truth.k or truth.k == 0:
        return False
    r, c = assign(truth.thetas, result.theta_hat)
    return bool(np.max(wrap_distance(truth.thetas[r], np.asarray(result.theta_hat)[c])) < SUCCESS_RADIUS / n)


def csr(truth: GroundTruth, result, n) -> float:
    """Component success ratio (simdata.csr :196-205): estimates near a true
    frequency plus true frequencies near an estimate, over K_hat + K."""
    rad = SUCCESS_RADIUS / n
    est = np.asarray(result.theta_hat, dtype=np.float64)

    def near(p, q):
        if len(p) == 0 or len(q) == 0:
            return 0
        return int(np.sum(np.min(wrap_distance(np.asarray(p)[:, None], np.asarray(q)[None, :]), axis=1) < rad))

    return float((near(est, truth.thetas) + near(truth.thetas, est)) / (est.size + truth.k))


# ------------------------------------------------------------ device path
@dataclass
class DeviceScenes:
    """A batch of scenes resident on the GPU (slse_sim_generate): y (T, G, M)
    complex, idx (T, M) 0-based observed positions, theta (T, K), alpha
    (T, G, K) complex, beta (T,), status (T,) (1 = separation infeasible)."""

    n: int
    m: int
    k: int
    g: int
    snr_db: float
    y: object
    idx: object
    theta: object
    alpha: object
    beta: object
    status: object

    @property
    def trials(self):
        return int(self.y.shape[0])

    def truth(self, t) -> GroundTruth:
        """Host GroundTruth of trial t."""
        return GroundTruth(k=self.k, thetas=self.theta[t].cpu().numpy(), alphas=self.alpha[t].cpu().numpy(),
                           beta_true=float(self.beta[t].item()), snr_db=self.snr_db)


def generate_device(n, m, k, snr_db, trials, seed, point=0, min_sep=None, snapshots=1, pairs=False,
                    intra_sep=0.0, device=None) -> DeviceScenes:
    """trials independent scenes on the GPU with generate's laws (or
    generate_pairs' with pairs=True: k = 2 x pairs); trial t of (seed, point)
    is the same whatever the batch it is drawn in."""
    import torch

    from . import _native

    lib = _native.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    m = n if m is None else int(m)
    min_sep = MIN_SEP_SCALE / n if min_sep is None else float(min_sep)
    if pairs:
        if (k // 2) * (intra_sep + 2 * min_sep) >= 1.0:
            raise InfeasibleSeparation(f"{k // 2} pairs of width {intra_sep:.4g} cannot fit in [0,1)")
    elif k * min_sep >= 1.0:
        raise InfeasibleSeparation(f"{k} frequencies with separation {min_sep:.4g} cannot fit in [0,1)")
    if not 2 <= m <= n:
        raise ValueError("m must satisfy 2 <= m <= n")
    g = int(snapshots)
    c, f = torch.complex128, torch.float64
    y = torch.empty((trials, g, m), dtype=c, device=dev)
    idx = torch.empty((trials, m), dtype=torch.int32, device=dev)
    th = torch.empty((trials, max(k, 1)), dtype=f, device=dev)
    al = torch.empty((trials, g, max(k, 1)), dtype=c, device=dev)
    be = torch.empty(trials, dtype=f, device=dev)
    st = torch.empty(trials, dtype=torch.int32, device=dev)
    ws = torch.empty(max(1, int(lib.slse_sim_workspace_bytes(n, trials))), dtype=torch.uint8, device=dev)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    with torch.cuda.device(dev):
        rc = lib.slse_sim_generate(ctypes.c_ulonglong(int(seed) & (2 ** 64 - 1)), ctypes.c_uint(int(point)), trials,
                                   n, m, k, g, float(snr_db), min_sep, 1 if pairs else 0, float(intra_sep), p(y),
                                   p(idx), p(th), p(al), p(be), p(st), p(ws),
                                   ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    _native.check(rc, "slse_sim_generate")
    if int(st.max().item()) != 0:
        raise InfeasibleSeparation("could not place the frequencies with the requested separation")
    return DeviceScenes(n=n, m=m, k=k, g=g, snr_db=float(snr_db), y=y, idx=idx, theta=th[:, :k], alpha=al[:, :, :k],
                        beta=be, status=st)


def metrics_device(scenes: DeviceScenes, result, theta_est=None, alpha_est=None):
    """NMSE and CSR of every trial on the GPU (slse_sim_metrics), block
    success with the Hungarian assignment on the host for the trials whose
    model order is right.  ``result`` is a BatchResult of the scenes (its
    SoA arrays are used).  Returns dict of numpy arrays nmse, csr, bsr, k_hat."""
    import torch

    from . import _native

    lib = _native.load()
    dev = scenes.y.device
    T, k, g, n = scenes.trials, scenes.k, scenes.g, scenes.n
    khat = np.asarray(result.k_hat, dtype=np.int32)
    th_e = np.ascontiguousarray(result.theta if theta_est is None else theta_est, dtype=np.float64)
    al_e = result.alpha if alpha_est is None else alpha_est
    al_e = np.ascontiguousarray(al_e if np.ndim(al_e) == 3 else np.asarray(al_e)[:, None, :], dtype=np.complex128)
    ks = max(1, th_e.shape[1])
    if th_e.shape[1] == 0:
        th_e = np.zeros((T, 1))
        al_e = np.zeros((T, g, 1), complex)
    th_d = torch.from_numpy(th_e).to(dev)
    al_d = torch.from_numpy(np.ascontiguousarray(al_e)).to(dev)
    kh_d = torch.from_numpy(khat).to(dev)
    nm = torch.empty(T, dtype=torch.float64, device=dev)
    cs = torch.empty(T, dtype=torch.float64, device=dev)
    md = torch.empty((T, max(k, 1)), dtype=torch.float64, device=dev)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    thc = scenes.theta.contiguous()
    alc = scenes.alpha.contiguous()
    with torch.cuda.device(dev):
        rc = lib.slse_sim_metrics(T, n, g, p(thc), p(alc), k, p(th_d), p(al_d), p(kh_d), ks, p(nm), p(cs), p(md),
                                  ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    _native.check(rc, "slse_sim_metrics")
    nm_h, cs_h = nm.cpu().numpy(), cs.cpu().numpy()
    md_h = md.cpu().numpy()
    th_true = thc.cpu().numpy()
    bsr = np.zeros(T, dtype=bool)
    for t in np.flatnonzero(khat == k):
        if k == 0 or np.max(md_h[t, :k]) >= SUCCESS_RADIUS / n:
            continue  # some true frequency has no estimate within 0.5/N: no assignment can succeed
        r, c = assign(th_true[t], th_e[t, :k])
        bsr[t] = bool(np.max(wrap_distance(th_true[t][r], th_e[t, :k][c])) < SUCCESS_RADIUS / n)
    return dict(nmse=nm_h, csr=cs_h, bsr=bsr, k_hat=khat)


def montecarlo(n, m, k, snr_db, trials, seed, point=0, opts=None, snapshots=1, pairs=False, intra_sep=0.0,
               min_sep=None, device=None):
    """One Monte-Carlo sweep point on the GPU: generate_device -> estimate_batch
    -> metrics_device.  Returns (metrics dict, BatchResult, DeviceScenes)."""
    from .estimator import EstimatorOptions, estimate_batch

    sc = generate_device(n, m, k, snr_db, trials, seed, point=point, min_sep=min_sep, snapshots=snapshots,
                         pairs=pairs, intra_sep=intra_sep, device=device)
    opts = opts or EstimatorOptions()
    y = sc.y[:, 0] if sc.g == 1 else sc.y
    if sc.m == n:
        res = estimate_batch(y, opts, device=device)
    else:
        res = estimate_batch(y, opts, device=device, n=n, observed_indices=sc.idx.cpu().numpy() + 1)
    return metrics_device(sc, res), res, sc
