"""Seeded synthetic problems for the BASELINE.json configs.

Per problem b: ``rng = np.random.default_rng([seed, cfg, b])`` (the
stream contract of the reference harness, simdata.py:12-14); frequencies by
sequential rejection sampling with wrap-around separation > sep/N
(simdata.py:61-73); amplitude law per config; noise variance from the
paper's SNR definition ||Psi alpha||^2 / (N beta) (simdata.py:96-99).
The reference benchmarks on no public dataset; these stand in for its
synthetic Monte-Carlo signals.
"""

from __future__ import annotations

import numpy as np

# cfg: (B, N, K, min_sep_scale, amplitude law, snr_db)   (BASELINE.json configs)
CONFIGS = {
    1: (1, 64, 4, 2.0, "unit", 20.0),
    2: (4096, 256, 16, 1.5, "cn", 15.0),
    3: (1024, 1024, 64, 2.0, "uniform", 20.0),
    4: (256, 4096, 256, 2.0, "cn", 20.0),
    5: (64, 16384, 512, 1.0, "loguniform", 10.0),
}


def _wrap(x, y):
    d = np.abs(x - y) % 1.0
    return np.minimum(d, 1.0 - d)


def problem(seed: int, cfg: int, b: int):
    """(y complex128[N], truth dict) for problem b of config cfg."""
    _, n, k, sep, law, snr = CONFIGS[cfg]
    rng = np.random.default_rng([seed, cfg, b])
    min_sep = sep / n
    th = []
    while len(th) < k:
        cand = rng.random()
        if not th or np.min(_wrap(cand, np.array(th))) > min_sep:
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
