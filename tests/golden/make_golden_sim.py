"""simdata golden fixtures from the REAL reference (build container only).

Runs ``superlse.simdata.generate`` / ``generate_pairs`` on seeded numpy
streams (the harness contract default_rng([base_seed, point, trial]),
simdata.py:12-14) and records the scenes (y, pattern, truth), and the
reference metrics (nmse, bsr_trial, csr) of perturbed estimates of each
scene, so tests/test_simdata.py can check the package's host generator
bit for bit and its host / device metrics on the same inputs.

Usage:  python tests/golden/make_golden_sim.py   (writes tests/golden/golden_sim.npz)
"""

import os
import sys
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from superlse import simdata as S  # noqa: E402

# (kind, n, m, k or pairs, snr, snapshots, intra_sep scale)
CASES = [
    ("gen", 64, None, 4, 20.0, 1, 0.0),
    ("gen", 128, 96, 10, 10.0, 1, 0.0),
    ("gen", 256, None, 16, 15.0, 2, 0.0),
    ("gen", 128, 64, 6, 0.0, 3, 0.0),
    ("pairs", 128, None, 5, 20.0, 1, 1.0),
    ("pairs", 128, 100, 4, 20.0, 1, 1.5),
]


def main():
    store = {}
    for ci, (kind, n, m, k, snr, g, intra) in enumerate(CASES):
        for trial in range(3):
            rng = np.random.default_rng([2026, ci, trial])
            if kind == "gen":
                obs, tr = S.generate(n, m, k, snr, rng, snapshots=g)
            else:
                obs, tr = S.generate_pairs(n, k, intra / n, snr, rng, snapshots=g, m_pattern=m)
            p = f"c{ci}_t{trial}_"
            store[p + "y"] = obs.y
            store[p + "idx"] = obs.observed_indices if not obs.is_complete else np.zeros(0, np.int64)
            store[p + "thetas"] = tr.thetas
            store[p + "alphas"] = tr.alphas
            store[p + "beta"] = tr.beta_true
            # estimates: truth perturbed (model order kept / one dropped / one spurious)
            prng = np.random.default_rng([7, ci, trial])
            est = []
            th = tr.thetas + prng.normal(0, 0.2 / n, tr.thetas.size)
            al = tr.alphas * (1 + 0.05 * prng.standard_normal(tr.alphas.shape))
            est.append((th % 1.0, al))
            est.append(((th[1:]) % 1.0, al[:, 1:]))
            est.append((np.append(th, prng.random()) % 1.0, np.concatenate([al, 0.1 * np.ones((g, 1))], axis=1)))
            for e, (et, ea) in enumerate(est):
                res = SimpleNamespace(theta_hat=et, alpha_hat=ea, k_hat=et.size)
                store[p + f"e{e}_theta"] = et
                store[p + f"e{e}_alpha"] = ea
                store[p + f"e{e}_nmse"] = S.nmse(tr, res, n)
                store[p + f"e{e}_bsr"] = S.bsr_trial(tr, res, n)
                store[p + f"e{e}_csr"] = S.csr(tr, res, n)
    np.savez_compressed(os.path.join(HERE, "golden_sim.npz"), cases=np.array(CASES, dtype=object).astype(str),
                        **store)
    print("cases", len(CASES))


if __name__ == "__main__":
    main()
