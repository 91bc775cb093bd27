"""Record, for every golden trajectory, the CPU oracle's smallest decision
margin (oracle.superlse_oracle.OracleResult.min_margin: how far the closest
Armijo / convergence / deactivation / beta decision was from flipping, in
units of that decision's roundoff scale) and every near-tie decision
(margin < golden_util.NEAR_TIE) with the objective-trace position it first
affects.

A near-tie decision can be flipped by any change of floating-point summation
order.  The parity tests accept a stage trace that departs from the golden
one only at or after the first near-tie position, and still require the
identical active-set history and final estimates.  Runs anywhere (no /root/reference needed).

Usage:  python tests/golden/make_margins.py [1 2 3 4 4x 5 deact]   (writes tests/golden/margins.json;
        with names, only those fixtures are recomputed and merged)
"""

import json
import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from golden_util import NEAR_TIE, load  # noqa: E402
from oracle import superlse_oracle as O  # noqa: E402


def _one(args):
    key, y = args
    # the goldens are solved at grid_factor = 4 (L = 4N), as the GPU tests
    r = O.estimate(y, O.OracleOptions(grid_factor=4))
    ties = [[int(pos), kind, float(mg)] for kind, mg, pos in r.margins if mg < NEAR_TIE]
    return key, {"min_margin": float(r.min_margin), "near_ties": ties}


def main():
    import multiprocessing as mp

    import numpy as np

    names = sys.argv[1:] or ["1", "2", "3", "4", "4x", "5", "deact"]
    jobs = []
    for name in names:
        path = os.path.join(HERE, f"golden_{'cfg' + name if name != 'deact' else 'deact'}.npz")
        if not os.path.exists(path):
            continue
        z = np.load(path)
        idx = [int(b) for b in z["problems"]] if "problems" in z.files else range(int(z["count"]))
        tag = f"cfg{name}" if name != "deact" else "deact"
        for b in idx:
            jobs.append((f"{tag}_p{b}", z[f"p{b}_y"]))
    target = os.path.join(HERE, "margins.json")
    out = {}
    if sys.argv[1:] and os.path.exists(target):  # partial run: merge into the existing table
        with open(target) as f:
            out = json.load(f)
    with mp.get_context("fork").Pool(min(8, len(jobs))) as pool:
        for key, val in pool.imap_unordered(_one, jobs):
            out[key] = val
            print(key, val["min_margin"], val["near_ties"], flush=True)
    with open(target, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
