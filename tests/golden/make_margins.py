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

Usage:  python tests/golden/make_margins.py   (writes tests/golden/margins.json)
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from golden_util import NEAR_TIE, load  # noqa: E402
from oracle import superlse_oracle as O  # noqa: E402


def main():
    out = {}
    for cfg in (1, 2, 3, 4):
        z = load(cfg)
        for b in range(int(z["count"])):
            r = O.estimate(z[f"p{b}_y"])
            ties = [[int(pos), kind, float(mg)] for kind, mg, pos in r.margins if mg < NEAR_TIE]
            out[f"cfg{cfg}_p{b}"] = {"min_margin": float(r.min_margin), "near_ties": ties}
            print(cfg, b, r.min_margin, ties, flush=True)
    with open(os.path.join(HERE, "margins.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
