"""Per-phase cycle profile of the persistent solver (one GPU).

Build the profiling variant first (nothing in the default build changes):
  SLSE_BUILD_OUT=build/variants/prof SLSE_BUILD_DEFS=-DSLSE_SOLVER_PROF python paper_1705_06073_b200/build.py
then run:
  SLSE_LIB=build/variants/prof/libsuperlse_b200.so python tools/solver_prof.py --config 2
Prints each phase's share of the solver CTAs' wall cycles (leader-thread
clock64, summed over problems).
"""

import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata  # noqa: E402
from paper_1705_06073_b200 import _native  # noqa: E402
from paper_1705_06073_b200.estimator import BatchSolver  # noqa: E402

PHASES = ["covariance column", "factor", "GS apply", "stats", "grid", "whole run", "rv wait (arrive)",
          "rv wait (depart)", "ctl: sweep", "ctl: try_activate", "ctl: deactivate", "ctl: lbfgs_step", "ctl: record",
          "ctl: beta EM", " (accept: stats incl)", " (accept: grad+push)"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
n = simdata.CONFIGS[a.config][1]
B = a.batch or simdata.CONFIGS[a.config][0]
Y = torch.from_numpy(simdata.batch(20261019, a.config, B)).cuda()
s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
s.solve(Y)  # warm-up
lib = _native.load()
out = (ctypes.c_ulonglong * 16)()
fns = {nt: getattr(lib, f"slse_solver_prof_{nt}") for nt in (32, 64, 128, 256, 512, 1024)}
fns["warps"] = lib.slse_solver_prof_warps
for fn in fns.values():
    fn(out, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.solve(Y)
e1.record()
torch.cuda.synchronize()
print(f"config {a.config}: B={B} N={n} solve {e0.elapsed_time(e1):.3f} ms")
for nt, fn in fns.items():
    fn(out, 0)
    v = list(out)
    if v[5] == 0:
        continue
    print(f"solver NT={nt}: total {v[5] / 1e9:.3f} G leader-cycles")
    for name, x in zip(PHASES[:5] + PHASES[6:16], v[:5] + v[6:16]):
        print(f"  {name:20s} {100.0 * x / v[5]:6.1f} %")
    print(f"  {'other':20s} {100.0 * (v[5] - sum(v[:5]) - sum(v[6:14])) / v[5]:6.1f} %")
