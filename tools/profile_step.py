"""Profiling driver (one GPU): one warm-up + one measured solve of a config
batch, then the standalone grid kernel; meant to be run under ncu."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, ops, simdata  # noqa: E402
from paper_1705_06073_b200.estimator import BatchSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--grids", type=int, default=2)
a = ap.parse_args()
cfg = a.config
B = a.batch or simdata.CONFIGS[cfg][0]
n = simdata.CONFIGS[cfg][1]
Y = torch.from_numpy(simdata.batch(20261019, cfg, B)).cuda()
s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
ev = []
for i in range(a.solves):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.solve(Y)
    e1.record()
    ev.append((e0, e1))
torch.cuda.synchronize()
print("solve ms:", [round(x.elapsed_time(y), 3) for x, y in ev])
h = s.host_outputs()
print("k_hat mean", h["k_hat"].mean(), "status nonzero", int(np.count_nonzero(h["status"])),
      "counters", h["counters"].sum(axis=0))
L = 4 * n
rho = torch.randn((B, n), dtype=torch.complex128, device="cuda")
w = torch.randn((B, n), dtype=torch.complex128, device="cuda")
dl = torch.rand(B, dtype=torch.float64, device="cuda") + 0.5
for i in range(a.grids):
    ops.grid_eval(rho, dl, w, L)
torch.cuda.synchronize()
print("ok")
