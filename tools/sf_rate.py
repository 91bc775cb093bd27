"""Semifast solver rate at the cfg1 / cfg2 shapes (complete data: the
reference's backend="auto" path below N = 512) and incomplete M = 0.75 N."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver

for cfg, B, frac in ((1, 1, 1.0), (2, 4096, 1.0), (2, 4096, 0.75), (2, 148, 1.0)):
    n = simdata.CONFIGS[cfg][1]
    Y = simdata.batch(20261019, cfg, B)
    m = int(round(frac * n))
    s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="semifast"), m=m)
    if m < n:
        rng = np.random.default_rng(3)
        idx = np.sort(rng.choice(n, size=m, replace=False)).astype(np.int32)
        s.set_pattern(idx)
        Y = Y[:, idx]
    Yd = torch.from_numpy(np.ascontiguousarray(Y)).cuda()
    s.solve(Yd); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.solve(Yd); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    h = s.host_outputs()
    print(f"semifast cfg{cfg} B={B} M={m}: {min(ts):.2f} ms = {B / min(ts) * 1000:.0f} problems/s; "
          f"status!=0 {int((h['status'] != 0).sum())}; k_hat mean {h['k_hat'].mean():.2f}", flush=True)
