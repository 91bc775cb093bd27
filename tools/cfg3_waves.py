import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver
Yall = simdata.batch(20261019, 3, 1184)
for B in (148, 296, 592, 888, 1024, 1184):
    Y = torch.from_numpy(np.ascontiguousarray(Yall[:B])).cuda()
    s = BatchSolver(1024, B, EstimatorOptions(grid_factor=4, backend="superfast"))
    s.solve(Y); torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    h = s.host_outputs()
    c = h['counters'][:, 0]
    print(f"cfg3 B={B}: {np.median(ms):.1f} ms = {B / np.median(ms) * 1000:.0f} problems/s; builds min/mean/max {c.min()}/{c.mean():.1f}/{c.max()}", flush=True)
