"""Tail effect of the one-problem-per-warp solver at cfg2: time per problem
for batches of 1, 1.73 (bench), 2, 3.46 problems per warp slot."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata  # noqa: E402
from paper_1705_06073_b200.estimator import BatchSolver  # noqa: E402
for B in (2368, 4096, 4736, 8192):
    Y = torch.from_numpy(simdata.batch(20261019, 2, B)).cuda()
    s = BatchSolver(256, B, EstimatorOptions(grid_factor=4, backend="superfast"))
    s.solve(Y); torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    t = float(np.median(ms))
    print(f"B={B}: {t:.2f} ms  {1000 * t / B:.2f} us/problem  {B / t * 1000:.0f} problems/s")
