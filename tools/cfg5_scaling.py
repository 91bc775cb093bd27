"""cfg5 batch time vs problems in flight (each on its own 2-CTA cluster): contention vs the slowest problem."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = simdata.CONFIGS[cfg][1]
full = simdata.CONFIGS[cfg][0]
Yall = simdata.batch(20261019, cfg, full)
for B, start in ((1, 0), (1, 1), (1, 2), (1, 3), (8, 0), (16, 0), (32, 0), (64, 0)) + (((full, 0),) if full > 64 else ()):
    Y = torch.from_numpy(np.ascontiguousarray(Yall[start:start + B])).cuda()
    s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
    s.solve(Y); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s.solve(Y); b.record(); torch.cuda.synchronize()
    h = s.host_outputs()
    print(f"cfg{cfg} B={B} start={start}: {a.elapsed_time(b):.1f} ms; builds per problem min/mean/max "
          f"{h['counters'][:, 0].min()}/{h['counters'][:, 0].mean():.1f}/{h['counters'][:, 0].max()}", flush=True)
