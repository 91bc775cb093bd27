"""Solve time of the package found under ROOT (argv[1]) at config cfg."""
import sys, os
root, cfg, B = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
sys.path.insert(0, root)
import torch
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver
n = simdata.CONFIGS[cfg][1]
Y = torch.from_numpy(simdata.batch(20261019, cfg, B)).cuda()
try:
    s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
except TypeError:
    s = BatchSolver(n, B, EstimatorOptions(grid_factor=4))
s.solve(Y); torch.cuda.synchronize()
ts = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{root} cfg{cfg} B={B}: {min(ts):.1f} ms")
