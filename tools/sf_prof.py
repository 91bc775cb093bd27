"""One warm-up and one timed semifast solve at the cfg2 shape (ncu target: -k regex:solve -s 1 -c 1)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
Y = torch.from_numpy(simdata.batch(20261019, 2, B)).cuda()
s = BatchSolver(256, B, EstimatorOptions(grid_factor=4, backend="semifast"))
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s.solve(Y); b.record(); torch.cuda.synchronize()
    print(f"semifast cfg2 B={B}: {a.elapsed_time(b):.2f} ms", flush=True)
h = s.host_outputs()
print("counters mean (builds, grids, stats, ls_trials):", h["counters"].mean(axis=0))
