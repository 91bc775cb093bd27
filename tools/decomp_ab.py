"""Full-batch solve time at a config with a given decomp_method (knobs build:
SLSE_SOLVER_NT / SLSE_NO_PAIR / SLSE_NO_CTA_PAIR select the layout)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver
cfg, B, method = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
n = simdata.CONFIGS[cfg][1]
Y = torch.from_numpy(simdata.batch(20261019, cfg, B)).cuda()
s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast", decomp_method=method))
s.solve(Y); torch.cuda.synchronize()
ts = []
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
h = s.host_outputs()
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SLSE_") and k != "SLSE_LIB")
print(f"cfg{cfg} B={B} {method} [{env}]: {min(ts):.1f} ms; status!=0 {int((h['status'] != 0).sum())}", flush=True)
