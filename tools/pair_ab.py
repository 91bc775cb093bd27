"""CTA-pair solver A/B at a superfast shape: time one full batch and dump
the SoA results (compare runs with and without SLSE_NO_CTA_PAIR=1 in a
-DSLSE_DEBUG_KNOBS build: the pair must give the same bits)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver

cfg = int(sys.argv[1]); B = int(sys.argv[2]); out = sys.argv[3]
n = simdata.CONFIGS[cfg][1]
Y = torch.from_numpy(simdata.batch(20261019, cfg, B)).cuda()
s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
s.solve(Y); torch.cuda.synchronize()
ts = []
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
h = s.host_outputs()
np.savez(out, **{k: np.asarray(v) for k, v in h.items() if k not in ("stage_seconds", "iter_seconds")})
print(f"cfg{cfg} B={B}: {min(ts):.1f} ms; status!=0 {int((h['status'] != 0).sum())}; k_hat mean {h['k_hat'].mean():.2f}", flush=True)
