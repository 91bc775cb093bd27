"""Every solver layout boundary at N = 4096 (CTA pair up to SMs/2 problems,
one 512-thread CTA per problem up to SMs, paired 256-thread CTAs above) and
N = 256 (128-thread CTAs / classic / warp mode): all problems finish with
status 0 and problem 0's result is the same in every batch."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch, simdata

sms = torch.cuda.get_device_properties(0).multi_processor_count
opts = EstimatorOptions(grid_factor=4, backend="superfast", max_outer_iterations=4)
for cfg, sizes in ((4, (1, 2, sms // 2, sms // 2 + 1, sms, sms + 1)), (2, (1, 5 * sms, 5 * sms + 1, 10 * sms, 10 * sms + 1))):
    ref = None
    for B in sizes:
        Y = simdata.batch(7, cfg, B)
        r = estimate_batch(Y, opts)
        assert np.all(r.status == 0), (cfg, B)
        t0 = r[0].objective_trace
        if ref is None:
            ref = t0
        d = float(np.max(np.abs(t0 - ref)) / np.max(np.abs(ref)))
        print(f"cfg{cfg} B={B}: ok, k_hat[0]={r.k_hat[0]} trace[0] rel diff vs first layout {d:.1e}", flush=True)
        assert d < 1e-9
