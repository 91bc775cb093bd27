"""Latency of one drop-in estimate() call (the reference's unit of work, estimator.py:117) per config shape:
whole call (Python + H2D + persistent kernel + D2H + LseResult) next to the kernel alone."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_06073_b200 as slse
from paper_1705_06073_b200 import simdata
from paper_1705_06073_b200.estimator import BatchSolver

for cfg, reps in ((1, 50), (2, 50), (3, 20), (4, 5)):
    n = simdata.CONFIGS[cfg][1]
    y, _ = simdata.problem(20261019, cfg, 0)
    for backend in ("superfast", "auto"):
        opts = slse.EstimatorOptions(grid_factor=4, backend=backend)
        obs = slse.Observation.complete(y)
        r = slse.estimate(obs, opts)
        ts = []
        for _ in range(reps):
            t = time.perf_counter(); r = slse.estimate(obs, opts); ts.append(time.perf_counter() - t)
        s = BatchSolver(n, 1, opts if backend == "superfast" else slse.EstimatorOptions(grid_factor=4, backend="superfast"))
        Y = torch.from_numpy(y[None, :].copy()).cuda()
        s.solve(Y); torch.cuda.synchronize()
        ks = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ks.append(a.elapsed_time(b))
        print(f"cfg{cfg} N={n} backend={backend}: estimate() median {1e3 * np.median(ts):.3f} ms (min {1e3 * min(ts):.3f}); "
              f"superfast kernel alone {np.median(ks):.3f} ms; k_hat {r.k_hat}; decomp {r.algorithms.get('decomp')}", flush=True)
