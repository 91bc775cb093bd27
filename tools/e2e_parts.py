"""Where the e2e time goes: H2D, solve, D2H + unpack (cfg2, one GPU)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata  # noqa: E402
from paper_1705_06073_b200.estimator import BatchResult, _cached_solver, estimate_batch  # noqa: E402
Y = simdata.batch(20261019, 2, 4096)
opts = EstimatorOptions(grid_factor=4, backend="superfast")
Yp = torch.from_numpy(Y).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = _cached_solver(256, 4096, opts, None, 1)
    t1 = time.perf_counter()
    yd = Yp.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s.solve(yd)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    h = s.host_outputs()
    t4 = time.perf_counter()
    r = BatchResult(h)
    chk = int(r.k_hat.sum()) + float(np.abs(r.alpha).sum())
    t5 = time.perf_counter()
    print(f"solver {1e3*(t1-t0):.2f}  h2d {1e3*(t2-t1):.2f}  solve {1e3*(t3-t2):.2f}  d2h {1e3*(t4-t3):.2f}  unpack {1e3*(t5-t4):.2f} ms")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = estimate_batch(Yp, opts)
    chk = int(res.k_hat.sum()) + float(np.abs(res.alpha).sum())
    print(f"estimate_batch {1e3*(time.perf_counter()-t0):.2f} ms")
