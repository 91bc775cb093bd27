import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1705_06073_b200 as slse
from paper_1705_06073_b200 import simdata
y, _ = simdata.problem(20261019, 5, 0)
opts = slse.EstimatorOptions(grid_factor=4, backend="superfast")
obs = slse.Observation.complete(y)
r = slse.estimate(obs, opts)
ts = []
for _ in range(3):
    t = time.perf_counter(); r = slse.estimate(obs, opts); ts.append(time.perf_counter() - t)
print(f"cfg5 single estimate(): median {np.median(ts):.3f} s, k_hat {r.k_hat}, decomp {r.algorithms.get('decomp')}")
