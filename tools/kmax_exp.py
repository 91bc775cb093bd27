"""Experiment: cfg2 solve time vs K_max (slab size; K_max also changes the
prior term, so compare builds too)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import EstimatorOptions, simdata
from paper_1705_06073_b200.estimator import BatchSolver
Y = torch.from_numpy(simdata.batch(20261019, 2)).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for km in (256, 128, 64, 32):
    s = BatchSolver(256, Y.shape[0], EstimatorOptions(grid_factor=4, backend="superfast", k_max=km))
    print("slab bytes/solver", s.workspace.numel() / 2368)
    for _ in range(2): s.solve(Y)
    ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.solve(Y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    h = s.host_outputs()
    print(f"k_max {km}: {min(ts):.2f} ms (median {sorted(ts)[2]:.2f}); builds {h['counters'][:,0].sum()} status!=0 {int((h['status']!=0).sum())}", flush=True)
