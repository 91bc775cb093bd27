"""Diagnostic: per-record objective-trace and stage differences of the GPU
solve against a golden trajectory fixture (tests/golden)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from golden_util import STAGES, load, near_ties, encode_events
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

cfg = sys.argv[1]
cfg = int(cfg) if cfg.isdigit() else cfg
method = sys.argv[2] if len(sys.argv) > 2 else "auto"
z = load(cfg)
probs = [int(b) for b in z["problems"]] if "problems" in z.files else list(range(int(z["count"])))
for b in probs:
    p = f"p{b}_"
    r = estimate_batch(z[p + "y"][None, :], EstimatorOptions(grid_factor=4, backend="superfast", decomp_method=method))[0]
    st = np.array([STAGES.index(s) for s in r.trace_stages]); gs = z[p + "stages"]
    tr = np.asarray(r.objective_trace); gt = z[p + "trace"]
    m = min(tr.size, gt.size)
    print(f"== cfg{cfg} p{b}: k_hat {r.k_hat} vs {int(z[p+'k_hat'])}; records {tr.size} vs {gt.size}; "
          f"events equal {np.array_equal(encode_events(r.events), z[p+'events'])}; ties {near_ties(cfg, b)}")
    for i in range(m):
        d = abs(tr[i] - gt[i]) / abs(gt[i])
        flag = " <" if d > 1e-9 or st[i] != gs[i] else ""
        print(f"  {i:3d} {STAGES[st[i]]:10s} {STAGES[gs[i]]:10s} {tr[i]:.12e} {gt[i]:.12e} {d:.2e}{flag}")
