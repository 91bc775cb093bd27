"""Builds per problem: GPU solver (2 bundle slots) vs the oracle's LRU(4)
engine (the reference's cache, model_core.py:416-444) on the same inputs."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import superlse_oracle as O
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

cfg = int(sys.argv[1]); count = int(sys.argv[2]); n = int(sys.argv[3]) if len(sys.argv) > 3 else None
k = int(sys.argv[4]) if len(sys.argv) > 4 else None
Y = O.generate_batch(20261019, cfg, count, n=n, k=k)
res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
for b in range(count):
    t = time.time()
    o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
    r = res[b]
    print(f"p{b}: gpu builds {r.counters['builds']} grids {r.counters['grids']} stats {r.counters['stats']} "
          f"trials {r.counters['line_search_trials']} | oracle builds {o.builds} | records {len(r.trace_stages)} vs "
          f"{len(o.trace_stages)} same={r.trace_stages == o.trace_stages} ({time.time()-t:.1f}s)", flush=True)
