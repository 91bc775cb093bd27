import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import superlse_oracle as O
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
for cfg, seed, b in ((1, 102, 18), (1, 103, 46), (2, 103, 60), (2, 104, 54)):
    Y = O.generate_batch(seed, cfg, 64)
    r = estimate_batch(Y[b:b+1], EstimatorOptions(grid_factor=4, backend="superfast"))[0]
    o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
    a, c = list(r.trace_stages), list(o.trace_stages)
    i = next((i for i in range(min(len(a), len(c))) if a[i] != c[i]), min(len(a), len(c)))
    print(f"cfg{cfg} seed {seed} p{b}: len gpu {len(a)} oracle {len(c)} first diff at {i}: gpu {a[i-1:i+3]} oracle {c[i-1:i+3]}")
    tg, to = np.asarray(r.objective_trace), np.asarray(o.objective_trace)
    m = min(len(tg), len(to))
    print("   objective rel diff before divergence:", float(np.max(np.abs(tg[:i] - to[:i]) / np.abs(to[:i]))) if i else None,
          " at i-1:", tg[i-1], to[i-1], " next:", tg[i:i+2], to[i:i+2])
    print("   final objective gpu/oracle:", tg[-1], to[-1], "iterations", r.iterations, o.iterations if hasattr(o,'iterations') else None,
          " theta diff", float(np.max(np.abs(np.sort(r.theta_hat) - np.sort(o.theta_hat)))))
