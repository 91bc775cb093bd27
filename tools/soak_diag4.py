"""cfg4 soak mismatches: GPU vs oracle port vs the REAL reference (baseline/_ref) on the same problems."""
import sys, os, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'baseline/_ref')
from golden_util import rel, wrap_distance
from oracle import superlse_oracle as O
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
import superlse
Y = O.generate_batch(301, 4, 16)
for b in (11, 12, 3):
    r = estimate_batch(Y[b:b+1], EstimatorOptions(grid_factor=4, backend="superfast"))[0]
    o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
    f = superlse.estimate(superlse.Observation.complete(Y[b]), superlse.EstimatorOptions(backend="superfast", grid_factor=4))
    fa = np.atleast_2d(np.asarray(f.alpha_hat))[0]
    print(f"p{b}: k_hat gpu {r.k_hat} oracle {o.k_hat} ref {f.k_hat}")
    print("   alpha rel: gpu-oracle", rel(r.alpha_hat[0], np.atleast_2d(o.alpha_hat)[0]), " gpu-ref", rel(r.alpha_hat[0], fa), " oracle-ref", rel(np.atleast_2d(o.alpha_hat)[0], fa))
    print("   theta wrap: gpu-oracle", float(np.max(wrap_distance(r.theta_hat, o.theta_hat))), " gpu-ref", float(np.max(wrap_distance(r.theta_hat, np.asarray(f.theta_hat)))),
          " oracle-ref", float(np.max(wrap_distance(np.asarray(o.theta_hat), np.asarray(f.theta_hat)))))
    print("   beta rel: gpu-ref", abs(r.beta_hat - f.beta_hat) / f.beta_hat, " oracle-ref", abs(o.beta_hat - f.beta_hat) / f.beta_hat)
