"""cfg5 seed 1002 problem 10: GPU vs the real reference with its default (NUFFT) and direct steering sums."""
import sys, os, time, numpy as np
import multiprocessing as mp
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'baseline/_ref')
from golden_util import rel, wrap_distance
from paper_1705_06073_b200 import EstimatorOptions, estimate_batch, simdata


def run(args):
    y, sm = args
    import superlse
    r = superlse.estimate(superlse.Observation.complete(y), superlse.EstimatorOptions(backend="superfast", grid_factor=4, steer_method=sm))
    return r.k_hat, np.asarray(r.theta_hat), np.asarray(r.alpha_hat), float(r.beta_hat), np.asarray(r.gamma_hat)


Y = simdata.batch(1002, 5, 16)
b = 10
g = estimate_batch(Y[b:b + 1], EstimatorOptions(grid_factor=4, backend="superfast"))[0]
with mp.get_context("fork").Pool(2) as pool:
    (ka, ta, aa, ba, ga), (kd, td, ad, bd, gd) = pool.map(run, [(Y[b], "auto"), (Y[b], "direct")])
aa, ad = np.atleast_2d(aa)[0], np.atleast_2d(ad)[0]
print("k_hat gpu / ref auto / ref direct:", g.k_hat, ka, kd)
print("alpha rel: gpu-refauto", rel(g.alpha_hat[0], aa), " gpu-refdirect", rel(g.alpha_hat[0], ad), " refauto-refdirect", rel(aa, ad))
print("theta: gpu-refauto", float(np.max(wrap_distance(g.theta_hat, ta))), " gpu-refdirect", float(np.max(wrap_distance(g.theta_hat, td))),
      " refauto-refdirect", float(np.max(wrap_distance(ta, td))))
print("beta rel: gpu-refauto", abs(g.beta_hat - ba) / ba, " gpu-refdirect", abs(g.beta_hat - bd) / bd, " refauto-refdirect", abs(ba - bd) / bd)
i = int(np.argmax(np.abs(g.alpha_hat[0] - aa)))
srt = np.sort(g.theta_hat)
j = int(np.searchsorted(srt, g.theta_hat[i]))
print("worst component: |alpha|", abs(aa[i]), "max |alpha|", float(np.max(np.abs(aa))), " nearest neighbour distance x N:",
      float(min(srt[j] - srt[j - 1] if j > 0 else 1, srt[(j + 1) % len(srt)] - srt[j] if j + 1 < len(srt) else 1) * 16384))
