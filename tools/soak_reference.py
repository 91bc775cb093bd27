"""Fresh-seed parity against the REAL reference (baseline/_ref, unmodified superlse) through both public APIs:
model order, frequencies (1e-8 wrap-around), amplitudes and noise variance (1e-6 relative), objective trace.
Usage: python tools/soak_reference.py [--configs 3,4,5] [--seed 777] [--count 16]"""
import argparse, os, sys
import multiprocessing as mp
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))


def _ref(y):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    import superlse
    r = superlse.estimate(superlse.Observation.complete(y), superlse.EstimatorOptions(backend="superfast", grid_factor=4))
    return (r.k_hat, np.asarray(r.theta_hat), np.asarray(r.alpha_hat), float(r.beta_hat), np.asarray(r.gamma_hat),
            np.asarray(r.objective_trace), bool(r.converged))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4,5")
    ap.add_argument("--seed", type=int, default=777)
    ap.add_argument("--count", type=int, default=16)
    a = ap.parse_args()
    from golden_util import AMP_TOL, THETA_TOL, rel, wrap_distance
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch, simdata
    bad = tot = 0
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for cfg in [int(c) for c in a.configs.split(",")]:
            Y = simdata.batch(a.seed, cfg, a.count)
            res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
            ref = pool.map(_ref, [Y[b] for b in range(Y.shape[0])], chunksize=1)
            worst = dict(theta=0.0, alpha=0.0, beta=0.0, trace=0.0)
            for b, (k, th, al, be, ga, tr, conv) in enumerate(ref):
                r = res[b]
                tot += 1
                why = []
                if r.status != 0: why.append(f"status {r.status}")
                if r.k_hat != k: why.append(f"k_hat {r.k_hat} vs {k}")
                if len(r.objective_trace) != len(tr): why.append(f"trace length {len(r.objective_trace)} vs {len(tr)}")
                if r.k_hat == k:
                    dt = float(np.max(wrap_distance(r.theta_hat, th), initial=0))
                    da = rel(r.alpha_hat[0], np.atleast_2d(al)[0])
                    db = abs(r.beta_hat - be) / be
                    worst["theta"] = max(worst["theta"], dt); worst["alpha"] = max(worst["alpha"], da)
                    worst["beta"] = max(worst["beta"], db)
                    m = min(len(r.objective_trace), len(tr))
                    worst["trace"] = max(worst["trace"], float(np.max(np.abs(np.asarray(r.objective_trace)[:m] - tr[:m]) / np.abs(tr[:m]))))
                    if dt >= THETA_TOL: why.append(f"theta {dt:.2e}")
                    if da >= AMP_TOL: why.append(f"alpha {da:.2e}")
                    if db >= AMP_TOL: why.append(f"beta {db:.2e}")
                if why:
                    bad += 1
                    print(f"DEVIATION cfg{cfg} seed {a.seed} problem {b}: {', '.join(why)}", flush=True)
            print(f"cfg{cfg} seed {a.seed}: {Y.shape[0]} problems vs the real reference; worst theta {worst['theta']:.2e} "
                  f"alpha {worst['alpha']:.2e} beta {worst['beta']:.2e} objective trace {worst['trace']:.2e}", flush=True)
    print(f"reference soak: {tot} problems, {bad} with deviations")


if __name__ == "__main__":
    main()
