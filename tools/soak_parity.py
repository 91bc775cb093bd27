"""Randomised parity soak: fresh seeds, GPU estimate_batch (superfast and semifast) vs the CPU oracle
on the same problems (model order, stage trace, active-set history, estimates).  Test infrastructure:
the oracle is only the checker.  Usage: python tools/soak_parity.py [--seeds 11,12,13] [--per-seed 64]"""
import argparse, os, sys
import multiprocessing as mp
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def _oracle(args):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import superlse_oracle as O
    y, backend = args
    o = O.estimate(y, O.OracleOptions(grid_factor=4, backend=backend)) if backend != "superfast" else \
        O.estimate(y, O.OracleOptions(grid_factor=4))
    return o.k_hat, list(o.trace_stages), o.events, np.asarray(o.theta_hat), np.asarray(o.alpha_hat), float(o.beta_hat)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", default="101,102,103,104")
    ap.add_argument("--per-seed", type=int, default=64)
    ap.add_argument("--configs", default="1,2")
    ap.add_argument("--backends", default="superfast,semifast")
    a = ap.parse_args()
    from golden_util import AMP_TOL, THETA_TOL, encode_events, rel, wrap_distance
    from oracle import superlse_oracle as O
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
    import inspect
    has_backend = "backend" in inspect.signature(O.OracleOptions).parameters
    bad = tot = 0
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for cfg in [int(c) for c in a.configs.split(",")]:
            for seed in [int(s) for s in a.seeds.split(",")]:
                Y = O.generate_batch(seed, cfg, a.per_seed)
                for backend in [x for x in a.backends.split(",") if x == "superfast" or has_backend]:
                    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend=backend))
                    ref = pool.map(_oracle, [(Y[b], backend) for b in range(Y.shape[0])], chunksize=1)
                    for b, (k, stages, events, th, al, be) in enumerate(ref):
                        r = res[b]
                        tot += 1
                        why = []
                        if r.status != 0: why.append(f"status {r.status}")
                        if r.k_hat != k: why.append(f"k_hat {r.k_hat} vs {k}")
                        if r.trace_stages != stages: why.append("stage trace")
                        if encode_events(r.events).tolist() != encode_events(events).tolist(): why.append("history")
                        if not why:
                            if np.max(wrap_distance(r.theta_hat, th), initial=0) >= THETA_TOL: why.append("theta")
                            if rel(r.alpha_hat[0], np.atleast_2d(al)[0]) >= AMP_TOL: why.append("alpha")
                            if abs(r.beta_hat - be) / be >= AMP_TOL: why.append("beta")
                        if why:
                            bad += 1
                            print(f"MISMATCH cfg{cfg} seed {seed} problem {b} backend {backend}: {', '.join(why)}", flush=True)
                    print(f"cfg{cfg} seed {seed} {backend}: {Y.shape[0]} problems checked ({bad} mismatches so far)", flush=True)
    print(f"soak: {tot} problem-runs, {bad} mismatches")


if __name__ == "__main__":
    main()
