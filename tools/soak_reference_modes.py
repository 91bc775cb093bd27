"""Fresh-seed parity against the REAL reference (baseline/_ref) for the other data forms of estimate():
incomplete data (random pattern, complex scales; the semifast backend) and MMV (G snapshots, superfast and semifast).
Usage: python tools/soak_reference_modes.py [--seed 909] [--count 32]"""
import argparse, os, sys
import multiprocessing as mp
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))


def _ref(args):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    import superlse
    y, n, idx, sc, backend = args
    obs = superlse.Observation.complete(y) if idx is None else superlse.Observation.incomplete(y, n, idx, sc)
    r = superlse.estimate(obs, superlse.EstimatorOptions(backend=backend, grid_factor=4))
    return r.k_hat, np.asarray(r.theta_hat), np.asarray(r.alpha_hat), float(r.beta_hat), len(r.objective_trace)


def scene(rng, n, k, g, snr_db):
    th = np.sort(rng.uniform(0, 1, k))
    while k > 1 and np.min(np.diff(np.concatenate([th, [th[0] + 1]]))) < 1.5 / n:
        th = np.sort(rng.uniform(0, 1, k))
    al = (rng.standard_normal((g, k)) + 1j * rng.standard_normal((g, k))) / np.sqrt(2)
    x = al @ np.exp(2j * np.pi * np.outer(th, np.arange(n)))
    p = np.mean(np.abs(x) ** 2)
    w = (rng.standard_normal((g, n)) + 1j * rng.standard_normal((g, n))) * np.sqrt(p / 10 ** (snr_db / 10) / 2)
    return x + w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=909)
    ap.add_argument("--count", type=int, default=32)
    a = ap.parse_args()
    from golden_util import AMP_TOL, THETA_TOL, rel, wrap_distance
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
    rng = np.random.default_rng(a.seed)
    cases = []
    for n, k in ((128, 6), (256, 12)):   # incomplete data, shared pattern with complex scales
        m = int(0.7 * n)
        idx = np.sort(rng.choice(n, size=m, replace=False)) + 1
        sc = rng.uniform(0.5, 1.5, m) * np.exp(2j * np.pi * rng.uniform(0, 1, m))
        Y = np.stack([(scene(rng, n, k, 1, 18.0)[0][idx - 1] * sc) for _ in range(a.count)])
        cases.append((f"incomplete N={n} M={m} K={k} (semifast)", Y, n, idx, sc, "semifast"))
    for n, k, g, backend in ((256, 10, 4, "superfast"), (128, 6, 3, "semifast"), (1024, 24, 2, "superfast")):
        Y = np.stack([scene(rng, n, k, g, 15.0) for _ in range(a.count)])
        cases.append((f"MMV N={n} G={g} K={k} ({backend})", Y, n, None, None, backend))
    bad = tot = 0
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for name, Y, n, idx, sc, backend in cases:
            if idx is None:
                res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend=backend))
            else:
                res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend=backend), n=n, observed_indices=idx, scales=sc)
            ref = pool.map(_ref, [(Y[b], n, idx, sc, backend) for b in range(Y.shape[0])], chunksize=1)
            worst = dict(theta=0.0, alpha=0.0, beta=0.0)
            for b, (k, th, al, be, nt) in enumerate(ref):
                r = res[b]
                tot += 1
                why = []
                if r.status != 0: why.append(f"status {r.status}")
                if r.k_hat != k: why.append(f"k_hat {r.k_hat} vs {k}")
                if abs(len(r.objective_trace) - nt) > 1: why.append(f"trace length {len(r.objective_trace)} vs {nt}")
                if r.k_hat == k:
                    dt = float(np.max(wrap_distance(r.theta_hat, th), initial=0))
                    da = rel(np.asarray(r.alpha_hat), np.atleast_2d(al))
                    db = abs(r.beta_hat - be) / be
                    worst["theta"] = max(worst["theta"], dt); worst["alpha"] = max(worst["alpha"], da); worst["beta"] = max(worst["beta"], db)
                    if dt >= THETA_TOL: why.append(f"theta {dt:.2e}")
                    if da >= AMP_TOL: why.append(f"alpha {da:.2e}")
                    if db >= AMP_TOL: why.append(f"beta {db:.2e}")
                if why:
                    bad += 1
                    print(f"DEVIATION {name} problem {b}: {', '.join(why)}", flush=True)
            print(f"{name}: {Y.shape[0]} problems vs the real reference; worst theta {worst['theta']:.2e} alpha {worst['alpha']:.2e} "
                  f"beta {worst['beta']:.2e}", flush=True)
    print(f"reference soak (incomplete / MMV): {tot} problems, {bad} with deviations")


if __name__ == "__main__":
    main()
