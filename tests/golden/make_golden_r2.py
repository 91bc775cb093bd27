"""Round-2 golden fixtures from the REAL reference (build container only).

Extends tests/golden/make_golden.py (same recorder, same per-call dump) to
the shapes and code paths round 1 left without reference evidence:

* ``golden_cfg5.npz`` -- the cfg5 shape (N = 16384, K = 512, L = 4N):
  trajectories of problems 0 and 1 with the reference's default
  (``steer_method="auto"``: NUFFT at N >= 512) and a second trajectory of
  each with ``steer_method="direct"`` (prefix ``p{b}d_``: the reference's own
  spread between its two statistics methods); per-call bundle quantities
  (``steer_method="direct"``, SURVEY.md 8(c) caveat) at the truth / final /
  empty states of problem 0 and the final state of problem 1.
* ``golden_cfg4x.npz`` -- cfg4 problems 1 and 2: trajectories plus
  per-call states truth / final (round 1 had one cfg4 trajectory and no
  per-call state).
* ``golden_deact.npz`` -- problems whose reference run REMOVES components
  (smlr.try_deactivate, smlr.py:203-225; estimator.py:235-242), found by
  scanning seeded near-resolution-limit problems (tools: the scan list in
  DEACT_CASES), with trajectories and the per-call state just before the
  first removal.

Large per-call vectors (omega sums, the activation grid) are stored
decimated at N >= 4096 (every DECIM-th entry, keys ending ``_dec``) to keep
the fixtures small; rho, delta, c and w are stored in full.

Usage:  python tests/golden/make_golden_r2.py [cfg5|cfg4x|deact ...]
"""

import multiprocessing as mp
import os
import re
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

import make_golden as MG  # noqa: E402  (imports /root/reference superlse)
from oracle.superlse_oracle import generate_problem  # noqa: E402

SEED = MG.SEED
DECIM = 16
BIG = ("om_s", "om_t", "om_v", "om_x", "q_grid", "s_grid")

# (seed, cfg-law, problem, N, K): reference runs that deactivate (scan in
# /tmp, recorded here; each verified again when the fixture is written)
DEACT_CASES = [
    (99, 5, 7, 128, 16),
    (99, 5, 0, 256, 32),
    (99, 5, 92, 128, 24),
    (99, 5, 72, 1024, 64),
]


def _traj(y, steer="auto"):
    """Reference trajectory (make_golden.run_instrumented with a steer method)."""
    from superlse import estimator as ref_est
    from superlse import model_core as ref_mc
    from superlse import smlr as ref_smlr
    import superlse

    if steer == "auto":
        return MG.run_instrumented(y)
    orig_est = superlse.estimate

    def est(obs, opts):
        opts.steer_method = steer
        return orig_est(obs, opts)

    superlse.estimate = est
    try:
        return MG.run_instrumented(y)
    finally:
        superlse.estimate = orig_est
    del ref_est, ref_mc, ref_smlr


def _store_traj(store, p, res, events):
    store[p + "k_hat"] = res.k_hat
    store[p + "theta_hat"] = res.theta_hat
    store[p + "gamma_hat"] = res.gamma_hat
    store[p + "alpha_hat"] = res.alpha_hat[0]
    store[p + "beta_hat"] = res.beta_hat
    store[p + "zeta_hat"] = res.zeta_hat
    store[p + "trace"] = res.objective_trace
    store[p + "stages"] = np.array([MG.STAGE_CODE[s] for s in res.trace_stages], dtype=np.int64)
    store[p + "iterations"] = res.iterations
    store[p + "converged"] = res.converged
    store[p + "events"] = MG.encode_events(events)
    store[p + "n_warnings"] = len(res.warnings)
    store[p + "seconds"] = res.wall_time_per_stage["total"]


def _store_call(store, p, y, th, ga, be, L, decim):
    for key, val in MG.per_call(y, th, ga, be, L).items():
        if decim > 1 and key in BIG:
            store[p + key + "_dec"] = val[::decim]
            store[p + key + "_max"] = float(np.max(np.abs(val)))  # the full vector's inf-norm (the rel denominator)
        else:
            store[p + key] = val


def job_traj(args):
    cfg, b, steer, n, k, seed = args
    y, truth = generate_problem(seed, cfg, b, n=n, k=k)
    res, events = _traj(y, steer)
    return args, y, truth, res, events


def job_call(args):
    cfg, b, name, th, ga, be, n, k, seed, decim = args
    y, _ = generate_problem(seed, cfg, b, n=n, k=k)
    L = 4 * y.size
    st = {}
    _store_call(st, "", y, th, ga, be, L, decim)
    return args[:3], st


def build_traj_fixture(cfg, problems, calls, out_name, extra_direct=(), nproc=8):
    """problems: problem indices; calls: {b: [state names]}; extra_direct: problems
    also traced with steer_method="direct" (prefix p{b}d_)."""
    jobs = [(cfg, b, "auto", None, None, SEED) for b in problems]
    jobs += [(cfg, b, "direct", None, None, SEED) for b in extra_direct]
    store = {}
    finals = {}
    truths = {}
    with mp.get_context("fork").Pool(min(nproc, len(jobs))) as pool:
        for (c, b, steer, _, _, _), y, truth, res, events in pool.imap_unordered(job_traj, jobs):
            p = f"p{b}_" if steer == "auto" else f"p{b}d_"
            store[f"p{b}_y"] = y
            _store_traj(store, p, res, events)
            if steer == "auto":
                finals[b] = (res.theta_hat, res.gamma_hat, res.beta_hat)
                truths[b] = (truth["thetas"], np.abs(truth["alphas"]) ** 2, truth["beta"])
            print(f"cfg{cfg} {p}: k_hat={res.k_hat} it={res.iterations} records={len(res.trace_stages)} "
                  f"events={len(events)} t={res.wall_time_per_stage['total']:.1f}s", flush=True)
    n = store[f"p{problems[0]}_y"].size
    decim = DECIM if n >= 4096 else 1
    cjobs = []
    for b, names in calls.items():
        for name in names:
            if name == "empty":
                y = store[f"p{b}_y"]
                th, ga, be = np.zeros(0), np.zeros(0), float(np.sum(np.abs(y) ** 2)) / n
            else:
                th, ga, be = (truths if name == "truth" else finals)[b]
            cjobs.append((cfg, b, name, th, ga, be, None, None, SEED, decim))
    with mp.get_context("fork").Pool(min(nproc, max(1, len(cjobs)))) as pool:
        for (c, b, name), st in pool.imap_unordered(job_call, cjobs):
            for key, val in st.items():
                store[f"p{b}_call_{name}_{key}"] = val
            print(f"cfg{cfg} p{b} call {name} done", flush=True)
    np.savez_compressed(os.path.join(HERE, out_name), seed=SEED, count=len(problems),
                        problems=np.array(problems), decim=decim, **store)


def build_deact_fixture(nproc=8):
    """Deactivating problems: trajectory + the state right before the first removal."""
    from superlse import smlr as ref_smlr

    store = {}
    rows = []
    jobs = [(law, b, "auto", n, k, seed) for seed, law, b, n, k in DEACT_CASES]
    with mp.get_context("fork").Pool(min(nproc, len(jobs))) as pool:
        results = pool.map(job_traj, jobs)
    for i, ((law, b, _, n, k, seed), y, truth, res, events) in enumerate(results):
        kinds = [e[0] for e in events]
        assert "deactivate" in kinds, (seed, law, b, n, k)
        p = f"p{i}_"
        store[p + "y"] = y
        _store_traj(store, p, res, events)
        rows.append((seed, law, b, n, k))
        print(f"deact case {i} {(seed, law, b, n, k)}: k_hat={res.k_hat} events={events}", flush=True)
    # per-call margins at the state right before the first removal of case 0
    captured = {}
    orig = ref_smlr.try_deactivate

    def deact(state, stats, recompute=None):
        if "state" not in captured:
            out, removed = orig(state, stats, recompute=recompute)
            if removed:
                captured["state"] = (state.theta[state.z].copy(), state.gamma[state.z].copy(), float(state.beta),
                                     float(state.zeta), int(state.k_max))
                captured["slots"] = state.active_indices.copy()
                captured["margins"] = ref_smlr.deactivation_margins(state, stats)
                captured["removed"] = list(removed)
            return out, removed
        return orig(state, stats, recompute=recompute)

    ref_smlr.try_deactivate = deact
    try:
        MG.run_instrumented(store["p0_y"])
    finally:
        ref_smlr.try_deactivate = orig
    th, ga, be, zeta, kmax = captured["state"]
    n = store["p0_y"].size
    for key, val in MG.per_call(store["p0_y"], th, ga, be, 4 * n).items():
        store["p0_call_predeact_" + key] = val
    store["p0_call_predeact_zeta"] = zeta
    store["p0_call_predeact_kmax"] = kmax
    store["p0_call_predeact_margins"] = np.asarray(captured["margins"], float)
    store["p0_call_predeact_removed"] = np.asarray(captured["removed"], np.int64)
    store["p0_call_predeact_slots"] = np.asarray(captured["slots"], np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_deact.npz"), count=len(rows), cases=np.array(rows, np.int64),
                        **store)


def refresh_calls(out_name, nproc=8):
    """Recompute the per-call entries of an existing fixture from its stored
    states (no trajectory rerun); the recomputed values must equal the stored
    ones, and the new keys (the full-vector inf-norms of decimated vectors)
    are added."""
    path = os.path.join(HERE, out_name)
    z = np.load(path)
    store = {k: z[k] for k in z.files}
    decim = int(z["decim"])
    cfg = 5 if "cfg5" in out_name else 4
    cjobs = []
    for k in z.files:
        m = re.match(r"p(\d+)_call_(\w+?)_thetas$", k)
        if m:
            b, name = int(m.group(1)), m.group(2)
            p = f"p{b}_call_{name}_"
            cjobs.append((cfg, b, name, z[p + "thetas"], z[p + "gammas"], float(z[p + "beta"]), None, None,
                          SEED, decim))
    with mp.get_context("fork").Pool(min(nproc, max(1, len(cjobs)))) as pool:
        for (c, b, name), st in pool.imap_unordered(job_call, cjobs):
            for key, val in st.items():
                full = f"p{b}_call_{name}_{key}"
                if full in store:
                    assert np.array_equal(np.asarray(store[full]), np.asarray(val)), full
                store[full] = val
            print(f"{out_name} p{b} call {name} refreshed", flush=True)
    np.savez_compressed(path, **store)


def add_direct(out_name, cfg, b):
    """Add problem b's steer_method="direct" reference trajectory (p{b}d_)
    to an existing fixture."""
    path = os.path.join(HERE, out_name)
    z = np.load(path)
    store = {k: z[k] for k in z.files}
    (_, _, _, _, _, _), y, _, res, events = job_traj((cfg, b, "direct", None, None, SEED))
    assert np.array_equal(y, store[f"p{b}_y"])
    _store_traj(store, f"p{b}d_", res, events)
    print(f"{out_name} p{b}d_: k_hat={res.k_hat} records={len(res.trace_stages)}", flush=True)
    np.savez_compressed(path, **store)


def main():
    what = sys.argv[1:] or ["deact", "cfg4x", "cfg5"]
    if "cfg5d1" in what:
        add_direct("golden_cfg5.npz", 5, 1)
        return
    if "refresh" in what:
        refresh_calls("golden_cfg4x.npz")
        refresh_calls("golden_cfg5.npz")
        return
    if "deact" in what:
        build_deact_fixture()
    if "cfg4x" in what:
        build_traj_fixture(4, [1, 2], {1: ["truth", "final"], 2: ["truth", "final"]}, "golden_cfg4x.npz")
    if "cfg5" in what:
        build_traj_fixture(5, [0, 1], {0: ["truth", "final", "empty"], 1: ["final"]}, "golden_cfg5.npz",
                           extra_direct=[0, 1])


if __name__ == "__main__":
    main()
