"""Semifast-backend golden fixtures from the REAL reference (build container only).

Runs the reference ``superlse.estimate`` with ``backend="semifast"``
(SemifastEngine / _SemifastBundle, model_core.py:316-409, 456-460) on

* complete data at the cfg1 / cfg2 shapes (N = 64, 256: where the
  reference's own ``backend="auto"`` picks semifast, model_core.py:469-470);
* incomplete data (``Observation.incomplete``, model_core.py:43-130): seeded
  random observation patterns, unit and complex scales, and one MMV (G = 2)
  case;

and records the trajectory (objective trace, stages, active-set history,
estimates) plus per-call semifast bundle quantities (data term,
e = Phi^H C^-1 y, the seven statistics, the activation grid) at the truth,
final, empty and "one zero variance" states (``steer_method="direct"``).

Inputs: y from ``oracle.superlse_oracle.generate_problem[_mmv]`` and the
pattern from ``pattern()`` below, so the GPU tests rebuild nothing from the
reference; every array they need is stored.

Usage:  python tests/golden/make_golden_sf.py   (writes tests/golden/golden_sf.npz)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import superlse  # noqa: E402
from superlse import estimator as ref_est  # noqa: E402
from superlse import model_core as ref_mc  # noqa: E402
from superlse import smlr as ref_smlr  # noqa: E402

from make_golden import SEED, STAGE_CODE, encode_events  # noqa: E402
from oracle.superlse_oracle import generate_problem, generate_problem_mmv  # noqa: E402

# (name, cfg law, problem, N, K, M or None (complete), scales kind, G)
CASES = [
    ("c1a", 1, 0, None, None, None, None, 1),
    ("c1b", 1, 1, None, None, None, None, 1),
    ("c1c", 1, 2, None, None, None, None, 1),
    ("c2a", 2, 0, None, None, None, None, 1),
    ("c2b", 2, 1, None, None, None, None, 1),
    ("i1a", 1, 3, 64, 4, 40, "ones", 1),
    ("i1b", 1, 4, 64, 4, 48, "complex", 1),
    ("i2a", 2, 2, 128, 8, 80, "complex", 1),
    ("i2b", 2, 3, 256, 12, 160, "ones", 1),
    ("m1a", 1, 5, 64, 4, 44, "complex", 2),
    # near-resolution-limit problems whose reference run removes components
    # (the superfast deactivation cases, make_golden_r2.DEACT_CASES), complete
    # and with a pattern
    ("d1a", 5, 7, 128, 16, None, None, 1, 99),
    ("d1b", 5, 92, 128, 24, 112, "ones", 1, 99),
]


def pattern(seed, b, n, m, kind):
    """Seeded observation pattern: 1-based sorted positions and scales."""
    rng = np.random.default_rng([seed, 77, b])
    idx = np.sort(rng.choice(n, size=m, replace=False)) + 1
    if kind == "ones":
        sc = np.ones(m, dtype=np.complex128)
    else:
        sc = rng.uniform(0.5, 1.5, m) * np.exp(2j * np.pi * rng.uniform(0.0, 1.0, m))
    return idx.astype(np.int64), sc.astype(np.complex128)


def make_obs(case):
    name, cfg, b, n, k, m, kind, g = case[:8]
    seed = case[8] if len(case) > 8 else SEED
    if g > 1:
        yf, truth = generate_problem_mmv(seed, cfg, b, g, n=n, k=k)
    else:
        yf, truth = generate_problem(seed, cfg, b, n=n, k=k)
        yf = yf[None, :]
    nn = yf.shape[-1]
    if m is None:
        return ref_mc.Observation.complete(yf), truth, None, None
    idx, sc = pattern(seed, b, nn, m, kind)
    y = sc[None, :] * yf[:, idx - 1]
    return ref_mc.Observation.incomplete(y, nn, idx, sc), truth, idx, sc


def run_instrumented(obs, grid_factor=4):
    """Reference semifast estimate() with the active-set history recorded."""
    events = []
    orig = (ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate)
    grid_len = ref_mc.default_grid_size(obs.n, grid_factor)

    def sweep(state, o, gs, tau=ref_smlr.DEFAULT_TAU):
        out = orig[0](state, o, gs, tau=tau)
        new = np.flatnonzero(out.z & ~state.z)
        if new.size:
            events.append(("sweep", [(int(s), int(round(out.theta[s] * grid_len))) for s in new]))
        return out

    def act(state, o, gs, tau=ref_smlr.DEFAULT_TAU):
        out = orig[1](state, o, gs, tau=tau)
        if out is not None:
            s = int(np.flatnonzero(out.z & ~state.z)[0])
            events.append(("activate", s, int(round(out.theta[s] * grid_len))))
        return out

    def deact(state, stats, recompute=None):
        out, removed = orig[2](state, stats, recompute=recompute)
        if removed:
            events.append(("deactivate", [int(r) for r in removed]))
        return out, removed

    ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate = sweep, act, deact
    try:
        res = superlse.estimate(obs, ref_est.EstimatorOptions(backend="semifast", grid_factor=grid_factor))
    finally:
        ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate = orig
    return res, events


def per_call(obs, thetas, gammas, beta, grid_len):
    """Semifast bundle quantities (model_core.py:316-409) with direct sums."""
    eng = ref_mc.SemifastEngine(obs, grid_size=grid_len, steer_method="direct")
    b = ref_mc._SemifastBundle(eng, np.asarray(thetas, float), np.asarray(gammas, float), float(beta))
    out = dict(thetas=np.asarray(thetas, float), gammas=np.asarray(gammas, float), beta=float(beta),
               data_term=b.data_term, e=b.e.T.copy())  # e: (G, N)
    g = b.grid()
    out["q_grid"] = g.q_grid  # (G, L)
    out["s_grid"] = g.s_grid
    if len(thetas):
        st = b.stats()
        for key in "qru":
            out["st_" + key] = getattr(st, key)  # (G, K)
        for key in "stvx":
            out["st_" + key] = getattr(st, key)
    return out


def main():
    store = {}
    names = []
    for case in CASES:
        name = case[0]
        obs, truth, idx, sc = make_obs(case)
        L = ref_mc.default_grid_size(obs.n, 4)
        res, events = run_instrumented(obs)
        p = name + "_"
        store[p + "y"] = obs.y  # (G, M)
        store[p + "n"] = obs.n
        if idx is not None:
            store[p + "idx"] = idx
            store[p + "scales"] = sc
        store[p + "k_hat"] = res.k_hat
        store[p + "theta_hat"] = res.theta_hat
        store[p + "gamma_hat"] = res.gamma_hat
        store[p + "alpha_hat"] = res.alpha_hat  # (G, k)
        store[p + "beta_hat"] = res.beta_hat
        store[p + "zeta_hat"] = res.zeta_hat
        store[p + "trace"] = res.objective_trace
        store[p + "stages"] = np.array([STAGE_CODE[s] for s in res.trace_stages], dtype=np.int64)
        store[p + "iterations"] = res.iterations
        store[p + "converged"] = res.converged
        store[p + "events"] = encode_events(events)
        # per-call states: truth, final, empty, and the final state with one
        # variance set to zero (outside the Cholesky's positive set, :325)
        th_t, ga_t = truth["thetas"], np.abs(truth["alphas"]) ** 2
        if ga_t.ndim > 1:
            ga_t = np.mean(ga_t, axis=0)
        states = {"truth": (th_t, ga_t, truth["beta"]),
                  "final": (res.theta_hat, res.gamma_hat, res.beta_hat),
                  "empty": (np.zeros(0), np.zeros(0), obs.energy() / obs.m)}
        if res.k_hat >= 2:
            gz = res.gamma_hat.copy()
            gz[1] = 0.0
            states["zgamma"] = (res.theta_hat, gz, res.beta_hat)
        for sname, (th, ga, be) in states.items():
            for key, val in per_call(obs, th, ga, be, L).items():
                store[f"{p}call_{sname}_{key}"] = val
        store[p + "states"] = np.array(list(states), dtype=object).astype(str)
        names.append(name)
        print(f"{name}: N={obs.n} M={obs.m} G={obs.g} k_hat={res.k_hat} records={len(res.trace_stages)} "
              f"events={len(events)} deact={sum(1 for e in events if e[0] == 'deactivate')}", flush=True)
    np.savez_compressed(os.path.join(HERE, "golden_sf.npz"), seed=SEED, names=np.array(names), **store)


if __name__ == "__main__":
    main()
