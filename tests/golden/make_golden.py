"""Generate golden fixtures from the REAL reference implementation.

Runs only in the build container (needs /root/reference, read-only): it
imports `superlse` from /root/reference/pkg/src, solves seeded config-shaped
problems with ``EstimatorOptions(backend="superfast", grid_factor=4)`` and
records

* the trajectory: objective trace, trace stages, model order after every
  record, and the active-set history (sweep / activate / deactivate events,
  captured by wrapping ``superlse.smlr`` entry points, estimator.py:168-242);
* per-call quantities of the superfast bundle (model_core.py:256-313) at a
  few states: Toeplitz column, rho, delta, C^-1 y, log-det, data term, the
  omega diagonal sums, the seven component statistics and the activation
  grid.  Statistics use ``steer_method="direct"`` (SURVEY.md 8(c) caveat).

Inputs come from ``oracle.superlse_oracle.generate_problem`` so the GPU
tests can regenerate the same y on a box without /root/reference.

Usage:  python tests/golden/make_golden.py   (writes tests/golden/*.npz)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import superlse  # noqa: E402
from superlse import estimator as ref_est  # noqa: E402
from superlse import model_core as ref_mc  # noqa: E402
from superlse import smlr as ref_smlr  # noqa: E402
from superlse import toeplitz as ref_tp  # noqa: E402

from oracle.superlse_oracle import generate_problem  # noqa: E402

SEED = 20261019
STAGE_CODE = {"init": 0, "beta": 1, "activate": 2, "zeta": 3, "refine": 4, "deactivate": 5}


def run_instrumented(y, grid_factor=4):
    """Reference estimate() with the active-set history recorded."""
    events = []
    orig = (ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate)
    grid_len = ref_mc.default_grid_size(y.size, grid_factor)

    def sweep(state, obs, gs, tau=ref_smlr.DEFAULT_TAU):
        out = orig[0](state, obs, gs, tau=tau)
        new = np.flatnonzero(out.z & ~state.z)
        if new.size:
            events.append(("sweep", [(int(s), int(round(out.theta[s] * grid_len))) for s in new]))
        return out

    def act(state, obs, gs, tau=ref_smlr.DEFAULT_TAU):
        out = orig[1](state, obs, gs, tau=tau)
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
        res = superlse.estimate(ref_mc.Observation.complete(y),
                                ref_est.EstimatorOptions(backend="superfast", grid_factor=grid_factor))
    finally:
        ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate = orig
    slots = None
    return res, events


def encode_events(events):
    """Flatten to int64 rows (kind, slot, grid_index): kind 0 sweep, 1 activate, 2 deactivate;
    a -1 row separates events."""
    rows = []
    for ev in events:
        if ev[0] == "sweep":
            rows += [(0, s, i) for s, i in ev[1]]
        elif ev[0] == "activate":
            rows.append((1, ev[1], ev[2]))
        else:
            rows += [(2, s, -1) for s in ev[1]]
        rows.append((-1, -1, -1))
    return np.array(rows, dtype=np.int64).reshape(-1, 3)



def per_call(y, thetas, gammas, beta, grid_len):
    obs = ref_mc.Observation.complete(y)
    eng = ref_mc.SuperfastEngine(obs, grid_size=grid_len, steer_method="direct")
    b = ref_mc._SuperfastBundle(eng, np.asarray(thetas, float), np.asarray(gammas, float), float(beta))
    col = ref_mc.nufft.steer_forward(np.asarray(thetas, float), np.asarray(gammas, complex), y.size,
                                     method="direct")
    col[0] = col[0].real + beta
    om = b.omegas()
    out = dict(thetas=np.asarray(thetas, float), gammas=np.asarray(gammas, float), beta=float(beta),
               c=col, rho=b.decomp.rho, delta=b.decomp.delta, w=b.w[:, 0],
               logdet=ref_tp.log_det(b.decomp), data_term=b.data_term,
               om_s=om["s"], om_t=om["t"], om_v=om["v"], om_x=om["x"])
    g = b.grid()
    out["q_grid"] = g.q_grid[0]
    out["s_grid"] = g.s_grid
    if len(thetas):
        st = b.stats()
        for k in "qru":
            out["st_" + k] = getattr(st, k)[0]
        for k in "stvx":
            out["st_" + k] = getattr(st, k)
    return out


def main():
    jobs = [  # (cfg, count, per_call?)
        (1, 6, True),
        (2, 4, True),
        (3, 1, True),
        (4, 1, False),
    ]
    for cfg, count, with_calls in jobs:
        store = {}
        for b in range(count):
            y, truth = generate_problem(SEED, cfg, b)
            n = y.size
            L = ref_mc.default_grid_size(n, 4)
            res, events = run_instrumented(y)
            p = f"p{b}_"
            store[p + "y"] = y
            store[p + "k_hat"] = res.k_hat
            store[p + "theta_hat"] = res.theta_hat
            store[p + "gamma_hat"] = res.gamma_hat
            store[p + "alpha_hat"] = res.alpha_hat[0]
            store[p + "beta_hat"] = res.beta_hat
            store[p + "zeta_hat"] = res.zeta_hat
            store[p + "trace"] = res.objective_trace
            store[p + "stages"] = np.array([STAGE_CODE[s] for s in res.trace_stages], dtype=np.int64)
            store[p + "iterations"] = res.iterations
            store[p + "converged"] = res.converged
            store[p + "events"] = encode_events(events)
            store[p + "n_warnings"] = len(res.warnings)
            print(f"cfg{cfg} p{b}: k_hat={res.k_hat} (K={truth['thetas'].size}) it={res.iterations} "
                  f"records={len(res.trace_stages)} events={len(events)} "
                  f"t={res.wall_time_per_stage['total']:.2f}s", flush=True)
            if with_calls and b < 2:
                states = {
                    "empty": ([], [], float(np.sum(np.abs(y) ** 2)) / n),
                    "truth": (truth["thetas"], np.abs(truth["alphas"]) ** 2, truth["beta"]),
                    "final": (res.theta_hat, res.gamma_hat, res.beta_hat),
                }
                for name, (th, ga, be) in states.items():
                    for key, val in per_call(y, th, ga, be, L).items():
                        store[f"{p}call_{name}_{key}"] = val
        np.savez_compressed(os.path.join(HERE, f"golden_cfg{cfg}.npz"), seed=SEED, count=count, **store)


if __name__ == "__main__":
    main()
