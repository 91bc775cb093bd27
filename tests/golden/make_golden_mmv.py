"""Generate MMV (G > 1 snapshots) golden fixtures from the REAL reference.

Runs only in the build container (imports `superlse` from
/root/reference/pkg/src, read-only).  Problems come from
oracle.superlse_oracle.generate_problem_mmv, so the GPU tests can rebuild y
without the reference.  Records, per problem, the trajectory (objective
trace, stages, active-set history, final estimates with alpha_hat (G, k))
and one per-call bundle at the truth state (w, data term, per-snapshot
q/r/u, q_grid (G, L)), plus the oracle's near-tie decisions.

Usage:  python tests/golden/make_golden_mmv.py   (writes tests/golden/golden_mmv.npz)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import superlse  # noqa: E402
from superlse import estimator as ref_est  # noqa: E402
from superlse import model_core as ref_mc  # noqa: E402
from superlse import smlr as ref_smlr  # noqa: E402
from superlse import toeplitz as ref_tp  # noqa: E402

from golden_util import NEAR_TIE  # noqa: E402
from make_golden import SEED, STAGE_CODE, encode_events  # noqa: E402
from oracle import superlse_oracle as O  # noqa: E402

CASES = [(1, 3, 4), (2, 2, 2)]  # (cfg shape, G, problems)


def run_instrumented(y, grid_factor=4):
    events = []
    orig = (ref_smlr.initial_activation_sweep, ref_smlr.try_activate, ref_smlr.try_deactivate)
    grid_len = ref_mc.default_grid_size(y.shape[-1], grid_factor)

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
    return res, events


def per_call(y, thetas, gammas, beta, grid_len):
    obs = ref_mc.Observation.complete(y)
    eng = ref_mc.SuperfastEngine(obs, grid_size=grid_len, steer_method="direct")
    b = ref_mc._SuperfastBundle(eng, np.asarray(thetas, float), np.asarray(gammas, float), float(beta))
    out = dict(thetas=np.asarray(thetas, float), gammas=np.asarray(gammas, float), beta=float(beta),
               rho=b.decomp.rho, delta=b.decomp.delta, w=b.w.T.copy(), logdet=ref_tp.log_det(b.decomp),
               data_term=b.data_term)
    g = b.grid()
    out["q_grid"] = g.q_grid
    out["s_grid"] = g.s_grid
    st = b.stats()
    for k in "qru":
        out["st_" + k] = getattr(st, k)
    for k in "stvx":
        out["st_" + k] = getattr(st, k)
    return out


def main():
    store = {}
    for cfg, G, count in CASES:
        for b in range(count):
            y, truth = O.generate_problem_mmv(SEED, cfg, b, G)
            n = y.shape[1]
            L = ref_mc.default_grid_size(n, 4)
            res, events = run_instrumented(y)
            p = f"c{cfg}g{G}_p{b}_"
            store[p + "y"] = y
            store[p + "k_hat"] = res.k_hat
            store[p + "theta_hat"] = res.theta_hat
            store[p + "gamma_hat"] = res.gamma_hat
            store[p + "alpha_hat"] = res.alpha_hat
            store[p + "beta_hat"] = res.beta_hat
            store[p + "trace"] = np.asarray(res.objective_trace)
            store[p + "stages"] = np.array([STAGE_CODE[s] for s in res.trace_stages])
            store[p + "iterations"] = res.iterations
            store[p + "converged"] = res.converged
            store[p + "events"] = encode_events(events)
            o = O.estimate(y, O.OracleOptions(grid_factor=4))
            ties = [[int(pos), kind, float(mg)] for kind, mg, pos in o.margins if mg < NEAR_TIE]
            store[p + "near_tie_pos"] = np.array([t[0] for t in ties], dtype=np.int64)
            pc = per_call(y, truth["thetas"], np.mean(np.abs(truth["alphas"]) ** 2, axis=0), truth["beta"], L)
            for k, v in pc.items():
                store[p + "call_" + k] = v
            print(cfg, G, b, "k_hat", res.k_hat, "iters", res.iterations, "ties", ties, flush=True)
    store["cases"] = np.array(CASES, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_mmv.npz"), **store)


if __name__ == "__main__":
    main()
