"""GPU parity of the semifast (Woodbury) backend -- complete and incomplete
data -- against fixtures written by the REAL reference
(tests/golden/make_golden_sf.py: superlse.estimate(..., backend="semifast"),
model_core._SemifastBundle :316-409, Observation.incomplete :43-130).

* per-call: data term, e = Phi^H C^-1 y, the seven statistics and the
  activation grid of one bundle at the truth / final / empty / zero-variance
  states, each at the north-star 1e-9 relative bar;
* trajectories: identical model order, stages and active-set history
  (deactivation included), trace within 1e-9 relative, estimates within the
  north-star bars -- through estimate_batch and the drop-in estimate();
* the K-capacity rerun path and batched per-problem patterns.
"""

import numpy as np
import pytest

from golden_util import AMP_TOL, CALL_TOL, STAGES, THETA_TOL, encode_events, rel, wrap_distance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _z():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_sf.npz"))


Z = None


def fx():
    global Z
    if Z is None:
        Z = _z()
    return Z


NAMES = ["c1a", "c1b", "c1c", "c2a", "c2b", "i1a", "i1b", "i2a", "i2b", "m1a", "d1a", "d1b"]


def _dev(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else np.asarray(a, dtype=dt))).cuda()


def _case(name):
    z = fx()
    p = name + "_"
    y = z[p + "y"]  # (G, M)
    n = int(z[p + "n"])
    idx = z[p + "idx"] if p + "idx" in z.files else None
    sc = z[p + "scales"] if p + "scales" in z.files else None
    return z, p, y, n, idx, sc


def _solve(name, opts=None, **kw):
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z, p, y, n, idx, sc = _case(name)
    opts = opts or EstimatorOptions(grid_factor=4, backend="semifast")
    yy = y[None, 0] if y.shape[0] == 1 else y[None]
    if idx is None:
        return estimate_batch(yy, opts, **kw)[0]
    return estimate_batch(yy, opts, n=n, observed_indices=idx, scales=sc, **kw)[0]


def _check_traj(r, z, p):
    assert r.status == 0
    assert r.k_hat == int(z[p + "k_hat"])
    stages = np.array([STAGES.index(s) for s in r.trace_stages])
    assert np.array_equal(stages, z[p + "stages"])
    assert np.array_equal(encode_events(r.events), z[p + "events"])
    gt = z[p + "trace"]
    assert np.max(np.abs(np.asarray(r.objective_trace) - gt) / np.abs(gt)) < CALL_TOL
    assert r.iterations == int(z[p + "iterations"])
    assert r.converged == bool(z[p + "converged"])
    assert np.max(wrap_distance(r.theta_hat, z[p + "theta_hat"]), initial=0) < THETA_TOL
    assert rel(r.alpha_hat, z[p + "alpha_hat"]) < AMP_TOL
    assert rel(r.gamma_hat, z[p + "gamma_hat"]) < AMP_TOL
    assert abs(r.beta_hat - float(z[p + "beta_hat"])) / float(z[p + "beta_hat"]) < AMP_TOL


@pytest.mark.parametrize("name", NAMES)
def test_semifast_trajectory_against_reference(name):
    z, p, *_ = _case(name)
    r = _solve(name)
    assert r.algorithms["backend"] == "semifast"
    _check_traj(r, z, p)
    if name == "d1a":
        assert any(ev[0] == "deactivate" for ev in r.events)


@pytest.mark.parametrize("name", ["c1a", "c2a", "i1b", "m1a"])
def test_semifast_dropin_estimate(name):
    """estimate(Observation) with the default backend="auto": semifast below
    N = 512 and for incomplete data (model_core.py:469-470), as the reference."""
    from paper_1705_06073_b200 import EstimatorOptions, Observation, estimate

    z, p, y, n, idx, sc = _case(name)
    obs = Observation.complete(y) if idx is None else Observation.incomplete(y, n, idx, sc)
    r = estimate(obs, EstimatorOptions(grid_factor=4))
    assert r.algorithms["backend"] == "semifast"
    _check_traj(r, z, p)


def test_superfast_rejects_incomplete():
    from paper_1705_06073_b200 import EstimatorOptions, Observation, estimate
    from paper_1705_06073_b200.errors import InvalidPattern

    z, p, y, n, idx, sc = _case("i1a")
    with pytest.raises(InvalidPattern):
        estimate(Observation.incomplete(y, n, idx, sc), EstimatorOptions(backend="superfast"))


def _states(name):
    z = fx()
    return [str(s) for s in z[name + "_states"]]


CALLS = [(nm, st) for nm in NAMES for st in ("truth", "final", "empty", "zgamma")]


@pytest.mark.parametrize("name,state", CALLS)
def test_semifast_bundle_against_reference(name, state):
    from paper_1705_06073_b200 import ops

    if state not in _states(name):
        pytest.skip("state not recorded")
    z, p, y, n, idx, sc = _case(name)
    q = f"{p}call_{state}_"
    th, ga, be = z[q + "thetas"], z[q + "gammas"], float(z[q + "beta"])
    k = th.size
    K = max(k, 1)
    L = z[q + "q_grid"].shape[-1]
    tht = _dev(np.pad(th, (0, K - k))[None, :], np.float64)
    gat = _dev(np.pad(ga, (0, K - k))[None, :], np.float64)
    kc = _dev(np.array([k]), np.int32)
    idx0 = _dev((idx - 1).astype(np.int32)) if idx is not None else None
    sct = _dev(sc.astype(np.complex128)) if sc is not None else None
    out = ops.semifast_bundle(tht, gat, kc, _dev(np.array([be])), _dev(y[None]), n, L, idx0, sct)
    assert int(out["status"].item()) == 0
    dt = float(z[q + "data_term"])
    assert abs(out["data_term"].item() - dt) <= CALL_TOL * abs(dt)
    assert rel(out["e"].cpu().numpy()[0], z[q + "e"]) < CALL_TOL
    assert rel(out["q_grid"].cpu().numpy()[0], z[q + "q_grid"]) < CALL_TOL
    assert rel(out["s_grid"].cpu().numpy()[0], z[q + "s_grid"]) < CALL_TOL
    if k:
        for key in "qru":
            assert rel(out[key].cpu().numpy()[0, :, :k], z[q + "st_" + key]) < CALL_TOL, key
        for key in "stvx":
            assert rel(out[key].cpu().numpy()[0, :k], z[q + "st_" + key]) < CALL_TOL, key


def test_semifast_kcap_rerun(monkeypatch):
    """A first attempt at K capacity 2 (smaller than the cfg2 active sets)
    stops those problems with status 3; estimate_batch re-solves them at
    K_max and returns the reference trajectory."""
    from paper_1705_06073_b200 import EstimatorOptions, estimator

    opts = EstimatorOptions(grid_factor=4, backend="semifast")
    z, p, y, n, idx, sc = _case("c2a")
    s = estimator.BatchSolver(n, 1, opts, k_cap=2)
    s.solve(_dev(y[0][None]))
    assert int(s.host_outputs()["status"][0]) == estimator.STATUS_KCAP
    monkeypatch.setattr(estimator, "SEMIFAST_FIRST_KCAP", 2)
    _check_traj(_solve("c2a", opts), z, p)


def test_semifast_batched_patterns():
    """One batch with a per-problem pattern (B, M) gives, problem by
    problem, the bits of the single-problem solves."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    opts = EstimatorOptions(grid_factor=4, backend="semifast")
    z = fx()
    y1, n1, i1, s1 = z["i1a_y"][0], int(z["i1a_n"]), z["i1a_idx"], z["i1a_scales"]
    rng = np.random.default_rng(5)
    ys, ids, scs = [], [], []
    for b in range(6):
        idx = np.sort(rng.choice(n1, size=i1.size, replace=False)) + 1
        sc = rng.uniform(0.5, 1.5, i1.size) * np.exp(2j * np.pi * rng.random(i1.size))
        full = np.zeros(n1, complex)
        full[i1 - 1] = y1 / s1
        ys.append(sc * (full[idx - 1] + 0.05 * (rng.standard_normal(i1.size) + 1j * rng.standard_normal(i1.size))))
        ids.append(idx)
        scs.append(sc)
    Y, I, S = np.stack(ys), np.stack(ids), np.stack(scs)
    res = estimate_batch(Y, opts, n=n1, observed_indices=I, scales=S)
    for b in range(Y.shape[0]):
        r1 = estimate_batch(Y[b:b + 1], opts, n=n1, observed_indices=I[b], scales=S[b])[0]
        rb = res[b]
        assert rb.status == 0 and r1.status == 0
        assert rb.k_hat == r1.k_hat
        assert np.array_equal(rb.objective_trace, r1.objective_trace)
        assert np.array_equal(rb.theta_hat, r1.theta_hat)


@pytest.mark.parametrize("n,k,m", [(64, 4, 40), (200, 8, 120), (512, 10, 300)])
def test_semifast_incomplete_batch_vs_oracle(n, k, m):
    """Seeded problems with per-problem random patterns and complex scales at
    sizes between the fixtures (N = 512 runs 128-thread CTAs over an
    L = 2048 grid): every CUDA trajectory vs the oracle's semifast
    restatement on the same input."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
    from oracle import superlse_oracle as O
    from test_gpu_parity import check_vs_oracle

    rng = np.random.default_rng([7, n, m])
    Y, I, S = [], [], []
    for b in range(6):
        yf, _ = O.generate_problem(41, 2, b, n=n, k=k)
        idx = np.sort(rng.choice(n, size=m, replace=False)) + 1
        sc = rng.uniform(0.5, 1.5, m) * np.exp(2j * np.pi * rng.random(m))
        Y.append(sc * yf[idx - 1])
        I.append(idx)
        S.append(sc)
    Y, I, S = np.stack(Y), np.stack(I), np.stack(S)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="semifast"), n=n, observed_indices=I, scales=S)
    for b in range(Y.shape[0]):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4, backend="semifast"), n=n, observed_indices=I[b],
                       scales=S[b])
        check_vs_oracle(res[b], o)


def test_semifast_edge_patterns():
    """Edge cases of the observation pattern against the oracle's semifast
    restatement: the minimum M = 2 (first and last sample), an incomplete
    call whose pattern is every sample (== complete semifast), and unit vs
    explicit unit scales."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
    from oracle import superlse_oracle as O

    opts = EstimatorOptions(grid_factor=4, backend="semifast")
    yf, _ = O.generate_problem(13, 1, 0)
    n = yf.size
    # M = 2
    idx = np.array([1, n])
    r = estimate_batch(yf[idx - 1][None], opts, n=n, observed_indices=idx)[0]
    o = O.estimate(yf[idx - 1], O.OracleOptions(grid_factor=4, backend="semifast"), n=n, observed_indices=idx)
    assert r.status == 0 and r.k_hat == o.k_hat
    assert r.trace_stages == o.trace_stages
    # full pattern through the incomplete API == complete data
    full = np.arange(1, n + 1)
    ri = estimate_batch(yf[None], opts, n=n, observed_indices=full, scales=np.ones(n, complex))[0]
    rc = estimate_batch(yf[None], opts)[0]
    assert ri.k_hat == rc.k_hat and ri.trace_stages == rc.trace_stages
    assert rel(ri.objective_trace, rc.objective_trace) < CALL_TOL
    assert np.max(wrap_distance(ri.theta_hat, rc.theta_hat), initial=0) < THETA_TOL


@pytest.mark.parametrize("n", [64, 256, 500])
def test_semifast_complete_gram_closed_form_vs_oracle(n):
    """Complete data takes the closed-form Gram sums (sf_gram_complete);
    the oracle's bundle takes the reference's direct sums (nufft.gram,
    nufft.py:184-210).  Frequencies at separations 0.2/N ... 3/N (the pairs
    below 0.5/N fall back to the direct sums), across the wrap-around point
    and far apart: data term, e, the seven statistics and the grid agree at
    the per-call bar."""
    from oracle import superlse_oracle as O
    from paper_1705_06073_b200 import ops

    rng = np.random.default_rng(n)
    base = np.array([0.11, 0.37, 0.62, 0.9995])
    seps = np.array([0.2, 0.49, 0.51, 1.0, 1.7, 3.0]) / n
    th = np.concatenate([base, 0.2 + np.cumsum(seps), [0.0004, 0.75]])  # 0.9995 / 0.0004: a pair across the wrap
    k = th.size
    ga = rng.uniform(0.5, 2.0, k)
    be = 0.05
    y = sum(np.sqrt(g) * np.exp(2j * np.pi * t * np.arange(n)) for g, t in zip(ga, th))
    y = y + np.sqrt(be / 2) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    L = 4 * (1 << int(np.ceil(np.log2(n))))
    ref = O.SemifastBundle(y[None], n, np.arange(1, n + 1), np.ones(n), th, ga, be)
    st = ref.stats()
    qg, sg = ref.grid(L)
    out = ops.semifast_bundle(_dev(th[None], np.float64), _dev(ga[None], np.float64), _dev(np.array([k]), np.int32),
                              _dev(np.array([be])), _dev(y[None]), n, L, None, None)
    assert int(out["status"].item()) == 0
    assert abs(out["data_term"].item() - ref.data_term) <= CALL_TOL * abs(ref.data_term)
    assert rel(out["q_grid"].cpu().numpy()[0], qg) < CALL_TOL
    assert rel(out["s_grid"].cpu().numpy()[0], sg) < CALL_TOL
    for key in "qru":
        assert rel(out[key].cpu().numpy()[0, :, :k], np.asarray(st[key]).reshape(1, -1)[:, :k]) < CALL_TOL, key
    for key in "stvx":
        assert rel(out[key].cpu().numpy()[0, :k], np.asarray(st[key])[:k]) < CALL_TOL, key
