"""GPU parity at the large shapes, on the deactivation path, and on the
reference suite's known-answer tests -- the holes round 1 left:

* cfg5 (N = 16384, L = 4N) and more cfg4 (N = 4096) problems against
  fixtures written by the REAL reference (tests/golden/make_golden_r2.py):
  whole trajectories (histories identical, stage trace held up to the first
  near tie the oracle records at L = 4N) and per-call bundle quantities;
* problems whose reference run removes components
  (smlr.try_deactivate, smlr.py:203-225; estimator.py:235-242);
* the reference's known-answer tests (pkg/tests/test_toeplitz.py,
  test_model_core.py, test_smlr.py) on the CUDA operators.

Per-call operators are checked DECOUPLED: each is fed the reference's own
inputs (its column, rho, delta, w), so the 1e-9 bar measures the operator,
not the conditioning of C (cond(C) ~ 1e4..1e6 at these shapes amplifies a
1e-12 column difference in C^-1 y).  Large vectors stored decimated in the
fixtures (omega sums, the activation grid) are compared at the stored
indices.
"""

import numpy as np
import pytest

from golden_util import AMP_TOL, CALL_TOL, STAGES, THETA_TOL, encode_events, load, near_ties, rel, wrap_distance
from oracle import superlse_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else np.asarray(a, dtype=dt))).cuda()


def _np(t):
    return t.cpu().numpy()


def check_traj(r, z, p, ties):
    """Identical history vs a golden trajectory (same contract as
    test_gpu_parity._check_traj)."""
    assert r.status == 0
    assert r.k_hat == int(z[p + "k_hat"])
    stages = np.array([STAGES.index(s) for s in r.trace_stages])
    gold = z[p + "stages"]
    same = np.array_equal(stages, gold)
    if not same:
        m = min(stages.size, gold.size)
        diff = np.flatnonzero(stages[:m] != gold[:m])
        first = int(diff[0]) if diff.size else m
        assert ties and first >= min(t[0] for t in ties), (first, ties)
    upto = len(stages) if same else min(t[0] for t in ties)
    tr = np.asarray(r.objective_trace)[:upto]
    gt = z[p + "trace"][:upto]
    return tr, gt, same


def check_estimates(r, z, p):
    assert np.array_equal(encode_events(r.events), z[p + "events"])
    assert r.converged == bool(z[p + "converged"])
    assert np.max(wrap_distance(r.theta_hat, z[p + "theta_hat"]), initial=0) < THETA_TOL
    assert rel(r.alpha_hat[0], z[p + "alpha_hat"]) < AMP_TOL
    assert rel(r.gamma_hat, z[p + "gamma_hat"]) < AMP_TOL
    assert abs(r.beta_hat - float(z[p + "beta_hat"])) / float(z[p + "beta_hat"]) < AMP_TOL


# objective-trace bar per shape: 1e-9 relative (north_star per-call bar)
# except at N = 16384.  There the reference's OWN algorithm switches move the
# trace by more than 1e-9: LD vs Schur by up to 2.7e-9, and
# its default NUFFT statistics vs exact direct sums (steer_method "auto" vs
# "direct", both stored in golden_cfg5.npz) by 5.2e-8 on problem 1 (records
# 23-24, L-BFGS refine steps: the step is accepted on an objective change
# near roundoff).  The bar is ~2x that spread, 1e-7; the events, model
# order and final estimates keep the north-star bars.
TRACE_TOL = {"4x": CALL_TOL, 5: 1e-7, "deact": CALL_TOL}



@pytest.mark.parametrize("cfg", ["4x", 5])
def test_large_trajectories_against_reference(cfg):
    """cfg4 problems 1-2 and cfg5 problems 0-1, batched: identical model
    order and active-set history, estimates within the north-star bars."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load(cfg)
    probs = [int(b) for b in z["problems"]]
    Y = np.stack([z[f"p{b}_y"] for b in probs])
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for i, b in enumerate(probs):
        r = res[i]
        p = f"p{b}_"
        tr, gt, same = check_traj(r, z, p, near_ties(cfg, b))
        assert np.max(np.abs(tr - gt) / np.abs(gt), initial=0) < TRACE_TOL[cfg]
        if same:
            assert r.iterations == int(z[p + "iterations"])
        check_estimates(r, z, p)
        if cfg == 5:
            # the reference run with exact direct sums (steer_method="direct")
            # gives the same history; the GPU matches it too
            trd, gtd, _ = check_traj(r, z, f"p{b}d_", near_ties(cfg, b))
            assert np.max(np.abs(trd - gtd) / np.abs(gtd), initial=0) < TRACE_TOL[cfg]
            check_estimates(r, z, f"p{b}d_")


def test_cfg5_levinson_inside_solver():
    """cfg5 problem 0 with the O(N^2) Schur-Levinson factorisation forced in
    the solver (decomp_method="levinson"): the same reference history as the
    superfast path -- the two factorisations are interchangeable, as the
    reference's own decompose() switch."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load(5)
    res = estimate_batch(z["p0_y"][None, :], EstimatorOptions(grid_factor=4, backend="superfast", decomp_method="levinson"))
    r = res[0]
    assert "levinson" in r.algorithms["decomp"]
    tr, gt, _ = check_traj(r, z, "p0_", near_ties(5, 0))
    assert np.max(np.abs(tr - gt) / np.abs(gt), initial=0) < TRACE_TOL[5]
    check_estimates(r, z, "p0_")


LARGE_CALLS = [("4x", 1, "truth"), ("4x", 1, "final"), ("4x", 2, "truth"), ("4x", 2, "final"),
               (5, 0, "truth"), (5, 0, "final"), (5, 0, "empty"), (5, 1, "final")]


def _golden_vec(z, key, n_full, decim):
    """(values, indices, inf-norm of the FULL golden vector) of a possibly
    decimated golden vector: the relative error is always taken against the
    full vector's inf-norm (north_star "relative" = ||d||/||ref||), which the
    fixture stores beside the decimated values (at the empty state the only
    nonzero omega lag, i = 0, is not on the decimated index set)."""
    if key in z.files:
        v = z[key]
        return v, np.arange(v.size), float(np.max(np.abs(v)))
    v = z[key + "_dec"]
    return v, np.arange(0, n_full, decim)[: v.size], float(z[key + "_max"])


@pytest.mark.parametrize("method", ["levinson", "schur"])
@pytest.mark.parametrize("cfg,b,state", LARGE_CALLS)
def test_large_per_call_against_reference(cfg, b, state, method):
    """Rows 1, 3-9 at N = 4096 / 16384 on the reference's bundle states,
    each operator on the reference's own inputs (see module docstring)."""
    from paper_1705_06073_b200 import ops

    z = load(cfg)
    decim = int(z["decim"])
    p = f"p{b}_call_{state}_"
    y = z[f"p{b}_y"]
    n = y.size
    L = 4 * n
    th, ga, be = z[p + "thetas"], z[p + "gammas"], float(z[p + "beta"])
    k = th.size
    K = max(k, 1)
    tht = _dev(np.pad(th, (0, K - k))[None, :], np.float64)
    gat = _dev(np.pad(ga, (0, K - k))[None, :], np.float64)
    kc = _dev(np.array([k]), np.int32)
    # row 1: the GPU's exactly reduced phases vs the reference's direct sum,
    # whose 2 pi n theta argument rounding is ~1e-11 relative at N = 16384
    c = ops.cov_column(tht, gat, kc, _dev(np.array([be])), n)
    assert rel(_np(c)[0], z[p + "c"]) < CALL_TOL
    # rows 2-4 on the reference column
    rho, delta, logdet, status = ops.toeplitz_factor(_dev(z[p + "c"][None, :]), method=method)
    assert int(status.item()) == 0
    assert rel(_np(rho)[0], z[p + "rho"]) < CALL_TOL
    assert rel(_np(delta)[0], z[p + "delta"]) < CALL_TOL
    ld = float(z[p + "logdet"])
    assert abs(logdet.item() - ld) <= CALL_TOL * max(1.0, abs(ld))
    # row 5-6 on the reference rho / delta
    rho_r = _dev(z[p + "rho"][None, :])
    dl_r = _dev(np.array([z[p + "delta"][-1]]))
    w, quad = ops.gs_apply(rho_r, dl_r, _dev(y[None, :]))
    assert rel(_np(w)[0], z[p + "w"]) < CALL_TOL
    dt = float(z[p + "data_term"])
    assert abs(ld + quad.item() - dt) <= CALL_TOL * abs(dt)
    # row 9 on the reference rho / w
    w_r = _dev(z[p + "w"][None, :])
    qg, sg = ops.grid_eval(rho_r, dl_r, w_r, L)
    for key, got in (("q_grid", _np(qg)[0]), ("s_grid", _np(sg)[0])):
        want, idx, den = _golden_vec(z, p + key, L, decim)
        assert np.max(np.abs(got[idx] - want)) / den < CALL_TOL, key
        assert abs(np.max(np.abs(got)) - den) <= CALL_TOL * den, key
    # row 7
    om = ops.omegas(rho_r, dl_r)
    for kind in "stvx":
        want, idx, den = _golden_vec(z, p + "om_" + kind, 2 * n - 1, decim)
        got = _np(om[kind])[0]
        assert np.max(np.abs(got[idx] - want)) / den < CALL_TOL, kind
        assert abs(np.max(np.abs(got)) - den) <= CALL_TOL * den, kind
    # row 8 (reference stats evaluated with exact direct sums)
    if k:
        st = ops.component_stats(tht, kc, rho_r, dl_r, w_r)
        for key in "qrustvx":
            assert rel(_np(st[key])[0, :k], z[p + "st_" + key]) < CALL_TOL, key


def test_large_chained_factor():
    """Chained rows 1 -> 3/4 at cfg5 (the GPU column into the GPU factor),
    both methods agreeing with the reference's rho/delta at the 1e-9 bar and
    with each other."""
    from paper_1705_06073_b200 import ops

    z = load(5)
    p = "p0_call_final_"
    n = z["p0_y"].size
    th, ga, be = z[p + "thetas"], z[p + "gammas"], float(z[p + "beta"])
    c = ops.cov_column(_dev(th[None, :]), _dev(ga[None, :]), _dev(np.array([th.size]), np.int32),
                       _dev(np.array([be])), n)
    out = {}
    for method in ("levinson", "schur"):
        rho, delta, logdet, status = ops.toeplitz_factor(c, method=method)
        assert int(status.item()) == 0
        assert rel(_np(rho)[0], z[p + "rho"]) < CALL_TOL, method
        assert rel(_np(delta)[0], z[p + "delta"]) < CALL_TOL, method
        out[method] = _np(rho)[0]
    assert rel(out["schur"], out["levinson"]) < 1e-10


# ------------------------------------------------------------ deactivation
def test_deactivation_trajectories_against_reference():
    """Problems whose reference run removes components: the GPU history
    holds the same deactivate events (slots and order), and the whole
    trajectory matches."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load("deact")
    count = int(z["count"])
    for b in range(count):
        assert 2 in z[f"p{b}_events"][:, 0], "fixture problem must deactivate"
    # ragged N across the cases: one batch per problem
    for b in range(count):
        p = f"p{b}_"
        r = estimate_batch(z[p + "y"][None, :], EstimatorOptions(grid_factor=4, backend="superfast"))[0]
        assert any(ev[0] == "deactivate" for ev in r.events)
        tr, gt, same = check_traj(r, z, p, near_ties("deact", b))
        assert np.max(np.abs(tr - gt) / np.abs(gt), initial=0) < TRACE_TOL["deact"]
        check_estimates(r, z, p)


def test_deactivation_margins_before_first_removal():
    """Row 11 at the reference state just before its first removal: the
    margins (smlr.deactivation_margins :174-200) on the reference's
    statistics, and the argmin = the removed component."""
    from paper_1705_06073_b200 import ops

    z = load("deact")
    p = "p0_call_predeact_"
    ga = z[p + "gammas"]
    k = ga.size
    kmax = int(z[p + "kmax"])
    st = {key: z[p + "st_" + key] for key in "qs"}
    kc = _dev(np.array([k]), np.int32)
    marg, idx = ops.deactivation_margins(_dev(st["q"][None, :]), _dev(st["s"][None, :]), _dev(ga[None, :]), kc,
                                         _dev(np.array([float(z[p + "zeta"])])), kmax)
    want = z[p + "margins"]
    got = _np(marg)[0, :k]
    assert rel(got, want) < CALL_TOL
    assert want.min() < 0.0
    i = int(idx.item())
    assert i == int(np.argmin(want))
    # the removed slot is the argmin-th active component (slot order)
    assert int(z[p + "slots"][i]) == int(z[p + "removed"][0])


def test_deactivation_batch_vs_oracle():
    """A batch of near-resolution-limit problems (cfg5 law, N = 128, K = 16)
    with the oracle on each: identical histories, deactivations included."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch
    from test_gpu_parity import check_vs_oracle

    Y = O.generate_batch(99, 5, 24, n=128, k=16)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    n_deact = 0
    for b in range(Y.shape[0]):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
        check_vs_oracle(res[b], o)
        n_deact += sum(1 for ev in o.events if ev[0] == "deactivate")
    assert n_deact >= 1  # problem 7 of this stream deactivates (golden_deact case 0)


# ------------------------------------------------ reference known answers
def _factor(c, method):
    from paper_1705_06073_b200 import ops

    return ops.toeplitz_factor(_dev(np.asarray(c, complex)[None, :]), method=method)


@pytest.mark.parametrize("method", ["levinson", "schur"])
def test_kat_factor_identity_and_2x2(method):
    """test_toeplitz.py:67-79 (LD on [1,0,0,0] and [2,1]) and :102-116 (Schur
    identity / scaled identity)."""
    if method == "levinson":
        rho, delta, _, st = _factor([1.0, 0.0, 0.0, 0.0], method)
        assert int(st.item()) == 0
        assert np.allclose(_np(rho)[0], [0, 0, 0, 1]) and np.allclose(_np(delta)[0], [1, 1, 1, 1])
        rho, delta, _, st = _factor([2.0, 1.0], method)
        assert np.allclose(_np(rho)[0], [-0.5, 1.0]) and np.allclose(_np(delta)[0], [2.0, 1.5])
    rho, delta, _, st = _factor(np.concatenate(([1.0], np.zeros(7))), method)
    e = np.zeros(8)
    e[-1] = 1
    assert np.allclose(_np(rho)[0], e) and np.allclose(_np(delta)[0], np.ones(8))
    beta, n = 2.75, 12
    rho, delta, _, st = _factor(np.concatenate(([beta], np.zeros(n - 1))), method)
    e = np.zeros(n)
    e[-1] = 1
    assert np.allclose(_np(rho)[0], e) and np.allclose(_np(delta)[0], beta * np.ones(n))


def _random_pd_toeplitz(n, rng, cond_floor=0.05):
    """Herglotz construction of test_toeplitz.py:22-29."""
    grid = 4 * n
    spectrum = cond_floor + rng.random(grid)
    c = grid * np.fft.ifft(spectrum)[:n] / grid
    c[0] = c[0].real
    return np.asarray(c)


@pytest.mark.parametrize("n", [2, 3, 9, 31, 64, 65, 100, 128])
def test_kat_schur_matches_levinson(n):
    """test_toeplitz.py:119-126 on the device: both factorisations of a
    random PD Toeplitz (Herglotz) agree within 1e-10, and the inverse they
    generate matches the dense inverse (:82-92, 1e-9)."""
    from scipy.linalg import toeplitz as dense_toeplitz

    rng = np.random.default_rng(500 + n)
    c = _random_pd_toeplitz(n, rng)
    r1, d1, _, s1 = _factor(c, "levinson")
    assert int(s1.item()) == 0
    if n >= 4:
        r2, d2, _, s2 = _factor(c, "schur")
        assert int(s2.item()) == 0
        assert np.max(np.abs(_np(r2) - _np(r1))) < 1e-10
        assert np.max(np.abs(_np(d2) - _np(d1))) < 1e-10 * _np(d1)[0, 0]
    rho, dl = _np(r1)[0], _np(d1)[0, -1]
    e1 = np.zeros(n, complex)
    e1[0] = 1
    t1 = dense_toeplitz(e1, rho[::-1])
    t0 = dense_toeplitz(np.concatenate(([0.0], rho[:-1])), np.zeros(n, complex))
    rec = (t1.conj().T @ t1 - t0 @ t0.conj().T) / dl
    dense_inv = np.linalg.inv(dense_toeplitz(c, np.conj(c)))
    assert np.linalg.norm(rec - dense_inv) / np.linalg.norm(dense_inv) < 1e-9


def test_kat_not_positive_definite():
    """test_toeplitz.py:95-99 and :129-134: an indefinite column returns
    status 1 (NotPositiveDefinite) from BOTH factorisations; a non-positive
    c_0 returns status 2 (HermitianToeplitz validation, :55-57)."""
    _, _, _, st = _factor([1.0, 2.0, 0.0], "levinson")
    assert int(st.item()) == 1
    c = np.zeros(40)
    c[0], c[1] = 1.0, 1.001
    for method in ("levinson", "schur"):
        _, _, _, st = _factor(c, method)
        assert int(st.item()) == 1, method
    # a PD prefix followed by an indefinite tail: the pivot fails deep inside
    # the superfast recursion (a leaf past the first) as well
    rng = np.random.default_rng(9)
    c = _random_pd_toeplitz(600, rng)
    c[300] += 5.0
    for method in ("levinson", "schur"):
        _, _, _, st = _factor(c, method)
        assert int(st.item()) == 1, method
    for method in ("levinson", "schur"):
        _, _, _, st = _factor([-1.0, 0.2, 0.0, 0.0], method)
        assert int(st.item()) == 2, method


@pytest.mark.parametrize("n,where", [(600, 254), (600, 255), (600, 256), (600, 257), (600, 511), (600, 512),
                                      (600, 598), (600, 599), (513, 511), (513, 512), (515, 513), (1030, 1027)])
def test_kat_not_positive_definite_at_leaf_boundaries(n, where):
    """The pivot fails at a chosen step of the superfast recursion: first /
    last pair of a 256-step block leaf, the single odd step that ends a leaf,
    the last step of the whole factorisation.  Both factorisations return
    status 1 (toeplitz.py:129-134), and the same column without the
    perturbation factors with status 0."""
    rng = np.random.default_rng(1000 + where)
    c = _random_pd_toeplitz(n, rng)
    for method in ("levinson", "schur"):
        _, _, _, st = _factor(c, method)
        assert int(st.item()) == 0, method
    bad = c.copy()
    bad[where] += 50.0 * abs(c[0])
    for method in ("levinson", "schur"):
        _, _, _, st = _factor(bad, method)
        assert int(st.item()) == 1, (method, where)


def test_kat_apply_inverse_and_logdet():
    """test_toeplitz.py:150-159 (identity; C^-1 [1,0] = [2/3, -1/3] for
    C = [[2,1],[1,2]]) and :184-190 (log det 0, ln 3, N ln beta)."""
    from paper_1705_06073_b200 import ops

    rho, delta, logdet, _ = _factor([2.0, 1.0], "levinson")
    w, _ = ops.gs_apply(rho, delta[:, -1].contiguous(), _dev(np.array([[1.0 + 0j, 0.0]])))
    assert np.allclose(_np(w)[0], [2.0 / 3.0, -1.0 / 3.0])
    assert np.isclose(logdet.item(), np.log(3.0))
    rng = np.random.default_rng(0)
    x = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    rho, delta, logdet, _ = _factor(np.concatenate(([1.0], np.zeros(5))), "levinson")
    w, _ = ops.gs_apply(rho, delta[:, -1].contiguous(), _dev(x[None, :]))
    assert np.allclose(_np(w)[0], x)
    assert logdet.item() == 0.0
    n, beta = 9, 0.37
    _, _, logdet, _ = _factor(np.concatenate(([beta], np.zeros(n - 1))), "levinson")
    assert np.isclose(logdet.item(), n * np.log(beta))


def test_kat_identity_diagonal_sums():
    """test_toeplitz.py:202-212: for C = I, omega_s(0) = N and omega_t(0) =
    2 pi N (N - 1) / 2, zero elsewhere."""
    from paper_1705_06073_b200 import ops

    n = 6
    rho, delta, _, _ = _factor(np.concatenate(([1.0], np.zeros(n - 1))), "levinson")
    om = ops.omegas(rho, delta[:, -1].contiguous())
    es = np.zeros(2 * n - 1)
    es[n - 1] = n
    et = np.zeros(2 * n - 1)
    et[n - 1] = 2 * np.pi * n * (n - 1) / 2
    assert np.allclose(_np(om["s"])[0], es)
    assert np.allclose(_np(om["t"])[0], et)


def test_kat_sherman_morrison_stats():
    """test_model_core.py:132-143: theta = 0, y = 1, C = beta I + gamma 11^H
    gives q_1 = s_1 = N / (beta + N gamma)."""
    from paper_1705_06073_b200 import ops

    n, beta, gamma = 16, 0.3, 1.7
    th, ga, kc = _dev(np.array([[0.0]])), _dev(np.array([[gamma]])), _dev(np.array([1]), np.int32)
    c = ops.cov_column(th, ga, kc, _dev(np.array([beta])), n)
    rho, delta, _, _ = ops.toeplitz_factor(c)
    dl = delta[:, -1].contiguous()
    w, _ = ops.gs_apply(rho, dl, _dev(np.ones((1, n), complex)))
    st = ops.component_stats(th, kc, rho, dl, w)
    want = n / (beta + n * gamma)
    assert np.isclose(_np(st["q"])[0, 0], want)
    assert np.isclose(_np(st["s"])[0, 0], want)


def test_kat_empty_state_grid():
    """test_model_core.py:174-184: with nothing active, s^G = N / beta and
    q^G = FFT_L(y / beta)."""
    from paper_1705_06073_b200 import ops

    rng = np.random.default_rng(11)
    n, beta, L = 16, 0.4, 64
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    c = np.zeros(n, complex)
    c[0] = beta
    rho, delta, _, _ = _factor(c, "levinson")
    dl = delta[:, -1].contiguous()
    w, _ = ops.gs_apply(rho, dl, _dev(y[None, :]))
    qg, sg = ops.grid_eval(rho, dl, w, L)
    assert np.allclose(_np(sg)[0], n / beta)
    assert np.allclose(_np(qg)[0], np.fft.fft(y / beta, n=L))


def test_kat_activation_on_grid_sinusoid():
    """test_smlr.py:158-180: a clean on-grid sinusoid at index 24 of L = 128
    is the activation argmin (and the estimator recovers it)."""
    from paper_1705_06073_b200 import EstimatorOptions, Observation, estimate, ops

    n, L = 32, 128
    theta_true = 24 / L
    y = 3.0 * np.exp(2j * np.pi * np.arange(n) * theta_true)
    beta, kmax = 0.05, 8
    c = np.zeros(n, complex)
    c[0] = beta
    rho, delta, _, _ = _factor(c, "levinson")
    dl = delta[:, -1].contiguous()
    w, _ = ops.gs_apply(rho, dl, _dev(y[None, :]))
    qg, sg = ops.grid_eval(rho, dl, w, L)
    energy = float(np.sum(np.abs(y) ** 2))
    gbar = energy / (n * 4)  # smlr._gamma_bar fallback (:53-59)
    _, idx = ops.activation_curve(qg, sg, _dev(np.array([gbar])), _dev(np.array([0.2])), kmax)
    assert int(idx.item()) == 24
    r = estimate(Observation.complete(y), EstimatorOptions(grid_factor=4, backend="superfast"))
    assert r.k_hat >= 1
    assert np.min(wrap_distance(r.theta_hat, theta_true)) < 1e-6
