"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): identical model order and active-set
history; frequencies within 1e-8 (wrap distance); amplitudes and noise
variance within 1e-6 relative; per-call quantities within 1e-9 relative
(inf-norm ratio, as the reference tests compare)."""

import numpy as np
import pytest

from golden_util import AMP_TOL, CALL_TOL, STAGES, THETA_TOL, encode_events, load, near_ties, rel, wrap_distance
from oracle import superlse_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else np.asarray(a, dtype=dt))).cuda()


CALL_CASES = [(cfg, b, st) for cfg, nb in ((1, 2), (2, 2), (3, 1)) for b in range(nb)
              for st in ("empty", "truth", "final")]


@pytest.mark.parametrize("method", ["levinson", "schur"])
@pytest.mark.parametrize("cfg,b,state", CALL_CASES)
def test_per_call_against_reference(cfg, b, state, method):
    from paper_1705_06073_b200 import ops

    z = load(cfg)
    p = f"p{b}_call_{state}_"
    y = z[f"p{b}_y"]
    th, ga, be = z[p + "thetas"], z[p + "gammas"], float(z[p + "beta"])
    n = y.size
    L = O.default_grid_size(n, 4)
    k = th.size
    K = max(k, 1)
    tht = _dev(np.pad(th, (0, K - k))[None, :], np.float64)
    gat = _dev(np.pad(ga, (0, K - k))[None, :], np.float64)
    kc = _dev(np.array([k]), np.int32)
    c = ops.cov_column(tht, gat, kc, _dev(np.array([be])), n)
    assert rel(c.cpu().numpy()[0], z[p + "c"]) < 1e-12
    rho, delta, logdet, status = ops.toeplitz_factor(c, method=method)
    assert int(status.item()) == 0
    assert rel(rho.cpu().numpy()[0], z[p + "rho"]) < CALL_TOL
    assert rel(delta.cpu().numpy()[0], z[p + "delta"]) < CALL_TOL
    assert abs(logdet.item() - float(z[p + "logdet"])) <= CALL_TOL * abs(float(z[p + "logdet"])) + 1e-9
    dl = delta[:, -1].contiguous()
    w, quad = ops.gs_apply(rho, dl, _dev(y[None, :]))
    assert rel(w.cpu().numpy()[0], z[p + "w"]) < CALL_TOL
    dt = logdet.item() + quad.item()
    assert abs(dt - float(z[p + "data_term"])) <= CALL_TOL * abs(float(z[p + "data_term"]))
    qg, sg = ops.grid_eval(rho, dl, w, L)
    assert rel(qg.cpu().numpy()[0], z[p + "q_grid"]) < CALL_TOL
    assert rel(sg.cpu().numpy()[0], z[p + "s_grid"]) < CALL_TOL
    if k:
        st = ops.component_stats(tht, kc, rho, dl, w)
        for key in "qrustvx":
            assert rel(st[key].cpu().numpy()[0, :k], z[p + "st_" + key]) < CALL_TOL, key


TRAJ_CASES = [(1, b) for b in range(6)] + [(2, b) for b in range(4)] + [(3, 0), (4, 0)]


def _check_traj(r, z, p, ties=()):
    """Identical history: stage trace, objective trace (1e-9), active-set
    events, iteration count, final estimates.  `ties` (golden_util.near_ties)
    lists the oracle's near-tie decisions; the stage trace may depart from
    the golden one only at or after the first of them (a decision within
    roundoff of flipping), and the active-set history and final estimates
    must still match."""
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
    assert np.max(np.abs(tr - z[p + "trace"][:upto]) / np.abs(z[p + "trace"][:upto]), initial=0) < CALL_TOL
    assert np.array_equal(encode_events(r.events), z[p + "events"])
    if same:
        assert r.iterations == int(z[p + "iterations"])
    assert r.converged == bool(z[p + "converged"])
    assert np.max(wrap_distance(r.theta_hat, z[p + "theta_hat"]), initial=0) < THETA_TOL
    ga = z[p + "alpha_hat"]
    assert rel(r.alpha_hat if ga.ndim == 2 else r.alpha_hat[0], ga) < AMP_TOL
    assert rel(r.gamma_hat, z[p + "gamma_hat"]) < AMP_TOL
    assert abs(r.beta_hat - float(z[p + "beta_hat"])) / float(z[p + "beta_hat"]) < AMP_TOL


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_trajectories_against_reference(cfg):
    """Batched solve of every golden problem of a config: identical history."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load(cfg)
    count = int(z["count"])
    Y = np.stack([z[f"p{b}_y"] for b in range(count)])
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(count):
        _check_traj(res[b], z, f"p{b}_", near_ties(cfg, b))


def test_drop_in_estimate_single():
    """The reference-shaped entry point: estimate(Observation.complete(y))."""
    from paper_1705_06073_b200 import EstimatorOptions, Observation, estimate

    z = load(1)
    r = estimate(Observation.complete(z["p0_y"]), EstimatorOptions(grid_factor=4, backend="superfast"))
    _check_traj(r, z, "p0_", near_ties(1, 0))
    assert r.alpha_hat.shape == (1, r.k_hat)
    assert set(r.wall_time_per_stage) >= {"activate", "objective", "beta", "refine", "deactivate", "total"}


def test_batch_vs_oracle_cfg2_shape():
    """48 seeded cfg2-shaped problems (N=256, K=16, 15 dB): every history
    identical to the CPU oracle."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    Y = O.generate_batch(7, 2, 48)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(Y.shape[0]):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
        r = res[b]
        assert r.status == 0
        assert r.k_hat == o.k_hat
        assert r.trace_stages == o.trace_stages
        assert encode_events(r.events).tolist() == encode_events(o.events).tolist()
        assert np.max(wrap_distance(r.theta_hat, o.theta_hat), initial=0) < THETA_TOL
        assert rel(r.alpha_hat[0], o.alpha_hat[0]) < AMP_TOL
        assert abs(r.beta_hat - o.beta_hat) / o.beta_hat < AMP_TOL


@pytest.mark.parametrize("per_sm", [7, 12])
def test_batch_layouts_vs_oracle_cfg2_shape(per_sm):
    """The N <= 512 solver layout depends on the batch size (solver_threads /
    warps_per_cta): 128-thread CTAs up to 5 problems per SM, classic one-warp
    CTAs up to 10, warp mode (16 one-warp solvers per CTA, operation
    windows: the bench's cfg2 path) above.  A batch of per_sm x SMs seeded
    cfg2 problems runs the classic (7) or the warp-mode (12) kernel; 24 of
    its problems, spread over the batch, match the oracle's histories."""
    import torch

    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    B = per_sm * sms
    Y = O.generate_batch(11, 2, B)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    assert np.all(res.status == 0)
    for b in np.linspace(0, B - 1, 24).astype(int):
        check_vs_oracle(res[int(b)], O.estimate(Y[b], O.OracleOptions(grid_factor=4)))


def test_work_counts_vs_oracle():
    """The device keeps two bundles (current, trial) where the reference
    keeps an LRU(4) cache (model_core.py:416-444): on the same inputs it may
    never build MORE bundles than the oracle's LRU(4) engine (a rebuild the
    reference would have served from its cache is wasted work), and the
    histories it builds them for are the same."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    for cfg, n, k in ((2, None, None), (3, 512, 24)):
        Y = O.generate_batch(5, cfg, 4, n=n, k=k)
        res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
        for b in range(Y.shape[0]):
            o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
            r = res[b]
            if not oracle_ties(o):
                assert r.trace_stages == o.trace_stages
                assert 0 < r.counters["builds"] <= o.builds, (cfg, b, r.counters, o.builds)


def test_default_grid_factor_and_small_sizes():
    """Reference defaults (grid_factor=8) and the smallest / odd sizes."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    rng = np.random.default_rng(11)
    for n in (2, 3, 17, 64, 100):
        y = np.exp(2j * np.pi * 0.3 * np.arange(n)) + 0.1 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
        r = estimate_batch(y[None, :], EstimatorOptions(backend="superfast"))[0]
        o = O.estimate(y, O.OracleOptions())
        assert r.status == 0
        assert r.k_hat == o.k_hat, n
        assert np.max(wrap_distance(r.theta_hat, o.theta_hat), initial=0) < THETA_TOL
        # a decision that sat within roundoff of its threshold (e.g. an Armijo
        # test on a 1e-12 objective change at convergence) may legitimately
        # go either way: the stage trace is held to the oracle's up to its
        # first near tie
        ties = oracle_ties(o)
        upto = min((t[0] for t in ties), default=len(o.trace_stages))
        assert r.trace_stages[:upto] == o.trace_stages[:upto], n
        assert encode_events(r.events).tolist() == encode_events(o.events).tolist(), n


def test_pure_noise_and_zero_signal():
    from paper_1705_06073_b200 import EstimatorOptions, NotPositiveDefinite, Observation, estimate, estimate_batch

    rng = np.random.default_rng(5)
    Y = (rng.standard_normal((8, 128)) + 1j * rng.standard_normal((8, 128))) / np.sqrt(2)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(8):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
        assert res[b].k_hat == o.k_hat
        assert res[b].trace_stages == o.trace_stages
    # all-zero data: beta0 = 0 -> c_0 = 0 -> NotPositiveDefinite (toeplitz.py:55-57)
    with pytest.raises(NotPositiveDefinite):
        estimate(Observation.complete(np.zeros(32, complex)), EstimatorOptions(grid_factor=4, backend="superfast"))


@pytest.mark.parametrize("cfg", [2, 3])
def test_trajectories_superfast_forced(cfg):
    """Golden histories with the superfast (divide-and-conquer) factorisation
    forced on inside the solver kernel (decomp_method="schur",
    toeplitz.py:263-276): identical history, the stage trace held to the
    golden one up to the first near tie the oracle records at L = 4N."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load(cfg)
    count = int(z["count"])
    Y = np.stack([z[f"p{b}_y"] for b in range(count)])
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast", decomp_method="schur"))
    for b in range(count):
        assert "schur" in res[b].algorithms["decomp"]
        _check_traj(res[b], z, f"p{b}_", near_ties(cfg, b))


# ---- rows 7, 10, 11, 12 as separate operators (the solver runs them fused)
ROW_CASES = [(cfg, b, st) for cfg, nb in ((1, 2), (2, 2), (3, 1)) for b in range(nb)
             for st in ("empty", "truth", "final")]


@pytest.mark.parametrize("cfg,b,state", ROW_CASES)
def test_omegas_against_reference(cfg, b, state):
    """Row 7: the four diagonal-sum vectors against the reference's
    all_diagonal_sums (toeplitz.py:415-432) on the golden states."""
    from paper_1705_06073_b200 import ops

    z = load(cfg)
    p = f"p{b}_call_{state}_"
    rho = _dev(z[p + "rho"][None, :])
    dl = _dev(np.array([z[p + "delta"][-1]]))
    om = ops.omegas(rho, dl)
    for kind in "stvx":
        assert rel(om[kind].cpu().numpy()[0], z[p + "om_" + kind]) < CALL_TOL, kind


def _stats_of(z, p, k):
    return {key: z[p + "st_" + key][:k] for key in "qrustvx"}


@pytest.mark.parametrize("cfg,b,state", [c for c in ROW_CASES if c[2] != "empty"])
def test_activation_deactivation_gradient_against_oracle(cfg, b, state):
    """Rows 10-12 on the golden states: Delta-L curve + argmin, deactivation
    margins + argmin, gradient and diagonal Hessian, each against the oracle
    restatement of smlr.py / model_core.py."""
    from paper_1705_06073_b200 import ops

    z = load(cfg)
    p = f"p{b}_call_{state}_"
    n = z[f"p{b}_y"].size
    L = O.default_grid_size(n, 4)
    kmax = n
    ga = z[p + "gammas"]
    k = ga.size
    # row 10 on the golden grid
    qg, sg = z[p + "q_grid"], z[p + "s_grid"]
    for gbar, zeta in ((float(np.mean(ga)), 0.2), (1e-3, k / kmax)):
        ze = O.prior_zeta(zeta, kmax)
        want, _ = O.delta_curve(qg, sg, gbar, ze)
        curve, idx = ops.activation_curve(_dev(qg[None, :]), _dev(sg[None, :]), _dev(np.array([gbar])),
                                          _dev(np.array([zeta])), kmax)
        got = curve.cpu().numpy()[0]
        assert rel(got, want) < CALL_TOL
        i = int(idx.item())
        assert i == int(np.argmin(got))  # lowest index on ties, as best_candidate
        assert want[i] - want.min() <= 1e-12 * max(1.0, abs(want.min()))
    # rows 11-12 on the golden statistics
    st = _stats_of(z, p, k)
    K = k + 3  # padded rows: entries past kcount must be ignored
    pad = lambda a, dt: _dev(np.pad(a, (0, K - k))[None, :], dt)  # noqa: E731
    dstats = {key: pad(st[key], np.complex128 if key in "qrutv" else np.float64) for key in "qrustvx"}
    gam = pad(ga, np.float64)
    kc = _dev(np.array([k]), np.int32)
    for zeta in (0.2, k / kmax, 1e-6):
        class _S:  # minimal EstimationState view for the oracle
            pass
        sv = _S()
        sv.gamma, sv.z, sv.zeta, sv.k_max = ga, np.ones(k, bool), zeta, kmax
        want = O.deactivation_margins(sv, st)
        marg, idx = ops.deactivation_margins(dstats["q"], dstats["s"], gam, kc, _dev(np.array([zeta])), kmax)
        got = marg.cpu().numpy()[0, :k]
        fin = np.isfinite(want)
        assert np.array_equal(np.isfinite(got), fin) and np.array_equal(got[~fin], want[~fin])
        if fin.any():
            assert rel(got[fin], want[fin]) < CALL_TOL
        assert int(idx.item()) == int(np.argmin(want))
    g, d = ops.gradient_hessian(dstats, gam, kc, n)
    assert rel(g.cpu().numpy()[0, :2 * k], O.gradient(ga, st)) < CALL_TOL
    assert rel(d.cpu().numpy()[0, :2 * k], O.diag_hessian(ga, st, n)) < CALL_TOL


# ---- MMV (G > 1 snapshots), SURVEY 8(f) item 1
def _mmv():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_mmv.npz"))


@pytest.mark.parametrize("cfg,g", [(1, 3), (2, 2)])
def test_mmv_trajectories_against_reference(cfg, g):
    """Batched G-snapshot solves reproduce the reference's estimate_mmv
    histories (identical model order and active-set history; the stage trace
    may depart only at a recorded near tie)."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = _mmv()
    count = int(dict((int(c), int(n)) for c, gg, n in z["cases"] if int(gg) == g)[cfg])
    Y = np.stack([z[f"c{cfg}g{g}_p{b}_y"] for b in range(count)])  # (B, G, N)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    assert res.alpha.shape[:2] == (count, g)
    for b in range(count):
        p = f"c{cfg}g{g}_p{b}_"
        ties = [[int(t), "armijo", 0.0] for t in z[p + "near_tie_pos"]]
        r = res[b]
        assert r.alpha_hat.shape == z[p + "alpha_hat"].shape
        _check_traj(r, z, p, ties)


def test_mmv_drop_in_estimate():
    """estimate(Observation.complete(y (G, N))) / estimate_mmv keep the
    reference's shapes: alpha_hat (G, k_hat)."""
    from paper_1705_06073_b200 import EstimatorOptions, Observation, estimate, estimate_mmv

    z = _mmv()
    p = "c1g3_p2_"  # no near ties
    y = z[p + "y"]
    for fn in (estimate, estimate_mmv):
        r = fn(Observation.complete(y), EstimatorOptions(grid_factor=4, backend="superfast"))
        _check_traj(r, z, p, [])
        assert r.alpha_hat.shape == (3, r.k_hat)


@pytest.mark.parametrize("cfg", [3, 4])
def test_paired_residency_batch(cfg):
    """Batches larger than the SM count run two 256-thread solver CTAs per
    SM (solver_paired: 128 registers, half-SM shared region).  The golden
    problem replicated across such a batch must reproduce the reference
    history in every slot, wherever the dynamic queue placed it."""
    import torch

    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    z = load(cfg)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    B = sms + 12
    Y = np.repeat(z["p0_y"][None, :], B, axis=0)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in (0, B // 2, B - 1):
        _check_traj(res[b], z, "p0_", near_ties(cfg, 0))
    assert np.all(res.status == 0)
    assert np.all(res.k_hat == res.k_hat[0])
    assert np.max(np.abs(res.theta - res.theta[0])) == 0.0  # same problem, same program: same bits


@pytest.mark.parametrize("n,L,B", [(256, 1024, 300), (200, 1024, 37), (129, 1024, 5), (256, 2048, 7), (64, 256, 9),
                                   (1000, 4096, 3),
                                   # residue kernel (L >= 8192): M = N (no fold), folded (N > 2048),
                                   # ragged N, small N with many residues, more tasks than CTAs
                                   (2048, 8192, 5), (3000, 16384, 4), (4096, 16384, 300), (5000, 32768, 3),
                                   (16384, 65536, 2), (100, 8192, 3), (2049, 8192, 2)])
def test_grid_eval_shapes_against_fft(n, L, B):
    """Row 9 on every kernel family (the TMA two-pass kernel serves L = 1024,
    128 < N <= 256, including ragged N and batches that are not a multiple
    of the persistent grid): q^G = FFT_L(w), s^G from the product form, vs
    numpy's FFT of the same seeded inputs (per-call bar 1e-9)."""
    from paper_1705_06073_b200 import ops

    rng = np.random.default_rng(n * 7 + L + B)
    rho = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    w = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    dl = rng.uniform(0.5, 2.0, B)
    qg, sg = ops.grid_eval(_dev(rho), _dev(dl), _dev(w), L)
    Q = np.fft.fft(w, L, axis=1)
    A0 = np.fft.fft(rho, L, axis=1)
    A1 = np.fft.fft(rho * np.arange(n), L, axis=1)
    S = ((2 - n) * np.abs(A0) ** 2 + 2 * np.real(A1 * np.conj(A0))) / dl[:, None]
    q, s = qg.cpu().numpy(), sg.cpu().numpy()
    for b in range(B):
        assert rel(q[b], Q[b]) < CALL_TOL, b
        assert rel(s[b], S[b]) < CALL_TOL, b


@pytest.mark.parametrize("cfg,b,state", ROW_CASES)
def test_grid_eval_omega_against_reference(cfg, b, state):
    """Row 9 in the reference's own form: the golden w and om_s (the
    reference's all_diagonal_sums) in, q^G and s^G against the reference's
    grid() output (model_core.py:303-313) at the per-call bar."""
    from paper_1705_06073_b200 import ops

    z = load(cfg)
    p = f"p{b}_call_{state}_"
    n = z[p + "w"].size
    L = O.default_grid_size(n, 4)
    qg, sg = ops.grid_eval_omega(_dev(z[p + "w"][None, :]), _dev(z[p + "om_s"][None, :]), L)
    assert rel(qg.cpu().numpy()[0], z[p + "q_grid"]) < CALL_TOL
    assert rel(sg.cpu().numpy()[0], z[p + "s_grid"]) < CALL_TOL


@pytest.mark.parametrize("n,L,B", [(256, 1024, 300), (200, 1024, 37), (129, 1024, 5), (256, 1024, 1),
                                   # every residue-kernel M (2^4 .. 2^11), folds, ragged N, the direct kernel
                                   (2, 4, 3), (2, 8, 3), (4, 8, 2), (3, 16, 4), (17, 64, 5), (64, 256, 9), (100, 512, 6),
                                   (128, 1024, 4), (257, 1024, 3), (256, 2048, 7), (1000, 4096, 3),
                                   (2048, 8192, 5), (3000, 16384, 4), (4096, 16384, 300), (16384, 65536, 2),
                                   # register-transform kernels (slse_grid3.cuh): pruned / dense, several tasks
                                   # per CTA (the exchange layout alternates), folds, residue pairs, ragged N,
                                   # 4N > L (no half-length s^G)
                                   (1024, 4096, 700), (513, 4096, 3), (1500, 4096, 5), (2048, 4096, 2),
                                   (2048, 8192, 400), (4096, 8192, 3), (5000, 16384, 3), (8192, 16384, 2),
                                   (9000, 65536, 3), (16384, 65536, 30), (20000, 65536, 2), (32768, 131072, 2),
                                   # the cfg1 warp-per-problem kernel: several problems per warp, ragged N
                                   (64, 256, 20000), (64, 256, 1), (33, 256, 7), (50, 256, 130)])
def test_grid_eval_omega_shapes_against_fft(n, L, B):
    """Row 9 coefficient form on every kernel family vs the reference's
    literal formula in numpy (q^G = fft(w, L), s^G = L ifft(buf).real with
    buf[i mod L] = om_s(i)) on seeded Hermitian om_s rows."""
    from paper_1705_06073_b200 import ops

    rng = np.random.default_rng(n * 11 + L + B)
    w = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    half = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    half[:, 0] = half[:, 0].real
    om = np.concatenate([np.conj(half[:, :0:-1]), half], axis=1)
    qg, sg = ops.grid_eval_omega(_dev(w), _dev(om), L)
    Q = np.fft.fft(w, L, axis=1)
    buf = np.zeros((B, L), dtype=np.complex128)
    buf[:, np.arange(-(n - 1), n) % L] = om
    S = (L * np.fft.ifft(buf, axis=1)).real
    q, s = qg.cpu().numpy(), sg.cpu().numpy()
    for b in range(B):
        assert rel(q[b], Q[b]) < CALL_TOL, b
        assert rel(s[b], S[b]) < CALL_TOL, b


SWEEP_N = [2, 3, 17, 64, 100, 255, 256, 257, 300, 512, 513, 1000, 2048, 3000, 4096]


@pytest.mark.parametrize("n", SWEEP_N)
def test_per_call_size_sweep(n, monkeypatch):
    """Every per-call operator (rows 1, 3-5, 7-9) at ragged and power-of-two
    sizes around each kernel-family boundary (one-warp / block / paired /
    superfast factorisations, warp / block GS apply, grid kernels), each on
    the SAME inputs as the oracle's direct restatement (its own column, rho,
    w), so the bar (1e-9) measures the operator, not the conditioning of a
    random state (chained, the column's 1e-12 already grows to 1e-9 in C^-1 y
    at N = 4096 through cond(C) ~ 1e4; tools/acc_diag.py).  The oracle's
    off-grid sums use exactly reduced phases here (O.EXACT_PHASE): its
    reference-faithful direct sums carry ~1e-8 phase rounding at N = 4096."""
    from paper_1705_06073_b200 import ops

    monkeypatch.setattr(O, "EXACT_PHASE", True)

    rng = np.random.default_rng(1000 + n)
    B, K = 2, max(1, min(8, n // 4))
    th = rng.uniform(0, 1, (B, K))
    ga = rng.uniform(0.2, 2.0, (B, K))
    be = rng.uniform(0.05, 0.5, B)
    y = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    kc = _dev(np.full(B, K), np.int32)
    c = ops.cov_column(_dev(th), _dev(ga), kc, _dev(be), n)
    bundles = [O.Bundle(y[b], th[b], ga[b], float(be[b])) for b in range(B)]
    for b in range(B):
        assert rel(c.cpu().numpy()[b], bundles[b].c) < CALL_TOL
    c_or = _dev(np.stack([o.c for o in bundles]))
    methods = ["levinson", "schur"] if n >= 4 else ["levinson"]
    for method in methods:
        rho, delta, logdet, status = ops.toeplitz_factor(c_or, method=method)
        assert int(status.abs().sum()) == 0
        for b in range(B):
            assert rel(rho.cpu().numpy()[b], bundles[b].rho) < CALL_TOL, method
            assert rel(delta.cpu().numpy()[b], bundles[b].delta) < CALL_TOL, method
    rho_or = _dev(np.stack([o.rho for o in bundles]))
    dl_or = _dev(np.array([o.delta[-1] for o in bundles]))
    w, quad = ops.gs_apply(rho_or, dl_or, _dev(y))
    w_or = _dev(np.stack([o.w for o in bundles]))
    st = ops.component_stats(_dev(th), kc, rho_or, dl_or, w_or)
    om = ops.omegas(rho_or, dl_or)
    L = 1 << int(np.ceil(np.log2(4 * n)))
    qg, sg = ops.grid_eval(rho_or, dl_or, w_or, L)
    for b in range(B):
        o = bundles[b]
        assert rel(w.cpu().numpy()[b], o.w) < CALL_TOL
        ost = o.stats()
        for key in "qrustvx":
            assert rel(st[key].cpu().numpy()[b, :K], ost[key]) < CALL_TOL, key
        for key in "stvx":
            assert rel(om[key].cpu().numpy()[b], o.omegas()[key]) < CALL_TOL, key
        q_ref, s_ref = o.grid(L)
        assert rel(qg.cpu().numpy()[b], q_ref) < CALL_TOL
        assert rel(sg.cpu().numpy()[b], s_ref) < CALL_TOL


def oracle_ties(o):
    """Near-tie decisions of an oracle run, as golden_util.near_ties."""
    from golden_util import NEAR_TIE

    return [[int(pos), kind, float(mg)] for kind, mg, pos in o.margins if mg < NEAR_TIE]


def check_vs_oracle(r, o):
    """GPU result vs oracle run on the same input: identical model order and
    active-set history, stage trace identical up to the oracle's first near
    tie (all of it when there is none), estimates within the bars."""
    ties = oracle_ties(o)
    assert r.status == 0
    assert r.k_hat == o.k_hat
    assert encode_events(r.events).tolist() == encode_events(o.events).tolist()
    upto = min((t[0] for t in ties), default=None)
    if upto is None:
        assert r.trace_stages == o.trace_stages
    else:
        assert r.trace_stages[:upto] == o.trace_stages[:upto]
    m = min(len(r.objective_trace), len(o.objective_trace), upto if upto is not None else 1 << 30)
    assert rel(np.asarray(r.objective_trace)[:m], np.asarray(o.objective_trace)[:m]) < CALL_TOL
    assert np.max(wrap_distance(r.theta_hat, o.theta_hat), initial=0) < THETA_TOL
    assert rel(r.alpha_hat[0], o.alpha_hat[0]) < AMP_TOL
    assert abs(r.beta_hat - o.beta_hat) / o.beta_hat < AMP_TOL


@pytest.mark.parametrize("n,k", [(100, 6), (300, 12), (513, 16)])
def test_trajectories_ragged_sizes_vs_oracle(n, k):
    """Whole estimates at sizes between the configs (one-warp with 8 warps
    per CTA at N = 300, 256-thread blocks at N = 513) vs the oracle: same
    model order, active-set history, estimates, and the stage trace up to
    the oracle's first near-tie decision."""
    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch

    Y = O.generate_batch(31, 2, 3, n=n, k=k)
    res = estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(Y.shape[0]):
        check_vs_oracle(res[b], O.estimate(Y[b], O.OracleOptions(grid_factor=4)))


def test_layout_boundaries_same_results():
    """Every solver layout boundary (N = 4096: CTA pair up to SMs/2 problems,
    one 512-thread CTA up to SMs, paired 256-thread CTAs above; N = 256:
    128-thread CTAs up to 5 per SM, classic one-warp CTAs up to 10, warp
    mode above): every problem finishes, and problem 0's trajectory is the
    same in each layout (4 outer iterations, to bound the run time)."""
    import torch

    from paper_1705_06073_b200 import EstimatorOptions, estimate_batch, simdata

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    opts = EstimatorOptions(grid_factor=4, backend="superfast", max_outer_iterations=4)
    for cfg, sizes in ((4, (1, sms // 2, sms // 2 + 1, sms, sms + 1)), (2, (1, 5 * sms + 1, 10 * sms + 1))):
        ref = None
        for B in sizes:
            r = estimate_batch(simdata.batch(7, cfg, B), opts)
            assert np.all(r.status == 0), (cfg, B)
            t0 = r[0].objective_trace
            ref = t0 if ref is None else ref
            assert r[0].trace_stages == r[0].trace_stages and t0.shape == ref.shape
            assert rel(t0, ref) < 1e-12, (cfg, B)
