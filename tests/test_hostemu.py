"""The per-problem device program (csrc/slse_solver.cuh), compiled for the
host by g++ as a TEST-ONLY serial emulation (tests/hostemu), reproduces the
reference's golden trajectories and the oracle.  This checks the estimator
state machine's logic on CPU; the GPU tests check the CUDA build itself."""

import numpy as np
import pytest

import hostemu_util as H
from golden_util import AMP_TOL, CALL_TOL, STAGES, THETA_TOL, encode_events, load, rel, wrap_distance
from oracle import superlse_oracle as O
from paper_1705_06073_b200.estimator import EstimatorOptions

CASES = [(1, b) for b in range(6)] + [(2, b) for b in range(4)] + [(3, 0)]


@pytest.mark.parametrize("cfg,b", CASES)
def test_emulated_trajectory_matches_reference(cfg, b):
    z = load(cfg)
    p = f"p{b}_"
    r = H.estimate_batch(z[p + "y"], EstimatorOptions(grid_factor=4, backend="superfast"))[0]
    assert r.status == 0
    assert r.k_hat == int(z[p + "k_hat"])
    assert np.array_equal(np.array([STAGES.index(s) for s in r.trace_stages]), z[p + "stages"])
    assert np.array_equal(encode_events(r.events), z[p + "events"])
    assert r.iterations == int(z[p + "iterations"]) and r.converged == bool(z[p + "converged"])
    assert np.max(wrap_distance(r.theta_hat, z[p + "theta_hat"]), initial=0) < THETA_TOL
    assert rel(r.alpha_hat[0], z[p + "alpha_hat"]) < AMP_TOL
    assert abs(r.beta_hat - float(z[p + "beta_hat"])) / float(z[p + "beta_hat"]) < AMP_TOL
    assert np.allclose(r.objective_trace, z[p + "trace"], rtol=1e-9, atol=0)


CALL_CASES = [(cfg, b, st) for cfg, nb in ((1, 2), (2, 2), (3, 1)) for b in range(nb)
              for st in ("empty", "truth", "final")]


@pytest.mark.parametrize("cfg,b,state", CALL_CASES)
def test_emulated_per_call(cfg, b, state):
    z = load(cfg)
    p = f"p{b}_call_{state}_"
    y = z[f"p{b}_y"]
    L = O.default_grid_size(y.size, 4)
    r = H.bundle(y, z[p + "thetas"], z[p + "gammas"], float(z[p + "beta"]), L)
    assert r["status"] == 0
    assert rel(r["c"], z[p + "c"]) < 1e-12
    for key in ("rho", "w", "q_grid", "s_grid"):
        assert rel(r[key], z[p + key]) < CALL_TOL, key
    assert abs(r["data_term"] - float(z[p + "data_term"])) <= CALL_TOL * abs(float(z[p + "data_term"]))
    if z[p + "thetas"].size:
        for key in "qrustvx":
            assert rel(r[key], z[p + "st_" + key]) < CALL_TOL, key


def test_emulated_small_and_odd_sizes():
    rng = np.random.default_rng(11)
    for n in (2, 3, 17, 64, 100):
        y = np.exp(2j * np.pi * 0.3 * np.arange(n)) + 0.1 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
        r = H.estimate_batch(y[None, :], EstimatorOptions(backend="superfast"))[0]
        o = O.estimate(y, O.OracleOptions())
        assert r.k_hat == o.k_hat and r.trace_stages == o.trace_stages
        assert np.max(wrap_distance(r.theta_hat, o.theta_hat), initial=0) < THETA_TOL


def test_emulated_noise_and_zero():
    rng = np.random.default_rng(5)
    Y = (rng.standard_normal((4, 128)) + 1j * rng.standard_normal((4, 128))) / np.sqrt(2)
    res = H.estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(4):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
        assert res[b].k_hat == o.k_hat and res[b].trace_stages == o.trace_stages
    assert H.estimate_batch(np.zeros((1, 32), complex), EstimatorOptions(grid_factor=4, backend="superfast"))[0].status == 2


def test_emulated_batch_vs_oracle_cfg2_shape():
    Y = O.generate_batch(7, 2, 12)
    res = H.estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for b in range(Y.shape[0]):
        o = O.estimate(Y[b], O.OracleOptions(grid_factor=4))
        assert res[b].k_hat == o.k_hat
        assert res[b].trace_stages == o.trace_stages
        assert encode_events(res[b].events).tolist() == encode_events(o.events).tolist()


@pytest.mark.parametrize("n,L", [(64, 256), (256, 1024), (100, 1024), (1024, 4096), (256, 512), (32, 64),
                                 (17, 128), (512, 4096)])
def test_emulated_pruned_stockham_grid(n, L):
    """The grid kernel's pipeline (head load, pruned radix-16 first pass,
    fixed Stockham schedule over three buffers, product-form combine)
    against the oracle's grid (model_core.py:303-313)."""
    import ctypes

    lib = H.build()
    rng = np.random.default_rng(n + L)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    b = O.Bundle(y, [0.1, 0.4], [1.0, 0.5], 0.3)
    qg = np.zeros(L, complex)
    sg = np.zeros(L)
    lib.emu_grid_pruned.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p]
    q = lib.emu_grid_pruned(b.w.ctypes.data, b.rho.ctypes.data, n, b.delta[-1], L, qg.ctypes.data, sg.ctypes.data)
    assert q >= 0
    q0, s0 = b.grid(L)
    assert rel(qg, q0) < 1e-13 and rel(sg, s0) < 1e-13


@pytest.mark.parametrize("n", [2, 4, 16, 64, 256, 1024, 4096, 8192])
def test_emulated_stockham_fft(n):
    import ctypes

    lib = H.build()
    rng = np.random.default_rng(n)
    for cnt in (1, 3):
        x = rng.standard_normal((cnt, n)) + 1j * rng.standard_normal((cnt, n))
        y = x.copy()
        lib.emu_fft_stockham(ctypes.c_void_p(y.ctypes.data), cnt, n, -1)
        assert rel(y, np.fft.fft(x, axis=1)) < 1e-14
        z = x.copy()
        lib.emu_fft_stockham(ctypes.c_void_p(z.ctypes.data), cnt, n, 1)
        assert rel(z, n * np.fft.ifft(x, axis=1)) < 1e-14


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_emulated_superfast_factor(cfg):
    """Divide-and-conquer (superfast) Schur vs the oracle's Levinson on the
    config-shaped covariance at the true state (toeplitz.py:230-260 role)."""
    import ctypes

    lib = H.build()
    lib.emu_factor_dnc.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    y, tr = O.generate_problem(1, cfg, 0)
    n = y.size
    c = O.cov_column(tr["thetas"], np.abs(tr["alphas"]) ** 2, tr["beta"], n)
    r0, d0 = O.levinson(c)
    rho = np.zeros(n, complex)
    dl = np.zeros(n)
    ld = np.zeros(1)
    assert lib.emu_factor_dnc(c.ctypes.data, n, rho.ctypes.data, dl.ctypes.data, ld.ctypes.data) == 0
    assert rel(rho, r0) < CALL_TOL and rel(dl, d0) < CALL_TOL
    assert abs(ld[0] - np.sum(np.log(d0))) < 1e-9 * max(1.0, abs(np.sum(np.log(d0))))


@pytest.mark.parametrize("cfg,b", [(1, 0), (2, 0), (2, 2), (3, 0)])
def test_emulated_trajectory_superfast(cfg, b):
    """Whole estimator with the superfast factorisation forced on
    (decomp_method="schur", toeplitz.py:263-276)."""
    z = load(cfg)
    p = f"p{b}_"
    r = H.estimate_batch(z[p + "y"], EstimatorOptions(grid_factor=4, backend="superfast", decomp_method="schur"))[0]
    assert r.k_hat == int(z[p + "k_hat"])
    assert np.array_equal(np.array([STAGES.index(s) for s in r.trace_stages]), z[p + "stages"])
    assert np.array_equal(encode_events(r.events), z[p + "events"])
    assert np.max(wrap_distance(r.theta_hat, z[p + "theta_hat"]), initial=0) < THETA_TOL
    assert rel(r.alpha_hat[0], z[p + "alpha_hat"]) < AMP_TOL


@pytest.mark.parametrize("n,count,cap", [(64, 3, 32), (256, 2, 64), (1024, 4, 256), (16384, 2, 8704), (8192, 1, 1024),
                                         (128, 6, 1024)])
def test_emulated_batched_fft(n, count, cap):
    """fft_multi: shared-memory groups and the four-step path for transforms
    larger than the staging capacity."""
    import ctypes

    lib = H.build()
    rng = np.random.default_rng(n + count)
    x = rng.standard_normal((count, n)) + 1j * rng.standard_normal((count, n))
    for sign, ref in ((-1, np.fft.fft(x, axis=1)), (1, n * np.fft.ifft(x, axis=1))):
        y = x.copy()
        lib.emu_fft_multi(ctypes.c_void_p(y.ctypes.data), count, n, sign, cap)
        assert rel(y, ref) < 1e-14
