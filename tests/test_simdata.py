"""simdata: the package's scene generator and metrics
against fixtures written by the REAL reference (tests/golden/make_golden_sim.py),
and the on-device generator / metrics (GPU) against the host ones."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1705_06073_b200 import simdata as S

Z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_sim.npz"))
CASES = [("gen", 64, None, 4, 20.0, 1, 0.0), ("gen", 128, 96, 10, 10.0, 1, 0.0), ("gen", 256, None, 16, 15.0, 2, 0.0),
         ("gen", 128, 64, 6, 0.0, 3, 0.0), ("pairs", 128, None, 5, 20.0, 1, 1.0), ("pairs", 128, 100, 4, 20.0, 1, 1.5)]


def _scene(ci, trial):
    kind, n, m, k, snr, g, intra = CASES[ci]
    rng = np.random.default_rng([2026, ci, trial])
    if kind == "gen":
        return S.generate(n, m, k, snr, rng, snapshots=g)
    return S.generate_pairs(n, k, intra / n, snr, rng, snapshots=g, m_pattern=m)


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_generate_bitwise_against_reference(ci):
    """Same numpy stream -> the reference's scene bit for bit (N < 512: both
    use direct steering sums)."""
    for trial in range(3):
        obs, tr = _scene(ci, trial)
        p = f"c{ci}_t{trial}_"
        assert np.array_equal(obs.y, Z[p + "y"])
        idx = Z[p + "idx"]
        if idx.size:
            assert np.array_equal(obs.observed_indices, idx)
        else:
            assert obs.is_complete
        assert np.array_equal(tr.thetas, Z[p + "thetas"])
        assert np.array_equal(tr.alphas, Z[p + "alphas"])
        assert tr.beta_true == float(Z[p + "beta"])


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_metrics_against_reference(ci):
    n = CASES[ci][1]
    for trial in range(3):
        obs, tr = _scene(ci, trial)
        p = f"c{ci}_t{trial}_"
        for e in range(3):
            th, al = Z[p + f"e{e}_theta"], Z[p + f"e{e}_alpha"]
            res = SimpleNamespace(theta_hat=th, alpha_hat=al, k_hat=th.size)
            assert abs(S.nmse(tr, res, n) - float(Z[p + f"e{e}_nmse"])) <= 1e-12 * float(Z[p + f"e{e}_nmse"])
            assert S.bsr_trial(tr, res, n) == bool(Z[p + f"e{e}_bsr"])
            assert S.csr(tr, res, n) == float(Z[p + f"e{e}_csr"])


def test_generate_infeasible():
    with pytest.raises(S.InfeasibleSeparation):
        S.generate(64, None, 40, 20.0, np.random.default_rng(0))


# ------------------------------------------------------------ device path
torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,k,g,pairs", [(128, None, 10, 1, False), (128, 96, 10, 1, False),
                                           (256, 200, 16, 3, False), (128, None, 10, 1, True)])
def test_device_generator_laws(n, m, k, g, pairs):
    """On-device scenes obey the generator's laws: pattern (first/last,
    sorted, unique), separation, |alpha| >= 0.2 offset law, the SNR
    definition of beta (recomputed from the device truth), noise moments;
    and a trial's scene does not depend on the batch it is drawn in."""
    sc = S.generate_device(n, m, k, 10.0, 64, seed=123, point=4, snapshots=g, pairs=pairs, intra_sep=1.0 / n)
    mm = n if m is None else m
    idx = sc.idx.cpu().numpy()
    th = sc.theta.cpu().numpy()
    al = sc.alpha.cpu().numpy()
    y = sc.y.cpu().numpy()
    be = sc.beta.cpu().numpy()
    noise = []
    for t in range(sc.trials):
        assert idx[t, 0] == 0 and idx[t, -1] == n - 1 and np.all(np.diff(idx[t]) > 0)
        d = S.wrap_distance(th[t][:, None], th[t][None, :]) + 2.0 * np.eye(k)
        if pairs:
            for j in range(0, k, 2):  # a pair's own members are intra_sep apart, the rest > 2/N
                d[j, j + 1] = d[j + 1, j] = 2.0
        assert np.min(d) > 2.0 / n
        assert np.min(np.abs(al[t])) >= 0.2
        clean = (np.exp(2j * np.pi * np.outer(idx[t], th[t])) @ al[t].T).T  # (G, M)
        assert abs(be[t] - np.mean(np.sum(np.abs(clean) ** 2, axis=1)) / (mm * 10.0)) <= 1e-12 * be[t]
        noise.append(((y[t] - clean) / np.sqrt(be[t] / 2.0)).ravel())
    z = np.concatenate(noise)
    assert abs(np.mean(z.real)) < 0.05 and abs(np.var(z.real) - 1.0) < 0.05 and abs(np.var(z.imag) - 1.0) < 0.05
    sub = S.generate_device(n, m, k, 10.0, 5, seed=123, point=4, snapshots=g, pairs=pairs, intra_sep=1.0 / n)
    assert torch.equal(sub.y, sc.y[:5]) and torch.equal(sub.theta, sc.theta[:5])


@pytest.mark.gpu
def test_device_metrics_against_host():
    """metrics_device (NMSE, CSR on the GPU, BSR with the host Hungarian) ==
    the host reference-semantics metrics on the same truth / estimates."""
    sc = S.generate_device(128, 96, 10, 20.0, 16, seed=9)
    T = sc.trials
    rng = np.random.default_rng(3)
    K = 12
    th = np.zeros((T, K))
    al = np.zeros((T, K), complex)
    kh = np.zeros(T, np.int32)
    for t in range(T):
        tr = sc.truth(t)
        kk = [10, 9, 11, 10][t % 4]
        e = (tr.thetas + rng.normal(0, 0.3 / 128, 10)) % 1.0
        a = tr.alphas[0] * (1 + 0.1 * rng.standard_normal(10))
        if kk < 10:
            e, a = e[:kk], a[:kk]
        elif kk > 10:
            e, a = np.append(e, rng.random()), np.append(a, 0.3)
        th[t, :kk], al[t, :kk], kh[t] = e, a, kk
    res = SimpleNamespace(k_hat=kh, theta=th, alpha=al)
    m = S.metrics_device(sc, res)
    for t in range(T):
        tr = sc.truth(t)
        r = SimpleNamespace(theta_hat=th[t, :kh[t]], alpha_hat=al[t, :kh[t]][None], k_hat=int(kh[t]))
        assert abs(m["nmse"][t] - S.nmse(tr, r, 128)) <= 1e-10 * S.nmse(tr, r, 128)
        assert m["csr"][t] == S.csr(tr, r, 128)
        assert m["bsr"][t] == S.bsr_trial(tr, r, 128)


@pytest.mark.gpu
def test_montecarlo_desk_scale():
    """Desk-scale Fig. 2 / Fig. 4 protocol points (SPEC acceptance 5, 7):
    N = 128, K = 10, SNR 20 dB, complete (superfast forced) and M/N = 0.75
    (semifast): BSR >= 0.8, CSR >= 0.95 over 64 device-drawn trials."""
    from paper_1705_06073_b200 import EstimatorOptions

    for m, backend in ((None, "superfast"), (96, "semifast")):
        met, res, sc = S.montecarlo(128, m, 10, 20.0, 64, seed=2026, point=1,
                                    opts=EstimatorOptions(backend=backend))
        assert np.all(res.status == 0)
        assert np.mean(met["bsr"]) >= 0.8, np.mean(met["bsr"])
        assert np.mean(met["csr"]) >= 0.95, np.mean(met["csr"])
