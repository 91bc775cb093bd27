"""CLI: signal-file schema round
trip, exit codes, and (GPU) estimate / benchmark end to end."""

import json
import os

import numpy as np
import pytest

from paper_1705_06073_b200 import cli, simdata as S


def test_generate_roundtrip_exact(tmp_path):
    sig, tru = tmp_path / "s.json", tmp_path / "t.json"
    assert cli.main(["generate", "--n", "96", "--m", "70", "--k", "5", "--snr", "15", "--seed", "4",
                     "--snapshots", "2", "--output", str(sig), "--truth", str(tru)]) == 0
    obs = cli.load_signal(str(sig))
    ref_obs, ref_tr = S.generate(96, 70, 5, 15.0, np.random.default_rng(4), snapshots=2)
    assert np.array_equal(obs.y, ref_obs.y)  # 17 significant digits: exact
    assert np.array_equal(obs.observed_indices, ref_obs.observed_indices)
    assert np.array_equal(obs.scales, ref_obs.scales)
    t = json.loads(tru.read_text())
    assert t["k"] == 5 and np.array_equal(np.array(t["thetas"]), ref_tr.thetas)


def test_generate_pairs_and_complete(tmp_path):
    sig = tmp_path / "p.json"
    assert cli.main(["generate", "--n", "128", "--pairs", "3", "--intra-sep", "1.0", "--seed", "1",
                     "--output", str(sig)]) == 0
    doc = json.loads(sig.read_text())
    assert doc["pattern"] == "complete" and doc["n"] == 128 and len(doc["snapshots"][0]) == 128


def test_input_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"n": 64, "pattern": "complete", "snapshots": [[1, 2]')
    assert cli.main(["estimate", str(bad)]) == 2
    assert cli.main(["estimate", str(tmp_path / "missing.json")]) == 2
    wrong = tmp_path / "wrong.json"
    wrong.write_text(json.dumps({"n": 4, "pattern": "complete", "snapshots": [[[1, 0], [0, 1], [1, 1]]]}))
    assert cli.main(["estimate", str(wrong)]) == 2  # M != n for complete data
    sig = tmp_path / "inc.json"
    cli.main(["generate", "--n", "64", "--m", "40", "--k", "3", "--output", str(sig)])
    assert cli.main(["estimate", str(sig), "--backend", "superfast"]) == 2  # InvalidPattern
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"sweep": "Nope", "points": [1]}))
    assert cli.main(["benchmark", str(cfg), "--output", str(tmp_path / "o.csv")]) == 2


def test_generate_infeasible_exit_2(tmp_path):
    assert cli.main(["generate", "--n", "32", "--k", "20", "--output", str(tmp_path / "x.json")]) == 2


@pytest.mark.gpu
def test_estimate_end_to_end(tmp_path):
    from paper_1705_06073_b200 import EstimatorOptions, estimate

    sig, out = tmp_path / "s.json", tmp_path / "r.json"
    cli.main(["generate", "--n", "128", "--m", "100", "--k", "6", "--snr", "20", "--seed", "3", "--output", str(sig)])
    assert cli.main(["estimate", str(sig), "--output", str(out), "--grid-factor", "4"]) == 0
    r = json.loads(out.read_text())
    direct = estimate(cli.load_signal(str(sig)), EstimatorOptions(grid_factor=4))
    assert r["backend"] == "semifast"
    assert r["k_hat"] == direct.k_hat
    assert np.array_equal(np.array(r["theta_hat"]), direct.theta_hat)
    assert r["trace_stages"] == direct.trace_stages


@pytest.mark.gpu
def test_benchmark_rows_and_determinism(tmp_path):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"sweep": "Snr", "n": 64, "k": 4, "points": [10, 20], "trial_count": 8,
                               "base_seed": 11, "grid_factor": 4}))
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["benchmark", str(cfg), "--output", str(a), "--no-wall"]) == 0
    assert cli.main(["benchmark", str(cfg), "--output", str(b), "--no-wall"]) == 0
    assert a.read_bytes() == b.read_bytes()
    lines = a.read_text().strip().split("\n")
    assert len(lines) == 1 + 16 + 2
    import csv
    rows = list(csv.DictReader(open(a)))
    trials = [r for r in rows if r["trial"] != "mean"]
    aggs = [r for r in rows if r["trial"] == "mean"]
    for p, ag in enumerate(aggs):
        bs = [int(r["bsr"]) for r in trials if int(r["point"]) == p]
        assert float(ag["bsr"]) == np.mean(bs)
