"""Command-line surface: the ``superlse`` console
script the reference declares (pkg/pyproject.toml:18-19)
but does not ship.

  python -m paper_1705_06073_b200.cli estimate SIGNAL.json [--output RESULT.json] [options]
  python -m paper_1705_06073_b200.cli generate --n N --k K --snr DB [--m M] [--snapshots G]
                                            [--pairs P --intra-sep S] [--seed S] --output SIGNAL.json
                                            [--truth TRUTH.json]
  python -m paper_1705_06073_b200.cli benchmark CONFIG.json --output TRIALS.csv [--no-wall]

Signal file: {"n": int, "pattern": "complete" | {"indices":
[int...], "scales": [[re, im]...]}, "snapshots": [[[re, im]...] ...]}, complex
numbers as [re, im] pairs of doubles written with 17 significant digits (so
generate -> estimate round-trips exactly).  Exit codes: 0 success, 2 input
error (unreadable / malformed file, schema, InvalidPattern, dimensions), 3
numerical failure (NotPositiveDefinite).

benchmark runs a seeded Monte-Carlo sweep: per point p and trial t the
scene comes from ``default_rng([base_seed, p, t])`` (the reference
harness's stream contract, simdata.py:12-14) through ``simdata.generate`` /
``generate_pairs``; each point's trials are solved as ONE batch on the GPU
(estimate_batch) and scored with simdata's metrics.  CSV: one row per trial
(sweep, point, value, trial, seed, n, m, k, snr_db, k_hat, nmse, bsr, csr,
wall_ms, iterations) then one aggregate row per point (trial = "mean"; bsr
= the exact mean of the trial booleans).  wall_ms is the point's batch time
divided by its trials; --no-wall writes 0 there so identical configs give
byte-identical files.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
import time

import numpy as np

EXIT_OK, EXIT_INPUT, EXIT_NUMERIC = 0, 2, 3
SWEEPS = ("Snr", "PairSeparation", "SubsamplingRatio", "RuntimeVsN", "RuntimeVsK", "PhaseTransition")


class InputError(Exception):
    """Malformed input (exit code 2)."""


def _c(z):
    return [float(f"{z.real:.17g}"), float(f"{z.imag:.17g}")]


def _dump(obj, path):
    text = json.dumps(obj, indent=None, separators=(",", ":"), allow_nan=True)
    if path in (None, "-"):
        sys.stdout.write(text + "\n")
    else:
        with open(path, "w") as f:
            f.write(text + "\n")


def _fmt17(x):
    return format(float(x), ".17g")


def signal_to_json(obs) -> str:
    """Observation -> the signal-file JSON text (17 significant digits)."""
    def cx(z):
        return "[" + _fmt17(z.real) + "," + _fmt17(z.imag) + "]"

    snaps = "[" + ",".join("[" + ",".join(cx(z) for z in row) + "]" for row in np.atleast_2d(obs.y)) + "]"
    if obs.is_complete:
        pat = '"complete"'
    else:
        pat = ('{"indices":[' + ",".join(str(int(i)) for i in obs.observed_indices) + '],"scales":[' +
               ",".join(cx(z) for z in obs.scales) + "]}")
    return '{"n":' + str(int(obs.n)) + ',"pattern":' + pat + ',"snapshots":' + snaps + "}"


def _complex_rows(a, what):
    try:
        arr = np.asarray(a, dtype=np.float64)
    except (TypeError, ValueError) as e:
        raise InputError(f"{what}: numbers expected ({e})")
    if arr.ndim < 1 or arr.shape[-1] != 2:
        raise InputError(f"{what}: complex values must be [re, im] pairs")
    return arr[..., 0] + 1j * arr[..., 1]


def load_signal(path):
    """Signal file -> Observation; InputError on any schema violation."""
    from .errors import SuperLseError
    from .model_core import Observation

    try:
        with open(path) as f:
            doc = json.load(f)
    except OSError as e:
        raise InputError(f"{path}: cannot read ({e.strerror})")
    except json.JSONDecodeError as e:
        raise InputError(f"{path}:{e.lineno}:{e.colno}: malformed JSON ({e.msg})")
    if not isinstance(doc, dict) or not {"n", "pattern", "snapshots"} <= set(doc):
        raise InputError(f"{path}: expected an object with keys n, pattern, snapshots")
    n = doc["n"]
    if not isinstance(n, int) or n < 2:
        raise InputError(f"{path}: n must be an integer >= 2")
    y = _complex_rows(doc["snapshots"], f"{path}: snapshots")
    if y.ndim != 2:
        raise InputError(f"{path}: snapshots must be a list of rows of [re, im] pairs")
    pat = doc["pattern"]
    try:
        if pat == "complete":
            return Observation(y=y, n=n)
        if not isinstance(pat, dict) or "indices" not in pat:
            raise InputError(f'{path}: pattern must be "complete" or {{"indices", "scales"}}')
        idx = np.asarray(pat["indices"], dtype=np.int64)
        sc = _complex_rows(pat["scales"], f"{path}: scales") if "scales" in pat else None
        return Observation.incomplete(y, n, idx, sc)
    except (ValueError, SuperLseError) as e:
        raise InputError(f"{path}: {e}")


def result_to_dict(res, backend=None):
    """LseResult -> JSON-ready dict (every field of estimator.py:53-66)."""
    alpha = np.atleast_2d(res.alpha_hat)
    out = {
        "k_hat": int(res.k_hat),
        "theta_hat": [float(x) for x in res.theta_hat],
        "alpha_hat": [[_c(z) for z in row] for row in alpha],
        "beta_hat": float(res.beta_hat),
        "gamma_hat": [float(x) for x in res.gamma_hat],
        "zeta_hat": float(res.zeta_hat),
        "objective_trace": [float(x) for x in res.objective_trace],
        "iterations": int(res.iterations),
        "converged": bool(res.converged),
        "trace_stages": list(res.trace_stages),
        "warnings": list(res.warnings),
        "wall_time_per_stage": {k: (list(map(float, v)) if isinstance(v, (list, tuple)) else float(v))
                                for k, v in res.wall_time_per_stage.items()},
    }
    if backend:
        out["backend"] = backend
    return out


def _options(args):
    from .estimator import EstimatorOptions

    kw = {}
    for name in ("backend", "tau", "grid_factor", "seed"):
        v = getattr(args, name, None)
        if v is not None:
            kw[name] = v
    if getattr(args, "max_iters", None) is not None:
        kw["max_outer_iterations"] = args.max_iters
    return EstimatorOptions(**kw)


def cmd_estimate(args) -> int:
    from .errors import DimensionMismatch, InvalidPattern, NotPositiveDefinite
    from .estimator import estimate

    try:
        obs = load_signal(args.input)
        opts = _options(args)
        res = estimate(obs, opts)
    except InputError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    except (InvalidPattern, DimensionMismatch, ValueError) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_INPUT
    except NotPositiveDefinite as e:
        print(f"error: NotPositiveDefinite: {e}", file=sys.stderr)
        return EXIT_NUMERIC
    _dump(result_to_dict(res, res.algorithms.get("backend")), args.output)
    return EXIT_OK


def truth_to_dict(tr):
    return {"k": int(tr.k), "thetas": [float(x) for x in tr.thetas],
            "alphas": [[_c(z) for z in row] for row in np.atleast_2d(tr.alphas)],
            "beta_true": float(tr.beta_true), "snr_db": float(tr.snr_db)}


def cmd_generate(args) -> int:
    from . import simdata as S
    from .errors import InfeasibleSeparation

    rng = np.random.default_rng(args.seed)
    try:
        if args.pairs:
            obs, tr = S.generate_pairs(args.n, args.pairs, args.intra_sep / args.n, args.snr, rng,
                                       snapshots=args.snapshots, m_pattern=args.m)
        else:
            obs, tr = S.generate(args.n, args.m, args.k, args.snr, rng, snapshots=args.snapshots)
    except (ValueError, InfeasibleSeparation) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_INPUT
    text = signal_to_json(obs)
    if args.output in (None, "-"):
        sys.stdout.write(text + "\n")
    else:
        with open(args.output, "w") as f:
            f.write(text + "\n")
    if args.truth:
        _dump(truth_to_dict(tr), args.truth)
    return EXIT_OK


# ------------------------------------------------------------ benchmark
def _points(cfg):
    sweep = cfg["sweep"]
    if sweep not in SWEEPS:
        raise InputError(f"sweep must be one of {SWEEPS}")
    pts = cfg.get("points")
    if not isinstance(pts, list) or not pts:
        raise InputError("points must be a nonempty list")
    return sweep, pts


def _point_params(cfg, sweep, value):
    """(n, m, k, snr, pairs, intra_sep) of one sweep point; the fixed
    parameters default to the figure captions (N = 128, SNR 20 dB, K = 10)."""
    n = int(cfg.get("n", 128))
    m = cfg.get("m")
    k = int(cfg.get("k", 10))
    snr = float(cfg.get("snr_db", 20.0))
    pairs = int(cfg.get("pairs", 0))
    intra = float(cfg.get("intra_sep", 1.0))
    if sweep == "Snr":
        snr = float(value)
    elif sweep == "PairSeparation":
        pairs = pairs or 5
        intra = float(value)
    elif sweep == "SubsamplingRatio":
        m = int(round(float(value) * n))
    elif sweep == "RuntimeVsN":
        n = int(value)
        if m is not None:
            m = int(round(float(cfg.get("m_ratio", m / cfg.get("n", 128))) * n))
    elif sweep == "RuntimeVsK":
        k = int(value)
    elif sweep == "PhaseTransition":
        if not (isinstance(value, list) and len(value) == 2):
            raise InputError("PhaseTransition points are [M/N, K] pairs")
        m, k = int(round(float(value[0]) * n)), int(value[1])
    if m is not None and int(m) >= n:
        m = None
    return n, (None if m is None else int(m)), k, snr, pairs, intra


COLUMNS = ["sweep", "point", "value", "trial", "seed", "n", "m", "k", "snr_db", "k_hat", "nmse", "bsr", "csr",
           "wall_ms", "iterations"]


def run_benchmark(cfg, device=None, no_wall=False):
    """Rows (dicts) of a benchmark config: trials per point solved as one
    GPU batch; scenes from the reference harness's seeded streams."""
    import torch

    from . import simdata as S
    from .estimator import EstimatorOptions, estimate_batch

    sweep, pts = _points(cfg)
    trials = int(cfg.get("trial_count", 100))
    base = int(cfg.get("base_seed", 0))
    ek = {k: cfg[k] for k in ("backend", "tau", "grid_factor", "max_outer_iterations") if k in cfg}
    opts = EstimatorOptions(**ek)
    g = int(cfg.get("snapshots", 1))
    rows, aggs = [], []
    for pi, value in enumerate(pts):
        n, m, k, snr, pairs, intra = _point_params(cfg, sweep, value)
        obs_l, tr_l = [], []
        for t in range(trials):
            rng = np.random.default_rng([base, pi, t])
            if pairs:
                obs, tr = S.generate_pairs(n, pairs, intra / n, snr, rng, snapshots=g, m_pattern=m)
            else:
                obs, tr = S.generate(n, m, k, snr, rng, snapshots=g)
            obs_l.append(obs)
            tr_l.append(tr)
        Y = np.stack([o.y if g > 1 else o.y[0] for o in obs_l])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if m is None:
            res = estimate_batch(Y, opts, device=device)
        else:
            res = estimate_batch(Y, opts, device=device, n=n,
                                 observed_indices=np.stack([o.observed_indices for o in obs_l]))
        wall = 0.0 if no_wall else 1000.0 * (time.perf_counter() - t0) / trials
        pr = []
        for t in range(trials):
            r = res[t]
            row = {"sweep": sweep, "point": pi, "value": json.dumps(value), "trial": t,
                   "seed": f"{base}/{pi}/{t}", "n": n, "m": n if m is None else m, "k": tr_l[t].k, "snr_db": snr,
                   "k_hat": r.k_hat, "nmse": S.nmse(tr_l[t], r, n), "bsr": int(S.bsr_trial(tr_l[t], r, n)),
                   "csr": S.csr(tr_l[t], r, n), "wall_ms": wall, "iterations": r.iterations}
            pr.append(row)
        rows += pr
        agg = dict(pr[0])
        agg.update(trial="mean", seed=f"{base}/{pi}/*", k_hat=float(np.mean([r["k_hat"] for r in pr])),
                   nmse=float(np.mean([r["nmse"] for r in pr])), bsr=float(np.mean([r["bsr"] for r in pr])),
                   csr=float(np.mean([r["csr"] for r in pr])), wall_ms=float(np.median([r["wall_ms"] for r in pr])),
                   iterations=float(np.mean([r["iterations"] for r in pr])))
        aggs.append(agg)
    return rows + aggs


def rows_to_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=COLUMNS, lineterminator="\n")
    w.writeheader()
    for r in rows:
        w.writerow({k: (_fmt17(v) if isinstance(v, float) else v) for k, v in r.items()})
    return buf.getvalue()


def cmd_benchmark(args) -> int:
    try:
        with open(args.config) as f:
            cfg = json.load(f)
        if not isinstance(cfg, dict) or "sweep" not in cfg:
            raise InputError(f"{args.config}: expected an object with a sweep")
        rows = run_benchmark(cfg, no_wall=args.no_wall)
    except OSError as e:
        print(f"error: {args.config}: cannot read ({e.strerror})", file=sys.stderr)
        return EXIT_INPUT
    except json.JSONDecodeError as e:
        print(f"error: {args.config}:{e.lineno}:{e.colno}: malformed JSON ({e.msg})", file=sys.stderr)
        return EXIT_INPUT
    except (InputError, ValueError, TypeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    text = rows_to_csv(rows)
    if args.output in (None, "-"):
        sys.stdout.write(text)
    else:
        with open(args.output, "w") as f:
            f.write(text)
    return EXIT_OK


def parser():
    ap = argparse.ArgumentParser(prog="superlse", description="B200 superfast line spectral estimation")
    sub = ap.add_subparsers(dest="cmd", required=True)
    e = sub.add_parser("estimate", help="estimate one signal file")
    e.add_argument("input")
    e.add_argument("--output", "-o")
    e.add_argument("--backend", choices=("auto", "superfast", "semifast"))
    e.add_argument("--seed", type=int)
    e.add_argument("--tau", type=float)
    e.add_argument("--grid-factor", dest="grid_factor", type=int)
    e.add_argument("--max-iters", dest="max_iters", type=int)
    g = sub.add_parser("generate", help="write a seeded synthetic signal (and its truth)")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--m", type=int)
    g.add_argument("--k", type=int, default=10)
    g.add_argument("--snr", type=float, default=20.0)
    g.add_argument("--snapshots", type=int, default=1)
    g.add_argument("--pairs", type=int, default=0)
    g.add_argument("--intra-sep", dest="intra_sep", type=float, default=1.0, help="pair separation in units of 1/N")
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--output", "-o")
    g.add_argument("--truth")
    b = sub.add_parser("benchmark", help="seeded Monte-Carlo sweep -> CSV")
    b.add_argument("config")
    b.add_argument("--output", "-o")
    b.add_argument("--no-wall", dest="no_wall", action="store_true")
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    return {"estimate": cmd_estimate, "generate": cmd_generate, "benchmark": cmd_benchmark}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
