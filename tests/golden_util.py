"""Helpers shared by the parity tests: golden fixture access and the
active-set-history encoding used by tests/golden/make_golden.py."""

import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STAGES = ("init", "beta", "activate", "zeta", "refine", "deactivate")


def load(cfg):
    """golden_cfg{cfg}.npz (cfg may be "4x"), or golden_deact.npz for cfg="deact"."""
    name = "golden_deact.npz" if cfg == "deact" else f"golden_cfg{cfg}.npz"
    return np.load(os.path.join(GOLDEN_DIR, name))


def encode_events(events):
    """(kind, slot, grid_index) rows; kind 0 sweep, 1 activate, 2 deactivate;
    a (-1, -1, -1) row closes each event."""
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


def wrap_distance(x, y):
    d = np.abs(np.asarray(x, float) - np.asarray(y, float)) % 1.0
    return np.minimum(d, 1.0 - d)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.max(np.abs(b)) if b.size else 1.0
    return float(np.max(np.abs(a - b)) / den) if b.size else 0.0


# Acceptance bars from BASELINE.json north_star.
THETA_TOL = 1e-8      # wrap-around distance
AMP_TOL = 1e-6        # amplitudes and noise variance, relative
CALL_TOL = 1e-9       # per-call quantities, relative (inf-norm / inf-norm)
# A decision closer than this to flipping, in units of its roundoff scale
# (1e-12 relative for objective comparisons), is a near tie (make_margins.py).
NEAR_TIE = 1.0


def near_ties(cfg, b):
    """Near-tie decisions of golden trajectory (cfg, b): [[trace_pos, kind, margin], ...]."""
    import json
    with open(os.path.join(GOLDEN_DIR, "margins.json")) as f:
        tag = "deact" if cfg == "deact" else f"cfg{cfg}"
        return json.load(f)[f"{tag}_p{b}"]["near_ties"]
