"""Accuracy of the per-call chain at large N vs the oracle (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import superlse_oracle as O  # noqa: E402
from paper_1705_06073_b200 import ops  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


d = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a if dt is None else np.asarray(a, dt))).cuda()
for n in (1000, 2048, 3000, 4096):
    rng = np.random.default_rng(1000 + n)
    B, K = 2, max(1, min(8, n // 4))
    th = rng.uniform(0, 1, (B, K)); ga = rng.uniform(0.2, 2.0, (B, K)); be = rng.uniform(0.05, 0.5, B)
    y = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    kc = d(np.full(B, K), np.int32)
    c = ops.cov_column(d(th), d(ga), kc, d(be), n)
    o = O.Bundle(y[0], th[0], ga[0], float(be[0]))
    # oracle rho into the GPU GS apply, and GPU rho into the oracle GS apply
    for m in ("levinson", "schur"):
        rho, delta, logdet, st = ops.toeplitz_factor(c, method=m)
        dl = delta[:, -1].contiguous()
        w, _ = ops.gs_apply(rho, dl, d(y))
        w_or, _ = ops.gs_apply(d(np.stack([o.rho, o.rho])), d(np.array([o.delta[-1]] * 2)), d(y))
        w_cpu_from_gpu_rho = O.gs_apply(rho.cpu().numpy()[0], float(dl.cpu().numpy()[0]), y[0])
        print(n, m, "c", rel(c.cpu().numpy()[0], o.c), "rho", rel(rho.cpu().numpy()[0], o.rho),
              "w", rel(w.cpu().numpy()[0], o.w), "w(gpu apply, oracle rho)", rel(w_or.cpu().numpy()[0], o.w),
              "w(oracle apply, gpu rho)", rel(w_cpu_from_gpu_rho, o.w))
