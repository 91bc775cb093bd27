"""Time the standalone Toeplitz factorisations (Schur-Levinson vs superfast)."""
import argparse, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import ops, simdata  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=148)
ap.add_argument("--methods", default="levinson,schur")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = {64: 1, 256: 2, 1024: 3, 4096: 4, 16384: 5}[a.n]
_, tr = simdata.problem(1, cfg, 0)
n = a.n
th = torch.tensor(tr["thetas"], dtype=torch.float64).cuda()[None, :].repeat(a.batch, 1).contiguous()
ga = torch.tensor(np.abs(tr["alphas"]) ** 2, dtype=torch.float64).cuda()[None, :].repeat(a.batch, 1).contiguous()
kc = torch.full((a.batch,), th.shape[1], dtype=torch.int32).cuda()
be = torch.full((a.batch,), tr["beta"], dtype=torch.float64).cuda()
c = ops.cov_column(th, ga, kc, be, n)
ref = None
for m in a.methods.split(","):
    ms = []
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rho, delta, logdet, st = ops.toeplitz_factor(c, method=m)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ms.append(e0.elapsed_time(e1))
    r0 = rho[0].cpu().numpy()
    if ref is None:
        ref = r0
    print(m, "ms per batch", [round(x, 3) for x in ms], "per problem-build us", round(1000 * np.mean(ms), 1),
          "status", int(st.abs().sum()), "rel diff vs first", float(np.max(np.abs(r0 - ref)) / np.max(np.abs(ref))))
