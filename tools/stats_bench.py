"""Standalone component-statistics kernel timing (rows 8 direct sums)."""
import argparse, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import ops  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=296)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=256)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
rho = torch.randn((a.B, a.N), dtype=torch.complex128, device="cuda", generator=g)
w = torch.randn((a.B, a.N), dtype=torch.complex128, device="cuda", generator=g)
th = torch.rand((a.B, a.K), dtype=torch.float64, device="cuda", generator=g)
kc = torch.full((a.B,), a.K, dtype=torch.int32, device="cuda")
dl = torch.rand(a.B, dtype=torch.float64, device="cuda", generator=g) + 0.5
for _ in range(2):
    ops.component_stats(th, kc, rho, dl, w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ops.component_stats(th, kc, rho, dl, w)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
pairs = a.B * a.K * a.N
print(f"stats B={a.B} N={a.N} K={a.K}: {ms:.3f} ms  {pairs / ms / 1e6:.2f} G(theta,n)/s  "
      f"~{30 * pairs / ms / 1e9:.1f} TF/s at 30 flop/pair")
