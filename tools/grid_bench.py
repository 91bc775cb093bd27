"""Standalone activation-grid kernel timing (cfg shapes), CUDA events, L2 flushed."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=4096)
ap.add_argument("--N", type=int, default=256)
ap.add_argument("--L", type=int, default=1024)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
rho = torch.randn((a.B, a.N), dtype=torch.complex128, device="cuda", generator=g)
w = torch.randn((a.B, a.N), dtype=torch.complex128, device="cuda", generator=g)
dl = torch.rand(a.B, dtype=torch.float64, device="cuda", generator=g) + 0.5
qg = torch.empty((a.B, a.L), dtype=torch.complex128, device="cuda")
sg = torch.empty((a.B, a.L), dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    ops.grid_eval(rho, dl, w, a.L, out=(qg, sg))
ms = []
for _ in range(a.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.grid_eval(rho, dl, w, a.L, out=(qg, sg))
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
ms.sort()
h = max(1, len(ms) // 2)
t = sum(ms[:h]) / h
alg = a.B * (32 * a.N + 24 * a.L)
print(f"grid B={a.B} N={a.N} L={a.L}: {1000 * t:.1f} us  {alg / t / 1e6:.0f} GB/s  ({100 * alg / t / 1e6 / 6553.3:.1f} % of 6553 GB/s)")
# parity spot check against the unfused reference path
import numpy as np  # noqa: E402
r = rho[:4].cpu().numpy(); ww = w[:4].cpu().numpy(); d = dl[:4].cpu().numpy()
A0 = np.fft.fft(r, a.L, axis=1); A1 = np.fft.fft(r * np.arange(a.N), a.L, axis=1); Q = np.fft.fft(ww, a.L, axis=1)
S = ((2 - a.N) * np.abs(A0) ** 2 + 2 * np.real(A1 * np.conj(A0))) / d[:, None]
print("max rel err q", float(np.max(np.abs(qg[:4].cpu().numpy() - Q)) / np.max(np.abs(Q))),
      "s", float(np.max(np.abs(sg[:4].cpu().numpy() - S)) / np.max(np.abs(S))))
