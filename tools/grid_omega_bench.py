"""Coefficient-form activation grid (slse_grid_eval_omega) vs the (w, rho)
form (slse_grid_eval): CUDA-event launch times with L2 flushed, GB/s of
algorithmic bytes (16N w + 16N om_s half / rho in, 24L out), a numpy
parity spot check against the reference's literal grid() formula, and a
pure-write / copy bandwidth probe on the same device."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_06073_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="256:1024:43008")  # N:L:B,...
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--probe", action="store_true")
ap.add_argument("--old", action="store_true")
a = ap.parse_args()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timeit(fn, reps):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    return ms[len(ms) // 2], ms[0]


if a.probe:
    buf = torch.empty(2 * 1024 ** 3 // 8, dtype=torch.float64, device="cuda")
    src = torch.empty(1024 ** 3 // 8, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    med, best = timeit(lambda: buf.fill_(1.0), 10)
    print(f"probe fill 2 GiB: {2 * 1024 ** 3 / best / 1e6:.0f} GB/s (best), {2 * 1024 ** 3 / med / 1e6:.0f} (median)")
    med, best = timeit(lambda: dst.copy_(src), 10)
    print(f"probe copy 1 GiB: {2 * 1024 ** 3 / best / 1e6:.0f} GB/s (best), {2 * 1024 ** 3 / med / 1e6:.0f} (median)")
    del buf, src, dst

for spec in a.shapes.split(","):
    N, L, B = (int(x) for x in spec.split(":"))
    g = torch.Generator(device="cuda").manual_seed(1)
    w = torch.randn((B, N), dtype=torch.complex128, device="cuda", generator=g)
    half = torch.randn((B, N), dtype=torch.complex128, device="cuda", generator=g)
    half[:, 0] = half[:, 0].real.to(torch.complex128)
    om = torch.cat([torch.flip(half[:, 1:], dims=[1]).conj(), half], dim=1).contiguous()
    del half
    qg = torch.empty((B, L), dtype=torch.complex128, device="cuda")
    sg = torch.empty((B, L), dtype=torch.float64, device="cuda")
    med, best = timeit(lambda: ops.grid_eval_omega(w, om, L, out=(qg, sg)), a.reps)
    alg = B * (32 * N + 24 * L)
    print(f"omega N={N} L={L} B={B}: median {1000 * med:.1f} us best {1000 * best:.1f} us  "
          f"{alg / med / 1e6:.0f} GB/s ({100 * alg / med / 1e6 / 6555.8:.1f} % of 6555.8)")
    k = min(B, 8)
    ww, oo = w[:k].cpu().numpy(), om[:k].cpu().numpy()
    Q = np.fft.fft(ww, L, axis=1)
    buf = np.zeros((k, L), dtype=np.complex128)
    buf[:, np.arange(-(N - 1), N) % L] = oo
    S = (L * np.fft.ifft(buf, axis=1)).real
    eq = float(np.max(np.abs(qg[:k].cpu().numpy() - Q)) / np.max(np.abs(Q)))
    es = float(np.max(np.abs(sg[:k].cpu().numpy() - S)) / np.max(np.abs(S)))
    last = B - 1
    eq2 = float(np.max(np.abs(qg[last].cpu().numpy() - np.fft.fft(w[last].cpu().numpy(), L))))
    print(f"   parity: rel err q {eq:.2e}  s {es:.2e}  (last problem q abs {eq2:.2e})")
    if a.old:
        rho = torch.randn((B, N), dtype=torch.complex128, device="cuda", generator=g)
        dl = torch.rand(B, dtype=torch.float64, device="cuda", generator=g) + 0.5
        med, best = timeit(lambda: ops.grid_eval(rho, dl, w, L, out=(qg, sg)), a.reps)
        print(f"   rho form: median {1000 * med:.1f} us  {alg / med / 1e6:.0f} GB/s")
        del rho
    del w, om, qg, sg
    torch.cuda.empty_cache()
