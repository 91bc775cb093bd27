import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1705_06073_b200 import ops
def run(n, L, B=3):
    rng = np.random.default_rng(1)
    rho = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    w = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    dl = np.ones(B)
    qg, sg = ops.grid_eval(torch.from_numpy(rho).cuda(), torch.from_numpy(dl).cuda(), torch.from_numpy(w).cuda(), L)
    Q = np.fft.fft(w, L, axis=1); A0 = np.fft.fft(rho, L, axis=1); A1 = np.fft.fft(rho * np.arange(n), L, axis=1)
    S = ((2 - n) * np.abs(A0) ** 2 + 2 * np.real(A1 * np.conj(A0)))
    q, s = qg.cpu().numpy(), sg.cpu().numpy()
    print(n, L, os.environ.get("SLSE_GRID_V2"), "q", np.max(np.abs(q - Q)) / np.max(np.abs(Q)), "s", np.max(np.abs(s - S)) / np.max(np.abs(S)))
for n, L in [(256, 2048), (512, 2048), (128, 2048), (1024, 2048), (129, 2048), (256, 1024), (100, 1024), (64, 1024)]:
    run(n, L)
