"""Multi-GPU sharding of independent problems.

One process per GPU (torch.distributed, NCCL on GPUs, gloo on CPU for the
tests).  Problems are independent, so the data path has no collective:
each rank solves a contiguous slice of the batch; the only communication is
one gather of the per-problem results at the end (and, in bench.py, a MAX
reduction of the elapsed time).
"""

from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int):
    """Contiguous slice [lo, hi) of `total` problems owned by `rank`
    (sizes differ by at most one; earlier ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


# fields gathered per problem (fixed-width, padded to the batch's k_max)
_SCALARS = ("k_hat", "status", "iterations", "flags", "beta", "zeta")
_VECTORS = ("theta", "gamma", "alpha", "slot")


def pack_results(h: dict, kmax: int) -> np.ndarray:
    """Host outputs of one shard -> one float64 matrix (rows = problems):
    6 scalars, then theta, gamma, alpha (re, im), slot, each padded to kmax."""
    B = h["k_hat"].shape[0]
    out = np.zeros((B, 6 + 5 * kmax), dtype=np.float64)
    for i, name in enumerate(_SCALARS):
        out[:, i] = h[name]
    o = 6
    for name in ("theta", "gamma"):
        v = h[name][:, :kmax]
        out[:, o:o + v.shape[1]] = v
        o += kmax
    a = h["alpha"]
    if a.ndim == 4:  # (B, G, K, 2) from BatchSolver.host_outputs
        if a.shape[1] != 1:
            raise NotImplementedError("pack_results gathers single-snapshot results (G = 1)")
        a = a[:, 0]
    a = a[:, :kmax]
    out[:, o:o + a.shape[1]] = a[..., 0]
    o += kmax
    out[:, o:o + a.shape[1]] = a[..., 1]
    o += kmax
    s = h["slot"][:, :kmax]
    out[:, o:o + s.shape[1]] = s
    return out


def unpack_results(m: np.ndarray, kmax: int) -> list:
    """Inverse of pack_results: per-problem dicts (k_hat, theta_hat, gamma_hat,
    alpha_hat, beta_hat, zeta_hat, status, iterations, converged, slots)."""
    res = []
    for row in m:
        k = int(row[0])
        o = 6
        th = row[o:o + k]
        ga = row[o + kmax:o + kmax + k]
        al = row[o + 2 * kmax:o + 2 * kmax + k] + 1j * row[o + 3 * kmax:o + 3 * kmax + k]
        sl = row[o + 4 * kmax:o + 4 * kmax + k].astype(np.int64)
        res.append(dict(k_hat=k, status=int(row[1]), iterations=int(row[2]), converged=bool(int(row[3]) & 1),
                        beta_hat=float(row[4]), zeta_hat=float(row[5]), theta_hat=th.copy(),
                        gamma_hat=ga.copy(), alpha_hat=al.reshape(1, k), slots=sl))
    return res


def gather_results(local: np.ndarray, total: int, group=None) -> np.ndarray:
    """All-gather the packed shards (equal widths) into the full (total, W)
    matrix in problem order.  Uses torch.distributed (NCCL or gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    width = local.shape[1]
    rows = max(shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world))
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros((rows, width), dtype=torch.float64, device=dev)
    lo, hi = shard_range(total, rank, world)
    buf[: hi - lo] = torch.from_numpy(local).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = np.zeros((total, width))
    for r in range(world):
        a, z = shard_range(total, r, world)
        out[a:z] = parts[r][: z - a].cpu().numpy()
    return out
