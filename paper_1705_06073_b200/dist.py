"""Multi-GPU sharding of independent problems.

One process per GPU (torch.distributed, NCCL on GPUs, gloo on CPU for the
tests).  Problems are independent, so the data path has no collective:
each rank solves a contiguous slice of the batch; the only communication is
one gather of the per-problem results at the end (and, in bench.py, a MAX
reduction of the elapsed time).

Public entry point: :func:`estimate_batch_distributed` -- every rank passes
the same (B, N) batch (the reference solves one problem per call,
estimator.py:117; this shards a named batch of them), solves its slice on
its own GPU through :func:`estimate_batch`, and receives the whole batch's
results in problem order.
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


class GatheredResult:
    """The whole batch's results after :func:`estimate_batch_distributed`:
    SoA arrays in problem order (k_hat, status, iterations, converged, beta,
    zeta (B,); theta, gamma, slot (B, K); alpha (B, K) complex, zero-padded
    past k_hat) plus per-problem dicts via indexing."""

    def __init__(self, m: np.ndarray, kmax: int, shard: tuple):
        self.kmax = kmax
        self.shard = shard  # this rank's [lo, hi)
        self._m = m
        o = 6
        self.k_hat = m[:, 0].astype(np.int64)
        self.status = m[:, 1].astype(np.int64)
        self.iterations = m[:, 2].astype(np.int64)
        self.converged = (m[:, 3].astype(np.int64) & 1) != 0
        self.beta = m[:, 4].copy()
        self.zeta = m[:, 5].copy()
        self.theta = m[:, o:o + kmax]
        self.gamma = m[:, o + kmax:o + 2 * kmax]
        self.alpha = m[:, o + 2 * kmax:o + 3 * kmax] + 1j * m[:, o + 3 * kmax:o + 4 * kmax]
        self.slot = m[:, o + 4 * kmax:o + 5 * kmax].astype(np.int64)
        self._items = None

    def __len__(self):
        return self._m.shape[0]

    def __getitem__(self, i):
        if self._items is None:
            self._items = unpack_results(self._m, self.kmax)
        return self._items[i]


def estimate_batch_distributed(y, opts=None, group=None, device=None, solve=None) -> GatheredResult:
    """Solve a batch of independent problems on every rank's GPU.

    Every rank of ``group`` calls this with the same ``y`` ((B, N) complex,
    numpy or a CPU torch tensor -- pinned input uploads asynchronously).
    Rank r solves problems ``shard_range(B, r, world)`` with
    :func:`paper_1705_06073_b200.estimate_batch` on ``device`` (default: the
    current CUDA device); the packed per-problem estimates are then
    all-gathered (one NCCL collective on GPUs, gloo on CPU) so every rank
    returns the full batch in problem order.  No collective runs on the
    data path.  ``solve`` replaces the per-rank solver (tests: the host
    emulation of the device program stands in for a GPU under gloo)."""
    import torch
    import torch.distributed as dist

    from .estimator import estimate_batch

    solve = solve or (lambda ys: estimate_batch(ys, opts, device=device))

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = int(y.shape[0])
    lo, hi = shard_range(total, rank, world)
    n = int(y.shape[-1])
    kmax = n if opts is None or getattr(opts, "k_max", None) is None else int(opts.k_max)
    if hi > lo:
        res = solve(y[lo:hi])
        kk = max(1, int(np.max(res.k_hat, initial=0)))
        h = {name: res.h[name] for name in _SCALARS}
        for name in _VECTORS:
            h[name] = res.h[name]
    else:
        kk = 1
        h = None
    # width of the gathered rows: the largest model order over all ranks
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
           else torch.device("cpu"))
    kt = torch.tensor([kk], dtype=torch.int64, device=dev)
    dist.all_reduce(kt, op=dist.ReduceOp.MAX, group=group)
    kk = min(int(kt.item()), kmax)
    if h is None:
        local = np.zeros((0, 6 + 5 * kk))
    else:
        local = pack_results(h, kk)
    return GatheredResult(gather_results(local, total, group), kk, (lo, hi))
