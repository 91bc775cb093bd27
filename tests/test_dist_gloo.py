"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 path: problem
sharding, per-rank solving (the host emulation of the device program stands
in for the GPU here) and the final result gather, compared against solving
the whole batch in one process."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_1705_06073_b200 import dist as D


def test_shard_range_partitions():
    for total in (0, 1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, Y, kmax, q):
    import torch.distributed as dist

    import hostemu_util as H
    from paper_1705_06073_b200.estimator import EstimatorOptions

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = D.shard_range(Y.shape[0], rank, world)
        res = H.estimate_batch(Y[lo:hi], EstimatorOptions(grid_factor=4, backend="superfast"))
        h = {"k_hat": np.array([r.k_hat for r in res]), "status": np.array([r.status for r in res]),
             "iterations": np.array([r.iterations for r in res]),
             "flags": np.array([int(r.converged) for r in res]), "beta": np.array([r.beta_hat for r in res]),
             "zeta": np.array([r.zeta_hat for r in res])}
        for name, attr in (("theta", "theta_hat"), ("gamma", "gamma_hat"), ("slot", "slots")):
            m = np.zeros((len(res), kmax))
            for i, r in enumerate(res):
                m[i, : r.k_hat] = getattr(r, attr)
            h[name] = m
        al = np.zeros((len(res), kmax, 2))
        for i, r in enumerate(res):
            al[i, : r.k_hat, 0] = r.alpha_hat[0].real
            al[i, : r.k_hat, 1] = r.alpha_hat[0].imag
        h["alpha"] = al
        full = D.gather_results(D.pack_results(h, kmax), Y.shape[0])
        if rank == 0:
            q.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_shard_and_gather():
    import hostemu_util as H
    from oracle import superlse_oracle as O
    from paper_1705_06073_b200.estimator import EstimatorOptions

    H.build()
    Y = O.generate_batch(3, 1, 5)  # 5 problems: uneven shards (3 + 2)
    kmax = 16
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, Y, kmax, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = D.unpack_results(full, kmax)
    ref = H.estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    for g, r in zip(got, ref):
        assert g["k_hat"] == r.k_hat
        assert np.array_equal(g["theta_hat"], r.theta_hat)
        assert np.array_equal(g["alpha_hat"], r.alpha_hat)
        assert g["beta_hat"] == r.beta_hat


def _worker_api(rank, world, port, Y, q):
    import torch.distributed as dist

    import hostemu_util as H
    from paper_1705_06073_b200.estimator import EstimatorOptions

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        opts = EstimatorOptions(grid_factor=4, backend="superfast")

        class _Res:  # the BatchResult surface estimate_batch_distributed reads
            def __init__(self, h):
                self.h = h
                self.k_hat = h["k_hat"]

        out = D.estimate_batch_distributed(Y, opts, solve=lambda ys: _Res(H.estimate_batch_raw(ys, opts)))
        q.put((rank, out.shard, out.k_hat, out.theta, out.alpha, out.beta))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_public_distributed_entry():
    """paper_1705_06073_b200.dist.estimate_batch_distributed at world size 2:
    every rank returns the whole batch (problem order) equal to solving it
    in one process."""
    import hostemu_util as H
    from oracle import superlse_oracle as O
    from paper_1705_06073_b200.estimator import EstimatorOptions

    H.build()
    Y = O.generate_batch(5, 1, 7)  # 7 problems: shards of 4 + 3
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_api, args=(r, 2, port, Y, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in range(2)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = H.estimate_batch(Y, EstimatorOptions(grid_factor=4, backend="superfast"))
    assert outs[0][1] == (0, 4) and outs[1][1] == (4, 7)
    for rank, shard, k_hat, theta, alpha, beta in outs:
        for b, r in enumerate(ref):
            assert k_hat[b] == r.k_hat
            assert np.array_equal(theta[b, : r.k_hat], r.theta_hat)
            assert np.array_equal(alpha[b, : r.k_hat], r.alpha_hat[0])
            assert beta[b] == r.beta_hat
