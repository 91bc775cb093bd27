"""Problems/s to convergence for every BASELINE config (one GPU), next to
the CPU oracle port on this host's cores (one problem per core, one round).

Usage: python tools/bench_configs.py [--configs 1,2,3,4,5] [--no-cpu] [--cpu-configs 1,2,3]
Prints one JSON line per config.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402  (cpu worker + seeds)


def gpu_rate(cfg, steps=2):
    import torch

    from paper_1705_06073_b200 import EstimatorOptions, simdata
    from paper_1705_06073_b200.estimator import BatchSolver

    B, n = simdata.CONFIGS[cfg][0], simdata.CONFIGS[cfg][1]
    Y = torch.from_numpy(simdata.batch(bench.SEED, cfg, B)).cuda()
    s = BatchSolver(n, B, EstimatorOptions(grid_factor=4, backend="superfast"))
    s.solve(Y)
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.solve(Y)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    h = s.host_outputs()
    return dict(batch=B, N=n, ms=float(np.mean(ms)), value=B / (np.mean(ms) / 1000.0),
                k_hat_mean=float(h["k_hat"].mean()), status_nonzero=int(np.count_nonzero(h["status"])),
                builds_per_problem=float(h["counters"][:, 0].mean()))


def cpu_rate(cfg):
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t = time.perf_counter()
        out = pool.map(bench._cpu_worker, [(bench.SEED, cfg, i) for i in range(cores)], chunksize=1)
        wall = time.perf_counter() - t
    return dict(value=cores / wall, cores=cores, mean_s=float(np.mean([o[0] for o in out])),
                sample=f"{cores} problems, one per core")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--cpu-configs", default="1,2,3")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    cpu_cfgs = {int(c) for c in a.cpu_configs.split(",") if c}
    for cfg in [int(c) for c in a.configs.split(",")]:
        line = {"config": f"cfg{cfg}", "gpu": gpu_rate(cfg)}
        if not a.no_cpu and cfg in cpu_cfgs:
            line["cpu_port"] = cpu_rate(cfg)
            line["speedup_vs_cpu"] = line["gpu"]["value"] / line["cpu_port"]["value"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
