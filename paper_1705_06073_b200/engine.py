"""Engine-level seam: GPU bundles behind the
reference's duck-typed engine protocol, so the reference's OWN Python outer
loop (estimator.estimate, estimator.py:117-275) can run on the B200
operators.

The protocol (estimator.py:147,161,169,175,199,215,218; model_core.py:416-472):
``engine.bundle(state)`` -> an object with ``data_term``, ``stats()`` ->
(q, r, u (G, K); s, t, v, x (K,)) and ``grid()`` -> (q_grid (G, L), s_grid (L,),
grid_size); ``engine.objective(state)``.  ``GpuEngine`` keeps the
reference's LRU(4) bundle cache keyed on the exact state bytes and builds
every bundle with the C-ABI operators:

* superfast (complete data): ops.cov_column -> ops.toeplitz_factor ->
  ops.gs_apply (build), ops.component_stats, ops.grid_eval;
* semifast (complete or incomplete): ops.semifast_bundle.

One launch per operator and a host copy per decision: this is the
incremental-adoption path; ``estimate`` / ``estimate_batch`` run the whole
loop in one persistent kernel and are what to use for throughput.

    from superlse import estimator
    estimator.make_engine = paper_1705_06073_b200.engine.make_engine
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidPattern, NoActiveComponents, NotPositiveDefinite
from .model_core import default_grid_size

SUPERFAST_MIN_N = 512  # model_core.py:469-470


@dataclass
class ComponentStats:
    """model_core.ComponentStats (:193-209): q, r, u (G, K); s, t, v, x (K,)."""
    q: np.ndarray
    r: np.ndarray
    u: np.ndarray
    s: np.ndarray
    t: np.ndarray
    v: np.ndarray
    x: np.ndarray


@dataclass
class GridStats:
    """model_core.GridStats (:211-216)."""
    q_grid: np.ndarray
    s_grid: np.ndarray
    grid_size: int


def _prior_term(k_hat, zeta, k_max):
    """model_core.prior_term (:230-239)."""
    ze = float(min(max(zeta, 0.5 / k_max), 0.5))
    return -(k_hat * np.log(ze) + (k_max - k_hat) * np.log1p(-ze))


class _GpuSuperfastBundle:
    def __init__(self, eng, thetas, gammas, beta):
        import torch

        from . import ops

        self.eng = eng
        self.thetas = np.asarray(thetas, dtype=np.float64)
        self.k = self.thetas.size
        dev = eng.device
        K = max(self.k, 1)
        self._th = torch.zeros((1, K), dtype=torch.float64, device=dev)
        ga = torch.zeros((1, K), dtype=torch.float64, device=dev)
        if self.k:
            self._th[0, :self.k] = torch.from_numpy(self.thetas)
            ga[0, :self.k] = torch.from_numpy(np.asarray(gammas, dtype=np.float64))
        self._kc = torch.tensor([self.k], dtype=torch.int32, device=dev)
        c = ops.cov_column(self._th, ga, self._kc, torch.tensor([float(beta)], dtype=torch.float64, device=dev),
                           eng.n)
        rho, delta, logdet, status = ops.toeplitz_factor(c)
        if int(status.item()) != 0:
            raise NotPositiveDefinite("covariance is not positive definite")
        self._rho = rho
        self._dl = delta_last = delta[:, -1].contiguous()
        self._w = []
        quad = 0.0
        for g in range(eng.g):
            w, q = ops.gs_apply(rho, delta_last, eng.y_dev[g:g + 1])
            self._w.append(w)
            quad += float(q.item())
        self.data_term = eng.g * float(logdet.item()) + quad  # model_core.py:268-270
        self._stats = None
        self._grid = None

    def stats(self):
        from . import ops

        if self._stats is None:
            if self.k == 0:
                raise NoActiveComponents("component statistics need an active component")
            qs, rs, us = [], [], []
            for w in self._w:
                st = ops.component_stats(self._th, self._kc, self._rho, self._dl, w)
                qs.append(st["q"][0, :self.k].cpu().numpy())
                rs.append(st["r"][0, :self.k].cpu().numpy())
                us.append(st["u"][0, :self.k].cpu().numpy())
            h = {k: st[k][0, :self.k].cpu().numpy() for k in "stvx"}
            self._stats = ComponentStats(q=np.stack(qs), r=np.stack(rs), u=np.stack(us), **h)
        return self._stats

    def grid(self):
        from . import ops

        if self._grid is None:
            L = self.eng.grid_size
            qg, sg = [], None
            for w in self._w:
                q, s = ops.grid_eval(self._rho, self._dl, w, L)
                qg.append(q[0].cpu().numpy())
                sg = s[0].cpu().numpy()
            self._grid = GridStats(q_grid=np.stack(qg), s_grid=sg, grid_size=L)
        return self._grid


class _GpuSemifastBundle:
    def __init__(self, eng, thetas, gammas, beta):
        import torch

        from . import ops

        self.thetas = np.asarray(thetas, dtype=np.float64)
        self.k = self.thetas.size
        dev = eng.device
        K = max(self.k, 1)
        th = torch.zeros((1, K), dtype=torch.float64, device=dev)
        ga = torch.zeros((1, K), dtype=torch.float64, device=dev)
        if self.k:
            th[0, :self.k] = torch.from_numpy(self.thetas)
            ga[0, :self.k] = torch.from_numpy(np.asarray(gammas, dtype=np.float64))
        kc = torch.tensor([self.k], dtype=torch.int32, device=dev)
        be = torch.tensor([float(beta)], dtype=torch.float64, device=dev)
        out = ops.semifast_bundle(th, ga, kc, be, eng.y_dev[None], eng.n, eng.grid_size, eng.idx_dev, eng.sc_dev)
        st = int(out["status"].item())
        if st != 0:
            raise NotPositiveDefinite("Sigma^{-1} is not positive definite")
        self.data_term = float(out["data_term"].item())
        self._out = out
        self._stats = None
        self._grid = None
        self.grid_size = eng.grid_size

    def stats(self):
        if self._stats is None:
            if self.k == 0:
                raise NoActiveComponents("component statistics need an active component")
            o = {k: v[0].cpu().numpy() for k, v in self._out.items() if k in "qrustvx"}
            k = self.k
            self._stats = ComponentStats(q=o["q"][:, :k], r=o["r"][:, :k], u=o["u"][:, :k], s=o["s"][:k],
                                         t=o["t"][:k], v=o["v"][:k], x=o["x"][:k])
        return self._stats

    def grid(self):
        if self._grid is None:
            self._grid = GridStats(q_grid=self._out["q_grid"][0].cpu().numpy(),
                                   s_grid=self._out["s_grid"][0].cpu().numpy(), grid_size=self.grid_size)
        return self._grid


class GpuEngine:
    """_Engine surface (model_core.py:416-444) with GPU bundles."""

    _CACHE = 4

    def __init__(self, obs, backend="superfast", grid_size=None, device=None):
        import torch

        self.obs = obs
        self.backend = backend
        self.n = obs.n
        self.g = obs.g
        self.grid_size = grid_size or default_grid_size(obs.n)
        self.device = torch.device(device) if device is not None else torch.device("cuda",
                                                                                   torch.cuda.current_device())
        y = np.ascontiguousarray(np.atleast_2d(obs.y), dtype=np.complex128)
        self.y_dev = torch.from_numpy(y).to(self.device)
        self.idx_dev = self.sc_dev = None
        if not obs.is_complete:
            if backend == "superfast":
                raise InvalidPattern("superfast backend requires the complete observation pattern")
            self.idx_dev = torch.from_numpy((np.asarray(obs.observed_indices) - 1).astype(np.int32)).to(self.device)
            self.sc_dev = torch.from_numpy(np.ascontiguousarray(obs.scales, dtype=np.complex128)).to(self.device)
        self._bundles = {}
        self._order = []

    def bundle(self, state):
        th = state.active_theta
        ga = state.active_gamma
        key = (th.tobytes(), ga.tobytes(), float(state.beta))
        hit = self._bundles.get(key)
        if hit is not None:
            return hit
        cls = _GpuSuperfastBundle if self.backend == "superfast" else _GpuSemifastBundle
        b = cls(self, th, ga, float(state.beta))
        self._bundles[key] = b
        self._order.append(key)
        if len(self._order) > self._CACHE:
            self._bundles.pop(self._order.pop(0), None)
        return b

    def objective(self, state):
        return self.bundle(state).data_term + _prior_term(state.k_hat, state.zeta, state.k_max)


def make_engine(obs, backend="auto", grid_size=None, decomp_method="auto", steer_method="auto"):
    """model_core.make_engine (:463-472) returning GPU engines."""
    if backend not in ("auto", "superfast", "semifast"):
        raise ValueError("backend must be one of ('auto', 'superfast', 'semifast')")
    if backend == "auto":
        backend = "superfast" if (obs.is_complete and obs.n >= SUPERFAST_MIN_N) else "semifast"
    return GpuEngine(obs, backend=backend, grid_size=grid_size)
