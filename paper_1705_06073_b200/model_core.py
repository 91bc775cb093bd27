"""Domain types of the drop-in boundary.

``Observation`` mirrors the reference's constructor contract
(model_core.py:43-130): y is coerced to complex128 of shape (G, M); complete
data means M == n.  Incomplete patterns are accepted by the type (so callers
can construct them) but the superfast path raises ``InvalidPattern`` for
them, exactly as ``SuperfastEngine`` does (model_core.py:450-453).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch

BACKENDS = ("auto", "superfast", "semifast")
BETA_FLOOR_SCALE = 1e-12  # model_core.py:36


@dataclass
class Observation:
    y: np.ndarray
    n: int
    observed_indices: np.ndarray = None
    scales: np.ndarray = None

    def __post_init__(self):
        y = np.atleast_2d(np.asarray(self.y, dtype=np.complex128))
        if y.ndim != 2:
            raise DimensionMismatch("y must have shape (G, M)")
        self.y = y
        if self.observed_indices is None:
            if y.shape[1] != self.n:
                raise DimensionMismatch(f"complete data needs M == n, got {y.shape[1]} != {self.n}")
            self.scales = None
        else:
            idx = np.asarray(self.observed_indices, dtype=np.int64)
            if idx.ndim != 1 or idx.size != y.shape[1]:
                raise DimensionMismatch("observed_indices must have length M")
            if np.any(np.diff(idx) <= 0):
                raise ValueError("observed_indices must be sorted and unique")
            if idx[0] < 1 or idx[-1] > self.n:
                raise ValueError("observed_indices must lie in 1..n")
            self.observed_indices = idx
            if self.scales is None:
                self.scales = np.ones(idx.size, dtype=np.complex128)
            else:
                self.scales = np.asarray(self.scales, dtype=np.complex128)
                if self.scales.shape != idx.shape:
                    raise DimensionMismatch("scales must have length M")

    @classmethod
    def complete(cls, y):
        y = np.atleast_2d(np.asarray(y, dtype=np.complex128))
        return cls(y=y, n=y.shape[1])

    @classmethod
    def incomplete(cls, y, n, observed_indices, scales=None):
        return cls(y=y, n=n, observed_indices=observed_indices, scales=scales)

    @property
    def is_complete(self):
        return self.observed_indices is None

    @property
    def m(self):
        return self.y.shape[1]

    @property
    def g(self):
        return self.y.shape[0]

    def energy(self):
        return float(np.mean(np.sum(np.abs(self.y) ** 2, axis=1)))

    def beta_floor(self):
        return BETA_FLOOR_SCALE * self.energy() / self.m


def default_grid_size(n, grid_factor=8):
    """model_core.py:224-227."""
    target = max(2 * n, grid_factor * n)
    return 1 << int(np.ceil(np.log2(target)))
