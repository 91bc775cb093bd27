"""Drop-in estimator boundary: ``estimate(obs, opts) -> LseResult``.

Same signature, options and result type as the reference
(estimator.py:34-66, 117-283).  The whole outer loop runs on the GPU: one
CTA per problem executes the estimator state machine (csrc/slse_solver.cuh)
and this module only packs inputs, launches ``slse_estimate_batch`` through
the C ABI and unpacks results.  ``estimate_batch`` is the batched entry
point (one problem per row).

Backends (model_core.make_engine :466-472): "superfast" (complete data,
Toeplitz / Gohberg-Semencul bundles, the north-star path) and "semifast"
(Woodbury bundles with a K x K Cholesky; complete or incomplete data,
``Observation.incomplete``); "auto" picks superfast for complete data with
N >= 512 and semifast otherwise, exactly as the reference.  Both run the
whole loop on the device (csrc/slse_solver.cuh; semifast bundles in
csrc/slse_semifast.cuh).  G >= 1 snapshots (MMV) on both.
"""

from __future__ import annotations

import ctypes
import dataclasses
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DimensionMismatch, InvalidPattern, NotPositiveDefinite, SuperLseError
from .model_core import BACKENDS, Observation, default_grid_size

DEFAULT_TAU = 5.0  # smlr.py:28
STAGE_NAMES = ("init", "beta", "activate", "zeta", "refine", "deactivate")
TIMER_NAMES = ("activate", "objective", "beta", "refine", "deactivate", "total")
FLAG_CONVERGED, FLAG_KMAX_CAP, FLAG_TRACE_FULL, FLAG_EVENTS_FULL = 1, 2, 4, 8
STATUS_OK, STATUS_NOT_PD, STATUS_BAD_DIAGONAL, STATUS_KCAP = 0, 1, 2, 3
SUPERFAST_MIN_N = 512  # model_core.py:469-470 ("auto": superfast for complete data from N = 512)
# First-attempt K capacity of semifast solves (0: the library default,
# min(K_max, 64)); problems whose active set outgrows it are re-solved at K_max.
SEMIFAST_FIRST_KCAP = 0
DECOMP_METHODS = {"auto": 0, "levinson": 1, "schur": 2}  # slse_options.decomp_method
STEER_METHODS = ("auto", "direct", "nufft")


@dataclass
class EstimatorOptions:
    """Knobs of the outer loop (estimator.py:34-50)."""

    grid_factor: int = 8
    tau: float = DEFAULT_TAU
    max_outer_iterations: int = 200
    convergence_tol_scale: float = 1e-7
    lbfgs_inner_max: int = 5
    newton_decrement_tol_scale: float = 1e-8
    backend: str = "auto"
    seed: int = None
    initial_sweep_iterations: int = 3
    lbfgs_memory: int = 10
    k_max: int = None
    decomp_method: str = "auto"
    steer_method: str = "auto"


@dataclass
class LseResult:
    """estimator.py:53-66, plus the active-set history (``events``) and
    per-problem counters the GPU path records."""

    k_hat: int
    theta_hat: np.ndarray
    alpha_hat: np.ndarray
    beta_hat: float
    gamma_hat: np.ndarray
    zeta_hat: float
    objective_trace: np.ndarray
    iterations: int
    wall_time_per_stage: dict
    converged: bool = True
    trace_stages: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    events: list = field(default_factory=list)
    trace_k: np.ndarray = None
    slots: np.ndarray = None
    counters: dict = field(default_factory=dict)
    status: int = STATUS_OK
    algorithms: dict = field(default_factory=dict)


def resolve_backend(opts: EstimatorOptions, n: int, complete: bool = True) -> str:
    """make_engine's choice (model_core.py:463-472)."""
    if opts.backend not in BACKENDS:
        raise ValueError(f"backend must be one of {BACKENDS}")
    b = opts.backend
    if b == "auto":
        b = "superfast" if (complete and n >= SUPERFAST_MIN_N) else "semifast"
    if b == "superfast" and not complete:
        raise InvalidPattern("superfast backend requires the complete observation pattern")
    return b


def _validate(opts: EstimatorOptions):
    if opts.backend not in BACKENDS:
        raise ValueError(f"backend must be one of {BACKENDS}")
    if opts.decomp_method not in DECOMP_METHODS:  # toeplitz.py:263-276
        raise ValueError(f"unknown decomposition method {opts.decomp_method!r}")
    if opts.steer_method not in STEER_METHODS:  # nufft.py:118-123
        raise ValueError(f"unknown method {opts.steer_method!r}")
    if not 1 <= opts.lbfgs_memory <= 16:
        raise ValueError("lbfgs_memory must lie in 1..16 on the GPU path")


def c_options(opts: EstimatorOptions, n: int, k_cap: int = 0) -> _native.SlseOptions:
    o = _native.SlseOptions()
    o.grid_factor = int(opts.grid_factor)
    o.tau = float(opts.tau)
    o.max_outer_iterations = int(opts.max_outer_iterations)
    o.convergence_tol_scale = float(opts.convergence_tol_scale)
    o.lbfgs_inner_max = int(opts.lbfgs_inner_max)
    o.newton_decrement_tol_scale = float(opts.newton_decrement_tol_scale)
    o.initial_sweep_iterations = int(opts.initial_sweep_iterations)
    o.lbfgs_memory = int(opts.lbfgs_memory)
    o.k_max = int(opts.k_max) if opts.k_max is not None else n
    o.trace_capacity = 2 + 13 * int(opts.max_outer_iterations)
    o.event_capacity = 4 * o.k_max + 64
    o.decomp_method = DECOMP_METHODS[opts.decomp_method]
    o.k_cap = int(k_cap)
    return o


def algorithms(opts: EstimatorOptions, n: int, backend: str = "superfast") -> dict:
    """The algorithms the device runs for these options (reported in
    LseResult.algorithms).  decomp_method selects the Toeplitz factorisation
    exactly as toeplitz.decompose does (:263-276; "auto" switches to the
    superfast divide-and-conquer Schur from N = 4096, the device crossover).
    Every off-grid Fourier sum (nufft.steer_forward / steer_adjoint /
    fourier_sum_two_sided) is evaluated EXACTLY on the device -- the values
    the reference's "direct" method computes (nufft.py:139-141,156-158), in
    the product form of SURVEY.md 8(a) rows 8-9 -- whatever steer_method
    says; the reference's "nufft" approximates the same sums to ~1e-10
    (SURVEY.md 8(c)), so it is accepted and served by the exact sums."""
    if backend == "semifast":
        return {"backend": "semifast", "decomp": "cholesky (Woodbury, K x K)",
                "steer": "direct (exact Gram / Fourier sums)", "steer_requested": opts.steer_method}
    dm = opts.decomp_method
    schur = dm == "schur" or (dm == "auto" and n >= 4096)
    return {"backend": "superfast",
            "decomp": "generalized_schur (superfast D&C)" if schur else "levinson (Schur-Levinson)",
            "steer": "direct (exact, product form)", "steer_requested": opts.steer_method}


class BatchOutputs:
    """Output arrays of one batched solve (torch tensors on one device, or
    numpy arrays for host-side consumers), laid out as slse_outputs."""

    def __init__(self, xp_empty, B, kmax, tcap, ecap, g=1, max_outer=200):
        e = xp_empty
        self.k_hat = e((B,), "i32")
        self.status = e((B,), "i32")
        self.iterations = e((B,), "i32")
        self.flags = e((B,), "i32")
        self.beta = e((B,), "f64")
        self.zeta = e((B,), "f64")
        self.theta = e((B, kmax), "f64")
        self.gamma = e((B, kmax), "f64")
        self.alpha = e((B, g, kmax, 2), "f64")  # [B, G, kmax] complex
        self.slot = e((B, kmax), "i32")
        self.trace = e((B, tcap), "f64")
        self.stage = e((B, tcap), "i32")
        self.trace_k = e((B, tcap), "i32")
        self.n_trace = e((B,), "i32")
        self.events = e((B, ecap, 3), "i32")
        self.n_events = e((B,), "i32")
        self.counters = e((B, 4), "i64")
        self.stage_seconds = e((B, 6), "f64")
        self.iter_seconds = e((B, max(1, max_outer)), "f64")

    def struct(self, ptr_of) -> _native.SlseOutputs:
        s = _native.SlseOutputs()
        for name in _native.OUTPUT_FIELDS:
            setattr(s, name, ptr_of(getattr(self, name)))
        return s


def decode_events(rows: np.ndarray):
    """(kind, slot, idx) rows -> [("sweep", [(slot, idx)...]) | ("activate", slot, idx) |
    ("deactivate", [slots])] (the encoding of tests/golden/make_golden.py)."""
    out = []
    cur = []
    for row in rows:
        kind, slot, idx = row
        if kind == -1:
            if cur:
                k0 = cur[0][0]
                if k0 == 0:
                    out.append(("sweep", [(s, i) for _, s, i in cur]))
                elif k0 == 1:
                    out.append(("activate", cur[0][1], cur[0][2]))
                else:
                    out.append(("deactivate", [s for _, s, _ in cur]))
            cur = []
        else:
            cur.append((int(kind), int(slot), int(idx)))
    return out


_STAGE_ARR = np.array(STAGE_NAMES, dtype=object)


def unpack_all(h: dict, algos: dict = None):
    """LseResult per problem from host (numpy) copies of the batch outputs.
    Per-problem arrays are views of ONE pageable copy per field (the caller
    owns them, as the reference's results, estimator.py:262-275; they do not
    keep the batch's pinned host block alive, and the batch is copied in a
    few large copies instead of six small ones per problem)."""
    B = h["k_hat"].shape[0]
    khat = h["k_hat"].tolist()
    ntr = h["n_trace"].tolist()
    nev = h["n_events"].tolist()
    flags = h["flags"].tolist()
    status = h["status"].tolist()
    iters = h["iterations"].tolist()
    beta = h["beta"].tolist()
    zeta = h["zeta"].tolist()
    alpha = np.array(h["alpha"]).view(np.complex128)[..., 0]  # (B, G, K), pageable copy
    names = _STAGE_ARR[np.clip(h["stage"], 0, len(STAGE_NAMES) - 1)]
    secs = h["stage_seconds"].tolist()
    ctr = h["counters"].tolist()
    theta, gamma, slot, trace, trace_k = (np.array(h[k]) for k in ("theta", "gamma", "slot", "trace", "trace_k"))
    events = h["events"]
    iter_s = h.get("iter_seconds")
    out = []
    for b in range(B):
        k, nt, fl = khat[b], ntr[b], flags[b]
        warns = []
        if fl & (FLAG_KMAX_CAP | FLAG_TRACE_FULL | FLAG_EVENTS_FULL):
            if fl & FLAG_KMAX_CAP:
                warns.append("activation loop hit the K_max cap")
            if fl & FLAG_TRACE_FULL:
                warns.append("objective trace truncated (trace capacity)")
            if fl & FLAG_EVENTS_FULL:
                warns.append("active-set history truncated (event capacity)")
        times = dict(zip(TIMER_NAMES, secs[b]))
        times["per_iteration"] = (iter_s[b, :min(iters[b], iter_s.shape[1])].tolist()
                                  if iter_s is not None else [])
        c = ctr[b]
        out.append(LseResult(
            k_hat=k,
            theta_hat=theta[b, :k],
            alpha_hat=alpha[b, :, :k],
            beta_hat=beta[b],
            gamma_hat=gamma[b, :k],
            zeta_hat=zeta[b],
            objective_trace=trace[b, :nt],
            iterations=iters[b],
            wall_time_per_stage=times,
            converged=bool(fl & FLAG_CONVERGED),
            trace_stages=names[b, :nt].tolist(),
            warnings=warns,
            events=decode_events(events[b, :nev[b]].tolist()),
            trace_k=trace_k[b, :nt],
            slots=slot[b, :k],
            counters=dict(builds=c[0], grids=c[1], stats=c[2], line_search_trials=c[3]),
            status=status[b],
            algorithms=dict(algos) if algos else {},
        ))
    return out


def unpack(h: dict, b: int, algos: dict = None) -> LseResult:
    """LseResult of problem b alone (see unpack_all)."""
    sub = {k: v[b:b + 1] for k, v in h.items()}
    return unpack_all(sub, algos)[0]


# ------------------------------------------------------------------ GPU path
def _torch():
    import torch

    return torch


_TORCH_DT = {"i32": "int32", "f64": "float64", "i64": "int64"}


class BatchSolver:
    """Reusable device buffers + launch for B problems of length N.

    ``solve(y_dev)`` launches on the current torch stream; inputs must be a
    contiguous complex128 (B, N) CUDA tensor.  ``results()`` copies back and
    unpacks.  No host synchronisation happens inside ``solve``."""

    def __init__(self, n: int, batch: int, opts: EstimatorOptions = None, device=None, g: int = 1, m: int = None,
                 backend: str = None, k_cap: int = 0):
        torch = _torch()
        self.opts = opts or EstimatorOptions()
        _validate(self.opts)
        self.m = int(m) if m is not None else n
        if self.m < 2:
            raise ValueError("need at least two observed samples")
        self.backend = backend or resolve_backend(self.opts, n, self.m == n)
        if self.backend == "superfast" and self.m != n:
            raise InvalidPattern("superfast backend requires the complete observation pattern")
        self.lib = _native.load()
        if not torch.cuda.is_available():
            raise SuperLseError("no CUDA device: the GPU estimator has no CPU fallback")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.batch, self.g = n, batch, int(g)
        if self.g < 1:
            raise ValueError("need at least one snapshot")
        self.copts = c_options(self.opts, self.m, k_cap)
        self.kmax = self.copts.k_max
        self.L = default_grid_size(n, self.opts.grid_factor)
        with torch.cuda.device(self.device):
            if self.backend == "semifast":
                ws = self.lib.slse_estimate_workspace_bytes_semifast(n, self.m, self.g, batch, ctypes.byref(self.copts))
            else:
                ws = self.lib.slse_estimate_workspace_bytes_mmv(n, self.g, batch, ctypes.byref(self.copts))
            if ws == 0:
                _native.check(-1, "slse_estimate_workspace_bytes")
            self.workspace = torch.empty(int(ws), dtype=torch.uint8, device=self.device)

            def empty(shape, dt):
                return torch.empty(shape, dtype=getattr(torch, _TORCH_DT[dt]), device=self.device)

            self.out = BatchOutputs(empty, batch, self.kmax, self.copts.trace_capacity, self.copts.event_capacity,
                                    g=self.g, max_outer=self.copts.max_outer_iterations)
        self.cout = self.out.struct(lambda t: t.data_ptr())
        self.algorithms = algorithms(self.opts, n, self.backend)
        self._stream = None
        self._pattern = None

    def set_pattern(self, idx0, scales=None):
        """Observation pattern of the semifast solve: 0-based positions
        (M,) shared by the batch or (B, M) per problem, and complex scales of
        the same shape (None = ones)."""
        torch = _torch()
        idx = torch.as_tensor(np.ascontiguousarray(idx0, dtype=np.int32)).to(self.device)
        if idx.shape[-1] != self.m or idx.dim() not in (1, 2) or (idx.dim() == 2 and idx.shape[0] != self.batch):
            raise DimensionMismatch("observed_indices must have shape (M,) or (B, M)")
        sc = None
        if scales is not None:
            sc = torch.as_tensor(np.ascontiguousarray(scales, dtype=np.complex128)).to(self.device)
            if tuple(sc.shape) != tuple(idx.shape):
                raise DimensionMismatch("scales must have the shape of observed_indices")
        self._pattern = (idx, sc, 0 if idx.dim() == 1 else self.m)

    def solve(self, y_dev, stream=None):
        torch = _torch()
        w = self.m if self.backend == "semifast" else self.n
        want = (self.batch, w) if self.g == 1 else (self.batch, self.g, w)
        if y_dev.dtype != torch.complex128 or not y_dev.is_contiguous() or tuple(y_dev.shape) != want:
            raise DimensionMismatch(f"y must be a contiguous complex128 tensor of shape {want}")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._stream = st
        if self.backend == "semifast":
            if self._pattern is None:  # complete data: the identity pattern
                self.set_pattern(np.arange(self.n, dtype=np.int32))
            idx, sc, stride = self._pattern
            rc = self.lib.slse_estimate_batch_semifast(
                ctypes.c_void_p(y_dev.data_ptr()), self.n, self.m, self.g, self.batch,
                ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(sc.data_ptr() if sc is not None else None), stride,
                ctypes.byref(self.copts), ctypes.byref(self.cout), ctypes.c_void_p(self.workspace.data_ptr()),
                ctypes.c_size_t(self.workspace.numel()), ctypes.c_void_p(st.cuda_stream))
            _native.check(rc, "slse_estimate_batch_semifast")
            return
        rc = self.lib.slse_estimate_batch_mmv(
            ctypes.c_void_p(y_dev.data_ptr()), self.n, self.g, self.batch, ctypes.byref(self.copts),
            ctypes.byref(self.cout), ctypes.c_void_p(self.workspace.data_ptr()),
            ctypes.c_size_t(self.workspace.numel()), ctypes.c_void_p(st.cuda_stream))
        _native.check(rc, "slse_estimate_batch_mmv")

    def _d2h(self, tensors: dict) -> dict:
        """Asynchronous copies into one fresh pinned block and one stream
        sync.  The returned arrays are views of that block and keep it alive;
        once the caller drops them, torch's caching host allocator hands the
        block to the next call, so steady-state calls neither pin new memory
        nor copy (or page-fault) the outputs a second time on the host."""
        torch = _torch()
        # copy on the stream the last solve() ran on (stream-ordered after it)
        st = self._stream if self._stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            ts = {name: t.contiguous() for name, t in tensors.items()}
            span = {name: (t.numel() * t.element_size() + 63) // 64 * 64 for name, t in ts.items()}
            buf = torch.empty(max(64, sum(span.values())), dtype=torch.uint8, pin_memory=True)
            off = 0
            host = {}
            for name, t in ts.items():
                nb = t.numel() * t.element_size()
                hb = buf[off:off + nb].view(t.dtype).view(t.shape)
                hb.copy_(t, non_blocking=True)
                host[name] = hb
                off += span[name]
        st.synchronize()
        return {name: hb.numpy() for name, hb in host.items()}

    def host_outputs(self) -> dict:
        """Host copies, trimmed to the longest trace / history / model order
        in the batch (one small D2H for the counts, then the used prefixes;
        two stream syncs in all)."""
        small = ("k_hat", "status", "iterations", "flags", "beta", "zeta", "n_trace", "n_events", "counters",
                 "stage_seconds")
        h = self._d2h({name: getattr(self.out, name) for name in small})
        kk = max(1, int(h["k_hat"].max(initial=0)))
        tt = max(1, int(h["n_trace"].max(initial=0)))
        ee = max(1, int(h["n_events"].max(initial=0)))
        o = self.out
        ii = max(1, min(int(h["iterations"].max(initial=0)), o.iter_seconds.shape[1]))
        big = {"theta": o.theta[:, :kk], "gamma": o.gamma[:, :kk], "alpha": o.alpha[:, :, :kk], "slot": o.slot[:, :kk],
               "trace": o.trace[:, :tt], "stage": o.stage[:, :tt], "trace_k": o.trace_k[:, :tt],
               "events": o.events[:, :ee], "iter_seconds": o.iter_seconds[:, :ii]}
        h.update(self._d2h(big))
        return h

    def results(self):
        return unpack_all(self.host_outputs(), self.algorithms)


class BatchResult:
    """Results of a batched solve: structure-of-arrays host copies (every
    estimate of every problem) plus list-like access to per-problem
    LseResult objects, built on first access.

    SoA fields (problem-major): k_hat, status, iterations, converged, beta,
    zeta (B,); theta, gamma, slot (B, K) zero-padded past k_hat; alpha
    complex (B, K), or (B, G, K) with G > 1 snapshots; trace (B, T) padded
    past n_trace.  The SoA arrays are zero-copy views of one pinned host
    block (no second host copy of the outputs); the block returns to torch's
    pinned-memory cache when the last of them is dropped.  The per-problem
    LseResult arrays are independent copies."""

    def __init__(self, h: dict, algos: dict = None):
        self.h = h
        self.algorithms = algos or {}
        self.k_hat = h["k_hat"]
        self.status = h["status"]
        self.iterations = h["iterations"]
        self.converged = (h["flags"] & FLAG_CONVERGED) != 0
        self.beta = h["beta"]
        self.zeta = h["zeta"]
        self.theta = h["theta"]
        self.gamma = h["gamma"]
        alpha = np.ascontiguousarray(h["alpha"]).view(np.complex128)[..., 0]  # (B, G, K)
        self.alpha = alpha[:, 0] if alpha.shape[1] == 1 else alpha
        self.slot = h["slot"]
        self.trace = h["trace"]
        self.n_trace = h["n_trace"]
        self._items = None

    def __len__(self):
        return int(self.k_hat.shape[0])

    def _all(self):
        if self._items is None:
            self._items = unpack_all(self.h, self.algorithms)
        return self._items

    def __getitem__(self, i):
        return self._all()[i]

    def __iter__(self):
        return iter(self._all())


_SOLVERS = threading.local()


def _cached_solver(n, batch, opts, device, g, m=None, backend=None, k_cap=0):
    """BatchSolver reuse across calls of one thread (device buffers and the
    workspace are sized by (N, M, B, G, options, backend, device)); results
    are host copies, so reuse by sequential calls is safe."""
    torch = _torch()
    opts = opts or EstimatorOptions()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (n, m, batch, g, dataclasses.astuple(opts), backend, k_cap, str(dev))
    cache = getattr(_SOLVERS, "cache", None)
    if cache is None:
        cache = _SOLVERS.cache = {}
    s = cache.get(key)
    if s is None:
        if len(cache) >= 4:
            cache.pop(next(iter(cache)))
        s = cache[key] = BatchSolver(n, batch, opts, device=dev, g=g, m=m, backend=backend, k_cap=k_cap)
    return s


def _check_pattern(n, m, observed_indices, scales, batch):
    """Observation's pattern contract (model_core.py:66-81) for a shared (M,)
    or per-problem (B, M) pattern: 1-based, sorted, unique, within 1..n.
    Returns 0-based int32 positions and complex scales (or None)."""
    idx = np.asarray(observed_indices, dtype=np.int64)
    if idx.ndim not in (1, 2) or idx.shape[-1] != m or (idx.ndim == 2 and idx.shape[0] != batch):
        raise DimensionMismatch("observed_indices must have length M (shape (M,) or (B, M))")
    if np.any(np.diff(idx, axis=-1) <= 0):
        raise ValueError("observed_indices must be sorted and unique")
    if idx.min() < 1 or idx.max() > n:
        raise ValueError("observed_indices must lie in 1..n")
    sc = None
    if scales is not None:
        sc = np.asarray(scales, dtype=np.complex128)
        if sc.shape != idx.shape:
            raise DimensionMismatch("scales must have length M")
    return (idx - 1).astype(np.int32), sc


def estimate_batch(y, opts: EstimatorOptions = None, device=None, return_solver=False, n: int = None,
                   observed_indices=None, scales=None) -> BatchResult:
    """Solve B independent problems, y: (B, M) complex, or (B, G, M) for G
    snapshots per problem sharing the frequencies (MMV).  Complete data
    (default): M = N.  Incomplete data (the semifast backend,
    model_core.Observation.incomplete): ``n`` and the 1-based
    ``observed_indices`` (M,) shared by the batch or (B, M) per problem, with
    optional complex ``scales`` of the same shape.  Accepts numpy or torch
    input; returns a BatchResult (SoA arrays + a sequence of LseResult in
    problem order).  Problems that hit a non-PD covariance carry ``status`` 1
    instead of raising."""
    torch = _torch()
    opts = opts or EstimatorOptions()
    if isinstance(y, torch.Tensor):
        yt = y
    else:
        yt = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(np.asarray(y, dtype=np.complex128))))
    if yt.dim() not in (2, 3):
        raise DimensionMismatch("y must have shape (B, M) or (B, G, M)")
    g = 1 if yt.dim() == 2 else int(yt.shape[1])
    if yt.dim() == 3 and g == 1:
        yt = yt[:, 0]
    m = int(yt.shape[-1])
    B = int(yt.shape[0])
    complete = observed_indices is None
    if complete:
        if n is not None and int(n) != m:
            raise DimensionMismatch(f"complete data needs M == n, got {m} != {n}")
        n = m
    n = int(n)
    backend = resolve_backend(opts, n, complete)
    pattern = None if complete else _check_pattern(n, m, observed_indices, scales, B)
    # pinned input (e.g. a torch.Tensor from pin_memory()) goes up
    # asynchronously; pageable numpy memory is copied by the driver directly
    # (cheaper than page-locking it for one transfer)
    pinned = yt.device.type == "cpu" and yt.is_pinned()
    k_cap = SEMIFAST_FIRST_KCAP
    while True:
        solver = _cached_solver(n, B, opts, device, g, m=m, backend=backend, k_cap=k_cap)
        ydev = yt.to(device=solver.device, dtype=torch.complex128, non_blocking=pinned).contiguous()
        if pattern is not None:
            solver.set_pattern(*pattern)
        else:
            solver._pattern = None
        solver.solve(ydev)
        h = solver.host_outputs()
        if backend != "semifast" or not np.any(h["status"] == STATUS_KCAP) or k_cap >= solver.kmax:
            break
        # a semifast active set outgrew the K capacity: rerun at full K_max
        # (whole batch; results are deterministic per problem)
        k_cap = solver.kmax
    res = BatchResult(h, solver.algorithms)
    return (res, solver) if return_solver else res


def estimate(obs: Observation, opts: EstimatorOptions = None) -> LseResult:
    """Fit the line-spectrum model (estimator.py:117-275) on the GPU."""
    opts = opts if opts is not None else EstimatorOptions()
    if obs.m < 2:
        raise ValueError("need at least two observed samples")
    _validate(opts)
    resolve_backend(opts, obs.n, obs.is_complete)  # InvalidPattern for superfast on incomplete data
    y = np.asarray(obs.y, dtype=np.complex128)
    if obs.is_complete:
        res = estimate_batch(y if obs.g == 1 else y[None], opts)[0]
    else:
        res = estimate_batch(y if obs.g == 1 else y[None], opts, n=obs.n, observed_indices=obs.observed_indices,
                             scales=obs.scales)[0]
    if res.status == STATUS_NOT_PD:
        raise NotPositiveDefinite("covariance lost positive definiteness during the fit")
    if res.status == STATUS_BAD_DIAGONAL:
        raise NotPositiveDefinite("diagonal entry c_0 must be real and positive")
    return res


def estimate_mmv(obs: Observation, opts: EstimatorOptions = None) -> LseResult:
    """estimator.py:278-283: snapshots share the frequencies; same path as
    estimate() (G = 1 included)."""
    return estimate(obs, opts)
