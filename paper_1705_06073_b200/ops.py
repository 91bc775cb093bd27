"""Per-call batched operators on CUDA tensors (the bundle pieces of
model_core._SuperfastBundle, model_core.py:256-313), each one launch of an
sm_100a kernel through the C ABI.  Complex arrays are complex128 tensors;
every call runs on the current torch stream and does not synchronise.

These are what the parity tests check call-by-call against the oracle; the
estimator itself runs all of them fused inside the solver kernel.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native
from .errors import NotPositiveDefinite


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _c128(t):
    assert t.dtype == torch.complex128 and t.is_cuda and t.is_contiguous()
    return t


def cov_column(theta, gamma, kcount, beta, n):
    """Row 1: c[b] = beta[b] e_0 + sum_{k<kcount[b]} gamma[b,k] psi(theta[b,k])
    (model_core.py:242-249).  theta/gamma: (B, K) float64; kcount: (B,) int32."""
    lib = _native.load()
    B, K = theta.shape
    c = torch.empty((B, n), dtype=torch.complex128, device=theta.device)
    _native.check(lib.slse_cov_column(_p(theta), _p(gamma), _p(kcount), K, _p(beta), n, B, _p(c), _stream()),
                  "slse_cov_column")
    return c


METHODS = {"auto": 0, "levinson": 1, "schur": 2}


def toeplitz_factor(c, with_delta=True, raise_on_error=False, method="auto"):
    """Rows 2-4: (rho, delta, logdet, status) of the Hermitian Toeplitz
    matrices with first columns c (B, N) (toeplitz.decompose, :263-276).
    method: "levinson" (Schur-Levinson, O(N^2)), "schur" (superfast
    divide-and-conquer, O(N log^2 N)) or "auto" (superfast from N >= 4096)."""
    lib = _native.load()
    _c128(c)
    B, n = c.shape
    rho = torch.empty_like(c)
    delta = torch.empty((B, n), dtype=torch.float64, device=c.device) if with_delta else None
    logdet = torch.empty(B, dtype=torch.float64, device=c.device)
    status = torch.empty(B, dtype=torch.int32, device=c.device)
    _native.check(lib.slse_toeplitz_factor_ex(_p(c), n, B, _p(rho), _p(delta), _p(logdet), _p(status),
                                              METHODS[method], _stream()), "slse_toeplitz_factor_ex")
    if raise_on_error and bool((status != 0).any()):
        raise NotPositiveDefinite("Toeplitz factorisation hit a non-positive pivot")
    return rho, delta, logdet, status


def gs_apply(rho, delta_last, y):
    """Row 5: (w = C^{-1} y, Re(y^H w)) (toeplitz.apply_inverse, :279-309)."""
    lib = _native.load()
    _c128(rho)
    _c128(y)
    B, n = rho.shape
    w = torch.empty_like(rho)
    quad = torch.empty(B, dtype=torch.float64, device=rho.device)
    _native.check(lib.slse_gs_apply(_p(rho), _p(delta_last.contiguous()), _p(y), n, B, _p(w), _p(quad), _stream()),
                  "slse_gs_apply")
    return w, quad


def component_stats(theta, kcount, rho, delta_last, w):
    """Row 8: dict of q, r, u, t, v (complex) and s, x (real), each (B, K)
    (model_core._SuperfastBundle.stats, :281-301)."""
    lib = _native.load()
    B, K = theta.shape
    n = rho.shape[1]
    dev = rho.device
    cz = lambda: torch.zeros((B, K), dtype=torch.complex128, device=dev)  # noqa: E731
    rz = lambda: torch.zeros((B, K), dtype=torch.float64, device=dev)  # noqa: E731
    q, r, u, t, v = cz(), cz(), cz(), cz(), cz()
    s, x = rz(), rz()
    _native.check(lib.slse_component_stats(_p(theta), _p(kcount), K, _p(rho), _p(delta_last.contiguous()), _p(w), n,
                                           B, _p(q), _p(r), _p(u), _p(s), _p(t), _p(v), _p(x), _stream()),
                  "slse_component_stats")
    return dict(q=q, r=r, u=u, s=s, t=t, v=v, x=x)


def grid_eval(rho, delta_last, w, L, out=None):
    """Row 9: (q_grid (B, L) complex, s_grid (B, L) real)
    (model_core._SuperfastBundle.grid, :303-313)."""
    lib = _native.load()
    B, n = rho.shape
    if out is None:
        qg = torch.empty((B, L), dtype=torch.complex128, device=rho.device)
        sg = torch.empty((B, L), dtype=torch.float64, device=rho.device)
    else:
        qg, sg = out
    _native.check(lib.slse_grid_eval(_p(rho), _p(delta_last.contiguous()), _p(w), n, L, B, _p(qg), _p(sg),
                                     _stream()), "slse_grid_eval")
    return qg, sg


def grid_eval_omega(w, om_s, L, out=None):
    """Row 9 in the reference's own form (model_core._SuperfastBundle.grid,
    :303-313): q_grid = FFT_L(w), s_grid = L IFFT_L(om_s wrapped).real, from
    w (B, N) and om_s (B, 2N-1) (the omegas() "s" diagonal sums); returns
    (q_grid (B, L) complex, s_grid (B, L) real)."""
    lib = _native.load()
    B, n = w.shape
    if om_s.shape != (B, 2 * n - 1):
        raise ValueError(f"om_s must be (B, 2N-1) = ({B}, {2 * n - 1}), got {tuple(om_s.shape)}")
    if out is None:
        qg = torch.empty((B, L), dtype=torch.complex128, device=w.device)
        sg = torch.empty((B, L), dtype=torch.float64, device=w.device)
    else:
        qg, sg = out
    _native.check(lib.slse_grid_eval_omega(_p(w), _p(om_s), n, L, B, _p(qg), _p(sg), _stream()),
                  "slse_grid_eval_omega")
    return qg, sg


def omegas(rho, delta_last):
    """Row 7: dict s, t, v, x of the diagonal sums omega(i), i = -(N-1)..N-1,
    each (B, 2N-1) complex (toeplitz.all_diagonal_sums, :415-432)."""
    lib = _native.load()
    B, n = rho.shape
    out = {k: torch.empty((B, 2 * n - 1), dtype=torch.complex128, device=rho.device) for k in "stvx"}
    _native.check(lib.slse_omegas(_p(rho), _p(delta_last.contiguous()), n, B, _p(out["s"]), _p(out["t"]),
                                  _p(out["v"]), _p(out["x"]), _stream()), "slse_omegas")
    return out


def activation_curve(q_grid, s_grid, gamma_bar, zeta, kmax, with_curve=True):
    """Row 10: (curve (B, L) float64 or None, argmin (B,) int32) of
    smlr._delta_objective_curve / best_candidate (:62-70, :84-96), G = 1."""
    lib = _native.load()
    B, L = s_grid.shape
    curve = torch.empty((B, L), dtype=torch.float64, device=s_grid.device) if with_curve else None
    idx = torch.empty(B, dtype=torch.int32, device=s_grid.device)
    _native.check(lib.slse_activation_curve(_p(q_grid), _p(s_grid), _p(gamma_bar.contiguous()), _p(zeta.contiguous()),
                                            kmax, L, B, _p(curve), _p(idx), _stream()), "slse_activation_curve")
    return curve, idx


def deactivation_margins(q, s, gamma, kcount, zeta, kmax):
    """Row 11: (margins (B, K) float64, argmin (B,) int32) of
    smlr.deactivation_margins (:174-200); entries past kcount[b] untouched."""
    lib = _native.load()
    B, K = s.shape
    margin = torch.zeros((B, K), dtype=torch.float64, device=s.device)
    idx = torch.empty(B, dtype=torch.int32, device=s.device)
    _native.check(lib.slse_deactivation_margins(_p(q), _p(s), _p(gamma), _p(kcount), K, _p(zeta.contiguous()), kmax,
                                                B, _p(margin), _p(idx), _stream()), "slse_deactivation_margins")
    return margin, idx


def gradient_hessian(stats, gamma, kcount, n):
    """Row 12: (g, d), each (B, 2K) float64: row b holds the theta block in
    [0, k) and the gamma block in [k, 2k), k = kcount[b]
    (model_core.gradient :497-505, diag_hessian :508-536)."""
    lib = _native.load()
    B, K = gamma.shape
    g = torch.zeros((B, 2 * K), dtype=torch.float64, device=gamma.device)
    d = torch.zeros((B, 2 * K), dtype=torch.float64, device=gamma.device)
    st = {k: v.contiguous() for k, v in stats.items()}
    _native.check(lib.slse_gradient_hessian(_p(st["q"]), _p(st["r"]), _p(st["u"]), _p(st["s"]), _p(st["t"]),
                                            _p(st["v"]), _p(st["x"]), _p(gamma), _p(kcount), K, n, B, _p(g), _p(d),
                                            _stream()), "slse_gradient_hessian")
    return g, d


def semifast_bundle(theta, gamma, kcount, beta, y, n, L, idx0=None, scales=None):
    """One semifast bundle per problem (model_core._SemifastBundle, :316-409):
    theta/gamma (B, K) float64 with kcount (B,) int32 active entries, beta
    (B,), y (B, M) or (B, G, M) complex observed samples, observation pattern
    idx0 (M,) or (B, M) 0-based int32 (None: complete, M = n) and complex
    scales of the same shape (None: ones), grid length L.  Returns a dict of
    data_term (B,), e (B, G, n), q, r, u (B, G, K), s, t, v, x (B, K),
    q_grid (B, G, L), s_grid (B, L), status (B,)."""
    lib = _native.load()
    _c128(y)
    dev = y.device
    B, K = theta.shape
    K = max(K, 1)
    g = 1 if y.dim() == 2 else int(y.shape[1])
    m = int(y.shape[-1])
    if idx0 is None:
        idx0 = torch.arange(n, dtype=torch.int32, device=dev)
    stride = 0 if idx0.dim() == 1 else m
    ws_bytes = lib.slse_semifast_bundle_workspace_bytes(n, m, g, B, L, K)
    if ws_bytes == 0:
        _native.check(-1, "slse_semifast_bundle_workspace_bytes")
    ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device=dev)
    c, f = torch.complex128, torch.float64
    out = dict(data_term=torch.empty(B, dtype=f, device=dev), e=torch.empty((B, g, n), dtype=c, device=dev),
               q=torch.zeros((B, g, K), dtype=c, device=dev), r=torch.zeros((B, g, K), dtype=c, device=dev),
               u=torch.zeros((B, g, K), dtype=c, device=dev), s=torch.zeros((B, K), dtype=f, device=dev),
               t=torch.zeros((B, K), dtype=c, device=dev), v=torch.zeros((B, K), dtype=c, device=dev),
               x=torch.zeros((B, K), dtype=f, device=dev), q_grid=torch.empty((B, g, L), dtype=c, device=dev),
               s_grid=torch.empty((B, L), dtype=f, device=dev), status=torch.empty(B, dtype=torch.int32, device=dev))
    th = theta if theta.shape[1] else torch.zeros((B, 1), dtype=f, device=dev)
    ga = gamma if gamma.shape[1] else torch.zeros((B, 1), dtype=f, device=dev)
    _native.check(lib.slse_semifast_bundle(
        _p(th.contiguous()), _p(ga.contiguous()), _p(kcount), K, _p(beta), _p(y), n, m, g, B, _p(idx0.contiguous()),
        _p(scales.contiguous() if scales is not None else None), stride, L,
        *[_p(out[k]) for k in ("data_term", "e", "q", "r", "u", "s", "t", "v", "x", "q_grid", "s_grid", "status")],
        _p(ws), ws_bytes, _stream()), "slse_semifast_bundle")
    return out
