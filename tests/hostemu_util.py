"""Build/load the TEST-ONLY host emulation of the device program
(tests/hostemu/slse_hostemu.cpp) and run it on numpy inputs."""

import ctypes
import os
import subprocess

import numpy as np

from paper_1705_06073_b200 import _native
from paper_1705_06073_b200.estimator import BatchOutputs, EstimatorOptions, c_options, unpack

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SRC = os.path.join(HERE, "hostemu", "slse_hostemu.cpp")
OUT = os.path.join(HERE, "hostemu", "_build", "libslse_hostemu.so")
CSRC = os.path.join(REPO, "paper_1705_06073_b200", "csrc")

_lib = None


def build():
    global _lib
    if _lib is not None:
        return _lib
    deps = [SRC] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(d) for d in deps):
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I" + os.path.join(REPO, "include"),
                        "-I" + CSRC, SRC, "-o", OUT], check=True)
    lib = ctypes.CDLL(OUT)
    lib.emu_estimate_batch.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(_native.SlseOptions), ctypes.POINTER(_native.SlseOutputs)]
    vp = ctypes.c_void_p
    lib.emu_bundle.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                               vp, vp, vp, vp, vp, vp, vp]
    _lib = lib
    return lib


_NP = {"i32": np.int32, "f64": np.float64, "i64": np.int64}


def estimate_batch_raw(Y, opts=None):
    """Host-output dict of the emulated batch (the layout of
    BatchSolver.host_outputs)."""
    lib = build()
    opts = opts or EstimatorOptions()
    Y = np.ascontiguousarray(np.atleast_2d(np.asarray(Y, dtype=np.complex128)))
    B, n = Y.shape
    co = c_options(opts, n)
    out = BatchOutputs(lambda shape, dt: np.zeros(shape, dtype=_NP[dt]), B, co.k_max, co.trace_capacity,
                       co.event_capacity, max_outer=co.max_outer_iterations)
    st = out.struct(lambda a: a.ctypes.data)
    lib.emu_estimate_batch(Y.ctypes.data, n, B, ctypes.byref(co), ctypes.byref(st))
    return {name: getattr(out, name) for name in _native.OUTPUT_FIELDS}


def estimate_batch(Y, opts=None):
    h = estimate_batch_raw(Y, opts)
    return [unpack(h, b) for b in range(h["k_hat"].shape[0])]


def bundle(y, thetas, gammas, beta, L):
    """Per-call quantities of one bundle: dict(c, rho, w, logdet, delta_last, data_term, q_grid, s_grid, stats)."""
    lib = build()
    y = np.ascontiguousarray(y, dtype=np.complex128)
    n = y.size
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    ga = np.ascontiguousarray(gammas, dtype=np.float64)
    k = th.size
    c = np.zeros(n, complex)
    rho = np.zeros(n, complex)
    w = np.zeros(n, complex)
    sc = np.zeros(3)
    qg = np.zeros(L, complex)
    sg = np.zeros(L)
    st = np.zeros(5 * 2 * k + 2 * k + 1)
    rc = lib.emu_bundle(y.ctypes.data, n, th.ctypes.data, ga.ctypes.data, k, float(beta), L, c.ctypes.data,
                        rho.ctypes.data, w.ctypes.data, sc.ctypes.data, qg.ctypes.data, sg.ctypes.data,
                        st.ctypes.data)
    out = dict(status=rc, c=c, rho=rho, w=w, logdet=sc[0], delta_last=sc[1], data_term=sc[2], q_grid=qg, s_grid=sg)
    if k:
        cs = st[: 10 * k].view(complex)
        out.update(q=cs[:k], r=cs[k:2 * k], u=cs[2 * k:3 * k], t=cs[3 * k:4 * k], v=cs[4 * k:5 * k],
                   s=st[10 * k:11 * k], x=st[11 * k:12 * k])
    return out
