"""ctypes binding of the C ABI in include/superlse_b200.h.

The shared library is the nvcc-built ``_lib/libsuperlse_b200.so`` (see
build.py).  There is no fallback: if it is missing or no CUDA device is
visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import SuperLseError

_LIB_PATH = os.environ.get("SLSE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                     "libsuperlse_b200.so")
ABI_VERSION = 3

c_int_p = ctypes.POINTER(ctypes.c_int32)


class SlseOptions(ctypes.Structure):
    """slse_options (include/superlse_b200.h)."""

    _fields_ = [
        ("grid_factor", ctypes.c_int),
        ("tau", ctypes.c_double),
        ("max_outer_iterations", ctypes.c_int),
        ("convergence_tol_scale", ctypes.c_double),
        ("lbfgs_inner_max", ctypes.c_int),
        ("newton_decrement_tol_scale", ctypes.c_double),
        ("initial_sweep_iterations", ctypes.c_int),
        ("lbfgs_memory", ctypes.c_int),
        ("k_max", ctypes.c_int),
        ("trace_capacity", ctypes.c_int),
        ("event_capacity", ctypes.c_int),
        ("decomp_method", ctypes.c_int),
        ("k_cap", ctypes.c_int),
    ]


OUTPUT_FIELDS = ("k_hat", "status", "iterations", "flags", "beta", "zeta", "theta", "gamma", "alpha", "slot",
                 "trace", "stage", "trace_k", "n_trace", "events", "n_events", "counters", "stage_seconds", "iter_seconds")


class SlseOutputs(ctypes.Structure):
    """slse_outputs (include/superlse_b200.h); all device pointers."""

    _fields_ = [(name, ctypes.c_void_p) for name in OUTPUT_FIELDS]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load (once) and return the CDLL; raises if the .so is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise SuperLseError(
            f"CUDA extension not built: {_LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i, d, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    sig = {
        "slse_abi_version": ([], i),
        "slse_last_error": ([], ctypes.c_char_p),
        "slse_device_info": ([c_int_p, c_int_p, c_int_p, c_int_p], i),
        "slse_default_options": ([ctypes.POINTER(SlseOptions)], None),
        "slse_cov_column": ([vp, vp, vp, i, vp, i, i, vp, vp], i),
        "slse_toeplitz_factor": ([vp, i, i, vp, vp, vp, vp, vp], i),
        "slse_toeplitz_factor_ex": ([vp, i, i, vp, vp, vp, vp, i, vp], i),
        "slse_gs_apply": ([vp, vp, vp, i, i, vp, vp, vp], i),
        "slse_component_stats": ([vp, vp, i, vp, vp, vp, i, i, vp, vp, vp, vp, vp, vp, vp, vp], i),
        "slse_grid_eval": ([vp, vp, vp, i, i, i, vp, vp, vp], i),
        "slse_grid_eval_omega": ([vp, vp, i, i, i, vp, vp, vp], i),
        "slse_omegas": ([vp, vp, i, i, vp, vp, vp, vp, vp], i),
        "slse_activation_curve": ([vp, vp, vp, vp, i, i, i, vp, vp, vp], i),
        "slse_deactivation_margins": ([vp, vp, vp, vp, i, vp, i, i, vp, vp, vp], i),
        "slse_gradient_hessian": ([vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp, vp, vp], i),
        "slse_estimate_workspace_bytes": ([i, i, ctypes.POINTER(SlseOptions)], sz),
        "slse_estimate_batch": ([vp, i, i, ctypes.POINTER(SlseOptions), ctypes.POINTER(SlseOutputs), vp, sz, vp], i),
        "slse_estimate_workspace_bytes_mmv": ([i, i, i, ctypes.POINTER(SlseOptions)], sz),
        "slse_estimate_batch_mmv": ([vp, i, i, i, ctypes.POINTER(SlseOptions), ctypes.POINTER(SlseOutputs), vp, sz,
                                     vp], i),
        "slse_estimate_workspace_bytes_semifast": ([i, i, i, i, ctypes.POINTER(SlseOptions)], sz),
        "slse_estimate_batch_semifast": ([vp, i, i, i, i, vp, vp, i, ctypes.POINTER(SlseOptions),
                                          ctypes.POINTER(SlseOutputs), vp, sz, vp], i),
        "slse_semifast_bundle_workspace_bytes": ([i, i, i, i, i, i], sz),
        "slse_semifast_bundle": ([vp, vp, vp, i, vp, vp, i, i, i, i, vp, vp, i, i] + [vp] * 13 + [sz, vp], i),
        "slse_sim_workspace_bytes": ([i, i], sz),
        "slse_sim_generate": ([ctypes.c_ulonglong, ctypes.c_uint, i, i, i, i, i, d, d, i, d] + [vp] * 8, i),
        "slse_sim_metrics": ([i, i, i, vp, vp, i, vp, vp, vp, i, vp, vp, vp, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.slse_abi_version() != ABI_VERSION:
        raise SuperLseError("libsuperlse_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = _lib.slse_last_error().decode() if _lib is not None else ""
        raise SuperLseError(f"{what} failed ({rc}): {msg}")
