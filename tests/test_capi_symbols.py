"""The C-ABI shared library builds, loads without a GPU and exports every
entry point include/superlse_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "superlse_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(slse_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1705_06073_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("slse_cov_column", "slse_toeplitz_factor", "slse_gs_apply", "slse_component_stats",
              "slse_grid_eval", "slse_estimate_batch", "slse_estimate_workspace_bytes"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_native_binding_loads_and_reports_abi(lib):
    from paper_1705_06073_b200 import _native

    L = _native.load()
    assert L.slse_abi_version() == _native.ABI_VERSION
    o = _native.SlseOptions()
    L.slse_default_options(ctypes.byref(o))
    assert (o.grid_factor, o.max_outer_iterations, o.lbfgs_memory, o.lbfgs_inner_max) == (8, 200, 10, 5)
    assert o.tau == 5.0 and o.convergence_tol_scale == 1e-7 and o.newton_decrement_tol_scale == 1e-8


def test_sm100a_cubin_present(lib):
    """The .so carries sm_100a SASS (no PTX-only / other-arch build)."""
    import shutil
    import subprocess

    from paper_1705_06073_b200 import build

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", build.LIBPATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
