"""In-tree build of the sm_100a shared library (libsuperlse_b200.so).

nvcc compiles the C-ABI translation unit and the four per-block-size
solver instantiations in parallel, then links one shared object into
``paper_1705_06073_b200/_lib/``.  The .so is git-ignored but travels to the
GPU box with the repo snapshot.  Nothing here needs a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(REPO, "include")
# Variant builds (tools/): SLSE_BUILD_DEFS adds -D flags, SLSE_BUILD_OUT
# redirects objects and the .so (the default build ignores both).
_OUT = os.environ.get("SLSE_BUILD_OUT")
LIBDIR = os.path.abspath(_OUT) if _OUT else os.path.join(PKG, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj") if _OUT else os.path.join(REPO, "build", "obj")
EXTRA_DEFS = os.environ.get("SLSE_BUILD_DEFS", "").split() if _OUT else []
LIBNAME = "libsuperlse_b200.so"
LIBPATH = os.path.join(LIBDIR, LIBNAME)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-Xcompiler", "-fPIC",
                     "-I" + INCLUDE, "-I" + CSRC]
SOLVE_NTS = (32, 64, 128, 256, 512, 1024)


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required)")
    return cand


def _sources():
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    hdrs.append(os.path.join(INCLUDE, "superlse_b200.h"))
    units = [("slse_capi", os.path.join(CSRC, "slse_capi.cu"), [])]
    for nt in SOLVE_NTS:
        units.append((f"slse_solve_{nt}", os.path.join(CSRC, "slse_solve_inst.cu"), [f"-DSLSE_NT={nt}"]))
    units.append(("slse_solve_warps", os.path.join(CSRC, "slse_solve_warps.cu"), ["-DSLSE_WARP_MODE"]))
    units.append(("slse_solve_sf", os.path.join(CSRC, "slse_solve_sf.cu"), ["-DSLSE_SEMIFAST"]))
    units.append(("slse_sim", os.path.join(CSRC, "slse_sim.cu"), []))
    return hdrs, units


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False) -> str:
    """Compile (if stale) and return the path of the shared library."""
    hdrs, units = _sources()
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdr_time = _newest(hdrs + [__file__])
    exe = nvcc()
    extra = ["-Xptxas", "-v"] if ptxas_info else []

    def compile_unit(u):
        name, src, defs = u
        obj = os.path.join(OBJDIR, name + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(hdr_time, os.path.getmtime(src)):
            return obj, ""
        cmd = [exe] + NVCC_FLAGS + extra + EXTRA_DEFS + defs + ["-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{res.stderr[-6000:]}")
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        results = list(ex.map(compile_unit, units))
    objs = [r[0] for r in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if force or not os.path.exists(LIBPATH) or os.path.getmtime(LIBPATH) < _newest(objs):
        cmd = [exe] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", LIBPATH] + objs
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stderr[-4000:]}")
    return LIBPATH


if __name__ == "__main__":
    t = build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(t)
