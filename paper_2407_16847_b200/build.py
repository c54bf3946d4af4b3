"""Build libsplat.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2407_16847_b200.build [--force] [-j N] [--diag]

Every translation unit in csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
paper_2407_16847_b200/libsplat.so with the CUDA runtime linked statically.

``--diag`` builds the diagnostics variant libsplat_diag.so (-DSPLAT_DIAG, plus
SPLAT_EXTRA_NVCC_FLAGS such as -DSPLAT_TRACE): profiling / ablation knobs read
from the environment.  Only tools/ load it (SPLAT_LIB=diag); the product
library, the tests and bench.py use libsplat.so, which has no knobs.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libsplat.so")
DIAG_BUILD = os.path.join(PKG, "build_diag")
DIAG_LIB = os.path.join(PKG, "libsplat_diag.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _flags(diag: bool):
    return FLAGS + (["-DSPLAT_DIAG"] + os.environ.get("SPLAT_EXTRA_NVCC_FLAGS", "").split() if diag else [])


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "splat.h")]


def _compile(src: str, force: bool, verbose: bool, diag: bool = False) -> str:
    obj = os.path.join(DIAG_BUILD if diag else BUILD, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if force or diag or not os.path.exists(obj) or os.path.getmtime(obj) < newest_dep:
        cmd = [NVCC, *ARCH, *_flags(diag), "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        subprocess.check_call(cmd)
    return obj


def build(force: bool = False, jobs: int = 8, verbose: bool = False, diag: bool = False) -> str:
    """Build libsplat.so (or, with diag=True, always rebuild libsplat_diag.so)."""
    os.makedirs(DIAG_BUILD if diag else BUILD, exist_ok=True)
    lib = DIAG_LIB if diag else LIB
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, diag), srcs))
    if diag or force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true", help="ptxas -v resource usage")
    ap.add_argument("--diag", action="store_true", help="diagnostics variant libsplat_diag.so (tools only)")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v, a.diag))
    sys.exit(0)
