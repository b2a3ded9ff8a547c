"""Build librelcp.so (sm_100a) in-tree with nvcc.

    python -m paper_2506_14097_b200.build [--force] [--ptxas-v]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "librelcp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "relcp.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu into one shared library (default: LIB).
    `defines` / `out` build tuning variants (e.g. SCATTER_MINB=6) side by side."""
    target = out or LIB
    if not force and out is None and not defines and not stale():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *(["-Xptxas", "-v"] if ptxas_v else []), *("-D" + d for d in defines),
           "-o", target + ".tmp", *sources()]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="--ptxas-v" in sys.argv))
