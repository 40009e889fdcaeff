"""Build libtetproj.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtetproj.so")
SOURCES = ["mesh_host.cpp", "rtree_host.cpp", "kernels.cu", "api.cu"]
HEADERS = ["internal.h"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "tetproj.h"))
    return any(os.path.getmtime(d) > t for d in deps)


MICRO_SRC = os.path.join(CSRC, "microbench.cu")
MICRO_LIB = os.path.join(HERE, "libtetmicro.so")


def build_micro(force: bool = False) -> str:
    """libtetmicro.so: roofline microbenchmarks (experiments/microbench.py)."""
    if force or not os.path.exists(MICRO_LIB) or os.path.getmtime(MICRO_LIB) < os.path.getmtime(MICRO_SRC):
        tmp = MICRO_LIB + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc(), "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", MICRO_SRC, "-o", tmp])
        os.replace(tmp, MICRO_LIB)
    return MICRO_LIB


DEBUG_LIB = os.path.join(HERE, "libtetproj_debug.so")


def build_debug(force: bool = False) -> str:
    """libtetproj_debug.so: the same sources with -DTETPROJ_DEBUG (device-side
    bounds checks that trap); loaded when TETPROJ_DEBUG_LIB=1."""
    if force or not os.path.exists(DEBUG_LIB) or any(
            os.path.getmtime(os.path.join(CSRC, f)) > os.path.getmtime(DEBUG_LIB)
            for f in SOURCES + HEADERS):
        tmp = DEBUG_LIB + f".tmp{os.getpid()}"
        flags = [f for f in NVCC_FLAGS if f not in ("-v", "-Xptxas")]
        cmd = [nvcc(), *flags, "-DTETPROJ_DEBUG",
               *[os.path.join(CSRC, f) for f in SOURCES], "-o", tmp]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libtetproj_debug.so")
        os.replace(tmp, DEBUG_LIB)
    return DEBUG_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *[os.path.join(CSRC, f) for f in SOURCES], "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libtetproj.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
