#!/usr/bin/env python
"""Build A/B variants of libtetproj with compile-time knobs (kernels.cu
TRACE_* macros) into paper_1908_06909_b200/variants/libtetproj_<name>.so;
bench.py / tests load one with TETPROJ_LIB_VARIANT=<name>.

  python tools/build_variants.py name=-DKNOB=1,-DOTHER=2 [name2=...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1908_06909_b200 import _build  # noqa: E402


def build(spec):
    name, flags = spec.split("=", 1)
    out_dir = os.path.join(os.path.dirname(_build.LIB), "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libtetproj_{name}.so")
    cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *[f for f in flags.split(",") if f],
           *[os.path.join(_build.CSRC, f) for f in _build.SOURCES], "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        return f"{name}: FAILED\n{r.stderr[-3000:]}"
    regs = [l for l in r.stderr.splitlines() if "Used" in l and "registers" in l]
    return f"{name}: ok ({len(regs)} kernels)"


if __name__ == "__main__":
    with ThreadPoolExecutor(8) as ex:
        for line in ex.map(build, sys.argv[1:]):
            print(line)
