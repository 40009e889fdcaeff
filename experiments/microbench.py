#!/usr/bin/env python
"""Measured roofline denominators for the walker:

  gather32_L2   random 32-B gathers (one 256-bit load each) from a 64 MB buffer
                (2^21 records; 32-bit xorshift index masked to the power of two)
  gather32_HBM  the same from a 8 GB buffer (DRAM-resident)
  gather16_L2   random 16-B gathers from a 64 MB buffer (the vertex gather)
  stream_L2     coalesced reads of a 64 MB buffer, 50 passes (L2 bandwidth)
  dfma          fp64 FMA rate (8 independent chains per thread)
  red_f64       RED.ADD.F64 to random addresses of an 8 MB array (L2 atomics)
  red_f32       RED.ADD.F32, same pattern
  red_*_coherent  8 addresses x 4 lanes per warp instruction (the walker's pattern)

Prints one JSON object; copied to profiles/ as rNN_microbench.json.
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1908_06909_b200", "csrc", "microbench.cu")
LIB = os.path.join(ROOT, "paper_1908_06909_b200", "libtetmicro.so")


def build():
    sys.path.insert(0, ROOT)
    from paper_1908_06909_b200 import _build
    _build.build_micro()
    L = C.CDLL(LIB)
    L.tetmicro_run.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int]
    L.tetmicro_run.restype = C.c_double
    return L


def main():
    L = build()
    sms = 148
    out = {"gpu": "B200 (sm_100a)"}
    blocks, threads, iters = sms * 16, 256, 256
    n = blocks * threads * iters
    ms = L.tetmicro_run(0, 64 << 20, iters, blocks, threads)
    out["gather32_L2_GBps"] = n * 32 / (ms / 1e3) / 1e9
    out["gather32_L2_Grec_per_s"] = n / (ms / 1e3) / 1e9
    ms = L.tetmicro_run(0, 8 << 30, iters, blocks, threads)
    out["gather32_HBM_GBps"] = n * 32 / (ms / 1e3) / 1e9
    out["gather32_HBM_Grec_per_s"] = n / (ms / 1e3) / 1e9
    ms = L.tetmicro_run(7, 64 << 20, iters, blocks, threads)
    out["gather16_L2_GBps"] = n * 16 / (ms / 1e3) / 1e9
    out["gather16_L2_Grec_per_s"] = n / (ms / 1e3) / 1e9
    passes = 50
    ms = L.tetmicro_run(1, 64 << 20, passes, sms * 8, 512)
    out["stream_L2_GBps"] = (64 << 20) * passes / (ms / 1e3) / 1e9
    it = 4096
    ms = L.tetmicro_run(2, 256, it, sms * 8, 256)
    out["dfma_TFLOPs"] = sms * 8 * 256 * it * 8 * 2 / (ms / 1e3) / 1e12
    it = 64
    ms = L.tetmicro_run(3, 8 << 20, it, sms * 16, 256)
    out["red_f64_Gops"] = sms * 16 * 256 * it / (ms / 1e3) / 1e9
    ms = L.tetmicro_run(4, 8 << 20, it, sms * 16, 256)
    out["red_f32_Gops"] = sms * 16 * 256 * it / (ms / 1e3) / 1e9
    ms = L.tetmicro_run(5, 8 << 20, it, sms * 16, 256)
    out["red_f64_coherent_Gops"] = sms * 16 * 256 * it / (ms / 1e3) / 1e9
    ms = L.tetmicro_run(6, 8 << 20, it, sms * 16, 256)
    out["red_f32_coherent_Gops"] = sms * 16 * 256 * it / (ms / 1e3) / 1e9
    print(json.dumps(out))
    path = os.path.join(ROOT, "gpurun_out", "microbench.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
