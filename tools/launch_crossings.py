#!/usr/bin/env python
"""Crossings of the walk launches that tools/gpu_r02_head_ncu.sh captures
(the first launch of each direction in bench.py's untimed statistics calls):
c3 launch 0 = angles [0, 256) (2^26 rays per launch), c5 launch 0 = [0, 64),
c2 / c4b / c4a = all angles.  Writes one JSON object to stdout."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402

LAUNCH0 = {"c3": 256, "c5": 64, "c2": None, "c4b": None, "c4a": None}


def main():
    out = {}
    for cfg, n in LAUNCH0.items():
        w = CF.workload(cfg)
        g = w.geom if n is None else w.geom.subset(np.arange(n))
        tm = T.TetMesh.from_mesh(w.mesh)
        _, st = tm.project(g, torch.from_numpy(w.mu).cuda(), stats=True)
        out[cfg] = {"angles": int(g.n_angles), "crossings": int(st["crossings"])}
        del tm
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
