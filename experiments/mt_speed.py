#!/usr/bin/env python
"""NEXT-1 measured: the paper's own traversal (Alg. 1/2, eps-guarded
Moller-Trumbore with escalation, fp64 and fp32) against the exact walk on
the same scans, forward and backward, through one plan per mode: walk
kernel time (CUDA events around each launch, tet_kernel_times), crossings/s
and the rays each mode loses.  The paper's walk runs on the record layout
in world coordinates (mt_trace_kernel); the exact walk is the FT16 walk."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402


def main(cfg="c3", reps=3):
    w = CF.workload(cfg)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    y = torch.from_numpy(CF.uniform_y(w.geom, 1000)).cuda()
    out = {"config": cfg, "tets": w.mesh.n_tets, "rays": w.geom.n_rays}
    for name, mode in (("exact", T.TET_TRAVERSE_EXACT), ("mt_f64", T.TET_TRAVERSE_MT_F64),
                       ("mt_f32", T.TET_TRAVERSE_MT_F32)):
        with tm.plan(w.geom, T.options(mode)) as pl:
            _, sf = pl.project(mu, stats=True)
            _, sb = pl.backproject(y, stats=True)
            torch.cuda.synchronize()
            T.tet_set_kernel_timing(tm.handle, True)
            T.tet_kernel_times(tm.handle)
            for _ in range(reps):
                pl.project(mu)
                pl.backproject(y)
            torch.cuda.synchronize()
            kt = T.tet_kernel_times(tm.handle)
            T.tet_set_kernel_timing(tm.handle, False)
        f_ms, b_ms = kt["forward"][0] / reps, kt["backward"][0] / reps
        out[name] = {"forward_ms": f_ms, "backward_ms": b_ms,
                     "forward_crossings_per_s": sf["crossings"] / (f_ms / 1e3),
                     "backward_crossings_per_s": sb["crossings"] / (b_ms / 1e3),
                     "crossings": sf["crossings"], "lost": sf["lost"], "stuck": sf["stuck"],
                     "escalations": sf["escalations"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c3"]))
