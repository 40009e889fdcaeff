#!/usr/bin/env python
"""NEXT-2 measurement: the paper's reconstruction loop on B200 -- OS-SART
with "blocks of 20 projections" and CGLS -- on the CUDA
operators, timed per iteration with CUDA events, through the plain calls
(every call runs the entry finder) and through PlannedOperators (one plan
per subset: the entry maps are built once, before the first iteration).

Workload: c3 (1.01 M-tet graded box, 512^2 cone beam, 360 angles), data
b = A mu_true simulated on the same mesh (fig:rec (a), known-mesh setting).
Prints one JSON line: ms per iteration and operator crossings/s for each
(solver, operators) pair, the plan build time, and the relative residual
after the timed iterations.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06909_b200 import solvers as S  # noqa: E402
from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


def main(cfg="c3", iters=3, block=20):
    w = CF.workload(cfg)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    b = tm.project(w.geom, mu)
    _, st = tm.project(w.geom, mu, stats=True)
    cross = st["crossings"]                    # per full projection (= per backprojection)
    calls = (lambda g, x: tm.project(g, x), lambda g, y: tm.backproject(g, y))
    res = {"config": cfg, "tets": w.mesh.n_tets, "rays": w.geom.n_rays, "crossings_per_pass": cross,
           "block": block, "iterations_timed": iters}
    for ops in ("calls", "plans"):
        po = T.PlannedOperators(tm)
        if ops == "plans":
            # build every subset's plan once (what a reconstruction does before
            # its first iteration); timed separately
            n_sub = (w.geom.n_angles + block - 1) // block
            subsets = [np.flatnonzero(np.arange(w.geom.n_angles) % n_sub == s) for s in range(n_sub)]
            _, t_plan = timed(lambda: [po.plan(S._subset(w.geom, idx)) for idx in subsets])
            po.plan(w.geom)
            res["plan_build_ms"] = t_plan
            P, B = po.project, po.backproject
        else:
            P, B = calls
        # OS-SART: one iteration = every subset once (A_s x and A_s^T r per
        # subset) after the weights (A 1, A^T 1) of the untimed setup
        S.os_sart(P, B, w.geom, b, torch.zeros_like(mu), n_iter=1, block=block)   # warm-up
        x, ms = timed(lambda: S.os_sart(P, B, w.geom, b, torch.zeros_like(mu), n_iter=iters,
                                        block=block))
        # the timed call also builds the weights: 2 passes; each iteration 2 passes
        passes = 2 + 2 * iters
        r = float((tm.project(w.geom, x) - b).norm() / b.norm())
        res[f"os_sart_{ops}"] = {"ms_total": ms, "passes": passes, "ms_per_pass": ms / passes,
                                 "crossings_per_s": passes * cross / (ms / 1e3),
                                 "rel_residual": r}
        S.cgls(P, B, w.geom, b, torch.zeros_like(mu), n_iter=1)                   # warm-up
        x, ms = timed(lambda: S.cgls(P, B, w.geom, b, torch.zeros_like(mu), n_iter=iters))
        passes = 2 + 2 * iters
        r = float((tm.project(w.geom, x) - b).norm() / b.norm())
        res[f"cgls_{ops}"] = {"ms_total": ms, "passes": passes, "ms_per_pass": ms / passes,
                              "crossings_per_s": passes * cross / (ms / 1e3), "rel_residual": r}
        po.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c3"]))
