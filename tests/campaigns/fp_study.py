#!/usr/bin/env python
"""NEXT-1: the paper's robustness study (fig:singledouble)
re-run on B200: the paper's own traversal (Alg. 1 epsilon-guarded
Möller-Trumbore + Alg. 2 epsilon escalation) in single and
double precision against the exact-SoS walker, on sliver meshes where rays run
through vertices / edges (c4a), classic Delaunay slivers (c4b) and the graded
CAD-like mesh (c3).

Prints one JSON line per (mesh, mode): rays hit, lost ("black dots": fewer
than two faces found even after 12 escalations), stuck (looping), epsilon
escalations per million crossings, and the fraction of hit pixels within
1e-4 of the exact projection.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402

CASES = [("c4a", dict(n_angles=16, n_u=256, n_v=256), dict(n_angles=4, n_u=48, n_v=48)),
         ("c4b", dict(n_angles=8, n_u=256, n_v=256), dict(n_angles=2, n_u=64, n_v=64)),
         ("c3", dict(n_angles=8, n_u=256, n_v=256), dict(n_angles=2, n_u=64, n_v=64))]
MODES = [("exact", T.TET_TRAVERSE_EXACT), ("mt_f64", T.TET_TRAVERSE_MT_F64),
         ("mt_f32", T.TET_TRAVERSE_MT_F32)]
KEYS = ("rays_hit", "crossings", "lost", "stuck", "escalations")


def study(w, with_oracle):
    """One line per mode; with_oracle: the CPU MT oracle (oracle/tetref_mt.inc,
    the same IEEE operations) on the same rays, its counts beside the GPU's."""
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    om = None
    if with_oracle:
        from oracle import tetref as O
        om = O.OracleMesh.from_mesh(w.mesh)
    ref = None
    lines = []
    for mname, mode in MODES:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p, st = tm.project(w.geom, mu, stats=True, opts=T.options(mode))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        p = p.cpu().numpy().astype(np.float64)
        if ref is None:
            ref = p
        hit = ref != 0
        floor = 1e-3 * float(np.abs(w.mu).mean()) * 3.46
        err = np.abs(p - ref) / np.maximum(np.abs(ref), floor)
        line = {"mesh": w.name, "tets": w.mesh.n_tets, "mode": mname, "rays": st["rays"],
                "detector": [w.geom.n_angles, w.geom.n_v, w.geom.n_u],
                "rays_hit": st["rays_hit"], "lost": st["lost"], "stuck": st["stuck"],
                "crossings": st["crossings"], "escalations": st["escalations"],
                "escalations_per_Mcrossing": 1e6 * st["escalations"] / max(st["crossings"], 1),
                "pixels_within_1e-4": float((err[hit] <= 1e-4).mean()) if hit.any() else None,
                "max_rel_err": float(err[hit].max()) if hit.any() else None,
                "seconds": dt}
        if om is not None and mode != T.TET_TRAVERSE_EXACT:
            from oracle import tetref as O
            t0 = time.perf_counter()
            q, ost = O.mt_project(om, w.geom, w.mu.astype(np.float64),
                                  single=mode == T.TET_TRAVERSE_MT_F32)
            line["oracle"] = {k: ost[k] for k in KEYS}
            line["oracle"]["seconds"] = time.perf_counter() - t0
            line["oracle_counts_equal"] = all(ost[k] == st[k] for k in KEYS)
            line["oracle_pixels_bitwise_equal"] = bool(
                np.array_equal(q.astype(np.float32).ravel(), p.astype(np.float32).ravel()))
        print(json.dumps(line), flush=True)
        lines.append(line)
    return lines


def main():
    out = []
    for name, kw, kw_small in CASES:
        out += study(CF.workload(name, **kw), False)
        out += study(CF.workload(name, **kw_small), True)
    path = os.path.join(ROOT, "gpurun_out", "fp_study.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
