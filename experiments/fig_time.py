#!/usr/bin/env python
"""NEXT-3: the paper's performance experiment (fig:time)
on B200: "computing times ... for regular tetrahedra meshes of increased
size", initialisation and ray propagation timed separately, one 1024x1024
cone-beam projection.  "The regular meshes have been created by linearly
increasing the number of points along each edge."

Mesh: Kuhn lattice n^3 (6 n^3 tets, 12 n^2 hull faces) in [-1/2,1/2]^3.
Prints one JSON line per n: entry-finder ms (initialisation), walk ms
(propagation), crossings, and crossings/s; the paper's claims are that the
propagation cost grows linearly with the edge length and the initialisation
cost only logarithmically (the paper's R*-tree, timed as init_rtree_ms; the
default detector-space raster as init_ms).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import geometry as G  # noqa: E402
from workloads import meshes as M  # noqa: E402


def main(ns=(8, 16, 24, 32, 48, 64, 96, 128), reps=5):
    R = np.sqrt(3) / 2
    geom = G.circular_cone([0.3], 4 * R, 8 * R, 1024, 1024, 3.6 * R / 1024, 3.6 * R / 1024)
    out = []
    for n in ns:
        mesh = M.kuhn_lattice(n)
        tm = T.TetMesh.from_mesh(mesh)
        mu = torch.ones(mesh.n_tets, device="cuda")
        proj = torch.empty((1, 1024, 1024), device="cuda")
        st = T.tet_project(tm.handle, geom, mu, proj, stats=True)
        T.tet_set_kernel_timing(tm.handle, True)
        T.tet_kernel_times(tm.handle)
        for _ in range(reps):
            T.tet_project(tm.handle, geom, mu, proj)
        torch.cuda.synchronize()
        kt = T.tet_kernel_times(tm.handle)
        # the paper's own initialisation: per-ray depth-first search of the
        # R*-tree over the hull faces (TET_ENTRY_RTREE)
        opts = T.options(entry=T.TET_ENTRY_RTREE)
        T.tet_project(tm.handle, geom, mu, proj, opts=opts)
        torch.cuda.synchronize()
        T.tet_kernel_times(tm.handle)
        for _ in range(reps):
            T.tet_project(tm.handle, geom, mu, proj, opts=opts)
        torch.cuda.synchronize()
        kt_r = T.tet_kernel_times(tm.handle)
        T.tet_set_kernel_timing(tm.handle, False)
        line = {"edge_points": n + 1, "tets": mesh.n_tets, "hull_faces": mesh.n_bfaces,
                "init_ms": kt["entry"][0] / reps, "init_rtree_ms": kt_r["entry"][0] / reps,
                "rtree_nodes": T.tet_mesh_features(tm.handle)["rtree_nodes"],
                "propagation_ms": kt["forward"][0] / reps,
                "crossings": st["crossings"], "rays_hit": st["rays_hit"],
                "crossings_per_s": st["crossings"] / (kt["forward"][0] / reps / 1e3),
                "lost": st["lost"], "stuck": st["stuck"]}
        print(json.dumps(line), flush=True)
        out.append(line)
    path = os.path.join(ROOT, "gpurun_out", "fig_time.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
