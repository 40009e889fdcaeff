#!/usr/bin/env python
"""Small workload touching every kernel family, for compute-sanitizer runs:
exact walker (forward/backward, degenerate c1 + lattice + ball), the three
entry finders, the paper-faithful MT walker, the permutes, plans (device and
host buffers, f64 accumulation).  Exits non-zero on any error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402
from workloads import geometry as G  # noqa: E402
from workloads import meshes as M  # noqa: E402


def run(mesh, geom, mu, y):
    tm = T.TetMesh.from_mesh(mesh)
    mu_d, y_d = torch.from_numpy(mu).cuda(), torch.from_numpy(y).cuda()
    for opts in (None, T.options(entry=T.TET_ENTRY_BVH), T.options(entry=T.TET_ENTRY_RTREE),
                 T.options(T.TET_TRAVERSE_MT_F64), T.options(T.TET_TRAVERSE_MT_F32)):
        p, st = tm.project(geom, mu_d, stats=True, opts=opts)
        x, st2 = tm.backproject(geom, y_d, stats=True, opts=opts)
        if opts is None:
            assert st["lost"] == st["stuck"] == st["entry_conflicts"] == 0, st
    with tm.plan(geom) as pl:
        p2 = pl.project(mu_d)
        pl.backproject(y_d)
        pl.backproject_f64(y_d)
        T.tet_plan_project(pl.handle, mu, np.zeros(geom.n_rays, np.float32))
        T.tet_plan_backproject(pl.handle, y, np.zeros(mesh.n_tets, np.float32))
        torch.cuda.synchronize()
    assert torch.equal(p2, tm.project(geom, mu_d))
    torch.cuda.synchronize()


def main():
    w = CF.workload("c1")
    run(w.mesh, w.geom, w.mu, w.y)
    m = M.random_small_mesh(40, 2)
    g = G.lattice_parallel((1 / 8,) * 3, (0, 0, 0), 19, 13, G.LATTICE_DIRS[:4])
    rng = np.random.default_rng(0)
    run(m, g, rng.uniform(0.5, 1.5, m.n_tets).astype(np.float32),
        rng.uniform(0.5, 1.5, g.n_rays).astype(np.float32))
    m = M.ball_mesh(h=0.25, seed=2)
    g = G.circular_cone(G.equidistant(2), 4.0, 8.0, 37, 29, 4.4 / 37, 4.4 / 29)
    run(m, g, rng.uniform(0.5, 1.5, m.n_tets).astype(np.float32),
        rng.uniform(0.5, 1.5, g.n_rays).astype(np.float32))
    print("sanitize case ok")


if __name__ == "__main__":
    main()
