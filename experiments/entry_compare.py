#!/usr/bin/env python
"""NEXT-3: entry finders compared -- per-(face, angle) exact rasterisation of
hull-face footprints (default) vs per-ray searches of a binary BVH and of the
paper's R*-tree (fan-out 4..10, depth-first) over the hull
faces.  All take the same exact decision: the projections must be
bit-identical.  One JSON line per config with the entry-finder milliseconds
of one forward projection."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from workloads import configs as CF  # noqa: E402


def main():
    out = []
    for name, kw in [("c2", {}), ("c3", dict(n_angles=90)), ("c4a", {}), ("c4b", {})]:
        w = CF.workload(name, **kw)
        tm = T.TetMesh.from_mesh(w.mesh)
        mu = torch.from_numpy(w.mu).cuda()
        res = {}
        for ename, mode in [("raster", T.TET_ENTRY_RASTER), ("bvh", T.TET_ENTRY_BVH),
                            ("rtree", T.TET_ENTRY_RTREE)]:
            opts = T.options(entry=mode)
            p, st = tm.project(w.geom, mu, stats=True, opts=opts)
            T.tet_set_kernel_timing(tm.handle, True)
            T.tet_kernel_times(tm.handle)
            for _ in range(3):
                tm.project(w.geom, mu, out=p, opts=opts)
            torch.cuda.synchronize()
            kt = T.tet_kernel_times(tm.handle)
            T.tet_set_kernel_timing(tm.handle, False)
            res[ename] = (p.clone(), st, kt["entry"][0] / 3, kt["forward"][0] / 3)
        same = all(torch.equal(res["raster"][0], res[k][0]) for k in ("bvh", "rtree"))
        line = {"config": name, "tets": w.mesh.n_tets, "hull_faces": w.mesh.n_bfaces,
                "rays": w.geom.n_rays, "identical": same,
                "raster_entry_ms": res["raster"][2], "bvh_entry_ms": res["bvh"][2],
                "rtree_entry_ms": res["rtree"][2], "walk_ms": res["raster"][3],
                "crossings_equal": all(res["raster"][1]["crossings"] == res[k][1]["crossings"]
                                       for k in ("bvh", "rtree"))}
        print(json.dumps(line), flush=True)
        out.append(line)
    path = os.path.join(ROOT, "gpurun_out", "entry_compare.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
