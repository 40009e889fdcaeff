#!/usr/bin/env python
"""A wider randomized parity campaign than tests/test_gpu_fuzz.py (same
generator, seeds [first, first + n)): random small meshes on a coarse
lattice (rays through vertices / edges / faces are common) under random cone
/ parallel / lattice-aligned scans, each entry finder in turn and both exact
walks, every case element by element against the CPU oracle with the
north-star tolerances (tests/gpu_util.check_parity).  Prints one JSON line:
cases, failures (seed + message), totals of rays, crossings and exact
fallbacks.

  python tests/campaigns/fuzz_campaign.py [first_seed] [n]
  python tests/campaigns/fuzz_campaign.py mt first_seed n      # the paper's walk vs the MT oracle
  python tests/campaigns/fuzz_campaign.py medium first_seed n  # 1e3-1e5-tet meshes
"""
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1908_06909_b200 import tetproj as T  # noqa: E402
from tests import gpu_util as U  # noqa: E402
from tests.test_gpu_fuzz import _case  # noqa: E402


def mt_case(seed):
    """The paper's Alg. 1/2 walk (fp64 for even seeds, fp32 for odd) vs the
    MT oracle: bit-identical projections, equal crossing / lost / stuck /
    escalation counts (tests/test_gpu_fuzz.py::test_random_scans_paper_mode_match_mt_oracle)."""
    import numpy as np
    import torch

    from oracle import tetref as O
    mesh, geom, mu, y = _case(seed)
    single = bool(seed % 2)
    tm = T.TetMesh.from_mesh(mesh)
    mode = T.TET_TRAVERSE_MT_F32 if single else T.TET_TRAVERSE_MT_F64
    p, st = tm.project(geom, torch.from_numpy(mu).cuda(), stats=True, opts=T.options(mode))
    q, ost = O.mt_project(O.OracleMesh.from_mesh(mesh), geom, mu.astype(np.float64), single=single)
    for k in ("rays_hit", "crossings", "lost", "stuck", "escalations"):
        assert st[k] == ost[k], (k, st, ost)
    np.testing.assert_array_equal(p.cpu().numpy().ravel(), q.astype(np.float32).ravel())
    return st


def main_mt(first, n):
    fails, lost, esc = [], 0, 0
    for seed in range(first, first + n):
        try:
            st = mt_case(seed)
            lost += st["lost"] + st["stuck"]
            esc += st["escalations"]
        except Exception as e:   # noqa: BLE001
            fails.append({"seed": seed, "error": repr(e)[:300]})
    print(json.dumps({"mode": "mt", "first_seed": first, "cases": n, "failures": fails,
                      "paper_walk_lost_or_stuck": lost, "escalations": esc}))


def medium_case(seed):
    """Medium meshes (ball Delaunay h in [0.15, 0.35]; jittered lattices n in
    [4, 14] with jitter 1e-4 / 1e-3 / 0.05 / 0.2 h -- slivers; graded boxes of
    2-8 k interior points; exact Kuhn lattices n in [2, 8] -- vertex and edge
    degeneracies) under random cone / parallel scans of 8-48^2 pixels, 1-4
    angles."""
    import numpy as np

    from workloads import geometry as G
    from workloads import meshes as M
    rng = np.random.default_rng(50_000 + seed)
    kind = seed % 4
    if kind == 0:
        mesh = M.ball_mesh(h=float(rng.uniform(0.15, 0.35)), seed=seed)
    elif kind == 1:
        mesh = M.jittered_lattice_mesh(int(rng.integers(4, 15)),
                                       float([1e-4, 1e-3, 0.05, 0.2][(seed // 4) % 4]), seed)
    elif kind == 3:   # exact Kuhn lattice: rays through vertices and edges
        mesh = M.kuhn_lattice(int(rng.integers(2, 9)))
    else:
        mesh = M.graded_box_mesh(int(rng.integers(2000, 8000)), seed=seed, per_edge=2, per_face=6)
    R = float(np.linalg.norm(mesh.verts, axis=1).max())
    n_u, n_v = int(rng.integers(8, 49)), int(rng.integers(8, 49))
    ang = rng.uniform(0, 2 * np.pi, int(rng.integers(1, 5)))
    if rng.uniform() < 0.6:
        dso = R * rng.uniform(1.5, 4)
        dsd = dso + R * rng.uniform(1.5, 4)
        mag = dsd / dso
        geom = G.circular_cone(ang, dso, dsd, n_u, n_v, 2.4 * R * mag / n_u, 2.4 * R * mag / n_v,
                               off_u=rng.uniform(-1, 1), off_v=rng.uniform(-1, 1))
    else:
        geom = G.circular_parallel(ang, n_u, n_v, 2.4 * R / n_u, 2.4 * R / n_v,
                                   off_u=rng.uniform(-1, 1), off_v=rng.uniform(-1, 1))
    mu = rng.uniform(0.3, 1.5, mesh.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    return mesh, geom, mu, y


def main_medium(first, n):
    fails, rays, cross, exact, tets = [], 0, 0, 0, 0
    for seed in range(first, first + n):
        try:
            mesh, geom, mu, y = medium_case(seed)
            entry = [T.TET_ENTRY_RASTER, T.TET_ENTRY_BVH, T.TET_ENTRY_RTREE][(seed // 3) % 3]
            r = U.check_parity(mesh, geom, mu, y, opts=T.options(entry=entry))
            rays += r["stats"]["rays"]
            cross += r["stats"]["crossings"]
            exact += r["stats"]["exact_fallbacks"]
            tets += mesh.n_tets
        except Exception as e:   # noqa: BLE001
            fails.append({"seed": seed, "error": repr(e)[:300],
                          "where": traceback.format_exc().splitlines()[-3:]})
    print(json.dumps({"mode": "medium", "first_seed": first, "cases": n, "failures": fails,
                      "tets": tets, "rays": rays, "crossings": cross, "exact_fallbacks": exact}))


def main(first=100, n=400):
    fails, rays, cross, exact = [], 0, 0, 0
    for seed in range(first, first + n):
        mesh, geom, mu, y = _case(seed)
        entry = [T.TET_ENTRY_RASTER, T.TET_ENTRY_BVH, T.TET_ENTRY_RTREE][seed % 3]
        walker = "rec" if seed % 5 == 4 else None
        if walker:
            os.environ["TETPROJ_WALKER"] = walker
        try:
            r = U.check_parity(mesh, geom, mu, y, opts=T.options(entry=entry))
            rays += r["stats"]["rays"]
            cross += r["stats"]["crossings"]
            exact += r["stats"]["exact_fallbacks"]
        except Exception as e:   # noqa: BLE001 -- record and continue
            fails.append({"seed": seed, "error": repr(e)[:300],
                          "where": traceback.format_exc().splitlines()[-3:]})
        finally:
            os.environ.pop("TETPROJ_WALKER", None)
    print(json.dumps({"first_seed": first, "cases": n, "failures": fails, "rays": rays,
                      "crossings": cross, "exact_fallbacks": exact}))


if __name__ == "__main__":
    if sys.argv[1:2] == ["mt"]:
        main_mt(*[int(x) for x in sys.argv[2:4]])
    elif sys.argv[1:2] == ["medium"]:
        main_medium(*[int(x) for x in sys.argv[2:4]])
    else:
        main(*[int(x) for x in sys.argv[1:3]])
