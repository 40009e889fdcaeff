"""Seeded randomized parity sweep (GPU): small random meshes (points on a
coarse lattice, so rays through vertices / edges / faces are common) under
random scans -- generic and lattice-aligned cone beams, lattice and generic
parallel beams, random detector sizes and angle counts -- each entry finder
(raster, BVH, R*-tree) and both walks (FT16 and the record walk), every case
element by element against the CPU oracle: identical crossing and hit
counts, forward per pixel and backprojection per tet within the north-star
tolerances, zero lost / stuck / conflicting rays."""
import os

import numpy as np
import pytest

from tests import gpu_util as U
from workloads import geometry as G
from workloads import meshes as M

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    mesh = M.random_small_mesh(int(rng.integers(15, 60)), 100 + seed, box=bool(seed % 3))
    n_u, n_v = int(rng.integers(3, 24)), int(rng.integers(3, 24))
    kind = seed % 4
    if kind == 0:       # generic cone beam
        dso = rng.uniform(3, 6)     # mesh radius <= sqrt(3): strictly between source and detector
        geom = G.circular_cone(rng.uniform(0, 2 * np.pi, int(rng.integers(1, 5))),
                               dso, dso + rng.uniform(2, 6), n_u, n_v,
                               rng.uniform(0.1, 0.5), rng.uniform(0.1, 0.5),
                               off_u=rng.uniform(-2, 2), off_v=rng.uniform(-2, 2))
    elif kind == 1:     # cone from lattice points through lattice pixel centres
        rows = []
        for _ in range(int(rng.integers(1, 4))):
            th = rng.uniform(0, 2 * np.pi)
            S = np.round(np.array([4 * np.sin(th), -4 * np.cos(th), rng.uniform(-1, 1)]) * 16) / 16
            Uv = np.array([0.0625, 0, 0]) if abs(np.cos(th)) > 0.5 else np.array([0, 0.0625, 0])
            V = np.array([0, 0, 0.0625])
            rows.append(np.concatenate([S, -S - (n_u // 2) * Uv - (n_v // 2) * V, Uv, V]))
        geom = G.explicit(G.BEAM_CONE, n_v, n_u, rows)
    elif kind == 2:     # lattice-aligned parallel rays
        dirs = [G.LATTICE_DIRS[i] for i in rng.choice(len(G.LATTICE_DIRS), 3, replace=False)]
        geom = G.lattice_parallel((1 / 16,) * 3, (0, 0, 0), n_u, n_v, dirs)
    else:               # generic parallel beam
        geom = G.circular_parallel(rng.uniform(0, 2 * np.pi, int(rng.integers(1, 5))), n_u, n_v,
                                   rng.uniform(0.1, 0.4), rng.uniform(0.1, 0.4),
                                   off_u=rng.uniform(-1, 1), off_v=rng.uniform(-1, 1))
    mu = rng.uniform(0.3, 1.5, mesh.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    return mesh, geom, mu, y


@pytest.mark.parametrize("seed", range(48))
def test_random_scans_match_oracle(seed):
    from paper_1908_06909_b200 import tetproj as T
    mesh, geom, mu, y = _case(seed)
    entry = [T.TET_ENTRY_RASTER, T.TET_ENTRY_BVH, T.TET_ENTRY_RTREE][seed % 3]
    walker = "rec" if seed % 5 == 4 else None
    if walker:
        os.environ["TETPROJ_WALKER"] = walker       # read at mesh creation
    try:
        U.check_parity(mesh, geom, mu, y, opts=T.options(entry=entry))
    finally:
        os.environ.pop("TETPROJ_WALKER", None)


@pytest.mark.parametrize("seed", range(12))
def test_random_scans_paper_mode_match_mt_oracle(seed):
    """The paper's Alg. 1/2 walk (fp64 for even seeds, fp32 for odd) on the
    same random scans: bit-identical projections and equal crossing, lost,
    stuck and escalation counts against the MT oracle."""
    import torch

    from oracle import tetref as O
    from paper_1908_06909_b200 import tetproj as T
    mesh, geom, mu, y = _case(seed)
    single = bool(seed % 2)
    tm = T.TetMesh.from_mesh(mesh)
    mode = T.TET_TRAVERSE_MT_F32 if single else T.TET_TRAVERSE_MT_F64
    p, st = tm.project(geom, torch.from_numpy(mu).cuda(), stats=True, opts=T.options(mode))
    q, ost = O.mt_project(O.OracleMesh.from_mesh(mesh), geom, mu.astype(np.float64), single=single)
    for k in ("rays_hit", "crossings", "lost", "stuck", "escalations"):
        assert st[k] == ost[k], (k, st, ost)
    np.testing.assert_array_equal(p.cpu().numpy().ravel(), q.astype(np.float32).ravel())


@pytest.mark.parametrize("seed", range(0, 48, 4))
def test_random_scans_through_plans(seed):
    """The same random scans through a plan (entry map built once, each entry
    finder in turn): bit-identical projections and equal statistics to the
    plan-less calls, backprojections equal up to the atomics' order."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    mesh, geom, mu, y = _case(seed)
    entry = [T.TET_ENTRY_RASTER, T.TET_ENTRY_BVH, T.TET_ENTRY_RTREE][(seed // 4) % 3]
    opts = T.options(entry=entry)
    tm = T.TetMesh.from_mesh(mesh)
    mu_d, y_d = torch.from_numpy(mu).cuda(), torch.from_numpy(y).cuda()
    p0, s0 = tm.project(geom, mu_d, stats=True, opts=opts)
    x0, t0 = tm.backproject(geom, y_d, stats=True, opts=opts)
    with tm.plan(geom, opts) as pl:
        p1, s1 = pl.project(mu_d, stats=True)
        x1, t1 = pl.backproject(y_d, stats=True)
        torch.cuda.synchronize()
    assert torch.equal(p0, p1)
    for k in ("rays_hit", "crossings", "lost", "stuck", "exact_fallbacks", "entry_conflicts"):
        assert s0[k] == s1[k] and t0[k] == t1[k], (k, s0, s1, t0, t1)
    np.testing.assert_allclose(x1.cpu().numpy(), x0.cpu().numpy(), rtol=2e-7, atol=1e-30)
