"""Plans (tet_plan_*, include/tetproj.h): a scan bound to a mesh, its entry
map computed once at creation -- PAPER.md Alg. 2 (lines 120-144) starts every
ray with "Read initial intersection element".  A plan's calls run the same
walk kernels on the same entry map as the plan-less calls, so projections are
bit-identical to them, statistics equal, backprojections equal up to the
order of the double atomics (rounded once to float); and both are within the
north-star tolerances of the CPU oracle."""
import numpy as np
import pytest

from tests import gpu_util as U
from workloads import configs as CF
from workloads import geometry as G

pytestmark = pytest.mark.gpu

CASES = {
    "c2": dict(n_angles=3, n_u=67, n_v=53),      # sphere, cone beam
    "c4a": dict(n_angles=4, n_u=72, n_v=40),     # slivers, lattice parallel rays (exact-heavy)
    "c4b": dict(n_angles=2, n_u=48, n_v=40),     # jittered lattice, sources on lattice points
}
STAT_KEYS = ("rays", "rays_hit", "crossings", "lost", "stuck", "exact_fallbacks",
             "entry_conflicts", "max_crossings_per_ray")


def _setup(case):
    import torch

    from paper_1908_06909_b200 import TetMesh
    w = CF.workload(case, **CASES[case])
    tm = TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu.astype(np.float32)).cuda()
    y = torch.from_numpy(w.y.astype(np.float32).ravel()).cuda()
    return w, tm, mu, y


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("entry", ["raster", "bvh", "rtree"])
def test_plan_matches_unplanned_and_oracle(case, entry):
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w, tm, mu, y = _setup(case)
    opts = T.options(entry={"raster": T.TET_ENTRY_RASTER, "bvh": T.TET_ENTRY_BVH,
                            "rtree": T.TET_ENTRY_RTREE}[entry])
    p0, s0 = tm.project(w.geom, mu, stats=True, opts=opts)
    x0, t0 = tm.backproject(w.geom, y, stats=True, opts=opts)
    with tm.plan(w.geom, opts) as pl:
        p1, s1 = pl.project(mu, stats=True)
        x1, t1 = pl.backproject(y, stats=True)
        p2, s2 = pl.project(mu, stats=True)          # the map is reused, not consumed
        x2 = pl.backproject(y, out=x1.clone(), accumulate=True)
    torch.cuda.synchronize()
    assert torch.equal(p1, p0) and torch.equal(p2, p0)
    for k in STAT_KEYS:
        assert s1[k] == s0[k] == s2[k], (k, s0, s1)
        assert t1[k] == t0[k], (k, t0, t1)
    assert s1["lost"] == s1["stuck"] == s1["entry_conflicts"] == 0
    xa, xb = x0.cpu().numpy().astype(np.float64), x1.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(xb, xa, rtol=2e-7, atol=0)
    np.testing.assert_allclose(x2.cpu().numpy(), 2 * x1.cpu().numpy(), rtol=2e-7, atol=0)
    pr, xr, ost, ost2 = U.run_oracle(w.mesh, w.geom, w.mu, w.y.ravel())
    assert s1["crossings"] == ost["crossings"] and s1["rays_hit"] == ost["rays_hit"]
    assert t1["crossings"] == ost2["crossings"]
    fe = U.fwd_errors(p1.cpu().numpy().astype(np.float64), pr, w.mu, w.mesh)
    be = U.back_errors(xb, xr)
    assert fe.max() <= U.FWD_TOL and be.max() <= U.BACK_TOL, (fe.max(), be.max())


def test_plan_host_buffers_and_f64():
    """Host (numpy) inputs and outputs through a plan -- the copy pipeline of
    the plan-less calls -- give the device results; backproject_f64
    accumulates the same sums in double."""
    import torch
    w, tm, mu, y = _setup("c2")
    with tm.plan(w.geom) as pl:
        p_dev = pl.project(mu).cpu().numpy()
        x_dev = pl.backproject(y).cpu().numpy()
        p_host = np.zeros(w.geom.n_rays, np.float32)
        x_host = np.zeros(tm.n_tets, np.float32)
        from paper_1908_06909_b200 import tetproj as T
        T.tet_plan_project(pl.handle, mu.cpu().numpy(), p_host)
        T.tet_plan_backproject(pl.handle, y.cpu().numpy(), x_host)
        acc = pl.backproject_f64(y)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(p_host, p_dev.ravel())
    np.testing.assert_allclose(x_host, x_dev, rtol=2e-7, atol=0)
    np.testing.assert_allclose(acc.cpu().numpy(), x_dev.astype(np.float64), rtol=1e-7, atol=0)


@pytest.mark.parametrize("mode", ["mt_f64", "mt_f32"])
def test_plan_paper_traversal_modes(mode):
    """The paper's Alg. 1/2 walk (TET_TRAVERSE_MT_*) from a plan: bit-identical
    to the plan-less call with the same options."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w, tm, mu, y = _setup("c2")
    opts = T.options(T.TET_TRAVERSE_MT_F64 if mode == "mt_f64" else T.TET_TRAVERSE_MT_F32)
    p0, s0 = tm.project(w.geom, mu, stats=True, opts=opts)
    with tm.plan(w.geom, opts) as pl:
        p1, s1 = pl.project(mu, stats=True)
    torch.cuda.synchronize()
    assert torch.equal(p0, p1)
    for k in ("crossings", "lost", "stuck", "escalations"):
        assert s0[k] == s1[k], (k, s0, s1)


def test_plan_rejects_bad_geometry():
    from paper_1908_06909_b200 import tetproj as T
    w, tm, mu, y = _setup("c2")
    g_inside = G.circular_cone([0.0], 0.5, 8.0, 8, 8, 0.1, 0.1)   # source inside the mesh
    with pytest.raises(T.TetProjError) as e:
        tm.plan(g_inside)
    assert e.value.status == T.TET_E_GEOMETRY
