"""CUDA path vs the CPU oracle, element by element (GPU only).

Tolerances (BASELINE.json north_star): forward <= 1e-4 relative per pixel,
backprojection <= 1e-4 relative per tet, adjoint <= 1e-5, zero lost/stuck
rays, and -- since both sides take the same exact combinatorial decisions --
identical crossing counts.
"""
import numpy as np
import pytest

from tests import gpu_util as U
from workloads import configs as CF
from workloads import geometry as G
from workloads import meshes as M

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_06909_b200 import tetproj
    tetproj.lib()


def test_c1_full():
    w = CF.workload("c1")
    r = U.check_parity(w.mesh, w.geom, w.mu, w.y, expect_exact_fallbacks=True)
    assert r["stats"]["rays_hit"] == 64


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_small_lattice_degenerate(seed):
    m = M.random_small_mesh(25 + 5 * seed, seed)
    geom = G.lattice_parallel((1 / 8,) * 3, (0, 0, 0), 19, 13, G.LATTICE_DIRS[seed::3][:5])
    rng = np.random.default_rng(seed)
    mu = rng.uniform(0.5, 1.5, m.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    U.check_parity(m, geom, mu, y, expect_exact_fallbacks=True)


def test_small_cone_through_vertices():
    m = M.random_small_mesh(40, 5)
    rows = []
    for th in (0.0, 1.0, 2.5, 4.0):
        S = np.round(np.array([4 * np.sin(th), -4 * np.cos(th), 0.25]) * 16) / 16
        Uv = np.array([0.0625, 0, 0]) if abs(np.cos(th)) > 0.5 else np.array([0, 0.0625, 0])
        V = np.array([0, 0, 0.0625])
        rows.append(np.concatenate([S, -S - 20 * Uv - 17 * V, Uv, V]))
    geom = G.explicit(G.BEAM_CONE, 35, 41, rows)
    rng = np.random.default_rng(0)
    mu = rng.uniform(0.5, 1.5, m.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    U.check_parity(m, geom, mu, y)


def test_c2_ball_ragged():
    w = CF.workload("c2", n_angles=3, n_u=67, n_v=53)
    U.check_parity(w.mesh, w.geom, w.mu, w.y)
    w2 = CF.workload("c2", n_angles=2, n_u=45, n_v=37, mu="uniform")
    U.check_parity(w2.mesh, w2.geom, w2.mu, w2.y)


def test_c3_graded_ragged():
    w = CF.workload("c3", n_angles=3, n_u=61, n_v=47)
    U.check_parity(w.mesh, w.geom, w.mu, w.y)


def test_c4a_sliver_lattice():
    w = CF.workload("c4a", n_angles=6, n_u=72, n_v=40)
    r = U.check_parity(w.mesh, w.geom, w.mu, w.y, expect_exact_fallbacks=True)
    assert r["stats"]["rays_hit"] > 0


def test_c4b_jittered_slivers():
    w = CF.workload("c4b", n_angles=2, n_u=48, n_v=40)
    U.check_parity(w.mesh, w.geom, w.mu, w.y)


def test_wide_cone_generic_frame():
    """Huge pixels: a 16x8 tile's rays spread over >45 degrees, so the block
    vote rejects every fixed shear axis and the generic per-ray frame runs."""
    m = M.ball_mesh(h=0.2, seed=2)
    geom = G.circular_cone(G.equidistant(3) + 0.4, 3.0, 4.5, 24, 20, 0.6, 0.6)
    rng = np.random.default_rng(4)
    mu = rng.uniform(0.2, 1.0, m.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    U.check_parity(m, geom, mu, y)


@pytest.mark.parametrize("beam", ["cone", "parallel"])
def test_many_angles_uniform_frame_chunks(beam):
    """300 angles on a small detector: the walk launches split at 256 angles
    (one block-uniform frame per angle in the launch parameters), and every
    angle's frame -- cone source / parallel shear, per-angle tau -- must give
    the oracle's crossings and values.  Angles are off the axes, so the
    blocks run the fixed-axis variants on the uniform frame."""
    m = M.ball_mesh(h=0.25, seed=3)
    ang = G.equidistant(300) + 0.013
    if beam == "cone":
        geom = G.circular_cone(ang, 3.0, 6.0, 13, 9, 0.4, 0.4, off_u=0.11, off_v=-0.07)
    else:
        geom = G.circular_parallel(ang, 13, 9, 0.19, 0.2, off_u=0.05, off_v=0.03)
    rng = np.random.default_rng(7)
    mu = rng.uniform(0.2, 1.0, m.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    r = U.check_parity(m, geom, mu, y)
    assert r["stats"]["rays_hit"] > geom.n_rays // 4


@pytest.mark.parametrize("finder", ["bvh", "rtree"])
@pytest.mark.parametrize("case", ["c1", "lattice", "c2"])
def test_bvh_entry_finder_identical(case, finder):
    """NEXT-3: the per-ray tree entry finders -- a binary BVH and the paper's
    R*-tree (fan-out 4..10) -- take the same exact
    decisions as the footprint rasteriser: identical projections and crossing
    counts, and parity with the oracle."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    if case == "c1":
        w = CF.workload("c1")
        mesh, geom, mu = w.mesh, w.geom, w.mu
    elif case == "lattice":
        mesh = M.random_small_mesh(40, 2)
        geom = G.lattice_parallel((1 / 8,) * 3, (0, 0, 0), 19, 13, G.LATTICE_DIRS[:6])
        mu = np.random.default_rng(1).uniform(0.5, 1.5, mesh.n_tets).astype(np.float32)
    else:
        w = CF.workload("c2", n_angles=4, n_u=80, n_v=64)
        mesh, geom, mu = w.mesh, w.geom, w.mu
    tm = T.TetMesh.from_mesh(mesh)
    mu_d = torch.from_numpy(mu).cuda()
    a, sa = tm.project(geom, mu_d, stats=True)
    mode = T.TET_ENTRY_BVH if finder == "bvh" else T.TET_ENTRY_RTREE
    b, sb = tm.project(geom, mu_d, stats=True, opts=T.options(entry=mode))
    assert torch.equal(a, b)
    assert sa["crossings"] == sb["crossings"] and sa["rays_hit"] == sb["rays_hit"]
    # and the tree-entry path against the oracle (forward, backward, adjoint)
    y = np.random.default_rng(2).uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    U.check_parity(mesh, geom, mu, y, opts=T.options(entry=mode))


def test_debug_build_bounds_checks():
    """All kernel families on the bounds-checked debug library (device-side
    traps on any out-of-range index); compute-sanitizer is closed on this pool."""
    import os
    import subprocess
    import sys

    from paper_1908_06909_b200 import _build
    _build.build_debug()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TETPROJ_DEBUG_LIB="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize case ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_empty_detector_misses_mesh():
    m = M.ball_mesh(h=0.3, seed=3)
    geom = G.circular_cone([0.0], 4.0, 8.0, 8, 8, 0.1, 0.1, off_u=200.0)
    mu = np.ones(m.n_tets, np.float32)
    y = np.ones(geom.n_rays, np.float32)
    p, x, st, st2, _ = U.run_gpu(m, geom, mu, y)
    assert st["rays_hit"] == 0 and np.all(p == 0) and np.all(x == 0)


def test_single_pixel_and_single_tet():
    m = M.single_tet()
    geom = G.explicit(G.BEAM_PARALLEL, 1, 1, [[1, 0, 0, 0, 0.25, 0.25, 1, 0, 0, 0, 1, 0]])
    p, x, st, st2, _ = U.run_gpu(m, geom, np.array([2.0], np.float32), np.array([3.0], np.float32))
    assert abs(p.ravel()[0] - 1.0) < 1e-6
    assert abs(x[0] - 1.5) < 1e-6                   # chord 0.5 * y 3


def test_host_pointers_and_accumulate():
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=2, n_u=33, n_v=29)
    tm = T.TetMesh.from_mesh(w.mesh)
    p_dev = tm.project(w.geom, torch.from_numpy(w.mu).cuda())
    p_host = np.zeros((w.geom.n_angles, w.geom.n_v, w.geom.n_u), np.float32)
    T.tet_project(tm.handle, w.geom, w.mu, p_host)
    np.testing.assert_array_equal(p_dev.cpu().numpy(), p_host)
    x_host = np.zeros(w.mesh.n_tets, np.float32)
    T.tet_backproject(tm.handle, w.geom, w.y, x_host)
    x2 = x_host.copy()
    T.tet_backproject(tm.handle, w.geom, w.y, x2, accumulate=True)
    np.testing.assert_allclose(x2, 2 * x_host, rtol=1e-6)
    acc = torch.zeros(w.mesh.n_tets, dtype=torch.float64, device="cuda")
    T.tet_backproject_f64(tm.handle, w.geom, torch.from_numpy(w.y.ravel()).cuda(), acc)
    np.testing.assert_allclose(acc.cpu().numpy().astype(np.float32), x_host, rtol=1e-6)


def test_host_pointers_pipelined_chunks():
    """Host buffers over several pipelined chunks (18.4 M rays: 2^22-ray
    chunks by the eighth-of-the-call rule): y / proj move chunk by
    chunk on a copy stream overlapped with tracing; results equal the
    device-pointer call (projections bit-exact, backprojection to f64-sum
    rounding)."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=70, n_u=512, n_v=512)    # 18.4 M rays: 5 chunks
    tm = T.TetMesh.from_mesh(w.mesh)
    p_dev = tm.project(w.geom, torch.from_numpy(w.mu).cuda())
    x_dev = tm.backproject(w.geom, torch.from_numpy(w.y).cuda())
    p_host = torch.empty(p_dev.shape, dtype=torch.float32).pin_memory()
    y_host = torch.from_numpy(w.y).pin_memory()
    x_host = np.zeros(w.mesh.n_tets, np.float32)
    T.tet_project(tm.handle, w.geom, w.mu, p_host.numpy())
    T.tet_backproject(tm.handle, w.geom, y_host.numpy(), x_host)
    np.testing.assert_array_equal(p_dev.cpu().numpy(), p_host.numpy())
    np.testing.assert_allclose(x_host, x_dev.cpu().numpy(), rtol=1e-6, atol=0)


def test_no_reorder_flag_same_result():
    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=2, n_u=31, n_v=27)
    a, xa, *_ = U.run_gpu(w.mesh, w.geom, w.mu, w.y)
    b, xb, *_ = U.run_gpu(w.mesh, w.geom, w.mu, w.y,
                          flags=T.TET_F_FIX_ORIENTATION | T.TET_F_NO_REORDER)
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(xa, xb, rtol=1e-6, atol=1e-7)


def test_errors_are_statuses():
    from paper_1908_06909_b200 import tetproj as T
    m = M.kuhn_cube()
    bad = m.nbrs.copy()
    bad[0, 0] = 5 if bad[0, 0] != 5 else 4
    with pytest.raises(T.TetProjError) as e:
        T.tet_mesh_create(m.verts, m.tets, bad, m.bfaces)
    assert e.value.status == T.TET_E_MESH
    a = M.kuhn_lattice(2)
    keep = [i for i in range(a.n_tets) if i % 7 != 3]
    nb, bf = M.build_graph(a.tets[keep])
    with pytest.raises(T.TetProjError) as e:
        T.tet_mesh_create(a.verts, a.tets[keep], nb, bf)
    assert e.value.status == T.TET_E_MESH            # non-manifold hull
    for make in (M.l_shaped_lattice, M.two_disjoint_tets):
        m = make()
        with pytest.raises(T.TetProjError) as e:
            T.tet_mesh_create(m.verts, m.tets, m.nbrs, m.bfaces)
        assert e.value.status == T.TET_E_NONCONVEX, str(e.value)
    tm = T.TetMesh.from_mesh(M.ball_mesh(h=0.3, seed=3))
    g_inside = G.circular_cone([0.0], 0.5, 8.0, 8, 8, 0.1, 0.1)   # source inside the mesh
    with pytest.raises(T.TetProjError) as e:
        tm.project(g_inside, np.ones(tm.n_tets, np.float32))
    assert e.value.status == T.TET_E_GEOMETRY


def test_full_size_c3_sampled():
    """BASELINE config c3 at full size, in bench.py's launch configuration:
    sampled rays vs the oracle one by one; backprojection via the adjoint and
    the total-sum identity sum_t (A^T 1)_t = sum_j (A 1)_j."""
    import torch

    from oracle import tetref as O
    w = CF.workload("c3")
    p, x, st, st2, tm = U.run_gpu(w.mesh, w.geom, w.mu, w.y)
    assert st["lost"] == st["stuck"] == st["entry_conflicts"] == 0
    assert st2["lost"] == st2["stuck"] == 0
    rng = np.random.default_rng(7)
    ids = np.sort(rng.choice(w.geom.n_rays, 3000, replace=False))
    om = O.OracleMesh.from_mesh(w.mesh)
    pr, _ = O.project(om, w.geom, w.mu.astype(np.float64), ray_ids=ids)
    fe = U.fwd_errors(p.ravel()[ids].astype(np.float64), pr, w.mu, w.mesh)
    assert fe.max() <= U.FWD_TOL
    lhs = float(np.dot(p.astype(np.float64).ravel(), w.y.astype(np.float64).ravel()))
    rhs = float(np.dot(w.mu.astype(np.float64), x.astype(np.float64)))
    assert abs(lhs - rhs) / abs(lhs) <= U.ADJ_TOL
    ones_t = torch.ones(w.mesh.n_tets, device="cuda")
    ones_r = torch.ones(w.geom.n_rays, device="cuda")
    rowsum = tm.project(w.geom, ones_t).double().sum().item()
    colsum = tm.backproject(w.geom, ones_r).double().sum().item()
    assert abs(rowsum - colsum) / rowsum <= U.ADJ_TOL


def _sampled_backprojection_check(tm, geom, mesh, om, ids, min_nonzero=1000):
    """Backprojection per tet at full size: y = 1 + (ray id mod 7) on the
    sampled rays and 0 elsewhere, so the oracle computes every tet's exact
    value from those rays alone (oracle backproject with ray_ids)."""
    import torch

    from oracle import tetref as O
    y = np.zeros(geom.n_rays, np.float32)
    y[ids] = 1.0 + (ids % 7).astype(np.float32)
    x = tm.backproject(geom, torch.from_numpy(y).cuda()).cpu().numpy().astype(np.float64)
    xr, _ = O.backproject(om, geom, y[ids], ray_ids=ids)
    assert np.count_nonzero(xr) > min_nonzero
    be = U.back_errors(x, xr)
    assert be.max() <= U.BACK_TOL, (be.max(), int(be.argmax()))


def test_full_size_c3_sampled_backprojection():
    """c3 at full size: every tet's backprojection of 3000 sampled rays."""
    from oracle import tetref as O
    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c3")
    tm = T.TetMesh.from_mesh(w.mesh)
    om = O.OracleMesh.from_mesh(w.mesh)
    ids = np.sort(np.random.default_rng(11).choice(w.geom.n_rays, 3000, replace=False))
    _sampled_backprojection_check(tm, w.geom, w.mesh, om, ids)


@pytest.mark.parametrize("cfg", ["c2", "c4a", "c4b"])
def test_full_size_sampled(cfg):
    """The other BASELINE configs at full size (c2 256^2 x 90, c4a 512^2 x 16
    lattice directions, c4b 512^2 x 32 with sources on lattice points), in
    bench.py's launch configuration: zero lost / stuck rays and zero entry
    conflicts over every ray (the c4 bar: "zero lost rays on sliver
    meshes"), 2000 sampled rays' projections against the oracle one by one,
    every tet's backprojection of those rays, and the adjoint identity."""
    from oracle import tetref as O
    w = CF.workload(cfg)
    p, x, st, st2, tm = U.run_gpu(w.mesh, w.geom, w.mu, w.y)
    assert st["lost"] == st["stuck"] == st["entry_conflicts"] == 0, st
    assert st2["lost"] == st2["stuck"] == 0, st2
    assert st["crossings"] == st2["crossings"] and st["rays_hit"] > 0
    om = O.OracleMesh.from_mesh(w.mesh)
    rng = np.random.default_rng(17)
    hit = np.flatnonzero(p.ravel() != 0)
    ids = np.sort(np.concatenate([rng.choice(w.geom.n_rays, 1000, replace=False),
                                  rng.choice(hit, 1000, replace=False)]))
    ids = np.unique(ids)
    pr, ost = O.project(om, w.geom, w.mu.astype(np.float64), ray_ids=ids)
    assert ost["lost"] == ost["stuck"] == 0
    fe = U.fwd_errors(p.ravel()[ids].astype(np.float64), pr, w.mu, w.mesh)
    assert fe.max() <= U.FWD_TOL, (fe.max(), int(ids[fe.argmax()]))
    lhs = float(np.dot(p.astype(np.float64).ravel(), w.y.astype(np.float64).ravel()))
    rhs = float(np.dot(w.mu.astype(np.float64), x.astype(np.float64)))
    assert abs(lhs - rhs) / abs(lhs) <= U.ADJ_TOL
    _sampled_backprojection_check(tm, w.geom, w.mesh, om, ids, min_nonzero=300)


def test_full_size_c5_mesh_sampled():
    """BASELINE config c5's 10.5 M-tet mesh at its full 1024^2 detector (8 of
    the 720 angles, evenly spaced -- the per-GPU work is angle-sharded): 2000
    sampled rays' projections one by one, every tet's backprojection of those
    rays, zero lost / stuck rays."""
    import torch

    from oracle import tetref as O
    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c5")
    geom = w.geom.subset(np.arange(0, w.geom.n_angles, w.geom.n_angles // 8))
    tm = T.TetMesh.from_mesh(w.mesh)
    p, st = tm.project(geom, torch.from_numpy(w.mu).cuda(), stats=True)
    assert st["lost"] == st["stuck"] == st["entry_conflicts"] == 0, st
    om = O.OracleMesh.from_mesh(w.mesh)
    ids = np.sort(np.random.default_rng(5).choice(geom.n_rays, 2000, replace=False))
    pr, ost = O.project(om, geom, w.mu.astype(np.float64), ray_ids=ids)
    fe = U.fwd_errors(p.cpu().numpy().ravel()[ids].astype(np.float64), pr, w.mu, w.mesh)
    assert fe.max() <= U.FWD_TOL, fe.max()
    _sampled_backprojection_check(tm, geom, w.mesh, om, ids)


def _mt_case(case):
    if case == "c2":                          # generic rays: no degeneracy
        w = CF.workload("c2", n_angles=2, n_u=64, n_v=48)
        return w.mesh, w.geom, w.mu, w.y.ravel()
    if case == "slivers":                     # fig:singledouble: Delaunay slivers
        m = M.jittered_lattice_mesh(12, 1e-4, 5)
        R = np.sqrt(3.0)
        geom = G.circular_cone(G.equidistant(4) + 0.1, 4 * R, 8 * R, 48, 48, 7.2 / 48, 7.2 / 48)
    else:                                     # fig:bad: lattice rays through vertices
        m = M.kuhn_lattice(4)
        geom = G.lattice_parallel((0.25,) * 3, (0, 0, 0), 11, 11, G.LATTICE_DIRS)
    rng = np.random.default_rng(3)
    mu = rng.uniform(0.5, 1.5, m.n_tets).astype(np.float32)
    y = rng.uniform(0.5, 1.5, geom.n_rays).astype(np.float32)
    return m, geom, mu, y


@pytest.mark.parametrize("case", ["c2", "slivers", "lattice"])
@pytest.mark.parametrize("single", [False, True])
def test_paper_mt_modes_match_mt_oracle(case, single):
    """NEXT-1: the paper's Alg. 1/2 walker (mt_trace_kernel) against the MT
    oracle (oracle/tetref_mt.inc), both IEEE operation for operation in the
    same precision: identical projections (bit for bit), identical crossing,
    lost, stuck and escalation counts -- including the rays the paper's
    method fails on (fp32 slivers, lattice rays) -- and the backprojection
    per tet within 1e-4 (atomic summation order)."""
    import torch

    from oracle import tetref as O
    from paper_1908_06909_b200 import tetproj as T
    mesh, geom, mu, y = _mt_case(case)
    tm = T.TetMesh.from_mesh(mesh)
    mode = T.TET_TRAVERSE_MT_F32 if single else T.TET_TRAVERSE_MT_F64
    p, st = tm.project(geom, torch.from_numpy(mu).cuda(), stats=True, opts=T.options(mode))
    x, stb = tm.backproject(geom, torch.from_numpy(y).cuda(), stats=True, opts=T.options(mode))
    om = O.OracleMesh.from_mesh(mesh)
    q, ost = O.mt_project(om, geom, mu.astype(np.float64), single=single)
    xr, ost2 = O.mt_backproject(om, geom, y.astype(np.float64), single=single)
    for k in ("rays_hit", "crossings", "lost", "stuck", "escalations"):
        assert st[k] == ost[k], (k, st, ost)
        assert stb[k] == ost2[k], (k, stb, ost2)
    np.testing.assert_array_equal(p.cpu().numpy().ravel(), q.astype(np.float32).ravel())
    be = U.back_errors(x.cpu().numpy().astype(np.float64), xr)
    assert be.max() <= U.BACK_TOL, be.max()


def test_kernel_times_are_busy_time():
    """tet_kernel_times reports the busy time of each kernel class (union of
    launch intervals): with a call's angle chunks alternating between two
    streams, the forward busy time never exceeds the call's own duration,
    and both chunks' launches are counted."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=300, n_u=40, n_v=32)      # 2 chunks (256 + 44)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    proj = torch.empty((w.geom.n_angles, w.geom.n_v, w.geom.n_u), device="cuda")
    T.tet_project(tm.handle, w.geom, mu, proj)               # warm
    torch.cuda.synchronize()
    T.tet_set_kernel_timing(tm.handle, True)
    T.tet_kernel_times(tm.handle)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    T.tet_project(tm.handle, w.geom, mu, proj)
    b.record()
    torch.cuda.synchronize()
    T.tet_set_kernel_timing(tm.handle, False)
    kt = T.tet_kernel_times(tm.handle)
    call_ms = a.elapsed_time(b)
    ms_f, n_f = kt["forward"]
    ms_e, n_e = kt["entry"]
    assert n_f == 2 and n_e == 2, kt
    assert 0 < ms_f <= call_ms * 1.001 + 0.01, (kt, call_ms)
    assert 0 < ms_e <= call_ms * 1.001 + 0.01, (kt, call_ms)


def test_exact_heavy_walk_shape_same_results():
    """A call whose statistics show > 5 % exact fallbacks per crossing makes the
    mesh's next calls run the exact-heavy walk shape (more registers, early
    gathers).  Same arithmetic: projections bit-identical, backprojections
    equal up to the order of the f64 atomic sums."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c4a", n_angles=4, n_u=64, n_v=40)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    y = torch.from_numpy(w.y.reshape(-1)).cuda()
    shape = (w.geom.n_angles, w.geom.n_v, w.geom.n_u)
    p0 = torch.empty(shape, device="cuda")
    x0 = torch.empty(w.mesh.n_tets, device="cuda")
    st = T.tet_project(tm.handle, w.geom, mu, p0, stats=True)    # fast shape; learns
    assert st["exact_fallbacks"] * 20 > st["crossings"], st
    T.tet_backproject(tm.handle, w.geom, y, x0)                   # exact-heavy shape
    p1 = torch.empty(shape, device="cuda")
    T.tet_project(tm.handle, w.geom, mu, p1)                      # exact-heavy shape
    torch.cuda.synchronize()
    assert torch.equal(p0, p1)
    # back to the fast shape: a call with statistics on generic rays
    w2 = CF.workload("c2", n_angles=2, n_u=33, n_v=29)
    tm2 = T.TetMesh.from_mesh(w2.mesh)
    x_fast = tm2.backproject(w2.geom, torch.from_numpy(w2.y).cuda())
    st2 = T.tet_project(tm2.handle, w2.geom, torch.from_numpy(w2.mu).cuda(),
                        torch.empty((2, 29, 33), device="cuda"), stats=True)
    assert st2["exact_fallbacks"] * 20 < st2["crossings"]
    x_again = tm2.backproject(w2.geom, torch.from_numpy(w2.y).cuda())
    torch.cuda.synchronize()
    np.testing.assert_allclose(x_again.cpu().numpy(), x_fast.cpu().numpy(), rtol=1e-6)
    # and the exact-heavy backward against the oracle
    _, xr, _, _ = U.run_oracle(w.mesh, w.geom, w.mu, w.y)
    be = U.back_errors(x0.cpu().numpy().astype(np.float64), xr)
    assert be.max() <= U.BACK_TOL, be.max()


def test_mesh_features_walk_selection():
    """The benchmark configs run the FT16 walk (16-B tags with apex
    coordinates) and carry both tree entry structures; TETPROJ_WALKER=rec
    (read at create) selects the record walk, with identical results."""
    import os

    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=2, n_u=48, n_v=40)
    tm = T.TetMesh.from_mesh(w.mesh)
    f = T.tet_mesh_features(tm.handle)
    assert f["walk"] == "ft16" and f["tag16_bytes"] == 64 * w.mesh.n_tets
    assert f["rtree_nodes"] > 0 and f["bvh_nodes"] > 0
    os.environ["TETPROJ_WALKER"] = "rec"
    try:
        tr = T.TetMesh.from_mesh(w.mesh)
    finally:
        del os.environ["TETPROJ_WALKER"]
    assert T.tet_mesh_features(tr.handle)["walk"] == "rec"
    mu = torch.from_numpy(w.mu).cuda()
    a, sa = tm.project(w.geom, mu, stats=True)
    b, sb = tr.project(w.geom, mu, stats=True)
    assert sa["crossings"] == sb["crossings"]
    np.testing.assert_allclose(a.cpu().numpy(), b.cpu().numpy(), rtol=1e-6, atol=1e-7)


def test_strict_flag_reports_failed_rays():
    """TET_F_STRICT: a call whose statistics show lost or stuck rays fails with
    TET_E_RAYS (header contract).  The exact walk never produces one; the
    paper's fp32 traversal on slivers does (fig:singledouble)."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    mesh, geom, mu, y = _mt_case("slivers")
    tm = T.TetMesh.from_mesh(mesh, flags=T.TET_F_FIX_ORIENTATION | T.TET_F_STRICT)
    mu_d = torch.from_numpy(mu).cuda()
    p, st = tm.project(geom, mu_d, stats=True)                 # exact: passes
    assert st["lost"] == st["stuck"] == 0
    with pytest.raises(T.TetProjError) as e:
        tm.project(geom, mu_d, opts=T.options(T.TET_TRAVERSE_MT_F32))
    assert e.value.status == T.TET_E_RAYS


def test_backproject_accumulate_device():
    """x += A^T y on device pointers: two accumulating calls give twice the
    backprojection, and match the oracle."""
    import torch

    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2", n_angles=2, n_u=40, n_v=32)
    tm = T.TetMesh.from_mesh(w.mesh)
    yd = torch.from_numpy(w.y).cuda()
    x = torch.zeros(w.mesh.n_tets, device="cuda")
    T.tet_backproject(tm.handle, w.geom, yd, x, accumulate=True)
    T.tet_backproject(tm.handle, w.geom, yd, x, accumulate=True)
    torch.cuda.synchronize()
    _, xr, _, _ = U.run_oracle(w.mesh, w.geom, w.mu, w.y)
    be = U.back_errors(x.cpu().numpy().astype(np.float64) / 2, xr)
    assert be.max() <= U.BACK_TOL, be.max()


def test_large_single_angle_detector_sampled():
    """Maximum-size edge case: ONE angle of a 4099 x 4097 detector (16.8 M
    rays in a single angle chunk: the largest grid of one walk launch, ragged
    in both directions), through a plan; sampled rays vs the oracle one by
    one, every tet's backprojection of the sampled rays, and the total-sum
    identity."""
    import torch

    from oracle import tetref as O
    from paper_1908_06909_b200 import tetproj as T
    w = CF.workload("c2")
    R = 1.0
    geom = G.circular_cone([0.37], 4 * R, 8 * R, 4099, 4097, 4.6 * R / 4099, 4.6 * R / 4097)
    tm = T.TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    with tm.plan(geom) as pl:
        p, st = pl.project(mu, stats=True)
        ones_r = torch.ones(geom.n_rays, device="cuda")
        colsum = pl.backproject(ones_r).double().sum().item()
        rowsum = pl.project(torch.ones_like(mu)).double().sum().item()
    assert st["rays"] == geom.n_rays and st["lost"] == st["stuck"] == st["entry_conflicts"] == 0
    assert st["rays_hit"] > 0.5 * geom.n_rays
    assert abs(rowsum - colsum) / rowsum <= U.ADJ_TOL
    rng = np.random.default_rng(11)
    ids = np.sort(rng.choice(geom.n_rays, 2000, replace=False))
    om = O.OracleMesh.from_mesh(w.mesh)
    pr, _ = O.project(om, geom, w.mu.astype(np.float64), ray_ids=ids)
    fe = U.fwd_errors(p.cpu().numpy().ravel()[ids].astype(np.float64), pr, w.mu, w.mesh)
    assert fe.max() <= U.FWD_TOL
    _sampled_backprojection_check(tm, geom, w.mesh, om, ids, min_nonzero=500)
