"""NEXT-2 solvers: OS-SART and CGLS (CPU with oracle operators; the GPU
variants run the same code on the CUDA operators)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_06909_b200 import solvers as S
from workloads import geometry as G
from workloads import meshes as M


def _problem(n_angles=24):
    mesh = M.random_small_mesh(30, 11)
    geom = G.circular_cone(G.equidistant(n_angles), 4.0, 8.0, 12, 12, 0.3, 0.3)
    rng = np.random.default_rng(3)
    mu = rng.uniform(0.2, 1.0, mesh.n_tets)
    return mesh, geom, mu


def _oracle_ops(mesh):
    from oracle import tetref as O
    om = O.OracleMesh.from_mesh(mesh)

    def project(g, x):
        p, st = O.project(om, g, x.numpy())
        assert st["lost"] == 0
        return torch.from_numpy(p)

    def backproject(g, y):
        x, _ = O.backproject(om, g, y.numpy().ravel())
        return torch.from_numpy(x)
    return project, backproject


def test_cgls_residual_decreases_and_recovers_known_mesh():
    mesh, geom, mu = _problem()
    P, B = _oracle_ops(mesh)
    b = P(geom, torch.from_numpy(mu))
    res = []
    x = S.cgls(P, B, geom, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=60,
               callback=lambda it, x, r: res.append(float(r.norm())))
    assert all(res[i + 1] <= res[i] * (1 + 1e-9) for i in range(len(res) - 1))
    assert res[-1] < 1e-2 * float(b.norm())
    # tets crossed by many rays are recovered (the known-mesh case of fig:rec (a))
    colsum = B(geom, torch.ones_like(b)).numpy()
    well = colsum > np.percentile(colsum, 50)
    assert np.median(np.abs(x.numpy()[well] - mu[well]) / mu[well]) < 0.1


def test_os_sart_reduces_error():
    mesh, geom, mu = _problem()
    P, B = _oracle_ops(mesh)
    b = P(geom, torch.from_numpy(mu))
    errs = []
    S.os_sart(P, B, geom, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=20, block=6,
              callback=lambda it, x: errs.append(float((P(geom, x) - b).norm())))
    assert errs[-1] < 0.1 * errs[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1908_06909_b200.dist import AngleSharding
        mesh, geom, mu = _problem()
        P, B = _oracle_ops(mesh)
        sh = AngleSharding(geom.n_angles, rank, world)
        g = sh.local_geometry(geom)
        b = P(g, torch.from_numpy(mu))
        x = S.cgls(P, B, g, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=15,
                   group=dist.group.WORLD)
        x2 = S.os_sart(P, B, g, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=3,
                       block=3, group=dist.group.WORLD)
        # uneven split (25 angles: 13 + 12) with subsets of the global scan:
        # both ranks must issue the same number of reductions (9 subsets)
        mesh25, geom25, mu25 = _problem(25)
        g25 = AngleSharding(25, rank, world).local_geometry(geom25)
        b25 = P(g25, torch.from_numpy(mu25))
        x3 = S.os_sart(P, B, g25, b25, torch.zeros(mesh25.n_tets, dtype=torch.float64), n_iter=3,
                       block=3, group=dist.group.WORLD)
        # more subsets than a rank has angles: empty subsets still join
        x4 = S.os_sart(P, B, g25, b25, torch.zeros(mesh25.n_tets, dtype=torch.float64), n_iter=2,
                       block=1, group=dist.group.WORLD)
        if rank == 0:
            np.savez(out, x=x.numpy(), x2=x2.numpy(), x3=x3.numpy(), x4=x4.numpy())
    finally:
        dist.destroy_process_group()


def test_distributed_cgls_matches_single_process(tmp_path):
    mesh, geom, mu = _problem()
    P, B = _oracle_ops(mesh)
    b = P(geom, torch.from_numpy(mu))
    x_ref = S.cgls(P, B, geom, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=15)
    out = str(tmp_path / "x.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    # CGLS is invariant to the row order of A: sharded == single process up
    # to the summation order of the reductions (amplified over 15 iterations)
    np.testing.assert_allclose(r["x"], x_ref.numpy(), rtol=1e-5, atol=1e-7)
    # OS-SART over the global subsets: sharded == single process
    x2_ref = S.os_sart(P, B, geom, b, torch.zeros(mesh.n_tets, dtype=torch.float64), n_iter=3,
                       block=3)
    np.testing.assert_allclose(r["x2"], x2_ref.numpy(), rtol=1e-9, atol=1e-12)
    mesh25, geom25, mu25 = _problem(25)
    b25 = P(geom25, torch.from_numpy(mu25))
    for key, it, blk in (("x3", 3, 3), ("x4", 2, 1)):
        ref = S.os_sart(P, B, geom25, b25, torch.zeros(mesh25.n_tets, dtype=torch.float64),
                        n_iter=it, block=blk)
        np.testing.assert_allclose(r[key], ref.numpy(), rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("ops", ["calls", "plans"])
def test_gpu_os_sart_known_mesh(ops):
    """OS-SART on the CUDA operators, the paper's known-mesh setting
    (fig:rec (a)): data simulated on the same mesh, 50 iterations, blocks of 20
    -- through the plain calls and through one plan per subset."""
    from paper_1908_06909_b200 import TetMesh
    from paper_1908_06909_b200.tetproj import PlannedOperators
    from workloads import configs as CF
    w = CF.workload("c2", n_angles=40, n_u=64, n_v=64)
    tm = TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    b = tm.project(w.geom, mu)
    res = []
    with PlannedOperators(tm) as po:
        P, B = ((lambda g, x: tm.project(g, x), lambda g, y: tm.backproject(g, y))
                if ops == "calls" else (po.project, po.backproject))
        x = S.os_sart(P, B, w.geom, b, torch.zeros_like(mu), n_iter=50, block=20,
                      callback=lambda it, x: res.append(float((tm.project(w.geom, x) - b).norm())))
        if ops == "plans":
            assert len(po.plans) == 2          # 40 angles in blocks of 20: one plan per subset
    assert res[-1] < 0.05 * float(b.norm())
    assert res[-1] < res[0]


@pytest.mark.gpu
@pytest.mark.parametrize("ops", ["calls", "plans"])
def test_gpu_solvers_match_oracle_operators(ops):
    """NEXT-2 parity: the same solver code on the CUDA operators and on the
    oracle operators, from the same data b, gives the same iterates -- every
    one of the first 5 CGLS and OS-SART iterates within 1e-4 (relative 2-norm)
    -- so the reconstruction path inherits the operator parity."""
    from paper_1908_06909_b200 import TetMesh
    mesh, geom, mu = _problem()
    P, B = _oracle_ops(mesh)
    tm = TetMesh.from_mesh(mesh)
    PG = lambda g, x: tm.project(g, x)          # noqa: E731
    BG = lambda g, y: tm.backproject(g, y)      # noqa: E731
    if ops == "plans":
        from paper_1908_06909_b200.tetproj import PlannedOperators
        po = PlannedOperators(tm)
        PG, BG = po.project, po.backproject
    b64 = P(geom, torch.from_numpy(mu))
    b32 = b64.float().cuda()
    z64 = torch.zeros(mesh.n_tets, dtype=torch.float64)
    z32 = torch.zeros(mesh.n_tets, dtype=torch.float32, device="cuda")
    for name, run in (("cgls", lambda Pp, Bb, b, z, cb: S.cgls(Pp, Bb, geom, b, z, n_iter=5,
                                                               callback=lambda it, x, r: cb(x))),
                      ("os_sart", lambda Pp, Bb, b, z, cb: S.os_sart(Pp, Bb, geom, b, z, n_iter=5,
                                                                     block=6,
                                                                     callback=lambda it, x: cb(x)))):
        xo, xg = [], []
        run(P, B, b64, z64, lambda x: xo.append(x.numpy().copy()))
        run(PG, BG, b32, z32, lambda x: xg.append(x.double().cpu().numpy()))
        assert len(xo) == len(xg) == 5, name
        for it, (a, g) in enumerate(zip(xo, xg)):
            rel = np.linalg.norm(g - a) / np.linalg.norm(a)
            assert rel <= 1e-4, (name, it, rel)
