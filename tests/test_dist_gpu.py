"""Multi-rank path on the GPU (a7, NEXT-2): two processes run the CUDA
operators on their angle shards and reduce the backprojection -- NCCL when
two GPUs exist, otherwise gloo with both ranks on cuda:0 (a logic check of
the sharded path; the reduction is the same call) -- and the result is
compared with the CPU oracle on the whole scan ("projections
are divided, while keeping the full mesh in each of the GPUs memories")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import gpu_util as U

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    ndev = torch.cuda.device_count()
    dev = rank % ndev
    torch.cuda.set_device(dev)
    if ndev >= world:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return dev


def _dist_worker(rank, world, port, out):
    dev = _init(rank, world, port)
    try:
        from paper_1908_06909_b200 import TetMesh
        from paper_1908_06909_b200 import dist as D
        from workloads import configs as CF
        w = CF.workload("c2", n_angles=5, n_u=61, n_v=47)        # 3 + 2 angles
        tm = TetMesh.from_mesh(w.mesh, device=dev)
        sh = D.sharding_for(w.geom)
        y_local = torch.from_numpy(np.ascontiguousarray(sh.local_stack(w.y))).cuda(dev)
        x = D.dist_backproject(tm, w.geom, y_local)
        x64 = D.dist_backproject(tm, w.geom, y_local, precision="f64")
        p_local, _ = D.dist_project(tm, w.geom, torch.from_numpy(w.mu).cuda(dev))
        with D.local_plan(tm, w.geom) as pl:     # the same through this rank's plan
            xp = D.dist_backproject(tm, w.geom, y_local, plan=pl)
            xp64 = D.dist_backproject(tm, w.geom, y_local, precision="f64", plan=pl)
            pp, _ = D.dist_project(tm, w.geom, torch.from_numpy(w.mu).cuda(dev), plan=pl)
            torch.cuda.synchronize()
        xs = D.dist_backproject(tm, w.geom, y_local, reduce="scatter")   # this rank's tet block
        lo, hi = D.tet_shard(tm.n_tets, rank, world)
        torch.cuda.synchronize()
        res = {"x": x.cpu().numpy(), "x64": x64.cpu().numpy(),
               "p": p_local.cpu().numpy(), "backend": dist.get_backend(),
               "xp": xp.cpu().numpy(), "xp64": xp64.cpu().numpy(), "pp": pp.cpu().numpy(),
               "xs": xs.cpu().numpy(), "lo": lo, "hi": hi}
        np.savez(f"{out}.{rank}.npz", **res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_cuda_operators_match_oracle(tmp_path):
    from workloads import configs as CF
    from paper_1908_06909_b200.dist import AngleSharding
    out = str(tmp_path / "r")
    mp.spawn(_dist_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    w = CF.workload("c2", n_angles=5, n_u=61, n_v=47)
    pr, xr, ost, _ = U.run_oracle(w.mesh, w.geom, w.mu, w.y)
    for rank in range(2):
        r = np.load(f"{out}.{rank}.npz")
        # every rank holds the reduced x = A^T y of the WHOLE scan
        be = U.back_errors(r["x"].astype(np.float64), xr)
        assert be.max() <= U.BACK_TOL, be.max()
        be64 = U.back_errors(r["x64"], xr)
        assert be64.max() <= U.BACK_TOL, be64.max()
        # and the forward rows of its own angles
        idx = AngleSharding(w.geom.n_angles, rank, 2).local_angles()
        fe = U.fwd_errors(r["p"].astype(np.float64), pr[idx], w.mu, w.mesh)
        assert fe.max() <= U.FWD_TOL, fe.max()
        # through the rank's plan: the same projection bits, the same sums
        np.testing.assert_array_equal(r["pp"], r["p"])
        np.testing.assert_allclose(r["xp"], r["x"], rtol=1e-6, atol=0)
        np.testing.assert_allclose(r["xp64"], r["x64"], rtol=1e-12, atol=0)
        # reduce-scatter: the rank's block of the same reduced sum
        lo, hi = int(r["lo"]), int(r["hi"])
        np.testing.assert_allclose(r["xs"][: hi - lo], r["x"][lo:hi], rtol=1e-6, atol=0)


def _cgls_worker(rank, world, port, out):
    dev = _init(rank, world, port)
    try:
        from paper_1908_06909_b200 import TetMesh
        from paper_1908_06909_b200 import solvers as S
        from paper_1908_06909_b200.dist import AngleSharding
        from workloads import configs as CF
        w = CF.workload("c2", n_angles=9, n_u=40, n_v=36)
        tm = TetMesh.from_mesh(w.mesh, device=dev)
        g = AngleSharding(w.geom.n_angles, rank, world).local_geometry(w.geom)
        mu = torch.from_numpy(w.mu).cuda(dev)
        b = tm.project(g, mu)
        x = S.cgls(lambda gg, v: tm.project(gg, v), lambda gg, yy: tm.backproject(gg, yy), g, b,
                   torch.zeros_like(mu), n_iter=6, group=dist.group.WORLD)
        torch.cuda.synchronize()
        np.save(f"{out}.{rank}.npy", x.cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gpu_cgls_matches_one_rank(tmp_path):
    """NEXT-2 on 2 ranks: CGLS with the angles sharded and A^T r / ||A p||^2
    all-reduced equals the single-process CGLS on the whole scan (CGLS does
    not depend on the row order of A) up to float rounding."""
    from paper_1908_06909_b200 import TetMesh
    from paper_1908_06909_b200 import solvers as S
    from workloads import configs as CF
    out = str(tmp_path / "c")
    mp.spawn(_cgls_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    w = CF.workload("c2", n_angles=9, n_u=40, n_v=36)
    tm = TetMesh.from_mesh(w.mesh)
    mu = torch.from_numpy(w.mu).cuda()
    b = tm.project(w.geom, mu)
    x1 = S.cgls(lambda gg, v: tm.project(gg, v), lambda gg, yy: tm.backproject(gg, yy), w.geom, b,
                torch.zeros_like(mu), n_iter=6).cpu().numpy().astype(np.float64)
    for rank in range(2):
        x2 = np.load(f"{out}.{rank}.npy").astype(np.float64)
        assert np.linalg.norm(x2 - x1) <= 1e-4 * np.linalg.norm(x1)
