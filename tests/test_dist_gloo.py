"""Multi-rank host logic on CPU: world_size-2 gloo processes shard the angles,
backproject their shard and all-reduce; the result must equal the
single-process backprojection (oracle used as the per-rank operator)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_06909_b200.dist import AngleSharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tetref as O
        from paper_1908_06909_b200 import dist as D
        from workloads import configs as CF
        w = CF.workload("c1")
        om = O.OracleMesh.from_mesh(w.mesh)

        def backproject(geom, y):
            x, st = O.backproject(om, geom, np.asarray(y).ravel())
            assert st["lost"] == 0
            return torch.from_numpy(x)

        def project(geom, mu):
            p, _ = O.project(om, geom, mu)
            return torch.from_numpy(p)

        sh = D.sharding_for(w.geom)
        y_local = sh.local_stack(w.y)
        x = D.dist_backproject(None, w.geom, y_local, backproject=backproject)
        # reduce-scatter: this rank's contiguous block of the same sum
        xs = D.dist_backproject(None, w.geom, y_local, backproject=backproject, reduce="scatter")
        lo, hi = D.tet_shard(x.numel(), rank, world)
        assert xs.numel() == -(-x.numel() // world)
        assert torch.allclose(xs[: hi - lo], x[lo:hi], rtol=1e-12, atol=1e-12)
        assert not xs[hi - lo:].any()
        p_local, sh2 = D.dist_project(None, w.geom, w.mu.astype(np.float64), project=project)
        # gather the forward stack to rank 0 for checking
        parts = [torch.zeros((len(AngleSharding(w.geom.n_angles, r, world).local_angles()),
                              w.geom.n_v, w.geom.n_u), dtype=torch.float64) for r in range(world)]
        dist.all_gather(parts, p_local)   # c1: 4 angles -> 2 per rank
        if rank == 0:
            np.savez(out_path, x=x.numpy(), **{f"p{r}": parts[r].numpy() for r in range(world)})
    finally:
        dist.destroy_process_group()


def test_sharding_partitions_angles():
    for n, w in [(4, 2), (360, 8), (7, 3), (1, 1), (8, 8), (41, 2)]:
        got = np.sort(np.concatenate([AngleSharding(n, r, w).local_angles() for r in range(w)]))
        np.testing.assert_array_equal(got, np.arange(n))
    # fewer angles than ranks: an empty rank would leave its peers waiting in
    # the all-reduce, so the sharding refuses it up front
    with pytest.raises(ValueError):
        AngleSharding(5, 0, 8)


def test_gloo_two_ranks_backprojection_allreduce(tmp_path):
    from oracle import tetref as O
    from workloads import configs as CF
    O.build()
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    w = CF.workload("c1")
    om = O.OracleMesh.from_mesh(w.mesh)
    x_ref, _ = O.backproject(om, w.geom, w.y.ravel())
    np.testing.assert_allclose(r["x"], x_ref, rtol=1e-12, atol=1e-12)
    p_ref, _ = O.project(om, w.geom, w.mu.astype(np.float64))
    for rank in range(2):
        idx = AngleSharding(w.geom.n_angles, rank, 2).local_angles()
        np.testing.assert_allclose(r[f"p{rank}"], p_ref[idx], rtol=1e-12, atol=1e-12)
