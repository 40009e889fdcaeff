"""Multi-GPU driver: projection angles sharded over ranks, mesh replicated,
one all-reduce for the backprojection.

"For our multi GPU approach, projections are divided, while keeping the full
mesh in each of the GPUs memories".  The forward projection
needs no communication (each rank owns the rows of its angles); the
backprojection x = A^T y = sum_r A_r^T y_r is the only exchange: one
``all_reduce(SUM)`` over the per-tet vector (NCCL over NVLink/NVSwitch on a
B200 box; gloo in the CPU tests).

The per-rank operators default to the CUDA library (TetMesh.project /
TetMesh.backproject); they are parameters only so the host logic (sharding,
geometry subsetting, reduction) can be exercised on CPU with another
implementation of the same operator.
"""
from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np


@dataclass(frozen=True)
class AngleSharding:
    """Rank r of W owns angles r, r+W, r+2W, ... (interleaved, so angle-
    dependent cost -- e.g. the silhouette of a box -- is balanced)."""
    n_angles: int
    rank: int
    world: int

    def __post_init__(self):
        if not (0 <= self.rank < self.world) or self.n_angles < 1:
            raise ValueError("bad sharding")
        if self.n_angles < self.world:
            # a rank without angles would have no local operator call to make
            # (the library rejects empty scans) and its peers would wait in
            # the all-reduce forever
            raise ValueError(f"{self.n_angles} angles cannot be sharded over {self.world} ranks")

    def local_angles(self) -> np.ndarray:
        return np.arange(self.rank, self.n_angles, self.world)

    def local_geometry(self, geom):
        """Geometry restricted to this rank's angles (same beam / detector)."""
        idx = self.local_angles()
        return SimpleNamespace(beam=geom.beam, n_v=geom.n_v, n_u=geom.n_u,
                               vecs=np.ascontiguousarray(np.asarray(geom.vecs)[idx]),
                               n_angles=len(idx), n_rays=len(idx) * geom.n_v * geom.n_u)

    def local_stack(self, y_full):
        """This rank's rows of a full [A][Nv][Nu] detector stack."""
        return y_full[self.local_angles()]


def _world(group):
    import torch.distributed as dist
    return dist.get_rank(group), dist.get_world_size(group)


def sharding_for(geom, group=None) -> AngleSharding:
    rank, world = _world(group)
    return AngleSharding(geom.n_angles, rank, world)


def local_plan(mesh, geom, group=None, opts=None):
    """A plan (tet_plan_create: geometry + entry map computed once) of this
    rank's angles of the full scan ``geom``, for ``dist_project`` /
    ``dist_backproject(plan=...)`` across iterations."""
    return mesh.plan(sharding_for(geom, group).local_geometry(geom), opts)


def _check_plan(plan, lg):
    g = plan.geom
    if (g.n_angles, g.n_v, g.n_u) != (lg.n_angles, lg.n_v, lg.n_u) or not np.array_equal(
            np.asarray(g.vecs), np.asarray(lg.vecs)):
        raise ValueError("plan is not of this rank's angles (use dist.local_plan)")


def dist_project(mesh, geom, mu, group=None, project=None, plan=None):
    """Forward projection of this rank's angles (no communication).
    Returns (local_proj, sharding).  ``plan``: this rank's ``local_plan``."""
    sh = sharding_for(geom, group)
    lg = sh.local_geometry(geom)
    if plan is not None:
        _check_plan(plan, lg)
        return plan.project(mu), sh
    fn = project if project is not None else mesh.project
    return fn(lg, mu), sh


def tet_shard(n_tets: int, rank: int, world: int):
    """[lo, hi) of the caller-order tets rank `rank` holds after
    ``dist_backproject(..., reduce="scatter")``: contiguous blocks of
    ceil(n_tets / world)."""
    s = -(-n_tets // world)
    lo = min(rank * s, n_tets)
    return lo, min(lo + s, n_tets)


def dist_backproject(mesh, geom, y_local, group=None, backproject=None, async_op=False,
                     precision: str = "f32", plan=None, reduce: str = "all"):
    """x = A^T y over all ranks: local backprojection of this rank's angles,
    then all_reduce(SUM).  ``y_local`` holds this rank's rows
    (``AngleSharding.local_stack``).  Returns the reduced per-tet tensor
    (or (tensor, work) when ``async_op``).

    precision "f32" (default): each rank's tet_backproject result (double
    accumulation on the device, rounded once to float) is summed in float --
    W ranks add at most W * 2^-24 relative (R15).  "f64": each rank
    accumulates into a double tensor (tet_backproject_f64) and the double
    partial sums are reduced; the result stays float64.  ``plan``: this
    rank's ``local_plan`` (the entry map is not recomputed).

    reduce "all" (default): every rank gets the whole x (all_reduce).
    "scatter": for a solver that shards x by tet, each rank
    gets only its block ``tet_shard(n_tets, rank, world)`` of the sum
    (reduce_scatter: half the all-reduce's traffic), zero-padded to
    ceil(n_tets / world) entries."""
    import torch.distributed as dist
    sh = sharding_for(geom, group)
    lg = sh.local_geometry(geom)
    if precision not in ("f32", "f64"):
        raise ValueError(f"precision must be 'f32' or 'f64', not {precision!r}")
    if plan is not None:
        _check_plan(plan, lg)
        x = plan.backproject_f64(y_local) if precision == "f64" else plan.backproject(y_local)
    elif backproject is not None:
        x = backproject(lg, y_local)
    elif precision == "f64":
        x = mesh.backproject_f64(lg, y_local)
    else:
        x = mesh.backproject(lg, y_local)
    if reduce == "scatter":
        import torch
        world = dist.get_world_size(group)
        s = -(-x.numel() // world)
        full = torch.zeros(s * world, dtype=x.dtype, device=x.device)
        full[: x.numel()] = x.reshape(-1)
        x = torch.empty(s, dtype=x.dtype, device=x.device)
        work = dist.reduce_scatter_tensor(x, full, op=dist.ReduceOp.SUM, group=group,
                                          async_op=async_op)
        return (x, work) if async_op else x
    if reduce != "all":
        raise ValueError(f"reduce must be 'all' or 'scatter', not {reduce!r}")
    work = dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    return (x, work) if async_op else x
