"""Iterative reconstruction on top of the operators.

"All algorithms require the computation of Ax (the projection operation) and
A^T b (the backprojection operations)"; the paper reconstructs
with OS-SART, "50 iterations with blocks of 20 projections".

Both solvers take the operators as callables so they run unchanged on one GPU
(``TetMesh.project`` / ``TetMesh.backproject``), on several GPUs (angles
sharded per rank; backprojections and inner products all-reduced over the
process group) and, in the CPU tests, on the oracle.  Vectors are torch
tensors on the operators' device; all arithmetic runs there.

    project(geom, x)      -> proj [A_geom, Nv, Nu]
    backproject(geom, y)  -> x    [T]
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np


def _subset(geom, idx):
    idx = np.asarray(idx)
    return SimpleNamespace(beam=geom.beam, n_v=geom.n_v, n_u=geom.n_u,
                           vecs=np.ascontiguousarray(np.asarray(geom.vecs)[idx]),
                           n_angles=len(idx), n_rays=len(idx) * geom.n_v * geom.n_u)


def _allreduce(t, group):
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def _global_angle_ids(n_local, group, angle_ids):
    """Global indices of this rank's angles and the global angle count.  With
    a process group and no explicit ids, the interleaved AngleSharding layout
    (rank r of W owns r, r+W, ...) is assumed; the count is all-reduced."""
    import torch
    if angle_ids is not None:
        ids = np.asarray(angle_ids, dtype=np.int64)
        if group is None:
            return ids, int(ids.max()) + 1 if ids.size else 0
    if group is None:
        return np.arange(n_local), n_local
    import torch.distributed as dist
    n = torch.tensor([n_local], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        n = n.cuda()
    dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
    total = int(n.item())
    if angle_ids is None:
        r, w = dist.get_rank(group), dist.get_world_size(group)
        ids = r + w * np.arange(n_local)
    return ids, total


def os_sart(project, backproject, geom, b, x0, n_iter: int = 50, block: int = 20,
            lam: float = 1.0, nonneg: bool = True, group=None, callback=None, angle_ids=None):
    """Ordered-subsets SART:

        x <- x + lam * V_s^-1 A_s^T ( W_s^-1 (b_s - A_s x) )

    over angle blocks s of size `block` of the GLOBAL scan (interleaved: block
    s holds global angles s, s+S, ... with S = ceil(n_angles / block)), with
    row weights W = A_s 1 and column weights V_s = A_s^T 1.  `geom` / `b` are
    THIS rank's angles (rows; ``angle_ids`` their global indices, default the
    AngleSharding layout); with a process group the column sums and
    backprojections are all-reduced, so every rank holds the same x, equal
    to the single-process iterate up to summation order.  Every rank joins
    every reduction, also for a subset it holds no angle of (it contributes
    zeros).  Zero weights leave the corresponding entries unchanged.
    """
    import torch
    x = x0.clone()
    ids, total = _global_angle_ids(geom.n_angles, group, angle_ids)
    n_sub = max(1, (total + block - 1) // block)
    subsets = [np.flatnonzero(ids % n_sub == s) for s in range(n_sub)]
    weights = []
    for idx in subsets:
        g = _subset(geom, idx)
        if len(idx):
            W = project(g, torch.ones_like(x))
            V = backproject(g, torch.ones_like(W))
        else:
            W, V = None, torch.zeros_like(x)
        weights.append((g, W, _allreduce(V, group)))
    for it in range(n_iter):
        for (g, W, V), idx in zip(weights, subsets):
            if len(idx):
                r = b[idx] - project(g, x)
                r = torch.where(W > 0, r / torch.where(W > 0, W, torch.ones_like(W)),
                                torch.zeros_like(r))
                upd = backproject(g, r.contiguous())
            else:
                upd = torch.zeros_like(x)
            upd = _allreduce(upd, group)
            x = x + lam * torch.where(V > 0, upd / torch.where(V > 0, V, torch.ones_like(V)),
                                      torch.zeros_like(upd))
            if nonneg:
                x = torch.clamp_min(x, 0.0)
        if callback is not None:
            callback(it, x)
    return x


def cgls(project, backproject, geom, b, x0, n_iter: int = 30, group=None, callback=None):
    """CGLS for min ||A x - b|| (PAPER.md:26 lists CGLS among the consumers).
    With a process group, A = [A_0; A_1; ...] over ranks: A x stays local,
    A^T r and ||A p||^2 are all-reduced."""
    import torch
    x = x0.clone()
    r = b - project(geom, x)
    s = _allreduce(backproject(geom, r.contiguous()), group)
    p = s.clone()
    gamma = float(torch.dot(s.double(), s.double()))
    for it in range(n_iter):
        q = project(geom, p)
        qq = _allreduce(torch.tensor([float(torch.dot(q.double().ravel(), q.double().ravel()))],
                                     dtype=torch.float64, device=q.device), group).item()
        if qq == 0 or gamma == 0:
            break
        alpha = gamma / qq
        x = x + alpha * p
        r = r - alpha * q
        s = _allreduce(backproject(geom, r.contiguous()), group)
        gamma_new = float(torch.dot(s.double(), s.double()))
        p = s + (gamma_new / gamma) * p
        gamma = gamma_new
        if callback is not None:
            callback(it, x, r)
    return x
