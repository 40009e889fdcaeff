"""Helpers shared by the GPU parity tests (CUDA path vs the CPU oracle)."""
from __future__ import annotations

import numpy as np

from oracle import tetref as O

FWD_TOL = 1e-4     # north_star: forward <= 1e-4 relative per pixel
BACK_TOL = 1e-4    # north_star: backprojection <= 1e-4 relative per tet
ADJ_TOL = 1e-5     # north_star: adjoint mismatch <= 1e-5


def hull_diameter(mesh) -> float:
    lo, hi = mesh.verts.min(0), mesh.verts.max(0)
    return float(np.linalg.norm(hi - lo))


def fwd_errors(g, r, mu, mesh):
    """Relative per-pixel errors with the floor of DESIGN.md R11."""
    floor = 1e-3 * float(np.abs(mu).mean()) * hull_diameter(mesh)
    return np.abs(g - r) / np.maximum(np.abs(r), floor)


def back_errors(g, r):
    nz = np.abs(r[r != 0])
    floor = 1e-3 * (float(np.median(nz)) if nz.size else 1.0)
    err = np.abs(g - r) / np.maximum(np.abs(r), floor)
    err[(g == 0) & (r == 0)] = 0.0
    return err


def run_gpu(mesh, geom, mu, y, device="cuda:0", flags=None, opts=None):
    import torch

    from paper_1908_06909_b200 import TetMesh
    kw = {} if flags is None else {"flags": flags}
    tm = TetMesh.from_mesh(mesh, device=0, **kw)
    dev = torch.device(device)
    proj, st = tm.project(geom, torch.from_numpy(np.ascontiguousarray(mu, np.float32)).to(dev),
                          stats=True, opts=opts)
    x, st2 = tm.backproject(geom, torch.from_numpy(np.ascontiguousarray(y, np.float32)).to(dev),
                            stats=True, opts=opts)
    torch.cuda.synchronize()
    return proj.cpu().numpy(), x.cpu().numpy(), st, st2, tm


def run_oracle(mesh, geom, mu, y):
    om = O.OracleMesh.from_mesh(mesh)
    p, st = O.project(om, geom, np.asarray(mu, np.float64))
    x, st2 = O.backproject(om, geom, np.asarray(y, np.float64))
    return p, x, st, st2


def check_parity(mesh, geom, mu, y, *, expect_exact_fallbacks=None, opts=None):
    """CUDA path (``opts``: traversal / entry-finder options, default exact +
    raster) vs the oracle: identical crossing and hit counts, per-pixel and
    per-tet values within the north-star tolerances, adjoint."""
    p, x, st, st2, _ = run_gpu(mesh, geom, mu, y, opts=opts)
    pr, xr, ost, ost2 = run_oracle(mesh, geom, mu, y)
    for s in (st, st2):
        assert s["lost"] == 0 and s["stuck"] == 0 and s["entry_conflicts"] == 0, s
        assert s["rays"] == geom.n_rays
    # same combinatorial paths: identical crossing counts and hit counts
    assert st["crossings"] == ost["crossings"], (st, ost)
    assert st2["crossings"] == ost2["crossings"], (st2, ost2)
    assert st["rays_hit"] == ost["rays_hit"]
    assert ost["lost"] == 0 and ost["stuck"] == 0
    fe = fwd_errors(p.astype(np.float64), pr, mu, mesh)
    be = back_errors(x.astype(np.float64), xr)
    assert fe.max() <= FWD_TOL, ("forward", fe.max(), np.unravel_index(fe.argmax(), fe.shape))
    assert be.max() <= BACK_TOL, ("back", be.max(), int(be.argmax()))
    # adjoint on the GPU outputs
    lhs = float(np.dot(p.astype(np.float64).ravel(), np.asarray(y, np.float64).ravel()))
    rhs = float(np.dot(np.asarray(mu, np.float64), x.astype(np.float64)))
    if lhs or rhs:
        assert abs(lhs - rhs) / max(abs(lhs), abs(rhs)) <= ADJ_TOL, (lhs, rhs)
    if expect_exact_fallbacks:
        assert st["exact_fallbacks"] > 0
    return {"fwd_max_rel": float(fe.max()), "back_max_rel": float(be.max()), "stats": st,
            "oracle": ost}
