"""BASELINE.json configs c1..c5 made concrete.

``workload(name, ...)`` returns a :class:`Workload` with the mesh, geometry
and seeded attenuation / detector values.  Detector size and angle count can
be overridden (keeping the detector's physical width) to build parity-sized
cases of the same shape.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import geometry as G
from . import meshes as M


@dataclass
class Workload:
    name: str
    mesh: M.Mesh
    geom: G.Geometry
    mu: np.ndarray       # float32 [T] attenuation per tet (caller order)
    y: np.ndarray        # float32 [A,Nv,Nu] detector values for backprojection
    desc: str = ""


def uniform_y(geom: G.Geometry, seed: int) -> np.ndarray:
    """y ~ U[0.5,1.5] (no cancellation in backprojected sums)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0.5, 1.5, (geom.n_angles, geom.n_v, geom.n_u)).astype(np.float32)


def uniform_mu(mesh: M.Mesh, seed: int, lo=0.0, hi=1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, mesh.n_tets).astype(np.float32)


def nested_balls_mu(mesh: M.Mesh) -> np.ndarray:
    """Background 0.5, an off-centre ball of 1 and a nested ball of 2 (the
    paper's 0/1/2 materials, with a positive background so
    relative checks see every tet)."""
    c = mesh.centroids()
    mu = np.full(mesh.n_tets, 0.5, dtype=np.float32)
    mu[np.linalg.norm(c - np.array([0.15, 0.1, 0.0]), axis=1) < 0.6] = 1.0
    mu[np.linalg.norm(c - np.array([0.3, 0.05, 0.1]), axis=1) < 0.25] = 2.0
    return mu


def cad_mu(mesh: M.Mesh) -> np.ndarray:
    inside = mesh.extra.get("inside")
    if inside is None:
        inside = M.cad_sdf(mesh.centroids()) < 0
    return np.where(np.asarray(inside, bool), 1.0, 0.05).astype(np.float32)


def _scaled_cone(n_angles, dso, dsd, width, n_u, n_v):
    return G.circular_cone(G.equidistant(n_angles), dso, dsd, n_u, n_v,
                           width / n_u, width / n_v)


def workload(name: str, n_angles: int | None = None, n_u: int | None = None,
             n_v: int | None = None, mu: str = "default", seed_y: int | None = None,
             angle_offset: int = 0) -> Workload:
    if name == "c1":
        mesh = M.kuhn_cube()
        A = n_angles or 4
        geom = G.circular_parallel(G.equidistant(A), n_u or 8, n_v or 8, 0.25, 0.25)
        mu_v = (np.arange(mesh.n_tets) + 1).astype(np.float32)
        desc = "Kuhn cube 6 tets, parallel 8x8 pitch 1/4, 4 angles"
        sy = 1
    elif name == "c2":
        mesh = M.cached(M.ball_mesh)
        geom = _scaled_cone(n_angles or 90, 4.0, 8.0, 4.4, n_u or 256, n_v or 256)
        mu_v = nested_balls_mu(mesh)
        desc = "perturbed-lattice ball ~1.0e5 tets, cone 256^2, 90 angles"
        sy = 3
    elif name in ("c3", "c5"):
        big = name == "c5"
        mesh = M.cached(M.graded_box_mesh, n_interior=1_560_000 if big else 150_000,
                        seed=4)
        R = np.sqrt(3.0)
        n = 1024 if big else 512
        geom = _scaled_cone(n_angles or (720 if big else 360), 4 * R, 8 * R, 7.2,
                            n_u or n, n_v or n)
        mu_v = cad_mu(mesh)
        desc = ("graded CAD-like box mesh, cone %dx%d, %d angles" %
                (geom.n_u, geom.n_v, geom.n_angles))
        sy = 4
    elif name == "c4a":
        mesh = M.sliver_kuhn_mesh(55)
        s = 2.0 ** -5
        dirs = G.LATTICE_DIRS[: (n_angles or 16)]
        geom = G.lattice_parallel((s, s, s * 2 ** -8), (0.0, 0.0, 0.0), n_u or 512,
                                  n_v or 512, dirs)
        mu_v = uniform_mu(mesh, 5, 0.5, 1.5)
        desc = "Kuhn sliver lattice (aspect 256), lattice-aligned parallel rays"
        sy = 5
    elif name == "c4b":
        n_l, jit = 55, 1e-4
        mesh = M.cached(M.jittered_lattice_mesh, n_l, jit, 5)
        R = np.sqrt(3.0)
        geom = _scaled_cone(n_angles or 32, 4 * R, 8 * R, 7.2, n_u or 512, n_v or 512)
        # "sources on lattice points" -- each source moves to
        # the nearest point of the (unjittered) mesh lattice, extended beyond
        # the mesh, so rays from it pass within 1e-4 h of lattice vertices
        h = 2.0 / n_l
        lo, step = -1 + 2 * jit * h, (2 - 4 * jit * h) / n_l
        S = geom.vecs[:, 0:3]
        geom.vecs[:, 0:3] = np.round((lo + np.round((S - lo) / step) * step) * 2.0 ** 22) / 2.0 ** 22
        mu_v = uniform_mu(mesh, 5, 0.5, 1.5)
        desc = ("Delaunay of 1e-4-jittered lattice (slivers), cone 512^2, 32 angles, "
                "sources on lattice points")
        sy = 5
    else:
        raise KeyError(name)
    if mu == "uniform":
        mu_v = uniform_mu(mesh, 3, 0.05, 1.0)
    if angle_offset:
        geom = geom.subset(np.arange(angle_offset, geom.n_angles))
    y = uniform_y(geom, seed_y if seed_y is not None else sy)
    return Workload(name, mesh, geom, mu_v, y, desc)
