"""Scan geometries -> the ABI's per-angle vectors (input generation only).

Each angle is 12 doubles (include/tetproj.h ``tet_geometry.vecs``):
  cone     : source S xyz | centre of pixel (v=0,u=0) xyz | u-step xyz | v-step xyz
  parallel : ray direction xyz | pixel (0,0) centre | u-step | v-step

Circular cone convention (the paper is silent and cites TIGRE, PAPER.md:177;
we use SPEC.md:357): rotation about z, S = Rz(th)(0,-DSO,0), detector centre
C = Rz(th)(0,DSD-DSO,0), u-axis Rz(th)(1,0,0)*du, v-axis (0,0,1)*dv, pixel
centre P(u,v) = C + (u-(Nu-1)/2) U + (v-(Nv-1)/2) V.  Angles are
equidistant, 2*pi*k/A ("circular trajectory in equidistant angles",
PAPER.md:187).  The parallel-beam analogue uses dir = Rz(th)(0,1,0) and a
detector plane through the origin.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BEAM_CONE = 0
BEAM_PARALLEL = 1


@dataclass
class Geometry:
    beam: int
    n_v: int
    n_u: int
    vecs: np.ndarray  # float64 [A,12]

    @property
    def n_angles(self) -> int:
        return int(self.vecs.shape[0])

    @property
    def n_rays(self) -> int:
        return self.n_angles * self.n_v * self.n_u

    def subset(self, angles) -> "Geometry":
        return Geometry(self.beam, self.n_v, self.n_u,
                        np.ascontiguousarray(self.vecs[np.asarray(angles)]))


def _rz(th):
    c, s = np.cos(th), np.sin(th)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def equidistant(n_angles: int) -> np.ndarray:
    return 2 * np.pi * np.arange(n_angles) / n_angles


def circular_cone(angles, dso, dsd, n_u, n_v, du, dv, off_u=0.0, off_v=0.0) -> Geometry:
    angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    vecs = np.empty((len(angles), 12))
    for i, th in enumerate(angles):
        R = _rz(th)
        S = R @ np.array([0.0, -dso, 0.0])
        C = R @ np.array([0.0, dsd - dso, 0.0])
        U = R @ np.array([du, 0.0, 0.0])
        V = np.array([0.0, 0.0, dv])
        P00 = C + (0 - (n_u - 1) / 2 + off_u) * U + (0 - (n_v - 1) / 2 + off_v) * V
        vecs[i] = np.concatenate([S, P00, U, V])
    return Geometry(BEAM_CONE, n_v, n_u, vecs)


def circular_parallel(angles, n_u, n_v, du, dv, off_u=0.0, off_v=0.0) -> Geometry:
    angles = np.atleast_1d(np.asarray(angles, dtype=np.float64))
    vecs = np.empty((len(angles), 12))
    for i, th in enumerate(angles):
        R = _rz(th)
        d = R @ np.array([0.0, 1.0, 0.0])
        U = R @ np.array([du, 0.0, 0.0])
        V = np.array([0.0, 0.0, dv])
        P00 = (0 - (n_u - 1) / 2 + off_u) * U + (0 - (n_v - 1) / 2 + off_v) * V
        vecs[i] = np.concatenate([d, P00, U, V])
    return Geometry(BEAM_PARALLEL, n_v, n_u, vecs)


def explicit(beam, n_v, n_u, rows) -> Geometry:
    return Geometry(beam, n_v, n_u, np.ascontiguousarray(np.asarray(rows, dtype=np.float64).reshape(-1, 12)))


# lattice directions for the sliver stress test
LATTICE_DIRS = [(0, 1, 0), (1, 0, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1),
                (1, 1, 1), (1, -1, 0), (1, 2, 3), (3, 1, 2), (2, 3, 1), (1, -1, 1),
                (1, 2, 0), (2, 1, 1), (1, 1, 2), (3, -2, 1)]


def lattice_parallel(step, center, n_u, n_v, dirs=LATTICE_DIRS) -> Geometry:
    """Parallel rays whose pixel centres are lattice points and whose
    directions are lattice vectors: every ray runs exactly through lattice
    vertices / edges / faces (a maximally degenerate workload)."""
    step = np.asarray(step, dtype=np.float64)
    center = np.asarray(center, dtype=np.float64)
    rows = []
    for d in dirs:
        d = np.asarray(d, dtype=np.float64)
        # two lattice vectors completing d to a basis
        cands = [np.array(c, dtype=np.float64) for c in
                 [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1)]]
        U = V = None
        for a in cands:
            if np.linalg.norm(np.cross(a, d)) == 0:
                continue
            for b in cands:
                if abs(np.linalg.det(np.stack([a, b, d]))) > 0.5:
                    U, V = a, b
                    break
            if U is not None:
                break
        Uw, Vw, dw = U * step, V * step, d * step
        P00 = center - (n_u // 2) * Uw - (n_v // 2) * Vw
        rows.append(np.concatenate([dw, P00, Uw, Vw]))
    return explicit(BEAM_PARALLEL, n_v, n_u, rows)
