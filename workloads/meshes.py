"""Synthetic tetrahedral meshes (input generators only).

Conventions (the C ABI's, include/tetproj.h):
  * ``tets[t] = (n0, n1, n2, n3)`` vertex indices (orientation NOT normalised
    here -- both the library and the oracle fix it with TET_F_FIX_ORIENTATION),
  * ``nbrs[t][k]`` = tet across the face opposite ``tets[t][k]``, ``-1`` on the
    hull (the face-opposite-node convention of the paper's graph, PAPER.md:38
    "nD+1 ordered neighbour indexes", read as in SPEC.md:38/95),
  * ``bfaces[b] = (t, k)`` with ``nbrs[t][k] == -1`` (the paper's list of
    "elements that bound the triangulated space").

All coordinates are multiples of 2**-20 (meshes of radius ~1) so that the
library's power-of-two grid snap is lossless
and the combinatorics produced by Qhull stay valid after snapping.
"""
from __future__ import annotations

import hashlib
import itertools
import os
from dataclasses import dataclass, field

import numpy as np

QUANT = 2.0 ** 20  # coordinates are multiples of 1/QUANT


@dataclass
class Mesh:
    name: str
    verts: np.ndarray   # float64 [V,3]
    tets: np.ndarray    # int32 [T,4]
    nbrs: np.ndarray    # int32 [T,4]
    bfaces: np.ndarray  # int32 [B,2]
    extra: dict = field(default_factory=dict)

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    @property
    def n_verts(self) -> int:
        return int(self.verts.shape[0])

    @property
    def n_bfaces(self) -> int:
        return int(self.bfaces.shape[0])

    def centroids(self) -> np.ndarray:
        return self.verts[self.tets].mean(axis=1)


# --------------------------------------------------------------------------
# combinatorial face matching (SPEC.md:59-67 build_graph; no geometry)
# --------------------------------------------------------------------------
def build_graph(tets: np.ndarray):
    """Neighbours by matching sorted face-node triples; returns (nbrs, bfaces)."""
    tets = np.asarray(tets, dtype=np.int64)
    T = tets.shape[0]
    # face k of tet t = the three nodes other than tets[t][k]
    others = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])
    faces = tets[:, others]                      # [T,4,3]
    faces = np.sort(faces, axis=2).reshape(-1, 3)  # [4T,3]
    owner = np.repeat(np.arange(T), 4)
    local = np.tile(np.arange(4), T)
    order = np.lexsort((faces[:, 2], faces[:, 1], faces[:, 0]))
    fs = faces[order]
    same = np.all(fs[1:] == fs[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("non-manifold input: a face is shared by >2 tets")
    nbrs = np.full((T, 4), -1, dtype=np.int64)
    i = np.nonzero(same)[0]
    a, b = order[i], order[i + 1]
    nbrs[owner[a], local[a]] = owner[b]
    nbrs[owner[b], local[b]] = owner[a]
    bt, bk = np.nonzero(nbrs < 0)
    bfaces = np.stack([bt, bk], axis=1)
    return nbrs.astype(np.int32), bfaces.astype(np.int32)


def _finish(name, verts, tets, extra=None) -> Mesh:
    verts = np.ascontiguousarray(verts, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int32)
    nbrs, bfaces = build_graph(tets)
    return Mesh(name, verts, tets, np.ascontiguousarray(nbrs),
                np.ascontiguousarray(bfaces), extra or {})


def _quantize(p: np.ndarray) -> np.ndarray:
    return np.round(p * QUANT) / QUANT


# --------------------------------------------------------------------------
# small exact meshes
# --------------------------------------------------------------------------
def single_tet() -> Mesh:
    """Unit tet (0,0,0),(1,0,0),(0,1,0),(0,0,1)."""
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    return _finish("single_tet", v, np.array([[0, 1, 2, 3]]))


def kuhn_lattice(n: int, lo=(-0.5, -0.5, -0.5), step=(None, None, None),
                 name: str | None = None) -> Mesh:
    """n^3 cubes, each split into the 6 Kuhn (Freudenthal) tets.

    Vertex (i,j,k) sits at lo + (i,j,k)*step.  For every permutation s of the
    axes, the tet  v0=(i,j,k), v1=v0+e_s0, v2=v1+e_s1, v3=v0+(1,1,1); the
    triangulation is conforming across cubes.
    """
    step = tuple((1.0 / n) if s is None else s for s in step)
    m = n + 1
    idx = lambda i, j, k: (i * m + j) * m + k  # noqa: E731
    g = np.arange(m)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    verts = np.stack([lo[0] + I.ravel() * step[0], lo[1] + J.ravel() * step[1],
                      lo[2] + K.ravel() * step[2]], axis=1)
    c = np.arange(n)
    ci, cj, ck = [a.ravel() for a in np.meshgrid(c, c, c, indexing="ij")]
    tets = []
    for perm in itertools.permutations(range(3)):
        pos = [ci.copy(), cj.copy(), ck.copy()]
        vs = [idx(*pos)]
        for ax in perm:
            pos[ax] = pos[ax] + 1
            vs.append(idx(*pos))
        tets.append(np.stack(vs, axis=1))
    tets = np.stack(tets, axis=1).reshape(-1, 4)
    return _finish(name or f"kuhn{n}", verts, tets)


def kuhn_cube() -> Mesh:
    """Unit cube [-1/2,1/2]^3 split into 6 tets (config c1)."""
    return kuhn_lattice(1, name="kuhn_cube")


def l_shaped_lattice() -> Mesh:
    """Kuhn lattice(2) minus its (+,+,+) cube: 42 tets whose hull is a closed
    2-manifold with reflex edges around the removed corner -- a valid graph
    mesh that violates only the paper's one precondition, "the volumetric
    mesh must be convex"."""
    a = kuhn_lattice(2)
    keep = np.arange(a.n_tets) // 6 != 7          # tet = cube * 6 + permutation
    return _finish("l_shaped", a.verts, a.tets[keep])


def two_disjoint_tets() -> Mesh:
    """Two separate unit tets: every hull edge is convex (each component is a
    tetrahedron), so only a global convexity check rejects it."""
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1],
                  [3, 0, 0], [4, 0, 0], [3, 1, 0], [3, 0, 1]], dtype=np.float64)
    return _finish("two_tets", v, np.array([[0, 1, 2, 3], [4, 5, 6, 7]]))


# --------------------------------------------------------------------------
# Delaunay meshes (Qhull through scipy)
# --------------------------------------------------------------------------
def _exact_orient_nonzero(verts_q: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """True where the tet has non-zero volume (float screen + exact recheck)."""
    p = verts_q[tets].astype(np.float64)
    d1, d2, d3 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]
    det = np.einsum("ij,ij->i", d1, np.cross(d2, d3))
    scale = (np.abs(d1).max(1) * np.abs(d2).max(1) * np.abs(d3).max(1)) + 1e-300
    ok = np.abs(det) > 1e-9 * scale
    for t in np.nonzero(~ok)[0]:
        q = [[int(x) for x in verts_q[n]] for n in tets[t]]
        a = [q[1][i] - q[0][i] for i in range(3)]
        b = [q[2][i] - q[0][i] for i in range(3)]
        c = [q[3][i] - q[0][i] for i in range(3)]
        e = (a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0])
             + a[2] * (b[0] * c[1] - b[1] * c[0]))
        ok[t] = e != 0
    return ok


def delaunay_mesh(points: np.ndarray, name: str, extra=None, quant: float = QUANT) -> Mesh:
    from scipy.spatial import Delaunay

    pts = np.unique(np.round(np.asarray(points, dtype=np.float64) * quant) / quant, axis=0)
    tri = Delaunay(pts)
    tets = tri.simplices.astype(np.int64)
    ok = _exact_orient_nonzero(np.round(pts * quant).astype(np.int64), tets)
    if not ok.all():
        raise RuntimeError(f"{name}: Qhull produced {int((~ok).sum())} flat tets")
    # the neighbour table from Qhull uses the same opposite-vertex convention,
    # but we rebuild it combinatorially so every mesh goes through one path.
    return _finish(name, pts, tets, extra)


def fibonacci_sphere(n: int, radius: float) -> np.ndarray:
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    theta = np.pi * (1 + 5 ** 0.5) * i
    return radius * np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi),
                              np.cos(phi)], axis=1)


def ball_mesh(h: float = 0.065, sigma: float = 0.2, radius: float = 1.0,
              seed: int = 2) -> Mesh:
    """Config c2: jittered lattice inside r < R - h/2 plus a Fibonacci sphere
    of floor(4 pi R^2 / h^2) points; Delaunay."""
    rng = np.random.default_rng(seed)
    g = np.arange(-radius, radius + h, h)
    P = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    P = P + rng.normal(0.0, sigma * h, P.shape)
    P = P[np.linalg.norm(P, axis=1) < radius - h / 2]
    S = fibonacci_sphere(int(4 * np.pi * radius ** 2 / h ** 2), radius)
    return delaunay_mesh(np.concatenate([P, S]), f"ball_h{h}_s{seed}",
                         {"radius": radius})


# ---- graded CAD-like box (configs c3 / c5) ------------------------------
def cad_sdf(x: np.ndarray) -> np.ndarray:
    """Signed distance (approx.) to a CAD-like part: a slab block with a
    cylindrical bore along z, unioned with a sphere boss (inside < 0)."""
    q = np.abs(x - np.array([0.0, 0.0, -0.1])) - np.array([0.6, 0.5, 0.35])
    box = np.linalg.norm(np.maximum(q, 0), axis=1) + np.minimum(q.max(1), 0)
    bore = 0.22 - np.linalg.norm(x[:, :2] - np.array([0.1, 0.0]), axis=1)
    part = np.maximum(box, bore)
    boss = np.linalg.norm(x - np.array([-0.25, 0.1, 0.35]), axis=1) - 0.3
    return np.minimum(part, boss)


def _box_boundary_points(rng, per_edge: int, per_face: int) -> np.ndarray:
    pts = [np.array(c, dtype=np.float64) for c in itertools.product((-1.0, 1.0), repeat=3)]
    # edge points (shared by two faces): jitter along the edge only
    for ax in range(3):
        for s1, s2 in itertools.product((-1.0, 1.0), repeat=2):
            t = (np.arange(1, per_edge + 1) / (per_edge + 1)) * 2 - 1
            t = t + rng.uniform(-0.25, 0.25, per_edge) * (2.0 / (per_edge + 1))
            for tv in t:
                p = np.empty(3)
                o = [a for a in range(3) if a != ax]
                p[ax], p[o[0]], p[o[1]] = tv, s1, s2
                pts.append(p)
    # face-interior points: jitter in-plane only, keeping the hull planar
    for ax in range(3):
        for s in (-1.0, 1.0):
            k = int(np.ceil(np.sqrt(per_face)))
            g = (np.arange(k) + 0.5) / k * 1.6 - 0.8
            U, V = np.meshgrid(g, g, indexing="ij")
            uv = np.stack([U.ravel(), V.ravel()], 1)[:per_face]
            uv = uv + rng.uniform(-0.3, 0.3, uv.shape) * (1.6 / k)
            o = [a for a in range(3) if a != ax]
            p = np.empty((uv.shape[0], 3))
            p[:, ax], p[:, o[0]], p[:, o[1]] = s, uv[:, 0], uv[:, 1]
            pts.extend(list(p))
    return np.array(pts)


def graded_box_mesh(n_interior: int = 150_000, h_min_frac: float = 0.18,
                    seed: int = 4, per_edge: int = 3, per_face: int = 16) -> Mesh:
    """Configs c3/c5: box [-1,1]^3 with a coarsely sampled hull (~300 hull
    faces, cf. "6x10^5 total elements, but contained only 192 boundary
    elements") and interior points whose density grows towards
    a CAD-like surface (fine surface, coarse interior)."""
    rng = np.random.default_rng(seed)
    bnd = _box_boundary_points(rng, per_edge, per_face)
    pts = []
    need = n_interior
    margin = 0.02
    while need > 0:
        c = rng.uniform(-1 + margin, 1 - margin, (max(4 * need, 10000), 3))
        d = np.abs(cad_sdf(c))
        w = h_min_frac + (1 - h_min_frac) * np.minimum(1.0, d / 0.35)  # h(x)/h_max
        acc = rng.uniform(0, 1, len(c)) < (h_min_frac / w) ** 3
        c = c[acc][:need]
        pts.append(c)
        need -= len(c)
    P = np.concatenate([bnd] + pts)
    m = delaunay_mesh(P, f"graded_box_n{n_interior}_s{seed}")
    inside = cad_sdf(m.centroids()) < 0
    m.extra["inside"] = inside
    return m


def jittered_lattice_mesh(n: int = 55, jitter: float = 1e-4, seed: int = 5) -> Mesh:
    """Config c4b: Delaunay of an (n+1)^3 lattice on [-1,1]^3 whose points are
    jittered by jitter*h (boundary points only in-plane) -> classic slivers
    ("high aspect ratios")."""
    h = 2.0 / n
    g = np.linspace(-1 + 2 * jitter * h, 1 - 2 * jitter * h, n + 1)  # jittered points stay in [-1,1]
    P = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    for attempt in range(8):
        # jitter in all directions (the hull is the convex hull of the jittered
        # boundary points); quantise finely (2^-22) so coplanar quadruples,
        # which make Qhull emit flat tets, are rare -- redraw if any appear.
        rng = np.random.default_rng([seed, attempt])
        J = rng.uniform(-1, 1, P.shape) * jitter * h
        try:
            return delaunay_mesh(P + J, f"jlattice_n{n}_j{jitter}_s{seed}", quant=2.0 ** 22)
        except RuntimeError:
            continue
    raise RuntimeError("could not draw a jittered lattice without flat tets")


def sliver_kuhn_mesh(n: int = 55) -> Mesh:
    """Config c4a: Kuhn lattice n^3 on integer coords scaled (1,1,2^-8):
    aspect ratio 256, every lattice ray runs through vertices/edges/faces."""
    s = 2.0 ** -5
    return kuhn_lattice(n, lo=(-n / 2 * s, -n / 2 * s, -n / 2 * s * 2 ** -8),
                        step=(s, s, s * 2 ** -8), name=f"sliver_kuhn{n}")


def random_small_mesh(n_points: int, seed: int, box: bool = True) -> Mesh:
    """Tiny Delaunay meshes for brute-force pins (points on a coarse 1/16
    lattice so rays through vertices/edges are frequent)."""
    for attempt in range(100):   # lattice points can make Qhull emit flat tets: redraw
        rng = np.random.default_rng([seed, attempt])
        if box:
            corners = np.array(list(itertools.product((-1.0, 1.0), repeat=3)))
            inner = rng.integers(-15, 16, (n_points, 3)) / 16.0
            P = np.concatenate([corners, inner])
        else:
            P = rng.integers(-16, 17, (n_points, 3)) / 16.0
        P = np.unique(P, axis=0)
        try:
            return delaunay_mesh(P, f"small_n{n_points}_s{seed}")
        except RuntimeError:
            continue
    raise RuntimeError("could not draw a non-degenerate small mesh")


# --------------------------------------------------------------------------
# cache (meshes are pure functions of their arguments)
# --------------------------------------------------------------------------
def cache_dir() -> str:
    d = os.environ.get("TETPROJ_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "tetproj"))
    os.makedirs(d, exist_ok=True)
    return d


def cached(fn, *args, **kw) -> Mesh:
    key = hashlib.sha1(repr((fn.__name__, args, sorted(kw.items()), 3)).encode()).hexdigest()[:16]
    path = os.path.join(cache_dir(), f"{fn.__name__}_{key}.npz")
    if os.path.exists(path):
        try:
            z = np.load(path, allow_pickle=False)
            extra = {k[6:]: z[k] for k in z.files if k.startswith("extra_")}
            return Mesh(str(z["name"]), z["verts"], z["tets"], z["nbrs"], z["bfaces"], extra)
        except Exception:
            pass
    m = fn(*args, **kw)
    tmp = path + f".tmp{os.getpid()}.npz"
    np.savez(tmp, name=m.name, verts=m.verts, tets=m.tets, nbrs=m.nbrs, bfaces=m.bfaces,
             **{f"extra_{k}": np.asarray(v) for k, v in m.extra.items()})
    os.replace(tmp, path)
    return m
