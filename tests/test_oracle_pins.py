"""Pins of the CPU oracle against things other than itself (CPU only).

* exact-rational brute force (every ray against every tet, tests/bruteforce.py)
* the SoS sign table against the full delta-polynomial
* closed forms: unit-tet chord, Kuhn cube axis integral (tests/golden/),
  box-hull slab chord, ball sandwich bounds
* invariants: adjoint, dense-A agreement, reversal, hull-chord conservation,
  isometry (signed axis permutations of mesh + rays)
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import tetref as O
from tests import bruteforce as BF
from workloads import configs as CF
from workloads import geometry as G
from workloads import meshes as M

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module", autouse=True)
def _build(oracle_lib):
    return oracle_lib


def _rel(a, b, floor=1e-300):
    return abs(a - b) / max(abs(a), abs(b), floor)


# ------------------------------------------------------------- SoS table --
def _degenerate_cases(rng, n):
    cases = []
    for _ in range(n):
        kind = rng.integers(0, 6)
        o = rng.integers(-3, 4, 3)
        p = o + rng.integers(-3, 4, 3)
        if np.all(p == o):
            p[0] += 1
        D = p - o
        a = rng.integers(-3, 4, 3)
        b = rng.integers(-3, 4, 3)
        if kind == 1:            # a on the line
            a = o + rng.integers(-2, 3) * D
        elif kind == 2:          # both on the line (edge along the ray)
            a = o + rng.integers(-2, 3) * D
            b = o + rng.integers(-2, 3) * D
        elif kind == 3:          # edge parallel to the ray
            b = a + rng.integers(1, 3) * D
        elif kind == 4:          # coplanar with the line
            b = o + rng.integers(-2, 3) * D + rng.integers(-2, 3) * (a - o)
        elif kind == 5:          # axis-aligned small coordinates
            a[rng.integers(0, 3)] = o[0]
        if np.all(a == b):
            b = b + np.array([0, 0, 1])
        cases.append((o, p, a, b))
    return cases


def test_sos_table_matches_delta_polynomial():
    rng = np.random.default_rng(11)
    n_zero_det = 0
    for o, p, a, b in _degenerate_cases(rng, 4000):
        want = BF.sos_sign_polynomial(o.tolist(), p.tolist(), a.tolist(), b.tolist())
        got = O.side(o, p, a, b)
        assert got == want, (o, p, a, b)
        assert got != 0
        assert O.side(o, p, b, a) == -got          # antisymmetric in the edge
        D = p - o
        n_zero_det += int(np.dot(D, np.cross(a - o, b - o)) == 0)
    assert n_zero_det > 1500                        # the cases are really degenerate


def test_sos_large_coordinates():
    """int128 range: coordinates near the +-2^31 grid span."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        o, p, a, b = [rng.integers(-2 ** 31 + 1, 2 ** 31 - 1, 3) for _ in range(4)]
        if rng.integers(0, 2):
            a = o + (p - o) // 2 * 0 + (p - o)       # a on the line
        want = BF.sos_sign_polynomial(o.tolist(), p.tolist(), a.tolist(), b.tolist())
        assert O.side(o, p, a, b) == want


# ----------------------------------------------------------- closed forms --
def test_unit_tet_chord_golden():
    ex = GOLD["unit_tet_chord"]
    m = M.single_tet()
    om = O.OracleMesh.from_mesh(m)
    d = ex["ray_dir"]
    geom = G.explicit(G.BEAM_PARALLEL, 1, 1, [d + ex["ray_point"] + [1, 0, 0, 0, 1, 0]])
    tets, ch = O.ray_path(om, geom, 0)
    assert list(tets) == [0]
    assert abs(ch[0] - ex["chord"]) < 1e-15
    val, st = O.project(om, geom, np.array([GOLD["unit_tet_integral_mu2"]["mu"]]))
    assert abs(val.ravel()[0] - GOLD["unit_tet_integral_mu2"]["integral"]) < 1e-15
    assert st["lost"] == 0 and st["stuck"] == 0


def test_kuhn_cube_axis_golden():
    ex = GOLD["kuhn_cube_axis_integral"]
    m = M.kuhn_cube()
    assert m.n_tets == GOLD["kuhn_cube_graph"]["n_tets"]
    assert m.n_bfaces == GOLD["kuhn_cube_graph"]["n_bfaces"]
    om = O.OracleMesh.from_mesh(m)
    for d in ex["ray_dirs"]:
        u = [1, 0, 0] if d[0] == 0 else [0, 1, 0]
        v = list(np.cross(d, u))
        geom = G.explicit(G.BEAM_PARALLEL, 1, 1, [d + ex["ray_point"] + u + v])
        val, st = O.project(om, geom, np.ones(6))
        assert abs(val.ravel()[0] - ex["integral"]) < 1e-14
        assert st["rays_hit"] == 1 and st["lost"] == 0


def test_c1_hit_count_and_hull_chord():
    w = CF.workload("c1")
    om = O.OracleMesh.from_mesh(w.mesh)
    val, st = O.project(om, w.geom, np.ones(6))
    assert st["rays_hit"] == 4 * GOLD["c1_hit_rays_per_angle"]["value"]
    assert st["lost"] == 0 and st["stuck"] == 0
    # every hit ray is axis-parallel through the unit cube: chord exactly 1
    assert np.all((np.abs(val - 1) < 1e-14) | (val == 0))


# ------------------------------------------------- brute-force agreement --
def _compare_with_bruteforce(mesh, geom, ray_ids):
    om = O.OracleMesh.from_mesh(mesh)
    Pg, g, C = BF.snap_verts(mesh.verts)
    assert om.g == g
    assert np.array_equal(om.vertex_grid(), np.array(Pg, dtype=np.int64))
    n_deg = 0
    for rid in ray_ids:
        o, p = BF.ray_points(geom, g, C, int(rid))
        oo, pp = O.ray_points(om, geom, int(rid))
        assert list(oo) == o and list(pp) == p
        L = math.sqrt(float(BF.dot(BF.sub(p, o), BF.sub(p, o)))) * g
        bf = BF.chords_of_ray(Pg, mesh.tets, o, p, g)
        tets, ch = O.ray_path(om, geom, int(rid))
        assert len(set(tets.tolist())) == len(tets)          # no tet twice
        eps = 1e-12 * L
        pos = {int(t): c for t, c in zip(tets, ch) if c > eps}
        bfpos = {t: c for t, c in bf.items() if c > eps}
        assert set(pos) == set(bfpos), (rid, sorted(pos), sorted(bfpos))
        for t in pos:
            assert abs(pos[t] - bfpos[t]) <= 1e-12 * L
        assert set(int(t) for t in tets) <= set(bf), rid      # visits only touched tets
        n_deg += len(bf) != len(bfpos)
    return n_deg


def test_bruteforce_c1_all_rays():
    w = CF.workload("c1")
    n_deg = _compare_with_bruteforce(w.mesh, w.geom, range(w.geom.n_rays))
    assert n_deg > 0            # c1 rays really hit degenerate configurations


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bruteforce_small_lattice_parallel(seed):
    m = M.random_small_mesh(25 + 5 * seed, seed)
    dirs = G.LATTICE_DIRS[seed::4][:4]
    geom = G.lattice_parallel((1 / 8, 1 / 8, 1 / 8), (0, 0, 0), 9, 9, dirs)
    n_deg = _compare_with_bruteforce(m, geom, range(geom.n_rays))
    assert n_deg > 0


@pytest.mark.parametrize("seed", [4, 5])
def test_bruteforce_small_cone_through_vertices(seed):
    """Cone source on a lattice point, pixel centres on lattice points: rays run
    through mesh vertices and edges."""
    m = M.random_small_mesh(30, seed)
    rows = []
    for th in (0.0, 1.0, 2.5):
        S = np.round(np.array([4 * math.sin(th), -4 * math.cos(th), 0.25]) * 16) / 16
        U = np.array([0.125, 0, 0]) if abs(math.cos(th)) > 0.5 else np.array([0, 0.125, 0])
        V = np.array([0, 0, 0.125])
        P00 = -S - 4 * U - 4 * V
        rows.append(np.concatenate([S, P00, U, V]))
    geom = G.explicit(G.BEAM_CONE, 9, 9, rows)
    _compare_with_bruteforce(m, geom, range(geom.n_rays))


def test_bruteforce_generic_rays():
    m = M.random_small_mesh(40, 7, box=False)
    geom = G.circular_cone(G.equidistant(3) + 0.123, 5.0, 10.0, 11, 9, 0.41, 0.43)
    _compare_with_bruteforce(m, geom, range(geom.n_rays))


def test_dense_matrix_project_backproject():
    """materialise A, compare A mu and A^T y with the oracle."""
    m = M.random_small_mesh(30, 9)
    geom = G.lattice_parallel((1 / 8,) * 3, (0, 0, 0), 9, 9, G.LATTICE_DIRS[:3])
    A = BF.dense_A(m, geom)
    om = O.OracleMesh.from_mesh(m)
    rng = np.random.default_rng(0)
    mu = rng.uniform(0.5, 1.5, m.n_tets)
    y = rng.uniform(0.5, 1.5, geom.n_rays)
    proj, st = O.project(om, geom, mu)
    x, st2 = O.backproject(om, geom, y)
    np.testing.assert_allclose(proj.ravel(), A @ mu, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(x, A.T @ y, rtol=1e-12, atol=1e-12)
    assert st["lost"] == st2["lost"] == 0


# ---------------------------------------------------------- invariants --
def _slab_chord(o, d, lo=-1.0, hi=1.0):
    t0, t1 = -np.inf, np.inf
    for i in range(3):
        if d[i] == 0:
            if not (lo <= o[i] <= hi):
                return 0.0
            continue
        a, b = (lo - o[i]) / d[i], (hi - o[i]) / d[i]
        t0, t1 = max(t0, min(a, b)), min(t1, max(a, b))
    return max(0.0, t1 - t0) * np.linalg.norm(d)


def test_box_hull_chord_conservation():
    """sum_i a_ij = chord of line j through the box hull."""
    m = M.graded_box_mesh(n_interior=1500, seed=8, per_face=4)
    om = O.OracleMesh.from_mesh(m)
    geom = G.circular_cone(G.equidistant(5) + 0.3, 4 * math.sqrt(3), 8 * math.sqrt(3), 24, 20,
                           0.3, 0.36)
    val, st = O.project(om, geom, np.ones(m.n_tets))
    assert st["lost"] == 0 and st["stuck"] == 0 and st["rays_hit"] > 100
    g = om.g
    for rid in range(geom.n_rays):
        o, p = O.ray_points(om, geom, rid)     # grid ints; box is [-1,1]^3 exactly
        o, p = o * g, p * g
        want = _slab_chord(o, p - o)
        assert abs(val.ravel()[rid] - want) <= 1e-12 * 4, rid


def test_ball_sandwich():
    """Faceted ball: chord_sphere(R_in) <= sum_i a_ij <= chord_sphere(R_out)."""
    m = M.ball_mesh(h=0.3, seed=3)
    om = O.OracleMesh.from_mesh(m)
    geom = G.circular_parallel([0.2, 1.7], 31, 31, 0.066, 0.066)
    val, st = O.project(om, geom, np.ones(m.n_tets))
    assert st["lost"] == 0 and st["stuck"] == 0
    V = m.verts
    R_out = np.linalg.norm(V, axis=1).max()
    R_in = np.inf
    for t, k in m.bfaces:
        f = [m.tets[t][j] for j in range(4) if j != k]
        n = np.cross(V[f[1]] - V[f[0]], V[f[2]] - V[f[0]])
        R_in = min(R_in, abs(np.dot(n, V[f[0]])) / np.linalg.norm(n))
    g = om.g
    for rid in range(geom.n_rays):
        o, p = O.ray_points(om, geom, rid)
        o, p = o * g, p * g
        d = (p - o) / np.linalg.norm(p - o)
        rho = np.linalg.norm(o - np.dot(o, d) * d)
        lo = 2 * math.sqrt(max(R_in ** 2 - rho ** 2, 0))
        hi = 2 * math.sqrt(max(R_out ** 2 - rho ** 2, 0))
        v = val.ravel()[rid]
        assert lo - 1e-12 <= v <= hi + 1e-12, (rid, lo, v, hi)


@pytest.mark.parametrize("name", ["c1", "small"])
def test_adjoint_double(name):
    if name == "c1":
        w = CF.workload("c1")
        mesh, geom = w.mesh, w.geom
    else:
        mesh = M.random_small_mesh(40, 3)
        geom = G.circular_cone(G.equidistant(4), 4.0, 8.0, 16, 16, 0.3, 0.3)
    om = O.OracleMesh.from_mesh(mesh)
    rng = np.random.default_rng(1)
    mu = rng.uniform(0, 1, mesh.n_tets)
    y = rng.uniform(0.5, 1.5, geom.n_rays)
    p, _ = O.project(om, geom, mu)
    x, _ = O.backproject(om, geom, y)
    lhs, rhs = float(p.ravel() @ y), float(mu @ x)
    assert _rel(lhs, rhs) <= 1e-12


def test_reversal_invariance():
    """Reversing every ray (o<->p) leaves every per-tet chord unchanged."""
    m = M.random_small_mesh(30, 6)
    fwd = G.lattice_parallel((1 / 8,) * 3, (0, 0, 0), 9, 9, G.LATTICE_DIRS[:4])
    rev = G.Geometry(fwd.beam, fwd.n_v, fwd.n_u, fwd.vecs.copy())
    rev.vecs[:, 0:3] *= -1.0
    om = O.OracleMesh.from_mesh(m)
    for rid in range(fwd.n_rays):
        t1, c1 = O.ray_path(om, fwd, rid)
        t2, c2 = O.ray_path(om, rev, rid)
        a = {int(t): c for t, c in zip(t1, c1) if c > 1e-15}
        b = {int(t): c for t, c in zip(t2, c2) if c > 1e-15}
        assert set(a) == set(b)
        for t in a:
            assert abs(a[t] - b[t]) < 1e-13


def test_orientation_fix_and_validation():
    m = M.kuhn_cube()
    t = m.tets.copy()
    n = m.nbrs.copy()
    t[:, [0, 1]] = t[:, [1, 0]]
    n[:, [0, 1]] = n[:, [1, 0]]
    b = np.array([(tt, {0: 1, 1: 0}.get(k, k)) for tt, k in m.bfaces], np.int32)
    om = O.OracleMesh(m.verts, t, n, b, fix=True)
    geom = CF.workload("c1").geom
    v1, _ = O.project(om, geom, np.arange(6) + 1.0)
    v0, _ = O.project(O.OracleMesh.from_mesh(m), geom, np.arange(6) + 1.0)
    np.testing.assert_array_equal(v0, v1)
    with pytest.raises(O.OracleError):
        O.OracleMesh(m.verts, t, n, b, fix=False)
    bad = m.nbrs.copy()
    bad[0, 0], bad[0, 1] = bad[0, 1], bad[0, 0]
    with pytest.raises(O.OracleError):
        O.OracleMesh(m.verts, m.tets, bad, m.bfaces)


@pytest.mark.parametrize("make", [M.l_shaped_lattice, M.two_disjoint_tets])
def test_nonconvex_rejected(make):
    """"The volumetric mesh must be convex" (§2.4).  Both meshes
    pass every other check (orientation, reciprocity, closed 2-manifold hull),
    so only the convexity check can reject them -- with code 3.  The L-shape
    has reflex hull edges; the two disjoint tets have none (each component is
    convex), so it needs the all-vertices-against-all-hull-planes form."""
    m = make()
    with pytest.raises(O.OracleError) as e:
        O.OracleMesh.from_mesh(m)
    assert e.value.code == 3, e.value
    # the same tets minus the offending part are accepted: a convex sub-mesh
    if make is M.two_disjoint_tets:
        O.OracleMesh(m.verts[:4], m.tets[:1], m.nbrs[:1], m.bfaces[m.bfaces[:, 0] == 0])


def test_carved_lattice_is_non_manifold():
    """Carving every 7th tet out of a lattice leaves a hull with a repeated
    directed edge: rejected as a mesh error (code 2) before convexity."""
    a = M.kuhn_lattice(2)
    keep = [i for i in range(a.n_tets) if i % 7 != 3]
    t = a.tets[keep]
    nb, bf = M.build_graph(t)
    with pytest.raises(O.OracleError) as e:
        O.OracleMesh(a.verts, t, nb, bf)
    assert e.value.code == 2, e.value


def test_stats_and_crossings_consistent():
    w = CF.workload("c1")
    om = O.OracleMesh.from_mesh(w.mesh)
    _, st = O.project(om, w.geom, w.mu)
    total = sum(len(O.ray_path(om, w.geom, r)[0]) for r in range(w.geom.n_rays))
    assert total == st["crossings"]
    _, st2 = O.backproject(om, w.geom, w.y)
    assert st2["crossings"] == st["crossings"]


# signed axis permutations: (perm, signs); odd ones flip every tet's orientation
_ISOMETRIES = [((1, 2, 0), (1, 1, 1)), ((1, 0, 2), (1, 1, 1)), ((0, 1, 2), (-1, 1, 1)),
               ((2, 1, 0), (1, -1, -1)), ((2, 0, 1), (-1, -1, -1))]


@pytest.mark.parametrize("perm,signs", _ISOMETRIES)
def test_isometry_invariance(perm, signs):
    """Eq. 1-3: a_ij is a length, so moving mesh and rays by the same
    isometry leaves every pixel and every per-tet value unchanged.  Signed axis
    permutations are exact on the snapping grid (SURVEY 8(b) Grid: c and r map
    with the vertices, rint is odd), so a dropped or transposed component in
    the predicate or the chord (which is not symmetric under these maps)
    breaks it.  Generic rays only: SoS (8(c) reading 6) is not invariant."""
    Q = np.zeros((3, 3))
    for i, (j, s) in enumerate(zip(perm, signs)):
        Q[i, j] = s
    m = M.random_small_mesh(40, 11)
    geom = G.circular_cone(G.equidistant(3) + 0.37, 4.0, 8.0, 13, 11, 0.37, 0.41,
                           off_u=0.21, off_v=-0.13)
    m2 = M.Mesh(m.name + "_iso", m.verts @ Q.T, m.tets, m.nbrs, m.bfaces)
    v2 = geom.vecs.reshape(-1, 4, 3) @ Q.T
    g2 = G.Geometry(geom.beam, geom.n_v, geom.n_u, np.ascontiguousarray(v2.reshape(-1, 12)))
    rng = np.random.default_rng(12)
    mu = rng.uniform(0.5, 1.5, m.n_tets)
    y = rng.uniform(0.5, 1.5, geom.n_rays)
    om, om2 = O.OracleMesh.from_mesh(m), O.OracleMesh.from_mesh(m2)
    p1, s1 = O.project(om, geom, mu)
    p2, s2 = O.project(om2, g2, mu)
    x1, _ = O.backproject(om, geom, y)
    x2, _ = O.backproject(om2, g2, y)
    assert s1["rays_hit"] > 50 and s1["lost"] == s2["lost"] == 0
    assert s1["crossings"] == s2["crossings"] and s1["rays_hit"] == s2["rays_hit"]
    np.testing.assert_allclose(p2, p1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(x2, x1, rtol=1e-12, atol=1e-12)
    assert np.count_nonzero(x1) > m.n_tets // 2
