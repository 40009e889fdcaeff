"""Pins of the NEXT-1 oracle -- the paper's own traversal, Alg. 1 (eps-guarded
Möller-Trumbore) inside Alg. 2 (eps escalation and the swap
check), oracle/tetref_mt.inc -- against things other than
itself (CPU only):

* SPEC.md's worked examples of Alg. 1 and of the tetra intersection
   and the Kuhn-cube closed form;
* exact rational linear algebra for the hit / miss decision and t of Alg. 1;
* the eps invariant the paper states: enlarging eps "increases the size of
  the triangle faces" while "keeping the value of the intersection parameter
  t unchanged";
* the exact SoS walker (an independent implementation) on generic rays:
  same tets, same values;
* fig:singledouble: on a sliver mesh double precision
  traces every ray while single precision leaves many rays unterminated.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import tetref as O
from workloads import configs as CF
from workloads import geometry as G
from workloads import meshes as M


@pytest.fixture(scope="module", autouse=True)
def _build(oracle_lib):
    return oracle_lib


@pytest.mark.parametrize("single", [False, True])
def test_alg1_spec_examples(single):
    tri = ([0, 0, 0], [1, 0, 0], [0, 1, 0])
    # S:140 planar case: hit at t = 1
    hit, t = O.mt_hit([0.25, 0.25, -1], [0.25, 0.25, 0], *tri, 0.0, single=single)
    assert hit and t == 1.0
    # S:141 ray in the z = 1 plane (parallel to the triangle): the |a| < 1e-8 branch
    hit, _ = O.mt_hit([0.25, 0.25, 1], [0.5, 0.25, 1], *tri, 0.0, single=single)
    assert not hit
    hit, _ = O.mt_hit([0.25, 0.25, 1], [0.5, 0.25, 1], *tri, 1e3, single=single)
    assert not hit                        # eps never rescues a parallel ray


def _exact_uvt(r1, r2, p1, p2, p3):
    """Solve R1 + t d = P1 + u E1 + v E2 by Cramer's rule in rationals."""
    F = [[Fraction(x) for x in v] for v in (r1, r2, p1, p2, p3)]
    R1, R2, P1, P2, P3 = F
    d = [R2[i] - R1[i] for i in range(3)]
    E1 = [P2[i] - P1[i] for i in range(3)]
    E2 = [P3[i] - P1[i] for i in range(3)]
    s = [R1[i] - P1[i] for i in range(3)]

    def det(a, b, c):   # columns a, b, c
        return (a[0] * (b[1] * c[2] - b[2] * c[1]) - b[0] * (a[1] * c[2] - a[2] * c[1])
                + c[0] * (a[1] * b[2] - a[2] * b[1]))
    nd = [-x for x in d]
    D = det(E1, E2, nd)            # [E1 E2 -d] (u v t)^T = s
    if D == 0:
        return None
    return det(s, E2, nd) / D, det(E1, s, nd) / D, det(E1, E2, s) / D


def test_alg1_against_exact_rational_solution():
    """Hit iff the exact barycentric (u, v) lie in the triangle (away from a
    1e-6 band around its edges), and then t equals the exact t to 1e-10."""
    rng = np.random.default_rng(21)
    n_hit = n_miss = 0
    for _ in range(3000):
        scale = 10.0 ** rng.uniform(-3, 3)
        P = rng.uniform(-1, 1, (3, 3)) * scale
        r1 = rng.uniform(-3, 3, 3) * scale
        target = P[0] + rng.uniform(-0.3, 1.0) * (P[1] - P[0]) + rng.uniform(-0.3, 1.0) * (P[2] - P[0])
        r2 = r1 + (target - r1) * rng.uniform(0.5, 2.0)
        ex = _exact_uvt(r1, r2, *P)
        if ex is None:
            continue
        u, v, t = (float(x) for x in ex)
        hit, tm = O.mt_hit(r1, r2, *P, 0.0)
        a_small = False
        d = r2 - r1
        E1, E2 = P[1] - P[0], P[2] - P[0]
        if abs(np.dot(E1, np.cross(d, E2))) < 1e-7:
            a_small = True        # the verbatim 1e-8 cutoff may reject it
        band = 1e-6
        if u > band and v > band and u + v < 1 - band and not a_small:
            assert hit, (u, v)
            assert abs(tm - t) <= 1e-10 * max(abs(t), 1.0), (tm, t)
            n_hit += 1
        elif u < -band or v < -band or u + v > 1 + band:
            assert not hit, (u, v)
            n_miss += 1
    assert n_hit > 500 and n_miss > 500


@pytest.mark.parametrize("single", [False, True])
def test_eps_inflates_faces_keeps_t(single):
    """the safety parameter "effectively increases the size of the
    triangle faces ... keeping the value of the intersection parameter t
    unchanged": a hit at eps stays a hit at every larger eps with the
    bitwise-identical t, and eps only ever adds hits."""
    rng = np.random.default_rng(5)
    eps_list = [0.0, 1e-9, 1e-7, 1e-5, 1e-3, 1e-1]
    grew = 0
    for _ in range(2000):
        P = rng.uniform(-1, 1, (3, 3))
        r1 = rng.uniform(-3, 3, 3)
        # aim at an edge or a vertex (the near-degenerate cases eps exists for)
        w = rng.choice([0.0, 1.0], 2) if rng.uniform() < 0.5 else rng.uniform(0, 1, 2) * [1, 0]
        target = P[0] + w[0] * (P[1] - P[0]) + w[1] * (P[2] - P[0])
        r2 = r1 + (target - r1) * 1.7
        first = None
        for eps in eps_list:
            hit, t = O.mt_hit(r1, r2, *P, eps, single=single)
            if first is not None:
                assert hit and t == first, (eps, t, first)
            elif hit:
                first = t
                grew += eps > 0
    assert grew > 10      # some of them need the safety parameter


@pytest.mark.parametrize("single", [False, True])
def test_tetra_and_cube_closed_forms(single):
    # unit tetra, ray along +x at (y, z) = (0.25, 0.25): chord 0.5
    m = M.single_tet()
    om = O.OracleMesh.from_mesh(m)
    geom = G.explicit(G.BEAM_PARALLEL, 1, 1, [[1, 0, 0, 0, 0.25, 0.25, 0, 1, 0, 0, 0, 1]])
    val, st = O.mt_project(om, geom, np.array([1.0]), single=single)
    assert abs(val.ravel()[0] - 0.5) < (1e-7 if single else 1e-15)
    assert st["crossings"] == 1 and st["lost"] == st["stuck"] == 0
    # Kuhn cube, generic axis-parallel ray: integral 1 through the 6 tets
    m = M.kuhn_cube()
    om = O.OracleMesh.from_mesh(m)
    geom = G.explicit(G.BEAM_PARALLEL, 1, 1, [[0, 0, 1, 0.1234, -0.0789, 0, 1, 0, 0, 0, 1, 0]])
    val, st = O.mt_project(om, geom, np.ones(6), single=single)
    assert abs(val.ravel()[0] - 1.0) < (1e-6 if single else 1e-14)
    assert st["lost"] == st["stuck"] == 0


def test_mt_f64_matches_exact_walker_on_generic_rays():
    """On rays in general position Alg. 2 and the exact SoS walker (a separate
    implementation: integer signs, brute-force face crossing) visit the same
    tets, and the chords agree to double rounding."""
    w = CF.workload("c2", n_angles=2, n_u=40, n_v=30)
    om = O.OracleMesh.from_mesh(w.mesh)
    mu = w.mu.astype(np.float64)
    p, st = O.project(om, w.geom, mu)
    q, st2 = O.mt_project(om, w.geom, mu)
    assert st2["crossings"] == st["crossings"] and st2["rays_hit"] == st["rays_hit"]
    assert st2["lost"] == st2["stuck"] == st2["escalations"] == 0
    np.testing.assert_allclose(q, p, rtol=1e-11, atol=1e-13)
    y = w.y.ravel().astype(np.float64)
    x, _ = O.backproject(om, w.geom, y)
    x2, _ = O.mt_backproject(om, w.geom, y)
    np.testing.assert_allclose(x2, x, rtol=1e-10, atol=1e-13)


def test_fig_singledouble_on_slivers():
    """fig:singledouble: on a mesh of slivers "the single
    precision numerical intersection code results in a high number of pixels
    where the ray-propagation integrals fail to terminate properly", while
    double precision traces them."""
    m = M.jittered_lattice_mesh(12, 1e-4, 5)
    om = O.OracleMesh.from_mesh(m)
    R = np.sqrt(3.0)
    geom = G.circular_cone(G.equidistant(4) + 0.1, 4 * R, 8 * R, 48, 48, 7.2 / 48, 7.2 / 48)
    mu = np.random.default_rng(0).uniform(0.5, 1.5, m.n_tets)
    p, st = O.project(om, geom, mu)
    q64, s64 = O.mt_project(om, geom, mu)
    q32, s32 = O.mt_project(om, geom, mu, single=True)
    assert s64["lost"] == s64["stuck"] == 0 and s64["crossings"] == st["crossings"]
    np.testing.assert_allclose(q64, p, rtol=1e-9, atol=1e-12)
    failed32 = s32["lost"] + s32["stuck"]
    assert failed32 > 0.1 * st["rays_hit"], s32


def test_swap_check_prevents_backtracking():
    """"An extra check thus needs to be performed when
    zero-length intersections are found, to ensure there is no backtracking
    by choosing the wrong face for the propagation of the ray, which can
    happen when a node exist with several tetrahedra" (fig:bad).  On lattice
    rays through the vertices of Kuhn meshes -- the fig:bad configuration --
    Alg. 2 with the swap check leaves fewer rays stuck and gives more rays
    the exact integral (the exact SoS walker's value) than without it."""
    for n in (2, 3, 4):
        m = M.kuhn_lattice(n)
        om = O.OracleMesh.from_mesh(m)
        geom = G.lattice_parallel((1 / n,) * 3, (0, 0, 0), 2 * n + 3, 2 * n + 3, G.LATTICE_DIRS)
        mu = np.ones(m.n_tets)
        p, _ = O.project(om, geom, mu)
        q1, s1 = O.mt_project(om, geom, mu, swap_check=True)
        q0, s0 = O.mt_project(om, geom, mu, swap_check=False)
        exact1 = int((np.abs(q1 - p) <= 1e-9 * np.maximum(p, 1)).sum())
        exact0 = int((np.abs(q0 - p) <= 1e-9 * np.maximum(p, 1)).sum())
        assert s1["stuck"] < s0["stuck"], (n, s1, s0)
        assert exact1 > exact0, (n, exact1, exact0)
