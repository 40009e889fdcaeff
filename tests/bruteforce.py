"""Exact-rational brute force used to PIN the oracle (tests only).

Independent of oracle/tetref.c: no Plücker signs, no walk, no SoS table.
For every (ray, tet) pair the line o + t (p - o) is clipped against the four
closed half-spaces of the tet with exact rational arithmetic (Python ints /
Fractions).  A face plane that contains the line is resolved by the limit of
the translated line o + w(d), w = (d, d^2, d^4), d -> 0+: the line is inside
that half-space iff the first non-zero component of the outward normal is
negative.  This is the limit definition a_ij = lim |line_j(d) ∩ T_i| of
DESIGN.md reading R2 (the chord is continuous in the line everywhere except
on coplanar configurations, where the translation decides).

Also here: the numeric contract's snapping written a third time (from the
DESIGN.md text) and the SoS sign evaluated from the full delta-polynomial.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


# ----------------------------------------------------------- snapping ------
def grid_of(verts: np.ndarray):
    """(g, C) per DESIGN.md 'Numeric contract'."""
    lo, hi = verts.min(0), verts.max(0)
    c = [0.5 * (float(lo[i]) + float(hi[i])) for i in range(3)]
    r = max(abs(float(verts[v, i]) - c[i]) for v in range(len(verts)) for i in range(3))
    m, k = math.frexp(64.0 * r)
    e = (k - 1 if m == 0.5 else k) - 30
    g = math.ldexp(1.0, e)
    C = [round(c[i] / g) * g for i in range(3)]   # Python round(): half-even
    return g, C


def snap_verts(verts: np.ndarray):
    g, C = grid_of(verts)
    return [[int(round((float(v[i]) - C[i]) / g)) for i in range(3)] for v in verts], g, C


def ray_points(geom, g, C, ray_id: int):
    per = geom.n_v * geom.n_u
    a, rem = divmod(ray_id, per)
    v, u = divmod(rem, geom.n_u)
    q = [float(x) for x in geom.vecs[a]]
    P00 = [int(round((q[3 + i] - C[i]) / g)) for i in range(3)]
    U = [int(round(q[6 + i] / g)) for i in range(3)]
    V = [int(round(q[9 + i] / g)) for i in range(3)]
    p = [P00[i] + u * U[i] + v * V[i] for i in range(3)]
    if geom.beam == 0:
        o = [int(round((q[i] - C[i]) / g)) for i in range(3)]
    else:
        mx = max(abs(q[0]), abs(q[1]), abs(q[2]))
        d = [int(round((q[i] / mx) * 1048576.0)) for i in range(3)]
        o = [p[i] - d[i] for i in range(3)]
    return o, p


# ------------------------------------------------------------ algebra ------
def sub(a, b):
    return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]


def dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


# ------------------------------------------------------------ clipping -----
def tet_interval(P, o, D):
    """Exact parameter interval [lo, hi] of line o + t D inside the closed tet
    with vertices P (4 integer 3-vectors), coplanar faces resolved by the
    translation limit.  Returns None when the limit line misses the tet."""
    lo = hi = None
    for k in range(4):
        a, b, c = [P[j] for j in range(4) if j != k]
        n = cross(sub(b, a), sub(c, a))
        if dot(n, sub(P[k], a)) > 0:
            n = [-n[0], -n[1], -n[2]]          # outward
        s0, sd = dot(n, sub(o, a)), dot(n, D)
        if sd == 0:
            if s0 > 0:
                return None
            if s0 == 0:
                first = next(x for x in n if x != 0)
                if first > 0:
                    return None
            continue
        ts = Fraction(-s0, sd)
        if sd > 0:
            hi = ts if hi is None else min(hi, ts)
        else:
            lo = ts if lo is None else max(lo, ts)
    if lo is None or hi is None or hi < lo:
        return None
    return lo, hi


def chords_of_ray(Pg, tets, o, p, g):
    """{tet: chord in world units} for every tet with a non-empty interval."""
    D = sub(p, o)
    L = math.sqrt(float(dot(D, D))) * g
    out = {}
    for t, tet in enumerate(tets):
        iv = tet_interval([Pg[int(n)] for n in tet], o, D)
        if iv is not None:
            out[t] = float(iv[1] - iv[0]) * L
    return out


def dense_A(mesh, geom, ray_ids=None):
    """Materialised A [n_rays, n_tets] (SPEC.md:295 dense-matrix oracle)."""
    Pg, g, C = snap_verts(mesh.verts)
    ids = range(geom.n_rays) if ray_ids is None else ray_ids
    A = np.zeros((len(ids), mesh.n_tets))
    for r, rid in enumerate(ids):
        o, p = ray_points(geom, g, C, int(rid))
        for t, ch in chords_of_ray(Pg, mesh.tets, o, p, g).items():
            A[r, t] = ch
    return A


# ---------------------------------------------------- SoS polynomial ------
def _padd(a, b):
    out = dict(a)
    for k, v in b.items():
        out[k] = out.get(k, 0) + v
    return out


def _pmul(a, b):
    out = {}
    for ka, va in a.items():
        for kb, vb in b.items():
            out[ka + kb] = out.get(ka + kb, 0) + va * vb
    return out


def _pneg(a):
    return {k: -v for k, v in a.items()}


def sos_sign_polynomial(o, p, a, b) -> int:
    """Sign, as delta -> 0+, of det[a - o(d), b - o(d), p(d) - o(d)] with
    o(d) = o + (d, d^2, d^4) and p(d) = p + (d, d^2, d^4) + (d^8, d^16, d^32):
    expand the full polynomial and take its lowest-order non-zero coefficient."""
    w = [{1: 1}, {2: 1}, {4: 1}]
    u = [{8: 1}, {16: 1}, {32: 1}]
    A = [_padd({0: a[i] - o[i]}, _pneg(w[i])) for i in range(3)]
    B = [_padd({0: b[i] - o[i]}, _pneg(w[i])) for i in range(3)]
    Dv = [_padd({0: p[i] - o[i]}, u[i]) for i in range(3)]

    def pc(x, y):  # polynomial cross product
        return [_padd(_pmul(x[1], y[2]), _pneg(_pmul(x[2], y[1]))),
                _padd(_pmul(x[2], y[0]), _pneg(_pmul(x[0], y[2]))),
                _padd(_pmul(x[0], y[1]), _pneg(_pmul(x[1], y[0])))]

    AB = pc(A, B)
    det = _padd(_padd(_pmul(Dv[0], AB[0]), _pmul(Dv[1], AB[1])), _pmul(Dv[2], AB[2]))
    for k in sorted(det):
        if det[k] != 0:
            return 1 if det[k] > 0 else -1
    return 0
