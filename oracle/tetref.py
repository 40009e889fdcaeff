"""ctypes binding of the CPU oracle (oracle/tetref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package ``paper_1908_06909_b200``.
"""
from __future__ import annotations

import ctypes as C
import os
import socket
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tetref.c")
LIB = os.path.join(HERE, "libtetref.so")
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11",
          "-shared", "-fPIC", "-Wall", "-Wno-unused-function"]


# host-specific build: outside the tree, so it never travels to another machine
NATIVE_LIB = os.path.join(tempfile.gettempdir(),
                          f"tetproj_oracle_native_{socket.gethostname()}.so")
_native = False


def _stale(lib):
    return not os.path.exists(lib) or os.path.getmtime(lib) < max(
        os.path.getmtime(os.path.join(HERE, f)) for f in ("tetref.c", "tetref.h", "tetref_mt.inc"))


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no -march=native: the .so travels)."""
    if force or _stale(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def use_native() -> None:
    """Load the same source compiled -O3 -march=native for THIS host (the
    CPU-baseline timing build of SURVEY 8(d)); built on the machine that runs
    it, never shipped.  Must be called before the first oracle call."""
    global _native
    if _lib is not None:
        return
    if _stale(NATIVE_LIB):
        tmp = NATIVE_LIB + f".tmp{os.getpid()}"
        flags = ["-O3", "-march=native"] + [f for f in CFLAGS if f != "-O2"]
        subprocess.check_call(["gcc", *flags, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, NATIVE_LIB)
    _native = True


def build_flags() -> str:
    return "gcc -O3 -march=native -fopenmp" if _native else "gcc -O2 -fopenmp"


class _Geom(C.Structure):
    _fields_ = [("beam", C.c_int32), ("n_angles", C.c_int32), ("n_v", C.c_int32),
                ("n_u", C.c_int32), ("vecs", C.POINTER(C.c_double))]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("rays", "rays_hit", "crossings", "lost", "stuck", "max_crossings")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class MtOptions(C.Structure):
    _fields_ = [("single", C.c_int32), ("max_escalations", C.c_int32), ("eps0", C.c_double),
                ("eps_growth", C.c_double), ("no_swap_check", C.c_int32), ("_pad", C.c_int32)]


class MtStats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("rays", "rays_hit", "crossings", "lost", "stuck", "max_crossings", "escalations")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(NATIVE_LIB if _native else build())
        P = C.c_void_p
        _lib.tetref_mesh_create.argtypes = [P, C.c_int64, P, P, C.c_int64, P, C.c_int64,
                                            C.c_uint32, C.POINTER(C.c_void_p)]
        _lib.tetref_mesh_destroy.argtypes = [P]
        _lib.tetref_last_error.restype = C.c_char_p
        _lib.tetref_grid_spacing.argtypes = [P]
        _lib.tetref_grid_spacing.restype = C.c_double
        for fn in (_lib.tetref_project, _lib.tetref_backproject):
            fn.argtypes = [P, C.POINTER(_Geom), P, C.c_int64, P, P, C.c_int,
                           C.POINTER(Stats)]
        _lib.tetref_ray_path.argtypes = [P, C.POINTER(_Geom), C.c_int64, C.c_int64, P, P,
                                         C.POINTER(C.c_int64)]
        _lib.tetref_side.argtypes = [P, P, P, P]
        _lib.tetref_ray_points.argtypes = [P, C.POINTER(_Geom), C.c_int64, P, P]
        _lib.tetref_vertex_grid.argtypes = [P, P]
        for fn in (_lib.tetref_mt_project, _lib.tetref_mt_backproject):
            fn.argtypes = [P, C.POINTER(_Geom), P, C.c_int64, P, P, C.POINTER(MtOptions), C.c_int,
                           C.POINTER(MtStats)]
        for fn in (_lib.tetref_mt_hit_f64, _lib.tetref_mt_hit_f32):
            fn.argtypes = [P, P, P, P, P, C.c_double, C.POINTER(C.c_double)]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tetref error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc:
        raise OracleError(rc, lib().tetref_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class OracleMesh:
    """Validated mesh on the host (orientation fixed when ``fix=True``)."""

    def __init__(self, verts, tets, nbrs, bfaces, fix: bool = True):
        self._keep = [np.ascontiguousarray(verts, np.float64), np.ascontiguousarray(tets, np.int32),
                      np.ascontiguousarray(nbrs, np.int32), np.ascontiguousarray(bfaces, np.int32)]
        v, t, n, b = self._keep
        h = C.c_void_p()
        _check(lib().tetref_mesh_create(_ptr(v), len(v), _ptr(t), _ptr(n), len(t), _ptr(b),
                                        len(b), 1 if fix else 0, C.byref(h)))
        self.h = h
        self.n_tets = len(t)
        self.n_verts = len(v)

    @classmethod
    def from_mesh(cls, m, fix=True):
        return cls(m.verts, m.tets, m.nbrs, m.bfaces, fix)

    def __del__(self):
        if getattr(self, "h", None):
            lib().tetref_mesh_destroy(self.h)
            self.h = None

    @property
    def g(self) -> float:
        return lib().tetref_grid_spacing(self.h)

    def vertex_grid(self) -> np.ndarray:
        out = np.empty((self.n_verts, 3), np.int64)
        lib().tetref_vertex_grid(self.h, _ptr(out))
        return out


def _geom(geom):
    vecs = np.ascontiguousarray(geom.vecs, np.float64)
    g = _Geom(geom.beam, geom.n_angles, geom.n_v, geom.n_u,
              vecs.ctypes.data_as(C.POINTER(C.c_double)))
    return g, vecs


def project(mesh: OracleMesh, geom, mu, ray_ids=None, nthreads: int = 0):
    """Eq. 2 on the listed rays (all rays when None).  Returns (values, stats)."""
    g, keep = _geom(geom)
    mu = np.ascontiguousarray(mu, np.float64)
    assert mu.shape == (mesh.n_tets,)
    if ray_ids is None:
        out = np.zeros(geom.n_rays)
        ids = None
    else:
        ids = np.ascontiguousarray(ray_ids, np.int64)
        out = np.zeros(len(ids))
    st = Stats()
    _check(lib().tetref_project(mesh.h, C.byref(g), _ptr(mu), 0 if ids is None else len(ids),
                                None if ids is None else _ptr(ids), _ptr(out), nthreads,
                                C.byref(st)))
    if ray_ids is None:
        out = out.reshape(geom.n_angles, geom.n_v, geom.n_u)
    return out, st.as_dict()


def backproject(mesh: OracleMesh, geom, y, ray_ids=None, nthreads: int = 0):
    """Eq. 3 over the listed rays (y given per listed ray, or the full stack)."""
    g, keep = _geom(geom)
    y = np.ascontiguousarray(np.asarray(y, np.float64).ravel())
    ids = None if ray_ids is None else np.ascontiguousarray(ray_ids, np.int64)
    n = geom.n_rays if ids is None else len(ids)
    assert y.shape == (n,)
    x = np.zeros(mesh.n_tets)
    st = Stats()
    _check(lib().tetref_backproject(mesh.h, C.byref(g), _ptr(y), 0 if ids is None else n,
                                    None if ids is None else _ptr(ids), _ptr(x), nthreads,
                                    C.byref(st)))
    return x, st.as_dict()


def ray_path(mesh: OracleMesh, geom, ray_id: int, cap: int = 1 << 16):
    g, keep = _geom(geom)
    tets = np.empty(cap, np.int32)
    chords = np.empty(cap, np.float64)
    n = C.c_int64()
    _check(lib().tetref_ray_path(mesh.h, C.byref(g), int(ray_id), cap, _ptr(tets), _ptr(chords),
                                 C.byref(n)))
    k = min(n.value, cap)
    return tets[:k].copy(), chords[:k].copy()


def ray_points(mesh: OracleMesh, geom, ray_id: int):
    g, keep = _geom(geom)
    o = np.empty(3, np.int64)
    p = np.empty(3, np.int64)
    _check(lib().tetref_ray_points(mesh.h, C.byref(g), int(ray_id), _ptr(o), _ptr(p)))
    return o, p


def side(o, p, a, b) -> int:
    arrs = [np.ascontiguousarray(x, np.int64) for x in (o, p, a, b)]
    return int(lib().tetref_side(*[_ptr(x) for x in arrs]))


# ---- NEXT-1: the paper's own traversal (Alg. 1 + Alg. 2), oracle/tetref_mt.inc ----
def mt_options(single=False, eps0=1e-9, eps_growth=10.0, max_escalations=12, swap_check=True):
    return MtOptions(1 if single else 0, max_escalations, eps0, eps_growth,
                     0 if swap_check else 1, 0)


def mt_project(mesh: OracleMesh, geom, mu, single=False, ray_ids=None, nthreads: int = 0,
               **kw):
    """Eq. 2 with the paper's eps-MT traversal in double or float."""
    g, keep = _geom(geom)
    mu = np.ascontiguousarray(mu, np.float64)
    ids = None if ray_ids is None else np.ascontiguousarray(ray_ids, np.int64)
    out = np.zeros(geom.n_rays if ids is None else len(ids))
    st = MtStats()
    opt = mt_options(single, **kw)
    _check(lib().tetref_mt_project(mesh.h, C.byref(g), _ptr(mu), 0 if ids is None else len(ids),
                                   None if ids is None else _ptr(ids), _ptr(out), C.byref(opt),
                                   nthreads, C.byref(st)))
    if ids is None:
        out = out.reshape(geom.n_angles, geom.n_v, geom.n_u)
    return out, st.as_dict()


def mt_backproject(mesh: OracleMesh, geom, y, single=False, ray_ids=None, nthreads: int = 0,
                   **kw):
    """Eq. 3 with the paper's eps-MT traversal in double or float."""
    g, keep = _geom(geom)
    y = np.ascontiguousarray(np.asarray(y, np.float64).ravel())
    ids = None if ray_ids is None else np.ascontiguousarray(ray_ids, np.int64)
    x = np.zeros(mesh.n_tets)
    st = MtStats()
    opt = mt_options(single, **kw)
    _check(lib().tetref_mt_backproject(mesh.h, C.byref(g), _ptr(y), 0 if ids is None else len(ids),
                                       None if ids is None else _ptr(ids), _ptr(x), C.byref(opt),
                                       nthreads, C.byref(st)))
    return x, st.as_dict()


def mt_hit(r1, r2, p1, p2, p3, eps, single=False):
    """Alg. 1 on one triangle: (hit, t)."""
    arrs = [np.ascontiguousarray(a, np.float64) for a in (r1, r2, p1, p2, p3)]
    t = C.c_double()
    fn = lib().tetref_mt_hit_f32 if single else lib().tetref_mt_hit_f64
    hit = fn(*[_ptr(a) for a in arrs], float(eps), C.byref(t))
    return bool(hit), t.value
