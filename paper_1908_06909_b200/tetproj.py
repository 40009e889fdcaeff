"""Thin ctypes binding of libtetproj (include/tetproj.h) -- argument
marshalling only; every step of the path runs in the CUDA library.

Names mirror the C ABI: ``tet_mesh_create``, ``tet_project``,
``tet_backproject``, ``tet_backproject_f64``, ``tet_mesh_info``,
``tet_mesh_destroy``.  Data arguments may be torch CUDA tensors (device
pointers, asynchronous on the current torch stream) or numpy arrays / torch
CPU tensors (host pointers; the library stages them through the device).

There is no CPU fallback: if ``libtetproj.so`` is missing or no CUDA device
is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _build

TET_OK, TET_E_ARG, TET_E_MESH, TET_E_NONCONVEX, TET_E_GEOMETRY, TET_E_CUDA, TET_E_NOMEM, \
    TET_E_RAYS = range(8)
TET_BEAM_CONE, TET_BEAM_PARALLEL = 0, 1
TET_F_FIX_ORIENTATION, TET_F_NO_REORDER, TET_F_STRICT = 1, 2, 4
_STATUS = ["TET_OK", "TET_E_ARG", "TET_E_MESH", "TET_E_NONCONVEX", "TET_E_GEOMETRY",
           "TET_E_CUDA", "TET_E_NOMEM", "TET_E_RAYS"]


class TetProjError(RuntimeError):
    def __init__(self, status: int, msg: str):
        name = _STATUS[status] if 0 <= status < len(_STATUS) else str(status)
        super().__init__(f"{name}: {msg}")
        self.status = status


class tet_geometry(C.Structure):
    _fields_ = [("beam", C.c_int32), ("n_angles", C.c_int32), ("n_v", C.c_int32),
                ("n_u", C.c_int32), ("vecs", C.POINTER(C.c_double))]


class tet_stats(C.Structure):
    _fields_ = [("rays", C.c_uint64), ("rays_hit", C.c_uint64), ("crossings", C.c_uint64),
                ("lost", C.c_uint64), ("stuck", C.c_uint64), ("exact_fallbacks", C.c_uint64),
                ("entry_conflicts", C.c_uint64), ("max_crossings_per_ray", C.c_uint32),
                ("_pad", C.c_uint32), ("escalations", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_ if k != "_pad"}


TET_TRAVERSE_EXACT, TET_TRAVERSE_MT_F64, TET_TRAVERSE_MT_F32 = 0, 1, 2


TET_ENTRY_RASTER, TET_ENTRY_BVH, TET_ENTRY_RTREE = 0, 1, 2


class tet_options(C.Structure):
    _fields_ = [("traversal", C.c_int32), ("max_escalations", C.c_int32), ("eps0", C.c_double),
                ("eps_growth", C.c_double), ("entry", C.c_int32), ("_reserved", C.c_int32)]


def options(traversal: int = TET_TRAVERSE_EXACT, eps0: float = 1e-9, eps_growth: float = 10.0,
            max_escalations: int = 12, entry: int = TET_ENTRY_RASTER) -> tet_options:
    """Traversal / entry-finder options; MT modes are the paper's Alg. 1/2
    (PAPER.md:79-144), TET_ENTRY_BVH the per-ray tree search."""
    return tet_options(traversal, max_escalations, eps0, eps_growth, entry, 0)


EXPORTS = ["tet_mesh_create", "tet_mesh_destroy", "tet_project", "tet_backproject",
           "tet_backproject_f64", "tet_mesh_info", "tet_mesh_features", "tet_last_error",
           "tet_set_kernel_timing", "tet_kernel_times", "tet_project_ex", "tet_backproject_ex",
           "tet_plan_create", "tet_plan_destroy", "tet_plan_project", "tet_plan_backproject",
           "tet_plan_backproject_f64"]
KERNEL_CLASSES = ["entry", "forward", "backward", "permute"]

_lib = None


def lib(build: bool = False) -> C.CDLL:
    """Load libtetproj.so (in-tree).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.DEBUG_LIB if os.environ.get("TETPROJ_DEBUG_LIB") == "1" else _build.LIB
    variant = os.environ.get("TETPROJ_LIB_VARIANT")   # A/B measurements (experiments/)
    if variant:
        path = os.path.join(os.path.dirname(_build.LIB), "variants", f"libtetproj_{variant}.so")
    if build or (not variant and os.environ.get("TETPROJ_DEBUG_LIB") != "1" and _build.stale()):
        _build.build()   # never load a library older than its sources
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_1908_06909_b200._build` "
                          "or __graft_entry__.build()")
    L = C.CDLL(path)
    P = C.c_void_p
    L.tet_mesh_create.argtypes = [P, C.c_int64, P, P, C.c_int64, P, C.c_int64, C.c_int,
                                  C.c_uint32, C.POINTER(C.c_void_p)]
    L.tet_mesh_destroy.argtypes = [P]
    L.tet_project.argtypes = [P, C.POINTER(tet_geometry), P, P, P, C.POINTER(tet_stats)]
    L.tet_backproject.argtypes = [P, C.POINTER(tet_geometry), P, P, C.c_int, P,
                                  C.POINTER(tet_stats)]
    L.tet_backproject_f64.argtypes = [P, C.POINTER(tet_geometry), P, P, P,
                                      C.POINTER(tet_stats)]
    L.tet_mesh_info.argtypes = [P, C.POINTER(C.c_int64)]
    L.tet_mesh_features.argtypes = [P, C.POINTER(C.c_int64)]
    L.tet_project_ex.argtypes = [P, C.POINTER(tet_geometry), P, P, C.POINTER(tet_options), P,
                                 C.POINTER(tet_stats)]
    L.tet_backproject_ex.argtypes = [P, C.POINTER(tet_geometry), P, P, C.c_int,
                                     C.POINTER(tet_options), P, C.POINTER(tet_stats)]
    L.tet_set_kernel_timing.argtypes = [P, C.c_int]
    L.tet_kernel_times.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.tet_plan_create.argtypes = [P, C.POINTER(tet_geometry), C.POINTER(tet_options), P,
                                  C.POINTER(C.c_void_p)]
    L.tet_plan_destroy.argtypes = [P, P]
    L.tet_plan_project.argtypes = [P, P, P, P, C.POINTER(tet_stats)]
    L.tet_plan_backproject.argtypes = [P, P, P, C.c_int, P, C.POINTER(tet_stats)]
    L.tet_plan_backproject_f64.argtypes = [P, P, P, P, C.POINTER(tet_stats)]
    L.tet_last_error.restype = C.c_char_p
    for f in EXPORTS:
        if f != "tet_last_error":
            getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _check(status: int):
    if status != TET_OK:
        raise TetProjError(status, lib().tet_last_error().decode())


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)


def _ptr(t, dtype, n):
    """(keepalive, void*) for a torch tensor (device or host) or numpy array."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            want = {np.float32: torch.float32, np.float64: torch.float64}[dtype]
            if t.dtype != want or not t.is_contiguous():
                raise TypeError(f"expected a contiguous {want} tensor")
            if t.numel() != n:
                raise ValueError(f"expected {n} elements, got {t.numel()}")
            return t, C.c_void_p(t.data_ptr())
    except ImportError:
        pass
    if not isinstance(t, np.ndarray) or t.dtype != dtype or not t.flags.c_contiguous:
        raise TypeError(f"expected a contiguous numpy {np.dtype(dtype).name} array")
    if t.size != n:
        raise ValueError(f"expected {n} elements, got {t.size}")
    return t, t.ctypes.data_as(C.c_void_p)


def _stream(stream, *tensors):
    if stream is not None:
        return C.c_void_p(int(stream))
    try:
        import torch
        for t in tensors:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    except ImportError:
        pass
    return C.c_void_p(0)


def _geom(g):
    vecs = np.ascontiguousarray(g.vecs, dtype=np.float64)
    assert vecs.shape == (g.n_angles, 12)
    s = tet_geometry(int(g.beam), int(g.n_angles), int(g.n_v), int(g.n_u),
                     vecs.ctypes.data_as(C.POINTER(C.c_double)))
    return s, vecs


@dataclass
class MeshHandle:
    ptr: C.c_void_p
    n_tets: int
    n_verts: int
    device: int

    def __del__(self):
        if self.ptr is not None and _lib is not None:
            _lib.tet_mesh_destroy(self.ptr)
            self.ptr = None


def tet_mesh_create(verts, tets, nbrs, bfaces, device: int = 0,
                    flags: int = TET_F_FIX_ORIENTATION) -> MeshHandle:
    v, pv = _host(verts, np.float64)
    t, pt = _host(tets, np.int32)
    n, pn = _host(nbrs, np.int32)
    b, pb = _host(bfaces, np.int32)
    assert v.ndim == 2 and v.shape[1] == 3 and t.shape[1:] == (4,) and n.shape == t.shape
    h = C.c_void_p()
    _check(lib().tet_mesh_create(pv, v.shape[0], pt, pn, t.shape[0], pb, b.shape[0], device,
                                 flags, C.byref(h)))
    return MeshHandle(h, int(t.shape[0]), int(v.shape[0]), device)


def tet_mesh_destroy(m: MeshHandle):
    if m.ptr is not None:
        _check(lib().tet_mesh_destroy(m.ptr))
        m.ptr = None


def tet_mesh_info(m: MeshHandle) -> dict:
    info = (C.c_int64 * 8)()
    _check(lib().tet_mesh_info(m.ptr, info))
    keys = ["n_verts", "n_tets", "n_bfaces", "device", "grid_exponent", "device_bytes",
            "l2_window_bytes", "reordered"]
    return dict(zip(keys, [int(x) for x in info]))


def tet_mesh_features(m: MeshHandle) -> dict:
    feat = (C.c_int64 * 4)()
    _check(lib().tet_mesh_features(m.ptr, feat))
    return {"walk": "ft16" if feat[0] else "rec", "tag16_bytes": int(feat[1]),
            "rtree_nodes": int(feat[2]), "bvh_nodes": int(feat[3])}


def tet_set_kernel_timing(m: MeshHandle, enable: bool = True):
    _check(lib().tet_set_kernel_timing(m.ptr, 1 if enable else 0))


def tet_kernel_times(m: MeshHandle) -> dict:
    """{class: (ms, launches)} accumulated since the last read (stream synced)."""
    ms = (C.c_double * 4)()
    n = (C.c_int64 * 4)()
    _check(lib().tet_kernel_times(m.ptr, ms, n))
    return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KERNEL_CLASSES)}


def tet_project(m: MeshHandle, geom, mu, proj, stream=None, stats: bool = False,
                opts: tet_options | None = None):
    """proj = A mu (Eq. 2).  Returns the stats dict when ``stats``."""
    g, keep = _geom(geom)
    _, pmu = _ptr(mu, np.float32, m.n_tets)
    _, pp = _ptr(proj, np.float32, geom.n_angles * geom.n_v * geom.n_u)
    st = tet_stats()
    sp = C.byref(st) if stats else None
    if opts is None:
        _check(lib().tet_project(m.ptr, C.byref(g), pmu, pp, _stream(stream, mu, proj), sp))
    else:
        _check(lib().tet_project_ex(m.ptr, C.byref(g), pmu, pp, C.byref(opts),
                                    _stream(stream, mu, proj), sp))
    return st.as_dict() if stats else None


def tet_backproject(m: MeshHandle, geom, proj, x, accumulate: bool = False, stream=None,
                    stats: bool = False, opts: tet_options | None = None):
    """x = A^T proj (Eq. 3), or x += A^T proj."""
    g, keep = _geom(geom)
    _, pp = _ptr(proj, np.float32, geom.n_angles * geom.n_v * geom.n_u)
    _, px = _ptr(x, np.float32, m.n_tets)
    st = tet_stats()
    sp = C.byref(st) if stats else None
    if opts is None:
        _check(lib().tet_backproject(m.ptr, C.byref(g), pp, px, 1 if accumulate else 0,
                                     _stream(stream, proj, x), sp))
    else:
        _check(lib().tet_backproject_ex(m.ptr, C.byref(g), pp, px, 1 if accumulate else 0,
                                        C.byref(opts), _stream(stream, proj, x), sp))
    return st.as_dict() if stats else None


def tet_backproject_f64(m: MeshHandle, geom, proj, acc, stream=None, stats: bool = False):
    """acc += A^T proj into a double device accumulator (multi-GPU partial sums)."""
    g, keep = _geom(geom)
    _, pp = _ptr(proj, np.float32, geom.n_angles * geom.n_v * geom.n_u)
    _, pa = _ptr(acc, np.float64, m.n_tets)
    st = tet_stats()
    _check(lib().tet_backproject_f64(m.ptr, C.byref(g), pp, pa, _stream(stream, proj, acc),
                                     C.byref(st) if stats else None))
    return st.as_dict() if stats else None


@dataclass
class PlanHandle:
    ptr: C.c_void_p
    mesh: MeshHandle          # the mesh must outlive the plan
    n_rays: int
    stream: int               # creation stream: the default stream of the destroy

    def __del__(self):
        if self.ptr is not None and _lib is not None and self.mesh.ptr is not None:
            _lib.tet_plan_destroy(self.ptr, C.c_void_p(self.stream))
            self.ptr = None


def tet_plan_create(m: MeshHandle, geom, opts: tet_options | None = None,
                    stream=None) -> PlanHandle:
    """Bind a scan to the mesh: geometry snapped once, entry map of every ray
    computed once (Alg. 2 "Read initial intersection element")."""
    g, keep = _geom(geom)
    h = C.c_void_p()
    sv = _stream(stream)
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                sv = C.c_void_p(torch.cuda.current_stream(m.device).cuda_stream)
        except ImportError:
            pass
    _check(lib().tet_plan_create(m.ptr, C.byref(g), C.byref(opts) if opts is not None else None,
                                 sv, C.byref(h)))
    return PlanHandle(h, m, geom.n_angles * geom.n_v * geom.n_u, int(sv.value or 0))


def tet_plan_destroy(p: PlanHandle, stream=None):
    if p.ptr is not None:
        _check(lib().tet_plan_destroy(p.ptr, C.c_void_p(int(stream)) if stream is not None
                                      else C.c_void_p(p.stream)))
        p.ptr = None


def tet_plan_project(p: PlanHandle, mu, proj, stream=None, stats: bool = False):
    _, pmu = _ptr(mu, np.float32, p.mesh.n_tets)
    _, pp = _ptr(proj, np.float32, p.n_rays)
    st = tet_stats()
    _check(lib().tet_plan_project(p.ptr, pmu, pp, _stream(stream, mu, proj),
                                  C.byref(st) if stats else None))
    return st.as_dict() if stats else None


def tet_plan_backproject(p: PlanHandle, proj, x, accumulate: bool = False, stream=None,
                         stats: bool = False):
    _, pp = _ptr(proj, np.float32, p.n_rays)
    _, px = _ptr(x, np.float32, p.mesh.n_tets)
    st = tet_stats()
    _check(lib().tet_plan_backproject(p.ptr, pp, px, 1 if accumulate else 0,
                                      _stream(stream, proj, x), C.byref(st) if stats else None))
    return st.as_dict() if stats else None


def tet_plan_backproject_f64(p: PlanHandle, proj, acc, stream=None, stats: bool = False):
    _, pp = _ptr(proj, np.float32, p.n_rays)
    _, pa = _ptr(acc, np.float64, p.mesh.n_tets)
    st = tet_stats()
    _check(lib().tet_plan_backproject_f64(p.ptr, pp, pa, _stream(stream, proj, acc),
                                          C.byref(st) if stats else None))
    return st.as_dict() if stats else None


class Plan:
    """A scan bound to a TetMesh (tet_plan_create): project / backproject
    without re-running the entry finder.  Use as a context manager or close()."""

    def __init__(self, mesh: "TetMesh", geom, opts: tet_options | None = None, stream=None):
        self.mesh = mesh
        self.geom = geom
        self.handle = tet_plan_create(mesh.handle, geom, opts, stream)

    def close(self, stream=None):
        tet_plan_destroy(self.handle, stream)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def project(self, mu, out=None, stats: bool = False):
        import torch
        if out is None:
            g = self.geom
            out = torch.empty((g.n_angles, g.n_v, g.n_u), dtype=torch.float32,
                              device=mu.device if isinstance(mu, torch.Tensor) else "cpu")
        st = tet_plan_project(self.handle, mu, out, stats=stats)
        return (out, st) if stats else out

    def backproject(self, proj, out=None, accumulate=False, stats: bool = False):
        import torch
        if out is None:
            out = torch.zeros(self.mesh.n_tets, dtype=torch.float32,
                              device=proj.device if isinstance(proj, torch.Tensor) else "cpu")
        st = tet_plan_backproject(self.handle, proj, out, accumulate, stats=stats)
        return (out, st) if stats else out

    def backproject_f64(self, proj, out=None, stats: bool = False):
        import torch
        if out is None:
            out = torch.zeros(self.mesh.n_tets, dtype=torch.float64,
                              device=proj.device if isinstance(proj, torch.Tensor) else "cpu")
        st = tet_plan_backproject_f64(self.handle, proj, out, stats=stats)
        return (out, st) if stats else out


class PlannedOperators:
    """``project(geom, mu)`` / ``backproject(geom, y)`` callables for the
    solvers (paper_1908_06909_b200.solvers) that bind each distinct scan --
    e.g. each OS-SART subset -- to a plan on first use, so the entry finder
    runs once per scan instead of once per call.  Plans live until close()."""

    def __init__(self, mesh: "TetMesh", opts: tet_options | None = None):
        self.mesh, self.opts, self.plans = mesh, opts, {}

    def plan(self, geom) -> Plan:
        vecs = np.ascontiguousarray(geom.vecs, dtype=np.float64)
        key = (int(geom.beam), int(geom.n_v), int(geom.n_u), vecs.tobytes())
        p = self.plans.get(key)
        if p is None:
            p = self.plans[key] = self.mesh.plan(geom, self.opts)
        return p

    def project(self, geom, mu):
        return self.plan(geom).project(mu)

    def backproject(self, geom, y):
        return self.plan(geom).backproject(y)

    def close(self):
        for p in self.plans.values():
            p.close()
        self.plans.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class TetMesh:
    """Convenience wrapper: a mesh resident on one GPU plus torch-facing ops."""

    def __init__(self, verts, tets, nbrs, bfaces, device: int = 0,
                 flags: int = TET_F_FIX_ORIENTATION):
        self.handle = tet_mesh_create(verts, tets, nbrs, bfaces, device, flags)
        self.device = device

    @classmethod
    def from_mesh(cls, mesh, device: int = 0, flags: int = TET_F_FIX_ORIENTATION):
        return cls(mesh.verts, mesh.tets, mesh.nbrs, mesh.bfaces, device, flags)

    @property
    def n_tets(self) -> int:
        return self.handle.n_tets

    def info(self) -> dict:
        return tet_mesh_info(self.handle)

    def plan(self, geom, opts: tet_options | None = None, stream=None) -> Plan:
        """Bind a scan: the entry finder runs once, here (tet_plan_create)."""
        return Plan(self, geom, opts, stream)

    def project(self, geom, mu, out=None, stats: bool = False, opts=None):
        import torch
        if out is None:
            out = torch.empty((geom.n_angles, geom.n_v, geom.n_u), dtype=torch.float32,
                              device=mu.device if isinstance(mu, torch.Tensor) else "cpu")
        st = tet_project(self.handle, geom, mu, out, stats=stats, opts=opts)
        return (out, st) if stats else out

    def backproject_f64(self, geom, proj, out=None, stats: bool = False):
        """acc = A^T proj in double (tet_backproject_f64 into a zeroed float64
        device tensor, or += into ``out``)."""
        import torch
        if out is None:
            out = torch.zeros(self.n_tets, dtype=torch.float64,
                              device=proj.device if isinstance(proj, torch.Tensor) else "cpu")
        st = tet_backproject_f64(self.handle, geom, proj, out, stats=stats)
        return (out, st) if stats else out

    def backproject(self, geom, proj, out=None, accumulate=False, stats: bool = False, opts=None):
        import torch
        if out is None:
            out = torch.zeros(self.n_tets, dtype=torch.float32,
                              device=proj.device if isinstance(proj, torch.Tensor) else "cpu")
        st = tet_backproject(self.handle, geom, proj, out, accumulate, stats=stats, opts=opts)
        return (out, st) if stats else out
