"""The C-ABI library loads and exports every symbol include/*.h declares;
argument errors come back as statuses (CPU only: no compute calls)."""
import ctypes as C
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(tet_[a-z0-9_]+)\s*\(", src))
    return names


def test_header_declares_the_north_star_calls():
    d = _declared()
    for n in ("tet_mesh_create", "tet_project", "tet_backproject", "tet_mesh_destroy",
              "tet_last_error"):
        assert n in d


def test_library_exports_every_declared_symbol():
    from paper_1908_06909_b200 import _build, tetproj
    _build.build()
    L = tetproj.lib()
    for n in _declared():
        assert hasattr(L, n), n
        assert n in tetproj.EXPORTS


def test_null_arguments_are_statuses():
    from paper_1908_06909_b200 import tetproj
    L = tetproj.lib(build=True)
    assert L.tet_mesh_create(None, 0, None, None, 0, None, 0, 0, 0, None) == tetproj.TET_E_ARG
    assert L.tet_project(None, None, None, None, None, None) == tetproj.TET_E_ARG
    assert L.tet_backproject(None, None, None, None, 0, None, None) == tetproj.TET_E_ARG
    assert L.tet_mesh_destroy(None) == tetproj.TET_OK
    h = C.c_void_p(1)
    assert L.tet_plan_create(None, None, None, None, C.byref(h)) == tetproj.TET_E_ARG
    assert h.value is None                      # *out cleared on error
    assert L.tet_plan_create(None, None, None, None, None) == tetproj.TET_E_ARG
    assert L.tet_plan_project(None, None, None, None, None) == tetproj.TET_E_ARG
    assert L.tet_plan_backproject(None, None, None, 0, None, None) == tetproj.TET_E_ARG
    assert L.tet_plan_backproject_f64(None, None, None, None, None) == tetproj.TET_E_ARG
    assert L.tet_plan_destroy(None, None) == tetproj.TET_OK
    assert isinstance(L.tet_last_error(), bytes)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1908_06909_b200 import tetproj
    from workloads import meshes as M
    m = M.kuhn_cube()
    with pytest.raises(tetproj.TetProjError) as e:
        tetproj.tet_mesh_create(m.verts, m.tets, m.nbrs, m.bfaces, device=0)
    assert e.value.status == tetproj.TET_E_CUDA


@pytest.mark.parametrize("case,want", [("l_shaped", "TET_E_NONCONVEX"),
                                       ("two_tets", "TET_E_NONCONVEX"),
                                       ("carved", "TET_E_MESH")])
def test_library_mesh_validation_statuses(case, want):
    """tet_mesh_create validates on the host before touching the device, so
    its exact checks are pinned here without a GPU: the L-shaped lattice
    (reflex hull edges) and two disjoint tets (no reflex edge: only the global
    all-vertices-against-all-hull-planes check catches it) are rejected as
    non-convex, a carved lattice as a non-manifold mesh."""
    from paper_1908_06909_b200 import tetproj
    from workloads import meshes as M
    if case == "l_shaped":
        m = M.l_shaped_lattice()
        t, nb, bf = m.tets, m.nbrs, m.bfaces
    elif case == "two_tets":
        m = M.two_disjoint_tets()
        t, nb, bf = m.tets, m.nbrs, m.bfaces
    else:
        m = M.kuhn_lattice(2)
        t = m.tets[[i for i in range(m.n_tets) if i % 7 != 3]]
        nb, bf = M.build_graph(t)
    with pytest.raises(tetproj.TetProjError) as e:
        tetproj.tet_mesh_create(m.verts, t, nb, bf, device=0)
    assert e.value.status == getattr(tetproj, want), str(e.value)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1908_06909_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if os.path.isfile(f) and f.endswith((".py", ".cu", ".cpp", ".h")):
            src = open(f).read()
            assert "import oracle" not in src and "from oracle" not in src, f
            assert "tetref" not in src, f
