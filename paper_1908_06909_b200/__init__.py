"""B200-native tetrahedral-mesh X-ray projector / backprojector (arXiv:1908.06909).

The product is the C-ABI library ``libtetproj.so`` (include/tetproj.h, CUDA
kernels for sm_100a in ``csrc/``); :mod:`.tetproj` is its thin ctypes binding
and :mod:`.dist` the multi-GPU angle-sharding driver.
"""
from .tetproj import (TET_BEAM_CONE, TET_BEAM_PARALLEL, TET_F_FIX_ORIENTATION,  # noqa: F401
                      TET_F_NO_REORDER, TET_F_STRICT, Plan, PlannedOperators, TetMesh,
                      TetProjError, tet_backproject, tet_backproject_f64, tet_mesh_create,
                      tet_mesh_destroy, tet_mesh_info, tet_plan_backproject, tet_plan_create,
                      tet_plan_destroy, tet_plan_project, tet_project)
