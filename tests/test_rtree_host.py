"""The R*-tree entry finder's host side (NEXT-3): built by
the product's own host code (rtree_host.cpp via prepare_mesh), compiled here
with g++ into a small harness, its invariants checked on CPU -- every hull
face in exactly one leaf, fan-out 4..10 below the root ("10 as maximum
number elements and 4 as minimum"), nested boxes.  Its GPU search is
checked against the oracle in tests/test_gpu_parity.py."""
import os
import struct
import subprocess

import numpy as np
import pytest

from workloads import configs as CF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1908_06909_b200", "csrc")


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("rt") / "rtree_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "native", "rtree_check.cpp"),
                           os.path.join(CSRC, "mesh_host.cpp"),
                           os.path.join(CSRC, "rtree_host.cpp"), "-o", exe])
    return exe


@pytest.mark.parametrize("cfg,faces", [("c1", 12), ("c2", 5944), ("c4a", 36300)])
def test_rtree_invariants(harness, tmp_path, cfg, faces):
    m = CF.workload(cfg, n_angles=1, n_u=2, n_v=2).mesh
    path = str(tmp_path / "mesh.bin")
    with open(path, "wb") as f:
        f.write(struct.pack("qqq", m.n_verts, m.n_tets, m.n_bfaces))
        for a, t in ((m.verts, np.float64), (m.tets, np.int32), (m.nbrs, np.int32),
                     (m.bfaces, np.int32)):
            f.write(np.ascontiguousarray(a, t).tobytes())
    out = subprocess.run([harness, path], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    nodes, n_faces, depth, bad = (int(x) for x in out.stdout.split())
    assert n_faces == faces and bad == 0
    # a balanced tree of fan-out 4..10 over B leaves entries is shallow
    assert depth <= int(np.ceil(np.log(max(faces, 2)) / np.log(4)))
