"""The C ABI from a C program (tests/native/abi_c_example.c): gcc builds it
against include/tetproj.h and the in-tree libtetproj.so.  On CPU the mesh
validates and creation reports TET_E_CUDA (no device); on the GPU one tet
and one ray give the closed-form chord 0.5: proj = 2 * 0.5,
x = 3 * 0.5, through a plan and without one."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run_example(tmp_path):
    from paper_1908_06909_b200 import _build
    _build.build()
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    libdir = os.path.dirname(_build.LIB)
    exe = str(tmp_path / "abi_c_example")
    subprocess.run([gcc, "-O1", "-Wall", "-Werror", os.path.join(ROOT, "tests", "native", "abi_c_example.c"),
                    "-o", exe, f"-L{libdir}", "-ltetproj", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=120).stdout
    return dict(line.split(" ", 1) for line in out.strip().splitlines())


def test_c_program_links_and_reports_statuses(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("the GPU variant below runs instead")
    r = _run_example(tmp_path)
    assert r["create"] == "5", r          # TET_E_CUDA: valid mesh, no device


@pytest.mark.gpu
def test_c_program_projects_one_tet(tmp_path):
    r = _run_example(tmp_path)
    assert r["create"] == "0" and r["plan"] == "0" and r["project"] == "0", r
    assert abs(float(r["proj"]) - 1.0) <= 1e-6 and r["crossings"] == "1" and r["lost"] == "0", r
    assert r["backproject"] == "0" and abs(float(r["x"]) - 1.5) <= 1e-6, r
    assert r["project_noplan"] == "0" and float(r["proj_noplan"]) == float(r["proj"]), r
