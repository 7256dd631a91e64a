"""The C ABI used from plain C (examples/poisson3d.c): the header compiles as C11 and the program
links against libajm.so (CPU); on a GPU it solves a 3D Poisson system (GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2407_03272_b200")


def _build(tmp_path):
    import paper_2407_03272_b200.build as b
    b.build()
    exe = str(tmp_path / "poisson3d")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "poisson3d.c"), "-L", LIBDIR, "-lajm",
                           f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", exe])
    return exe


def test_c_example_builds_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_solves(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = _build(tmp_path)
    out = subprocess.run([exe, "32", "1e-10"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout)
    assert r["status"] == 0 and r["rel_residual"] <= 1e-10
    import paper_2407_03272_b200 as ajm
    assert r["max_abs_err"] <= 1e-6 and r["abi"] == ajm.ABI_VERSION
