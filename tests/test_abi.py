"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol
include/ajm.h declares, and rejects bad arguments before touching a device.  No compute calls."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2407_03272_b200 as ajm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ajm.h")).read()
    decl = r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(ajm_[a-z_]+)\s*\("
    return sorted(set(re.findall(decl, src, flags=re.M)))


def test_library_built_and_loads():
    from paper_2407_03272_b200 import build
    build.build()
    L = ajm.lib()
    assert L.ajm_abi_version() == ajm.ABI_VERSION


def test_exports_every_header_symbol():
    syms = _header_symbols()
    assert set(syms) == set(ajm.ABI_SYMBOLS)
    L = ajm.lib()
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", ajm.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_sm100a_code_present():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ajm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_args_without_device():
    L = ajm.lib()
    h = ctypes.c_void_p()
    st = L.ajm_create(ctypes.byref(h), 0, 0, None, None, None, None, 0, None, 0, None)
    assert st == 1  # AJM_ERR_INVALID_ARG
    assert b"n must be" in L.ajm_last_error(None)
    st = L.ajm_create(None, 4, 4, None, None, None, None, 0, None, 0, None)
    assert st == 1
    st = L.ajm_create(ctypes.byref(h), 1 << 31, 4, None, None, None, None, 0, None, 0, None)
    assert st == 10  # AJM_ERR_UNSUPPORTED
    res = ajm.ajm_result_t()
    pol = ajm.ajm_policy_t(1, 1, 2)
    st = L.ajm_solve(None, None, 1e-6, 10, pol, None, ctypes.byref(res), None, None, None, 0, None)
    assert st == 1
    assert L.ajm_destroy(None) == 0


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2407_03272_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ajm_oracle" not in txt, f


def test_output_arguments_are_not_silently_converted():
    """Outputs (x_out, histories) are written in place: the binding raises on a wrong dtype or a
    non-contiguous buffer instead of handing the library a temporary copy."""
    import numpy as np
    import torch
    with pytest.raises(TypeError):
        ajm._ptr(np.zeros(4, dtype=np.float32), np.float64, output=True)
    with pytest.raises(TypeError):
        ajm._ptr(np.zeros((4, 2))[:, 0], np.float64, output=True)
    with pytest.raises(TypeError):
        ajm._ptr(torch.zeros(4, dtype=torch.float32), np.float64, output=True)
    with pytest.raises(TypeError):
        ajm._ptr(torch.zeros(4, 2, dtype=torch.float64)[:, 0], np.float64, output=True)
    a = np.zeros(4)
    p, keep = ajm._ptr(a, np.float64, output=True)
    assert keep is a and p.value == a.ctypes.data
    t = torch.zeros(4, dtype=torch.float64)
    p, keep = ajm._ptr(t, np.float64, output=True)
    assert keep is t and p.value == t.data_ptr()
    # inputs are still converted
    p, keep = ajm._ptr(np.zeros(4, dtype=np.float32), np.float64)
    assert keep.dtype == np.float64
