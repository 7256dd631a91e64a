"""Build libajm.so (the C-ABI library of include/ajm.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libajm.so")
SOURCES = [os.path.join(CSRC, "ajm.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "ajm_kernels.cuh"), os.path.join(ROOT, "include", "ajm.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",          # no multiply-add contraction anywhere (R14)
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2,-fopenmp",  # OpenMP: the host layout planner's O(n) passes
    "-shared", "-cudart", "static", "-lgomp",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-o", tmp, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libajm.so")
    log = os.path.join(HERE, "csrc", "ptxas_log.txt")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if verbose:
        sys.stdout.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
