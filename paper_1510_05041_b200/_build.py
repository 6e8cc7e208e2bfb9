"""Build libblasx_cuda.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

The .so is git-ignored but travels with the repo snapshot to the GPU box; nothing is
JIT-compiled at import time."""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libblasx_cuda.so")
SOURCES = ["blasx_cuda.cu"]
DEPS = ["bx_gemm_dmma.cuh", "bx_trsm.cuh", "bx_sgemm_tc.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = SOURCES + DEPS + [os.path.join("..", "..", "include", "blasx_cuda.h")]
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in files
               if os.path.exists(os.path.join(CSRC, f)))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libblasx_cuda.so")
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
