"""Build libblasx_cuda.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a),
and libblasx.so, the legacy cblas / Fortran BLAS ABI (plain C++, no CUDA; include/blasx_cblas.h).

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
CBLAS_LIB = os.path.join(PKG, "libblasx.so")
CBLAS_SRC = os.path.join(CSRC, "blasx_cblas.c")
CC = os.environ.get("CC", "gcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = SOURCES + DEPS + [os.path.join("..", "..", "include", "blasx_cuda.h")]
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in files
               if os.path.exists(os.path.join(CSRC, f)))


def _site_packages() -> str:
    import site
    for p in site.getsitepackages():
        if os.path.isdir(os.path.join(p, "numpy")):
            return p
    return ""


def _libpython() -> str:
    import sysconfig
    v = sysconfig.get_config_var("LDVERSION") or f"{sys.version_info[0]}.{sys.version_info[1]}"
    return f"libpython{v}.so.1.0"


def build_cblas(force: bool = False) -> str:
    """libblasx.so: plain C (gcc), no C++ runtime; bakes in this interpreter's site-packages and libpython name
    (used when the library has to start an embedded interpreter; overridable by $BLASX_SITE /
    $BLASX_LIBPYTHON)."""
    hdr = os.path.join(PKG, "..", "include", "blasx_cblas.h")
    if (not force and os.path.exists(CBLAS_LIB)
            and os.path.getmtime(CBLAS_LIB) >= max(os.path.getmtime(CBLAS_SRC), os.path.getmtime(hdr))):
        return CBLAS_LIB
    cmd = [CC, "-O2", "-std=gnu11", "-shared", "-fPIC", "-Wall", "-fvisibility=hidden",
           f'-DBLASX_SITE="{_site_packages()}"', f'-DBLASX_LIBPYTHON="{_libpython()}"',
           "-o", CBLAS_LIB, CBLAS_SRC, "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("gcc failed building libblasx.so")
    return CBLAS_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_cblas(force)
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
