"""CPU-side checks of the C ABI: the library builds/loads and exports exactly what
include/blasx_cuda.h declares (no CUDA calls are made)."""

import ctypes
import os
import re

from conftest import ROOT
from paper_1510_05041_b200 import _native

HEADER = os.path.join(ROOT, "include", "blasx_cuda.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^int\s+(bx_\w+)\s*\(", src, flags=re.M)))


def test_header_and_binding_agree():
    assert declared() == _native.exported_symbols()


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native._LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
