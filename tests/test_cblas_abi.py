"""Legacy BLAS ABI (libblasx.so, include/blasx_cblas.h).

CPU: the library builds, exports exactly the declared symbols, validates arguments like
reference BLAS (xerbla numbering, buffers untouched), takes the quick returns, and maps
CblasRowMajor / Fortran calls onto the right column-major RoutineCall — checked numerically
in-process through ctypes with the fake engine standing in for the GPUs.
GPU: a plain C program linked against libblasx.so (embedded interpreter) runs every routine
against naive loops (tests/c/cblas_app.c)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_1510_05041_b200 import _build

HEADER = os.path.join(ROOT, "include", "blasx_cblas.h")
APP_SRC = os.path.join(ROOT, "tests", "c", "cblas_app.c")

ROW, COL = 101, 102
NT, T = 111, 112
UP, LO = 121, 122
NU, UN = 131, 132
LEFT, RIGHT = 141, 142


@pytest.fixture(scope="module")
def libpath():
    return _build.build_cblas()


@pytest.fixture(scope="module")
def app(libpath, tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("capp") / "cblas_app")
    pkg = os.path.dirname(libpath)
    subprocess.run(["gcc", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", exe, APP_SRC,
                    "-L", pkg, "-lblasx", f"-Wl,-rpath,{pkg}", "-lm"], check=True)
    return exe


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:void|int)\s+(\w+)\s*\(", src, flags=re.M)))


def test_exports_match_header(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(line.split()[-1] for line in out.splitlines() if " T " in line)
    assert exported == declared()


def test_c_program_argument_checks(app):
    r = subprocess.run([app, "args"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "On entry to cblas_dgemm parameter number 9 had an illegal value" in r.stderr
    assert "On entry to DGEMM parameter number 13 had an illegal value" in r.stderr


def test_c_program_quick_returns(app):
    r = subprocess.run([app, "quick"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


# ----------------------------------------------------------------------------- in-process

D, I, P = ctypes.c_double, ctypes.c_int, ctypes.c_void_p


@pytest.fixture(scope="module")
def lib(libpath):
    L = ctypes.CDLL(libpath)
    L.blasx_last_status.restype = I
    L.cblas_dgemm.argtypes = [I, I, I, I, I, I, D, P, I, P, I, D, P, I]
    L.cblas_sgemm.argtypes = [I, I, I, I, I, I, ctypes.c_float, P, I, P, I, ctypes.c_float, P, I]
    L.cblas_dsyrk.argtypes = [I, I, I, I, I, D, P, I, D, P, I]
    L.cblas_dsyr2k.argtypes = [I, I, I, I, I, D, P, I, P, I, D, P, I]
    L.cblas_dsymm.argtypes = [I, I, I, I, I, D, P, I, P, I, D, P, I]
    L.cblas_dtrmm.argtypes = [I, I, I, I, I, I, I, D, P, I, P, I]
    L.cblas_dtrsm.argtypes = [I, I, I, I, I, I, I, D, P, I, P, I]
    return L


@pytest.fixture
def fake(monkeypatch):
    """Route run_call to the fake engine on one (fake) device."""
    from fake_engine import FakeEngine
    from paper_1510_05041_b200 import engine, scheduler
    from paper_1510_05041_b200.devices import DeviceDesc, Topology
    eng = FakeEngine(1, seed=5, arena_bytes=256 << 20)
    monkeypatch.setattr(engine, "get_engine", lambda *a, **k: eng)
    monkeypatch.setattr(scheduler, "discover_topology",
                        lambda: Topology([DeviceDesc(0, arena_capacity=256 << 20)]))
    return eng


def ptr(a):
    return a.ctypes.data


def test_inprocess_xerbla_leaves_buffers(lib, capfd):
    c = np.full(16, 3.0)
    lib.cblas_dgemm(COL, NT, NT, 4, 4, 4, 1.0, ptr(c), 4, ptr(c), 4, 1.0, ptr(c), 2)
    assert lib.blasx_last_status() == -14
    assert (c == 3.0).all()
    assert "parameter number 14" in capfd.readouterr().err


@pytest.mark.parametrize("ta,tb", [(NT, NT), (T, NT), (NT, T), (T, T)])
def test_rowmajor_dgemm_maps_to_colmajor(lib, fake, ta, tb):
    rng = np.random.default_rng(1)
    m, n, k = 70, 45, 33
    A = rng.uniform(-1, 1, (k, m) if ta == T else (m, k))       # row-major (C order) storage
    B = rng.uniform(-1, 1, (n, k) if tb == T else (k, n))
    C = rng.uniform(-1, 1, (m, n))
    ref = 0.5 * (A.T if ta == T else A) @ (B.T if tb == T else B) - 2.0 * C
    A, B = np.ascontiguousarray(A), np.ascontiguousarray(B)
    lib.cblas_dgemm(ROW, ta, tb, m, n, k, 0.5, ptr(A), A.shape[1], ptr(B), B.shape[1], -2.0,
                    ptr(C), n)
    assert lib.blasx_last_status() == 0
    np.testing.assert_allclose(C, ref, rtol=1e-12, atol=1e-12)


def test_colmajor_dgemm_with_padded_ld(lib, fake):
    rng = np.random.default_rng(2)
    m, n, k, ld = 50, 40, 30, 53
    Ab = rng.uniform(-1, 1, ld * k)
    Bb = rng.uniform(-1, 1, ld * n)
    Cb = rng.uniform(-1, 1, ld * n)
    view = lambda b, r, c: b[:ld * c].reshape(c, ld).T[:r]
    ref = view(Ab, m, k) @ view(Bb, k, n) + view(Cb, m, n)
    pad_before = Cb.reshape(n, ld)[:, m:].copy()
    lib.cblas_dgemm(COL, NT, NT, m, n, k, 1.0, ptr(Ab), ld, ptr(Bb), ld, 1.0, ptr(Cb), ld)
    assert lib.blasx_last_status() == 0
    np.testing.assert_allclose(view(Cb, m, n), ref, rtol=1e-12, atol=1e-12)
    assert (Cb.reshape(n, ld)[:, m:] == pad_before).all()       # rows beyond m untouched


@pytest.mark.parametrize("order", [ROW, COL])
@pytest.mark.parametrize("uplo", [UP, LO])
def test_syrk_syr2k_triangle_and_layout(lib, fake, order, uplo):
    rng = np.random.default_rng(3)
    n, k = 48, 20
    A = rng.uniform(-1, 1, (n, k))
    B = rng.uniform(-1, 1, (n, k))
    C0 = rng.uniform(-1, 1, (n, n))
    # storage in the caller's layout
    st = (lambda x: np.ascontiguousarray(x)) if order == ROW else (lambda x: np.asfortranarray(x))
    ld_a = k if order == ROW else n
    tri = np.tril if uplo == LO else np.triu
    other = (lambda x: np.triu(x, 1)) if uplo == LO else (lambda x: np.tril(x, -1))
    a, c = st(A), st(C0.copy())
    lib.cblas_dsyrk(order, uplo, NT, n, k, 1.5, ptr(a), ld_a, 0.5, ptr(c), n)
    assert lib.blasx_last_status() == 0
    full = 1.5 * A @ A.T + 0.5 * C0
    np.testing.assert_allclose(tri(c), tri(full), rtol=1e-12, atol=1e-12)
    assert (other(c) == other(C0)).all()
    a, b, c = st(A), st(B), st(C0.copy())
    lib.cblas_dsyr2k(order, uplo, NT, n, k, 1.0, ptr(a), ld_a, ptr(b), ld_a, 0.0, ptr(c), n)
    full = A @ B.T + B @ A.T
    np.testing.assert_allclose(tri(c), tri(full), rtol=1e-12, atol=1e-12)
    assert (other(c) == other(C0)).all()


@pytest.mark.parametrize("order", [ROW, COL])
@pytest.mark.parametrize("side", [LEFT, RIGHT])
def test_symm_trmm_trsm_layouts(lib, fake, order, side):
    rng = np.random.default_rng(4)
    m, n = 40, 28
    q = m if side == LEFT else n
    st = (lambda x: np.ascontiguousarray(x)) if order == ROW else (lambda x: np.asfortranarray(x))
    ldb = n if order == ROW else m
    S = rng.uniform(-1, 1, (q, q))
    B = rng.uniform(-1, 1, (m, n))
    C0 = rng.uniform(-1, 1, (m, n))
    sym = np.triu(S) + np.triu(S, 1).T                         # uplo = upper
    a, b, c = st(S), st(B), st(C0.copy())
    lib.cblas_dsymm(order, side, UP, m, n, 1.0, ptr(a), q, ptr(b), ldb, 1.0, ptr(c), ldb)
    assert lib.blasx_last_status() == 0
    ref = (sym @ B if side == LEFT else B @ sym) + C0
    np.testing.assert_allclose(c, ref, rtol=1e-12, atol=1e-12)

    L = np.tril(rng.uniform(-1, 1, (q, q))) / q + np.diag(1.0 + rng.uniform(0, 1, q))
    a = st(L + np.triu(np.full((q, q), np.nan), 1))            # unstored triangle never read
    b = st(B.copy())
    lib.cblas_dtrmm(order, side, LO, T, NU, m, n, 2.0, ptr(a), q, ptr(b), ldb)
    assert lib.blasx_last_status() == 0
    ref = 2.0 * (L.T @ B if side == LEFT else B @ L.T)
    np.testing.assert_allclose(b, ref, rtol=1e-12, atol=1e-12)
    lib.cblas_dtrsm(order, side, LO, T, NU, m, n, 0.5, ptr(a), q, ptr(b), ldb)
    assert lib.blasx_last_status() == 0
    np.testing.assert_allclose(b, B, rtol=1e-10, atol=1e-10)


def test_singular_trsm_status(lib, fake):
    q = 16
    a = np.asfortranarray(np.eye(q))
    a[5, 5] = 0.0
    b = np.asfortranarray(np.ones((q, 4)))
    lib.cblas_dtrsm(COL, LEFT, UP, NT, NU, q, 4, 1.0, ptr(a), q, ptr(b), q)
    assert lib.blasx_last_status() == 6


@pytest.mark.gpu
def test_c_program_on_gpu(app):
    r = subprocess.run([app, "compute", "300"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "compute: 0 failures" in r.stdout
