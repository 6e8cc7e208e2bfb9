"""Small calls that launch every kernel of libblasx_cuda.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool memcheck python tools/sanitize_small.py

FP64 task GEMM (interior and edge CTAs, all transposes, triangle epilogue, deferred beta
axpy, triangular-operand k-ranges), TRMM materialise, TRSM (inverse-based diagonal step:
identity + panel/leaf substitution + apply; and the substitution-only path), the tcgen05
SGEMM kernels (1-SM, 2-SM cluster, persistent) and the 3xTF32 split, host<->device tile
copies and the batched copy path.  Each call is checked against numpy so a kernel that a
sanitizer run disturbed is also caught."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1510_05041_b200 import RunOptions, _native, build_call, run_call  # noqa: E402


def check(name, call, opts, ref_fn, rtol):
    a = call.a.matrix.as_2d().astype(np.float64)
    b = call.b.matrix.as_2d().astype(np.float64) if call.b is not None else None
    c0 = call.c.matrix.as_2d().astype(np.float64)
    run_call(call, options=opts)
    got = call.c.matrix.as_2d().astype(np.float64)
    ref = ref_fn(a, b, c0)
    err = float(np.max(np.abs(got - ref)) / max(1e-30, np.max(np.abs(ref))))
    print(f"{name:40s} rel err {err:.2e}", flush=True)
    assert err < rtol, (name, err)


def tri(a, uplo, trans=False, unit=False):
    m = np.tril(a) if uplo == "lower" else np.triu(a)
    if unit:
        np.fill_diagonal(m, 1.0)
    return m.T if trans else m


def sgemm(lib):
    for variant in [int(v) for v in os.environ.get("BX_SAN_SGEMM", "0,1,2,3").split(",") if v]:
        lib.bx_set_sgemm_variant(variant)
        for precise in (False, True):
            call = build_call("gemm", m=600, n=520, k=512, tile_size=256, seed=6, beta=1.0,
                              dtype=np.float32)
            check(f"sgemm variant={variant} precise={precise}", call,
                  RunOptions(chunk_steps=2, sgemm_precise=precise), lambda a, b, c: a @ b + c, 2e-3)
    lib.bx_set_sgemm_variant(3)


def main():
    lib = _native.load()
    o = RunOptions(chunk_steps=2)
    if os.environ.get("BX_SAN_ONLY_SGEMM"):
        return sgemm(lib)
    for ta in (False, True):
        for tb in (False, True):
            call = build_call("gemm", m=700, n=600, k=520, tile_size=256, seed=1, alpha=0.5, beta=0.5,
                              trans_a=ta, trans_b=tb)
            check(f"dgemm ta={ta} tb={tb}", call, o,
                  lambda a, b, c, ta=ta, tb=tb: 0.5 * (a.T if ta else a) @ (b.T if tb else b) + 0.5 * c, 1e-12)
    call = build_call("syrk", m=600, n=600, k=300, tile_size=256, seed=2, beta=1.0, uplo="lower")
    check("dsyrk lower", call, o, lambda a, b, c: np.where(np.tril(np.ones_like(c)) > 0, a @ a.T + c, c), 1e-12)
    call = build_call("syr2k", m=600, n=600, k=300, tile_size=256, seed=3, beta=0.0, uplo="upper")
    check("dsyr2k upper", call, o,
          lambda a, b, c: np.where(np.triu(np.ones_like(c)) > 0, a @ b.T + b @ a.T, c), 1e-12)
    for side, uplo, trans in (("left", "lower", False), ("right", "upper", True)):
        call = build_call("trmm", m=600, n=520, k=600, tile_size=256, seed=4, side=side, uplo=uplo,
                          trans_a=trans, trsm_scaled=True)
        check(f"dtrmm {side} {uplo} trans={trans}", call, o,
              lambda a, b, c, s=side, u=uplo, t=trans: tri(a, u, t) @ c if s == "left" else c @ tri(a, u, t),
              1e-11)
    for side, uplo, trans, inv in (("left", "lower", False, 128), ("right", "upper", True, 128),
                                   ("left", "upper", False, 0)):
        call = build_call("trsm", m=600, n=520, k=600, tile_size=256, seed=5, side=side, uplo=uplo,
                          trans_a=trans, trsm_scaled=True)
        check(f"dtrsm {side} {uplo} trans={trans} inv={inv}", call,
              RunOptions(chunk_steps=2, trsm_inverse_min=inv),
              lambda a, b, c, s=side, u=uplo, t=trans: np.linalg.solve(tri(a, u, t), c) if s == "left"
              else np.linalg.solve(tri(a, u, t).T, c.T).T, 1e-10)
    sgemm(lib)
    print("sanitize_small: all kernels ran and matched", flush=True)


if __name__ == "__main__":
    main()
