/* libblasx.so: the legacy BLAS ABI (include/blasx_cblas.h) over the tiled multi-GPU runtime.
 *
 * BLASX's backward compatibility: an unmodified program that calls
 * cblas_dgemm / dgemm_ (linked, or LD_PRELOADed) is served by the runtime.  The runtime's host
 * side (planner, scheduler, tile cache) is Python by design, so each entry point hands its
 * arguments — CBLAS enums, sizes, scalars, raw host addresses — to
 * paper_1510_05041_b200/cblas.py, which validates them like reference BLAS, maps row-major
 * onto column-major and runs the call through run_call (reference scheduler.py:665-669).
 *
 * Attaching to Python without linking libpython: a Python process (ctypes.CDLL, an extension)
 * already exports the C API, found with dlsym(RTLD_DEFAULT); a plain C / Fortran process gets
 * an embedded interpreter from libpython (dlopen), started once with the build's
 * site-packages and this repository on sys.path, with the GIL released between calls so any
 * thread may enter through PyGILState_Ensure.  No torch, no CUDA here: the kernels live in
 * libblasx_cuda.so, loaded by the Python runtime.
 */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <libgen.h>

#include <pthread.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/blasx_cblas.h"

#ifndef BLASX_SITE
#define BLASX_SITE ""
#endif
#ifndef BLASX_LIBPYTHON
#define BLASX_LIBPYTHON "libpython3.12.so.1.0"
#endif

typedef void PyObj;
typedef struct {
    int (*IsInitialized)(void);
    void (*InitializeEx)(int);
    void *(*EvalSaveThread)(void);
    int (*GILEnsure)(void);
    void (*GILRelease)(int);
    PyObj *(*ImportModule)(const char *);
    PyObj *(*GetAttrString)(PyObj *, const char *);
    PyObj *(*CallObject)(PyObj *, PyObj *);
    PyObj *(*VaBuildValue)(const char *, va_list);
    long (*LongAsLong)(PyObj *);
    void (*DecRef)(PyObj *);
    void (*ErrPrint)(void);
    int (*RunSimpleString)(const char *);
} PyApi;

static PyApi py;
static pthread_once_t g_once = PTHREAD_ONCE_INIT;
static int g_ok = 0;
static PyObj *g_mod = NULL;
static __thread int g_status = 0;

#define SYM(h, name, field)                                                        \
    ((*(void **)&py.field = dlsym(h, name)) != NULL ||                             \
     (fprintf(stderr, "blasx: Python C API symbol %s not found\n", name), 0))

static int load_api(void *h) {
    return SYM(h, "Py_IsInitialized", IsInitialized) && SYM(h, "Py_InitializeEx", InitializeEx) &&
           SYM(h, "PyEval_SaveThread", EvalSaveThread) && SYM(h, "PyGILState_Ensure", GILEnsure) &&
           SYM(h, "PyGILState_Release", GILRelease) && SYM(h, "PyImport_ImportModule", ImportModule) &&
           SYM(h, "PyObject_GetAttrString", GetAttrString) &&
           SYM(h, "PyObject_CallObject", CallObject) && SYM(h, "Py_VaBuildValue", VaBuildValue) &&
           SYM(h, "PyLong_AsLong", LongAsLong) && SYM(h, "Py_DecRef", DecRef) &&
           SYM(h, "PyErr_Print", ErrPrint) && SYM(h, "PyRun_SimpleString", RunSimpleString);
}

/* repository root = the directory above the one holding this library */
static void repo_root(char *out, size_t n) {
    Dl_info info;
    char buf[4096];
    out[0] = 0;
    if (!dladdr((void *)&blasx_last_status, &info) || !info.dli_fname) return;
    snprintf(buf, sizeof buf, "%s", info.dli_fname);
    char *pkg = dirname(buf);
    char buf2[4096];
    snprintf(buf2, sizeof buf2, "%s", pkg);
    snprintf(out, n, "%s", dirname(buf2));
}

static void attach_once(void) {
    void *self = RTLD_DEFAULT;                         /* (void *)0 on glibc: test the symbol */
    if (!dlsym(RTLD_DEFAULT, "Py_IsInitialized")) {
        const char *lib = getenv("BLASX_LIBPYTHON");
        self = dlopen(lib && *lib ? lib : BLASX_LIBPYTHON, RTLD_NOW | RTLD_GLOBAL);
        if (!self) {
            fprintf(stderr, "blasx: cannot load %s: %s\n", lib && *lib ? lib : BLASX_LIBPYTHON, dlerror());
            return;
        }
    }
    if (!load_api(self)) return;
    int embedded = !py.IsInitialized();
    if (embedded) py.InitializeEx(0);                  /* no signal handlers: the host program owns them */
    int st = embedded ? 0 : py.GILEnsure();            /* a running host interpreter: take its GIL */
    char root[4096], code[16384];
    repo_root(root, sizeof root);
    const char *site = getenv("BLASX_SITE");
    if (!site || !*site) site = BLASX_SITE;
    snprintf(code, sizeof code,
             "import sys\n"
             "for _p, _front in ((r'''%s''', False), (r'''%s''', True)):\n"
             "    if _p and _p not in sys.path:\n"
             "        sys.path.insert(0, _p) if _front else sys.path.append(_p)\n",
             site, root);
    if (py.RunSimpleString(code) == 0) {
        g_mod = py.ImportModule("paper_1510_05041_b200.cblas");
        if (!g_mod) py.ErrPrint();
    }
    g_ok = g_mod != NULL;
    if (embedded) py.EvalSaveThread();                 /* release the GIL for PyGILState_Ensure callers */
    else py.GILRelease(st);
}

static int invoke(const char *fn, const char *fmt, ...) {
    pthread_once(&g_once, attach_once);
    if (!g_ok) return g_status = -100;
    int st = py.GILEnsure();
    int rc = -100;
    PyObj *f = py.GetAttrString(g_mod, fn);
    if (f) {
        va_list ap;
        va_start(ap, fmt);
        PyObj *args = py.VaBuildValue(fmt, ap);
        va_end(ap);
        if (args) {
            PyObj *r = py.CallObject(f, args);
            py.DecRef(args);
            if (r) {
                rc = (int)py.LongAsLong(r);
                py.DecRef(r);
            } else {
                py.ErrPrint();
            }
        } else {
            py.ErrPrint();
        }
        py.DecRef(f);
    } else {
        py.ErrPrint();
    }
    py.GILRelease(st);
    return g_status = rc;
}

typedef unsigned long long u64;
static inline u64 P(const void *p) { return (u64)(uintptr_t)p; }

static int f_trans(const char *c) {
    switch (c ? *c : 0) {
        case 'N': case 'n': return CblasNoTrans;
        case 'T': case 't': return CblasTrans;
        case 'C': case 'c': return CblasConjTrans;
        default: return 0;
    }
}
static int f_uplo(const char *c) {
    switch (c ? *c : 0) {
        case 'U': case 'u': return CblasUpper;
        case 'L': case 'l': return CblasLower;
        default: return 0;
    }
}
static int f_diag(const char *c) {
    switch (c ? *c : 0) {
        case 'N': case 'n': return CblasNonUnit;
        case 'U': case 'u': return CblasUnit;
        default: return 0;
    }
}
static int f_side(const char *c) {
    switch (c ? *c : 0) {
        case 'L': case 'l': return CblasLeft;
        case 'R': case 'r': return CblasRight;
        default: return 0;
    }
}

/* argument tuples of cblas.py's functions (api: 1 = cblas numbering, 0 = Fortran numbering) */
static const char *GEMM_FMT = "(iiiiiiidKiKidKii)";
static const char *SYRK_FMT = "(iiiiiidKidKi)";
static const char *SYR2K_FMT = "(iiiiiidKiKidKi)";
static const char *SYMM_FMT = "(iiiiiidKiKidKi)";
static const char *TRI_FMT = "(iiiiiiiidKiKi)";

#pragma GCC visibility push(default)

int blasx_last_status(void) { return g_status; }

void blasx_set_tile(int tile) { invoke("set_tile", "(i)", tile); }

int blasx_get_tile(void) { return invoke("get_tile", "()"); }

void cblas_dgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE transa, enum CBLAS_TRANSPOSE transb,
                 int m, int n, int k, double alpha, const double *A, int lda, const double *B,
                 int ldb, double beta, double *C, int ldc) {
    invoke("gemm", GEMM_FMT, 1, (int)order, (int)transa, (int)transb, m, n, k, alpha, P(A), lda,
           P(B), ldb, beta, P(C), ldc, 8);
}

void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE transa, enum CBLAS_TRANSPOSE transb,
                 int m, int n, int k, float alpha, const float *A, int lda, const float *B,
                 int ldb, float beta, float *C, int ldc) {
    invoke("gemm", GEMM_FMT, 1, (int)order, (int)transa, (int)transb, m, n, k, (double)alpha, P(A),
           lda, P(B), ldb, (double)beta, P(C), ldc, 4);
}

void cblas_dsyrk(enum CBLAS_ORDER order, enum CBLAS_UPLO uplo, enum CBLAS_TRANSPOSE trans, int n,
                 int k, double alpha, const double *A, int lda, double beta, double *C, int ldc) {
    invoke("syrk", SYRK_FMT, 1, (int)order, (int)uplo, (int)trans, n, k, alpha, P(A), lda, beta,
           P(C), ldc);
}

void cblas_dsyr2k(enum CBLAS_ORDER order, enum CBLAS_UPLO uplo, enum CBLAS_TRANSPOSE trans, int n,
                  int k, double alpha, const double *A, int lda, const double *B, int ldb,
                  double beta, double *C, int ldc) {
    invoke("syr2k", SYR2K_FMT, 1, (int)order, (int)uplo, (int)trans, n, k, alpha, P(A), lda, P(B),
           ldb, beta, P(C), ldc);
}

void cblas_dsymm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo, int m, int n,
                 double alpha, const double *A, int lda, const double *B, int ldb, double beta,
                 double *C, int ldc) {
    invoke("symm", SYMM_FMT, 1, (int)order, (int)side, (int)uplo, m, n, alpha, P(A), lda, P(B), ldb,
           beta, P(C), ldc);
}

void cblas_dtrmm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo,
                 enum CBLAS_TRANSPOSE transa, enum CBLAS_DIAG diag, int m, int n, double alpha,
                 const double *A, int lda, double *B, int ldb) {
    invoke("trmm", TRI_FMT, 1, (int)order, (int)side, (int)uplo, (int)transa, (int)diag, m, n, alpha,
           P(A), lda, P(B), ldb);
}

void cblas_dtrsm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo,
                 enum CBLAS_TRANSPOSE transa, enum CBLAS_DIAG diag, int m, int n, double alpha,
                 const double *A, int lda, double *B, int ldb) {
    invoke("trsm", TRI_FMT, 1, (int)order, (int)side, (int)uplo, (int)transa, (int)diag, m, n, alpha,
           P(A), lda, P(B), ldb);
}

void dgemm_(const char *transa, const char *transb, const int *m, const int *n, const int *k,
            const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
            const double *beta, double *C, const int *ldc) {
    invoke("gemm", GEMM_FMT, 0, (int)CblasColMajor, f_trans(transa), f_trans(transb), *m, *n, *k,
           *alpha, P(A), *lda, P(B), *ldb, *beta, P(C), *ldc, 8);
}

void sgemm_(const char *transa, const char *transb, const int *m, const int *n, const int *k,
            const float *alpha, const float *A, const int *lda, const float *B, const int *ldb,
            const float *beta, float *C, const int *ldc) {
    invoke("gemm", GEMM_FMT, 0, (int)CblasColMajor, f_trans(transa), f_trans(transb), *m, *n, *k,
           (double)*alpha, P(A), *lda, P(B), *ldb, (double)*beta, P(C), *ldc, 4);
}

void dsyrk_(const char *uplo, const char *trans, const int *n, const int *k, const double *alpha,
            const double *A, const int *lda, const double *beta, double *C, const int *ldc) {
    invoke("syrk", SYRK_FMT, 0, (int)CblasColMajor, f_uplo(uplo), f_trans(trans), *n, *k, *alpha,
           P(A), *lda, *beta, P(C), *ldc);
}

void dsyr2k_(const char *uplo, const char *trans, const int *n, const int *k, const double *alpha,
             const double *A, const int *lda, const double *B, const int *ldb, const double *beta,
             double *C, const int *ldc) {
    invoke("syr2k", SYR2K_FMT, 0, (int)CblasColMajor, f_uplo(uplo), f_trans(trans), *n, *k, *alpha,
           P(A), *lda, P(B), *ldb, *beta, P(C), *ldc);
}

void dsymm_(const char *side, const char *uplo, const int *m, const int *n, const double *alpha,
            const double *A, const int *lda, const double *B, const int *ldb, const double *beta,
            double *C, const int *ldc) {
    invoke("symm", SYMM_FMT, 0, (int)CblasColMajor, f_side(side), f_uplo(uplo), *m, *n, *alpha, P(A),
           *lda, P(B), *ldb, *beta, P(C), *ldc);
}

void dtrmm_(const char *side, const char *uplo, const char *transa, const char *diag, const int *m,
            const int *n, const double *alpha, const double *A, const int *lda, double *B,
            const int *ldb) {
    invoke("trmm", TRI_FMT, 0, (int)CblasColMajor, f_side(side), f_uplo(uplo), f_trans(transa),
           f_diag(diag), *m, *n, *alpha, P(A), *lda, P(B), *ldb);
}

void dtrsm_(const char *side, const char *uplo, const char *transa, const char *diag, const int *m,
            const int *n, const double *alpha, const double *A, const int *lda, double *B,
            const int *ldb) {
    invoke("trsm", TRI_FMT, 0, (int)CblasColMajor, f_side(side), f_uplo(uplo), f_trans(transa),
           f_diag(diag), *m, *n, *alpha, P(A), *lda, P(B), *ldb);
}

#pragma GCC visibility pop
