/* Legacy BLAS ABI of the B200 engine: libblasx.so.
 *
 * The paper's backward-compatibility story:
 * an unmodified application linked against (or LD_PRELOADing) libblasx.so gets its level-3
 * calls served by the tiled multi-GPU runtime.  Every entry point builds the same
 * RoutineCall the cblas-style Python API builds (paper_1510_05041_b200/blas.py, which mirrors
 * /root/reference/pkg/src/tileblas/routines.py:49-67) and runs it through run_call
 * (scheduler.py:665-669 of the reference): host-resident column-major operands, output in
 * place.  The runtime's host side is Python (the north star keeps planner / scheduler / cache
 * in Python), so this library attaches to the process's interpreter, or starts an embedded
 * one when the caller is a plain C/Fortran program.
 *
 * Semantics follow reference BLAS / CBLAS: CblasRowMajor is mapped onto the column-major
 * routine (swapped operands / flipped flags), illegal arguments print the xerbla message
 * "** On entry to <NAME> parameter number <i> had an illegal value" and return without
 * touching any buffer, m==0 / n==0 return immediately, and beta==0 never reads C.
 * Unlike reference BLAS, a singular triangle in DTRSM is reported (status 6) instead of
 * producing inf/nan; blasx_last_status() returns the status of the calling thread's last
 * call (codes below).
 */
#ifndef BLASX_CBLAS_H
#define BLASX_CBLAS_H

#ifdef __cplusplus
extern "C" {
#endif

enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
enum CBLAS_UPLO { CblasUpper = 121, CblasLower = 122 };
enum CBLAS_DIAG { CblasNonUnit = 131, CblasUnit = 132 };
enum CBLAS_SIDE { CblasLeft = 141, CblasRight = 142 };

/* Status of the calling thread's last call:
 *    0  ok
 *   -i  parameter i was illegal (xerbla numbering: 1-based; cblas_* count Order as 1,
 *       the Fortran entry points start at their first argument)
 *    5  invalid argument rejected by the runtime (InvalidArgumentError)
 *    6  singular triangular matrix (SingularMatrixError; DTRSM only)
 *    7  device arena exhausted (ArenaOutOfMemoryError / CapacityDeadlockError)
 *   -100 the runtime could not be attached (no Python, package not importable, no GPU) */
int blasx_last_status(void);

/* Tile size used by the legacy entry points (default 1024, or $BLASX_TILE at first use). */
void blasx_set_tile(int tile);
int blasx_get_tile(void);

/* C <- alpha op(A) op(B) + beta C.  Replaces routines.py `gemm` (RoutineCall kind "gemm"). */
void cblas_dgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE transa, enum CBLAS_TRANSPOSE transb,
                 int m, int n, int k, double alpha, const double *A, int lda, const double *B,
                 int ldb, double beta, double *C, int ldc);
/* Single precision: TF32 tensor-core tile kernel with fp32 accumulation. */
void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE transa, enum CBLAS_TRANSPOSE transb,
                 int m, int n, int k, float alpha, const float *A, int lda, const float *B,
                 int ldb, float beta, float *C, int ldc);
/* stored triangle of C <- alpha op(A) op(A)^T + beta C   (routines.py `syrk`). */
void cblas_dsyrk(enum CBLAS_ORDER order, enum CBLAS_UPLO uplo, enum CBLAS_TRANSPOSE trans, int n,
                 int k, double alpha, const double *A, int lda, double beta, double *C, int ldc);
/* stored triangle of C <- alpha (op(A) op(B)^T + op(B) op(A)^T) + beta C   (`syr2k`). */
void cblas_dsyr2k(enum CBLAS_ORDER order, enum CBLAS_UPLO uplo, enum CBLAS_TRANSPOSE trans, int n,
                  int k, double alpha, const double *A, int lda, const double *B, int ldb,
                  double beta, double *C, int ldc);
/* C <- alpha sym(A) B + beta C (left) / alpha B sym(A) + beta C (right)   (`symm`). */
void cblas_dsymm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo, int m, int n,
                 double alpha, const double *A, int lda, const double *B, int ldb, double beta,
                 double *C, int ldc);
/* B <- alpha op(tri(A)) B / alpha B op(tri(A)), in place   (`trmm`). */
void cblas_dtrmm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo,
                 enum CBLAS_TRANSPOSE transa, enum CBLAS_DIAG diag, int m, int n, double alpha,
                 const double *A, int lda, double *B, int ldb);
/* op(tri(A)) X = alpha B / X op(tri(A)) = alpha B, X over B   (`trsm`). */
void cblas_dtrsm(enum CBLAS_ORDER order, enum CBLAS_SIDE side, enum CBLAS_UPLO uplo,
                 enum CBLAS_TRANSPOSE transa, enum CBLAS_DIAG diag, int m, int n, double alpha,
                 const double *A, int lda, double *B, int ldb);

/* Fortran 77 BLAS (column-major, every argument by reference; trailing hidden character
 * lengths are accepted and ignored). */
void dgemm_(const char *transa, const char *transb, const int *m, const int *n, const int *k,
            const double *alpha, const double *A, const int *lda, const double *B, const int *ldb,
            const double *beta, double *C, const int *ldc);
void sgemm_(const char *transa, const char *transb, const int *m, const int *n, const int *k,
            const float *alpha, const float *A, const int *lda, const float *B, const int *ldb,
            const float *beta, float *C, const int *ldc);
void dsyrk_(const char *uplo, const char *trans, const int *n, const int *k, const double *alpha,
            const double *A, const int *lda, const double *beta, double *C, const int *ldc);
void dsyr2k_(const char *uplo, const char *trans, const int *n, const int *k, const double *alpha,
             const double *A, const int *lda, const double *B, const int *ldb, const double *beta,
             double *C, const int *ldc);
void dsymm_(const char *side, const char *uplo, const int *m, const int *n, const double *alpha,
            const double *A, const int *lda, const double *B, const int *ldb, const double *beta,
            double *C, const int *ldc);
void dtrmm_(const char *side, const char *uplo, const char *transa, const char *diag, const int *m,
            const int *n, const double *alpha, const double *A, const int *lda, double *B,
            const int *ldb);
void dtrsm_(const char *side, const char *uplo, const char *transa, const char *diag, const int *m,
            const int *n, const double *alpha, const double *A, const int *lda, double *B,
            const int *ldb);

#ifdef __cplusplus
}
#endif
#endif
