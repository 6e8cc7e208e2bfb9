/* A legacy BLAS application: links libblasx.so like it would link any cblas / Fortran BLAS.
 * Built and run by tests/test_cblas_abi.py.
 *   cblas_app args     illegal arguments -> xerbla message + status, buffers untouched
 *   cblas_app quick    quick returns (m=0, alpha=0 / k=0 scaling) - no device needed
 *   cblas_app compute  every routine (cblas row/col-major + Fortran) vs naive loops (GPU) */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "blasx_cblas.h"

static int fails = 0;
#define CHECK(c, ...) do { if (!(c)) { fails++; printf("FAIL %s:%d ", __FILE__, __LINE__); printf(__VA_ARGS__); printf("\n"); } } while (0)

static double rnd(unsigned *s) { *s = *s * 1103515245u + 12345u; return ((*s >> 8) & 0xffff) / 32768.0 - 1.0; }
static double *mat(int n, unsigned seed) { double *p = malloc(sizeof(double) * (n ? n : 1)); for (int i = 0; i < n; i++) p[i] = rnd(&seed); return p; }

/* element (i,j) of a stored matrix in either layout */
#define EL(p, ld, i, j, row) (*((row) ? &(p)[(long)(i) * (ld) + (j)] : &(p)[(long)(j) * (ld) + (i)]))

static double maxdiff(const double *a, const double *b, int n) { double m = 0; for (int i = 0; i < n; i++) { double d = fabs(a[i] - b[i]); if (d > m || d != d) m = d != d ? 1e300 : d; } return m; }

static void ref_gemm(int row, int ta, int tb, int m, int n, int k, double al, const double *A, int lda, const double *B, int ldb, double be, double *C, int ldc) {
    for (int i = 0; i < m; i++) for (int j = 0; j < n; j++) {
        double s = 0;
        for (int p = 0; p < k; p++) s += (ta ? EL(A, lda, p, i, row) : EL(A, lda, i, p, row)) * (tb ? EL(B, ldb, j, p, row) : EL(B, ldb, p, j, row));
        double c0 = be == 0 ? 0 : be * EL(C, ldc, i, j, row);
        EL(C, ldc, i, j, row) = al * s + c0;
    }
}

static int args_mode(void) {
    double A[16] = {0}, B[16] = {0}, C[16];
    for (int i = 0; i < 16; i++) C[i] = 7;
    cblas_dgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, 4, 4, 4, 1.0, A, 2, B, 4, 1.0, C, 4);
    CHECK(blasx_last_status() == -9, "lda<m -> param 9, got %d", blasx_last_status());
    cblas_dgemm(CblasRowMajor, CblasNoTrans, CblasTrans, 4, 4, 3, 1.0, A, 2, B, 4, 1.0, C, 4);
    CHECK(blasx_last_status() == -9, "row-major lda<k -> param 9, got %d", blasx_last_status());
    cblas_dgemm((enum CBLAS_ORDER)7, CblasNoTrans, CblasNoTrans, 4, 4, 4, 1.0, A, 4, B, 4, 1.0, C, 4);
    CHECK(blasx_last_status() == -1, "bad order -> 1, got %d", blasx_last_status());
    cblas_dgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, -1, 4, 4, 1.0, A, 4, B, 4, 1.0, C, 4);
    CHECK(blasx_last_status() == -4, "m<0 -> 4, got %d", blasx_last_status());
    int m = 4, n = 4, k = 4, bad = 1; double one = 1.0;
    dgemm_("X", "N", &m, &n, &k, &one, A, &m, B, &k, &one, C, &bad);
    CHECK(blasx_last_status() == -1, "fortran bad transa -> 1, got %d", blasx_last_status());
    dgemm_("N", "N", &m, &n, &k, &one, A, &m, B, &k, &one, C, &bad);
    CHECK(blasx_last_status() == -13, "fortran ldc -> 13, got %d", blasx_last_status());
    cblas_dsyrk(CblasColMajor, (enum CBLAS_UPLO)0, CblasNoTrans, 4, 4, 1.0, A, 4, 1.0, C, 4);
    CHECK(blasx_last_status() == -2, "syrk uplo -> 2, got %d", blasx_last_status());
    cblas_dtrsm(CblasColMajor, CblasLeft, CblasLower, CblasNoTrans, (enum CBLAS_DIAG)5, 4, 4, 1.0, A, 4, B, 4);
    CHECK(blasx_last_status() == -5, "trsm diag -> 5, got %d", blasx_last_status());
    cblas_dtrmm(CblasColMajor, CblasRight, CblasLower, CblasNoTrans, CblasUnit, 4, 4, 1.0, A, 3, B, 4);
    CHECK(blasx_last_status() == -10, "trmm lda -> 10, got %d", blasx_last_status());
    cblas_dsymm(CblasColMajor, CblasLeft, CblasUpper, 4, 4, 1.0, A, 4, B, 4, 1.0, C, 3);
    CHECK(blasx_last_status() == -13, "symm ldc -> 13, got %d", blasx_last_status());
    cblas_dsyr2k(CblasColMajor, CblasLower, CblasTrans, 4, 5, 1.0, A, 4, B, 5, 1.0, C, 4);
    CHECK(blasx_last_status() == -8, "syr2k lda<k (trans) -> 8, got %d", blasx_last_status());
    for (int i = 0; i < 16; i++) CHECK(C[i] == 7, "C touched by an illegal call");
    return 0;
}

static int quick_mode(void) {
    double C[12], A[12], B[12];
    for (int i = 0; i < 12; i++) { C[i] = i + 1; A[i] = NAN; B[i] = NAN; }
    cblas_dgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, 0, 3, 4, 1.0, A, 1, B, 4, 2.0, C, 1);
    CHECK(blasx_last_status() == 0 && C[0] == 1, "m=0 quick return");
    cblas_dgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, 3, 3, 4, 0.0, A, 3, B, 4, 2.0, C, 4);
    CHECK(blasx_last_status() == 0, "alpha=0 status %d", blasx_last_status());
    for (int j = 0; j < 3; j++) for (int i = 0; i < 4; i++)
        CHECK(C[j * 4 + i] == (i < 3 ? 2.0 : 1.0) * (j * 4 + i + 1), "alpha=0 scaling C[%d,%d]=%g", i, j, C[j * 4 + i]);
    cblas_dgemm(CblasRowMajor, CblasNoTrans, CblasNoTrans, 2, 2, 0, 1.0, A, 1, B, 2, 0.0, C, 4);
    CHECK(C[0] == 0 && C[1] == 0 && C[4] == 0 && C[5] == 0 && C[2] != 0, "k=0 beta=0 zeroes C (row-major)");
    double Bt[6] = {1, 2, 3, 4, 5, 6};
    cblas_dtrsm(CblasColMajor, CblasLeft, CblasLower, CblasNoTrans, CblasNonUnit, 2, 3, 0.0, A, 2, Bt, 2);
    for (int i = 0; i < 6; i++) CHECK(Bt[i] == 0, "trsm alpha=0 zeroes B");
    blasx_set_tile(256);
    CHECK(blasx_get_tile() == 256, "tile setter");
    return 0;
}

static int compute_mode(int n) {
    int k = n - 37, lda = n + 3;
    unsigned seed = 1;
    for (int row = 0; row < 2; row++)
    for (int ta = 0; ta < 2; ta++) for (int tb = 0; tb < 2; tb++) {
        int m = n, nn = n - 5;
        double *A = mat(lda * n, seed++), *B = mat(lda * n, seed++), *C = mat(lda * n, seed++);
        double *R = malloc(sizeof(double) * lda * n); memcpy(R, C, sizeof(double) * lda * n);
        cblas_dgemm(row ? CblasRowMajor : CblasColMajor, ta ? CblasTrans : CblasNoTrans, tb ? CblasTrans : CblasNoTrans,
                    m, nn, k, 0.75, A, lda, B, lda, -0.5, C, lda);
        ref_gemm(row, ta, tb, m, nn, k, 0.75, A, lda, B, lda, -0.5, R, lda);
        double d = maxdiff(C, R, lda * n);
        CHECK(blasx_last_status() == 0 && d < 1e-10, "dgemm row=%d ta=%d tb=%d: status %d maxdiff %g", row, ta, tb, blasx_last_status(), d);
        free(A); free(B); free(C); free(R);
    }
    /* Fortran dgemm_ */
    {
        int m = n, nn = n, kk = n, ld = n; double al = 1.0, be = 1.0;
        double *A = mat(n * n, 11), *B = mat(n * n, 12), *C = mat(n * n, 13), *R = malloc(sizeof(double) * n * n);
        memcpy(R, C, sizeof(double) * n * n);
        dgemm_("T", "n", &m, &nn, &kk, &al, A, &ld, B, &ld, &be, C, &ld);
        ref_gemm(0, 1, 0, n, n, n, 1.0, A, n, B, n, 1.0, R, n);
        double d = maxdiff(C, R, n * n);
        CHECK(blasx_last_status() == 0 && d < 1e-10, "dgemm_: maxdiff %g", d);
        free(A); free(B); free(C); free(R);
    }
    /* syrk / syr2k (row-major lower == col-major upper of the transposed storage) */
    for (int row = 0; row < 2; row++) {
        double *A = mat(n * n, 21), *B = mat(n * n, 22), *C = mat(n * n, 23), *R = malloc(sizeof(double) * n * n), *R2 = malloc(sizeof(double) * n * n);
        memcpy(R, C, sizeof(double) * n * n);
        cblas_dsyrk(row ? CblasRowMajor : CblasColMajor, CblasLower, CblasNoTrans, n, n, 1.0, A, n, 1.0, C, n);
        /* reference: full product restricted to the lower triangle, in the caller's layout */
        memcpy(R2, R, sizeof(double) * n * n);
        ref_gemm(row, 0, 1, n, n, n, 1.0, A, n, A, n, 1.0, R2, n);
        for (int i = 0; i < n; i++) for (int j = 0; j <= i; j++) EL(R, n, i, j, row) = EL(R2, n, i, j, row);
        double d = maxdiff(C, R, n * n);
        CHECK(blasx_last_status() == 0 && d < 1e-10, "dsyrk row=%d: maxdiff %g", row, d);
        memcpy(R, C, sizeof(double) * n * n);
        cblas_dsyr2k(row ? CblasRowMajor : CblasColMajor, CblasUpper, CblasTrans, n, n, 0.5, A, n, B, n, 0.0, C, n);
        for (int i = 0; i < n * n; i++) R2[i] = 0;
        ref_gemm(row, 1, 0, n, n, n, 0.5, A, n, B, n, 0.0, R2, n);
        double *R3 = calloc(n * n, sizeof(double));
        ref_gemm(row, 1, 0, n, n, n, 0.5, B, n, A, n, 0.0, R3, n);
        for (int i = 0; i < n; i++) for (int j = i; j < n; j++) EL(R, n, i, j, row) = EL(R2, n, i, j, row) + EL(R3, n, i, j, row);
        d = maxdiff(C, R, n * n);
        CHECK(blasx_last_status() == 0 && d < 1e-10, "dsyr2k row=%d: maxdiff %g", row, d);
        free(A); free(B); free(C); free(R); free(R2); free(R3);
    }
    /* symm left upper: C = A_sym B + C */
    for (int row = 0; row < 2; row++) {
        double *A = mat(n * n, 31), *B = mat(n * n, 32), *C = mat(n * n, 33), *R = malloc(sizeof(double) * n * n), *S = malloc(sizeof(double) * n * n);
        memcpy(R, C, sizeof(double) * n * n);
        for (int i = 0; i < n; i++) for (int j = 0; j < n; j++) EL(S, n, i, j, row) = i <= j ? EL(A, n, i, j, row) : EL(A, n, j, i, row);
        cblas_dsymm(row ? CblasRowMajor : CblasColMajor, CblasLeft, CblasUpper, n, n, 1.0, A, n, B, n, 1.0, C, n);
        ref_gemm(row, 0, 0, n, n, n, 1.0, S, n, B, n, 1.0, R, n);
        double d = maxdiff(C, R, n * n);
        CHECK(blasx_last_status() == 0 && d < 1e-10, "dsymm row=%d: maxdiff %g", row, d);
        free(A); free(B); free(C); free(R); free(S);
    }
    /* trmm / trsm round trip: B -> tri(A) B -> solve back */
    for (int row = 0; row < 2; row++) for (int side = 0; side < 2; side++) {
        double *A = mat(n * n, 41), *B = mat(n * n, 42), *B0 = malloc(sizeof(double) * n * n);
        for (int i = 0; i < n; i++) for (int j = 0; j < n; j++) {
            double v = EL(A, n, i, j, row) / n;
            EL(A, n, i, j, row) = i == j ? (v >= 0 ? 1.0 + fabs(v) * n : -1.0 - fabs(v) * n) : v;
        }
        memcpy(B0, B, sizeof(double) * n * n);
        enum CBLAS_ORDER o = row ? CblasRowMajor : CblasColMajor;
        enum CBLAS_SIDE s = side ? CblasRight : CblasLeft;
        cblas_dtrmm(o, s, CblasLower, CblasNoTrans, CblasNonUnit, n, n, 2.0, A, n, B, n);
        int st1 = blasx_last_status();
        cblas_dtrsm(o, s, CblasLower, CblasNoTrans, CblasNonUnit, n, n, 0.5, A, n, B, n);
        double d = maxdiff(B, B0, n * n);
        CHECK(st1 == 0 && blasx_last_status() == 0 && d < 1e-9, "trmm/trsm row=%d side=%d: maxdiff %g", row, side, d);
        free(A); free(B); free(B0);
    }
    /* singular triangle is reported */
    {
        double *A = mat(n * n, 51), *B = mat(n * n, 52);
        for (int i = 0; i < n; i++) A[(long)i * n + i] = 1.0;
        A[(long)(n / 2) * n + n / 2] = 0.0;
        cblas_dtrsm(CblasColMajor, CblasLeft, CblasUpper, CblasNoTrans, CblasNonUnit, n, n, 1.0, A, n, B, n);
        CHECK(blasx_last_status() == 6, "singular trsm status %d", blasx_last_status());
        free(A); free(B);
    }
    /* sgemm (TF32): normwise check */
    {
        float *A = malloc(4 * n * n), *B = malloc(4 * n * n), *C = malloc(4 * n * n);
        unsigned s2 = 9;
        for (int i = 0; i < n * n; i++) { A[i] = (float)rnd(&s2); B[i] = (float)rnd(&s2); C[i] = 0; }
        cblas_sgemm(CblasColMajor, CblasNoTrans, CblasNoTrans, n, n, n, 1.0f, A, n, B, n, 0.0f, C, n);
        double num = 0, den = 0;
        for (int i = 0; i < n; i++) for (int j = 0; j < n; j++) {
            double s = 0; for (int p = 0; p < n; p++) s += (double)A[p * n + i] * B[j * n + p];
            num += (C[j * n + i] - s) * (C[j * n + i] - s); den += s * s;
        }
        CHECK(blasx_last_status() == 0 && sqrt(num / den) < 2e-3, "sgemm rel err %g", sqrt(num / den));
        free(A); free(B); free(C);
    }
    return 0;
}

int main(int argc, char **argv) {
    const char *mode = argc > 1 ? argv[1] : "args";
    if (!strcmp(mode, "args")) args_mode();
    else if (!strcmp(mode, "quick")) quick_mode();
    else compute_mode(argc > 2 ? atoi(argv[2]) : 300);
    printf("%s: %d failures\n", mode, fails);
    return fails ? 1 : 0;
}
