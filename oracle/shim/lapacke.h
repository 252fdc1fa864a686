/* TEST INFRASTRUCTURE (oracle build only).
 * Five-prototype LAPACKE shim so the reference's dense.cpp compiles without a
 * system liblapacke. The dense analysis layer (reference proj/src/dense.cpp:25,
 * 40,51,60,76) is OFF the solve path this repo accelerates; the stubs in
 * lapacke_stub.c return an error code so any accidental use fails loudly. */
#ifndef ORACLE_LAPACKE_SHIM_H
#define ORACLE_LAPACKE_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
#define LAPACK_COL_MAJOR 102
typedef int lapack_int;
lapack_int LAPACKE_dsyevd(int layout, char jobz, char uplo, lapack_int n, double* a,
                          lapack_int lda, double* w);
lapack_int LAPACKE_dsygvd(int layout, lapack_int itype, char jobz, char uplo, lapack_int n,
                          double* a, lapack_int lda, double* b, lapack_int ldb, double* w);
lapack_int LAPACKE_dpotrf(int layout, char uplo, lapack_int n, double* a, lapack_int lda);
lapack_int LAPACKE_dpotrs(int layout, char uplo, lapack_int n, lapack_int nrhs,
                          const double* a, lapack_int lda, double* b, lapack_int ldb);
lapack_int LAPACKE_dgels(int layout, char trans, lapack_int m, lapack_int n, lapack_int nrhs,
                         double* a, lapack_int lda, double* b, lapack_int ldb);
#ifdef __cplusplus
}
#endif
#endif
