/* TEST INFRASTRUCTURE: LAPACKE stubs for the oracle build (see lapacke.h).
 * Every stub reports failure (-1); nothing on the MINRES/IC(0) solve path
 * calls them. */
#include "lapacke.h"
lapack_int LAPACKE_dsyevd(int l, char j, char u, lapack_int n, double* a, lapack_int lda,
                          double* w) {
  (void)l; (void)j; (void)u; (void)n; (void)a; (void)lda; (void)w;
  return -1;
}
lapack_int LAPACKE_dsygvd(int l, lapack_int it, char j, char u, lapack_int n, double* a,
                          lapack_int lda, double* b, lapack_int ldb, double* w) {
  (void)l; (void)it; (void)j; (void)u; (void)n; (void)a; (void)lda; (void)b; (void)ldb; (void)w;
  return -1;
}
lapack_int LAPACKE_dpotrf(int l, char u, lapack_int n, double* a, lapack_int lda) {
  (void)l; (void)u; (void)n; (void)a; (void)lda;
  return -1;
}
lapack_int LAPACKE_dpotrs(int l, char u, lapack_int n, lapack_int r, const double* a,
                          lapack_int lda, double* b, lapack_int ldb) {
  (void)l; (void)u; (void)n; (void)r; (void)a; (void)lda; (void)b; (void)ldb;
  return -1;
}
lapack_int LAPACKE_dgels(int l, char t, lapack_int m, lapack_int n, lapack_int r, double* a,
                         lapack_int lda, double* b, lapack_int ldb) {
  (void)l; (void)t; (void)m; (void)n; (void)r; (void)a; (void)lda; (void)b; (void)ldb;
  return -1;
}
