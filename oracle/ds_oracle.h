/* TEST INFRASTRUCTURE — CPU oracle for the MINRES + IC(0) block-preconditioned
 * Stokes solve. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it; the product path never does.
 *
 * Plain-C restatement of the reference's solve stage (scalar kernel path),
 * each function citing the reference file:line it follows. Pinned against the
 * reference itself (oracle/_ref/libdivstokes_ref.so built from
 * /root/reference/proj/src by oracle/Makefile) in tests/test_oracle.py:
 * with the reference forced to its scalar kernels the two agree bit for bit
 * on RCM, permutation, IC(0), the IC(0) apply and the full solves; with the
 * reference's default AVX2 kernels they agree to round-off.
 */
#ifndef DS_ORACLE_H
#define DS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n_rows, n_cols;
  const int64_t* rp;
  const int32_t* ci;
  const double* v;
} or_csr;

/* block kinds — same values as DSGPU_BLOCK_* in include/dsgpu.h */
enum { OR_JACOBI = 0, OR_PCG_JACOBI = 1, OR_PCG_IC0 = 2 };

/* status codes — same values as DSGPU_* in include/dsgpu.h */
enum {
  OR_OK = 0,
  OR_E_INDEFINITE_PRECOND = 1,
  OR_E_NEG_CURVATURE = 2,
  OR_E_BAD_INPUT = 3,
  OR_E_NONPOS_DIAG = 5,
  OR_E_BREAKDOWN = 6
};

typedef struct {
  int iterations;
  int converged;
  double wall_seconds;      /* MINRES only (solvers.cpp:27,120-121) */
  double setup_seconds;     /* RCM + permute + IC(0) */
  double mean_inner_top;
  double mean_inner_bottom;
  int hist_len;
  int status;
  int failed_block;         /* 0 velocity, 1 pressure, -1 none */
  int breakdown_row;
  long inner_top, apps_top, inner_bottom, apps_bottom;
} or_report;

double or_dot(const double* a, const double* b, int64_t n);
void or_spmv(const or_csr* a, const double* x, double* y);
int or_rcm(int n, const int64_t* rp, const int32_t* ci, int32_t* perm);
void or_permute(int n, const int64_t* rp, const int32_t* ci, const double* v,
                const int32_t* perm, int64_t* out_rp, int32_t* out_ci, double* out_v);
int64_t or_lower_nnz(int n, const int64_t* rp, const int32_t* ci);
int or_ic0(int n, const int64_t* rp, const int32_t* ci, const double* v, int64_t* l_rp,
           int32_t* l_ci, double* l_v, int* bad_row);
void or_ic0_solve(int n, const int64_t* l_rp, const int32_t* l_ci, const double* l_v,
                  const double* r, double* z);
int or_pcg(const or_csr* a, const double* b, int pre_kind, const or_csr* l_factor,
           double tol, int max_iter, double* x, int* iterations, int* converged);
int or_solve_stokes(const or_csr* A, const or_csr* B, const or_csr* Bt, const or_csr* Q_nu,
                    const or_csr* Q_filter, const double* f, int top_kind, int bottom_kind,
                    double outer_tol, double inner_tol, int max_iter, int stop_euclid,
                    int inner_cap, double* u, double* p, or_report* rep, double* hist_m,
                    double* hist_e, int hist_cap);

#ifdef __cplusplus
}
#endif
#endif
