/* dshost — C ABI of the native host side (input producer + preconditioner
 * setup) that feeds the B200 solve (include/dsgpu.h).
 *
 * In the reference these steps live in its own C++ (SURVEY.md §3.2):
 *   assemble_stokes            proj/src/assembly.cpp:340-361
 *   rcm_permutation            proj/src/reorder.cpp:9-55
 *   permute_symmetric          proj/src/csr.cpp:113-124
 *   ic0                        proj/src/cholesky.cpp:84-134
 * A reference-side integration keeps calling those; this
 * library is the framework's own native equivalent, so bench/tests can build
 * BASELINE's systems (2D bit-identical to the reference, and 3D, which the
 * reference lacks) without the reference present.
 *
 * Conventions: CSR = int64 row_ptr, int32 cols (sorted, unique), f64 vals —
 * the reference CsrMatrix layout (proj/include/divstokes/csr.hpp:12-16).
 * Return 0 on success, a DSHOST_E_* code otherwise; dshost_last_error()
 * holds a message (thread-local).
 */
#ifndef DSHOST_H
#define DSHOST_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DSHOST_OK = 0,
  DSHOST_E_INVALID = 3,   /* std::invalid_argument in the reference */
  DSHOST_E_BREAKDOWN = 6, /* FactorBreakdown (proj/include/divstokes/cholesky.hpp:13-19) */
  DSHOST_E_INTERNAL = 7,
  DSHOST_E_RUNTIME = 8    /* std::runtime_error in the reference (I/O, file format) */
};

/* case ids: BASELINE psi-MMS forcing, lid-driven cavity (2D), seeded
 * uniform[-1,1] velocity RHS (std::mt19937_64 + uniform_real_distribution) */
enum { DSHOST_CASE_PSI_MMS = 0, DSHOST_CASE_CAVITY = 1, DSHOST_CASE_RANDOM = 3 };
/* block ids for dshost_block */
enum { DSHOST_A = 0, DSHOST_B = 1, DSHOST_BT = 2, DSHOST_Q = 3, DSHOST_Q_NU = 4 };

typedef struct dshost_system dshost_system;

const char* dshost_last_error(void);

/* Divergence-conforming B-spline Stokes system on the unit square (dim 2) or
 * cube (dim 3), k' = degree of the pressure space, n_elem elements per
 * direction, viscosity nu. Replaces build_pair + assemble_stokes
 * (proj/src/spaces.cpp:28-82, proj/src/assembly.cpp:340-361). */
int dshost_assemble(int dim, int k_prime, int n_elem, int case_id, double nu, uint64_t seed,
                    dshost_system** out);
void dshost_free(dshost_system* s);
int dshost_dims(const dshost_system* s, int* n_u, int* n_p, int64_t* nnz5);
/* Borrowed pointers into the system (valid until dshost_free). */
int dshost_block(const dshost_system* s, int which, int* n_rows, int* n_cols,
                 const int64_t** row_ptr, const int32_t** cols, const double** vals);
const double* dshost_rhs(const dshost_system* s);

/* rcm_permutation (perm[k] = original index at position k). */
int dshost_rcm(int n, const int64_t* row_ptr, const int32_t* cols, int32_t* perm);
/* permute_symmetric: out arrays sized n+1 / nnz. */
int dshost_permute(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                   const int32_t* perm, int64_t* out_row_ptr, int32_t* out_cols,
                   double* out_vals);
int64_t dshost_lower_nnz(int n, const int64_t* row_ptr, const int32_t* cols);
/* ic0: L arrays sized n+1 / dshost_lower_nnz; *bad_row = breakdown row. */
int dshost_ic0(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
               int64_t* l_row_ptr, int32_t* l_cols, double* l_vals, int* bad_row);

/* ---- Matrix Market wire format (proj/src/csr.cpp:126-175) ------------- */
/* write_matrix_market: the reference's dump format byte for byte (header,
 * size line, 1-based "i j v" lines at 17 significant digits; symmetric =
 * lower triangle only). */
int dshost_write_matrix_market(const char* path, int n_rows, int n_cols, const int64_t* row_ptr,
                               const int32_t* cols, const double* vals, int symmetric);
/* read_matrix_market: the CSR the reference's reader builds (symmetric
 * entries mirrored, duplicates summed, csr_from_triplets ordering). Errors:
 * DSHOST_E_RUNTIME (cannot open, bad header / type / size line, truncated
 * entry list), DSHOST_E_INVALID (index out of range). */
typedef struct dshost_csr dshost_csr;
int dshost_read_matrix_market(const char* path, dshost_csr** out);
/* Borrowed pointers into the matrix (valid until dshost_csr_free). */
int dshost_csr_view(const dshost_csr* m, int* n_rows, int* n_cols, const int64_t** row_ptr,
                    const int32_t** cols, const double** vals);
void dshost_csr_free(dshost_csr* m);

#ifdef __cplusplus
}
#endif
#endif
