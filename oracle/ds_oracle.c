/* TEST INFRASTRUCTURE — see ds_oracle.h. Plain-C restatement of the
 * reference's solve stage; compiled with -ffp-contract=off so every
 * multiply/add rounds exactly like the reference's scalar kernels. */
#define _POSIX_C_SOURCE 199309L
#include "ds_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* scalar::dot, proj/src/kernels.cpp:17-21 */
double or_dot(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* scalar::axpy, proj/src/kernels.cpp:23-25 */
static void or_axpy(double alpha, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

/* scalar::spmv_csr, proj/src/kernels.cpp:31-38 */
void or_spmv(const or_csr* a, const double* x, double* y) {
  for (int i = 0; i < a->n_rows; ++i) {
    double acc = 0.0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) acc += a->v[k] * x[a->ci[k]];
    y[i] = acc;
  }
}

/* CsrMatrix::pattern_symmetric, proj/src/csr.cpp:82-86: transpose pattern
 * equals the pattern. */
static int pattern_symmetric(int n, const int64_t* rp, const int32_t* ci) {
  int64_t nnz = rp[n];
  int64_t* trp = calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* tci = malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
  int64_t* next = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  for (int64_t k = 0; k < nnz; ++k) trp[ci[k] + 1]++;
  for (int i = 0; i < n; ++i) trp[i + 1] += trp[i];
  for (int i = 0; i < n; ++i) next[i] = trp[i];
  for (int i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) tci[next[ci[k]]++] = i;
  int ok = 1;
  for (int i = 0; i <= n && ok; ++i) ok = trp[i] == rp[i];
  for (int64_t k = 0; k < nnz && ok; ++k) ok = tci[k] == ci[k];
  free(trp);
  free(tci);
  free(next);
  return ok;
}

static const int* g_degree; /* comparator context (single-threaded oracle) */
static int cmp_degree_index(const void* pa, const void* pb) {
  const int a = *(const int*)pa, b = *(const int*)pb;
  if (g_degree[a] != g_degree[b]) return g_degree[a] < g_degree[b] ? -1 : 1;
  return (a > b) - (a < b);
}

/* rcm_permutation, proj/src/reorder.cpp:9-55. Returns 0, or -1 for a
 * nonsymmetric pattern (the reference throws std::invalid_argument). */
int or_rcm(int n, const int64_t* rp, const int32_t* ci, int32_t* perm) {
  if (!pattern_symmetric(n, rp, ci)) return -1;
  int* degree = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    int d = 0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] != i) ++d;
    degree[i] = d;
  }
  int* order = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  char* visited = calloc((size_t)(n > 0 ? n : 1), 1);
  int* nb = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int len = 0;
  g_degree = degree;
  for (int scan = 0; scan < n; ++scan) {
    if (visited[scan]) continue;
    int start = scan;
    for (int v = scan; v < n; ++v)
      if (!visited[v] && degree[v] < degree[start]) start = v;
    visited[start] = 1;
    order[len++] = start;
    for (int head = len - 1; head < len; ++head) {
      const int u = order[head];
      int cnt = 0;
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        const int v = ci[k];
        if (v != u && !visited[v]) {
          visited[v] = 1;
          nb[cnt++] = v;
        }
      }
      qsort(nb, (size_t)cnt, sizeof(int), cmp_degree_index);
      memcpy(order + len, nb, sizeof(int) * (size_t)cnt);
      len += cnt;
      if (len == n) break;
    }
  }
  for (int i = 0; i < n; ++i) perm[i] = order[n - 1 - i];
  free(degree);
  free(order);
  free(visited);
  free(nb);
  return 0;
}

static int cmp_col_pos(const void* pa, const void* pb) {
  const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  /* packed (col << 32 | original position): column order, stable */
  return (a > b) - (a < b);
}

/* permute_symmetric, proj/src/csr.cpp:113-124 (B(i,j) = A(perm[i], perm[j]),
 * rebuilt through csr_from_triplets :88-111; duplicates cannot occur). */
void or_permute(int n, const int64_t* rp, const int32_t* ci, const double* v,
                const int32_t* perm, int64_t* out_rp, int32_t* out_ci, double* out_v) {
  int* inv = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) inv[perm[i]] = i;
  int64_t maxlen = 0;
  for (int i = 0; i < n; ++i)
    if (rp[i + 1] - rp[i] > maxlen) maxlen = rp[i + 1] - rp[i];
  int64_t* key = malloc(sizeof(int64_t) * (size_t)(maxlen > 0 ? maxlen : 1));
  out_rp[0] = 0;
  for (int r = 0; r < n; ++r) {
    const int old = perm[r];
    const int64_t len = rp[old + 1] - rp[old];
    for (int64_t k = 0; k < len; ++k)
      key[k] = ((int64_t)inv[ci[rp[old] + k]] << 32) | (int64_t)k;
    qsort(key, (size_t)len, sizeof(int64_t), cmp_col_pos);
    const int64_t base = out_rp[r];
    for (int64_t k = 0; k < len; ++k) {
      out_ci[base + k] = (int32_t)(key[k] >> 32);
      double sum = 0.0; /* csr_from_triplets sums from 0.0 (csr.cpp:99-102) */
      sum += v[rp[old] + (key[k] & 0xffffffffLL)];
      out_v[base + k] = sum;
    }
    out_rp[r + 1] = base + len;
  }
  free(inv);
  free(key);
}

int64_t or_lower_nnz(int n, const int64_t* rp, const int32_t* ci) {
  int64_t c = 0;
  for (int i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] <= i) ++c;
  return c;
}

/* ic0, proj/src/cholesky.cpp:84-134. Returns OR_OK, OR_E_BAD_INPUT (missing
 * diagonal) or OR_E_BREAKDOWN with *bad_row set (FactorBreakdown). */
int or_ic0(int n, const int64_t* rp, const int32_t* ci, const double* v, int64_t* l_rp,
           int32_t* l_ci, double* l_v, int* bad_row) {
  *bad_row = -1;
  l_rp[0] = 0;
  int64_t pos = 0;
  for (int i = 0; i < n; ++i) {
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] <= i) {
        l_ci[pos] = ci[k];
        l_v[pos] = v[k];
        ++pos;
      }
    l_rp[i + 1] = pos;
  }
  for (int i = 0; i < n; ++i) {
    const int64_t ib = l_rp[i], ie = l_rp[i + 1];
    if (ie == ib || l_ci[ie - 1] != i) {
      *bad_row = i;
      return OR_E_BAD_INPUT;
    }
    for (int64_t ku = ib; ku < ie - 1; ++ku) {
      const int j = l_ci[ku];
      double s = l_v[ku];
      int64_t pi = ib, pj = l_rp[j];
      const int64_t je = l_rp[j + 1] - 1;
      while (pi < ku && pj < je) {
        if (l_ci[pi] == l_ci[pj])
          s -= l_v[pi++] * l_v[pj++];
        else if (l_ci[pi] < l_ci[pj])
          ++pi;
        else
          ++pj;
      }
      l_v[ku] = s / l_v[je];
    }
    double d = l_v[ie - 1];
    for (int64_t k = ib; k < ie - 1; ++k) d -= l_v[k] * l_v[k];
    if (!(d > 0.0)) {
      *bad_row = i;
      return OR_E_BREAKDOWN;
    }
    l_v[ie - 1] = sqrt(d);
  }
  return OR_OK;
}

/* Ic0Factor::solve, proj/src/cholesky.cpp:136-152: row-oriented forward
 * sweep, column-oriented (scatter) backward sweep over the same L. */
void or_ic0_solve(int n, const int64_t* l_rp, const int32_t* l_ci, const double* l_v,
                  const double* r, double* z) {
  for (int i = 0; i < n; ++i) {
    double s = r[i];
    const int64_t end = l_rp[i + 1] - 1;
    for (int64_t k = l_rp[i]; k < end; ++k) s -= l_v[k] * z[l_ci[k]];
    z[i] = s / l_v[end];
  }
  for (int i = n - 1; i >= 0; --i) {
    const int64_t end = l_rp[i + 1] - 1;
    const double zi = z[i] / l_v[end];
    z[i] = zi;
    for (int64_t k = l_rp[i]; k < end; ++k) z[l_ci[k]] -= l_v[k] * zi;
  }
}

/* ---- blocks (proj/src/precond.cpp:32-118) -------------------------------- */

typedef struct {
  int kind, n;
  double tol;
  int cap;
  or_csr m;            /* operator in the block's ordering */
  int64_t *m_rp;       /* owned permuted copy (IC0) */
  int32_t* m_ci;
  double* m_v;
  int32_t* perm;       /* IC0 only */
  or_csr l;            /* IC0 factor */
  int64_t* l_rp;
  int32_t* l_ci;
  double* l_v;
  double* inv_diag;    /* JACOBI / PCG_JACOBI */
  double *rhs, *sol, *r, *z, *p, *q; /* work */
  long inner, apps;
} or_block;

static int diag_of(const or_csr* a, double* d) {
  for (int i = 0; i < a->n_rows; ++i) {
    d[i] = 0.0;
    /* CsrMatrix::at via lower_bound, proj/src/csr.cpp:13-18 */
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k)
      if (a->ci[k] == i) d[i] = a->v[k];
  }
  return 0;
}

static int block_init(or_block* b, const or_csr* m, int kind, double tol, int cap, int* bad_row) {
  memset(b, 0, sizeof(*b));
  b->kind = kind;
  b->n = m->n_rows;
  b->tol = tol;
  b->cap = cap;
  const int n = b->n;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  b->rhs = calloc(nn, sizeof(double));
  b->sol = calloc(nn, sizeof(double));
  b->r = calloc(nn, sizeof(double));
  b->z = calloc(nn, sizeof(double));
  b->p = calloc(nn, sizeof(double));
  b->q = calloc(nn, sizeof(double));
  if (kind == OR_PCG_IC0) {
    /* PcgBlock ctor, precond.cpp:61-64: rcm -> permute -> ic0 */
    b->perm = malloc(sizeof(int32_t) * nn);
    if (or_rcm(n, m->rp, m->ci, b->perm) != 0) return OR_E_BAD_INPUT;
    const int64_t nnz = m->rp[n];
    b->m_rp = malloc(sizeof(int64_t) * (nn + 1));
    b->m_ci = malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    b->m_v = malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    or_permute(n, m->rp, m->ci, m->v, b->perm, b->m_rp, b->m_ci, b->m_v);
    b->m = (or_csr){n, n, b->m_rp, b->m_ci, b->m_v};
    const int64_t lnnz = or_lower_nnz(n, b->m_rp, b->m_ci);
    b->l_rp = malloc(sizeof(int64_t) * (nn + 1));
    b->l_ci = malloc(sizeof(int32_t) * (size_t)(lnnz > 0 ? lnnz : 1));
    b->l_v = malloc(sizeof(double) * (size_t)(lnnz > 0 ? lnnz : 1));
    const int rc = or_ic0(n, b->m_rp, b->m_ci, b->m_v, b->l_rp, b->l_ci, b->l_v, bad_row);
    if (rc != OR_OK) return rc;
    b->l = (or_csr){n, n, b->l_rp, b->l_ci, b->l_v};
  } else {
    /* JacobiBlock ctor (precond.cpp:34-39) / PcgBlock jacobi (:65-71) */
    b->m = *m;
    b->inv_diag = malloc(sizeof(double) * nn);
    diag_of(m, b->inv_diag);
    for (int i = 0; i < n; ++i) {
      if (!(b->inv_diag[i] > 0.0)) return OR_E_NONPOS_DIAG;
      b->inv_diag[i] = 1.0 / b->inv_diag[i];
    }
  }
  return OR_OK;
}

static void block_free(or_block* b) {
  free(b->m_rp); free(b->m_ci); free(b->m_v); free(b->perm);
  free(b->l_rp); free(b->l_ci); free(b->l_v); free(b->inv_diag);
  free(b->rhs); free(b->sol); free(b->r); free(b->z); free(b->p); free(b->q);
}

static void block_pre(const or_block* b, const double* x, double* y) {
  if (b->kind == OR_PCG_IC0)
    or_ic0_solve(b->n, b->l_rp, b->l_ci, b->l_v, x, y);
  else
    for (int i = 0; i < b->n; ++i) y[i] = b->inv_diag[i] * x[i];
}

/* pcg, proj/src/solvers.cpp:125-159 (zero initial guess). Work vectors
 * supplied by the block. Returns OR_OK / OR_E_INDEFINITE_PRECOND /
 * OR_E_NEG_CURVATURE. */
static int pcg_core(const or_block* b, const double* rhs, double* x, double* r, double* z,
                    double* p, double* q, int* iters, int* conv) {
  const int n = b->n;
  *iters = 0;
  *conv = 0;
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  memcpy(r, rhs, sizeof(double) * (size_t)n);
  block_pre(b, r, z);
  double rho = or_dot(r, z, n);
  if (rho < 0.0) return OR_E_INDEFINITE_PRECOND;
  const double rho0 = rho;
  if (rho0 == 0.0) {
    *conv = 1;
    return OR_OK;
  }
  memcpy(p, z, sizeof(double) * (size_t)n);
  for (int it = 1; it <= b->cap; ++it) {
    or_spmv(&b->m, p, q);
    const double curv = or_dot(p, q, n);
    if (curv <= 0.0) return OR_E_NEG_CURVATURE;
    const double alpha = rho / curv;
    or_axpy(alpha, p, x, n);
    or_axpy(-alpha, q, r, n);
    block_pre(b, r, z);
    const double rho_next = or_dot(r, z, n);
    if (rho_next < 0.0) return OR_E_INDEFINITE_PRECOND;
    *iters = it;
    if (sqrt(rho_next / rho0) <= b->tol) {
      *conv = 1;
      return OR_OK;
    }
    const double beta = rho_next / rho;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_next;
  }
  return OR_OK;
}

int or_pcg(const or_csr* a, const double* b, int pre_kind, const or_csr* l_factor, double tol,
           int max_iter, double* x, int* iterations, int* converged) {
  or_block blk;
  memset(&blk, 0, sizeof(blk));
  const int n = a->n_rows;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  blk.n = n;
  blk.m = *a;
  blk.tol = tol;
  blk.cap = max_iter;
  blk.kind = pre_kind == 2 ? OR_PCG_IC0 : OR_PCG_JACOBI;
  double* inv = NULL;
  if (pre_kind == 2) {
    blk.l_rp = (int64_t*)l_factor->rp;
    blk.l_ci = (int32_t*)l_factor->ci;
    blk.l_v = (double*)l_factor->v;
  } else {
    inv = malloc(sizeof(double) * nn);
    diag_of(a, inv);
    for (int i = 0; i < n; ++i) inv[i] = pre_kind == 1 ? 1.0 / inv[i] : 1.0;
    blk.inv_diag = inv;
  }
  double* r = calloc(nn, sizeof(double));
  double* z = calloc(nn, sizeof(double));
  double* p = calloc(nn, sizeof(double));
  double* q = calloc(nn, sizeof(double));
  const int rc = pcg_core(&blk, b, x, r, z, p, q, iterations, converged);
  free(r); free(z); free(p); free(q); free(inv);
  return rc;
}

/* PcgBlock::apply (precond.cpp:75-100) / JacobiBlock::apply (:40-43) */
static int block_apply(or_block* b, const double* r, double* z) {
  const int n = b->n;
  if (b->kind == OR_JACOBI) {
    for (int i = 0; i < n; ++i) z[i] = b->inv_diag[i] * r[i];
    ++b->apps;
    return OR_OK;
  }
  if (b->perm)
    for (int i = 0; i < n; ++i) b->rhs[i] = r[b->perm[i]];
  else
    memcpy(b->rhs, r, sizeof(double) * (size_t)n);
  int it = 0, conv = 0;
  const int rc = pcg_core(b, b->rhs, b->sol, b->r, b->z, b->p, b->q, &it, &conv);
  if (rc != OR_OK) return rc;
  b->inner += it;
  ++b->apps;
  if (b->perm)
    for (int i = 0; i < n; ++i) z[b->perm[i]] = b->sol[i];
  else
    memcpy(z, b->sol, sizeof(double) * (size_t)n);
  return OR_OK;
}

typedef struct {
  or_block* top;
  or_block* bottom;
  int n_top, n_bottom;
  int failed_block;
} or_precond;

/* BlockDiagPreconditioner::apply, precond.cpp:139-148 */
static int precond_apply(or_precond* m, const double* r, double* z) {
  int rc = block_apply(m->top, r, z);
  if (rc != OR_OK) return rc;
  if (or_dot(z, r, m->n_top) < 0.0) {
    m->failed_block = 0;
    return OR_E_INDEFINITE_PRECOND;
  }
  rc = block_apply(m->bottom, r + m->n_top, z + m->n_top);
  if (rc != OR_OK) return rc;
  if (or_dot(z + m->n_top, r + m->n_top, m->n_bottom) < 0.0) {
    m->failed_block = 1;
    return OR_E_INDEFINITE_PRECOND;
  }
  return OR_OK;
}

/* StokesSystem::apply, proj/src/assembly.cpp:363-372 */
static void saddle_apply(const or_csr* A, const or_csr* B, const or_csr* Bt, const double* x,
                         double* y, double* tmp) {
  const int nu = A->n_rows;
  or_spmv(A, x, y);
  or_spmv(Bt, x + nu, tmp);
  for (int i = 0; i < nu; ++i) y[i] += tmp[i];
  or_spmv(B, x, y + nu);
}

/* minres, proj/src/solvers.cpp:24-123 (x0 = 0), driven as in solve_stokes,
 * proj/src/precond.cpp:245-299. */
int or_solve_stokes(const or_csr* A, const or_csr* B, const or_csr* Bt, const or_csr* Q_nu,
                    const or_csr* Q_filter, const double* f, int top_kind, int bottom_kind,
                    double outer_tol, double inner_tol, int max_iter, int stop_euclid,
                    int inner_cap, double* u, double* p, or_report* rep, double* hist_m,
                    double* hist_e, int hist_cap) {
  memset(rep, 0, sizeof(*rep));
  rep->failed_block = -1;
  rep->breakdown_row = -1;
  const int n_u = A->n_rows, n_p = Q_nu->n_rows, n = n_u + n_p;
  or_block top, bottom;
  const double t_setup = now_s();
  int bad = -1;
  int rc = block_init(&top, A, top_kind, inner_tol, inner_cap, &bad);
  if (rc == OR_OK) {
    rc = block_init(&bottom, Q_nu, bottom_kind, inner_tol, inner_cap, &bad);
    if (rc != OR_OK) block_free(&bottom);
  }
  rep->setup_seconds = now_s() - t_setup;
  if (rc != OR_OK) {
    block_free(&top);
    rep->status = rc;
    rep->breakdown_row = bad;
    return rc;
  }
  or_precond M = {&top, &bottom, n_u, n_p, -1};

  const size_t nn = (size_t)n;
  double* b = calloc(nn, sizeof(double));
  for (int i = 0; i < n_u; ++i) b[i] = f[i];
  double *x = calloc(nn, 8), *r1 = calloc(nn, 8), *r2 = calloc(nn, 8), *y = calloc(nn, 8);
  double *v = calloc(nn, 8), *w = calloc(nn, 8), *w1 = calloc(nn, 8), *w2 = calloc(nn, 8);
  double *res = calloc(nn, 8), *av = calloc(nn, 8), *aw = calloc(nn, 8);
  double *aw1 = calloc(nn, 8), *aw2 = calloc(nn, 8), *tmp = calloc((size_t)n_u + 1, 8);
  double* t;
#define SWAP(a, b) (t = (a), (a) = (b), (b) = t)

  const double t0 = now_s();
  memcpy(r1, b, sizeof(double) * nn);
  memcpy(res, r1, sizeof(double) * nn);
  const double rnorm0 = sqrt(or_dot(res, res, n));
  rc = precond_apply(&M, r1, y);
  int hl = 0;
  if (rc != OR_OK) goto done;
  double beta1 = or_dot(r1, y, n);
  if (beta1 < 0.0) {
    rc = OR_E_INDEFINITE_PRECOND;
    goto done;
  }
  beta1 = sqrt(beta1);
  if (hl < hist_cap) {
    if (hist_m) hist_m[hl] = 1.0;
    if (hist_e) hist_e[hl] = 1.0;
  }
  ++hl;
  if (beta1 == 0.0) {
    rep->converged = 1;
    goto done;
  }
  memcpy(r2, r1, sizeof(double) * nn);
  {
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1;
    double cs = -1.0, sn = 0.0, oldeps = 0.0;
    for (int it = 1; it <= max_iter; ++it) {
      const double s = 1.0 / beta;
      for (int i = 0; i < n; ++i) v[i] = s * y[i];
      saddle_apply(A, B, Bt, v, av, tmp);
      memcpy(y, av, sizeof(double) * nn);
      if (it >= 2) or_axpy(-beta / oldb, r1, y, n);
      const double alfa = or_dot(v, y, n);
      or_axpy(-alfa / beta, r2, y, n);
      SWAP(r1, r2);
      SWAP(r2, y);
      rc = precond_apply(&M, r2, y);
      if (rc != OR_OK) goto done;
      oldb = beta;
      const double betasq = or_dot(r2, y, n);
      if (betasq < 0.0) {
        rc = OR_E_INDEFINITE_PRECOND;
        goto done;
      }
      beta = sqrt(betasq);
      oldeps = epsln;
      const double delta = cs * dbar + sn * alfa;
      const double gbar = sn * dbar - cs * alfa;
      epsln = sn * beta;
      dbar = -cs * beta;
      double gamma = sqrt(gbar * gbar + beta * beta);
      if (gamma < 2.220446049250313e-16) gamma = 2.220446049250313e-16;
      cs = gbar / gamma;
      sn = beta / gamma;
      const double phi = cs * phibar;
      phibar = sn * phibar;
      SWAP(w1, w2);
      SWAP(w2, w);
      SWAP(aw1, aw2);
      SWAP(aw2, aw);
      for (int i = 0; i < n; ++i) {
        w[i] = (v[i] - oldeps * w1[i] - delta * w2[i]) / gamma;
        aw[i] = (av[i] - oldeps * aw1[i] - delta * aw2[i]) / gamma;
      }
      or_axpy(phi, w, x, n);
      or_axpy(-phi, aw, res, n);
      rep->iterations = it;
      const double relres_m = phibar / beta1;
      const double relres_e = rnorm0 > 0.0 ? sqrt(or_dot(res, res, n)) / rnorm0 : 0.0;
      if (hl < hist_cap) {
        if (hist_m) hist_m[hl] = relres_m;
        if (hist_e) hist_e[hl] = relres_e;
      }
      ++hl;
      const double stop_value = stop_euclid ? relres_e : relres_m;
      if (stop_value <= outer_tol) {
        rep->converged = 1;
        break;
      }
      if (beta == 0.0) {
        rep->converged = relres_m <= outer_tol;
        break;
      }
    }
  }
done:
  rep->wall_seconds = now_s() - t0;
  rep->hist_len = hl;
  rep->status = rc;
  rep->failed_block = M.failed_block;
  memcpy(u, x, sizeof(double) * (size_t)n_u);
  memcpy(p, x + n_u, sizeof(double) * (size_t)n_p);
  if (rc == OR_OK && Q_filter) {
    /* zero-mean filter, precond.cpp:266-284, kernel = all ones (identity
     * map: constant_pressure_coefficients, analysis.cpp:270-290) */
    double* kern = malloc(sizeof(double) * (size_t)(n_p > 0 ? n_p : 1));
    double* btk = malloc(sizeof(double) * (size_t)(n_u > 0 ? n_u : 1));
    double* qk = malloc(sizeof(double) * (size_t)(n_p > 0 ? n_p : 1));
    for (int i = 0; i < n_p; ++i) kern[i] = 1.0;
    or_spmv(Bt, kern, btk);
    double resid = 0.0, bscale = 0.0;
    for (int i = 0; i < n_u; ++i) resid = fmax(resid, fabs(btk[i]));
    for (int64_t k = 0; k < B->rp[B->n_rows]; ++k) bscale = fmax(bscale, fabs(B->v[k]));
    if (resid <= 1e-10 * bscale) {
      or_spmv(Q_filter, kern, qk);
      double num = 0.0, den = 0.0;
      for (int i = 0; i < n_p; ++i) {
        num += qk[i] * p[i];
        den += qk[i] * kern[i];
      }
      const double mean = num / den;
      for (int i = 0; i < n_p; ++i) p[i] -= mean * kern[i];
    }
    free(kern);
    free(btk);
    free(qk);
  }
  rep->inner_top = top.inner;
  rep->apps_top = top.apps;
  rep->inner_bottom = bottom.inner;
  rep->apps_bottom = bottom.apps;
  if (top_kind != OR_JACOBI && top.apps > 0) rep->mean_inner_top = (double)top.inner / top.apps;
  if (bottom_kind != OR_JACOBI && bottom.apps > 0)
    rep->mean_inner_bottom = (double)bottom.inner / bottom.apps;
  free(b); free(x); free(r1); free(r2); free(y); free(v); free(w); free(w1); free(w2);
  free(res); free(av); free(aw); free(aw1); free(aw2); free(tmp);
  block_free(&top);
  block_free(&bottom);
#undef SWAP
  return rc;
}
