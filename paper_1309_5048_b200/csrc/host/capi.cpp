// extern "C" surface of the host library (include/dshost.h).
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "../../../include/dshost.h"
#include "dshost.hpp"

struct dshost_system {
  dshost::System sys;
};
struct dshost_csr {
  dshost::Csr m;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return DSHOST_OK;
  } catch (const dshost::Ic0Breakdown& e) {
    g_err = "factorization breakdown: nonpositive pivot at row " + std::to_string(e.row);
    return DSHOST_E_BREAKDOWN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DSHOST_E_INVALID;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return DSHOST_E_INVALID;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return DSHOST_E_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DSHOST_E_INTERNAL;
  }
}

dshost::Csr view(int n_rows, int n_cols, const int64_t* rp, const int32_t* ci, const double* v) {
  dshost::Csr m;
  m.n_rows = n_rows;
  m.n_cols = n_cols;
  m.rp.assign(rp, rp + n_rows + 1);
  m.ci.assign(ci, ci + rp[n_rows]);
  if (v)
    m.v.assign(v, v + rp[n_rows]);
  else
    m.v.assign(rp[n_rows], 1.0);
  return m;
}
}  // namespace

extern "C" {

const char* dshost_last_error(void) { return g_err.c_str(); }

int dshost_assemble(int dim, int k_prime, int n_elem, int case_id, double nu, uint64_t seed,
                    dshost_system** out) {
  *out = nullptr;
  return guard([&] {
    auto* s = new dshost_system{dshost::assemble(dim, k_prime, n_elem, case_id, nu, seed)};
    *out = s;
  });
}

void dshost_free(dshost_system* s) { delete s; }

int dshost_dims(const dshost_system* s, int* n_u, int* n_p, int64_t* nnz5) {
  *n_u = s->sys.n_u;
  *n_p = s->sys.n_p;
  nnz5[0] = s->sys.A.nnz();
  nnz5[1] = s->sys.B.nnz();
  nnz5[2] = s->sys.Bt.nnz();
  nnz5[3] = s->sys.Q.nnz();
  nnz5[4] = s->sys.Q_nu.nnz();
  return DSHOST_OK;
}

int dshost_block(const dshost_system* s, int which, int* n_rows, int* n_cols,
                 const int64_t** row_ptr, const int32_t** cols, const double** vals) {
  const dshost::Csr* m[5] = {&s->sys.A, &s->sys.B, &s->sys.Bt, &s->sys.Q, &s->sys.Q_nu};
  if (which < 0 || which > 4) {
    g_err = "dshost_block: bad block id";
    return DSHOST_E_INVALID;
  }
  *n_rows = m[which]->n_rows;
  *n_cols = m[which]->n_cols;
  *row_ptr = m[which]->rp.data();
  *cols = m[which]->ci.data();
  *vals = m[which]->v.data();
  return DSHOST_OK;
}

const double* dshost_rhs(const dshost_system* s) { return s->sys.f.data(); }

int dshost_rcm(int n, const int64_t* row_ptr, const int32_t* cols, int32_t* perm) {
  return guard([&] {
    const auto p = dshost::rcm_permutation(view(n, n, row_ptr, cols, nullptr));
    std::memcpy(perm, p.data(), sizeof(int32_t) * n);
  });
}

int dshost_permute(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                   const int32_t* perm, int64_t* out_row_ptr, int32_t* out_cols,
                   double* out_vals) {
  return guard([&] {
    const std::vector<int32_t> p(perm, perm + n);
    const dshost::Csr b = dshost::permute_symmetric(view(n, n, row_ptr, cols, vals), p);
    std::memcpy(out_row_ptr, b.rp.data(), sizeof(int64_t) * (n + 1));
    std::memcpy(out_cols, b.ci.data(), sizeof(int32_t) * b.ci.size());
    std::memcpy(out_vals, b.v.data(), sizeof(double) * b.v.size());
  });
}

int64_t dshost_lower_nnz(int n, const int64_t* row_ptr, const int32_t* cols) {
  int64_t c = 0;
  for (int i = 0; i < n; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
      if (cols[k] <= i) ++c;
  return c;
}

int dshost_ic0(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
               int64_t* l_row_ptr, int32_t* l_cols, double* l_vals, int* bad_row) {
  *bad_row = -1;
  return guard([&] {
    try {
      const dshost::Csr L = dshost::ic0(view(n, n, row_ptr, cols, vals));
      std::memcpy(l_row_ptr, L.rp.data(), sizeof(int64_t) * (n + 1));
      std::memcpy(l_cols, L.ci.data(), sizeof(int32_t) * L.ci.size());
      std::memcpy(l_vals, L.v.data(), sizeof(double) * L.v.size());
    } catch (const dshost::Ic0Breakdown& e) {
      *bad_row = e.row;
      throw;
    }
  });
}

int dshost_write_matrix_market(const char* path, int n_rows, int n_cols, const int64_t* row_ptr,
                               const int32_t* cols, const double* vals, int symmetric) {
  return guard([&] {
    if (!path || n_rows < 0 || n_cols < 0 || !row_ptr) throw std::invalid_argument("write_matrix_market: bad input");
    dshost::write_matrix_market(view(n_rows, n_cols, row_ptr, cols, vals), path, symmetric != 0);
  });
}

int dshost_read_matrix_market(const char* path, dshost_csr** out) {
  *out = nullptr;
  return guard([&] {
    if (!path) throw std::invalid_argument("read_matrix_market: null path");
    auto* m = new dshost_csr{dshost::read_matrix_market(path)};
    *out = m;
  });
}

int dshost_csr_view(const dshost_csr* m, int* n_rows, int* n_cols, const int64_t** row_ptr,
                    const int32_t** cols, const double** vals) {
  if (!m) {
    g_err = "dshost_csr_view: null matrix";
    return DSHOST_E_INVALID;
  }
  *n_rows = m->m.n_rows;
  *n_cols = m->m.n_cols;
  *row_ptr = m->m.rp.data();
  *cols = m->m.ci.data();
  *vals = m->m.v.data();
  return DSHOST_OK;
}

void dshost_csr_free(dshost_csr* m) { delete m; }

}  // extern "C"
