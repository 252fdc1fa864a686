// TEST INFRASTRUCTURE — never shipped, never on the product path.
//
// extern "C" driver over the UNMODIFIED reference library (divstokes, built
// from /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load it. It exposes exactly what the parity checks need:
//   * the reference's own assembly of the 2D systems BASELINE names
//     (build_pair + assemble_stokes, proj/src/spaces.cpp:28-82,
//     proj/src/assembly.cpp:340-361), plus the BASELINE cases the reference
//     lacks (psi-MMS forcing and the seeded uniform RHS);
//   * the reference solve (make_strategy + solve_stokes,
//     proj/src/precond.cpp:161-193, 245-299), including the
//     "IC0-PCG(A)+Diag(Q)" composition built through the public
//     BlockSolver interface (proj/include/divstokes/precond.hpp:14-22) from the
//     public rcm_permutation / permute_symmetric / ic0 / pcg calls in the same
//     order as PcgBlock (proj/src/precond.cpp:59-100);
//   * the solver-layer primitives (rcm_permutation, permute_symmetric, ic0,
//     Ic0Factor::solve, spmv, minres, pcg) for kernel-level parity.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "divstokes/assembly.hpp"
#include "divstokes/cases.hpp"
#include "divstokes/cholesky.hpp"
#include "divstokes/csr.hpp"
#include "divstokes/kernels.hpp"
#include "divstokes/precond.hpp"
#include "divstokes/reorder.hpp"
#include "divstokes/solvers.hpp"
#include "divstokes/spaces.hpp"

using namespace divstokes;

namespace {

void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
  }
}

// Exception taxonomy -> return codes (mirrors include/dsgpu.h DSGPU_E_*).
template <class F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const FactorBreakdown& e) {
    set_err(err, errlen, e.what());
    return 4;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch (const std::domain_error& e) {
    set_err(err, errlen, e.what());
    return 3;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

// BASELINE psi-MMS: u = curl psi = (psi_y, -psi_x),
// psi = X(x) Y(y), X = x^2 (1-x)^2, p = sin(pi x) sin(pi y);
// f = -nu lap(u) + grad p (div u = 0).
Vec2 psi_mms_force(Vec2 q, double nu) {
  const double x = q.x, y = q.y;
  const double X = x * x * (1.0 - x) * (1.0 - x);
  const double X1 = ((4.0 * x - 6.0) * x + 2.0) * x;
  const double X2 = (12.0 * x - 12.0) * x + 2.0;
  const double X3 = 24.0 * x - 12.0;
  const double Y = y * y * (1.0 - y) * (1.0 - y);
  const double Y1 = ((4.0 * y - 6.0) * y + 2.0) * y;
  const double Y2 = (12.0 * y - 12.0) * y + 2.0;
  const double Y3 = 24.0 * y - 12.0;
  const double lap_u1 = X2 * Y1 + X * Y3;
  const double lap_u2 = -(X3 * Y + X1 * Y2);
  const double px = M_PI * std::cos(M_PI * x) * std::sin(M_PI * y);
  const double py = M_PI * std::sin(M_PI * x) * std::cos(M_PI * y);
  return {-nu * lap_u1 + px, -nu * lap_u2 + py};
}

CsrMatrix csr_from_arrays(int n_rows, int n_cols, const int64_t* rp, const int32_t* ci,
                          const double* v) {
  CsrMatrix m;
  m.n_rows = n_rows;
  m.n_cols = n_cols;
  m.row_ptr.assign(rp, rp + n_rows + 1);
  const int64_t nnz = rp[n_rows];
  m.cols.assign(ci, ci + nnz);
  m.vals.assign(v, v + nnz);
  return m;
}

void csr_to_arrays(const CsrMatrix& m, int64_t* rp, int32_t* ci, double* v) {
  std::memcpy(rp, m.row_ptr.data(), sizeof(int64_t) * (m.n_rows + 1));
  std::memcpy(ci, m.cols.data(), sizeof(int32_t) * m.cols.size());
  std::memcpy(v, m.vals.data(), sizeof(double) * m.vals.size());
}

// Caller-side composition for the G2 strategy, through the public
// BlockSolver interface; same construction order as PcgBlock
// (proj/src/precond.cpp:59-73) and same apply (:75-100).
class Ic0PcgBlock final : public BlockSolver {
 public:
  Ic0PcgBlock(const CsrMatrix& m, double tol, int cap) : tol_(tol), cap_(cap) {
    perm_ = rcm_permutation(m);
    matrix_ = permute_symmetric(m, perm_);
    factor_ = std::make_unique<Ic0Factor>(ic0(matrix_));
  }
  void apply(const double* r, double* z) override {
    const int n = matrix_.n_rows;
    std::vector<double> rhs(n), sol;
    for (int i = 0; i < n; ++i) rhs[i] = r[perm_[i]];
    LinearOperator op = [this](const double* x, double* y) { matrix_.multiply(x, y); };
    LinearOperator pre = [this](const double* x, double* y) { factor_->solve(x, y); };
    const PcgResult res = pcg(op, rhs, pre, tol_, cap_, sol);
    inner_ += res.iterations;
    ++apps_;
    for (int i = 0; i < n; ++i) z[perm_[i]] = sol[i];
  }
  std::string label() const override { return "pcg(rcm+ic0)"; }
  bool iterative() const override { return true; }
  long inner_iterations() const override { return inner_; }
  long applications() const override { return apps_; }

 private:
  CsrMatrix matrix_;
  std::vector<int> perm_;
  std::unique_ptr<Ic0Factor> factor_;
  double tol_;
  int cap_;
  long inner_ = 0, apps_ = 0;
};

class DiagBlock final : public BlockSolver {
 public:
  explicit DiagBlock(const CsrMatrix& m) : inv_(m.diagonal()) {
    for (auto& d : inv_) {
      if (!(d > 0.0)) throw std::domain_error("jacobi block: nonpositive diagonal");
      d = 1.0 / d;
    }
  }
  void apply(const double* r, double* z) override {
    for (std::size_t i = 0; i < inv_.size(); ++i) z[i] = inv_[i] * r[i];
    ++apps_;
  }
  std::string label() const override { return "jacobi-diagonal"; }
  long applications() const override { return apps_; }

 private:
  std::vector<double> inv_;
  long apps_ = 0;
};

}  // namespace

extern "C" {

struct ref_system {
  StokesSystem sys;
};

// case_id: 0 psi-MMS (BASELINE C1/C2), 1 lid-driven cavity, 2 reference
// square (e^x MMS), 3 seeded uniform[-1,1] velocity RHS (BASELINE C3).
ref_system* ref_assemble(int case_id, int k_prime, int n_elem, double nu,
                         unsigned long long seed, char* err, int errlen) {
  ref_system* out = nullptr;
  const int rc = guarded(err, errlen, [&] {
    auto pair = std::make_shared<const DiscretePair>(build_pair(k_prime, n_elem));
    ProblemConfig cfg;
    std::shared_ptr<const GeometricMap> map = map_square();
    if (case_id == 0) {
      cfg.nu = nu;
      cfg.body_force = [nu](Vec2 x) { return psi_mms_force(x, nu); };
    } else if (case_id == 1) {
      const CaseDefinition def = case_cavity();
      cfg = def.problem_config();
      map = def.map;
    } else if (case_id == 2) {
      const CaseDefinition def = case_square(nu);
      cfg = def.problem_config();
      map = def.map;
    } else if (case_id == 3) {
      cfg.nu = nu;
    } else {
      throw std::invalid_argument("ref_assemble: unknown case id");
    }
    auto* s = new ref_system{assemble_stokes(pair, map, cfg)};
    if (case_id == 3) {
      std::mt19937_64 gen(seed);
      std::uniform_real_distribution<double> dist(-1.0, 1.0);
      for (auto& v : s->sys.f) v = dist(gen);
    }
    out = s;
  });
  return rc == 0 ? out : nullptr;
}

// System from external CSR blocks (3D or any producer). pair/map stay null,
// so solve_stokes skips its zero-mean filter (proj/src/precond.cpp:266).
ref_system* ref_from_csr(int n_u, int n_p, const int64_t* a_rp, const int32_t* a_ci,
                         const double* a_v, const int64_t* b_rp, const int32_t* b_ci,
                         const double* b_v, const int64_t* q_rp, const int32_t* q_ci,
                         const double* q_v, double nu, const double* f) {
  auto* s = new ref_system;
  s->sys.A = csr_from_arrays(n_u, n_u, a_rp, a_ci, a_v);
  s->sys.B = csr_from_arrays(n_p, n_u, b_rp, b_ci, b_v);
  s->sys.Bt = s->sys.B.transposed();
  s->sys.Q = csr_from_arrays(n_p, n_p, q_rp, q_ci, q_v);
  s->sys.Q_nu = s->sys.Q;
  for (auto& v : s->sys.Q_nu.vals) v *= 1.0 / (2.0 * nu);
  s->sys.f.assign(f, f + n_u);
  s->sys.nu = nu;
  return s;
}

void ref_free(ref_system* s) { delete s; }

void ref_dims(const ref_system* s, int* n_u, int* n_p, int64_t* nnz5) {
  *n_u = s->sys.n_u();
  *n_p = s->sys.n_p();
  nnz5[0] = s->sys.A.nnz();
  nnz5[1] = s->sys.B.nnz();
  nnz5[2] = s->sys.Bt.nnz();
  nnz5[3] = s->sys.Q.nnz();
  nnz5[4] = s->sys.Q_nu.nnz();
}

// which: 0 A, 1 B, 2 Bt, 3 Q, 4 Q_nu
void ref_export(const ref_system* s, int which, int64_t* rp, int32_t* ci, double* v) {
  const CsrMatrix* m[5] = {&s->sys.A, &s->sys.B, &s->sys.Bt, &s->sys.Q, &s->sys.Q_nu};
  csr_to_arrays(*m[which], rp, ci, v);
}

void ref_rhs(const ref_system* s, double* f) {
  std::memcpy(f, s->sys.f.data(), sizeof(double) * s->sys.f.size());
}

void ref_set_rhs(ref_system* s, const double* f) {
  std::memcpy(s->sys.f.data(), f, sizeof(double) * s->sys.f.size());
}

// StokesSystem::apply (proj/src/assembly.cpp:363-372).
void ref_apply(const ref_system* s, const double* x, double* y) { s->sys.apply(x, y); }

// Select the scalar kernels (proj/src/kernels.cpp:15-40) instead of the
// auto-detected AVX2 ones, so the C restatement can be pinned bit-exactly.
int ref_force_scalar(int on) {
  kernels::force_isa(on ? kernels::Isa::scalar : kernels::Isa::avx2);
  return static_cast<int>(kernels::active_isa());
}

// report7: iterations, converged, minres wall s, mean inner top, mean inner
// bottom, setup s (make_strategy), history length.
int ref_solve(ref_system* s, const char* strategy, double outer_tol, double inner_tol,
              int max_iter, int stop_euclid, double* u, double* p, double* report7,
              double* hist_m, double* hist_e, int hist_cap, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const std::string name(strategy);
    const auto t0 = std::chrono::steady_clock::now();
    BlockDiagPreconditioner precond;
    if (name == "IC0-PCG(A)+Diag(Q)") {
      precond.name = name;
      precond.n_top = s->sys.n_u();
      precond.n_bottom = s->sys.n_p();
      precond.top = std::make_unique<Ic0PcgBlock>(s->sys.A, inner_tol, 100000);
      precond.bottom = std::make_unique<DiagBlock>(s->sys.Q_nu);
    } else {
      precond = make_strategy(name, s->sys, inner_tol);
    }
    const double setup =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    SolverOptions opt;
    opt.outer_tol = outer_tol;
    opt.inner_tol = inner_tol;
    opt.max_iter = max_iter;
    opt.stop = stop_euclid ? MinresStop::euclidean : MinresStop::preconditioned;
    const StokesSolution sol = solve_stokes(s->sys, precond, opt);
    std::memcpy(u, sol.u.data(), sizeof(double) * sol.u.size());
    std::memcpy(p, sol.p.data(), sizeof(double) * sol.p.size());
    report7[0] = sol.report.iterations;
    report7[1] = sol.report.converged ? 1.0 : 0.0;
    report7[2] = sol.report.wall_seconds;
    report7[3] = sol.report.mean_inner_top;
    report7[4] = sol.report.mean_inner_bottom;
    report7[5] = setup;
    const int len = static_cast<int>(sol.report.residual_history.size());
    report7[6] = len;
    for (int i = 0; i < len && i < hist_cap; ++i) {
      if (hist_m) hist_m[i] = sol.report.residual_history[i];
      if (hist_e) hist_e[i] = sol.report.euclid_history[i];
    }
  });
}

// ---- a preconditioner kept across solves ---------------------------------
// make_strategy (proj/src/precond.cpp:161-193) once, then any number of
// solve_stokes(system, precond, options) calls (precond.cpp:245-290): at 96^3
// the reference's RCM + permute + ic0 is ~15 minutes, so the bounded
// (max_iter = k) and the full C5 solves share it. The block counters are
// cumulative in the reference; the per-call inner means are counter deltas.
struct ref_precond {
  BlockDiagPreconditioner p;
};

ref_precond* ref_precond_make(ref_system* s, const char* strategy, double inner_tol,
                              double* setup_seconds, char* err, int errlen) {
  ref_precond* out = nullptr;
  const int rc = guarded(err, errlen, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    auto* h = new ref_precond{make_strategy(strategy, s->sys, inner_tol)};
    *setup_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out = h;
  });
  return rc == 0 ? out : nullptr;
}

void ref_precond_free(ref_precond* h) { delete h; }

int ref_solve_with(ref_system* s, ref_precond* h, double outer_tol, double inner_tol,
                   int max_iter, int stop_euclid, double* u, double* p, double* report7,
                   double* hist_m, double* hist_e, int hist_cap, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    SolverOptions opt;
    opt.outer_tol = outer_tol;
    opt.inner_tol = inner_tol;
    opt.max_iter = max_iter;
    opt.stop = stop_euclid ? MinresStop::euclidean : MinresStop::preconditioned;
    const long it0 = h->p.top->inner_iterations(), ap0 = h->p.top->applications();
    const long ib0 = h->p.bottom->inner_iterations(), ab0 = h->p.bottom->applications();
    const StokesSolution sol = solve_stokes(s->sys, h->p, opt);
    std::memcpy(u, sol.u.data(), sizeof(double) * sol.u.size());
    std::memcpy(p, sol.p.data(), sizeof(double) * sol.p.size());
    const long at = h->p.top->applications() - ap0, ab = h->p.bottom->applications() - ab0;
    report7[0] = sol.report.iterations;
    report7[1] = sol.report.converged ? 1.0 : 0.0;
    report7[2] = sol.report.wall_seconds;
    report7[3] = at > 0 ? static_cast<double>(h->p.top->inner_iterations() - it0) / at : 0.0;
    report7[4] = ab > 0 ? static_cast<double>(h->p.bottom->inner_iterations() - ib0) / ab : 0.0;
    report7[5] = 0.0;
    const int len = static_cast<int>(sol.report.residual_history.size());
    report7[6] = len;
    for (int i = 0; i < len && i < hist_cap; ++i) {
      if (hist_m) hist_m[i] = sol.report.residual_history[i];
      if (hist_e) hist_e[i] = sol.report.euclid_history[i];
    }
  });
}

// MINRES from an initial guess: the reference's own minres (solvers.cpp:24-123) with
// MinresOptions::x0 (solvers.hpp:34) on the saddle operator and a kept
// preconditioner, exactly as solve_stokes sets it up (precond.cpp:245-258) --
// solve_stokes itself never passes x0, and its zero-mean pressure filter is not
// applied here. x0 / x: [u; p] in the original ordering.
int ref_minres_x0(ref_system* s, ref_precond* h, const double* x0, double outer_tol, int max_iter,
                  int stop_euclid, double* x, double* report3, double* hist_e, int hist_cap, char* err,
                  int errlen) {
  return guarded(err, errlen, [&] {
    const int n = s->sys.n_u() + s->sys.n_p();
    std::vector<double> b(n, 0.0), guess(x0, x0 + n);
    for (int i = 0; i < s->sys.n_u(); ++i) b[i] = s->sys.f[i];
    MinresOptions mopt;
    mopt.tol = outer_tol;
    mopt.max_iter = max_iter;
    mopt.stop = stop_euclid ? MinresStop::euclidean : MinresStop::preconditioned;
    mopt.x0 = &guess;
    SolveReport rep;
    LinearOperator op = [&](const double* in, double* out) { s->sys.apply(in, out); };
    const std::vector<double> sol = minres(op, b, h->p.as_operator(), mopt, rep);
    std::memcpy(x, sol.data(), sizeof(double) * n);
    report3[0] = rep.iterations;
    report3[1] = rep.converged ? 1.0 : 0.0;
    const int len = static_cast<int>(rep.euclid_history.size());
    report3[2] = len;
    for (int i = 0; i < len && i < hist_cap; ++i)
      if (hist_e) hist_e[i] = rep.euclid_history[i];
  });
}

// ---- solver-layer primitives -------------------------------------------

void ref_spmv(int n_rows, int n_cols, const int64_t* rp, const int32_t* ci, const double* v,
              const double* x, double* y) {
  (void)n_cols;
  kernels::spmv_csr(n_rows, rp, ci, v, x, y);
}

int ref_rcm(int n, const int64_t* rp, const int32_t* ci, int32_t* perm, char* err,
            int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<double> ones(rp[n], 1.0);
    const CsrMatrix m = csr_from_arrays(n, n, rp, ci, ones.data());
    const std::vector<int> p = rcm_permutation(m);
    for (int i = 0; i < n; ++i) perm[i] = p[i];
  });
}

int ref_bandwidth(int n, const int64_t* rp, const int32_t* ci) {
  std::vector<double> ones(rp[n], 1.0);
  return bandwidth(csr_from_arrays(n, n, rp, ci, ones.data()));
}

// Output arrays sized nnz(A) (permutation keeps the pattern size).
int ref_permute(int n, const int64_t* rp, const int32_t* ci, const double* v,
                const int32_t* perm, int64_t* out_rp, int32_t* out_ci, double* out_v,
                char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const CsrMatrix m = csr_from_arrays(n, n, rp, ci, v);
    const std::vector<int> p(perm, perm + n);
    csr_to_arrays(permute_symmetric(m, p), out_rp, out_ci, out_v);
  });
}

// L arrays sized nnz(lower(A)); *bad_row receives FactorBreakdown::row.
int ref_ic0(int n, const int64_t* rp, const int32_t* ci, const double* v, int64_t* l_rp,
            int32_t* l_ci, double* l_v, int* bad_row, char* err, int errlen) {
  *bad_row = -1;
  return guarded(err, errlen, [&] {
    try {
      const Ic0Factor f = ic0(csr_from_arrays(n, n, rp, ci, v));
      csr_to_arrays(f.lower, l_rp, l_ci, l_v);
    } catch (const FactorBreakdown& e) {
      *bad_row = e.row;
      throw;
    }
  });
}

void ref_ic0_solve(int n, const int64_t* l_rp, const int32_t* l_ci, const double* l_v,
                   const double* r, double* z) {
  Ic0Factor f{csr_from_arrays(n, n, l_rp, l_ci, l_v)};
  f.solve(r, z);
}

// pcg / minres on a CSR operator with a simple preconditioner:
// pre_kind 0 identity, 1 Jacobi (diag^-1), 2 IC(0) of the same matrix (no
// reordering). report3: iterations, converged, (minres) last relres.
int ref_pcg_csr(int n, const int64_t* rp, const int32_t* ci, const double* v, const double* b,
                int pre_kind, double tol, int max_iter, double* x, double* report3, char* err,
                int errlen) {
  return guarded(err, errlen, [&] {
    const CsrMatrix m = csr_from_arrays(n, n, rp, ci, v);
    std::vector<double> d = m.diagonal();
    std::unique_ptr<Ic0Factor> f;
    if (pre_kind == 2) f = std::make_unique<Ic0Factor>(ic0(m));
    LinearOperator op = [&m](const double* xx, double* yy) { m.multiply(xx, yy); };
    LinearOperator pre = [&](const double* r, double* z) {
      if (pre_kind == 0)
        for (int i = 0; i < n; ++i) z[i] = r[i];
      else if (pre_kind == 1)
        for (int i = 0; i < n; ++i) z[i] = r[i] / d[i];
      else
        f->solve(r, z);
    };
    std::vector<double> bb(b, b + n), sol;
    const PcgResult res = pcg(op, bb, pre, tol, max_iter, sol);
    std::memcpy(x, sol.data(), sizeof(double) * n);
    report3[0] = res.iterations;
    report3[1] = res.converged ? 1.0 : 0.0;
    report3[2] = 0.0;
  });
}

int ref_minres_csr(int n, const int64_t* rp, const int32_t* ci, const double* v,
                   const double* b, int pre_kind, double tol, int max_iter, int stop_euclid,
                   double* x, double* report3, double* hist_m, double* hist_e, int hist_cap,
                   char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const CsrMatrix m = csr_from_arrays(n, n, rp, ci, v);
    std::vector<double> d = m.diagonal();
    LinearOperator op = [&m](const double* xx, double* yy) { m.multiply(xx, yy); };
    LinearOperator pre = [&](const double* r, double* z) {
      if (pre_kind == 0)
        for (int i = 0; i < n; ++i) z[i] = r[i];
      else
        for (int i = 0; i < n; ++i) z[i] = r[i] / std::fabs(d[i]);
    };
    MinresOptions opt;
    opt.tol = tol;
    opt.max_iter = max_iter;
    opt.stop = stop_euclid ? MinresStop::euclidean : MinresStop::preconditioned;
    SolveReport rep;
    std::vector<double> bb(b, b + n);
    const std::vector<double> sol = minres(op, bb, pre, opt, rep);
    std::memcpy(x, sol.data(), sizeof(double) * n);
    report3[0] = rep.iterations;
    report3[1] = rep.converged ? 1.0 : 0.0;
    report3[2] = rep.residual_history.size();
    for (int i = 0; i < static_cast<int>(rep.residual_history.size()) && i < hist_cap; ++i) {
      if (hist_m) hist_m[i] = rep.residual_history[i];
      if (hist_e) hist_e[i] = rep.euclid_history[i];
    }
  });
}

// ---- Matrix Market wire format (csr.cpp:126-175), for the dump / load
// parity of the framework's reader and writer ---------------------------

int ref_write_mm(int n_rows, int n_cols, const int64_t* rp, const int32_t* ci, const double* v,
                 const char* path, int symmetric, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    write_matrix_market(csr_from_arrays(n_rows, n_cols, rp, ci, v), path, symmetric != 0);
  });
}

// Two calls: ref_read_mm returns the matrix (heap) and its sizes; ref_mm_take
// copies it out and frees it.
void* ref_read_mm(const char* path, int* n_rows, int* n_cols, int64_t* nnz, char* err, int errlen) {
  CsrMatrix* out = nullptr;
  const int rc = guarded(err, errlen, [&] {
    out = new CsrMatrix(read_matrix_market(path));
    *n_rows = out->n_rows;
    *n_cols = out->n_cols;
    *nnz = static_cast<int64_t>(out->cols.size());
  });
  return rc ? nullptr : out;
}

void ref_mm_take(void* m, int64_t* rp, int32_t* ci, double* v) {
  auto* a = static_cast<CsrMatrix*>(m);
  std::copy(a->row_ptr.begin(), a->row_ptr.end(), rp);
  std::copy(a->cols.begin(), a->cols.end(), ci);
  std::copy(a->vals.begin(), a->vals.end(), v);
  delete a;
}

}  // extern "C"
