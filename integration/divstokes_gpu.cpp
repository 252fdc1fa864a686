// Reference-side shim over the C ABI (include/dsgpu.h). Compiled against the
// reference headers; uses only the reference's public API.
#include "divstokes_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>
#include <vector>

#include "divstokes/analysis.hpp"
#include "divstokes/cholesky.hpp"
#include "divstokes/reorder.hpp"
#include "dsgpu.h"

namespace divstokes_gpu {
namespace {

using divstokes::CsrMatrix;

dsgpu_csr view(const CsrMatrix& m) {
  return dsgpu_csr{m.n_rows, m.n_cols, m.row_ptr.data(), m.cols.data(), m.vals.data()};
}

struct BlockSetup {
  int kind = DSGPU_BLOCK_JACOBI;
  std::vector<int32_t> perm;
  CsrMatrix factor;
};

BlockSetup prepare(const CsrMatrix& m, int kind) {
  BlockSetup b;
  b.kind = kind;
  if (kind == DSGPU_BLOCK_PCG_IC0) {
    const std::vector<int> p = divstokes::rcm_permutation(m);
    b.perm.assign(p.begin(), p.end());
    b.factor = divstokes::ic0(divstokes::permute_symmetric(m, p)).lower;
  }
  return b;
}

[[noreturn]] void rethrow(int code, const char* msg) {
  switch (code) {
    case DSGPU_E_INDEFINITE_PRECOND:
    case DSGPU_E_NEG_CURVATURE:
      throw std::runtime_error(msg);
    case DSGPU_E_NONPOS_DIAG:
      throw std::domain_error(msg);
    case DSGPU_E_BAD_INPUT:
    case DSGPU_E_UNSUPPORTED:
      throw std::invalid_argument(msg);
    default:
      throw std::runtime_error(std::string("dsgpu: ") + msg);
  }
}

}  // namespace

divstokes::StokesSolution solve_stokes(const divstokes::StokesSystem& sys,
                                       const std::string& strategy,
                                       const divstokes::SolverOptions& options, int device) {
  int top, bottom;
  if (strategy == "IC0-PCG(A,Q)") {
    top = bottom = DSGPU_BLOCK_PCG_IC0;
  } else if (strategy == "IC0-PCG(A)+Diag(Q)") {
    top = DSGPU_BLOCK_PCG_IC0;
    bottom = DSGPU_BLOCK_JACOBI;
  } else if (strategy == "PCG(A,Q)") {
    top = bottom = DSGPU_BLOCK_PCG_JACOBI;
  } else if (strategy == "PCG(A)+Diag(Q)") {
    top = DSGPU_BLOCK_PCG_JACOBI;
    bottom = DSGPU_BLOCK_JACOBI;
  } else if (strategy == "Diag(A,Q)") {
    top = bottom = DSGPU_BLOCK_JACOBI;
  } else {
    throw std::invalid_argument("unknown or host-only preconditioning strategy: " + strategy);
  }
  const BlockSetup bt = prepare(sys.A, top), bb = prepare(sys.Q_nu, bottom);

  dsgpu_handle* h = nullptr;
  int rc = dsgpu_create(device, &h);
  if (rc) rethrow(rc, dsgpu_last_error(nullptr));
  std::unique_ptr<dsgpu_handle, void (*)(dsgpu_handle*)> guard(h, dsgpu_destroy);
  const dsgpu_csr A = view(sys.A), B = view(sys.B), Bt = view(sys.Bt), Qn = view(sys.Q_nu);
  const dsgpu_csr LA = view(bt.factor), LQ = view(bb.factor);
  rc = dsgpu_setup(h, &A, &B, &Bt, &Qn, top, bt.perm.empty() ? nullptr : bt.perm.data(),
                   bt.perm.empty() ? nullptr : &LA, bottom,
                   bb.perm.empty() ? nullptr : bb.perm.data(), bb.perm.empty() ? nullptr : &LQ,
                   nullptr /* filter applied below with the reference's kernel vector */);
  if (rc) rethrow(rc, dsgpu_last_error(h));

  dsgpu_opts o;
  dsgpu_default_opts(&o);
  o.outer_tol = options.outer_tol;
  o.inner_tol = options.inner_tol;
  o.max_iter = options.max_iter;
  o.stop = options.stop == divstokes::MinresStop::euclidean ? DSGPU_STOP_EUCLIDEAN
                                                            : DSGPU_STOP_PRECONDITIONED;
  divstokes::StokesSolution sol;
  sol.u.assign(sys.n_u(), 0.0);
  sol.p.assign(sys.n_p(), 0.0);
  std::vector<double> hm(options.max_iter + 1), he(options.max_iter + 1);
  dsgpu_report rep{};
  rc = dsgpu_solve(h, sys.f.data(), &o, sol.u.data(), sol.p.data(), &rep, hm.data(), he.data(),
                   static_cast<int32_t>(hm.size()));
  if (rc) rethrow(rc, dsgpu_last_error(h));
  sol.report.iterations = rep.iterations;
  sol.report.converged = rep.converged != 0;
  sol.report.wall_seconds = rep.wall_seconds;
  sol.report.mean_inner_top = rep.mean_inner_top;
  sol.report.mean_inner_bottom = rep.mean_inner_bottom;
  const int len = std::min<int>(rep.hist_len, static_cast<int>(hm.size()));
  sol.report.residual_history.assign(hm.begin(), hm.begin() + len);
  sol.report.euclid_history.assign(he.begin(), he.begin() + len);

  // zero-mean filter exactly as solve_stokes (precond.cpp:266-284)
  if (sys.pair && sys.map) {
    const std::vector<double> kernel =
        divstokes::constant_pressure_coefficients(*sys.pair, *sys.map);
    std::vector<double> btk(sys.n_u());
    sys.Bt.multiply(kernel.data(), btk.data());
    double resid = 0.0, bscale = 0.0;
    for (const double v : btk) resid = std::max(resid, std::abs(v));
    for (const double v : sys.B.vals) bscale = std::max(bscale, std::abs(v));
    if (resid <= 1e-10 * bscale) {
      const std::vector<double> qk = sys.Q.multiply(kernel);
      double num = 0.0, den = 0.0;
      for (int i = 0; i < sys.n_p(); ++i) {
        num += qk[i] * sol.p[i];
        den += qk[i] * kernel[i];
      }
      const double mean = num / den;
      for (int i = 0; i < sys.n_p(); ++i) sol.p[i] -= mean * kernel[i];
    }
  }
  return sol;
}

}  // namespace divstokes_gpu

// extern "C" hook used by tests/test_gpu_integration.py (through
// oracle/ref_driver's ref_system handle layout: a StokesSystem first member).
extern "C" int divstokes_gpu_solve(const void* ref_system, const char* strategy,
                                   double outer_tol, double inner_tol, int max_iter,
                                   double* u, double* p, double* report4, char* err, int errlen) {
  try {
    const auto* sys = static_cast<const divstokes::StokesSystem*>(ref_system);
    divstokes::SolverOptions opt;
    opt.outer_tol = outer_tol;
    opt.inner_tol = inner_tol;
    opt.max_iter = max_iter;
    const divstokes::StokesSolution s = divstokes_gpu::solve_stokes(*sys, strategy, opt);
    std::copy(s.u.begin(), s.u.end(), u);
    std::copy(s.p.begin(), s.p.end(), p);
    report4[0] = s.report.iterations;
    report4[1] = s.report.converged ? 1.0 : 0.0;
    report4[2] = s.report.mean_inner_top;
    report4[3] = s.report.mean_inner_bottom;
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen > 0) {
      std::string m = e.what();
      m = m.substr(0, errlen - 1);
      std::copy(m.begin(), m.end(), err);
      err[m.size()] = '\0';
    }
    return 1;
  }
}
