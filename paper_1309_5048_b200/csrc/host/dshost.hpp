// Host-side input producer and setup for the B200 Stokes solve.
//
// The reference keeps assembly, RCM and the IC(0) factor on the host in C++
// (L1 reorder/cholesky, L4 spaces/assembly). This is a native
// re-design of that host side so the framework can build its own inputs:
//   * divergence-conforming B-spline pair + Stokes assembly for the unit
//     square (2D) and unit cube (3D), pattern-first (CSR pattern from the
//     tensor-product support overlap, values accumulated in place), which
//     reproduces the reference's 2D matrices bit for bit (the per-entry
//     summation order equals the reference's triplet insertion order,
//     proj/src/assembly.cpp:106-295 + csr_from_triplets proj/src/csr.cpp:88-111);
//   * rcm_permutation / permute_symmetric / ic0 with the reference's exact
//     rules (proj/src/reorder.cpp:9-55, proj/src/csr.cpp:113-124,
//     proj/src/cholesky.cpp:84-134), so the factor handed to the GPU is
//     bit-identical to the one PcgBlock builds (proj/src/precond.cpp:61-64).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dshost {

struct Csr {
  int n_rows = 0, n_cols = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  int64_t nnz() const { return static_cast<int64_t>(ci.size()); }
};

// ---- splines / quadrature ---------------------------------------------------
struct Space1D {
  int p = 0;        // degree
  int n = 0;        // basis count
  int nelem = 0;
  std::vector<double> t;       // open knot vector, interior multiplicity 1
  std::vector<double> breaks;  // j / nelem
  std::vector<int> first;      // first supported basis per element
  int find_span(double x) const;
  // values (row 0) and first derivatives (row 1) of the p+1 supported
  // functions; returns the first supported index
  int eval(double x, double* val, double* der) const;
  // element support range [lo, hi] of basis i
  int supp_lo(int i) const { return i - p < 0 ? 0 : i - p; }
  int supp_hi(int i) const { return i > nelem - 1 ? nelem - 1 : i; }
};
Space1D make_space(int degree, int nelem);

struct Gauss {
  std::vector<double> x, w;  // on [0,1]
};
Gauss gauss_legendre(int n);

// ---- systems ----------------------------------------------------------------
enum CaseId { kPsiMms = 0, kCavity = 1, kRandom = 3 };

struct System {
  int dim = 2, k_prime = 2, n_elem = 0;
  double nu = 1.0, c_pen = 0.0;
  int n_u = 0, n_p = 0;
  Csr A, B, Bt, Q, Q_nu;
  std::vector<double> f;
};

// Throws std::invalid_argument on bad parameters.
System assemble(int dim, int k_prime, int n_elem, int case_id, double nu, uint64_t seed);

// ---- sparse setup (reference-exact) -------------------------------------
Csr transpose(const Csr& a);
bool pattern_symmetric(const Csr& a);
std::vector<int32_t> rcm_permutation(const Csr& a);  // throws on nonsymmetric pattern
Csr permute_symmetric(const Csr& a, const std::vector<int32_t>& perm);
// Matrix Market dump / load (proj/src/csr.cpp:126-175), mmio.cpp
void write_matrix_market(const Csr& a, const std::string& path, bool symmetric);
Csr read_matrix_market(const std::string& path);
// IC(0) of a; throws ic0_breakdown{row} or std::invalid_argument (missing diagonal)
struct Ic0Breakdown {
  int row;
};
Csr ic0(const Csr& a);

}  // namespace dshost
