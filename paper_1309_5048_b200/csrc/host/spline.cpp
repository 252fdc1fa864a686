// B-spline spaces and Gauss rules for the host assembler.
//
// Evaluation restates the published Cox-de Boor derivative algorithm
// (Piegl & Tiller A2.3), the same algorithm the reference uses
// (proj/src/spline.cpp:67-126), with identical operation order so the 2D
// matrices reproduce the reference's bit for bit. The Gauss rule restates the
// Newton/Legendre-recurrence construction of proj/src/quadrature.cpp:11-40.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "dshost.hpp"

namespace dshost {

Space1D make_space(int degree, int nelem) {
  if (degree < 0 || nelem < 1) throw std::invalid_argument("make_space: bad degree/nelem");
  Space1D s;
  s.p = degree;
  s.nelem = nelem;
  s.breaks.resize(nelem + 1);
  for (int j = 0; j <= nelem; ++j) s.breaks[j] = static_cast<double>(j) / nelem;
  // open knots, maximal regularity (interior multiplicity 1)
  s.t.assign(degree + 1, s.breaks.front());
  for (int j = 1; j < nelem; ++j) s.t.push_back(s.breaks[j]);
  s.t.insert(s.t.end(), degree + 1, s.breaks.back());
  s.n = static_cast<int>(s.t.size()) - degree - 1;
  s.first.resize(nelem);
  for (int e = 0; e < nelem; ++e) s.first[e] = s.find_span(0.5 * (s.breaks[e] + s.breaks[e + 1])) - degree;
  return s;
}

int Space1D::find_span(double x) const {
  if (x >= t[n]) return n - 1;  // left limit at the right end
  // last knot <= x among t[p..n] (right limit at interior knots)
  const auto it = std::upper_bound(t.begin() + p, t.begin() + n + 1, x);
  return static_cast<int>(it - t.begin()) - 1;
}

int Space1D::eval(double x, double* val, double* der) const {
  if (!(x >= 0.0 && x <= 1.0)) throw std::domain_error("spline eval: x outside [0,1]");
  const int span = find_span(x);
  const int P = p;
  // triangular table of basis values (upper part) and knot differences
  // (lower part), then one derivative order from it
  double ndu[8][8], left[8], right[8], a[2][8];
  if (P > 6) throw std::invalid_argument("spline eval: degree > 6 unsupported");
  ndu[0][0] = 1.0;
  for (int j = 1; j <= P; ++j) {
    left[j] = x - t[span + 1 - j];
    right[j] = t[span + j] - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];
      const double tmp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * tmp;
      saved = left[j - r] * tmp;
    }
    ndu[j][j] = saved;
  }
  for (int j = 0; j <= P; ++j) {
    val[j] = ndu[j][P];
    der[j] = 0.0;
  }
  if (P >= 1) {
    const int k = 1, pk = P - 1;
    for (int r = 0; r <= P; ++r) {
      a[0][0] = 1.0;
      double d = 0.0;
      const int rk = r - k;
      if (r >= k) {
        a[1][0] = a[0][0] / ndu[pk + 1][rk];
        d = a[1][0] * ndu[rk][pk];
      }
      // the middle loop (j1..j2) is empty for the first derivative
      if (r <= pk) {
        a[1][k] = -a[0][k - 1] / ndu[pk + 1][r];
        d += a[1][k] * ndu[r][pk];
      }
      der[r] = d;
    }
    for (int j = 0; j <= P; ++j) der[j] *= static_cast<double>(P);
  }
  return span - P;
}

namespace {
// Legendre P_n and P_{n-1} at x by the three-term recurrence
// k P_k = (2k - 1) x P_{k-1} - (k - 1) P_{k-2}.
struct LegendrePair {
  double pn, pnm1;
};
LegendrePair legendre_pair(int n, double x) {
  LegendrePair r{x, 1.0};
  for (int k = 2; k <= n; ++k) {
    const double next = ((2 * k - 1) * x * r.pn - (k - 1) * r.pnm1) / k;
    r.pnm1 = r.pn;
    r.pn = next;
  }
  return r;
}
}  // namespace

// n-point Gauss-Legendre rule on [0, 1]. The quadrature points feed the
// assembly, whose matrices are compared bit for bit with the reference's
// (tests/test_host.py), so the nodes must be the reference's doubles
// (proj/src/quadrature.cpp:11-40), not merely accurate ones: the same Chebyshev
// starting guess, Newton on P_n with P_n' = n (x P_n - P_{n-1}) / (x^2 - 1), the
// same stopping rule and the same weight formula, evaluated in the same order.
// The rule is symmetric; only the roots x > 0 are iterated.
Gauss gauss_legendre(int n) {
  if (n < 1) throw std::invalid_argument("gauss_legendre: need n >= 1");
  Gauss g;
  g.x.assign(n, 0.0);
  g.w.assign(n, 0.0);
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double root = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double slope = 0.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
      const LegendrePair p = legendre_pair(n, root);
      slope = n * (root * p.pn - p.pnm1) / (root * root - 1.0);
      const double step = p.pn / slope;
      root -= step;
      if (std::abs(step) < 1e-15) break;
    }
    const double weight = 2.0 / ((1.0 - root * root) * slope * slope);
    const int mirror = n - 1 - i;
    g.x[i] = 0.5 * (1.0 - root);
    g.x[mirror] = 0.5 * (1.0 + root);
    g.w[i] = g.w[mirror] = 0.5 * weight;
  }
  return g;
}

}  // namespace dshost
