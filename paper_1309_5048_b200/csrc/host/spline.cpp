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

Gauss gauss_legendre(int n) {
  if (n < 1) throw std::invalid_argument("gauss_legendre: need n >= 1");
  Gauss g;
  g.x.resize(n);
  g.w.resize(n);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = pk;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    g.x[i] = 0.5 * (1.0 - x);
    g.x[n - 1 - i] = 0.5 * (1.0 + x);
    g.w[i] = 0.5 * w;
    g.w[n - 1 - i] = 0.5 * w;
  }
  return g;
}

}  // namespace dshost
