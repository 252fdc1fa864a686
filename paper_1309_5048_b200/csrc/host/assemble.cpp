// Pattern-first assembly of the divergence-conforming B-spline Stokes system
// on the unit square (D=2) and unit cube (D=3), identity map.
//
// Discretization (reference proj/src/spaces.cpp:28-82, assembly.cpp:106-295):
//   velocity component c has degree p = k'+1 in direction c and p-1 in the
//   others (maximal regularity); pressure has degree p-1 everywhere; the DOFs
//   with nonzero normal trace (first/last index of component c in direction
//   c) are removed; velocity ids run over component 0 (x fastest), then 1
//   (then 2); pressure ids are lexicographic.
//   A = 2 nu (grad^s u, grad^s v) - Nitsche terms with C_pen = 5 (k'+1) /
//   h_F on every boundary face; B = -(div u, q); Q = (p, q); Q_nu = Q/(2 nu).
//   (p+1)-point Gauss rule per direction.
//
// Why pattern-first: the reference builds ~nv^2 triplets per element and a
// stable sort (csr_from_triplets), which does not scale to the 3D configs.
// Here the CSR pattern is generated from the tensor-product support overlap
// (two basis functions couple iff they share an element) and element
// contributions are added into their slots in element order, then face order
// -- exactly the reference's triplet insertion order, so in 2D every entry is
// the same floating-point sum as the reference's (bit-identical matrices; see
// tests/test_host.py). Local element matrices are computed in parallel
// batches (OpenMP) and scattered serially in element order, so the result does
// not depend on the thread count.
#include <algorithm>
#include <array>
#include <cmath>
#include <random>
#include <stdexcept>

#include "dshost.hpp"

namespace dshost {
namespace {

template <int D>
struct Pair {
  int kp = 0, p = 0, N = 0;
  Space1D hi, lo;
  // basis counts per (component c or pressure D, direction d)
  int nb[D + 1][D];
  std::vector<int> vid[D];  // tensor flat -> velocity id or -1
  int n_u = 0, n_p = 0;

  const Space1D& space(int c, int d) const { return (c < D && c == d) ? hi : lo; }
  int flat(int c, const int* idx) const {
    int f = 0;
    for (int d = D - 1; d >= 0; --d) f = f * nb[c][d] + idx[d];
    return f;
  }
  int dim(int c) const {
    int n = 1;
    for (int d = 0; d < D; ++d) n *= nb[c][d];
    return n;
  }
};

template <int D>
Pair<D> build_pair(int k_prime, int N) {
  if (k_prime < 1) throw std::invalid_argument("build_pair: k' must be >= 1");
  if (N < 2) throw std::invalid_argument("build_pair: need at least 2 elements per direction");
  Pair<D> P;
  P.kp = k_prime;
  P.p = k_prime + 1;
  P.N = N;
  P.hi = make_space(P.p, N);
  P.lo = make_space(P.p - 1, N);
  for (int c = 0; c <= D; ++c)
    for (int d = 0; d < D; ++d) P.nb[c][d] = P.space(c, d).n;
  int next = 0;
  for (int c = 0; c < D; ++c) {
    P.vid[c].assign(P.dim(c), -1);
    int idx[D] = {};
    const int total = P.dim(c);
    for (int f = 0; f < total; ++f) {
      int rem = f;
      for (int d = 0; d < D; ++d) {
        idx[d] = rem % P.nb[c][d];
        rem /= P.nb[c][d];
      }
      const bool removed = idx[c] == 0 || idx[c] == P.nb[c][c] - 1;
      if (!removed) P.vid[c][f] = next++;
    }
  }
  P.n_u = next;
  P.n_p = P.dim(D);
  return P;
}

// ---- forcing ---------------------------------------------------------------
// BASELINE psi-MMS. 2D: u = curl psi = (psi_y, -psi_x),
// psi = X(x) Y(y), X = x^2 (1-x)^2, p = sin(pi x) sin(pi y). 3D: u =
// curl(psi, psi, psi), psi = X Y Z, p = sin(pi x) sin(pi y) sin(pi z).
// f = -nu lap u + grad p (div u = 0).
struct Poly {
  double f, f1, f2, f3;
  explicit Poly(double x)
      : f(x * x * (1.0 - x) * (1.0 - x)),
        f1(((4.0 * x - 6.0) * x + 2.0) * x),
        f2((12.0 * x - 12.0) * x + 2.0),
        f3(24.0 * x - 12.0) {}
};

void psi_mms_force2(const double* q, double nu, double* out) {
  const Poly X(q[0]), Y(q[1]);
  const double lap_u1 = X.f2 * Y.f1 + X.f * Y.f3;
  const double lap_u2 = -(X.f3 * Y.f + X.f1 * Y.f2);
  const double px = M_PI * std::cos(M_PI * q[0]) * std::sin(M_PI * q[1]);
  const double py = M_PI * std::sin(M_PI * q[0]) * std::cos(M_PI * q[1]);
  out[0] = -nu * lap_u1 + px;
  out[1] = -nu * lap_u2 + py;
}

void psi_mms_force3(const double* q, double nu, double* out) {
  const Poly X(q[0]), Y(q[1]), Z(q[2]);
  // lap of the gradient components of psi
  const double lap_px = X.f3 * Y.f * Z.f + X.f1 * Y.f2 * Z.f + X.f1 * Y.f * Z.f2;
  const double lap_py = X.f2 * Y.f1 * Z.f + X.f * Y.f3 * Z.f + X.f * Y.f1 * Z.f2;
  const double lap_pz = X.f2 * Y.f * Z.f1 + X.f * Y.f2 * Z.f1 + X.f * Y.f * Z.f3;
  const double s[3] = {std::sin(M_PI * q[0]), std::sin(M_PI * q[1]), std::sin(M_PI * q[2])};
  const double c[3] = {std::cos(M_PI * q[0]), std::cos(M_PI * q[1]), std::cos(M_PI * q[2])};
  out[0] = -nu * (lap_py - lap_pz) + M_PI * c[0] * s[1] * s[2];
  out[1] = -nu * (lap_pz - lap_px) + M_PI * s[0] * c[1] * s[2];
  out[2] = -nu * (lap_px - lap_py) + M_PI * s[0] * s[1] * c[2];
}

// ---- pattern ------------------------------------------------------------------
// Rows of basis (space S, index i) couple with basis j of space S' iff their
// element supports intersect: j in [lo_S(i), min(n'-1, hi_S(i) + p')].
inline void overlap(const Space1D& s, int i, const Space1D& t, int& j0, int& j1) {
  j0 = s.supp_lo(i);
  j1 = std::min(t.n - 1, s.supp_hi(i) + t.p);
}

// Enumerate the sorted global column list of one row. Row basis: component
// rc (D = pressure) at multi-index ridx. Column family: velocity (all
// components, kept ids) or pressure.
template <int D, class Emit>
void row_cols(const Pair<D>& P, int rc, const int* ridx, bool vel_cols, Emit&& emit) {
  const int c_lo = vel_cols ? 0 : D, c_hi = vel_cols ? D - 1 : D;
  for (int cc = c_lo; cc <= c_hi; ++cc) {
    int j0[D], j1[D];
    for (int d = 0; d < D; ++d) overlap(P.space(rc, d), ridx[d], P.space(cc, d), j0[d], j1[d]);
    int idx[D];
    for (int d = 0; d < D; ++d) idx[d] = j0[d];
    while (true) {
      const int f = P.flat(cc, idx);
      const int id = cc < D ? P.vid[cc][f] : f;
      if (id >= 0) emit(cc < D ? id : f);
      int d = 0;
      for (; d < D; ++d) {
        if (++idx[d] <= j1[d]) break;
        idx[d] = j0[d];
      }
      if (d == D) break;
    }
  }
}

template <int D>
Csr build_pattern(const Pair<D>& P, bool vel_rows, bool vel_cols) {
  Csr m;
  m.n_rows = vel_rows ? P.n_u : P.n_p;
  m.n_cols = vel_cols ? P.n_u : P.n_p;
  m.rp.assign(m.n_rows + 1, 0);
  // two passes: count, fill
  for (int pass = 0; pass < 2; ++pass) {
    int64_t pos = 0;
    const int c_lo = vel_rows ? 0 : D, c_hi = vel_rows ? D - 1 : D;
    for (int rc = c_lo; rc <= c_hi; ++rc) {
      const int total = P.dim(rc);
      int idx[D];
      for (int f = 0; f < total; ++f) {
        int rem = f;
        for (int d = 0; d < D; ++d) {
          idx[d] = rem % P.nb[rc][d];
          rem /= P.nb[rc][d];
        }
        const int row = rc < D ? P.vid[rc][f] : f;
        if (row < 0) continue;
        if (pass == 0) {
          int64_t cnt = 0;
          row_cols<D>(P, rc, idx, vel_cols, [&](int) { ++cnt; });
          m.rp[row + 1] = cnt;
        } else {
          int64_t at = m.rp[row];
          row_cols<D>(P, rc, idx, vel_cols, [&](int col) { m.ci[at++] = col; });
        }
        (void)pos;
      }
    }
    if (pass == 0) {
      for (int i = 0; i < m.n_rows; ++i) m.rp[i + 1] += m.rp[i];
      m.ci.resize(m.rp[m.n_rows]);
      m.v.assign(m.rp[m.n_rows], 0.0);
    }
  }
  return m;
}

inline int64_t slot(const Csr& m, int row, int col) {
  const auto b = m.ci.begin() + m.rp[row], e = m.ci.begin() + m.rp[row + 1];
  const auto it = std::lower_bound(b, e, col);
  return it - m.ci.begin();
}

// ---- per-point basis data ----------------------------------------------------
template <int D>
struct VelPoint {
  int comp;
  double v;            // value of the (only nonzero) component
  double s[D][D];      // symmetric gradient
  double divhat;
};

// 1D tables at the Gauss points of every element: [e][a][0..p]
struct Tab1 {
  int p = 0, q = 0;
  std::vector<double> val, der;
  void build(const Space1D& s, const Gauss& g) {
    p = s.p;
    q = static_cast<int>(g.x.size());
    val.assign(static_cast<size_t>(s.nelem) * q * (p + 1), 0.0);
    der.assign(val.size(), 0.0);
    for (int e = 0; e < s.nelem; ++e)
      for (int a = 0; a < q; ++a) {
        const double x = s.breaks[e] + (s.breaks[e + 1] - s.breaks[e]) * g.x[a];
        s.eval(x, &val[(static_cast<size_t>(e) * q + a) * (p + 1)],
               &der[(static_cast<size_t>(e) * q + a) * (p + 1)]);
      }
  }
  const double* v(int e, int a) const { return &val[(static_cast<size_t>(e) * q + a) * (p + 1)]; }
  const double* d(int e, int a) const { return &der[(static_cast<size_t>(e) * q + a) * (p + 1)]; }
};

// Local velocity basis of one element: per local index its component and
// per-direction local offsets (0..deg); ordering = component, then z, y, x
// (x fastest), reference proj/src/spaces.cpp:84-106.
template <int D>
struct LocalLayout {
  int nv = 0, np = 0;
  std::vector<int> comp;
  std::vector<std::array<int, D>> off;
  std::vector<std::array<int, D>> poff;
  explicit LocalLayout(const Pair<D>& P) {
    for (int c = 0; c <= D; ++c) {
      int deg[D], idx[D] = {};
      int cnt = 1;
      for (int d = 0; d < D; ++d) {
        deg[d] = P.space(c, d).p;
        cnt *= deg[d] + 1;
      }
      for (int f = 0; f < cnt; ++f) {
        int rem = f;
        for (int d = 0; d < D; ++d) {
          idx[d] = rem % (deg[d] + 1);
          rem /= deg[d] + 1;
        }
        std::array<int, D> o;
        for (int d = 0; d < D; ++d) o[d] = idx[d];
        if (c < D) {
          comp.push_back(c);
          off.push_back(o);
        } else {
          poff.push_back(o);
        }
      }
    }
    nv = static_cast<int>(comp.size());
    np = static_cast<int>(poff.size());
  }
};

// Velocity basis data at one point from per-direction tables.
// tv[c][d] / td[c][d]: value / derivative tables of space(c, d).
template <int D>
void eval_vel(const LocalLayout<D>& L, const double* const tv[D][D], const double* const td[D][D],
              std::vector<VelPoint<D>>& out) {
  out.resize(L.nv);
  for (int i = 0; i < L.nv; ++i) {
    const int c = L.comp[i];
    const auto& o = L.off[i];
    double vhat = tv[c][0][o[0]];
    for (int d = 1; d < D; ++d) vhat = vhat * tv[c][d][o[d]];
    double g[D];  // gradhat row c
    for (int k = 0; k < D; ++k) {
      double acc = (k == 0) ? td[c][0][o[0]] : tv[c][0][o[0]];
      for (int d = 1; d < D; ++d) acc = acc * ((k == d) ? td[c][d][o[d]] : tv[c][d][o[d]]);
      g[k] = acc;
    }
    VelPoint<D>& vp = out[i];
    vp.comp = c;
    vp.v = vhat;
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) vp.s[a][b] = 0.0;
    vp.s[c][c] = g[c];
    for (int b = 0; b < D; ++b)
      if (b != c) {
        // 0.5 (grad_cb + grad_bc); only row c of gradhat is nonzero
        const double sym = (c < b) ? 0.5 * (g[b] + 0.0) : 0.5 * (0.0 + g[b]);
        vp.s[c][b] = vp.s[b][c] = sym;
      }
    vp.divhat = g[c];
  }
}

template <int D>
inline double contraction(const VelPoint<D>& a, const VelPoint<D>& b) {
  double acc = a.s[0][0] * b.s[0][0];
  for (int d = 1; d < D; ++d) acc = acc + a.s[d][d] * b.s[d][d];
  for (int x = 0; x < D; ++x)
    for (int y = x + 1; y < D; ++y) acc = acc + 2.0 * a.s[x][y] * b.s[x][y];
  return acc;
}

template <int D>
inline double vdot(const VelPoint<D>& a, const VelPoint<D>& b) {
  // full-vector dot in component order; zero components contribute +-0
  double acc = (a.comp == 0 ? a.v : 0.0) * (b.comp == 0 ? b.v : 0.0);
  for (int d = 1; d < D; ++d) acc = acc + (a.comp == d ? a.v : 0.0) * (b.comp == d ? b.v : 0.0);
  return acc;
}

template <int D>
System assemble_dim(int k_prime, int N, int case_id, double nu, uint64_t seed) {
  const Pair<D> P = build_pair<D>(k_prime, N);
  const LocalLayout<D> L(P);
  const int nv = L.nv, np = L.np;
  const int q = P.p + 1;
  const Gauss g = gauss_legendre(q);
  const double two_nu = 2.0 * nu;
  const double c_pen = 5.0 * (k_prime + 1);

  System S;
  S.dim = D;
  S.k_prime = k_prime;
  S.n_elem = N;
  S.nu = nu;
  S.c_pen = c_pen;
  S.n_u = P.n_u;
  S.n_p = P.n_p;
  S.A = build_pattern<D>(P, true, true);
  S.B = build_pattern<D>(P, false, true);
  S.Q = build_pattern<D>(P, false, false);
  S.f.assign(P.n_u, 0.0);
  const bool body = case_id == kPsiMms;

  Tab1 th, tl;
  th.build(P.hi, g);
  tl.build(P.lo, g);
  auto tab = [&](int c, int d) -> const Tab1& { return (c < D && c == d) ? th : tl; };

  int n_elem_total = 1;
  for (int d = 0; d < D; ++d) n_elem_total *= N;

  const int batch = 256;
  const size_t la = static_cast<size_t>(nv) * nv, lb = static_cast<size_t>(np) * nv,
               lq = static_cast<size_t>(np) * np;
  std::vector<double> bufA(batch * la), bufB(batch * lb), bufQ(batch * lq), bufF(batch * nv);

  for (int e0 = 0; e0 < n_elem_total; e0 += batch) {
    const int e1 = std::min(n_elem_total, e0 + batch);
#pragma omp parallel for schedule(dynamic, 4)
    for (int e = e0; e < e1; ++e) {
      double* al = &bufA[(e - e0) * la];
      double* bl = &bufB[(e - e0) * lb];
      double* ql = &bufQ[(e - e0) * lq];
      double* fl = &bufF[(e - e0) * nv];
      std::fill(al, al + la, 0.0);
      std::fill(bl, bl + lb, 0.0);
      std::fill(ql, ql + lq, 0.0);
      std::fill(fl, fl + nv, 0.0);
      int ei[D];
      {
        int rem = e;
        for (int d = 0; d < D; ++d) {
          ei[d] = rem % N;
          rem /= N;
        }
      }
      double x0[D], hx[D];
      for (int d = 0; d < D; ++d) {
        x0[d] = P.hi.breaks[ei[d]];
        hx[d] = P.hi.breaks[ei[d] + 1] - P.hi.breaks[ei[d]];
      }
      double area = hx[0];
      for (int d = 1; d < D; ++d) area = area * hx[d];
      std::vector<VelPoint<D>> vel;
      std::vector<double> press(np);
      int qa[D] = {};
      const int nq = (D == 2) ? q * q : q * q * q;
      for (int qq = 0; qq < nq; ++qq) {
        // point order: x outermost, last direction innermost
        {
          int rem = qq;
          for (int d = D - 1; d >= 0; --d) {
            qa[d] = rem % q;
            rem /= q;
          }
        }
        double w = g.w[qa[0]];
        for (int d = 1; d < D; ++d) w = w * g.w[qa[d]];
        w = w * area;
        const double wj = w * 1.0;  // det DF = 1 (identity map)
        const double* tv[D][D];
        const double* td[D][D];
        for (int c = 0; c < D; ++c)
          for (int d = 0; d < D; ++d) {
            tv[c][d] = tab(c, d).v(ei[d], qa[d]);
            td[c][d] = tab(c, d).d(ei[d], qa[d]);
          }
        eval_vel<D>(L, tv, td, vel);
        for (int k = 0; k < np; ++k) {
          const auto& o = L.poff[k];
          double pv = tl.v(ei[0], qa[0])[o[0]];
          for (int d = 1; d < D; ++d) pv = pv * tl.v(ei[d], qa[d])[o[d]];
          press[k] = pv;
        }
        const double wt = wj * two_nu;
        for (int i = 0; i < nv; ++i)
          for (int j = 0; j <= i; ++j) al[i * nv + j] += wt * contraction<D>(vel[i], vel[j]);
        const double bscale = -w / 1.0;
        for (int k = 0; k < np; ++k) {
          const double sp = bscale * press[k];
          for (int j = 0; j < nv; ++j) bl[k * nv + j] += sp * vel[j].divhat;
        }
        const double qscale = w / 1.0;
        for (int k = 0; k < np; ++k) {
          const double sp = qscale * press[k];
          for (int l = 0; l <= k; ++l) ql[k * np + l] += sp * press[l];
        }
        if (body) {
          double xq[D], fv[D];
          for (int d = 0; d < D; ++d) xq[d] = x0[d] + hx[d] * g.x[qa[d]];
          if (D == 2)
            psi_mms_force2(xq, nu, fv);
          else
            psi_mms_force3(xq, nu, fv);
          for (int i = 0; i < nv; ++i) {
            // dot(f, v_i) over all components in order
            double acc = fv[0] * (vel[i].comp == 0 ? vel[i].v : 0.0);
            for (int d = 1; d < D; ++d) acc = acc + fv[d] * (vel[i].comp == d ? vel[i].v : 0.0);
            fl[i] += wj * acc;
          }
        }
      }
    }
    // serial scatter in element order (= reference triplet order)
    for (int e = e0; e < e1; ++e) {
      const double* al = &bufA[(e - e0) * la];
      const double* bl = &bufB[(e - e0) * lb];
      const double* ql = &bufQ[(e - e0) * lq];
      const double* fl = &bufF[(e - e0) * nv];
      int ei[D];
      {
        int rem = e;
        for (int d = 0; d < D; ++d) {
          ei[d] = rem % N;
          rem /= N;
        }
      }
      std::vector<int> vids(nv), pids(np);
      for (int i = 0; i < nv; ++i) {
        int idx[D];
        for (int d = 0; d < D; ++d) idx[d] = P.space(L.comp[i], d).first[ei[d]] + L.off[i][d];
        vids[i] = P.vid[L.comp[i]][P.flat(L.comp[i], idx)];
      }
      for (int k = 0; k < np; ++k) {
        int idx[D];
        for (int d = 0; d < D; ++d) idx[d] = P.lo.first[ei[d]] + L.poff[k][d];
        pids[k] = P.flat(D, idx);
      }
      for (int i = 0; i < nv; ++i) {
        if (vids[i] < 0) continue;
        for (int j = 0; j <= i; ++j) {
          if (vids[j] < 0) continue;
          const double v = al[i * nv + j];
          S.A.v[slot(S.A, vids[i], vids[j])] += v;
          if (i != j) S.A.v[slot(S.A, vids[j], vids[i])] += v;
        }
      }
      for (int k = 0; k < np; ++k)
        for (int j = 0; j < nv; ++j) {
          if (vids[j] < 0) continue;
          S.B.v[slot(S.B, pids[k], vids[j])] += bl[k * nv + j];
        }
      for (int k = 0; k < np; ++k)
        for (int l = 0; l <= k; ++l) {
          const double v = ql[k * np + l];
          S.Q.v[slot(S.Q, pids[k], pids[l])] += v;
          if (k != l) S.Q.v[slot(S.Q, pids[l], pids[k])] += v;
        }
      if (body)
        for (int i = 0; i < nv; ++i)
          if (vids[i] >= 0) S.f[vids[i]] += fl[i];
    }
  }

  // Nitsche face terms (reference assembly.cpp:230-293): sides in the order
  // x=0, x=1, y=0, y=1 (, z=0, z=1); faces in lexicographic order of the
  // tangential element indices; nodes in lexicographic order of the
  // tangential Gauss indices (first tangential direction outermost).
  {
    std::vector<double> face_a(static_cast<size_t>(nv) * nv), face_f(nv);
    std::vector<VelPoint<D>> vel;
    double tnv[D][D][8], tnd[D][D][8];
    for (int side = 0; side < 2 * D; ++side) {
      const int nd = side / 2;     // normal direction
      const int hi_side = side % 2;
      double nrm[D] = {};
      nrm[nd] = hi_side ? 1.0 : -1.0;
      int tdirs[D - 1], t = 0;
      for (int d = 0; d < D; ++d)
        if (d != nd) tdirs[t++] = d;
      int n_faces = 1;
      for (int k = 0; k < D - 1; ++k) n_faces *= N;
      for (int fidx = 0; fidx < n_faces; ++fidx) {
        // tangential element indices: last tangential direction slowest
        int ei[D];
        {
          int rem = fidx;
          for (int k = D - 2; k >= 0; --k) {
            ei[tdirs[k]] = rem % N;
            rem /= N;
          }
        }
        // for D=2 the single tangential index is fidx itself
        ei[nd] = hi_side ? N - 1 : 0;
        std::fill(face_a.begin(), face_a.end(), 0.0);
        std::fill(face_f.begin(), face_f.end(), 0.0);
        // h_F: face extent (2D: arc length; 3D: sqrt of the face area)
        double h_F = 0.0;
        int n_nodes = 1;
        for (int k = 0; k < D - 1; ++k) n_nodes *= q;
        for (int node = 0; node < n_nodes; ++node) {
          int qa[D - 1];
          int rem = node;
          for (int k = D - 2; k >= 0; --k) {
            qa[k] = rem % q;
            rem /= q;
          }
          double weight = 1.0;
          for (int k = 0; k < D - 1; ++k) {
            const int d = tdirs[k];
            const double wk = (P.hi.breaks[ei[d] + 1] - P.hi.breaks[ei[d]]) * g.w[qa[k]];
            weight = (k == 0) ? wk : weight * wk;
          }
          h_F += weight * 1.0;
        }
        if (D == 3) h_F = std::sqrt(h_F);
        const double pen = c_pen / h_F;
        for (int node = 0; node < n_nodes; ++node) {
          int qa[D - 1];
          int rem = node;
          for (int k = D - 2; k >= 0; --k) {
            qa[k] = rem % q;
            rem /= q;
          }
          double xh[D];
          double weight = 1.0;
          for (int k = 0; k < D - 1; ++k) {
            const int d = tdirs[k];
            const double t0 = P.hi.breaks[ei[d]], t1 = P.hi.breaks[ei[d] + 1];
            xh[d] = t0 + (t1 - t0) * g.x[qa[k]];
            const double wk = (t1 - t0) * g.w[qa[k]];
            weight = (k == 0) ? wk : weight * wk;
          }
          xh[nd] = hi_side ? 1.0 : 0.0;
          const double* tv[D][D];
          const double* td[D][D];
          for (int c = 0; c < D; ++c)
            for (int d = 0; d < D; ++d) {
              P.space(c, d).eval(xh[d], tnv[c][d], tnd[c][d]);
              tv[c][d] = tnv[c][d];
              td[c][d] = tnd[c][d];
            }
          eval_vel<D>(L, tv, td, vel);
          const double ds = weight * 1.0;
          std::vector<std::array<double, D>> tn(nv);
          for (int i = 0; i < nv; ++i)
            for (int a = 0; a < D; ++a) {
              double acc = vel[i].s[a][0] * nrm[0];
              for (int b = 1; b < D; ++b) acc = acc + vel[i].s[a][b] * nrm[b];
              tn[i][a] = acc;
            }
          auto tdot = [&](int i, int j) {  // dot(tn_i, v_j)
            double acc = tn[i][0] * (vel[j].comp == 0 ? vel[j].v : 0.0);
            for (int a = 1; a < D; ++a) acc = acc + tn[i][a] * (vel[j].comp == a ? vel[j].v : 0.0);
            return acc;
          };
          const double dsn = ds * two_nu;
          for (int i = 0; i < nv; ++i)
            for (int j = 0; j <= i; ++j) {
              const double eta = tdot(i, j) + tdot(j, i) - pen * vdot<D>(vel[i], vel[j]);
              face_a[i * nv + j] -= dsn * eta;
            }
          if (case_id == kCavity && D == 2 && side == 3) {
            // lid data g = (1, 0) on y = 1 (reference case_cavity, cases.cpp:208-218)
            const double gv[2] = {1.0, 0.0};
            for (int i = 0; i < nv; ++i) {
              const double tg = tn[i][0] * gv[0] + tn[i][1] * gv[1];
              const double gvv = gv[0] * (vel[i].comp == 0 ? vel[i].v : 0.0) +
                                 gv[1] * (vel[i].comp == 1 ? vel[i].v : 0.0);
              face_f[i] += dsn * (-tg + pen * gvv);
            }
          }
        }
        // scatter (element dof map of the face element)
        std::vector<int> vids(nv);
        for (int i = 0; i < nv; ++i) {
          int idx[D];
          for (int d = 0; d < D; ++d) idx[d] = P.space(L.comp[i], d).first[ei[d]] + L.off[i][d];
          vids[i] = P.vid[L.comp[i]][P.flat(L.comp[i], idx)];
        }
        for (int i = 0; i < nv; ++i) {
          if (vids[i] < 0) continue;
          for (int j = 0; j <= i; ++j) {
            if (vids[j] < 0) continue;
            const double v = face_a[i * nv + j];
            S.A.v[slot(S.A, vids[i], vids[j])] += v;
            if (i != j) S.A.v[slot(S.A, vids[j], vids[i])] += v;
          }
        }
        if (case_id == kCavity)
          for (int i = 0; i < nv; ++i)
            if (vids[i] >= 0) S.f[vids[i]] += face_f[i];
      }
    }
  }

  S.Bt = transpose(S.B);
  S.Q_nu = S.Q;
  const double scale = 1.0 / (2.0 * nu);
  for (auto& v : S.Q_nu.v) v *= scale;
  if (case_id == kRandom) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (auto& v : S.f) v = dist(gen);
  }
  return S;
}

}  // namespace

System assemble(int dim, int k_prime, int n_elem, int case_id, double nu, uint64_t seed) {
  if (case_id != kPsiMms && case_id != kCavity && case_id != kRandom)
    throw std::invalid_argument("assemble: unknown case id");
  if (case_id == kCavity && dim != 2) throw std::invalid_argument("assemble: cavity is 2D only");
  if (!(nu > 0.0)) throw std::invalid_argument("assemble: nu must be positive");
  if (dim == 2) return assemble_dim<2>(k_prime, n_elem, case_id, nu, seed);
  if (dim == 3) return assemble_dim<3>(k_prime, n_elem, case_id, nu, seed);
  throw std::invalid_argument("assemble: dim must be 2 or 3");
}

}  // namespace dshost
