// Host sparse setup: transpose, RCM, symmetric permutation, IC(0).
//
// Same deterministic rules as the reference so the factor the GPU receives
// is the one PcgBlock would build (proj/src/precond.cpp:61-64):
//   rcm_permutation   proj/src/reorder.cpp:9-55
//   permute_symmetric proj/src/csr.cpp:113-124 (+ csr_from_triplets :88-111)
//   ic0               proj/src/cholesky.cpp:84-134
// Written for scale (no triplet sort: rows are permuted and sorted in place,
// which yields the same CSR since a permutation creates no duplicates).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>

#include "dshost.hpp"

namespace dshost {

Csr transpose(const Csr& a) {
  Csr t;
  t.n_rows = a.n_cols;
  t.n_cols = a.n_rows;
  t.rp.assign(static_cast<size_t>(a.n_cols) + 1, 0);
  for (const auto c : a.ci) ++t.rp[c + 1];
  for (int i = 0; i < a.n_cols; ++i) t.rp[i + 1] += t.rp[i];
  t.ci.resize(a.ci.size());
  t.v.resize(a.v.size());
  std::vector<int64_t> next(t.rp.begin(), t.rp.end() - 1);
  for (int i = 0; i < a.n_rows; ++i)
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
      const int64_t pos = next[a.ci[k]]++;
      t.ci[pos] = i;
      t.v[pos] = a.v[k];
    }
  return t;
}

bool pattern_symmetric(const Csr& a) {
  if (a.n_rows != a.n_cols) return false;
  const Csr t = transpose(a);
  return t.rp == a.rp && t.ci == a.ci;
}

std::vector<int32_t> rcm_permutation(const Csr& a) {
  if (!pattern_symmetric(a)) throw std::invalid_argument("rcm_permutation: pattern is not symmetric");
  const int n = a.n_rows;
  std::vector<int> degree(n);
  for (int i = 0; i < n; ++i) {
    int d = 0;
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (a.ci[k] != i) ++d;
    degree[i] = d;
  }
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<char> visited(n, 0);
  std::vector<int> nb;
  // Component roots: minimum degree, lowest index among the unvisited
  // vertices at or after the scan position.
  for (int scan = 0; scan < n; ++scan) {
    if (visited[scan]) continue;
    int start = scan;
    for (int v = scan; v < n; ++v)
      if (!visited[v] && degree[v] < degree[start]) start = v;
    visited[start] = 1;
    order.push_back(start);
    for (size_t head = order.size() - 1; head < order.size(); ++head) {
      const int u = order[head];
      nb.clear();
      for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
        const int v = a.ci[k];
        if (v != u && !visited[v]) {
          visited[v] = 1;
          nb.push_back(v);
        }
      }
      std::sort(nb.begin(), nb.end(), [&](int x, int y) {
        return degree[x] != degree[y] ? degree[x] < degree[y] : x < y;
      });
      order.insert(order.end(), nb.begin(), nb.end());
      if (static_cast<int>(order.size()) == n) break;
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

Csr permute_symmetric(const Csr& a, const std::vector<int32_t>& perm) {
  if (a.n_rows != a.n_cols || static_cast<int>(perm.size()) != a.n_rows)
    throw std::invalid_argument("permute_symmetric: bad inputs");
  const int n = a.n_rows;
  std::vector<int32_t> inv(n);
  for (int i = 0; i < n; ++i) inv[perm[i]] = i;
  Csr b;
  b.n_rows = b.n_cols = n;
  b.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (int r = 0; r < n; ++r) b.rp[r + 1] = b.rp[r] + (a.rp[perm[r] + 1] - a.rp[perm[r]]);
  b.ci.resize(a.ci.size());
  b.v.resize(a.v.size());
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> row;
#pragma omp for schedule(dynamic, 256)
    for (int r = 0; r < n; ++r) {
      const int old = perm[r];
      row.clear();
      for (int64_t k = a.rp[old]; k < a.rp[old + 1]; ++k) row.emplace_back(inv[a.ci[k]], a.v[k]);
      std::sort(row.begin(), row.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      int64_t at = b.rp[r];
      for (const auto& e : row) {
        b.ci[at] = e.first;
        double sum = 0.0;  // csr_from_triplets sums from 0.0
        sum += e.second;
        b.v[at++] = sum;
      }
    }
  }
  return b;
}

Csr ic0(const Csr& a) {
  if (a.n_rows != a.n_cols) throw std::invalid_argument("ic0: matrix not square");
  const int n = a.n_rows;
  Csr L;
  L.n_rows = L.n_cols = n;
  L.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
      if (a.ci[k] <= i) ++L.rp[i + 1];
  for (int i = 0; i < n; ++i) L.rp[i + 1] += L.rp[i];
  L.ci.resize(L.rp[n]);
  L.v.resize(L.rp[n]);
  {
    int64_t pos = 0;
    for (int i = 0; i < n; ++i)
      for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k)
        if (a.ci[k] <= i) {
          L.ci[pos] = a.ci[k];
          L.v[pos] = a.v[k];
          ++pos;
        }
  }
  for (int i = 0; i < n; ++i) {
    const int64_t ib = L.rp[i], ie = L.rp[i + 1];
    if (ie == ib || L.ci[ie - 1] != i)
      throw std::invalid_argument("ic0: structurally missing diagonal at row " + std::to_string(i));
    for (int64_t ku = ib; ku < ie - 1; ++ku) {
      const int j = L.ci[ku];
      // sparse dot of rows i and j below column j (sorted merge)
      double s = L.v[ku];
      int64_t pi = ib, pj = L.rp[j];
      const int64_t je = L.rp[j + 1] - 1;
      while (pi < ku && pj < je) {
        if (L.ci[pi] == L.ci[pj])
          s -= L.v[pi++] * L.v[pj++];
        else if (L.ci[pi] < L.ci[pj])
          ++pi;
        else
          ++pj;
      }
      L.v[ku] = s / L.v[je];
    }
    double d = L.v[ie - 1];
    for (int64_t k = ib; k < ie - 1; ++k) d -= L.v[k] * L.v[k];
    if (!(d > 0.0)) throw Ic0Breakdown{i};
    L.v[ie - 1] = std::sqrt(d);
  }
  return L;
}

}  // namespace dshost
