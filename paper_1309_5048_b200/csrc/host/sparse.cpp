// Host sparse setup: transpose, RCM, symmetric permutation, IC(0).
//
// Same deterministic rules as the reference so the factor the GPU receives
// is the one PcgBlock would build (proj/src/precond.cpp:61-64):
//   rcm_permutation   proj/src/reorder.cpp:9-55
//   permute_symmetric proj/src/csr.cpp:113-124 (+ csr_from_triplets :88-111)
//   ic0               proj/src/cholesky.cpp:84-134
// Written for scale and in parallel (OpenMP): a level-synchronous RCM, a
// row-wise permutation without a triplet sort (a permutation creates no
// duplicates), and a dataflow-scheduled IC(0); each reproduces the reference's
// result bit for bit (tests/test_host.py) by keeping its order of operations,
// not its loop structure.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
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

// Structural symmetry without materializing a transpose: every entry (i, j)
// is looked up in row j (sorted columns), rows in parallel.
bool pattern_symmetric(const Csr& a) {
  if (a.n_rows != a.n_cols) return false;
  const int n = a.n_rows;
  int ok = 1;
#pragma omp parallel for schedule(dynamic, 1024) reduction(min : ok)
  for (int i = 0; i < n; ++i) {
    if (!ok) continue;
    for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) {
      const int j = a.ci[k];
      const int32_t* b = a.ci.data() + a.rp[j];
      const int32_t* e = a.ci.data() + a.rp[j + 1];
      if (!std::binary_search(b, e, i)) {
        ok = 0;
        break;
      }
    }
  }
  return ok != 0;
}

// Reverse Cuthill-McKee, level-synchronous. The reference walks a FIFO queue
// and appends each vertex's unvisited neighbours sorted by (degree, index)
// (proj/src/reorder.cpp:9-55); the vertex that discovers v is therefore the
// EARLIEST queue member adjacent to v. Here a whole BFS level is expanded at
// once: every frontier vertex pushes its queue position onto its unvisited
// neighbours (atomic min), the newly reached vertices are collected and sorted
// by (position of the discovering vertex, degree, index) -- the same total
// order, hence the same permutation -- with the edge scans in parallel.
// Component roots: minimum degree, lowest index among the unvisited vertices
// at or after the scan position (same rule as the reference).
std::vector<int32_t> rcm_permutation(const Csr& a) {
  if (!pattern_symmetric(a)) throw std::invalid_argument("rcm_permutation: pattern is not symmetric");
  const int n = a.n_rows;
  std::vector<int32_t> degree(n);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    const int32_t* b = a.ci.data() + a.rp[i];
    const int32_t* e = a.ci.data() + a.rp[i + 1];
    degree[i] = static_cast<int32_t>(e - b) - (std::binary_search(b, e, i) ? 1 : 0);
  }
  constexpr int32_t kFree = INT32_MAX;       // not reached yet
  std::vector<int32_t> finder(n, kFree);     // queue position of the discovering vertex; -1: placed
  std::vector<int32_t> order(n);
  int placed = 0;
  std::vector<int32_t> next;
  for (int scan = 0; scan < n; ++scan) {
    if (finder[scan] != kFree) continue;
    int root = scan;
    for (int v = scan; v < n; ++v)
      if (finder[v] == kFree && degree[v] < degree[root]) root = v;
    finder[root] = -1;
    order[placed] = root;
    int lo = placed, hi = ++placed;  // current level = order[lo, hi)
    while (lo < hi) {
      next.clear();
#pragma omp parallel
      {
        std::vector<int32_t> mine;
#pragma omp for schedule(dynamic, 64) nowait
        for (int q = lo; q < hi; ++q) {
          const int u = order[q];
          for (int64_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
            const int v = a.ci[k];
            int32_t cur = __atomic_load_n(&finder[v], __ATOMIC_RELAXED);
            while (cur > q) {  // placed vertices hold -1 and never match
              if (__atomic_compare_exchange_n(&finder[v], &cur, q, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
                if (cur == kFree) mine.push_back(v);  // first to reach v: it collects it
                break;
              }
            }
          }
        }
#pragma omp critical
        next.insert(next.end(), mine.begin(), mine.end());
      }
      std::sort(next.begin(), next.end(), [&](int32_t x, int32_t y) {
        if (finder[x] != finder[y]) return finder[x] < finder[y];
        if (degree[x] != degree[y]) return degree[x] < degree[y];
        return x < y;
      });
      lo = hi;
      for (const int32_t v : next) {
        order[placed++] = v;
        finder[v] = -1;
      }
      hi = placed;
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
    // one 64-bit key per entry: (new column << 32) | position in the old row --
    // sorting plain integers is ~2x faster than sorting (column, value) pairs
    std::vector<uint64_t> key;
#pragma omp for schedule(dynamic, 256)
    for (int r = 0; r < n; ++r) {
      const int old = perm[r];
      const int64_t k0 = a.rp[old], len = a.rp[old + 1] - k0;
      key.resize(static_cast<size_t>(len));
      for (int64_t k = 0; k < len; ++k)
        key[k] = (static_cast<uint64_t>(static_cast<uint32_t>(inv[a.ci[k0 + k]])) << 32) | static_cast<uint32_t>(k);
      std::sort(key.begin(), key.end());
      int64_t at = b.rp[r];
      for (int64_t k = 0; k < len; ++k) {
        b.ci[at] = static_cast<int32_t>(key[k] >> 32);
        double sum = 0.0;  // csr_from_triplets sums from 0.0
        sum += a.v[k0 + static_cast<uint32_t>(key[k])];
        b.v[at++] = sum;
      }
    }
  }
  return b;
}

// IC(0), dataflow-parallel and bit-identical to the reference's row-by-row
// sweep (proj/src/cholesky.cpp:84-134). Entry (i, j) is
//   L_ij = (a_ij - sum_{c < j, c in row i and row j} L_ic L_jc) / L_jj
// with the products subtracted in ascending column order -- the order in which
// the reference's sorted merge meets the common columns. Here row i's columns
// are scattered into a position map and row j is walked once, looking each of
// its columns up in the map: the same products in the same order, without the
// merge. Rows are handed out in increasing order to the threads; entry (i, j)
// waits only for row j's completion flag, so a row overlaps all of its
// predecessors except its newest dependencies (the smallest unfinished row
// always progresses: no deadlock). A nonpositive pivot marks the row; the
// smallest marked row is the reference's first failing row (every row before
// it is exact).
Csr ic0(const Csr& a) {
  if (a.n_rows != a.n_cols) throw std::invalid_argument("ic0: matrix not square");
  const int n = a.n_rows;
  Csr L;
  L.n_rows = L.n_cols = n;
  L.rp.assign(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    const int32_t* b = a.ci.data() + a.rp[i];
    const int32_t* e = a.ci.data() + a.rp[i + 1];
    L.rp[i + 1] = std::upper_bound(b, e, i) - b;  // columns <= i
  }
  for (int i = 0; i < n; ++i) L.rp[i + 1] += L.rp[i];
  L.ci.resize(L.rp[n]);
  L.v.resize(L.rp[n]);
  int missing = n;
#pragma omp parallel for schedule(static) reduction(min : missing)
  for (int i = 0; i < n; ++i) {
    const int64_t len = L.rp[i + 1] - L.rp[i];
    std::copy_n(a.ci.data() + a.rp[i], len, L.ci.data() + L.rp[i]);
    std::copy_n(a.v.data() + a.rp[i], len, L.v.data() + L.rp[i]);
    if (len == 0 || L.ci[L.rp[i + 1] - 1] != i) missing = std::min(missing, i);
  }
  // rows before the first structurally missing diagonal are factored first: a
  // breakdown there is what the reference's row-by-row loop would report
  const int n_run = missing;
  std::vector<unsigned char> done(n, 0);
  int next_row = 0, bad = n;
#pragma omp parallel
  {
    std::vector<int32_t> where(n, -1);  // column -> position in the current row
    for (;;) {
      const int i = __atomic_fetch_add(&next_row, 1, __ATOMIC_RELAXED);
      if (i >= n_run) break;
      const int64_t ib = L.rp[i], id = L.rp[i + 1] - 1;  // id: the diagonal
      for (int64_t k = ib; k < id; ++k) where[L.ci[k]] = static_cast<int32_t>(k - ib);
      for (int64_t ku = ib; ku < id; ++ku) {
        const int j = L.ci[ku];
        while (!__atomic_load_n(&done[j], __ATOMIC_ACQUIRE)) __builtin_ia32_pause();
        double s = L.v[ku];
        const int32_t upto = static_cast<int32_t>(ku - ib);  // row i's entries before column j
        const int64_t jd = L.rp[j + 1] - 1;
        for (int64_t kj = L.rp[j]; kj < jd; ++kj) {
          const int32_t m = where[L.ci[kj]];
          if (m >= 0 && m < upto) s -= L.v[ib + m] * L.v[kj];
        }
        L.v[ku] = s / L.v[jd];
      }
      double d = L.v[id];
      for (int64_t k = ib; k < id; ++k) {
        d -= L.v[k] * L.v[k];
        where[L.ci[k]] = -1;
      }
      if (!(d > 0.0)) {
        int cur = __atomic_load_n(&bad, __ATOMIC_RELAXED);
        while (i < cur && !__atomic_compare_exchange_n(&bad, &cur, i, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
        }
      }
      L.v[id] = std::sqrt(d);
      __atomic_store_n(&done[i], 1, __ATOMIC_RELEASE);
    }
  }
  if (bad < n) throw Ic0Breakdown{bad};
  if (missing < n)
    throw std::invalid_argument("ic0: structurally missing diagonal at row " + std::to_string(missing));
  return L;
}

}  // namespace dshost
