// Host planner of the multi-GPU row partition (partition.hpp).
#include "partition.hpp"

#include <algorithm>
#include <stdexcept>

namespace dsgpu {

namespace {
// world + 1 bounds of [0, rows) with equal shares of cost(i) = nnz of row (+ vector work)
std::vector<int32_t> balanced_bounds(int rows, int world, const int64_t* rp, int row0) {
  std::vector<int32_t> b(world + 1, rows);
  b[0] = 0;
  const double base = static_cast<double>(rp[row0]);
  const double total = static_cast<double>(rp[row0 + rows]) - base + 24.0 * rows;
  int c = 1;
  for (int i = 0; i < rows && c < world; ++i) {
    const double done = static_cast<double>(rp[row0 + i + 1]) - base + 24.0 * (i + 1);
    while (c < world && done >= total * c / world) b[c++] = i + 1;
  }
  return b;
}
}  // namespace

int RowPartition::owner_of(int col) const {
  const std::vector<int32_t>& b = col < n_u ? ub : pb;
  const int c = col < n_u ? col : col - n_u;
  return static_cast<int>(std::upper_bound(b.begin() + 1, b.end(), c) - b.begin()) - 1;
}

int RowPartition::local_of(int r, int col) const {
  const RankPart& P = rank[r];
  return col < n_u ? col - P.u0 : (P.u1 - P.u0) + (col - n_u) - P.p0;
}

RowPartition partition_rows(int n, int n_u, const int64_t* k_rp, const int32_t* k_ci, const double* k_v,
                            const int32_t* k_na, int world) {
  if (world < 1 || n_u < 0 || n_u > n) throw std::invalid_argument("partition_rows: bad arguments");
  RowPartition R;
  R.world = world;
  R.n = n;
  R.n_u = n_u;
  R.ub = balanced_bounds(n_u, world, k_rp, 0);
  R.pb = balanced_bounds(n - n_u, world, k_rp, n_u);
  R.rank.resize(world);
#pragma omp parallel for schedule(static, 1)
  for (int r = 0; r < world; ++r) {
    RankPart& P = R.rank[r];
    P.u0 = R.ub[r];
    P.u1 = R.ub[r + 1];
    P.p0 = R.pb[r];
    P.p1 = R.pb[r + 1];
    const int nown = P.n_own();
    auto owned = [&](int c) { return c < n_u ? (c >= P.u0 && c < P.u1) : (c - n_u >= P.p0 && c - n_u < P.p1); };
    // halo columns: those of the A' parts first (per source), then the rest
    std::vector<int32_t> ha, hk;
    auto rows_do = [&](auto&& f) {
      for (int i = P.u0; i < P.u1; ++i) f(i);
      for (int i = n_u + P.p0; i < n_u + P.p1; ++i) f(i);
    };
    rows_do([&](int i) {
      const int64_t s = k_rp[i], e = k_rp[i + 1];
      const int64_t a_end = i < n_u ? s + k_na[i] : s;
      for (int64_t k = s; k < e; ++k)
        if (!owned(k_ci[k])) (k < a_end ? ha : hk).push_back(k_ci[k]);
    });
    auto uniq = [](std::vector<int32_t>& v) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    };
    uniq(ha);
    uniq(hk);
    {  // hk := hk \ ha
      std::vector<int32_t> d;
      std::set_difference(hk.begin(), hk.end(), ha.begin(), ha.end(), std::back_inserter(d));
      hk.swap(d);
    }
    P.src_ptr.assign(world + 1, 0);
    P.a_cnt.assign(world, 0);
    std::vector<std::vector<int32_t>> seg_a(world), seg_k(world);
    for (const int32_t c : ha) seg_a[R.owner_of(c)].push_back(c);
    for (const int32_t c : hk) seg_k[R.owner_of(c)].push_back(c);
    for (int s = 0; s < world; ++s) {
      P.a_cnt[s] = static_cast<int32_t>(seg_a[s].size());
      P.halo.insert(P.halo.end(), seg_a[s].begin(), seg_a[s].end());
      P.halo.insert(P.halo.end(), seg_k[s].begin(), seg_k[s].end());
      P.src_ptr[s + 1] = static_cast<int32_t>(P.halo.size());
    }
    P.halo_a = static_cast<int>(ha.size());
    // global column -> local index
    std::vector<std::pair<int32_t, int32_t>> hmap(P.halo.size());
    for (size_t k = 0; k < P.halo.size(); ++k) hmap[k] = {P.halo[k], static_cast<int32_t>(nown + k)};
    std::sort(hmap.begin(), hmap.end());
    auto local = [&](int c) {
      if (owned(c)) return R.local_of(r, c);
      const auto it = std::lower_bound(hmap.begin(), hmap.end(), std::make_pair(static_cast<int32_t>(c), INT32_MIN));
      return static_cast<int>(it->second);
    };
    P.rp.assign(1, 0);
    rows_do([&](int i) {
      for (int64_t k = k_rp[i]; k < k_rp[i + 1]; ++k) {
        P.ci.push_back(local(k_ci[k]));
        P.v.push_back(k_v[k]);
      }
      P.rp.push_back(static_cast<int64_t>(P.ci.size()));
      if (i < n_u) P.na.push_back(k_na[i]);
    });
  }
  return R;
}

}  // namespace dsgpu

// Test hook (host only): partitions a square operator (n rows, the first n_u of
// them "velocity" rows whose first na[i] entries are the A part; na may be
// NULL = whole row) over `world` ranks and evaluates y = K x the way the ranks
// would: each rank gathers its halo from the owners' slices, multiplies its
// local rows, and writes its slice of y. bounds: 2 (world + 1) ints (velocity
// bounds, pressure bounds); halo_counts: world x world (row r: entries rank r
// reads from each source).
extern "C" int dsgpu_debug_partition_spmv(int n, int n_u, const int64_t* rp, const int32_t* ci, const double* v,
                                          const int32_t* na, int world, int32_t* bounds, int64_t* halo_counts,
                                          const double* x, double* y) {
  try {
    std::vector<int32_t> na_full;
    if (!na) {
      na_full.resize(n_u);
      for (int i = 0; i < n_u; ++i) na_full[i] = static_cast<int32_t>(rp[i + 1] - rp[i]);
      na = na_full.data();
    }
    const dsgpu::RowPartition R = dsgpu::partition_rows(n, n_u, rp, ci, v, na, world);
    for (int r = 0; r <= world; ++r) {
      bounds[r] = R.ub[r];
      bounds[world + 1 + r] = R.pb[r];
    }
    // every rank's owned slice of x (what lives in its HBM)
    std::vector<std::vector<double>> own(world);
    for (int r = 0; r < world; ++r) {
      const dsgpu::RankPart& P = R.rank[r];
      own[r].resize(P.n_own());
      for (int i = P.u0; i < P.u1; ++i) own[r][i - P.u0] = x[i];
      for (int i = P.p0; i < P.p1; ++i) own[r][(P.u1 - P.u0) + i - P.p0] = x[n_u + i];
    }
    for (int r = 0; r < world; ++r) {
      const dsgpu::RankPart& P = R.rank[r];
      std::vector<double> loc(own[r]);
      loc.resize(P.n_own() + P.halo.size());
      for (int s = 0; s < world; ++s) {
        halo_counts[static_cast<size_t>(r) * world + s] = P.src_ptr[s + 1] - P.src_ptr[s];
        for (int k = P.src_ptr[s]; k < P.src_ptr[s + 1]; ++k)  // the peer read
          loc[P.n_own() + k] = own[s][R.local_of(s, P.halo[k])];
      }
      int row = 0;
      auto out = [&](int gi) {
        double acc = 0.0;
        for (int64_t k = P.rp[row]; k < P.rp[row + 1]; ++k) acc += P.v[k] * loc[P.ci[k]];
        y[gi] = acc;
        ++row;
      };
      for (int i = P.u0; i < P.u1; ++i) out(i);
      for (int i = P.p0; i < P.p1; ++i) out(n_u + i);
    }
    return DSGPU_OK;
  } catch (const std::exception&) {
    return DSGPU_E_BAD_INPUT;
  }
}
