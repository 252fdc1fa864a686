// Host-side preprocessing for dsgpu_setup: builds the RCM-basis saddle
// operator, the block operators and the level-grouped triangular sweeps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>

#include "dsgpu_internal.hpp"

namespace dsgpu {
namespace {

void check_csr(const dsgpu_csr* m, int rows, int cols, const char* name) {
  if (!m || !m->row_ptr || m->n_rows != rows || m->n_cols != cols)
    throw std::invalid_argument(std::string("dsgpu_setup: bad dimensions for ") + name);
  if (m->row_ptr[0] != 0) throw std::invalid_argument(std::string(name) + ": row_ptr[0] != 0");
  for (int i = 0; i < rows; ++i)
    if (m->row_ptr[i + 1] < m->row_ptr[i])
      throw std::invalid_argument(std::string(name) + ": row_ptr not monotone");
  const int64_t nnz = m->row_ptr[rows];
  if (nnz > 0 && (!m->cols || !m->vals))
    throw std::invalid_argument(std::string(name) + ": null cols/vals");
  for (int64_t k = 0; k < nnz; ++k)
    if (m->cols[k] < 0 || m->cols[k] >= cols)
      throw std::invalid_argument(std::string(name) + ": column index out of range");
}

std::vector<int32_t> inverse(const std::vector<int32_t>& perm, int n, const char* name) {
  std::vector<int32_t> inv(n, -1);
  for (int i = 0; i < n; ++i) {
    const int p = perm[i];
    if (p < 0 || p >= n || inv[p] >= 0)
      throw std::invalid_argument(std::string(name) + ": not a permutation");
    inv[p] = i;
  }
  return inv;
}

double diag_at(const dsgpu_csr* m, int i) {
  // CsrMatrix::at (proj/src/csr.cpp:13-18): zero outside the pattern
  const int32_t* b = m->cols + m->row_ptr[i];
  const int32_t* e = m->cols + m->row_ptr[i + 1];
  const int32_t* it = std::lower_bound(b, e, i);
  return (it == e || *it != i) ? 0.0 : m->vals[it - m->cols];
}

}  // namespace

void build_sweeps(const dsgpu_csr& L, HostSweep& fwd, HostSweep& bwd) {
  const int n = L.n_rows;
  // validate: lower triangular, diagonal stored last and nonzero
  for (int i = 0; i < n; ++i) {
    const int64_t b = L.row_ptr[i], e = L.row_ptr[i + 1];
    if (e == b || L.cols[e - 1] != i)
      throw std::invalid_argument("IC(0) factor: missing diagonal at row " + std::to_string(i));
    for (int64_t k = b; k < e - 1; ++k)
      if (L.cols[k] >= i || (k > b && L.cols[k] <= L.cols[k - 1]))
        throw std::invalid_argument("IC(0) factor: not strictly lower/sorted at row " +
                                    std::to_string(i));
  }
  // backward rows: U row c = {(k, L_kc) : k > c}, k descending
  std::vector<int64_t> urp(n + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int64_t k = L.row_ptr[i]; k < L.row_ptr[i + 1] - 1; ++k) ++urp[L.cols[k] + 1];
  for (int i = 0; i < n; ++i) urp[i + 1] += urp[i];
  std::vector<int32_t> uci(urp[n]);
  std::vector<double> uv(urp[n]);
  {
    std::vector<int64_t> next(urp.begin(), urp.end() - 1);
    for (int i = n - 1; i >= 0; --i)  // descending source row
      for (int64_t k = L.row_ptr[i]; k < L.row_ptr[i + 1] - 1; ++k) {
        const int c = L.cols[k];
        uci[next[c]] = i;
        uv[next[c]] = L.vals[k];
        ++next[c];
      }
  }

  auto build = [n](HostSweep& s, const std::vector<int64_t>& rp, const int32_t* ci,
                   const double* v, const std::vector<double>& diag, bool reverse) {
    s.n = n;
    s.diag = diag;
    std::vector<int> level(n, 0);
    int max_level = -1;
    for (int t = 0; t < n; ++t) {
      const int i = reverse ? n - 1 - t : t;
      int lv = 0;
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) lv = std::max(lv, level[ci[k]] + 1);
      level[i] = lv;
      max_level = std::max(max_level, lv);
    }
    s.n_levels = max_level + 1;
    // bucket rows by level (ascending row index inside a level)
    std::vector<int> cnt(s.n_levels + 1, 0);
    for (int i = 0; i < n; ++i) ++cnt[level[i] + 1];
    for (int l = 0; l < s.n_levels; ++l) cnt[l + 1] += cnt[l];
    std::vector<int> order(n);
    {
      std::vector<int> pos(cnt.begin(), cnt.end() - 1);
      for (int i = 0; i < n; ++i) order[pos[level[i]]++] = i;
    }
    s.gptr.assign(1, 0);
    s.gwidth.clear();
    s.grows.clear();
    for (int l = 0; l < s.n_levels; ++l)
      for (int a = cnt[l]; a < cnt[l + 1]; a += kLanes) {
        const int b = std::min(cnt[l + 1], a + kLanes);
        int width = 0;
        for (int t = a; t < b; ++t)
          width = std::max<int>(width, static_cast<int>(rp[order[t] + 1] - rp[order[t]]));
        s.gwidth.push_back(width);
        for (int lane = 0; lane < kLanes; ++lane) s.grows.push_back(a + lane < b ? order[a + lane] : -1);
        s.gptr.push_back(s.gptr.back() + static_cast<int64_t>(width) * kLanes);
      }
    s.n_groups = static_cast<int>(s.gwidth.size());
    s.cols.assign(s.gptr.back(), -1);
    s.vals.assign(s.gptr.back(), 0.0);
    for (int g = 0; g < s.n_groups; ++g)
      for (int lane = 0; lane < kLanes; ++lane) {
        const int r = s.grows[static_cast<size_t>(g) * kLanes + lane];
        if (r < 0) continue;
        int kk = 0;
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k, ++kk) {
          s.cols[s.gptr[g] + static_cast<int64_t>(kk) * kLanes + lane] = ci[k];
          s.vals[s.gptr[g] + static_cast<int64_t>(kk) * kLanes + lane] = v[k];
        }
      }
  };

  std::vector<double> diag(n);
  for (int i = 0; i < n; ++i) diag[i] = L.vals[L.row_ptr[i + 1] - 1];
  // forward rows: L row i without its diagonal (columns ascending)
  std::vector<int64_t> frp(n + 1, 0);
  std::vector<int32_t> fci;
  std::vector<double> fv;
  fci.reserve(L.row_ptr[n] - n);
  fv.reserve(L.row_ptr[n] - n);
  for (int i = 0; i < n; ++i) {
    for (int64_t k = L.row_ptr[i]; k < L.row_ptr[i + 1] - 1; ++k) {
      fci.push_back(L.cols[k]);
      fv.push_back(L.vals[k]);
    }
    frp[i + 1] = static_cast<int64_t>(fci.size());
  }
  build(fwd, frp, fci.data(), fv.data(), diag, false);
  build(bwd, urp, uci.data(), uv.data(), diag, true);
}

void build_plan(HostPlan& P, const dsgpu_csr* A, const dsgpu_csr* B, const dsgpu_csr* Bt,
                const dsgpu_csr* Q_nu, int top_kind, const int32_t* perm_A, const dsgpu_csr* L_A,
                int bottom_kind, const int32_t* perm_Q, const dsgpu_csr* L_Q,
                const dsgpu_csr* Q_filter, int blocked) {
  if (!A || !B || !Bt || !Q_nu) throw std::invalid_argument("dsgpu_setup: null block");
  const int n_u = A->n_rows, n_p = Q_nu->n_rows;
  if (n_u <= 0 || n_p <= 0) throw std::invalid_argument("dsgpu_setup: empty system");
  check_csr(A, n_u, n_u, "A");
  check_csr(B, n_p, n_u, "B");
  check_csr(Bt, n_u, n_p, "Bt");
  check_csr(Q_nu, n_p, n_p, "Q_nu");
  for (int kind : {top_kind, bottom_kind})
    if (kind < DSGPU_BLOCK_JACOBI || kind > DSGPU_BLOCK_PCG_IC0)
      throw std::invalid_argument("dsgpu_setup: unknown block kind");
  P.n_u = n_u;
  P.n_p = n_p;
  P.n = n_u + n_p;

  const dsgpu_csr* mats[2] = {A, Q_nu};
  const int kinds[2] = {top_kind, bottom_kind};
  const int32_t* perms[2] = {perm_A, perm_Q};
  const dsgpu_csr* facs[2] = {L_A, L_Q};
  std::vector<int32_t> inv[2];
  for (int b = 0; b < 2; ++b) {
    HostBlock& hb = P.blk[b];
    hb.kind = kinds[b];
    hb.n = mats[b]->n_rows;
    hb.off = b == 0 ? 0 : n_u;
    if (hb.kind == DSGPU_BLOCK_PCG_IC0) {
      if (!perms[b] || !facs[b])
        throw std::invalid_argument("dsgpu_setup: IC0 block needs its permutation and factor");
      check_csr(facs[b], hb.n, hb.n, b == 0 ? "L_A" : "L_Q");
      hb.perm.assign(perms[b], perms[b] + hb.n);
    } else {
      hb.perm.resize(hb.n);
      std::iota(hb.perm.begin(), hb.perm.end(), 0);
    }
    inv[b] = inverse(hb.perm, hb.n, b == 0 ? "perm_A" : "perm_Q");
  }

  // K' rows, each part padded to a multiple of 4 entries (128-bit loads)
  auto pad4 = [](int64_t len) { return (len + 3) / 4 * 4; };
  P.k_rp.assign(P.n + 1, 0);
  P.k_na.assign(n_u, 0);
  for (int r = 0; r < n_u; ++r) {
    const int o = P.blk[0].perm[r];
    P.k_na[r] = static_cast<int32_t>(pad4(A->row_ptr[o + 1] - A->row_ptr[o]));
    P.k_rp[r + 1] = P.k_rp[r] + P.k_na[r] + pad4(Bt->row_ptr[o + 1] - Bt->row_ptr[o]);
  }
  for (int r = 0; r < n_p; ++r) {
    const int o = P.blk[1].perm[r];
    P.k_rp[n_u + r + 1] = P.k_rp[n_u + r] + pad4(B->row_ptr[o + 1] - B->row_ptr[o]);
  }
  P.nnz_a = A->row_ptr[n_u];
  P.nnz_k = A->row_ptr[n_u] + Bt->row_ptr[n_u] + B->row_ptr[n_p];
  P.nnz_q = Q_nu->row_ptr[n_p];
  P.k_ci.resize(P.k_rp[P.n]);
  P.k_v.resize(P.k_rp[P.n]);
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> row;
#pragma omp for schedule(dynamic, 256)
    for (int r = 0; r < P.n; ++r) {
      int64_t at = P.k_rp[r];
      auto emit = [&](const dsgpu_csr* m, int o, const std::vector<int32_t>& iv, int shift) {
        row.clear();
        for (int64_t k = m->row_ptr[o]; k < m->row_ptr[o + 1]; ++k)
          row.emplace_back(iv[m->cols[k]] + shift, m->vals[k]);
        std::sort(row.begin(), row.end(),
                  [](const auto& a, const auto& b) { return a.first < b.first; });
        for (const auto& e : row) {
          P.k_ci[at] = e.first;
          P.k_v[at++] = e.second;
        }
        for (; at % 4 != 0; ++at) {  // pad (row starts are multiples of 4)
          P.k_ci[at] = r;
          P.k_v[at] = 0.0;
        }
      };
      if (r < n_u) {
        const int o = P.blk[0].perm[r];
        emit(A, o, inv[0], 0);
        emit(Bt, o, inv[1], n_u);
      } else {
        emit(B, P.blk[1].perm[r - n_u], inv[0], 0);
      }
    }
  }

  for (int b = 0; b < 2; ++b) {
    HostBlock& hb = P.blk[b];
    const dsgpu_csr* m = mats[b];
    if (hb.kind != DSGPU_BLOCK_PCG_IC0) {
      // JacobiBlock / PcgBlock(jacobi): inverse diagonal, nonpositive -> domain_error
      hb.dinv.resize(hb.n);
      for (int i = 0; i < hb.n; ++i) {
        const double d = diag_at(m, i);
        if (!(d > 0.0)) throw std::domain_error("jacobi block: nonpositive diagonal");
        hb.dinv[i] = 1.0 / d;
      }
    }
    if (b == 1 && hb.kind != DSGPU_BLOCK_JACOBI) {
      // permuted Q_nu operator for the pressure PCG
      hb.rp.assign(hb.n + 1, 0);
      for (int r = 0; r < hb.n; ++r)
        hb.rp[r + 1] = hb.rp[r] + pad4(m->row_ptr[hb.perm[r] + 1] - m->row_ptr[hb.perm[r]]);
      hb.ci.resize(hb.rp[hb.n]);
      hb.v.resize(hb.rp[hb.n]);
      std::vector<std::pair<int32_t, double>> row;
      for (int r = 0; r < hb.n; ++r) {
        const int o = hb.perm[r];
        row.clear();
        for (int64_t k = m->row_ptr[o]; k < m->row_ptr[o + 1]; ++k)
          row.emplace_back(inv[b][m->cols[k]], m->vals[k]);
        std::sort(row.begin(), row.end(),
                  [](const auto& x, const auto& y) { return x.first < y.first; });
        int64_t at = hb.rp[r];
        for (const auto& e : row) {
          hb.ci[at] = e.first;
          hb.v[at++] = e.second;
        }
        for (; at < hb.rp[r + 1]; ++at) {
          hb.ci[at] = r;
          hb.v[at] = 0.0;
        }
      }
    }
    if (hb.kind == DSGPU_BLOCK_PCG_IC0 && blocked) {
      build_bsweeps(*facs[b], hb.bfwd, hb.bbwd);
    } else if (hb.kind == DSGPU_BLOCK_PCG_IC0) {
      build_sweeps(*facs[b], hb.fwd, hb.bwd);
      const dsgpu_csr* L = facs[b];
      hb.lrp.assign(L->row_ptr, L->row_ptr + hb.n + 1);
      hb.lci.assign(L->cols, L->cols + hb.lrp[hb.n]);
      hb.lv.assign(L->vals, L->vals + hb.lrp[hb.n]);
    }
  }

  P.filter = false;
  if (Q_filter) {
    check_csr(Q_filter, n_p, n_p, "Q_filter");
    // solve_stokes's zero-mean filter test (precond.cpp:266-274), kernel = 1
    double resid = 0.0, bscale = 0.0;
    for (int i = 0; i < n_u; ++i) {
      double acc = 0.0;
      for (int64_t k = Bt->row_ptr[i]; k < Bt->row_ptr[i + 1]; ++k) acc += Bt->vals[k] * 1.0;
      resid = std::max(resid, std::abs(acc));
    }
    for (int64_t k = 0; k < B->row_ptr[n_p]; ++k) bscale = std::max(bscale, std::abs(B->vals[k]));
    if (resid <= 1e-10 * bscale) {
      P.filter = true;
      std::vector<double> qk(n_p);
      double den = 0.0;
      for (int i = 0; i < n_p; ++i) {
        double acc = 0.0;
        for (int64_t k = Q_filter->row_ptr[i]; k < Q_filter->row_ptr[i + 1]; ++k)
          acc += Q_filter->vals[k] * 1.0;
        qk[i] = acc;
        den += qk[i] * 1.0;
      }
      P.qk.resize(n_p);
      for (int r = 0; r < n_p; ++r) P.qk[r] = qk[P.blk[1].perm[r]];
      P.filter_den = den;
    }
  }
}

}  // namespace dsgpu

namespace dsgpu {

// Dependency rows of a level-grouped SELL sweep.
DepRows rows_from_sweep(const HostSweep& s) {
  DepRows r;
  r.n = s.n;
  r.level.assign(s.n, 0);
  r.ent.assign(s.n, {});
  r.w.assign(s.n, {});
  r.diag = s.diag;
  for (int g = 0; g < s.n_groups; ++g)
    for (int l = 0; l < kLanes; ++l) {
      const int row = s.grows[static_cast<size_t>(g) * kLanes + l];
      if (row < 0) continue;
      for (int k = 0; k < s.gwidth[g]; ++k) {
        const int64_t at = s.gptr[g] + static_cast<int64_t>(k) * kLanes + l;
        if (s.cols[at] >= 0) r.ent[row].emplace_back(s.cols[at], s.vals[at]);
      }
    }
  // levels in dependency order (rows of a group's lanes all share a level)
  int lv = 0;
  for (int g = 0; g < s.n_groups; ++g) {
    for (int l = 0; l < kLanes; ++l) {
      const int row = s.grows[static_cast<size_t>(g) * kLanes + l];
      if (row < 0) continue;
      int v = 0;
      for (const auto& e : r.ent[row]) v = std::max(v, r.level[e.first] + 1);
      r.level[row] = v;
      lv = std::max(lv, v);
    }
  }
  return r;
}

DepRows merge_levels(const DepRows& in, int M) {
  if (M <= 1) return in;
  const int n = in.n;
  DepRows out;
  out.n = n;
  out.diag = in.diag;
  out.level.resize(n);
  for (int i = 0; i < n; ++i) out.level[i] = in.level[i] / M;
  out.ent.assign(n, {});
  out.w.assign(n, {});
  // rows in original level order, so every in-block dependency is final first
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return in.level[a] < in.level[b]; });
  std::vector<double> acc_a(n, 0.0), acc_w(n, 0.0);
  std::vector<char> has_a(n, 0), has_w(n, 0);
  std::vector<int> list_a, list_w;
  for (const int i : order) {
    const int blk = out.level[i];
    list_a.clear();
    list_w.clear();
    auto add_a = [&](int k, double v) {
      if (!has_a[k]) { has_a[k] = 1; acc_a[k] = 0.0; list_a.push_back(k); }
      acc_a[k] += v;
    };
    auto add_w = [&](int j, double v) {
      if (!has_w[j]) { has_w[j] = 1; acc_w[j] = 0.0; list_w.push_back(j); }
      acc_w[j] += v;
    };
    for (const auto& e : in.ent[i]) {
      const int j = e.first;
      if (out.level[j] == blk) {
        // substitute y_j = (b_j + sum w_jl b_l - sum a'_jk y_k) / d_j
        const double c = e.second / in.diag[j];
        add_w(j, -c);
        for (const auto& x : out.w[j]) add_w(x.first, -c * x.second);
        for (const auto& x : out.ent[j]) add_a(x.first, -c * x.second);
      } else {
        add_a(j, e.second);
      }
    }
    for (const int k : list_a) {
      out.ent[i].emplace_back(k, acc_a[k]);
      has_a[k] = 0;
    }
    for (const int j : list_w) {
      out.w[i].emplace_back(j, acc_w[j]);
      has_w[j] = 0;
    }
  }
  return out;
}

namespace {
// groups: rows of one level, <= 32 per group, ascending row index
void make_groups(const DepRows& r, std::vector<int>& gof, std::vector<int>& lof,
                 std::vector<std::vector<int>>& groups) {
  const int n = r.n;
  int L = 0;
  for (int i = 0; i < n; ++i) L = std::max(L, r.level[i] + 1);
  std::vector<std::vector<int>> by(L);
  for (int i = 0; i < n; ++i) by[r.level[i]].push_back(i);
  groups.clear();
  gof.assign(n, -1);
  lof.assign(n, -1);
  for (int l = 0; l < L; ++l)
    for (size_t a = 0; a < by[l].size(); a += kLanes) {
      groups.emplace_back();
      for (size_t t = a; t < std::min(by[l].size(), a + kLanes); ++t) {
        gof[by[l][t]] = static_cast<int>(groups.size()) - 1;
        lof[by[l][t]] = static_cast<int>(t - a);
        groups.back().push_back(by[l][t]);
      }
    }
}
}  // namespace

int flow_b_needed(const DepRows& r) {
  std::vector<int> gof, lof;
  std::vector<std::vector<int>> groups;
  make_groups(r, gof, lof, groups);
  int need = 0;
  for (int i = 0; i < r.n; ++i) {
    int c = 0;
    for (const auto& e : r.ent[i]) c += gof[e.first] >= gof[i] - 2;
    need = std::max(need, c);
  }
  return need;
}

// Staged sweep plan (see HostFlow in dsgpu_internal.hpp).
void build_flow(const DepRows& r, int tb, int ring, HostFlow& f) {
  const int n = r.n;
  f = HostFlow{};
  f.n = n;
  f.tb = tb;
  f.ring = ring;
  // smem index of an entry's x: the full vector (row) or the ring slot
  const int zero_idx = ring ? kXRing * kLanes : n;
  f.diag = r.diag;
  f.dinv.resize(n);
  for (int i = 0; i < n; ++i) f.dinv[i] = 1.0 / r.diag[i];
  std::vector<int> gof, lof;
  std::vector<std::vector<int>> groups;
  make_groups(r, gof, lof, groups);
  f.G = static_cast<int>(groups.size());
  for (int i = 0; i < n; ++i) f.n_levels = std::max(f.n_levels, r.level[i] + 1);
  f.pptr.assign(1, 0);
  f.wptr.assign(1, 0);
  f.cptr.assign(1, 0);
  f.gptr.assign(1, 0);
  f.acol.assign(static_cast<size_t>(f.G) * kTA * kLanes, 8 * zero_idx);
  f.aval.assign(f.acol.size(), 0.0);
  f.bcol.assign(static_cast<size_t>(f.G) * tb * kLanes, 8 * zero_idx);
  f.bval.assign(f.bcol.size(), 0.0);
  auto sidx = [&](int row) { return ring ? (gof[row] % kXRing) * kLanes + lof[row] : row; };
  // A window: groups g-flowd+1 .. g-3 are gathered by the co-main warp
  const int flowd = std::getenv("DSGPU_FLOWD") ? std::max(3, std::atoi(std::getenv("DSGPU_FLOWD"))) : kFlowD;
  std::vector<std::pair<int, double>> P[kLanes], A[kLanes], B[kLanes], GP[kLanes];
  for (int g = 0; g < f.G; ++g) {
    const std::vector<int>& rows = groups[g];
    const int nr = static_cast<int>(rows.size());
    int pw = 0, need = -1, ww = 0, gw = 0, gneed = -1;
    std::vector<int> cneed_g;
    for (int l = 0; l < nr; ++l) {
      P[l].clear();
      A[l].clear();
      B[l].clear();
      GP[l].clear();
      std::vector<std::pair<int, double>> e = r.ent[rows[l]];
      std::stable_sort(e.begin(), e.end(),
                       [&](const auto& a, const auto& b) { return gof[a.first] < gof[b.first]; });
      for (const auto& x : e) {
        const int dg = gof[x.first];
        if (dg >= g - 2)
          B[l].push_back(x);
        else if (dg > g - flowd)
          A[l].push_back(x);
        else
          P[l].push_back(x);
      }
      while (static_cast<int>(A[l].size()) > kTA) {  // oldest A entries go to the helpers
        P[l].push_back(A[l].front());
        A[l].erase(A[l].begin());
      }
      if (static_cast<int>(B[l].size()) > tb)
        throw std::invalid_argument("flow sweep: B capacity exceeded");
      if (ring) {  // prefix entries too old for the ring come from global memory
        std::vector<std::pair<int, double>> keep;
        for (const auto& x : P[l])
          (gof[x.first] >= g - kXRing + 2 ? keep : GP[l]).push_back(x);
        P[l].swap(keep);
        for (const auto& x : GP[l]) gneed = std::max(gneed, gof[x.first]);
        gw = std::max(gw, static_cast<int>(GP[l].size()));
      }
      for (const auto& x : P[l]) need = std::max(need, gof[x.first]);

      pw = std::max(pw, static_cast<int>(P[l].size()));
      ww = std::max(ww, static_cast<int>(r.w[rows[l]].size()));
    }
    // widths padded to whole chunks; lists lane-interleaved with stride 32 so
    // the helpers load them with constant offsets and no predicates
    // prefix widths: kPW-entry chunks then one kPL-entry last chunk
    pw = pw > 0 ? kPL + (std::max(pw - kPL, 0) + kPW - 1) / kPW * kPW : 0;
    gw = (gw + kPW - 1) / kPW * kPW;
    // prefix lists are right-aligned (padding first) so every lane's newest
    // entries share the last chunk and older chunks can go early
    for (int l = 0; l < nr; ++l) {
      const int shift = pw - static_cast<int>(P[l].size());
      for (size_t k = 0; k < P[l].size(); ++k) {  // per-chunk newest dependency
        const int pos = static_cast<int>(k) + shift;
        const size_t c = pos >= pw - kPL ? (pw - kPL) / kPW : pos / kPW;
        if (cneed_g.size() <= c) cneed_g.resize(c + 1, -1);
        cneed_g[c] = std::max(cneed_g[c], gof[P[l][k].first]);
      }
    }
    cneed_g.resize(pw > 0 ? (pw - kPL) / kPW + 1 : 0, -1);
    f.nr.push_back(nr);
    f.need.push_back(need);
    for (const int c : cneed_g) f.cneed.push_back(c);
    f.cptr.push_back(f.cptr.back() + static_cast<int32_t>(cneed_g.size()));
    f.pw.push_back(pw);
    f.ww.push_back(ww);
    f.gw.push_back(gw);
    f.gneed.push_back(gneed);
    for (int l = 0; l < kLanes; ++l) f.grows.push_back(l < nr ? rows[l] : -1);
    const int64_t pb = f.pptr.back(), wb = f.wptr.back(), gb = f.gptr.back();
    f.gcols.resize(gb + static_cast<int64_t>(gw) * kLanes, n);
    f.gvals.resize(gb + static_cast<int64_t>(gw) * kLanes, 0.0);
    f.pcols.resize(pb + static_cast<int64_t>(pw) * kLanes, 8 * zero_idx);
    f.pvals.resize(pb + static_cast<int64_t>(pw) * kLanes, 0.0);
    f.wcols.resize(wb + static_cast<int64_t>(ww) * kLanes, n);
    f.wvals.resize(wb + static_cast<int64_t>(ww) * kLanes, 0.0);
    for (int l = 0; l < nr; ++l) {
      const int64_t shift = pw - static_cast<int64_t>(P[l].size());
      for (size_t k = 0; k < P[l].size(); ++k) {
        f.pcols[pb + (static_cast<int64_t>(k) + shift) * kLanes + l] = 8 * sidx(P[l][k].first);
        f.pvals[pb + (static_cast<int64_t>(k) + shift) * kLanes + l] = P[l][k].second;
      }
      for (size_t k = 0; k < GP[l].size(); ++k) {
        f.gcols[gb + static_cast<int64_t>(k) * kLanes + l] = GP[l][k].first;
        f.gvals[gb + static_cast<int64_t>(k) * kLanes + l] = GP[l][k].second;
      }
      const auto& wl = r.w[rows[l]];
      for (size_t k = 0; k < wl.size(); ++k) {
        f.wcols[wb + static_cast<int64_t>(k) * kLanes + l] = wl[k].first;
        f.wvals[wb + static_cast<int64_t>(k) * kLanes + l] = wl[k].second;
      }
      for (size_t k = 0; k < A[l].size(); ++k) {
        const size_t at = (static_cast<size_t>(g) * kTA + k) * kLanes + l;
        f.acol[at] = 8 * sidx(A[l][k].first);
        f.aval[at] = A[l][k].second;
      }
      for (size_t k = 0; k < B[l].size(); ++k) {
        const size_t at = (static_cast<size_t>(g) * tb + k) * kLanes + l;
        f.bcol[at] = 8 * sidx(B[l][k].first);
        f.bval[at] = B[l][k].second;
      }
    }
    f.pptr.push_back(pb + static_cast<int64_t>(pw) * kLanes);
    f.wptr.push_back(wb + static_cast<int64_t>(ww) * kLanes);
    f.gptr.push_back(gb + static_cast<int64_t>(gw) * kLanes);
  }
  // pre-formatted static slot blocks (TMA bulk-copied into the ring)
  const SlotLayout lay(tb);
  f.stat.assign(static_cast<size_t>(f.G) * lay.bytes, 0);
  for (int g = 0; g < f.G; ++g) {
    uint8_t* blk = f.stat.data() + static_cast<size_t>(g) * lay.bytes;
    auto put_d = [&](int off, int idx, double v) { std::memcpy(blk + off + 8 * idx, &v, 8); };
    auto put_i = [&](int off, int idx, int32_t v) { std::memcpy(blk + off + 4 * idx, &v, 4); };
    for (int l = 0; l < kLanes; ++l) {
      const int row = f.grows[static_cast<size_t>(g) * kLanes + l];
      put_d(lay.dd, 2 * l, row >= 0 ? f.diag[row] : 1.0);
      put_d(lay.dd, 2 * l + 1, row >= 0 ? f.dinv[row] : 1.0);
      put_i(lay.rows, l, row);
      for (int k = 0; k < kTA; ++k) {
        const size_t at = (static_cast<size_t>(g) * kTA + k) * kLanes + l;
        std::memcpy(blk + lay.aval + SlotLayout::f64_at(k, l), &f.aval[at], 8);
        std::memcpy(blk + lay.acol + SlotLayout::i32_at(k, l), &f.acol[at], 4);
      }
      for (int k = 0; k < tb; ++k) {
        const size_t at = (static_cast<size_t>(g) * tb + k) * kLanes + l;
        std::memcpy(blk + lay.bval + SlotLayout::f64_at(k, l), &f.bval[at], 8);
        std::memcpy(blk + lay.bcol + SlotLayout::i32_at(k, l), &f.bcol[at], 4);
      }
    }
    put_i(lay.meta, 0, f.nr[g]);
    int nb = 0;  // B entries of the widest lane (left-aligned): the main warp skips empty 4-chunks
    for (int k = 0; k < tb; ++k)
      for (int l = 0; l < kLanes; ++l)
        if (f.bcol[(static_cast<size_t>(g) * tb + k) * kLanes + l] != 8 * zero_idx) nb = k + 1;
    put_i(lay.meta, 1, (nb + 3) / 4);
  }
}

// Diagnostics (env DSGPU_FLOW_STATS): how far ahead of the main warp the
// helpers' newest dependency lies, and the entry mix per group.
static void flow_stats(const HostFlow& f, const char* name) {
  if (!std::getenv("DSGPU_FLOW_STATS")) return;
  const int zero_idx = f.ring ? kXRing * kLanes : f.n;
  long hist[12] = {};  // last-chunk slack 0..9, >=10, none
  double sa = 0, sb = 0, sp = 0, sw = 0, sn = 0;
  for (int g = 0; g < f.G; ++g) {
    const int c1 = f.cptr[g + 1], c0 = f.cptr[g];
    const int slack = c1 > c0 ? g - f.cneed[c1 - 1] : 1 << 20;
    hist[slack < 10 ? slack : slack < (1 << 20) ? 10 : 11]++;
    int na = 0, nb = 0;
    for (int k = 0; k < kTA; ++k)
      for (int l = 0; l < kLanes; ++l)
        if (f.acol[(static_cast<size_t>(g) * kTA + k) * kLanes + l] != 8 * zero_idx) { ++na; break; }
    for (int k = 0; k < f.tb; ++k)
      for (int l = 0; l < kLanes; ++l)
        if (f.bval[(static_cast<size_t>(g) * f.tb + k) * kLanes + l] != 0.0) { ++nb; break; }

    sa += na;
    sb += nb;
    sp += f.pw[g];
    sw += f.ww[g];
    sn += f.nr[g];
  }
  const double G = f.G > 0 ? f.G : 1;
  std::fprintf(stderr,
               "[flow %s] n=%d G=%d merge=%d tb=%d ring=%d rows/group %.1f | A %.2f B %.2f P %.2f W %.2f "
               "per group | last-chunk slack 2:%ld 3:%ld 4:%ld 5:%ld 6:%ld 7:%ld 8:%ld 9:%ld >=10:%ld none:%ld\n",
               name, f.n, f.G, f.merge, f.tb, f.ring, sn / G, sa / G, sb / G, sp / G, sw / G, hist[2],
               hist[3], hist[4], hist[5], hist[6], hist[7], hist[8], hist[9], hist[10], hist[11]);
}

// Staged plans for every IC(0) block with one shared B capacity; lowers the
// merge factor until the B entries fit kTBMax. Returns the capacity used.
// Host memory: at most one DepRows (~16 B per factor entry) is alive at a
// time -- a first pass only measures the B capacity, the second rebuilds each
// direction's rows and turns them into its flow -- and each exact column-order
// sweep (only needed by DSGPU_EXACT, which does not come here) is released once
// its flow exists. At 96^3 (717M factor entries) this is the difference
// between fitting the GPU box's host memory and not.
int build_block_flows(HostPlan& P, int merge, int* merge_used, size_t smem_budget, int force_ring_n) {
  auto rows_of = [](const HostSweep& s, int M) {
    DepRows r = rows_from_sweep(s);
    if (M > 1) return merge_levels(r, M);
    return r;  // moved: no copy when M <= 1
  };
  auto release = [](HostSweep& s) {  // keep n, n_groups, n_levels
    std::vector<int64_t>().swap(s.gptr);
    std::vector<int32_t>().swap(s.gwidth);
    std::vector<int32_t>().swap(s.grows);
    std::vector<int32_t>().swap(s.cols);
    std::vector<double>().swap(s.vals);
    std::vector<double>().swap(s.diag);
  };
  for (int M = std::max(1, merge);; M = M > 1 ? M / 2 : 0) {
    if (M == 0) throw std::invalid_argument("flow sweep: dependency fan-in too large");
    int need = 1;
    for (int b = 0; b < 2 && need <= kTBMax; ++b) {
      if (P.blk[b].kind != DSGPU_BLOCK_PCG_IC0) continue;
      need = std::max(need, flow_b_needed(rows_of(P.blk[b].fwd, M)));
      if (need <= kTBMax) need = std::max(need, flow_b_needed(rows_of(P.blk[b].bwd, M)));
    }
    if (need > kTBMax) continue;
    const int tb = need <= 8 ? 8 : 16;
    // one kernel variant per handle: ring mode for all IC blocks if any block's
    // full-vector workspace (flow_smem_bytes) does not fit shared memory
    int ring = 0;
    for (int b = 0; b < 2; ++b)
      if (P.blk[b].kind == DSGPU_BLOCK_PCG_IC0 &&
          (flow_smem_bytes(P.blk[b].n, SlotLayout(tb).bytes) > smem_budget ||
           P.blk[b].n >= force_ring_n))
        ring = 1;
    for (int b = 0; b < 2; ++b) {
      if (P.blk[b].kind != DSGPU_BLOCK_PCG_IC0) continue;
      build_flow(rows_of(P.blk[b].fwd, M), tb, ring, P.blk[b].ffwd);
      release(P.blk[b].fwd);
      build_flow(rows_of(P.blk[b].bwd, M), tb, ring, P.blk[b].fbwd);
      release(P.blk[b].bwd);
      P.blk[b].ffwd.merge = P.blk[b].fbwd.merge = M;
      flow_stats(P.blk[b].ffwd, b == 0 ? "A fwd" : "Q fwd");
      flow_stats(P.blk[b].fbwd, b == 0 ? "A bwd" : "Q bwd");
    }
    if (merge_used) *merge_used = M;
    return tb;
  }
}

}  // namespace dsgpu
