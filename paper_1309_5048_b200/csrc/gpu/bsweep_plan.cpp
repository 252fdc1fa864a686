// Host-side plan of the blocked triangular sweeps (bsweep.hpp): dense
// 16 x 16 blocks next to the diagonal, lane-interleaved sparse lists for the
// rest. Parallel over groups (OpenMP); two passes (widths, then fill).
#include "bsweep.hpp"

#include <omp.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

namespace dsgpu {
namespace {

using Ent = std::pair<int32_t, double>;  // (sweep-order column, value)

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// rows(p, ent, diag): strictly-lower entries of sweep row p with their
// sweep-order columns ASCENDING (oldest dependency first), and the diagonal.
template <class RowFn>
void build_dir(int n, int dir, RowFn rows, HostBSweep& s) {
  const int G = (n + kBsB - 1) / kBsB;
  s = HostBSweep{};
  s.n = n;
  s.G = G;
  s.dir = dir;
  s.mw.assign(G, 0);
  s.ms.assign(G, 0);
  s.fw.assign(G, 0);
  // ---- pass 1: list widths -------------------------------------------------
#pragma omp parallel
  {
    std::vector<Ent> ent;
#pragma omp for schedule(dynamic, 64)
    for (int g = 0; g < G; ++g) {
      int wm = 0, wf = 0;
      for (int r = 0; r < kBsB; ++r) {
        const int p = g * kBsB + r;
        if (p >= n) break;
        double d;
        rows(p, ent, d);
        int cm = 0, cf = 0;
        for (const Ent& e : ent) {
          const int dg = g - e.first / kBsB;
          if (dg > kBsR)
            ++cf;
          else if (dg > kBsK)
            ++cm;
        }
        wm = std::max(wm, (cm + 1) / 2);
        wf = std::max(wf, (cf + 1) / 2);
      }
      s.mw[g] = round_up(wm, kBsMC);
      s.fw[g] = round_up(wf, kBsFC);
    }
  }
  s.mptr.assign(G + 1, 0);
  s.fptr.assign(G + 1, 0);
  s.fcptr.assign(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    s.mptr[g + 1] = s.mptr[g] + static_cast<int64_t>(s.mw[g]) * 32;
    s.fptr[g + 1] = s.fptr[g] + static_cast<int64_t>(s.fw[g]) * 32;
    s.fcptr[g + 1] = s.fcptr[g] + s.fw[g] / kBsFC;
  }
  s.mcols.assign(s.mptr[G], kBsZero);
  s.mvals.assign(s.mptr[G], 0.0);
  s.fcols.assign(s.fptr[G], n);
  s.fvals.assign(s.fptr[G], 0.0);
  s.fneed.assign(s.fcptr[G], -1);
  s.slots.assign(static_cast<size_t>(G + kBsK + 1) * kBsSlotBytes, 0);
  s.tblk.assign(static_cast<size_t>(G) * kBsBlock, 0);
  int64_t nd = 0, nm = 0, nf = 0;
  // ---- pass 2: fill ----------------------------------------------------------
#pragma omp parallel reduction(+ : nd, nm, nf)
  {
    std::vector<Ent> ent, mid, far;
    std::vector<int> mneed;
#pragma omp for schedule(dynamic, 64)
    for (int g = 0; g < G; ++g) {
      long double D[kBsB][kBsB] = {};
      long double E[kBsK][kBsB][kBsB] = {};
      const int wm = s.mw[g], wf = s.fw[g];
      int32_t* mc = s.mcols.data() + s.mptr[g];
      double* mv = s.mvals.data() + s.mptr[g];
      int32_t* fc = s.fcols.data() + s.fptr[g];
      double* fv = s.fvals.data() + s.fptr[g];
      int32_t* fneed = s.fneed.data() + s.fcptr[g];
      mneed.assign(wm / kBsMC, -1);
      for (int r = 0; r < kBsB; ++r) {
        const int p = g * kBsB + r;
        if (p >= n) {
          D[r][r] = 1.0L;  // padding row: y = 0
          continue;
        }
        double d;
        rows(p, ent, d);
        D[r][r] = d;
        mid.clear();
        far.clear();
        for (const Ent& e : ent) {
          const int gq = e.first / kBsB, c = e.first % kBsB, dg = g - gq;
          if (dg == 0)
            D[r][c] = e.second;
          else if (dg <= kBsK)
            E[dg - 1][r][c] = e.second;
          else if (dg <= kBsR)
            mid.push_back(e);
          else
            far.push_back(e);
        }
        nd += static_cast<int64_t>(ent.size()) - static_cast<int64_t>(mid.size() + far.size());
        nm += static_cast<int64_t>(mid.size());
        nf += static_cast<int64_t>(far.size());
        // a row's list is dealt alternately to its two lanes (r, r + 16), each
        // lane's entries oldest first and RIGHT-aligned in the group's width,
        // so the newest dependencies of all lanes share the last chunks
        for (int h = 0; h < 2; ++h) {
          const int lane = r + 16 * h;
          const int lm = (static_cast<int>(mid.size()) + 1 - h) / 2;
          for (int k = 0; k < lm; ++k) {
            const Ent& e = mid[2 * k + h];
            const int pos = wm - lm + k;
            const int gq = e.first / kBsB, c = e.first % kBsB;
            mc[bs_i32_at(pos, lane)] = ((gq % kBsR) * kBsB + c) * 8;
            mv[bs_f64_at(pos, lane)] = e.second;
            mneed[pos / kBsMC] = std::max(mneed[pos / kBsMC], gq);
          }
          const int lf = (static_cast<int>(far.size()) + 1 - h) / 2;
          for (int k = 0; k < lf; ++k) {
            const Ent& e = far[2 * k + h];
            const int pos = wf - lf + k;
            fc[bs_i32_at(pos, lane)] = dir ? n - 1 - e.first : e.first;
            fv[bs_f64_at(pos, lane)] = e.second;
            fneed[pos / kBsFC] = std::max(fneed[pos / kBsFC], e.first / kBsB);
          }
        }
      }
      // far padding gathers a real, already published entry (times 0): the
      // group's oldest far column, which every lane's first chunk waits for anyway
      if (wf > 0) {
        int32_t oldest = INT32_MAX;
        for (int r = 0; r < kBsB; ++r) {
          const int p = g * kBsB + r;
          if (p >= n) break;
          double d;
          rows(p, ent, d);
          if (!ent.empty() && g - ent.front().first / kBsB > kBsR) oldest = std::min(oldest, ent.front().first);
        }
        const int32_t pad = dir ? n - 1 - oldest : oldest;
        for (int lane = 0; lane < 32; ++lane)
          for (int k = 0; k < wf; ++k)
            if (fv[bs_f64_at(k, lane)] == 0.0 && fc[bs_i32_at(k, lane)] == n) fc[bs_i32_at(k, lane)] = pad;
      }
      // leading mid chunks that are computable two groups early
      int early = 0;
      while (early < wm / kBsMC && mneed[early] <= g - kBsK - 3) ++early;
      s.ms[g] = early * kBsMC;
      // T = D^{-1} (forward substitution, long double), F_k = T E_k
      long double T[kBsB][kBsB] = {};
      for (int c = 0; c < kBsB; ++c)
        for (int r = c; r < kBsB; ++r) {
          long double acc = r == c ? 1.0L : 0.0L;
          for (int m = c; m < r; ++m) acc -= D[r][m] * T[m][c];
          T[r][c] = acc / D[r][r];
        }
      uint8_t* slot = s.slots.data() + static_cast<size_t>(g) * kBsSlotBytes;
      uint8_t* tb = s.tblk.data() + static_cast<size_t>(g) * kBsBlock;
      auto put = [&](int block, int r, int c, long double v) {  // block kBsK: T (its own array)
        const int lane = r + 16 * (c >> 3), q = (c & 7) >> 1;
        const double dv = static_cast<double>(v);
        uint8_t* base = block == kBsK ? tb : slot + static_cast<size_t>(block) * kBsBlock;
        std::memcpy(base + ((q * 32) + lane) * 16 + (c & 1) * 8, &dv, 8);
      };
      for (int k = 0; k < kBsK; ++k)
        for (int r = 0; r < kBsB; ++r)
          for (int c = 0; c < kBsB; ++c) {
            long double acc = 0.0L;
            for (int m = 0; m <= r; ++m) acc += T[r][m] * E[k][m][c];
            put(k, r, c, acc);
          }
      for (int r = 0; r < kBsB; ++r)
        for (int c = 0; c < kBsB; ++c) put(kBsK, r, c, T[r][c]);
    }
  }
  s.nnz_dense = nd;
  s.nnz_mid = nm;
  s.nnz_far = nf;
}

}  // namespace

void build_bsweeps(const dsgpu_csr& L, HostBSweep& fwd, HostBSweep& bwd) {
  const int n = L.n_rows;
  if (n <= 0 || L.n_cols != n || !L.row_ptr || !L.cols || !L.vals)
    throw std::invalid_argument("IC(0) factor: bad dimensions");
  int64_t bad = -1;
  int bw = 0;
#pragma omp parallel for reduction(max : bad, bw) schedule(static)
  for (int i = 0; i < n; ++i) {
    const int64_t b = L.row_ptr[i], e = L.row_ptr[i + 1];
    if (e <= b || L.cols[e - 1] != i || !(L.vals[e - 1] != 0.0)) {
      bad = std::max<int64_t>(bad, i);
      continue;
    }
    for (int64_t k = b; k < e - 1; ++k)
      if (L.cols[k] < 0 || L.cols[k] >= i || (k > b && L.cols[k] <= L.cols[k - 1])) bad = std::max<int64_t>(bad, i);
    if (e - 1 > b) bw = std::max(bw, i - L.cols[b]);
  }
  if (bad >= 0)
    throw std::invalid_argument("IC(0) factor: row " + std::to_string(bad) +
                                " is not strictly lower / sorted with a nonzero diagonal last");
  build_dir(
      n, 0,
      [&](int p, std::vector<Ent>& ent, double& diag) {
        const int64_t b = L.row_ptr[p], e = L.row_ptr[p + 1] - 1;
        ent.resize(static_cast<size_t>(e - b));
        for (int64_t k = b; k < e; ++k) ent[k - b] = Ent(L.cols[k], L.vals[k]);
        diag = L.vals[e];
      },
      fwd);
  // L^T by columns (strictly lower part of L, rows ascending inside a column).
  // L is banded (row i reaches back at most bw columns), so the thread that
  // owns columns [c0, c1) only scans rows [c0, c1 + bw).
  std::vector<int64_t> crp(static_cast<size_t>(n) + 1, 0);
  const int T = omp_get_max_threads();
  auto scan = [&](int c0, int c1, auto&& visit) {
    const int r1 = static_cast<int>(std::min<int64_t>(n, static_cast<int64_t>(c1) + bw));
    for (int i = c0; i < r1; ++i) {
      const int32_t* b = L.cols + L.row_ptr[i];
      const int32_t* e = L.cols + L.row_ptr[i + 1] - 1;
      const int32_t* lo = std::lower_bound(b, e, c0);
      const int32_t* hi = std::lower_bound(lo, e, c1);
      for (const int32_t* q = lo; q < hi; ++q) visit(*q, i, L.vals[q - L.cols]);
    }
  };
#pragma omp parallel for schedule(static, 1)
  for (int t = 0; t < T; ++t) {
    const int c0 = static_cast<int>(static_cast<int64_t>(n) * t / T);
    const int c1 = static_cast<int>(static_cast<int64_t>(n) * (t + 1) / T);
    scan(c0, c1, [&](int c, int, double) { ++crp[c + 1]; });
  }
  for (int c = 0; c < n; ++c) crp[c + 1] += crp[c];
  std::vector<int32_t> crow(static_cast<size_t>(crp[n]));
  std::vector<double> cval(static_cast<size_t>(crp[n]));
#pragma omp parallel for schedule(static, 1)
  for (int t = 0; t < T; ++t) {
    const int c0 = static_cast<int>(static_cast<int64_t>(n) * t / T);
    const int c1 = static_cast<int>(static_cast<int64_t>(n) * (t + 1) / T);
    std::vector<int64_t> next(crp.begin() + c0, crp.begin() + c1);
    scan(c0, c1, [&](int c, int i, double v) {
      const int64_t at = next[c - c0]++;
      crow[at] = i;
      cval[at] = v;
    });
  }
  build_dir(
      n, 1,
      [&](int p, std::vector<Ent>& ent, double& diag) {
        const int i = n - 1 - p;  // factor column i = row i of L^T
        const int64_t b = crp[i], e = crp[i + 1];
        ent.resize(static_cast<size_t>(e - b));
        for (int64_t k = e - 1; k >= b; --k) ent[e - 1 - k] = Ent(n - 1 - crow[k], cval[k]);
        diag = L.vals[L.row_ptr[i + 1] - 1];
      },
      bwd);
}

void bsweep_host_apply(const HostBSweep& s, const double* rhs, double* x) {
  const int n = s.n;
  auto orig = [&](int p) { return s.dir ? n - 1 - p : p; };
  std::vector<double> y(static_cast<size_t>(s.G + 1) * kBsB, 0.0);  // sweep order
  auto blk = [&](int g, int block, int r, int c) {
    const int lane = r + 16 * (c >> 3), q = (c & 7) >> 1;
    double v;
    const uint8_t* base = block == kBsK ? s.tblk.data() + static_cast<size_t>(g) * kBsBlock
                                        : s.slots.data() + static_cast<size_t>(g) * kBsSlotBytes +
                                              static_cast<size_t>(block) * kBsBlock;
    std::memcpy(&v, base + ((q * 32) + lane) * 16 + (c & 1) * 8, 8);
    return v;
  };
  for (int g = 0; g < s.G; ++g) {
    double t[kBsB];
    for (int r = 0; r < kBsB; ++r) {
      const int p = g * kBsB + r;
      double part[2];
      for (int h = 0; h < 2; ++h) {
        const int lane = r + 16 * h;
        double acc = (h == 0 && p < n) ? rhs[orig(p)] : 0.0;
        for (int k = 0; k < s.fw[g]; ++k) {
          const int32_t c = s.fcols[s.fptr[g] + bs_i32_at(k, lane)];
          if (c < n) acc -= s.fvals[s.fptr[g] + bs_f64_at(k, lane)] * x[c];
        }
        for (int k = 0; k < s.mw[g]; ++k) {
          const int32_t off = s.mcols[s.mptr[g] + bs_i32_at(k, lane)];
          if (off == kBsZero) continue;
          const int slot = off / 8 / kBsB, c = off / 8 % kBsB;
          int back = ((g - slot) % kBsR + kBsR) % kBsR;
          if (back == 0) back = kBsR;
          acc -= s.mvals[s.mptr[g] + bs_f64_at(k, lane)] * y[static_cast<size_t>(g - back) * kBsB + c];
        }
        part[h] = acc;
      }
      t[r] = part[0] + part[1];
    }
    for (int r = 0; r < kBsB; ++r) {
      double c = 0.0;
      for (int m = 0; m < kBsB; ++m) c += blk(g, kBsK, r, m) * t[m];
      double acc = 0.0;
      for (int k = 1; k <= kBsK && k <= g; ++k)
        for (int m = 0; m < kBsB; ++m) acc += blk(g, k - 1, r, m) * y[static_cast<size_t>(g - k) * kBsB + m];
      const double v = c - acc;
      y[static_cast<size_t>(g) * kBsB + r] = v;
      const int p = g * kBsB + r;
      if (p < n) x[orig(p)] = v;
    }
  }
}

}  // namespace dsgpu

// Test hook (no device involved): the blocked-sweep PLAN of the factor L
// evaluated on the host, z = (L L^T)^{-1} r, so the plan's structure and
// coefficients can be checked against the plain substitution without a GPU.
// stats8: G, factor entries in dense blocks / mid lists / far lists of the
// forward sweep, widest mid list, widest far list, padded mid, padded far entries.
extern "C" int dsgpu_debug_bsweep_host(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                                       const double* r, double* z, int64_t* stats8) {
  try {
    dsgpu_csr L{n, n, row_ptr, cols, vals};
    dsgpu::HostBSweep f, b;
    dsgpu::build_bsweeps(L, f, b);
    std::vector<double> y(static_cast<size_t>(n) + 1, 0.0), zz(static_cast<size_t>(n) + 1, 0.0);
    dsgpu::bsweep_host_apply(f, r, y.data());
    dsgpu::bsweep_host_apply(b, y.data(), zz.data());
    std::memcpy(z, zz.data(), sizeof(double) * n);
    if (stats8) {
      stats8[0] = f.G;
      stats8[1] = f.nnz_dense;
      stats8[2] = f.nnz_mid;
      stats8[3] = f.nnz_far;
      stats8[4] = *std::max_element(f.mw.begin(), f.mw.end());
      stats8[5] = *std::max_element(f.fw.begin(), f.fw.end());
      stats8[6] = f.mptr.back();
      stats8[7] = f.fptr.back();
    }
    return DSGPU_OK;
  } catch (const std::exception&) {
    return DSGPU_E_BAD_INPUT;
  }
}
