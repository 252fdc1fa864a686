// Row partition of the RCM-basis saddle operator K' across the GPUs of one
// NVLink/NVSwitch box (BASELINE north_star): every rank owns
// one contiguous range of velocity rows and one of pressure rows (each block
// balanced by its nonzeros), the vectors are partitioned the same way, and
// each rank's SpMV reads the columns it does not own -- its HALO -- from the
// owners' memory (NVLink peer loads, gathered once per SpMV into a local strip
// behind the owned entries). Dot products are sums of per-rank partials in
// rank order (a fixed order: every rank computes the same value). The IC(0)
// sweeps are replicated: every rank applies the whole factor to the whole
// (all-gathered) block residual, so the preconditioner is the single-GPU one.
#pragma once

#include <cstdint>
#include <vector>

#include "dsgpu.h"

namespace dsgpu {

struct RankPart {
  int u0 = 0, u1 = 0;  // owned velocity rows [u0, u1) of K'
  int p0 = 0, p1 = 0;  // owned pressure rows [p0, p1) (block-local: K' row n_u + p)
  int n_own() const { return (u1 - u0) + (p1 - p0); }
  // local operator: the owned rows (velocity rows first), columns renumbered:
  // owned velocity entry u -> u - u0, owned pressure entry p -> (u1 - u0) + p - p0,
  // halo entry -> n_own + its position in `halo`; entries keep their order, so a
  // row's sum is the single-GPU sum bit for bit
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  std::vector<int32_t> na;         // velocity rows: length of the A' part
  // halo: global K' columns (ascending inside each source rank's segment),
  // grouped by owner; src_ptr[s] .. src_ptr[s+1] are the entries owned by rank s
  std::vector<int32_t> halo;
  std::vector<int32_t> src_ptr;    // world + 1
  int halo_a = 0;                  // halo entries [.. per source] that the A' part needs come first in
                                   // each segment: a_cnt[s] of them
  std::vector<int32_t> a_cnt;      // world
};

struct RowPartition {
  int world = 1, n = 0, n_u = 0;
  std::vector<int32_t> ub, pb;     // world + 1 bounds of the velocity / pressure ranges
  std::vector<RankPart> rank;
  int owner_of(int col) const;     // rank owning global K' column `col`
  int local_of(int r, int col) const;  // index of an OWNED column in rank r's local vector
};

// k_rp / k_ci / k_v: K' (n rows); k_na[i]: A' entries of velocity row i (first in the row).
RowPartition partition_rows(int n, int n_u, const int64_t* k_rp, const int32_t* k_ci, const double* k_v,
                            const int32_t* k_na, int world);

}  // namespace dsgpu
