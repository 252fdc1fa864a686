// Internal plan shared by the host-side setup (setup.cpp) and the device
// solver (solver.cu). Everything lives in the RCM basis diag(P_A, P_Q).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "bsweep.hpp"
#include "dsgpu.h"

namespace dsgpu {

constexpr int kLanes = 32;  // rows per triangular-solve group (one warp)

// One triangular sweep, level-scheduled and sync-free:
//   * rows are grouped by dependency level (level(i) = 1 + max level of the
//     rows it reads); each level is cut into groups of <= 32 rows;
//   * groups are ordered by level and dealt round-robin to the warps of ONE
//     CTA; a warp spins (shared memory) only on rows of earlier levels, so no
//     CTA- or grid-wide barrier is needed between levels;
//   * group entries are stored lane-interleaved (SELL-32): entry k of lane l
//     at ptr[g] + 32 k + l, so a warp's loads are coalesced; padding cols = -1.
// The forward sweep walks L's rows with columns ascending; the backward sweep
// walks U = L^T's rows (L's columns) with the contributing rows DESCENDING,
// which is exactly the order in which the reference's column-oriented
// backward scatter subtracts them (proj/src/cholesky.cpp:145-151) -- so with
// separate mul/sub roundings the device result is bit-identical.
struct HostSweep {
  int n = 0;
  int n_groups = 0, n_levels = 0;
  std::vector<int64_t> gptr;   // n_groups + 1 (entries)
  std::vector<int32_t> gwidth; // n_groups
  std::vector<int32_t> grows;  // n_groups * 32, -1 = idle lane
  std::vector<int32_t> cols;   // SELL entries
  std::vector<double> vals;
  std::vector<double> diag;    // n
};

// Staged ("flow") sweep plan: the production triangular-solve layout.
// One CTA runs a sweep with four roles:
//   * one MAIN warp walks the groups strictly in order; for group g it
//     gathers the "B" entries (dependencies on groups g-1 and g-2) from the
//     shared-memory x workspace it wrote itself, subtracts them from the
//     co-main's partial sum and scales by the reciprocal diagonal with one
//     Markstein correction (= the correctly rounded quotient). Nothing else
//     is on its per-level chain;
//   * one CO-MAIN warp (another SM sub-partition) runs two groups behind the
//     critical path: for group g it gathers the "A" entries (dependencies on
//     groups g-D+1 .. g-3) from shared memory and hands acc_pre = psum - A to
//     the main warp;
//   * HELPER warps run further ahead: for group g they wait until the groups
//     each chunk of the row's "prefix" entries (all older dependencies)
//     depends on are done and stage psum = rhs - sum;
//   * a PRODUCER thread streams each group's static data (diagonal, A/B
//     entries) into a shared-memory ring with TMA bulk copies.
// Within a row the entries are summed in dependency-level order with tree
// reductions (reassociated w.r.t. the reference's column order: results
// agree to round-off); the factor and the operation are the
// same. kTA / TB are the per-lane capacities for A and B entries.
constexpr int kTA = 16, kRing = 16, kSRing = 8, kFlowD = 7;
// Ring mode (systems whose solution vector does not fit shared memory): the
// last kXRing groups' results live in a shared-memory ring, older ones in
// global memory (published every kFenceEvery groups after a fence).
constexpr int kXRing = 64, kFenceEvery = 8;
// remote helpers: warps sharing one group's older-than-ring list (power of 2)
constexpr int kRSplit = 4;
// Supported per-lane B capacities (templates); the plan picks the smallest that fits.
constexpr int kTBMax = 16;
constexpr int kPW = 16;  // helper prefix-list chunk (entries per lane)
constexpr int kPL = 4;   // the last (newest) chunk: small, it is summed after the final wait

// Dependency form of one triangular sweep: row i computes
//   y_i = (sum_j w_ij b_j - sum_k a_ik y_k) / d_i      (w_ii = 1 implied)
// The plain sweep has no w entries; level merging (merge_levels) adds them.
struct DepRows {
  int n = 0;
  std::vector<int> level;
  std::vector<std::vector<std::pair<int, double>>> ent;  // a_ik
  std::vector<std::vector<std::pair<int, double>>> w;    // w_ij, j != i
  std::vector<double> diag;
};

// Byte layout of one group's static data, identical in HBM (one contiguous
// block per group, copied by a TMA bulk copy) and in the shared-memory ring
// slot. Arrays are lane-interleaved in 16-byte units so the warps read them
// with 128-bit shared loads, conflict-free:
//   dd[32]{diag, dinv} | aval[kTA/2][32]{2 x f64} | bval[tb/2][32]{2 x f64} |
//   acol[kTA/4][32]{4 x i32} | bcol[tb/4][32]{4 x i32} | rows[32] i32 |
//   meta{nr, 0, 0, 0}. acol / bcol are byte offsets into the x workspace.
struct SlotLayout {
  int dd, aval, bval, acol, bcol, rows, meta, bytes;
  constexpr explicit SlotLayout(int tb)
      : dd(0), aval(512), bval(512 + 256 * kTA), acol(bval + 256 * tb), bcol(acol + 128 * kTA),
        rows(bcol + 128 * tb), meta(rows + 128), bytes(meta + 16) {}
  // byte offset of element k of lane l in a pair-interleaved f64 array / a
  // quad-interleaved i32 array
  static constexpr int f64_at(int k, int l) { return ((k >> 1) * 32 + l) * 16 + (k & 1) * 8; }
  static constexpr int i32_at(int k, int l) { return ((k >> 2) * 32 + l) * 16 + (k & 3) * 4; }
};

struct HostFlow {
  int n = 0, G = 0, n_levels = 0, tb = 4, merge = 1;
  int ring = 0;                              // 1: ring mode (see kXRing)
  std::vector<int32_t> gw, gneed;            // ring mode: global-prefix width / newest dep group
  std::vector<int64_t> gptr;                 // G + 1
  std::vector<int32_t> gcols;                // rows (pad = n, gx[n] = 0)
  std::vector<double> gvals;
  std::vector<uint8_t> stat;                 // G * SlotLayout(tb).bytes
  std::vector<int32_t> nr, need, pw, ww, grows;  // per group (grows: G*32)
  std::vector<int64_t> pptr, wptr;           // G + 1, lane-interleaved (stride 32; pw, gw in whole kPW chunks)
  std::vector<int32_t> cptr, cneed;          // per kPW-entry chunk of the prefix list: newest dep group
  std::vector<int32_t> pcols, wcols;         // pcols: byte offsets into the x workspace (pad: the zero slot); wcols: rows (pad n)
  std::vector<double> pvals, wvals;
  std::vector<int32_t> acol;                 // G*kTA*32: byte offsets into the x workspace, pad = 8n
  std::vector<double> aval;
  std::vector<int32_t> bcol;                 // G*tb*32: byte offsets into the x workspace, pad = 8n
  std::vector<double> bval;
  std::vector<double> diag, dinv;            // n
};

struct HostBlock {
  int kind = DSGPU_BLOCK_JACOBI;
  int n = 0, off = 0;
  std::vector<int32_t> perm;     // block ordering -> original index (empty = identity)
  // operator in block ordering (bottom block; the top block reads K's A part)
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  std::vector<double> dinv;      // Jacobi / Jacobi-PCG
  std::vector<int64_t> lrp;      // IC0-PCG: the factor L (block ordering), as given
  std::vector<int32_t> lci;
  std::vector<double> lv;
  HostSweep fwd, bwd;            // IC0-PCG, exact column-order sweeps (bit-identical mode)
  HostFlow ffwd, fbwd;           // IC0-PCG, staged level sweeps
  HostBSweep bfwd, bbwd;         // IC0-PCG, blocked sweeps (production, bsweep.hpp)
};

struct HostPlan {
  int n_u = 0, n_p = 0, n = 0;
  // K' = diag(P_A,P_Q) K diag(P_A,P_Q)^T: velocity rows = [A' | Bt'] (A'
  // entries first, k_na per row), pressure rows = [B'].
  // 128-bit-load layout: every row part ([A'], [Bt'], [B']) is padded to a
  // multiple of 4 entries (pad: the row's own column, value 0), so k_rp / k_na
  // count padded entries; nnz_* keep the true counts.
  std::vector<int64_t> k_rp;
  std::vector<int32_t> k_ci;
  std::vector<double> k_v;
  std::vector<int32_t> k_na;
  int64_t nnz_k = 0, nnz_a = 0, nnz_q = 0;
  HostBlock blk[2];
  bool filter = false;
  std::vector<double> qk;  // Q 1 in the pressure block ordering
  double filter_den = 0.0;
};

// Throws std::invalid_argument / std::domain_error on bad input. blocked != 0:
// the IC(0) blocks get blocked sweeps (bsweep.hpp); otherwise the level-grouped
// exact sweeps plus a copy of the factor (staged / partitioned-inverse modes).
void build_plan(HostPlan& plan, const dsgpu_csr* A, const dsgpu_csr* B, const dsgpu_csr* Bt,
                const dsgpu_csr* Q_nu, int top_kind, const int32_t* perm_A, const dsgpu_csr* L_A,
                int bottom_kind, const int32_t* perm_Q, const dsgpu_csr* L_Q,
                const dsgpu_csr* Q_filter, int blocked);

void build_sweeps(const dsgpu_csr& L, HostSweep& fwd, HostSweep& bwd);
DepRows rows_from_sweep(const HostSweep& s);
// Exact algebraic merge of M consecutive dependency levels into one:
// within each block, dependencies are substituted away (fill in a_ik, and a
// right-hand-side transform w_ij over the block's rows). Depth / M.
DepRows merge_levels(const DepRows& r, int M);
// Largest number of B entries (dependencies on groups g-1 and g-2) of any row.
int flow_b_needed(const DepRows& r);
void build_flow(const DepRows& r, int tb, int ring, HostFlow& f);
// Shared memory of one staged sweep with `slots` x entries (rows in full mode,
// kXRing*32 in ring mode); mirrors FlowSmem in solver.cu.
inline size_t flow_smem_bytes(int slots, int slot_bytes) {
  return (static_cast<size_t>(slots + 1) * 8 + 127) / 128 * 128 +
         static_cast<size_t>(kSRing) * slot_bytes + kRing * 32 * 8 + kRing * 32 * 8 + kSRing * 8 +
         (2 * kRing + 2 * kSRing) * 4 + 64;
}
// Ring mode when a full-vector workspace exceeds smem_budget (or n >= force_ring_n).
int build_block_flows(HostPlan& P, int merge, int* merge_used, size_t smem_budget, int force_ring_n);

}  // namespace dsgpu
