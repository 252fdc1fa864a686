// Blocked triangular sweep ("block sweep"): the production form of the IC(0)
// forward / backward solves (reference Ic0Factor::solve,
// proj/src/cholesky.cpp:136-152) on B200.
//
// The rows of the (RCM-ordered) factor are cut into groups of kBsB = 16
// CONSECUTIVE rows (not dependency levels). With D_g the 16 x 16 diagonal
// block of group g and E_{g,h} its coupling to group h < g,
//
//   y_g = D_g^{-1} ( r_g - sum_{h<g} E_{g,h} y_h )
//       = T_g ( r_g - sum_{h < g-K} E_{g,h} y_h )  -  sum_{k=1..K} F_{g,k} y_{g-k},
//
// T_g = D_g^{-1} and F_{g,k} = D_g^{-1} E_{g,g-k} formed once at setup as
// DENSE 16 x 16 blocks (the factor is quasi-dense next to its diagonal: at
// 32^3 a row has 12 of its 235 entries within the previous 32 rows). The
// sequential chain is then one dense 16 x 16 product per group, done by ONE
// warp out of shared memory, instead of one step per dependency level
// (32^3: 7,153 groups vs 10,715 levels of 10.7 rows).
//
// Roles (per triangular solve one "sweep CTA", or -- the production form -- a
// CTA PAIR of a 2-CTA cluster: a chain CTA with the main / second main /
// producer / publisher warps and a list CTA with the co-mains and a relay warp,
// exchanging y_g and c_g as tagged units through distributed shared memory;
// plus far-worker CTAs):
//   * MAIN warp: y_g = c_g - q_g - F_{g,1} y_{g-1} - F_{g,2} y_{g-2}; lane (r, h)
//     owns row r and columns 8h..8h+7 of each block (two lanes per row, combined
//     by one shuffle). y_{g-1} is broadcast through the shared-memory y ring.
//   * SECOND MAIN warp: q_g = sum_{k=3..K} F_{g,k} y_{g-k}, accumulated as the
//     y's appear (two steps of slack before the main warp needs q_g).
//   * CO-MAIN warps (kBsNC, round-robin over groups): c_g = T_g (r_g - far_g
//     - mid_g): the "mid" entries (groups g-R .. g-K-1) are gathered from the y
//     ring; the "far" partial sums come from the far workers. Each co-main
//     stages its NEXT group's mid list in shared memory with cp.async while it
//     works on the current one, so the lists' HBM latency is off its path.
//   * PRODUCER lane: TMA bulk copies of each group's dense blocks (F_1..F_K)
//     into a shared-memory slot ring.
//   * PUBLISHER warp: copies finished groups from the y ring to the result
//     vector in global memory (plain, and as tagged units for the far workers),
//     so the main warp never touches global memory.
//   * FAR WORKERS (warps of other CTAs): for each group the partial sums of
//     the entries older than the ring (col group < g-R), gathered from the
//     published result vector; they run far ahead of the main warp and stream
//     ~85 % of the factor at HBM/L2 speed on as many SMs as needed.
// The backward solve is the same sweep on the reversed ordering (row p of the
// sweep = row n-1-p of the factor; L^T's rows are L's columns).
//
// Arithmetic: T_g and F_{g,k} are formed in long double and rounded once; the
// sweep itself is fp64. The result is the same operator (L L^T)^{-1} applied
// with a different association (measured agreement with the reference's
// Ic0Factor::solve: see tests/test_gpu_parity.py); the exact column-order
// sweep stays available behind DSGPU_EXACT=1.
#pragma once

#include <cstdint>
#include <vector>

#include "dsgpu.h"

// Tuning constants (overridable at build time for A/B runs: make EXTRA_DEFS=-DDSGPU_BS_K=4 ...)
#ifndef DSGPU_BS_K
#define DSGPU_BS_K 6
#endif
#ifndef DSGPU_BS_R
#define DSGPU_BS_R 32
#endif
#ifndef DSGPU_BS_NC
#define DSGPU_BS_NC 8
#endif
#ifndef DSGPU_BS_STAGE
#define DSGPU_BS_STAGE 16
#endif
#ifndef DSGPU_BS_NC2
#define DSGPU_BS_NC2 12
#endif

namespace dsgpu {

constexpr int kBsB = 16;     // rows per group
constexpr int kBsK = DSGPU_BS_K;      // dense pre-multiplied coupling blocks: F_1, F_2 on the main warp,
                             //   F_3..F_K on the second main warp
constexpr int kBsRQ = 8;     // q ring (second main warp -> main), groups (power of two)
constexpr int kBsR = DSGPU_BS_R;     // y ring depth in groups; older entries are "far"
constexpr int kBsNC = DSGPU_BS_NC;     // co-main warps
constexpr int kBsNC2 = DSGPU_BS_NC2;  // co-main warps of the list CTA when the sweep runs on a CTA pair
constexpr int kBsRC = 16;    // c ring (co-main -> main), groups (power of two)
constexpr int kBsRL = 16;    // y landing ring of the list CTA (chain CTA -> relay warp), groups (power of two)
constexpr int kBsMC = 4;     // mid-list chunk (entries per lane)
constexpr int kBsFC = 8;     // far-list chunk (entries per lane)
constexpr int kBsStage = DSGPU_BS_STAGE;  // mid-list entries per lane staged ahead in shared memory (cp.async)
constexpr int kBsStageBytes = kBsStage / kBsMC * 3 * 512;  // per buffer: chunks x (int4 + 2 double2) x 32 lanes
constexpr int kBsBlock = kBsB * kBsB * 8;              // bytes of one dense block
constexpr int kBsSlotBytes = kBsK * kBsBlock;          // F_1..F_K (T_g travels separately: co-mains load it)
constexpr int kBsZero = kBsR * kBsB * 8;               // byte offset of the ring's zero slot

// Lane-unit layouts. A dense block: lane l = (row r = l & 15, half h = l >> 4)
// owns columns 8h..8h+7 as four 16-byte units; unit q of lane l sits at byte
// ((q * 32) + l) * 16 (conflict-free 128-bit shared loads). Sparse lists: entry
// k of lane l at int32 index ((k / 4) * 32 + l) * 4 + k % 4 and double index
// ((k / 2) * 32 + l) * 2 + k % 2 from the group's base (coalesced 128-bit loads).
inline int64_t bs_i32_at(int k, int l) { return (static_cast<int64_t>(k >> 2) * 32 + l) * 4 + (k & 3); }
inline int64_t bs_f64_at(int k, int l) { return (static_cast<int64_t>(k >> 1) * 32 + l) * 2 + (k & 1); }

struct HostBSweep {
  int n = 0, G = 0, dir = 0;        // dir 0: forward (L), 1: backward (L^T, reversed ordering)
  std::vector<uint8_t> slots;        // (G + kBsK + 1) * kBsSlotBytes: zero blocks behind the last group, so the
                                     //   main warps never clamp a look-ahead index
  std::vector<uint8_t> tblk;         // G * kBsBlock: T_g = D_g^{-1} (read by the co-mains straight from global memory)
  std::vector<int32_t> mw, ms;       // mid list: width (multiple of kBsMC), leading entries that only
                                     //   need groups <= g-K-3 (multiple of kBsMC)
  std::vector<int64_t> mptr;         // G + 1, element offset of the group's lists (width * 32 each)
  std::vector<int32_t> mcols;        // byte offsets into the y ring (pad: kBsZero)
  std::vector<double> mvals;
  std::vector<int32_t> fw;           // far list: width (multiple of kBsFC; 0 = none)
  std::vector<int64_t> fptr;         // G + 1
  std::vector<int32_t> fcols;        // rows of the result vector (original ordering); padding entries
                                     //   (value 0) point at the group's oldest far column
  std::vector<double> fvals;
  std::vector<int32_t> fcptr;        // G + 1: first chunk of the group in fneed
  std::vector<int32_t> fneed;        // per chunk: newest group it depends on (-1: none)
  int64_t nnz_dense = 0, nnz_mid = 0, nnz_far = 0;  // factor entries by class (statistics)
};

// Builds both sweeps of the factor L (lower triangular CSR, columns ascending,
// diagonal last in each row, as Ic0Factor::lower). Throws std::invalid_argument.
void build_bsweeps(const dsgpu_csr& L, HostBSweep& fwd, HostBSweep& bwd);

// CPU evaluation of one sweep plan (tests: the plan against the plain
// substitution): x = T^{-1} rhs in the sweep's own arithmetic order.
void bsweep_host_apply(const HostBSweep& s, const double* rhs, double* x);

// The sweep runs on ONE CTA (part 0: every role) or on a CTA PAIR of a 2-CTA
// thread-block cluster (part 1, "chain": main, second main, producer, publisher
// -- the dense blocks; part 2, "lists": the co-mains and a relay warp that
// receives the chain CTA's results through distributed shared memory), so that
// the chain's latency-critical shared-memory loads do not queue behind the
// lists' bulk traffic on one SM's shared-memory pipe.
enum { kBsWhole = 0, kBsChain = 1, kBsLists = 2 };

// Shared memory of a sweep CTA with a slot ring of `ns` slots (same carve-up as
// BsSmem in bsweep.cuh; the chain CTA of a pair may use a deeper ring ns1).
inline size_t bs_smem_bytes_part(int ns, int part) {
  const int nc = part == kBsLists ? kBsNC2 : (part == kBsChain ? 0 : kBsNC);
  const int nslot = part == kBsLists ? 0 : ns;
  return static_cast<size_t>(kBsZero) + 128            // y ring + zero slot
         + kBsRC * kBsB * 16                            // c ring / y landing ring (tagged 16-byte units)
         + kBsRQ * 32 * 8                               // q ring
         + static_cast<size_t>(nslot) * kBsSlotBytes    // dense-block slots
         + static_cast<size_t>(nc) * 2 * kBsStageBytes  // co-main mid-list staging (double-buffered)
         + static_cast<size_t>(nslot) * 8               // mbarriers
         + (2 * nslot + kBsRQ + 8) * 4 + 128;           // sready, base_use, qready, progress words
}
inline size_t bs_smem_bytes(int ns) { return bs_smem_bytes_part(ns, kBsWhole); }
inline size_t bs_smem_bytes_pair(int ns) {
  return bs_smem_bytes_part(ns, kBsChain) > bs_smem_bytes_part(ns, kBsLists) ? bs_smem_bytes_part(ns, kBsChain)
                                                                              : bs_smem_bytes_part(ns, kBsLists);
}

}  // namespace dsgpu
