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
// Who does what (measured reasons in DESIGN.md):
//   * SWEEP CTA (one SM) -- only the dense near-diagonal part, because one SM
//     moves 128 B/clk through shared memory and every byte it touches costs:
//       - MAIN warp: y_g = c_g - q_g - F_{g,1} y_{g-1} - F_{g,2} y_{g-2}; lane
//         (r, h) owns row r and columns 8h..8h+7 of each block (two lanes per
//         row, one shuffle). Only F_{g,1} y_{g-1} is on the dependent chain.
//       - SECOND MAIN warp: q_g = sum_{k=3..K} F_{g,k} y_{g-k}, accumulated as
//         the y's appear (two steps of slack).
//       - PRODUCER lane: TMA bulk copies of each group's F_1..F_K into a
//         shared-memory slot ring. PUBLISHER warp: the plain result vector.
//   * WORKER warps on all the other SMs (one group per warp, round-robin):
//     c_g = T_g ( r_g - sum_{h < g-K} E_{g,h} y_h ): the whole sparse part of
//     the factor (97 % of its entries at 32^3), streamed once from HBM as
//     lane-interleaved lists, y gathered from L2.
// Every cross-SM hand-off (y to the workers, c to the main warp, the
// right-hand side) travels as self-validating 16-byte units {low word, tag,
// high word, tag} -- two 8-byte halves, each carrying the sweep's tag, like
// NCCL's LL protocol -- polled by the consumer: no fence, no flag. Measured
// (tools/bs_lab.cu): 175 cycles per hop against 2,260 for data + fence + flag.
// A worker needs y_{g-K-1} before it can finish c_g, and the main warp needs c_g
// K steps later: K sets that slack.
// The backward solve is the same sweep on the reversed ordering (row p of the
// sweep = row n-1-p of the factor; L^T's rows are L's columns).
//
// Arithmetic: T_g and F_{g,k} are formed in long double and rounded once; the
// sweep itself is fp64. The result is the same operator (L L^T)^{-1} applied
// with a different association (measured agreement with the reference's
// Ic0Factor::solve: ~1e-15, see tests/test_gpu_parity.py); the exact
// column-order sweep stays available behind DSGPU_EXACT=1.
#pragma once

#include <cstdint>
#include <vector>

#include "dsgpu.h"

namespace dsgpu {

constexpr int kBsB = 16;     // rows per group
constexpr int kBsK = 6;      // dense pre-multiplied coupling blocks: F_1, F_2 on the main warp,
                             //   F_3..F_K on the second main warp
constexpr int kBsR = 16;     // y ring depth in groups (main -> second main, publisher); power of two
constexpr int kBsRQ = 8;     // q ring (second main warp -> main), groups (power of two)
constexpr int kBsLC = 8;     // list chunk (entries per lane)
constexpr int kBsBlock = kBsB * kBsB * 8;        // bytes of one dense block
constexpr int kBsSlotBytes = kBsK * kBsBlock;    // F_1..F_K of one group

// Lane-unit layouts. A dense block: lane l = (row r = l & 15, half h = l >> 4)
// owns columns 8h..8h+7 as four 16-byte units; unit q of lane l sits at byte
// ((q * 32) + l) * 16 (conflict-free 128-bit loads). Sparse lists: entry k of
// lane l at int32 index ((k / 4) * 32 + l) * 4 + k % 4 and double index
// ((k / 2) * 32 + l) * 2 + k % 2 from the group's base (coalesced 128-bit loads);
// a row's entries are dealt alternately to its two lanes, oldest first,
// right-aligned in the group's width.
inline int64_t bs_i32_at(int k, int l) { return (static_cast<int64_t>(k >> 2) * 32 + l) * 4 + (k & 3); }
inline int64_t bs_f64_at(int k, int l) { return (static_cast<int64_t>(k >> 1) * 32 + l) * 2 + (k & 1); }

struct HostBSweep {
  int n = 0, G = 0, dir = 0;        // dir 0: forward (L), 1: backward (L^T, reversed ordering)
  std::vector<uint8_t> slots;        // (G + kBsK + 1) * kBsSlotBytes: zero groups behind the last one, so
                                     //   the main warps never clamp a look-ahead index
  std::vector<uint8_t> tblk;         // G * kBsBlock: T_g = D_g^{-1} (workers)
  std::vector<int32_t> lw;           // list width of a group (multiple of kBsLC; 0 = none)
  std::vector<int64_t> lptr;         // G + 1: element offset of the group's lists (width * 32 each)
  std::vector<int32_t> lcols;        // rows of the result vector (original ordering); padding entries
                                     //   (value 0) point at the group's oldest column
  std::vector<double> lvals;
  int64_t nnz_dense = 0, nnz_list = 0;  // factor entries in dense blocks / in the lists
};

// Builds both sweeps of the factor L (lower triangular CSR, columns ascending,
// diagonal last in each row, as Ic0Factor::lower). Throws std::invalid_argument.
void build_bsweeps(const dsgpu_csr& L, HostBSweep& fwd, HostBSweep& bwd);

// CPU evaluation of one sweep plan (tests: the plan against the plain
// substitution): x = T^{-1} rhs in the sweep's own arithmetic order.
void bsweep_host_apply(const HostBSweep& s, const double* rhs, double* x);

// Shared memory of the sweep CTA with a slot ring of `ns` slots.
inline size_t bs_smem_bytes(int ns) {
  return static_cast<size_t>(kBsR) * kBsB * 8 + 128      // y ring
         + kBsRQ * 32 * 8                                 // q ring
         + static_cast<size_t>(ns) * kBsSlotBytes         // dense-block slots
         + static_cast<size_t>(ns) * 8                    // mbarriers
         + (2 * ns + kBsRQ + 8) * 4 + 256;                // sready, base_use, qready, progress words
}

}  // namespace dsgpu
