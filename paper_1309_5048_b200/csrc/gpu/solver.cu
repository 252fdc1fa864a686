// B200 (sm_100a) MINRES + block-diagonal IC(0)/PCG preconditioned Stokes
// solve, behind the C ABI of include/dsgpu.h.
//
// Execution model: ONE cooperative persistent kernel runs the whole
// preconditioned MINRES (reference proj/src/solvers.cpp:24-123) including the
// inner PCG of each preconditioner block (solvers.cpp:125-159, driven as
// PcgBlock::apply, precond.cpp:75-100) and the IC(0) applies
// (cholesky.cpp:136-152). Scalars never leave the device: every CTA reduces
// the same per-CTA partials in the same fixed order and takes identical
// control decisions, so the only cross-CTA synchronization is one grid
// barrier per dependent phase:
//   outer iteration  : [w/aw/x/res update of it-1 + v = y/beta + saddle SpMV
//                       + alpha partial]  |  [precond]
//   precond start    : [r := input; IC sweeps or Jacobi]          | reduce rho
//   inner PCG step   : [q = A p (p = z + beta p on the fly)]      | reduce kappa
//                      [r -= alpha q; IC sweeps; x += alpha p]    | reduce rho'
// The IC(0) sweeps of a block run inside one CTA (sync-free, level-grouped,
// see dsgpu_internal.hpp) while the other CTAs do the element-wise updates;
// the top (velocity) and bottom (pressure) blocks run concurrently on
// different CTAs, their PCG loops in lockstep.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "dsgpu_internal.hpp"
#include "kernels.cuh"
#include "partition.hpp"
#include "pi.cuh"
#include "bsweep.cuh"

using namespace dsgpu;
using namespace dsgpu::dev;

namespace {

constexpr int kThreads = 512;
constexpr int kDefaultMerge = 2;
constexpr int kWarps = kThreads / 32;

enum Slot { SL_BB = 0, SL_RES, SL_ALPHA, SL_RHO0, SL_RHO1, SL_KAP0, SL_KAP1, SL_ZR0, SL_ZR1, SL_NUM, NSLOT };

struct DSweep {
  int n_groups;
  const int64_t* gptr;
  const int32_t* gwidth;
  const int32_t* grows;
  const int32_t* cols;
  const double* vals;
  const double* diag;
};

struct DFlow {
  int G;
  const int32_t *nr, *pw, *ww, *grows, *pcols, *wcols;
  const int64_t *pptr, *wptr;
  const double *pvals, *wvals;
  const uint8_t* stat;  // G * SlotLayout(tb).bytes, 16-byte aligned
  int ring;
  const int32_t *gw, *gneed, *gcols;
  const int64_t* gptr;
  const double* gvals;
  const int32_t *cptr, *cneed;  // prefix-list chunks: newest dependency group of each
  int rsplit;                   // remote helpers: warps per group's older-than-ring list (<= kRSplit)
};

struct DBlock {
  int kind, n, off, ic_cta;
  const int64_t* rp;  // operator rows (block ordering)
  const int32_t* ci;
  const double* v;
  const int32_t* na;  // top block: (padded) A-part length of each K row (nullptr: full row)
  int lanes;          // lanes per row of the block SpMV (row_partial)
  const double* dinv;
  DSweep fwd, bwd;    // exact column-order sweeps (bit-identical mode)
  DFlow ffwd, fbwd;   // staged sweeps (production)
  int exact;          // 1: use the exact sweeps
  double *r, *z, *q, *p0, *p1;  // PCG work (block-local, length n)
  double* y;                    // forward-sweep result (staged mode), n + 1 (y[n] = 0)
  double* bb;                   // materialized right-hand side (staged mode), n + 1
  // ring mode: partial sums of the entries older than the ring are computed by
  // "remote" helper CTAs and handed over through global memory
  double* rpsum;                // max(G) * kRSplit * 32
  unsigned* rflag;              // max(G) * kRSplit: sweep tag once rpsum[g][part] is final
  unsigned long long* gprog;    // (sweep tag << 32) | groups published by the main warp
  int remote_cta0, n_remote;    // remote helper CTAs (0: none)
  int pi;                       // 1: partitioned-inverse IC(0) apply (pi.cuh), all CTAs
  DPi pim;
  // blocked sweeps (bsweep.cuh): remote_cta0 / n_remote name the far-worker CTAs
  int bs, bs_ns;                // 1: blocked sweeps; slot-ring depth
  DBSweep bfwd, bbwd;
  uint4* bs_bt;                 // n: tagged right-hand side, written by the rows' owners (every GPU's workers)
  uint4* bs_gt;                 // n + 1: tagged copy of the sweep result (far workers gather it)
  uint4* bs_fps;                // max(G) * 16: tagged far partial sums
};

// Multi-GPU state of one rank (partition.hpp). Every rank runs
// the same persistent kernel on its own rows; all cross-GPU traffic goes through
// peer memory (the ranks' arenas, mapped into every rank with CUDA IPC):
//   * halo: before an SpMV the ranks copy the vector entries their rows need
//     from the owners' vectors (NVLink peer loads);
//   * dot products: every grid-barrier reduction is followed by an exchange of
//     the per-GPU sums through peer mailboxes (stores + release flag, summed in
//     rank order on every GPU: identical values everywhere);
//   * IC(0): every rank pushes its rows of the block residual, tagged, into
//     every rank's right-hand-side buffer and all ranks run the whole sweep
//     (replicated: the preconditioner is the single-GPU one).
constexpr int kMaxWorld = 8;
struct MultiGpu {
  int world, rank;
  char* arena[kMaxWorld];          // base of every rank's arena in THIS rank's address space
  const int2* halo_y;              // {K' column, owner}: entries of y this rank's rows read but do not own
  int n_halo_y;
  const int2* halo_p[2];           // the same for the block operators (block-local column, owner)
  int n_halo_p[2];
  double* xsum;                    // [2][kMaxWorld][NSLOT] mailbox (in the arena)
  unsigned* xflag;                 // [2][kMaxWorld]
};
template <class T>
__device__ __forceinline__ T* peer_ptr(const MultiGpu& m, T* p, int r) {
  return reinterpret_cast<T*>(m.arena[r] + (reinterpret_cast<char*>(p) - m.arena[m.rank]));
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DevReport {
  int iterations, converged, status, failed_block, hist_len, pad;
  double relres_m, relres_e;
  long long inner[2], apps[2];
};

// Request / completion mailbox of one IC(0) server CTA (one per IC block).
// Workers post a request with st.release on `req`; the server answers with the
// CTA's <r, z> on `rz` and st.release on `done`.
enum { IC_OP_S1 = 1, IC_OP_L2 = 2, IC_OP_EXIT = 3 };
struct alignas(128) Mailbox {
  unsigned req;
  int op;
  double alpha;          // L2: r -= alpha q
  const double* src0;    // S1: r = src0 (+ coef src1), also stored to dst
  const double* src1;
  double coef;
  double* dst;
  alignas(128) unsigned done;
  double rz;
};

struct Args {
  int n, n_u, n_p;
  const int64_t* k_rp;
  const int32_t* k_ci;
  const double* k_v;
  const int32_t *row_lo, *row_hi;  // per worker CTA: its rows [row_lo, row_hi) of K' (within one block)
  int k_lanes;               // lanes per row of the saddle SpMV (row_partial)
  MultiGpu mg;               // world > 1: the row-partitioned solve across the box's GPUs
  DBlock blk[2];
  const double* f_in;        // n_u, original order
  const double* u0_in;       // initial guess (MinresOptions::x0, solvers.hpp:34), original order; null: x0 = 0
  const double* p0_in;
  const int32_t* perm_u;     // block ordering -> original
  const int32_t* perm_p;
  double* u_out;             // n_u, original order
  double* p_out;             // n_p, original order
  double *x, *y, *v, *av, *res;
  double* rbuf[4];
  double* w[3];
  double* aw[3];
  const double* qk;
  double filter_den;
  int filter;
  double* partial;           // [2][NSLOT][G]
  unsigned* bar;             // count @ [0], gen @ [32], abort @ [64]
  double* hist_m;
  double* hist_e;
  int hist_cap;
  double outer_tol, inner_tol;
  int max_iter, stop_euclid, inner_cap;
  DevReport* rep;
  int smem_half;  // doubles per dataflow array (largest IC block)
  unsigned launch_id;  // distinguishes the sweep tags of successive launches
  int n_srv;           // CTAs [0, n_srv) are IC(0) servers (CTA b serves block b; with bs_pair CTAs 2b, 2b + 1)
  int bs_pair;         // blocked sweeps on CTA pairs (2-CTA clusters: chain + lists, bsweep.hpp)
  Mailbox* mbox;       // [2]
};

// ---------------------------------------------------------------------------
// triangular sweep (one CTA): x = T^{-1} rhs with T unit-free rows
// x_i = (rhs_i - sum_k T_ik x_k) / d_i, entries in stored order, no FMA.
template <class Rhs, class Out>
__device__ void sweep(const DSweep& s, double* xs, int n, Rhs rhs, Out out, unsigned* abort_flag) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    const int row = s.grows[static_cast<int64_t>(g) * 32 + lane];
    double acc = row >= 0 ? rhs(row) : 0.0;
    const int width = s.gwidth[g];
    const int32_t* cp = s.cols + s.gptr[g] + lane;
    const double* vp = s.vals + s.gptr[g] + lane;
    int k = 0;
    for (; k + 4 <= width; k += 4) {
      const int c0 = cp[0], c1 = cp[32], c2 = cp[64], c3 = cp[96];
      const double v0 = vp[0], v1 = vp[32], v2 = vp[64], v3 = vp[96];
      cp += 128;
      vp += 128;
      if (c0 >= 0) acc = sub_rn(acc, mul_rn(v0, slot_wait(xs, c0, abort_flag)));
      if (c1 >= 0) acc = sub_rn(acc, mul_rn(v1, slot_wait(xs, c1, abort_flag)));
      if (c2 >= 0) acc = sub_rn(acc, mul_rn(v2, slot_wait(xs, c2, abort_flag)));
      if (c3 >= 0) acc = sub_rn(acc, mul_rn(v3, slot_wait(xs, c3, abort_flag)));
    }
    for (; k < width; ++k) {
      const int c0 = cp[0];
      const double v0 = vp[0];
      cp += 32;
      vp += 32;
      if (c0 >= 0) acc = sub_rn(acc, mul_rn(v0, slot_wait(xs, c0, abort_flag)));
    }
    if (row >= 0) {
      const double xi = div_rn(acc, s.diag[row]);
      slot_publish(xs, row, xi);
      out(row, xi);
    }
  }
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Staged dataflow sweep (production): see HostFlow in dsgpu_internal.hpp.
// Shared memory: xs[n+1] (results; xs[n] = 0 is the padding slot) followed by
// a ring of kRing slots. Executed by every thread of one CTA; on return
// (after a CTA barrier) xs holds the solution.
template <int N>
__device__ __forceinline__ double tree_sum(double* p) {
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int k = 0; k + w < N; k += 2 * w) p[k] = add_rn(p[k], p[k + w]);
  return p[0];
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  unsigned lo, hi, rlo, rhi;
  asm volatile("mov.b64 {%0,%1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rlo) : "r"(lo), "r"(src));
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rhi) : "r"(hi), "r"(src));
  double out;
  asm volatile("mov.b64 %0, {%1,%2};" : "=d"(out) : "r"(rlo), "r"(rhi));
  return out;
}

// Shared-memory workspace of one staged sweep: xs[n+1] | ring of kSRing static
// slots (SlotLayout, filled by TMA bulk copies) | psum[kRing][32] (helpers ->
// co-main) | apre[kRing][32] (co-main -> main) | mbarriers | flags | progress.
struct FlowSmem {
  double* xs;
  uint8_t* slots;
  double* psum;
  double* apre;
  uint64_t* mbar;
  volatile int* pready;   // psum of group g staged (helpers)
  volatile int* aready;   // acc_pre of group g staged (co-main)
  volatile int* sready;   // static data of group g landed (producer, after its mbarrier)
  volatile int* progress;
  volatile int* gprogress;  // ring mode: groups whose results are visible in global memory
  int* base_use;  // completed mbarrier phases per slot before this sweep
  int slot_bytes;
  // n = number of x slots (rows in full mode, kXRing*32 in ring mode); xs[n] = 0
  __device__ FlowSmem(double* base, int n, int sb) : slot_bytes(sb) {
    xs = base;
    const size_t xbytes = (static_cast<size_t>(n + 1) * 8 + 127) / 128 * 128;
    slots = reinterpret_cast<uint8_t*>(base) + xbytes;
    psum = reinterpret_cast<double*>(slots + static_cast<size_t>(kSRing) * sb);
    apre = psum + kRing * 32;
    mbar = reinterpret_cast<uint64_t*>(apre + kRing * 32);
    pready = reinterpret_cast<volatile int*>(mbar + kSRing);
    aready = pready + kRing;
    sready = aready + kRing;
    progress = sready + kSRing;
    gprogress = progress + 1;
    base_use = const_cast<int*>(gprogress) + 1;
  }
  static size_t bytes(int n, int sb) { return flow_smem_bytes(n, sb); }
};

// Once per kernel launch and CTA, before any staged sweep: the ring's
// mbarriers are initialized once and then only ever advance (re-initializing
// an mbarrier the bulk-copy unit has used is not safe).
template <int TB>
__device__ void flow_setup(double* smem, int n, int ring) {
  FlowSmem S(smem, ring ? kXRing * 32 : n, SlotLayout(TB).bytes);
  for (int i = threadIdx.x; i < kSRing; i += blockDim.x) {
    mbar_init(S.mbar + i, 1);
    S.base_use[i] = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

// diagnostics: [0] main-warp cycles, [1] main cycles waiting for slots,
// [2] groups processed by the main warp (summed over sweeps), [3] abort code,
// [4] main cycles waiting for the producer (static slot data), [5] helper
// cycles waiting for their ring-list dependencies, [6] helper cycles waiting
// for remote partial sums, [7] helper cycles in total (all helper warps),
// [8..11] groups by main's distance when the helper published them (g minus
// groups done: <=1, 2-3, 4-6, >=7), [12..15] the same at the helper's start of
// the group (<=3, 4-7, 8-11, >=12), [16] helper cycles from the end of the
// last dependency wait to the prefix-sum publication, [17] groups whose last
// dependency wait had to spin
__device__ unsigned long long g_flow_dbg[32];
// helper polling back-off (ns); DSGPU_HSLEEP overrides it (experiments)
__device__ unsigned g_hsleep = 20;
// timing experiments only (DSGPU_NOWAIT=1): the main warp does not wait for
// the co-mains (results are wrong); isolates the main warp's own loop cost
__device__ int g_nowait = 0;
// phase diagnostics of the persistent kernel: [0] CTA0 cycles in grid barriers,
// [1] CTA0 cycles in IC(0) applies, [2] CTA2 cycles in grid barriers,
// [3] barriers, [4] CTA0 kernel cycles, [5] CTA1 cycles in IC(0) applies
__device__ unsigned long long g_phase_dbg[8];
// SpMV phases of the persistent kernel as worker CTA 0 sees them (diag build):
// M1 (outer saddle SpMV): [0] cycles of its own rows, [1] phases, [2] stored
// entries of its rows, [3] cycles through the phase's grid barrier; L1 (inner
// A-block SpMV): [4] own cycles, [5] phases, [6] stored entries of its rows,
// [7] cycles through the barrier (the pressure block's SpMV included)
__device__ unsigned long long g_spmv_dbg[8];
#ifdef DSGPU_DIAG
#define PHASE_DIAG(...) __VA_ARGS__
#else
#define PHASE_DIAG(...)
#endif

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Hand-off state of one ring-mode sweep with remote helpers.
struct FlowRemote {
  double* rpsum;
  unsigned* rflag;
  unsigned long long* gprog;
  unsigned tag;  // unique per sweep within a launch, launch id in the top bits
  int on;        // remote helpers active
};

__device__ __forceinline__ unsigned sweep_tag(unsigned launch_id, unsigned sweep_no) {
  return ((launch_id & 0xFFFu) << 20) | (sweep_no & 0xFFFFFu);
}

// Remote helpers (other CTAs): for every group, the partial sum of the entries
// older than the shared-memory ring, from the results the main warp has
// published in global memory. rank / nranks: this CTA among the remote CTAs.
__device__ void flow_remote(const DFlow& s, int n, const double* __restrict__ gx, FlowRemote R,
                            int rank, int nranks, unsigned* abort_flag) {
  constexpr int PW = 16;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int wid = rank * nw + (threadIdx.x >> 5), W = nranks * nw;
  // task t = (group g, part): kRSplit consecutive warps share one group's list
  // (chunks part, part + kRSplit, ...) so its partial sum is ready kRSplit x
  // sooner; each part publishes its own slot and flag
  const int S = s.rsplit;
  for (int t = wid; t < s.G * S; t += W) {
    const int g = t / S, part = t - g * S;
    const int gw = __ldg(s.gw + g);
    if (gw == 0) continue;
    const int gneed = __ldg(s.gneed + g);
    const int64_t gb = __ldg(s.gptr + g);
    const unsigned need = static_cast<unsigned>(gneed + 1);
    double acc = 0.0;
    SpinGuard sg(abort_flag);
    const int32_t* gc = s.gcols + gb + part * PW * 32 + lane;
    const double* gv = s.gvals + gb + part * PW * 32 + lane;
    bool waited = false;
    for (int k0 = part * PW; k0 < gw; k0 += S * PW, gc += S * PW * 32, gv += S * PW * 32) {
      int pc[PW];
      double pv[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) {  // widths are whole chunks, pads are (n, 0)
        pc[q] = __ldg(gc + q * 32);
        pv[q] = __ldg(gv + q * 32);
      }
      if (!waited) {
        waited = true;
        for (;;) {  // the tag must match: stale words of other sweeps never count
          const unsigned long long v = ld_acquire_u64(R.gprog);
          if (static_cast<unsigned>(v >> 32) == R.tag && static_cast<unsigned>(v) >= need) break;
          __nanosleep(100);
          if (sg.expired()) {
            g_flow_dbg[3] = 1000000000ull * 7 + 100000ull * s.G + g;
            break;
          }
        }
      }
      double pp[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) pp[q] = mul_rn(pv[q], __ldcg(gx + pc[q]));
      acc = add_rn(acc, tree_sum<PW>(pp));
    }
    __stcg(R.rpsum + static_cast<int64_t>(t) * 32 + lane, acc);
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(R.rflag + t, R.tag);
  }
}

// gx: ring mode only -- results are written there (global, n+1 with gx[n] = 0).
template <int TB, bool RING>
__device__ void flow_sweep(const DFlow& s_in, int n, double* smem, const double* __restrict__ b,
                           double* gx, FlowRemote R, unsigned* abort_flag) {
  // Local copy of the plan's header: reached through a generic pointer in the
  // persistent kernel, its fields would be reloaded after every volatile
  // shared-memory access otherwise.
  const DFlow s = s_in;
  const int G = s.G;
  const SlotLayout lay(TB);
  const int xcount = RING ? kXRing * 32 : n;
  FlowSmem S(smem, xcount, lay.bytes);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // x workspace read through byte offsets (one shared load, no index scaling)
  auto xs_at = [&](int boff) {
    return *reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(S.xs) + boff);
  };
  for (int i = threadIdx.x; i < kRing; i += blockDim.x) {
    S.pready[i] = -1;
    S.aready[i] = -1;
    if (i < kSRing) S.sready[i] = -1;
  }
  if (threadIdx.x == 0) {
    *S.progress = 0;
    *S.gprogress = 0;
    S.xs[xcount] = 0.0;
  }
  __syncthreads();
  // roles: main = last warp; producer = lane 0 of the warp 4 below it (same
  // SM sub-partition, nearly idle); co-mains = the kCo warps before main (other
  // sub-partition); helpers = the remaining warps off main's sub-partition.
  constexpr int kCo = 2;  // co-main warps (round-robin over groups)
  const int mainw = nw - 1, prodw = nw - 5;
  const int cid = warp < mainw && warp >= mainw - kCo ? mainw - 1 - warp : -1;
  int hid = -1, nh = 0;
  for (int w = 0; w < nw; ++w)
    if (w != mainw && !(w < mainw && w >= mainw - kCo) && (w & 3) != (mainw & 3)) {
      if (w == warp) hid = nh;
      ++nh;
    }
  auto ld_f64 = [&](const uint8_t* arr, double* out, int cnt) {
    const double2* p = reinterpret_cast<const double2*>(arr) + lane;
#pragma unroll
    for (int j = 0; j < cnt / 2; ++j) {
      const double2 t = p[j * 32];
      out[2 * j] = t.x;
      out[2 * j + 1] = t.y;
    }
  };
  auto ld_i32 = [&](const uint8_t* arr, int* out, int cnt) {
    const int4* p = reinterpret_cast<const int4*>(arr) + lane;
#pragma unroll
    for (int j = 0; j < cnt / 4; ++j) {
      const int4 t = p[j * 32];
      out[4 * j] = t.x;
      out[4 * j + 1] = t.y;
      out[4 * j + 2] = t.z;
      out[4 * j + 3] = t.w;
    }
  };
  auto slot_of = [&](int gg) { return S.slots + (static_cast<unsigned>(gg) & (kSRing - 1)) * lay.bytes; };
  static_assert(kTA % 4 == 0 && TB % 4 == 0 && (kRing & (kRing - 1)) == 0 &&
                    (kSRing & (kSRing - 1)) == 0, "slot layout");
  if (warp == mainw && G > 0) {
    // iteration g: gather the B operands (groups g-1, g-2: written by this
    // warp) from xs, take the co-main's acc_pre(g), x(g) = (acc_pre - B) / d.
    // Group g+1's B offsets are loaded one iteration ahead.
    int bcn[TB];
    const long long t_main0 = clock64();
    long long wait_cyc = 0, wait_s = 0;
    int pf_s = -2;  // sready of g+1, prefetched one iteration ahead
    auto wait_static = [&](int gg) {
      if (pf_s != gg) {
        SpinGuard sg(abort_flag);
        while (S.sready[gg & (kSRing - 1)] != gg)
          if (sg.expired()) {
            g_flow_dbg[3] = 1000000000ull * 1 + 100000ull * G + gg;
            break;
          }
        const long long w = clock64() - sg.t0;
        wait_cyc += w;
        wait_s += w;
      }
    };
    const int glast = G - 1;
    wait_static(0);
    ld_i32(S.slots + lay.bcol, bcn, TB);
    for (int g = 0; g < G; ++g) {
      const uint8_t* base = slot_of(g);
      // (1) B operands and values in halves of at most 8 (register pressure)
      constexpr int TH = TB < 8 ? TB : 8;
      double bsum[TB / TH];
#pragma unroll
      for (int hh = 0; hh < TB / TH; ++hh) {
        double xb[TH], bv[TH], pb[TH];
#pragma unroll
        for (int k = 0; k < TH; ++k) xb[k] = xs_at(bcn[hh * TH + k]);
        const double2* bvp = reinterpret_cast<const double2*>(base + lay.bval) + lane + hh * (TH / 2) * 32;
#pragma unroll
        for (int j = 0; j < TH / 2; ++j) {
          const double2 t = bvp[j * 32];
          bv[2 * j] = t.x;
          bv[2 * j + 1] = t.y;
        }
#pragma unroll
        for (int k = 0; k < TH; ++k) pb[k] = mul_rn(bv[k], xb[k]);
        bsum[hh] = tree_sum<TH>(pb);
      }
      // (2) this group's static values (landed: checked in iteration g-1)
      const double2 ddv = reinterpret_cast<const double2*>(base + lay.dd)[lane];
      const int row = reinterpret_cast<const int*>(base + lay.rows)[lane];
      const int nr = *reinterpret_cast<const int*>(base + lay.meta);
      // (3) next group's B offsets
      const int g1 = g + 1 < G ? g + 1 : glast;
      wait_static(g1);
      int bcn1[TB];
      ld_i32(slot_of(g1) + lay.bcol, bcn1, TB);
      pf_s = S.sready[(g + 2 < G ? g + 2 : glast) & (kSRing - 1)];
      // (4) acc_pre(g) from the co-mains
      const int sa = g & (kRing - 1);
      if (!g_nowait && S.aready[sa] != g) {
        SpinGuard sg(abort_flag);
        while (S.aready[sa] != g)
          if (sg.expired()) {
            g_flow_dbg[3] = 1000000000ull * 2 + 100000ull * G + g;
            break;
          }
        wait_cyc += clock64() - sg.t0;
      }
      const double ap = S.apre[sa * 32 + lane];
      // (5) the critical chain
      const double acc = sub_rn(ap, tree_sum<TB / TH>(bsum));
      // correctly rounded acc / d from the reciprocal (one Markstein step)
      const double q0 = mul_rn(acc, ddv.y);
      const double rr = fma(-q0, ddv.x, acc);
      const double x = fma(rr, ddv.y, q0);
      if (RING) {
        S.xs[(g & (kXRing - 1)) * 32 + lane] = x;
        if (lane < nr) gx[row] = x;
      } else if (lane < nr) {
        S.xs[row] = x;
      }
      __syncwarp();
      if (lane == 0) *S.progress = g + 1;
      if (RING && ((g + 1) % kFenceEvery == 0 || g + 1 == G)) {
        __threadfence();  // publish older results in global memory
        __syncwarp();
        if (lane == 0) {
          *S.gprogress = g + 1;
          if (R.on)  // ordered by the fence above
            st_relaxed_u64(R.gprog, (static_cast<unsigned long long>(R.tag) << 32) | (g + 1));
        }
      }
#pragma unroll
      for (int k = 0; k < TB; ++k) bcn[k] = bcn1[k];
    }
    if (lane == 0) {
      atomicAdd(&g_flow_dbg[0], static_cast<unsigned long long>(clock64() - t_main0));
      atomicAdd(&g_flow_dbg[1], static_cast<unsigned long long>(wait_cyc));
      atomicAdd(&g_flow_dbg[2], static_cast<unsigned long long>(G));
      atomicAdd(&g_flow_dbg[4], static_cast<unsigned long long>(wait_s));
    }
  } else if (cid >= 0) {
    // co-main: acc_pre(h) = psum(h) - A(h); A's dependencies are groups <= h-3
    long long wait_co = 0, t_work = 0;
    unsigned cpub[4] = {0, 0, 0, 0}, cwhy[2] = {0, 0};
    for (int h = cid; h < G; h += kCo) {
      SpinGuard sg(abort_flag);
      while (S.sready[h & (kSRing - 1)] != h)
        if (sg.expired()) {
          g_flow_dbg[3] = 1000000000ull * 9 + 100000ull * G + h;
          break;
        }
      const uint8_t* base = slot_of(h);
      double av[kTA];
      int ac[kTA];
      ld_i32(base + lay.acol, ac, kTA);
      ld_f64(base + lay.aval, av, kTA);
      const int sp = h & (kRing - 1);
      const long long t0 = clock64();
      cwhy[0] += S.pready[sp] != h;
      cwhy[1] += *S.progress < h - 2;
      while (S.pready[sp] != h || *S.progress < h - 2)
        if (sg.expired()) {
          g_flow_dbg[3] = 1000000000ull * 10 + 100000ull * G + h;
          break;
        }
      const long long t1 = clock64();
      wait_co += t1 - t0;
      const double ps = S.psum[sp * 32 + lane];
      double pa[kTA];
#pragma unroll
      for (int k = 0; k < kTA; ++k) pa[k] = mul_rn(av[k], xs_at(ac[k]));
      S.apre[sp * 32 + lane] = sub_rn(ps, tree_sum<kTA>(pa));
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        S.aready[sp] = h;
      }
      t_work += clock64() - t1;
      const int dist = h - *S.progress;
      ++cpub[dist <= 0 ? 0 : dist == 1 ? 1 : dist == 2 ? 2 : 3];
    }
    if (lane == 0) {
      atomicAdd(&g_flow_dbg[18], static_cast<unsigned long long>(wait_co));
      atomicAdd(&g_flow_dbg[23], static_cast<unsigned long long>(t_work));
      for (int i = 0; i < 4; ++i) atomicAdd(&g_flow_dbg[24 + i], static_cast<unsigned long long>(cpub[i]));
      atomicAdd(&g_flow_dbg[28], static_cast<unsigned long long>(cwhy[0]));
      atomicAdd(&g_flow_dbg[29], static_cast<unsigned long long>(cwhy[1]));
    }
  } else if (warp == prodw) {
    if (lane == 0) {
      int issued = 0, done = 0;
      SpinGuard sg(abort_flag);
      while (done < G) {
        bool idle = true;
        // issue: the slot's previous group (issued - kRing) was loaded by main
        // iteration issued - kRing - 1
        if (issued < G && *S.progress >= issued - kSRing + 2) {
          const int sl = issued % kSRing;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(S.mbar + sl, lay.bytes);
          bulk_g2s(S.slots + static_cast<size_t>(sl) * lay.bytes,
                   s.stat + static_cast<size_t>(issued) * lay.bytes, lay.bytes, S.mbar + sl);
          ++issued;
          idle = false;
        }
        // complete: publish the oldest outstanding copy once it has landed
        if (done < issued) {
          const int sl = done % kSRing;
          if (mbar_test(S.mbar + sl, (S.base_use[sl] + done / kSRing) & 1)) {
            S.sready[sl] = done;
            ++done;
            idle = false;
          }
        }
        if (idle) {
          if (sg.expired()) {
            g_flow_dbg[3] = 1000000000ull * 3 + 100000ull * G + done;
            break;
          }
        } else {
          sg.t0 = clock64();
        }
      }
    }
  } else if (hid >= 0) {
    constexpr int PW = kPW;
    const long long th0 = clock64();
    long long tw_need = 0, tw_rem = 0;
    unsigned hpub[4] = {0, 0, 0, 0}, hstart[4] = {0, 0, 0, 0};
    long long t_post = 0, t_pa = 0, t_pb = 0, t_pc = 0, t_pd = 0;
    unsigned n_spun = 0;
    int g = hid;
    int nr = 0, pw = 0;
    int64_t pb0 = 0;
    if (g < G) {
      nr = __ldg(s.nr + g);
      pw = __ldg(s.pw + g);
      pb0 = __ldg(s.pptr + g);
    }
    for (; g < G; g += nh) {
      const int sl = g % kRing;
      const int gn = g + nh;
      {
        const int dist = g - *S.progress;
        ++hstart[dist <= 3 ? 0 : dist <= 7 ? 1 : dist <= 11 ? 2 : 3];
      }
      int nrn = 0, pwn = 0;
      int64_t pbn = 0;
      if (gn < G) {
        nrn = __ldg(s.nr + gn);
        pwn = __ldg(s.pw + gn);
        pbn = __ldg(s.pptr + gn);
      }
      int row = -1;
      double rhs = 0.0;
      if (lane < nr) {
        row = __ldg(s.grows + static_cast<int64_t>(g) * 32 + lane);
        rhs = b[row];
        const int ww = __ldg(s.ww + g);
        const int64_t wb = __ldg(s.wptr + g);
        for (int k = 0; k < ww; ++k) {  // level-merge right-hand-side transform
          const int j = __ldg(s.wcols + wb + k * 32 + lane);
          rhs = add_rn(rhs, mul_rn(__ldg(s.wvals + wb + k * 32 + lane), b[j]));
        }
      }
      const int32_t* cp = s.pcols + pb0 + lane;
      const double* vp = s.pvals + pb0 + lane;
      // acc = rhs - (older entries) - (chunk sums): consuming rhs first keeps
      // its global load off the path after the last dependency wait
      double acc = lane < nr ? rhs : 0.0;
      SpinGuard sg(abort_flag);
      if (RING && R.on) {  // entries older than the ring: remote helpers' partial sum
        if (__ldg(s.gw + g) > 0) {
          const long long t0 = clock64();
          double rp[kRSplit];
#pragma unroll
          for (int q = 0; q < kRSplit; ++q) {
            rp[q] = 0.0;
            if (q < s.rsplit) {
              while (ld_acquire(R.rflag + g * s.rsplit + q) != R.tag) {
                __nanosleep(20);
                if (sg.expired()) {
                  g_flow_dbg[3] = 1000000000ull * 8 + 100000ull * G + g;
                  break;
                }
              }
              rp[q] = __ldcg(R.rpsum + (static_cast<int64_t>(g) * s.rsplit + q) * 32 + lane);
            }
          }
          tw_rem += clock64() - t0;
          acc = sub_rn(acc, tree_sum<kRSplit>(rp));
        }
      } else if (RING) {  // entries older than the ring: global memory, once published
        const int gw = __ldg(s.gw + g);
        if (gw > 0) {
          const int gneed = __ldg(s.gneed + g);
          const int64_t gb = __ldg(s.gptr + g);
          while (*S.gprogress <= gneed) {
            __nanosleep(20);
            if (sg.expired()) {
              g_flow_dbg[3] = 1000000000ull * 6 + 100000ull * G + g;
              break;
            }
          }
          const int32_t* gc = s.gcols + gb + lane;
          const double* gv = s.gvals + gb + lane;
          for (int k0 = 0; k0 < gw; k0 += PW, gc += PW * 32, gv += PW * 32) {
            int pc[PW];
            double pv[PW];
#pragma unroll
            for (int q = 0; q < PW; ++q) {
              pc[q] = __ldg(gc + q * 32);
              pv[q] = __ldg(gv + q * 32);
            }
            double pp[PW];
#pragma unroll
            for (int q = 0; q < PW; ++q) pp[q] = mul_rn(pv[q], __ldcg(gx + pc[q]));
            acc = sub_rn(acc, tree_sum<PW>(pp));
          }
        }
      }
      // ring-list entries, oldest chunk first; each chunk waits for its own
      // newest dependency, so the next chunk's loads overlap that wait
      // kPW-entry chunks, then the small last chunk (the newest entries)
      const int nbig = pw > 0 ? (pw - kPL) / PW : -1;
      long long t_last = clock64();
      bool spun = false;
      int seen = 0;  // last progress value observed
      const int c0 = pw > 0 ? __ldg(s.cptr + g) : 0;
      auto chunk = [&](auto width, int ch) {
        constexpr int CW = decltype(width)::value;
        const int32_t* cq = cp + ch * (PW * 32);
        const double* vq = vp + ch * (PW * 32);
        const int cn = __ldg(s.cneed + c0 + ch);
        int pc[CW];
        double pv[CW];
#pragma unroll
        for (int q = 0; q < CW; ++q) {
          pc[q] = __ldg(cq + q * 32);
          pv[q] = __ldg(vq + q * 32);
        }
        const long long t0 = clock64();
        spun = false;
        while ((seen = *S.progress) <= cn) {
          spun = true;
          __nanosleep(g_hsleep);
          if (sg.expired()) {
            g_flow_dbg[3] = 1000000ull * (blockIdx.x + 1) + 1000ull * 4 + (g % 1000);
            break;
          }
        }
        t_last = clock64();
        tw_need += t_last - t0;
        double pp[CW];
#pragma unroll
        for (int q = 0; q < CW; ++q) pp[q] = mul_rn(pv[q], xs_at(pc[q]));
        acc = sub_rn(acc, tree_sum<CW>(pp));
      };
      for (int ch = 0; ch < nbig; ++ch) chunk(std::integral_constant<int, PW>(), ch);
      if (nbig >= 0) chunk(std::integral_constant<int, kPL>(), nbig);
      if (lane >= nr) acc = 0.0;
      const long long t_a = clock64();
      // psum slot reuse: group g - kRing's psum was consumed before the main
      // warp's iteration g - kRing (skip the read when already observed)
      while (seen < g - kRing + 2 && (seen = *S.progress) < g - kRing + 2) {
        __nanosleep(20);
        if (sg.expired()) {
          g_flow_dbg[3] = 1000000ull * (blockIdx.x + 1) + 1000ull * 5 + (g % 1000);
          break;
        }
      }
      const long long t_b = clock64();
      S.psum[sl * 32 + lane] = acc;
      __syncwarp();
      const long long t_c = clock64();
      if (lane == 0) {
        __threadfence_block();
        S.pready[sl] = g;
      }
      const long long t_d = clock64();
      t_pa += t_a - t_last;
      t_pb += t_b - t_a;
      t_pc += t_c - t_b;
      t_pd += t_d - t_c;
      {
        const int dist = g - *S.progress;
        ++hpub[dist <= 1 ? 0 : dist <= 3 ? 1 : dist <= 6 ? 2 : 3];
        t_post += clock64() - t_last;
        n_spun += spun;
      }
      nr = nrn;
      pw = pwn;
      pb0 = pbn;
    }
    if (lane == 0) {
      atomicAdd(&g_flow_dbg[5], static_cast<unsigned long long>(tw_need));
      atomicAdd(&g_flow_dbg[6], static_cast<unsigned long long>(tw_rem));
      atomicAdd(&g_flow_dbg[7], static_cast<unsigned long long>(clock64() - th0));
      atomicAdd(&g_flow_dbg[16], static_cast<unsigned long long>(t_post));
      atomicAdd(&g_flow_dbg[19], static_cast<unsigned long long>(t_pa));
      atomicAdd(&g_flow_dbg[20], static_cast<unsigned long long>(t_pb));
      atomicAdd(&g_flow_dbg[21], static_cast<unsigned long long>(t_pc));
      atomicAdd(&g_flow_dbg[22], static_cast<unsigned long long>(t_pd));
      atomicAdd(&g_flow_dbg[17], static_cast<unsigned long long>(n_spun));
      for (int i = 0; i < 4; ++i) {
        atomicAdd(&g_flow_dbg[8 + i], static_cast<unsigned long long>(hpub[i]));
        atomicAdd(&g_flow_dbg[12 + i], static_cast<unsigned long long>(hstart[i]));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < kSRing) {
    const int sl = threadIdx.x;
    if (G > sl) S.base_use[sl] += (G - 1 - sl) / kSRing + 1;
  }
  __syncthreads();
}

// IC(0) apply z = (L L^T)^{-1} r (Ic0Factor::solve) in one CTA; returns the
// CTA sum of r_i z_i in warp 0. rhs(row) yields r_row (and may write it).
template <int TB, bool RING, class Rhs>
__device__ double ic_apply(const DBlock& B, Rhs rhs, double* xf, double* xb, double* red,
                           unsigned* abort_flag, unsigned launch_id = 0, unsigned sweep_no = 0,
                           bool rhs_is_local = true, int part = kBsWhole) {
  double* z = B.z;
  const double* r = B.r;
  double rz = 0.0;
  if (B.exact) {
    sweep(B.fwd, xf, B.n, rhs, [](int, double) {}, abort_flag);
    sweep(
        B.bwd, xb, B.n, [&](int row) { return xf[row]; },
        [&](int row, double zi) {
          z[row] = zi;
          rz += r[row] * zi;
        },
        abort_flag);
    return block_sum(rz, red);
  }
  // staged sweeps: materialize the right-hand side once (it may update r)
  double* bb = B.bb;
  double* y = B.y;
  if constexpr (TB != 0) {
    for (int i = threadIdx.x; i < B.n; i += blockDim.x) bb[i] = rhs(i);
    __syncthreads();
  }
  if constexpr (TB == 0) {
    // blocked sweeps (bsweep.cuh). The tagged right-hand side B.bs_bt was
    // written by the rows' owners (the worker CTAs of every GPU: precond());
    // the stand-alone kernel passes rhs_is_local and writes it here.
    (void)bb;
    const unsigned tag_f = sweep_tag(launch_id, sweep_no), tag_b = sweep_tag(launch_id, sweep_no + 1);
    if (rhs_is_local && part != kBsLists)
      for (int i = threadIdx.x; i < B.n; i += blockDim.x) __stcg(B.bs_bt + i, bs_pack(rhs(i), tag_f));
    const int workers = B.n_remote * static_cast<int>(blockDim.x >> 5);
    bsweep<kBsK>(B.bfwd, xf, B.bs_ns, B.bs_bt, tag_f, nullptr, y,
                 BsFar{B.bs_gt, B.bs_fps, tag_f, workers}, abort_flag, part);
    bsweep<kBsK>(B.bbwd, xf, B.bs_ns, nullptr, tag_b, y, z, BsFar{B.bs_gt, B.bs_fps, tag_b, workers}, abort_flag,
                 part);
    if (part == kBsLists) return 0.0;  // the chain CTA answers
    // <r, z> over the whole block from the tagged right-hand side (complete: the
    // forward sweep has read every entry of it)
    for (int i = threadIdx.x; i < B.n; i += blockDim.x) rz += bs_value(__ldcg(B.bs_bt + i)) * z[i];
    return block_sum(rz, red);
  } else if constexpr (RING) {
    // results go straight to global memory (y, then z)
    const int on = B.n_remote > 0;
    flow_sweep<TB, true>(B.ffwd, B.n, xf, bb, y,
                         FlowRemote{B.rpsum, B.rflag, B.gprog, sweep_tag(launch_id, sweep_no), on},
                         abort_flag);
    flow_sweep<TB, true>(B.fbwd, B.n, xf, y, z,
                         FlowRemote{B.rpsum, B.rflag, B.gprog, sweep_tag(launch_id, sweep_no + 1), on},
                         abort_flag);
    for (int i = threadIdx.x; i < B.n; i += blockDim.x) rz += r[i] * z[i];
    return block_sum(rz, red);
  } else {
    const FlowRemote none{nullptr, nullptr, nullptr, 0u, 0};
    flow_sweep<TB, false>(B.ffwd, B.n, xf, bb, nullptr, none, abort_flag);
    for (int i = threadIdx.x; i < B.n; i += blockDim.x) y[i] = xf[i];
    __syncthreads();
    flow_sweep<TB, false>(B.fbwd, B.n, xf, y, nullptr, none, abort_flag);
    for (int i = threadIdx.x; i < B.n; i += blockDim.x) {
      const double zi = xf[i];
      z[i] = zi;
      rz += r[i] * zi;
    }
    return block_sum(rz, red);
  }
}

// What a remote helper CTA does while the IC CTA runs one IC(0) apply.
__device__ __noinline__ void ic_apply_remote(const DBlock& B, int rank, unsigned* abort_flag, unsigned launch_id,
                                             unsigned sweep_no) {
  if (B.bs) {  // far workers of the blocked sweeps: every warp of this CTA
    const int nw = blockDim.x >> 5, W = B.n_remote * nw, wid = rank * nw + (threadIdx.x >> 5);
    bs_far(B.bfwd, BsFar{B.bs_gt, B.bs_fps, sweep_tag(launch_id, sweep_no), W}, wid, W, abort_flag);
    bs_far(B.bbwd, BsFar{B.bs_gt, B.bs_fps, sweep_tag(launch_id, sweep_no + 1), W}, wid, W, abort_flag);
    return;
  }
  flow_remote(B.ffwd, B.n, B.y,
              FlowRemote{B.rpsum, B.rflag, B.gprog, sweep_tag(launch_id, sweep_no), 1}, rank,
              B.n_remote, abort_flag);
  flow_remote(B.fbwd, B.n, B.z,
              FlowRemote{B.rpsum, B.rflag, B.gprog, sweep_tag(launch_id, sweep_no + 1), 1}, rank,
              B.n_remote, abort_flag);
}

struct Input {
  const double* src0;
  const double* src1;
  double coef;
  double* dst;
  __device__ __forceinline__ double at(int i) const {
    return src1 ? add_rn(src0[i], mul_rn(coef, src1[i])) : src0[i];
  }
  __device__ __forceinline__ const double* materialized() const { return dst ? dst : src0; }
};

struct Ctx {
  const Args& a;
  int cta, G, r0, r1;
  unsigned epoch;
  double* red;
  double* sums;
  double* xf;
  double* xb;
  unsigned* abort_flag;
  unsigned sweeps[2] = {0u, 0u};  // IC(0) sweeps issued per block (same count in every CTA)
  unsigned req[2] = {0u, 0u};     // IC(0) server requests posted per block
  unsigned pi_par = 0u;           // partitioned-inverse applies issued (buffer-set parity)
  int status = DSGPU_OK, failed_block = -1;

  // worker CTAs only: cta / G index the workers (blockIdx.x - n_srv)
  __device__ Ctx(const Args& args, int vblock, int vgrid, double* red_, double* sums_, double* xs)
      : a(args), cta(vblock - args.n_srv), G(vgrid - args.n_srv), epoch(0), red(red_),
        sums(sums_) {
    r0 = a.row_lo[cta];
    r1 = a.row_hi[cta];
    xf = xs;
    xb = xs + a.smem_half;
    abort_flag = a.bar + 64;
  }
  // remote-helper rank of this CTA for block b, or -1
  __device__ int remote_rank(int b) const {
    const DBlock& B = a.blk[b];
    const int k = cta - B.remote_cta0;
    return (B.n_remote > 0 && k >= 0 && k < B.n_remote) ? k : -1;
  }
  __device__ double* part(int slot) {
    return a.partial + (static_cast<size_t>(epoch & 1) * NSLOT + slot) * G;
  }
  // thread 0 of warp 0 publishes a CTA partial (value valid in warp 0)
  __device__ void put(int slot, double v) {
    if (threadIdx.x == 0) part(slot)[cta] = v;
  }
  // grid barrier, then reduce `mask` slots of this epoch into sums[]
  __device__ bool sync_reduce(unsigned mask) {
    PHASE_DIAG(const long long tb0 = clock64();)
    const bool ok = grid_sync(a.bar, a.bar + 32, abort_flag, static_cast<unsigned>(G));
    PHASE_DIAG(if (threadIdx.x == 0) {
      if (cta == 0) {
        atomicAdd(&g_phase_dbg[0], static_cast<unsigned long long>(clock64() - tb0));
        atomicAdd(&g_phase_dbg[3], 1ull);
      }
      if (cta == 1) atomicAdd(&g_phase_dbg[2], static_cast<unsigned long long>(clock64() - tb0));
    })
    if (ok) {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      if (warp < NSLOT && (mask >> warp) & 1u) {
        const double* p = part(warp);
        double s = 0.0;
        for (int c = lane; c < G; c += 32) s += __ldcg(p + c);
        s = warp_sum(s);
        if (lane == 0) sums[warp] = s;
      }
    }
    __syncthreads();
    ++epoch;
    if (ok && a.mg.world > 1) return cross_gpu_reduce(mask);
    return ok;
  }
  // After the local reduction: exchange the per-GPU sums through the peers'
  // mailboxes and add them in rank order (every CTA of every GPU gets the same
  // values). Mailboxes are double-buffered by epoch parity; the epoch word
  // carries the launch id, so nothing has to be reset between launches.
  __device__ bool cross_gpu_reduce(unsigned mask) {
    const MultiGpu& m = a.mg;
    const unsigned ep = (a.launch_id << 20) | (epoch & 0xFFFFFu);
    const int par = static_cast<int>(epoch & 1u);
    if (cta == 0) {
      if (threadIdx.x < NSLOT)
        for (int r = 0; r < m.world; ++r)
          if (r != m.rank)
            *reinterpret_cast<volatile double*>(peer_ptr(m, m.xsum, r) + (par * kMaxWorld + m.rank) * NSLOT + threadIdx.x) =
                sums[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        for (int r = 0; r < m.world; ++r)
          if (r != m.rank) st_release_sys(peer_ptr(m, m.xflag, r) + par * kMaxWorld + m.rank, ep);
      }
    }
    __shared__ int xok_sh;
    if (threadIdx.x == 0) {
      int ok = 1;
      const long long t0 = clock64();
      const unsigned long long w0 = wall_ns();
      for (int r = 0; r < m.world && ok; ++r) {
        if (r == m.rank) continue;
        while (ld_acquire_sys(m.xflag + par * kMaxWorld + r) != ep) {
          if (*reinterpret_cast<volatile unsigned*>(abort_flag) ||
              (clock64() - t0 > kSpinTimeoutCycles && wall_ns() - w0 > g_spin_timeout_ns)) {
            atomicCAS(abort_flag, 0u, kAbortTimeout);
            ok = 0;
            break;
          }
        }
      }
      xok_sh = ok;
    }
    __syncthreads();
    double total = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool mine = warp < NSLOT && ((mask >> warp) & 1u) && lane == 0;
    if (mine)
      for (int r = 0; r < m.world; ++r)
        total += r == m.rank ? sums[warp]
                             : *reinterpret_cast<volatile double*>(m.xsum + (par * kMaxWorld + r) * NSLOT + warp);
    __syncthreads();
    if (mine) sums[warp] = total;
    __syncthreads();
    return xok_sh != 0;
  }
  // Halo: copy the entries of vector v (length-n K' indexing, or block-local)
  // that this rank's rows read but do not own from their owners; then a local
  // grid barrier so every CTA sees them. Call right after a cross-GPU barrier.
  __device__ bool gather_halo(double* v, const int2* halo, int count) {
    const MultiGpu& m = a.mg;
    for (int k = cta * blockDim.x + threadIdx.x; k < count; k += G * blockDim.x) {
      const int2 e = halo[k];
      v[e.x] = *reinterpret_cast<volatile const double*>(peer_ptr(m, v, e.y) + e.x);
    }
    return grid_sync(a.bar, a.bar + 32, abort_flag, static_cast<unsigned>(G));
  }
  // post an IC(0) apply of block b to its server (the lead worker thread);
  // every worker counts the request
  __device__ void post(int b, int op, double alpha, const Input* in) {
    ++req[b];
    if (cta == 0 && threadIdx.x == 0) {
      Mailbox* m = a.mbox + b;
      m->op = op;
      m->alpha = alpha;
      if (in) {
        m->src0 = in->src0;
        m->src1 = in->src1;
        m->coef = in->coef;
        m->dst = in->dst;
      }
      st_release(&m->req, req[b]);
    }
  }
  // wait for the server's answer to the latest request of block b; <r, z>
  __device__ double ic_result(int b) {
    __shared__ double rz_sh;
    __shared__ int ok_sh;
    if (threadIdx.x == 0) {
      Mailbox* m = a.mbox + b;
      int ok = 1;
      const long long t0 = clock64();
      const unsigned long long w0 = wall_ns();
      while (ld_acquire(&m->done) != req[b]) {
        if (*reinterpret_cast<volatile unsigned*>(abort_flag) ||
            (clock64() - t0 > kSpinTimeoutCycles && wall_ns() - w0 > g_spin_timeout_ns)) {
          atomicCAS(abort_flag, 0u, kAbortTimeout);
          ok = 0;
          break;
        }
      }
      __threadfence();
      rz_sh = ok ? *reinterpret_cast<volatile double*>(&m->rz) : 0.0;
      ok_sh = ok;
    }
    __syncthreads();
    if (!ok_sh) status = DSGPU_E_CUDA;
    return rz_sh;
  }
  // one row of block B's residual into every rank's tagged right-hand-side buffer
  __device__ __forceinline__ void push_rhs(const DBlock& B, int li, double v, unsigned tag) const {
    const uint4 w = bs_pack(v, tag);
    __stcg(B.bs_bt + li, w);
    for (int r = 0; r < a.mg.world; ++r)
      if (r != a.mg.rank) __stcg(peer_ptr(a.mg, B.bs_bt, r) + li, w);
  }
  // rows of this CTA inside block b: [lo, hi) in global vector indices
  __device__ void block_rows(int b, int& lo, int& hi) const {
    lo = max(r0, a.blk[b].off);
    hi = min(r1, a.blk[b].off + a.blk[b].n);
  }
};

// Preconditioner application z = M^{-1} rin (BlockDiagPreconditioner::apply,
// precond.cpp:139-148). Writes zout (length n), returns the two guard dots
// <z_b, r_b> in zr[] (identical in all CTAs). False on error.
// Partitioned-inverse IC(0) apply of the active PI blocks by all worker CTAs;
// adds each block's CTA partial of <r, z> to rho_p[b] (warp 0 of the CTA).
template <bool PI>
__device__ void pi_blocks(Ctx& C, const bool act[2], const PiRhs* rhs, double rho_p[2]) {
  if constexpr (PI) {
    const Args& a = C.a;
    extern __shared__ double xs_dyn[];
    double rho0 = 0.0, rho1 = 0.0;
    pi_apply(a.blk[0].pim, a.blk[1].pim, act[0], act[1], rhs[0], rhs[1], a.blk[0].z, a.blk[1].z,
                    C.pi_par & 1u, C.cta, C.G, xs_dyn, C.abort_flag, rho0, rho1);
    ++C.pi_par;
    const bool l0 = (threadIdx.x & 31) == 0;
    if (act[0]) rho_p[0] += block_sum(l0 ? rho0 : 0.0, C.red);
    if (act[1]) rho_p[1] += block_sum(l0 ? rho1 : 0.0, C.red);
  }
}

template <int TB, bool RING, bool PI>
__device__ bool precond(Ctx& C, const Input& in, double* zout, double zr[2],
                        long long inner[2], long long apps[2]) {
  const Args& a = C.a;
  const int tid = threadIdx.x;
  double rho_p[2] = {0.0, 0.0}, zr_p[2] = {0.0, 0.0};
  // ---- S1: r := input; z := M_b^{-1} r; x := 0 -------------------------
  // IC(0) blocks: the block's server CTA computes r and z (requests posted
  // here, answered at the next reduction); ring mode: remote helper CTAs.
  // PI blocks: every CTA joins the partitioned-inverse apply; r (and the
  // materialized input) are written after the reduction, by their owners.
  if constexpr (TB == 0) {
    // blocked sweeps: every worker CTA (of every GPU) writes its rows of the
    // block residual r := input -- plain for its own PCG, tagged into every
    // rank's right-hand-side buffer for the (replicated) sweeps. Tagged units
    // validate themselves: no barrier between this and the sweep.
    for (int b = 0; b < 2; ++b) {
      const DBlock& B = a.blk[b];
      if (B.kind != DSGPU_BLOCK_PCG_IC0) continue;
      int lo, hi;
      C.block_rows(b, lo, hi);
      const unsigned tag = sweep_tag(a.launch_id, C.sweeps[b]);
      for (int i = lo + tid; i < hi; i += blockDim.x) {
        const double ri = in.at(i);
        if (in.dst) in.dst[i] = ri;
        B.r[i - B.off] = ri;
        C.push_rhs(B, i - B.off, ri, tag);
      }
    }
  }
  for (int b = 0; b < 2; ++b)
    if (!PI && a.blk[b].kind == DSGPU_BLOCK_PCG_IC0) C.post(b, IC_OP_S1, 0.0, &in);
  for (int b = 0; b < 2; ++b) {
    const DBlock& B = a.blk[b];
    if constexpr (!PI && RING)
      if (B.kind == DSGPU_BLOCK_PCG_IC0 && C.remote_rank(b) >= 0)
        ic_apply_remote(B, C.remote_rank(b), C.abort_flag, a.launch_id, C.sweeps[b]);
    if (B.kind == DSGPU_BLOCK_PCG_IC0) C.sweeps[b] += 2;
  }
  if constexpr (PI) {
    bool act[2];
    PiRhs rhs[2];
    for (int b = 0; b < 2; ++b) {
      act[b] = a.blk[b].kind == DSGPU_BLOCK_PCG_IC0;
      rhs[b].src0 = in.src0;
      rhs[b].src1 = in.src1;
      rhs[b].coef = in.coef;
      rhs[b].off = a.blk[b].off;
    }
    pi_blocks<PI>(C, act, rhs, rho_p);
  }
  for (int b = 0; b < 2; ++b) {
    const DBlock& B = a.blk[b];
    int lo, hi;
    C.block_rows(b, lo, hi);
    double acc = 0.0;
    for (int i = lo + tid; i < hi; i += blockDim.x) {
      const int li = i - B.off;
      if (B.kind == DSGPU_BLOCK_JACOBI) {
        const double ri = in.at(i);
        if (in.dst) in.dst[i] = ri;
        const double zi = mul_rn(B.dinv[li], ri);
        zout[i] = zi;
        acc += zi * ri;
      } else if (B.kind == DSGPU_BLOCK_PCG_JACOBI) {
        const double ri = in.at(i);
        if (in.dst) in.dst[i] = ri;
        B.r[li] = ri;
        const double zi = mul_rn(B.dinv[li], ri);
        B.z[li] = zi;
        zout[i] = 0.0;
        acc += ri * zi;
      } else {
        zout[i] = 0.0;
      }
    }
    const double s = block_sum(acc, C.red);
    if (B.kind == DSGPU_BLOCK_JACOBI) zr_p[b] = s;
    if (B.kind == DSGPU_BLOCK_PCG_JACOBI) rho_p[b] = s;
  }
  C.put(SL_RHO0, rho_p[0]);
  C.put(SL_RHO1, rho_p[1]);
  C.put(SL_ZR0, zr_p[0]);
  C.put(SL_ZR1, zr_p[1]);
  if (!C.sync_reduce((1u << SL_RHO0) | (1u << SL_RHO1) | (1u << SL_ZR0) | (1u << SL_ZR1)))
    return false;
  if constexpr (PI) {  // deferred: r := input (and the materialized input) for owned rows
    for (int b = 0; b < 2; ++b) {
      const DBlock& B = a.blk[b];
      if (B.kind != DSGPU_BLOCK_PCG_IC0) continue;
      int lo, hi;
      C.block_rows(b, lo, hi);
      for (int i = lo + tid; i < hi; i += blockDim.x) {
        const double ri = in.at(i);
        if (in.dst) in.dst[i] = ri;
        B.r[i - B.off] = ri;
      }
    }
  }

  bool active[2] = {false, false};
  double rho[2] = {0, 0}, rho0[2] = {0, 0}, beta[2] = {0, 0}, alpha[2] = {0, 0};
  int it[2] = {0, 0};
  for (int b = 0; b < 2; ++b) {
    const DBlock& B = a.blk[b];
    if (B.kind == DSGPU_BLOCK_JACOBI) {
      zr[b] = C.sums[SL_ZR0 + b];
      ++apps[b];
      continue;
    }
    rho[b] = (B.kind == DSGPU_BLOCK_PCG_IC0 && !PI) ? C.ic_result(b) : C.sums[SL_RHO0 + b];
    if (C.status != DSGPU_OK) return false;
    if (rho[b] < 0.0) {  // pcg: preconditioner is not positive definite
      C.status = DSGPU_E_INDEFINITE_PRECOND;
      C.failed_block = b;
      return false;
    }
    rho0[b] = rho[b];
    active[b] = rho0[b] != 0.0;
    zr[b] = 0.0;  // x = 0 if the block returns immediately
  }
  const double* rin = in.materialized();
  int pp = 0;  // p ping-pong: read p[pp], write p[pp ^ 1]
  int k = 0;
  while (active[0] || active[1]) {
    // ---- L1: q = A p_new, p_new = z (+ beta p_old) -----------------------
    double kap_p[2] = {0.0, 0.0};
    if (a.mg.world > 1 && k > 0) {  // the other ranks' entries of p_old that these rows read
      for (int b = 0; b < 2; ++b)
        if (active[b] && a.mg.n_halo_p[b] > 0 &&
            !C.gather_halo(pp ? a.blk[b].p1 : a.blk[b].p0, a.mg.halo_p[b], a.mg.n_halo_p[b]))
          return false;
    }
    PHASE_DIAG(const long long tl1 = clock64();)
    {
      const int lane = tid & 31, warp = tid >> 5;
      for (int b = 0; b < 2; ++b) {
        if (!active[b]) continue;
        const DBlock& B = a.blk[b];
        int lo, hi;
        C.block_rows(b, lo, hi);
        PHASE_DIAG(const long long tb1 = clock64();)
        const double* z = B.z;
        const double* po = pp ? B.p1 : B.p0;
        double* pn = pp ? B.p0 : B.p1;
        const double bt = beta[b];
        const bool first = k == 0;
        double acc_k = 0.0;
        const int sub = lane & (B.lanes - 1);
        spmv_rows(
            lo, hi, B.lanes, B.ci, B.v,
            [&](int i, int64_t& s, int& len) {
              const int li = i - B.off;
              s = B.rp[li];
              len = B.na ? B.na[li] : static_cast<int>(B.rp[li + 1] - s);
            },
            [&](int j) { return first ? z[j] : add_rn(z[j], mul_rn(bt, po[j])); },
            [&](int i, bool ok, double acc) {
              if (ok && sub == 0) {
                const int li = i - B.off;
                const double pi = first ? z[li] : add_rn(z[li], mul_rn(bt, po[li]));
                pn[li] = pi;
                B.q[li] = acc;
                acc_k += pi * acc;
              }
            });
        kap_p[b] = block_sum(acc_k, C.red);
        PHASE_DIAG(if (b == 0 && C.cta == 0 && tid == 0 && hi > lo) {
          atomicAdd(&g_spmv_dbg[4], static_cast<unsigned long long>(clock64() - tb1));
          atomicAdd(&g_spmv_dbg[5], 1ull);
          g_spmv_dbg[6] = static_cast<unsigned long long>(B.rp[hi - B.off] - B.rp[lo - B.off]);
        })
      }
    }
    C.put(SL_KAP0, kap_p[0]);
    C.put(SL_KAP1, kap_p[1]);
    if (!C.sync_reduce((1u << SL_KAP0) | (1u << SL_KAP1))) return false;
    PHASE_DIAG(if (active[0] && C.cta == 0 && tid == 0)
                 atomicAdd(&g_spmv_dbg[7], static_cast<unsigned long long>(clock64() - tl1));)
    for (int b = 0; b < 2; ++b) {
      if (!active[b]) continue;
      const double kap = C.sums[SL_KAP0 + b];
      if (kap <= 0.0) {  // pcg: operator is not positive definite
        C.status = DSGPU_E_NEG_CURVATURE;
        C.failed_block = b;
        return false;
      }
      alpha[b] = div_rn(rho[b], kap);
    }
    // ---- L2: r -= alpha q; z = M^{-1} r; x += alpha p -------------------
    double rho_n[2] = {0.0, 0.0}, zr_n[2] = {0.0, 0.0};
    if constexpr (TB == 0) {  // r -= alpha q by the rows' owners, tagged for the sweeps (as in S1)
      for (int b = 0; b < 2; ++b) {
        const DBlock& B = a.blk[b];
        if (!active[b] || B.kind != DSGPU_BLOCK_PCG_IC0) continue;
        int lo, hi;
        C.block_rows(b, lo, hi);
        const unsigned tag = sweep_tag(a.launch_id, C.sweeps[b]);
        const double na = -alpha[b];
        for (int i = lo + tid; i < hi; i += blockDim.x) {
          const int li = i - B.off;
          const double ri = add_rn(B.r[li], mul_rn(na, B.q[li]));
          B.r[li] = ri;
          C.push_rhs(B, li, ri, tag);
        }
      }
    }
    for (int b = 0; b < 2; ++b)
      if (!PI && active[b] && a.blk[b].kind == DSGPU_BLOCK_PCG_IC0) C.post(b, IC_OP_L2, alpha[b], nullptr);
    for (int b = 0; b < 2; ++b) {
      const DBlock& B = a.blk[b];
      if constexpr (!PI && RING)
        if (active[b] && B.kind == DSGPU_BLOCK_PCG_IC0 && C.remote_rank(b) >= 0)
          ic_apply_remote(B, C.remote_rank(b), C.abort_flag, a.launch_id, C.sweeps[b]);
      if (active[b] && B.kind == DSGPU_BLOCK_PCG_IC0) C.sweeps[b] += 2;
    }
    if constexpr (PI) {
      bool act[2];
      PiRhs rhs[2];
      for (int b = 0; b < 2; ++b) {
        act[b] = active[b] && a.blk[b].kind == DSGPU_BLOCK_PCG_IC0;
        rhs[b].r = a.blk[b].r;
        rhs[b].q = a.blk[b].q;
        rhs[b].na = -alpha[b];
      }
      pi_blocks<PI>(C, act, rhs, rho_n);
    }
    for (int b = 0; b < 2; ++b) {
      if (!active[b]) continue;
      const DBlock& B = a.blk[b];
      int lo, hi;
      C.block_rows(b, lo, hi);
      const double* pn = pp ? B.p0 : B.p1;
      const double al = alpha[b], na = -alpha[b];
      double acc_r = 0.0, acc_z = 0.0;
      for (int i = lo + tid; i < hi; i += blockDim.x) {
        const int li = i - B.off;
        if (B.kind == DSGPU_BLOCK_PCG_JACOBI) {
          const double ri = add_rn(B.r[li], mul_rn(na, B.q[li]));
          B.r[li] = ri;
          const double zi = mul_rn(B.dinv[li], ri);
          B.z[li] = zi;
          acc_r += ri * zi;
        }
        const double xi = add_rn(zout[i], mul_rn(al, pn[li]));
        zout[i] = xi;
        acc_z += xi * rin[i];
      }
      const double sr = block_sum(acc_r, C.red);
      const double sz = block_sum(acc_z, C.red);
      if (B.kind == DSGPU_BLOCK_PCG_JACOBI) rho_n[b] = sr;
      zr_n[b] = sz;
    }
    C.put(SL_RHO0, rho_n[0]);
    C.put(SL_RHO1, rho_n[1]);
    C.put(SL_ZR0, zr_n[0]);
    C.put(SL_ZR1, zr_n[1]);
    if (!C.sync_reduce((1u << SL_RHO0) | (1u << SL_RHO1) | (1u << SL_ZR0) | (1u << SL_ZR1)))
      return false;
    if constexpr (PI) {  // deferred: r -= alpha q for owned rows
      for (int b = 0; b < 2; ++b) {
        const DBlock& B = a.blk[b];
        if (!active[b] || B.kind != DSGPU_BLOCK_PCG_IC0) continue;
        int lo, hi;
        C.block_rows(b, lo, hi);
        const double na = -alpha[b];
        for (int i = lo + tid; i < hi; i += blockDim.x) {
          const int li = i - B.off;
          B.r[li] = add_rn(B.r[li], mul_rn(na, B.q[li]));
        }
      }
    }
    for (int b = 0; b < 2; ++b) {
      if (!active[b]) continue;
      const double rn = (a.blk[b].kind == DSGPU_BLOCK_PCG_IC0 && !PI) ? C.ic_result(b) : C.sums[SL_RHO0 + b];
      if (C.status != DSGPU_OK) return false;
      if (rn < 0.0) {
        C.status = DSGPU_E_INDEFINITE_PRECOND;
        C.failed_block = b;
        return false;
      }
      ++it[b];
      zr[b] = C.sums[SL_ZR0 + b];
      if (sqrt_rn(div_rn(rn, rho0[b])) <= a.inner_tol || it[b] >= a.inner_cap) {
        active[b] = false;
      } else {
        beta[b] = div_rn(rn, rho[b]);
        rho[b] = rn;
      }
    }
    pp ^= 1;
    ++k;
  }
  for (int b = 0; b < 2; ++b)
    if (a.blk[b].kind != DSGPU_BLOCK_JACOBI) {
      inner[b] += it[b];
      ++apps[b];
    }
  return true;
}

// IC(0) server CTA of block b: answers the workers' apply requests until told
// to exit. Runs no MINRES code, so the sweep's registers are its own.
// (not inlined: its register allocation stays separate from the MINRES code's)
template <int TB, bool RING>
__device__ __noinline__ void ic_server(const Args& a, int vblock, double* xs, double* red) {
  // bs_pair: server CTAs 2b (chain) and 2b + 1 (lists) are one 2-CTA cluster serving block b
  const int b = (TB == 0 && a.bs_pair) ? vblock >> 1 : vblock;
  const int part = (TB == 0 && a.bs_pair) ? (vblock & 1 ? kBsLists : kBsChain) : kBsWhole;
  const DBlock& B = a.blk[b];
  if (B.kind != DSGPU_BLOCK_PCG_IC0) return;
  Mailbox* m = a.mbox + b;
  unsigned* abort_flag = a.bar + 64;
  __shared__ int op_sh;
  __shared__ double al_sh, coef_sh;
  __shared__ const double* src0_sh;
  __shared__ const double* src1_sh;
  __shared__ double* dst_sh;
  if constexpr (TB == 0) {
    if (!B.exact) bs_setup(xs, B.bs_ns, part);
  } else {
    if (!B.exact) flow_setup<TB>(xs, B.n, B.ffwd.ring);
  }
  for (unsigned seq = 1;; ++seq) {
    if (threadIdx.x == 0) {
      int op = IC_OP_EXIT;
      const long long t0 = clock64();
      const unsigned long long w0 = wall_ns();
      for (;;) {
        if (ld_acquire(&m->req) == seq) {
          op = *reinterpret_cast<volatile int*>(&m->op);
          break;
        }
        if (*reinterpret_cast<volatile unsigned*>(abort_flag)) break;
        if (clock64() - t0 > 4 * kSpinTimeoutCycles && wall_ns() - w0 > 4 * g_spin_timeout_ns) {
          atomicCAS(abort_flag, 0u, kAbortTimeout);  // workers gone: give up
          break;
        }
      }
      op_sh = op;
      al_sh = *reinterpret_cast<volatile double*>(&m->alpha);
      src0_sh = m->src0;
      src1_sh = m->src1;
      coef_sh = m->coef;
      dst_sh = m->dst;
    }
    __syncthreads();
    const int op = op_sh;
    if (op == IC_OP_EXIT) break;
    PHASE_DIAG(const long long ti0 = clock64();)
    const unsigned sweep_no = 2 * (seq - 1);
    double rz;
    if (op == IC_OP_S1) {
      const double* src0 = src0_sh;
      const double* src1 = src1_sh;
      const double coef = coef_sh;
      double* dst = dst_sh;
      double* r = B.r;
      const int off = B.off;
      rz = ic_apply<TB, RING>(
          B,
          [&](int row) {
            const int i = off + row;
            const double ri = src1 ? add_rn(src0[i], mul_rn(coef, src1[i])) : src0[i];
            if (dst) dst[i] = ri;
            r[row] = ri;
            return ri;
          },
          xs, xs + a.smem_half, red, abort_flag, a.launch_id, sweep_no, TB != 0, part);
    } else {
      double* r = B.r;
      const double* q = B.q;
      const double na = -al_sh;
      rz = ic_apply<TB, RING>(
          B,
          [&](int row) {
            const double ri = add_rn(r[row], mul_rn(na, q[row]));
            r[row] = ri;
            return ri;
          },
          xs, xs + a.smem_half, red, abort_flag, a.launch_id, sweep_no, TB != 0, part);
    }
    __syncthreads();  // every thread's r, z (and dst) written
    if (threadIdx.x == 0 && part != kBsLists) {
      m->rz = rz;
      __threadfence();
      st_release(&m->done, seq);
      PHASE_DIAG(atomicAdd(&g_phase_dbg[b == 0 ? 1 : 5], static_cast<unsigned long long>(clock64() - ti0));)
    }
  }
  if constexpr (TB == 0) {
    if (part != kBsWhole && !B.exact) bs_cluster_sync();  // neither CTA leaves while the other may still store into it
  }
}

// MINRES vector recurrences of one row (solvers.cpp:93-101, one fused pass):
// w = (v - oldeps w1 - delta w2) / gamma and the same for aw = K w; x += phi w;
// res -= phi aw. Returns res_i^2 (the caller's ||res|| reduction). Rounds like
// the reference's scalar C++ (explicit mul/add/div, no FMA contraction).
__device__ __forceinline__ double minres_update_row(int i, const double* v, const double* av, const double* w1,
                                                    const double* w2, const double* aw1, const double* aw2,
                                                    double* wn, double* awn, double* x, double* res,
                                                    double oldeps, double delta, double gamma, double phi) {
  const double wv = div_rn(sub_rn(sub_rn(v[i], mul_rn(oldeps, w1[i])), mul_rn(delta, w2[i])), gamma);
  const double awv = div_rn(sub_rn(sub_rn(av[i], mul_rn(oldeps, aw1[i])), mul_rn(delta, aw2[i])), gamma);
  wn[i] = wv;
  awn[i] = awv;
  x[i] = add_rn(x[i], mul_rn(phi, wv));
  const double rv = add_rn(res[i], mul_rn(-phi, awv));
  res[i] = rv;
  return rv * rv;
}

// Warm start (MinresOptions::x0): r1 = res = b - K x0 for the rows [r0, r1) of this
// CTA; returns the thread's share of ||r1||^2. Out of line: it runs once per
// solve and must not cost the solve loop a register.
__device__ __noinline__ double warm_residual(const Args& a, int r0, int r1, double* bvec) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = a.k_lanes, sub = lane & (L - 1), ng = kWarps * (32 / L);
  const int gid = warp * (32 / L) + lane / L;
  const double* x0v = a.x;
  double acc = 0.0;
  for (int base = r0; base < r1; base += ng) {
    const int i = base + gid;
    const bool ok = i < r1;
    double kx = 0.0;
    if (ok) {
      const int64_t ks = a.k_rp[i];
      kx = row_partial(a.k_ci + ks, a.k_v + ks, static_cast<int>(a.k_rp[i + 1] - ks), sub, L,
                       [&](int j) { return x0v[j]; });
    }
    kx = group_sum(kx, L);
    if (ok && sub == 0) {
      const double ri = sub_rn(bvec[i], kx);
      bvec[i] = ri;
      a.res[i] = ri;
      acc += ri * ri;
    }
  }
  return acc;
}

// The whole solve as seen by CTA `vblock` of a grid of `vgrid` CTAs (the real
// grid for minres_kernel; one rank's share of the grid for the multi-rank
// emulation kernel below).
template <int TB, bool RING, bool PI, bool WARM = false>
__device__ __forceinline__ void minres_body(const Args& a, int vblock, int vgrid) {
  extern __shared__ double xs_dyn[];
  __shared__ double red[32];
  __shared__ double sums[NSLOT];
  if constexpr (!PI) {  // (the PI variant must not even instantiate the sweeps)
    if (vblock < a.n_srv) {
      ic_server<TB, RING>(a, vblock, xs_dyn, red);
      return;
    }
  }
  if (PI) pi_prologue();
  Ctx C(a, vblock, vgrid, red, sums, xs_dyn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  PHASE_DIAG(const long long t_kernel0 = clock64();)
  const int r0 = C.r0, r1 = C.r1;
  long long inner[2] = {0, 0}, apps[2] = {0, 0};
  int iterations = 0, converged = 0, hist_len = 0;
  double relres_m = 1.0, relres_e = 1.0;
  const bool writer = (C.cta == 0 && tid == 0);

  // ---- P0: b = [f'; 0]; x = x0 (or 0); r1 = res = b - K x0; w* = aw* = 0; ||res||^2
  // (solvers.cpp:29-42)
  double* bvec = a.rbuf[0];
  {
    // (a separate instantiation: the cold kernel's code -- and its register
    // allocation -- carry no trace of the warm start)
    constexpr bool warm = WARM;
    double acc = 0.0;
    for (int i = r0 + tid; i < r1; i += blockDim.x) {
      const double bi = i < a.n_u ? a.f_in[a.perm_u[i]] : 0.0;
      bvec[i] = bi;
      a.res[i] = bi;
      a.x[i] = warm ? (i < a.n_u ? a.u0_in[a.perm_u[i]] : a.p0_in[a.perm_p[i - a.n_u]]) : 0.0;
      a.w[0][i] = a.w[1][i] = a.w[2][i] = 0.0;
      a.aw[0][i] = a.aw[1][i] = a.aw[2][i] = 0.0;
      if (!warm) acc += bi * bi;
    }
    if constexpr (warm) {  // r1 = b - K x0 once every CTA's part of x0 is in place
      if (!C.sync_reduce(0u)) goto finish;
      acc = warm_residual(a, r0, r1, bvec);
    }
    C.put(SL_BB, block_sum(acc, red));
    if (PI)  // both partitioned-inverse buffer sets start out "not yet computed"
      for (int b = 0; b < 2; ++b)
        if (a.blk[b].pi)
          for (int s = 0; s < 2; ++s) {
            unsigned long long* o = reinterpret_cast<unsigned long long*>(a.blk[b].pim.set[s]);
            for (int k = C.cta * blockDim.x + tid; k < 4 * a.blk[b].pim.n; k += C.G * blockDim.x) o[k] = kSentinel;
          }
  }
  if (!C.sync_reduce(1u << SL_BB)) goto finish;
  {
    const double rnorm0 = sqrt_rn(sums[SL_BB]);
    double* r1v = a.rbuf[0];
    double* r2v = a.rbuf[0];
    double* spare = a.rbuf[1];
    double* free4 = a.rbuf[2];
    double* y = a.y;
    double zr[2];
    if (!precond<TB, RING, PI>(C, Input{r1v, nullptr, 0.0, nullptr}, y, zr, inner, apps)) goto finish;
    if (zr[0] < 0.0 || zr[1] < 0.0) {  // BlockDiagPreconditioner guards
      C.status = DSGPU_E_INDEFINITE_PRECOND;
      C.failed_block = zr[0] < 0.0 ? 0 : 1;
      goto finish;
    }
    double beta1 = zr[0] + zr[1];
    if (beta1 < 0.0) {
      C.status = DSGPU_E_INDEFINITE_PRECOND;
      goto finish;
    }
    beta1 = sqrt_rn(beta1);
    if (writer && a.hist_cap > 0) {
      a.hist_m[0] = 1.0;
      a.hist_e[0] = 1.0;
    }
    hist_len = 1;
    if (beta1 == 0.0) {
      converged = 1;
      goto finish;
    }
    if (a.max_iter == 0) goto finish;  // x = x0 = 0, no iteration (solvers.cpp:62)
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1;
    double cs = -1.0, sn = 0.0, oldeps = 0.0;
    double delta = 0.0, gamma = 1.0, phi = 0.0;
    int wi = 0;  // w[wi] = current w; rotation per reference swaps
    bool pending = false;
    bool do_spmv = true;
    PHASE_DIAG(long long tm1 = 0;)
    for (int it = 1;; ++it) {
      // ---- M1: finish iteration it-1 (vector recurrences) + SpMV of it --
      double acc_res = 0.0, acc_alpha = 0.0;
      if (pending) {
        // w1<->w2, w2<->w  =>  w1 = old w2, w2 = old w, w = old w1
        const int iw = wi, iw1 = (wi + 1) % 3, iw2 = (wi + 2) % 3;  // current roles
        const int nw = iw1;            // new w reuses old w1's buffer
        const double* w1 = a.w[iw2];   // new w1 = old w2
        const double* w2 = a.w[iw];    // new w2 = old w
        double* wn = a.w[nw];
        const double* aw1 = a.aw[iw2];
        const double* aw2 = a.aw[iw];
        double* awn = a.aw[nw];
        wi = nw;
        for (int i = r0 + tid; i < r1; i += blockDim.x)
          acc_res += minres_update_row(i, a.v, a.av, w1, w2, aw1, aw2, wn, awn, a.x, a.res, oldeps, delta,
                                       gamma, phi);
        C.put(SL_RES, block_sum(acc_res, red));
      }
      if (do_spmv && a.mg.world > 1 && !C.gather_halo(y, a.mg.halo_y, a.mg.n_halo_y)) goto finish;
      if (do_spmv) {
        const double s = div_rn(1.0, beta);
        const double c1 = it >= 2 ? div_rn(-beta, oldb) : 0.0;
        for (int i = r0 + tid; i < r1; i += blockDim.x) a.v[i] = mul_rn(s, y[i]);
        __syncthreads();  // old av consumed above before the new av is written
        // (one trip per lane in flight: the pipelined spmv_rows of the inner SpMV measured
        // slower here -- C3 152 -> 181 us, C4 294 -> 302 us per phase, profiles/r02_phases_spmv.md)
        const int L = a.k_lanes, sub = lane & (L - 1), ng = kWarps * (32 / L);
        const int gid = warp * (32 / L) + lane / L;
        PHASE_DIAG(tm1 = clock64();)
        for (int base = r0; base < r1; base += ng) {
          const int i = base + gid;
          const bool ok = i < r1;
          double acc = 0.0;
          if (ok) {
            const int64_t ks = a.k_rp[i];
            acc = row_partial(a.k_ci + ks, a.k_v + ks, static_cast<int>(a.k_rp[i + 1] - ks), sub, L,
                              [&](int j) { return mul_rn(s, y[j]); });
          }
          acc = group_sum(acc, L);
          if (ok && sub == 0) {
            a.av[i] = acc;
            const double t = it >= 2 ? add_rn(acc, mul_rn(c1, r1v[i])) : acc;
            spare[i] = t;
            acc_alpha += mul_rn(s, y[i]) * t;
          }
        }
        C.put(SL_ALPHA, block_sum(acc_alpha, red));
        PHASE_DIAG(if (writer) {
          atomicAdd(&g_spmv_dbg[0], static_cast<unsigned long long>(clock64() - tm1));
          atomicAdd(&g_spmv_dbg[1], 1ull);
          g_spmv_dbg[2] = static_cast<unsigned long long>(a.k_rp[r1] - a.k_rp[r0]);
        })
      }
      if (!C.sync_reduce((pending ? (1u << SL_RES) : 0u) | (do_spmv ? (1u << SL_ALPHA) : 0u)))
        goto finish;
      PHASE_DIAG(if (writer && do_spmv) atomicAdd(&g_spmv_dbg[3], static_cast<unsigned long long>(clock64() - tm1));)
      if (pending) {
        // stop test of iteration it-1 (solvers.cpp:102-117)
        relres_e = rnorm0 > 0.0 ? div_rn(sqrt_rn(sums[SL_RES]), rnorm0) : 0.0;
        iterations = it - 1;
        if (writer && hist_len < a.hist_cap) {
          a.hist_m[hist_len] = relres_m;
          a.hist_e[hist_len] = relres_e;
        }
        ++hist_len;
        const double stop_value = a.stop_euclid ? relres_e : relres_m;
        if (stop_value <= a.outer_tol) {
          converged = 1;
          break;
        }
        if (beta == 0.0) {
          converged = relres_m <= a.outer_tol;
          break;
        }
        if (!do_spmv) break;  // max_iter reached
      }
      const double alfa = sums[SL_ALPHA];
      // ---- precond: r2_new = spare - (alfa/beta) r2;  y = M^{-1} r2_new ----
      if (!precond<TB, RING, PI>(C, Input{spare, r2v, div_rn(-alfa, beta), spare}, y, zr, inner, apps))
        goto finish;
      {
        double* nr1 = r2v;
        double* nr2 = spare;
        double* nsp = (r1v != r2v) ? r1v : free4;
        r1v = nr1;
        r2v = nr2;
        spare = nsp;
      }
      if (zr[0] < 0.0 || zr[1] < 0.0) {
        C.status = DSGPU_E_INDEFINITE_PRECOND;
        C.failed_block = zr[0] < 0.0 ? 0 : 1;
        goto finish;
      }
      oldb = beta;
      const double betasq = zr[0] + zr[1];
      if (betasq < 0.0) {
        C.status = DSGPU_E_INDEFINITE_PRECOND;
        goto finish;
      }
      beta = sqrt_rn(betasq);
      // Givens (solvers.cpp:79-91)
      oldeps = epsln;
      delta = add_rn(mul_rn(cs, dbar), mul_rn(sn, alfa));
      const double gbar = sub_rn(mul_rn(sn, dbar), mul_rn(cs, alfa));
      epsln = mul_rn(sn, beta);
      dbar = mul_rn(-cs, beta);
      gamma = sqrt_rn(add_rn(mul_rn(gbar, gbar), mul_rn(beta, beta)));
      gamma = fmax(gamma, 2.220446049250313e-16);
      cs = div_rn(gbar, gamma);
      sn = div_rn(beta, gamma);
      phi = mul_rn(cs, phibar);
      phibar = mul_rn(sn, phibar);
      relres_m = div_rn(phibar, beta1);
      pending = true;
      do_spmv = (it < a.max_iter) && beta != 0.0;
      if (it >= a.max_iter) iterations = it;
    }
  }
finish:
  // ---- F: zero-mean pressure filter + un-permute -------------------------
  {
    double mean = 0.0;
    if (a.filter && C.status == DSGPU_OK) {
      double acc = 0.0;
      const int lo = max(r0, a.n_u);
      for (int i = lo + tid; i < r1; i += blockDim.x) acc += a.qk[i - a.n_u] * a.x[i];
      C.put(SL_NUM, block_sum(acc, red));
      if (C.sync_reduce(1u << SL_NUM)) mean = div_rn(sums[SL_NUM], a.filter_den);
    }
    for (int i = r0 + tid; i < r1; i += blockDim.x) {
      if (i < a.n_u)
        a.u_out[a.perm_u[i]] = a.x[i];
      else
        a.p_out[a.perm_p[i - a.n_u]] = a.filter ? sub_rn(a.x[i], mul_rn(mean, 1.0)) : a.x[i];
    }
  }
  PHASE_DIAG(if (threadIdx.x == 0 && C.cta == 0)
               atomicAdd(&g_phase_dbg[4], static_cast<unsigned long long>(clock64() - t_kernel0));)
  if (writer && !PI)  // release the IC(0) servers
    for (int b = 0; b < 2; ++b)
      if (a.blk[b].kind == DSGPU_BLOCK_PCG_IC0) {
        a.mbox[b].op = IC_OP_EXIT;
        st_release(&a.mbox[b].req, C.req[b] + 1);
      }
  if (writer) {
    DevReport* R = a.rep;
    R->iterations = iterations;
    R->converged = converged;
    R->status = C.status;
    R->failed_block = C.failed_block;
    R->hist_len = hist_len;
    R->relres_m = relres_m;
    R->relres_e = relres_e;
    R->inner[0] = inner[0];
    R->inner[1] = inner[1];
    R->apps[0] = apps[0];
    R->apps[1] = apps[1];
    const unsigned ab = *reinterpret_cast<volatile unsigned*>(a.bar + 64);
    if (ab) R->status = ab == kAbortTimeout ? DSGPU_E_TIMEOUT : DSGPU_E_CUDA;
  }
}

template <int TB, bool RING, bool PI, bool WARM = false>
__global__ void __launch_bounds__(kThreads, 1) minres_kernel(const __grid_constant__ Args a) {
  minres_body<TB, RING, PI, WARM>(a, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
}

// Multi-rank emulation on ONE GPU (tests of the multi-GPU data plane where
// only one GPU exists): a single cooperative launch whose grid is `world`
// consecutive groups of `per_rank` CTAs; group r runs rank r's solve with rank
// r's argument block, and the "peer" arenas are the other groups' arenas in the
// same address space. All CTAs are co-resident (cooperative launch), so the
// cross-rank waits make progress exactly as they do across GPUs.
__global__ void __launch_bounds__(kThreads, 1) minres_emul_kernel(const Args* all, int per_rank) {
  const int r = static_cast<int>(blockIdx.x) / per_rank;
  minres_body<0, true, false>(all[r], static_cast<int>(blockIdx.x) % per_rank, per_rank);
}

// ---- standalone kernels (parity / microbenchmarks) -------------------------
template <int TB, bool RING>
__global__ void __launch_bounds__(kThreads, 1)
    ic_apply_kernel(const __grid_constant__ DBlock B, const double* r, unsigned* abort_flag,
                    unsigned launch_id, int pair) {
  extern __shared__ double xs_dyn[];
  __shared__ double red[32];
  // B.r = r (input), B.z = output, B.y = forward-sweep scratch (set by the host).
  // Ring mode: the CTAs after the sweep CTA (pair: after the sweep CTA pair, a
  // 2-CTA cluster as in the solve) are the remote helpers / far workers.
  const int lead = (TB == 0 && pair) ? 2 : 1;
  if (RING && static_cast<int>(blockIdx.x) >= lead) {
    ic_apply_remote(B, blockIdx.x - lead, abort_flag, launch_id, 0u);
    return;
  }
  const int part = (TB == 0 && pair) ? (blockIdx.x ? kBsLists : kBsChain) : kBsWhole;
  if constexpr (TB == 0) {
    if (!B.exact) bs_setup(xs_dyn, B.bs_ns, part);
  } else {
    if (!B.exact) flow_setup<TB>(xs_dyn, B.n, B.ffwd.ring);
  }
  ic_apply<TB, RING>(B, [&](int row) { return r[row]; }, xs_dyn, xs_dyn + B.n, red, abort_flag,
                     launch_id, 0u, true, part);
  if constexpr (TB == 0) {
    if (part != kBsWhole) bs_cluster_sync();
  }
}

// One partitioned-inverse IC(0) apply z = (L L^T)^{-1} r of one block by all
// CTAs (cooperative launch); the buffer set `par` must hold sentinels.
__global__ void __launch_bounds__(kThreads, 1)
    pi_apply_kernel(const __grid_constant__ DPi P, const double* r, double* z, unsigned par, unsigned* abort_flag) {
  extern __shared__ double xs_dyn[];
  pi_prologue();
  PiRhs rhs;
  rhs.src0 = r;
  double rho0 = 0.0, rho1 = 0.0;
  pi_apply(P, DPi{}, true, false, rhs, rhs, z, nullptr, par, blockIdx.x, gridDim.x, xs_dyn, abort_flag, rho0,
                  rho1);
}

__global__ void fill_sentinel(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    reinterpret_cast<unsigned long long*>(p)[i] = kSentinel;
}

using MinresFn = void (*)(Args);
using IcFn = void (*)(DBlock, const double*, unsigned*, unsigned, int);
// warm: the instantiation that starts from an initial guess (blocked sweeps and
// partitioned inverse only -- the modes the policy selects; nullptr otherwise)
MinresFn minres_for(int tb, bool ring, bool pi, bool warm = false) {
  if (warm) {
    if (tb == 0) return minres_kernel<0, true, false, true>;
    if (pi) return minres_kernel<8, false, true, true>;
    return nullptr;
  }
  if (tb == 0) return minres_kernel<0, true, false>;  // blocked sweeps
  if (pi) return minres_kernel<8, false, true>;
  if (ring) return tb <= 8 ? minres_kernel<8, true, false> : minres_kernel<16, true, false>;
  return tb <= 8 ? minres_kernel<8, false, false> : minres_kernel<16, false, false>;
}
IcFn ic_for(int tb, bool ring) {
  if (tb == 0) return ic_apply_kernel<0, true>;  // blocked sweeps
  if (ring) return tb <= 8 ? ic_apply_kernel<8, true> : ic_apply_kernel<16, true>;
  return tb <= 8 ? ic_apply_kernel<8, false> : ic_apply_kernel<16, false>;
}

// y = M x, warp per row; na != nullptr limits each row to its first na[i] entries
// (padded rows, L lanes per row: row_partial in kernels.cuh; launch with
// spmv_grid(n_rows, L) CTAs of 256 threads)
__global__ void spmv_kernel(int n_rows, const int64_t* rp, const int32_t* ci, const double* v,
                            const int32_t* na, const double* x, double* y, int L) {
  const int lane = threadIdx.x & 31, sub = lane & (L - 1);
  const int row = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L);
  const bool ok = row < n_rows;
  double acc = 0.0;
  if (ok) {
    const int64_t s = rp[row];
    const int len = na ? na[row] : static_cast<int>(rp[row + 1] - s);
    acc = row_partial(ci + s, v + s, len, sub, L, [&](int j) { return x[j]; });
  }
  acc = group_sum(acc, L);
  if (ok && sub == 0) y[row] = acc;
}
inline unsigned spmv_grid(int n_rows, int L) {
  return static_cast<unsigned>((static_cast<int64_t>(n_rows) * L + 255) / 256);
}

// Stand-alone form of the persistent kernel's fused MINRES vector pass (the
// roofline measurement of part (3)/(4) of the hot path): minres_update_row over
// all rows + the ||res||^2 warp-shuffle / block reduction, one partial per CTA.
// 12 vectors streamed once: 8 reads + 4 writes = 96 bytes per row.
__global__ void __launch_bounds__(kThreads) minres_vec_kernel(int n, const double* v, const double* av,
                                                              const double* w1, const double* w2,
                                                              const double* aw1, const double* aw2, double* wn,
                                                              double* awn, double* x, double* res,
                                                              double* partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc += minres_update_row(i, v, av, w1, w2, aw1, aw2, wn, awn, x, res, 0.25, 0.5, 1.5, 1e-3);
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void gather_kernel(int n, const int32_t* perm, const double* src, double* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}
__global__ void scatter_kernel(int n, const int32_t* perm, const double* src, double* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[perm[i]] = src[i];
}

// ---- device memory -----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct dsgpu_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  bool ready = false;
  HostPlan plan;
  std::vector<DevBuf> bufs;
  Args args{};
  int grid = 0;
  size_t smem = 0;
  int64_t levels[4] = {0, 0, 0, 0};
  double* d_f = nullptr;
  double* d_u = nullptr;
  double* d_p = nullptr;
  double* d_tmp[3] = {nullptr, nullptr, nullptr};
  DevReport* d_rep = nullptr;
  int64_t nnz_k = 0, nnz_a = 0, nnz_l[2] = {0, 0}, nnz_q = 0;
  bool exact = false;
  bool ring = false;
  bool pi = false;            // partitioned-inverse IC(0) applies (pi.cuh)
  bool bs = false;            // blocked sweeps (bsweep.cuh)
  bool force_pi = false;      // the early model chose the partitioned inverse
  int bs_ns = kBsK + 3;       // dense-block slot ring depth (minimum K + 3: the second main warp looks K groups ahead)
  double *d_u0 = nullptr, *d_p0 = nullptr;  // initial guess of the next solve (dsgpu_set_initial_guess)
  bool warm = false;
  bool bs_pair = false;       // the solve's IC(0) servers are CTA pairs (2-CTA clusters; DSGPU_BS_PAIR=0: single CTAs)
  int far_ctas[2] = {0, 0};   // far-worker CTAs per IC block
  PiPlan pip[2];
  int pi_cbase = 0, pi_cslot = 0;  // chain coefficient prefetch slots (doubles)
  int pi_steps = 0;           // dependent chain steps per IC(0) apply (both sweeps)
  int tb = 4, merge = 1;
  int remote_max = 8;         // remote helper CTAs per IC block (ring mode)
  int sms = 148;
  unsigned launch_id = 0;     // 1..4095, cycled per launch (sweep tags)
  unsigned next_launch_id() {
    launch_id = launch_id % (world > 1 ? 2047u : 4095u) + 1u;
    return launch_id;
  }
  // Solves of a multi-GPU handle take their ids from their own counter (upper
  // half of the 12-bit id space): the ranks' tags and reduction epochs agree as
  // long as every rank has made the same number of SOLVE calls, whatever
  // stand-alone kernels each rank ran in between.
  unsigned solve_id = 0;
  unsigned next_solve_id() {
    if (world == 1) return next_launch_id();
    solve_id = solve_id % 2047u + 1u;
    return 2048u + solve_id;
  }

  // multi-GPU (dsgpu_create_multi): this rank, the world size, and the arena --
  // ONE allocation holding every buffer another rank reads or writes (the
  // iterate y, the PCG directions, the tagged right-hand sides, the reduction
  // mailboxes), exported to the peers as one CUDA IPC handle; the same layout
  // on every rank, so a peer's copy of a buffer sits at the same offset.
  int rank = 0, world = 1;
  char* arena = nullptr;
  size_t arena_size = 0, arena_used = 0;
  void* peer_arena[kMaxWorld] = {};
  bool peers_open = false;
  template <class T>
  T* arena_alloc(size_t count) {
    const size_t bytes = (std::max<size_t>(count, 1) * sizeof(T) + 255) / 256 * 256;
    if (!arena || arena_used + bytes > arena_size) throw std::runtime_error("arena exhausted");
    T* p = reinterpret_cast<T*>(arena + arena_used);
    arena_used += bytes;
    return p;
  }
  template <class T>
  T* alloc(size_t count) {
    DevBuf b;
    b.bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (cudaMalloc(&b.p, b.bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    bufs.push_back(b);
    return static_cast<T*>(b.p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* d = alloc<T>(v.size());
    if (!v.empty() &&
        cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      throw std::runtime_error("cudaMemcpy H2D failed");
    return d;
  }
  void free_all() {
    if (peers_open)
      for (int r = 0; r < world; ++r)
        if (r != rank && peer_arena[r]) cudaIpcCloseMemHandle(peer_arena[r]);
    peers_open = false;
    for (auto& p : peer_arena) p = nullptr;
    for (auto& b : bufs) cudaFree(b.p);
    bufs.clear();
    d_u0 = d_p0 = nullptr;
    warm = false;
    arena = nullptr;
    arena_size = arena_used = 0;
    ready = false;
  }
};

namespace {

thread_local std::string g_err;

int fail(dsgpu_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return code;
}

int cuda_check(dsgpu_handle* h, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DSGPU_OK;
  return fail(h, DSGPU_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

DFlow upload_flow(dsgpu_handle* h, const HostFlow& f) {
  DFlow d{};
  d.G = f.G;
  d.nr = h->upload(f.nr);
  d.cptr = h->upload(f.cptr);
  d.cneed = h->upload(f.cneed);
  d.pw = h->upload(f.pw);
  d.grows = h->upload(f.grows);
  d.pcols = h->upload(f.pcols);
  d.pptr = h->upload(f.pptr);
  d.pvals = h->upload(f.pvals);
  d.ww = h->upload(f.ww);
  d.stat = h->upload(f.stat);
  d.ring = f.ring;
  d.gw = h->upload(f.gw);
  d.gneed = h->upload(f.gneed);
  d.gptr = h->upload(f.gptr);
  d.gcols = h->upload(f.gcols);
  d.gvals = h->upload(f.gvals);
  d.wptr = h->upload(f.wptr);
  d.wcols = h->upload(f.wcols);
  d.wvals = h->upload(f.wvals);
  // remote split: lists of >= 4 chunks per group on average get kRSplit warps,
  // short ones 1 (a split only adds flags to wait on); DSGPU_RSPLIT overrides
  double chunks = 0.0;
  for (const int32_t w : f.gw) chunks += w / 16.0;
  chunks /= std::max(1, f.G);
  d.rsplit = chunks >= 4.0 ? kRSplit : 1;
  if (const char* env = std::getenv("DSGPU_RSPLIT"))
    d.rsplit = std::min(kRSplit, std::max(1, std::atoi(env)));
  return d;
}

DBSweep upload_bsweep(dsgpu_handle* h, HostBSweep& s) {
  DBSweep d{};
  d.n = s.n;
  d.G = s.G;
  d.dir = s.dir;
  d.slots = h->upload(s.slots);
  d.tblk = h->upload(s.tblk);
  d.mw = h->upload(s.mw);
  d.ms = h->upload(s.ms);
  d.mptr = h->upload(s.mptr);
  d.mcols = h->upload(s.mcols);
  d.mvals = h->upload(s.mvals);
  d.fw = h->upload(s.fw);
  d.fptr = h->upload(s.fptr);
  d.fcols = h->upload(s.fcols);
  d.fvals = h->upload(s.fvals);
  d.fcptr = h->upload(s.fcptr);
  d.fneed = h->upload(s.fneed);
  // the device copy is the plan from here on (96^3: 13 GB of lists per sweep)
  std::vector<uint8_t>().swap(s.slots);
  std::vector<uint8_t>().swap(s.tblk);
  std::vector<int32_t>().swap(s.mcols);
  std::vector<double>().swap(s.mvals);
  std::vector<int32_t>().swap(s.fcols);
  std::vector<double>().swap(s.fvals);
  return d;
}

// Dynamic shared memory limit of a kernel: raised once to the device maximum
// (the attribute belongs to the function, not to a handle: a per-handle value
// would be lowered by the next, smaller system's setup).
cudaError_t raise_smem_limit(const void* fn, int smem_optin) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const int want = smem_optin - static_cast<int>(fa.sharedSizeBytes);
  if (fa.maxDynamicSharedSizeBytes >= want) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
}

DSweep upload_sweep(dsgpu_handle* h, const HostSweep& s) {
  DSweep d{};
  d.n_groups = s.n_groups;
  d.gptr = h->upload(s.gptr);
  d.gwidth = h->upload(s.gwidth);
  d.grows = h->upload(s.grows);
  d.cols = h->upload(s.cols);
  d.vals = h->upload(s.vals);
  d.diag = h->upload(s.diag);
  return d;
}

// Partitioned-inverse mode (pi.hpp) for the IC(0) blocks. Block size = the
// factor's lower bandwidth x m, with m the candidate (0.5, 1, 1.5; DSGPU_PI_B
// fixes it) of least modelled apply time; the pressure block is cut into no
// more blocks than the velocity block so both chains share steps. Off (staged
// sweeps) when DSGPU_PI=0, when the windows do not fit shared memory, when the
// block inverses would exceed half the free HBM, or when the cost model
// predicts the staged sweeps to be competitive. DSGPU_PI=1 skips the model.
//
// Cost model (B200, measured: profiles/r01_configs_c3_c4.jsonl,
// r01_knobs_c3_pib.jsonl, r01_ic_ncu_c3_c4.md). A PI apply streams every
// coefficient once (both blocks' chains run together, 3.9 TB/s measured by
// ncu at C3) and pays a latency per chain step; a staged sweep pays per
// dependency level and the two blocks' sweeps run concurrently:
//   t_pi     = 8 n_coef / 3.9 TB/s + 2 us x steps
//   t_staged = 0.6 us x max_b (levels_fwd + levels_bwd)
// PI when t_pi < 0.7 t_staged: C2 (m = 1.5: 58 steps, latency-bound), C3
// (m = 0.5: 2.0 ms per velocity apply vs 3.1 ms at m = 1.5 and 8.6 ms
// staged); not C4/C5 (3D, lower bandwidth 23k+: tens of GB of block inverses;
// C4 PI 14 ms per apply vs 14.5 ms staged, staged solve 1.4x faster).
bool choose_pi(dsgpu_handle* h, const HostPlan& P, size_t smem_budget) {
  bool force = h->force_pi;
  if (const char* env = std::getenv("DSGPU_PI")) {
    if (std::atoi(env) == 0) return false;
    force = true;
  }
  std::vector<double> mults = {0.5, 1.0, 1.5};
  if (const char* env = std::getenv("DSGPU_PI_B")) mults = {std::atof(env)};
  double staged_levels = 0.0;
  int bw[2] = {0, 0};
  for (int b = 0; b < 2; ++b) {
    const HostBlock& hb = P.blk[b];
    if (hb.kind != DSGPU_BLOCK_PCG_IC0) continue;
    staged_levels = std::max(staged_levels, static_cast<double>(hb.fwd.n_levels + hb.bwd.n_levels));
    bw[b] = pi_bandwidth(hb.n, hb.lrp.data(), hb.lci.data());
  }
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  double best = 0.0;
  bool found = false;
  for (const double mult : mults) {
    PiPlan pp[2];
    int nb0 = 0;
    size_t bytes = 0;
    for (int b = 0; b < 2; ++b) {
      const HostBlock& hb = P.blk[b];
      if (hb.kind != DSGPU_BLOCK_PCG_IC0) continue;
      int bsz = std::max(1, static_cast<int>(std::ceil(std::max(1, bw[b]) * mult)));
      if (b == 1 && nb0 > 0) bsz = std::max(bsz, (hb.n + nb0 - 1) / nb0);
      pp[b] = pi_plan(hb.n, hb.lrp.data(), hb.lci.data(), bsz);
      if (b == 0) nb0 = pp[0].nb;
      bytes += sizeof(double) * (static_cast<size_t>(pp[b].n_coef) + 8ull * hb.n);
    }
    const size_t smem = sizeof(double) * static_cast<size_t>(pp[0].wmax + pp[1].wmax + 32);
    if (smem > smem_budget || bytes > free_b / 2) continue;
    const int steps = 2 * std::max(pp[0].nb, pp[1].nb);
    const double coef_bytes = 8.0 * static_cast<double>(pp[0].n_coef + pp[1].n_coef);
    const double t_pi = coef_bytes / 3.9e12 + 2e-6 * steps;
    if (!found || t_pi < best) {
      found = true;
      best = t_pi;
      h->pip[0] = pp[0];
      h->pip[1] = pp[1];
      h->pi_steps = steps;
    }
  }
  if (!found) return false;
  const double t_staged = 0.6e-6 * staged_levels;
  return force || best < 0.7 * t_staged;
}

// Early mode choice (before the plan exists, on the caller's factor arrays):
// modelled time of one partitioned-inverse apply against one blocked-sweep
// apply. The partitioned inverse wins where the factor's bandwidth is small
// (2D systems: its block inverses are tens of MB and its chain a few dozen
// steps); the blocked sweeps win where the inverses would be GBs (3D).
//   t_pi = 8 n_coef / 3.9 TB/s + 2 us x steps    (as in choose_pi)
//   t_bs = 0.35 us x 2 ceil(n / 16)              (measured: 0.28-0.39 us per 16-row group)
bool prefers_partitioned_inverse(const dsgpu_csr* fac[2], const int kinds[2], size_t smem_budget) {
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  int bw[2] = {0, 0};
  double t_bs = 0.0;
  for (int b = 0; b < 2; ++b) {
    if (kinds[b] != DSGPU_BLOCK_PCG_IC0 || !fac[b]) continue;
    bw[b] = pi_bandwidth(fac[b]->n_rows, fac[b]->row_ptr, fac[b]->cols);
    t_bs = std::max(t_bs, 0.35e-6 * 2.0 * ((fac[b]->n_rows + kBsB - 1) / kBsB));
  }
  double best = -1.0;
  for (const double mult : {0.5, 1.0, 1.5}) {
    PiPlan pp[2];
    int nb0 = 0;
    size_t bytes = 0;
    bool ok = true;
    for (int b = 0; b < 2 && ok; ++b) {
      if (kinds[b] != DSGPU_BLOCK_PCG_IC0 || !fac[b]) continue;
      const int n = fac[b]->n_rows;
      int bsz = std::max(1, static_cast<int>(std::ceil(std::max(1, bw[b]) * mult)));
      if (b == 1 && nb0 > 0) bsz = std::max(bsz, (n + nb0 - 1) / nb0);
      // the inverses alone are ~ n * bsz doubles: skip the exact plan when that cannot fit
      if (static_cast<double>(n) * bsz * 8.0 > static_cast<double>(free_b) / 2) {
        ok = false;
        break;
      }
      pp[b] = pi_plan(n, fac[b]->row_ptr, fac[b]->cols, bsz);
      if (b == 0) nb0 = pp[0].nb;
      bytes += sizeof(double) * (static_cast<size_t>(pp[b].n_coef) + 8ull * n);
    }
    if (!ok) continue;
    const size_t smem = sizeof(double) * static_cast<size_t>(pp[0].wmax + pp[1].wmax + 32);
    if (smem > smem_budget || bytes > free_b / 2) continue;
    const double t_pi = 8.0 * static_cast<double>(pp[0].n_coef + pp[1].n_coef) / 3.9e12 +
                        2e-6 * 2 * std::max(pp[0].nb, pp[1].nb);
    if (best < 0.0 || t_pi < best) best = t_pi;
  }
  return best >= 0.0 && best < 0.8 * t_bs;
}

// Shared memory of the PI kernels: both chain windows, then (when it fits)
// one coefficient-prefetch slot per warp.
size_t pi_smem(dsgpu_handle* h, size_t budget) {
  const int win = h->pip[0].wmax + h->pip[1].wmax;
  h->pi_cbase = (win + 31) / 32 * 32;
  h->pi_cslot = (std::max(h->pip[0].wmax, h->pip[1].wmax) + 1) / 2 * 2;
  size_t bytes = sizeof(double) * (static_cast<size_t>(h->pi_cbase) + static_cast<size_t>(kWarps) * h->pi_cslot);
  if (bytes > budget) {
    h->pi_cslot = 0;
    bytes = sizeof(double) * static_cast<size_t>(h->pi_cbase);
  }
  return bytes;
}

}  // namespace

extern "C" {

const char* dsgpu_last_error(const dsgpu_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }

void dsgpu_default_opts(dsgpu_opts* o) {
  o->outer_tol = 1e-12;
  o->inner_tol = 1e-6;
  o->max_iter = 20000;
  o->stop = DSGPU_STOP_EUCLIDEAN;
  o->inner_cap = 100000;
}

int dsgpu_create(int device, dsgpu_handle** out) {
  *out = nullptr;
  auto h = std::make_unique<dsgpu_handle>();
  h->device = device;
  int rc = cuda_check(nullptr, cudaSetDevice(device), "cudaSetDevice");
  if (rc) return rc;
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) return fail(nullptr, DSGPU_E_CUDA, "device lacks cooperative launch");
  rc = cuda_check(nullptr, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking),
                  "cudaStreamCreate");
  if (rc) return rc;
  *out = h.release();
  return DSGPU_OK;
}

int dsgpu_create_multi(int rank, int world, int device, dsgpu_handle** out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world) {
    g_err = "dsgpu_create_multi: need 0 <= rank < world <= 8";
    return DSGPU_E_BAD_INPUT;
  }
  const int rc = dsgpu_create(device, out);
  if (rc) return rc;
  (*out)->rank = rank;
  (*out)->world = world;
  return DSGPU_OK;
}

int dsgpu_multi_ipc_export(dsgpu_handle* h, void* handle64) {
  if (!h || !h->ready || !handle64) return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_multi_ipc_export: not set up");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handle size");
  cudaSetDevice(h->device);
  cudaIpcMemHandle_t m;
  const int rc = cuda_check(h, cudaIpcGetMemHandle(&m, h->arena), "cudaIpcGetMemHandle");
  if (rc) return rc;
  std::memcpy(handle64, &m, 64);
  return DSGPU_OK;
}

int dsgpu_multi_ipc_import(dsgpu_handle* h, const void* handles) {
  if (!h || !h->ready || !handles) return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_multi_ipc_import: not set up");
  cudaSetDevice(h->device);
  h->peer_arena[h->rank] = h->arena;
  h->args.mg.arena[h->rank] = h->arena;
  for (int r = 0; r < h->world; ++r) {
    if (r == h->rank) continue;
    cudaIpcMemHandle_t m;
    std::memcpy(&m, static_cast<const char*>(handles) + 64 * r, 64);
    void* p = nullptr;
    const int rc = cuda_check(h, cudaIpcOpenMemHandle(&p, m, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    if (rc) return rc;
    h->peer_arena[r] = p;
    h->args.mg.arena[r] = static_cast<char*>(p);
  }
  h->peers_open = true;
  return DSGPU_OK;
}

void dsgpu_destroy(dsgpu_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  h->free_all();
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int dsgpu_setup(dsgpu_handle* h, const dsgpu_csr* A, const dsgpu_csr* B, const dsgpu_csr* Bt,
                const dsgpu_csr* Q_nu, int top_kind, const int32_t* perm_A, const dsgpu_csr* L_A,
                int bottom_kind, const int32_t* perm_Q, const dsgpu_csr* L_Q,
                const dsgpu_csr* Q_filter) {
  if (!h) return fail(nullptr, DSGPU_E_BAD_INPUT, "null handle");
  cudaSetDevice(h->device);
  h->free_all();
  h->plan = HostPlan{};
  for (auto& l : h->levels) l = 0;
  // IC(0) apply mode: blocked sweeps unless DSGPU_SWEEP=legacy (or one of the
  // legacy knobs DSGPU_PI / DSGPU_EXACT is set): staged level sweeps or the
  // partitioned inverse by the cost model, or the exact column-order sweeps
  h->exact = std::getenv("DSGPU_EXACT") && std::atoi(std::getenv("DSGPU_EXACT")) != 0;
  h->force_pi = false;
  {
    const char* sw = std::getenv("DSGPU_SWEEP");
    const bool any_ic0 = top_kind == DSGPU_BLOCK_PCG_IC0 || bottom_kind == DSGPU_BLOCK_PCG_IC0;
    if (h->exact || !any_ic0) {
      h->bs = false;
    } else if (sw) {
      h->bs = std::string(sw) == "bs";  // "legacy": round-1 cost model (partitioned inverse / staged sweeps)
    } else if (std::getenv("DSGPU_PI")) {
      h->bs = false;
    } else {  // auto: partitioned inverse where its model wins (2D), blocked sweeps otherwise
      int smem_optin = 0;
      cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
      const dsgpu_csr* fac[2] = {L_A, L_Q};
      const int kinds[2] = {top_kind, bottom_kind};
      bool pi = false;
      try {
        if ((top_kind != DSGPU_BLOCK_PCG_IC0 || (L_A && L_A->row_ptr && L_A->cols)) &&
            (bottom_kind != DSGPU_BLOCK_PCG_IC0 || (L_Q && L_Q->row_ptr && L_Q->cols)))
          pi = prefers_partitioned_inverse(fac, kinds, static_cast<size_t>(smem_optin) - 2048);
      } catch (const std::exception&) {
        pi = false;  // malformed factor: build_plan reports it
      }
      h->bs = !pi;
      h->force_pi = pi;
    }
  }
  try {
    build_plan(h->plan, A, B, Bt, Q_nu, top_kind, perm_A, L_A, bottom_kind, perm_Q, L_Q,
               Q_filter, h->bs ? 1 : 0);
  } catch (const std::domain_error& e) {
    return fail(h, DSGPU_E_NONPOS_DIAG, e.what());
  } catch (const std::exception& e) {
    return fail(h, DSGPU_E_BAD_INPUT, e.what());
  }
  HostPlan& P = h->plan;
  const int64_t L_nnz[2] = {(top_kind == DSGPU_BLOCK_PCG_IC0 && L_A) ? L_A->row_ptr[L_A->n_rows] : 0,
                            (bottom_kind == DSGPU_BLOCK_PCG_IC0 && L_Q) ? L_Q->row_ptr[L_Q->n_rows] : 0};
  try {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    h->sms = sms;
    if (const char* env = std::getenv("DSGPU_REMOTE")) h->remote_max = std::max(0, std::atoi(env));
    if (const char* env = std::getenv("DSGPU_TIMEOUT_S")) {
      const unsigned long long ns = static_cast<unsigned long long>(std::max(0.001, std::atof(env)) * 1e9);
      cudaMemcpyToSymbol(g_spin_timeout_ns, &ns, sizeof(ns));
    }
    if (const char* env = std::getenv("DSGPU_NOWAIT")) {
      const int v = std::atoi(env);
      cudaMemcpyToSymbol(g_nowait, &v, sizeof(v));
    }
    if (const char* env = std::getenv("DSGPU_HSLEEP")) {
      const unsigned ns = static_cast<unsigned>(std::max(0, std::atoi(env)));
      cudaMemcpyToSymbol(g_hsleep, &ns, sizeof(ns));
    }
    // smem: two dataflow arrays of the largest IC block
    int nmax = 0;
    for (int b = 0; b < 2; ++b)
      if (P.blk[b].kind == DSGPU_BLOCK_PCG_IC0) nmax = std::max(nmax, P.blk[b].n);
    int smem_optin_pi = 0;
    cudaDeviceGetAttribute(&smem_optin_pi, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    h->pi = !h->exact && !h->bs && nmax > 0 && choose_pi(h, P, static_cast<size_t>(smem_optin_pi) - 2048);
    h->ring = false;
    h->tb = 4;
    if (h->bs && nmax == 0) h->bs = false;  // no IC(0) block: nothing to sweep
    if (h->bs) {
      h->tb = 0;  // selects the blocked-sweep kernels (minres_for / ic_for)
      h->ring = true;
      // CTA pairs need groups that fit the 18-bit group tag and the column-order
      // ("exact") sweep off
      h->bs_pair = !h->exact;
      for (int b = 0; b < 2; ++b)
        if (P.blk[b].kind == DSGPU_BLOCK_PCG_IC0 && (P.blk[b].n + kBsB - 1) / kBsB >= (1 << 18) - 2) h->bs_pair = false;
      if (const char* env = std::getenv("DSGPU_BS_PAIR")) h->bs_pair = h->bs_pair && std::atoi(env) != 0;
      // slot ring: K + 3 at least; the chain CTA of a pair has room for 12 (C4: 1.24 -> 1.17 s)
      h->bs_ns = h->bs_pair ? std::max(kBsK + 3, 12) : kBsK + 3;
      if (const char* env = std::getenv("DSGPU_BS_SLOTS")) h->bs_ns = std::max(kBsK + 3, std::atoi(env));
    }
    if (!h->exact && !h->pi && !h->bs && nmax > 0) {
      const int merge = std::getenv("DSGPU_MERGE") ? std::atoi(std::getenv("DSGPU_MERGE")) : kDefaultMerge;
      // ring mode when the full solution vector + ring would not fit shared memory
      int smem_optin0 = 0;
      cudaDeviceGetAttribute(&smem_optin0, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
      const size_t budget = static_cast<size_t>(smem_optin0) - 2048;
      const int force_ring_n = std::getenv("DSGPU_RING_N") ? std::atoi(std::getenv("DSGPU_RING_N")) : (1 << 30);
      h->tb = build_block_flows(P, merge, &h->merge, budget, force_ring_n);
      h->ring = (P.blk[0].kind == DSGPU_BLOCK_PCG_IC0 && P.blk[0].ffwd.ring) ||
                (P.blk[1].kind == DSGPU_BLOCK_PCG_IC0 && P.blk[1].ffwd.ring);
      nmax = 0;  // shared-memory footprint per block (x slots)
      for (int b = 0; b < 2; ++b)
        if (P.blk[b].kind == DSGPU_BLOCK_PCG_IC0)
          nmax = std::max(nmax, P.blk[b].ffwd.ring ? kXRing * 32 : P.blk[b].n);
    }
    h->smem = h->exact ? static_cast<size_t>(2) * nmax * sizeof(double)
                       : FlowSmem::bytes(nmax, SlotLayout(h->tb).bytes);
    if (h->pi) h->smem = pi_smem(h, static_cast<size_t>(smem_optin_pi) - 2048);
    // CTA pairs need less shared memory per CTA than the single-CTA sweep (no slot
    // ring in the list CTA, no list staging in the chain CTA): the smaller
    // carve-out leaves the SpMV CTAs of the same kernel more L1
    if (h->bs) h->smem = h->bs_pair ? bs_smem_bytes_pair(h->bs_ns) : bs_smem_bytes(h->bs_ns);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    const size_t static_smem = 1024;
    if (h->smem + static_smem > static_cast<size_t>(smem_optin))
      return fail(h, DSGPU_E_UNSUPPORTED,
                  "IC(0) block too large for the shared-memory dataflow sweep in this build (n=" +
                      std::to_string(nmax) + ")");
    int rc = cuda_check(h, raise_smem_limit(reinterpret_cast<const void*>(minres_for(h->tb, h->ring, h->pi)), smem_optin),
                        "cudaFuncSetAttribute");
    if (rc) return rc;
    rc = cuda_check(h,
                    raise_smem_limit(h->pi ? reinterpret_cast<const void*>(pi_apply_kernel)
                                           : reinterpret_cast<const void*>(ic_for(h->tb, h->ring)),
                                     smem_optin),
                    "cudaFuncSetAttribute");
    if (rc) return rc;
    int per_sm = 0;
    rc = cuda_check(h,
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, minres_for(h->tb, h->ring, h->pi), kThreads,
                                                                  h->smem),
                    "occupancy");
    if (rc) return rc;
    if (per_sm < 1) return fail(h, DSGPU_E_CUDA, "minres kernel cannot be resident");
    if (h->bs_pair) {  // every 2-CTA cluster of a full grid must be resident at once
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(sms & ~1);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = h->smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclus = 0;
      if (cudaOccupancyMaxActiveClusters(&nclus, reinterpret_cast<const void*>(minres_for(h->tb, h->ring, h->pi)), &cfg) !=
              cudaSuccess ||
          2 * nclus < (sms & ~1)) {
        cudaGetLastError();
        h->bs_pair = false;  // single-CTA servers, cooperative launch
        h->bs_ns = kBsK + 3;
        h->smem = bs_smem_bytes(h->bs_ns);
      }
    }
    // grid: IC(0) server CTAs (one per block, CTA b serves block b) + worker
    // CTAs, one per SM, fewer for tiny systems (barrier cost grows with CTAs)
    const int64_t nnz = P.nnz_k;
    if (!h->bs) h->bs_pair = false;
    const int n_srv =
        (!h->pi && (P.blk[0].kind == DSGPU_BLOCK_PCG_IC0 || P.blk[1].kind == DSGPU_BLOCK_PCG_IC0))
            ? (h->bs_pair ? 4 : 2)
            : 0;
    if (n_srv == 0) h->bs_pair = false;
    const int wmax = sms - n_srv;
    int G = static_cast<int>(std::min<int64_t>(wmax, std::max<int64_t>(2, (nnz + 16383) / 16384)));
    G = std::max(G, 2);
    if (h->pi) G = wmax;  // the partitioned-inverse chain wants every SM
    if (h->ring && !h->bs) G = std::min(wmax, std::max(G, 1 + 2 * h->remote_max));  // room for remote helpers
    if (const char* env = std::getenv("DSGPU_GRID")) G = std::max(2, std::min(wmax, std::atoi(env)));
    if (h->bs) {
      // far-worker CTAs of the blocked sweeps: workers 1.. of the grid (worker 0
      // posts the requests), split between the blocks; a block without far
      // entries (everything within the y ring) needs none
      int want[2] = {32, 8};
      if (const char* env = std::getenv("DSGPU_FAR_A")) want[0] = std::max(0, std::atoi(env));
      if (const char* env = std::getenv("DSGPU_FAR_Q")) want[1] = std::max(0, std::atoi(env));
      for (int b = 0; b < 2; ++b)
        if (P.blk[b].kind != DSGPU_BLOCK_PCG_IC0 || P.blk[b].bfwd.nnz_far + P.blk[b].bbwd.nnz_far == 0) want[b] = 0;
      if (!std::getenv("DSGPU_GRID")) G = std::min(wmax, std::max(G, 1 + want[0] + want[1]));
      while (want[0] + want[1] > G - 1) {  // small grids: shrink the larger share first
        int& w = want[0] >= want[1] ? want[0] : want[1];
        --w;
      }
      h->far_ctas[0] = want[0];
      h->far_ctas[1] = want[1];
    }
    if (h->bs_pair && (G & 1)) G += (G < wmax) ? 1 : -1;  // 2-CTA clusters: an even grid
    h->grid = n_srv + G;  // G = worker CTAs below
    // K-row partition balanced by nnz + per-row vector work
    // This rank's rows (partition.hpp: one velocity range and one pressure range,
    // the whole system when world == 1) and their split over the worker CTAs:
    // every CTA works inside ONE block, its rows balanced by nonzeros + vector work.
    RowPartition part;
    if (h->world > 1) {
      if (!h->bs)
        return fail(h, DSGPU_E_UNSUPPORTED, "multi-GPU solves use the blocked sweeps (an IC(0) velocity block)");
      for (int b = 0; b < 2; ++b)
        if (P.blk[b].kind == DSGPU_BLOCK_PCG_JACOBI)
          return fail(h, DSGPU_E_UNSUPPORTED, "multi-GPU solves: Jacobi-PCG blocks are not partitioned");
      part = partition_rows(P.n, P.n_u, P.k_rp.data(), P.k_ci.data(), P.k_v.data(), P.k_na.data(), h->world);
    }
    const int own_u0 = h->world > 1 ? part.rank[h->rank].u0 : 0, own_u1 = h->world > 1 ? part.rank[h->rank].u1 : P.n_u;
    const int own_p0 = h->world > 1 ? part.rank[h->rank].p0 : 0, own_p1 = h->world > 1 ? part.rank[h->rank].p1 : P.n_p;
    std::vector<int32_t> row_lo(G, 0), row_hi(G, 0);
    {
      auto cost = [&](int lo, int hi) { return static_cast<double>(P.k_rp[hi] - P.k_rp[lo]) + 24.0 * (hi - lo); };
      const double cu = cost(own_u0, own_u1), cp = cost(P.n_u + own_p0, P.n_u + own_p1);
      int Gu = static_cast<int>(std::lround(G * cu / std::max(1.0, cu + cp)));
      Gu = std::max(own_u1 > own_u0 ? 1 : 0, std::min(Gu, G - (own_p1 > own_p0 ? 1 : 0)));
      auto split = [&](int lo, int hi, int c0, int c1) {  // rows [lo, hi) over the CTAs [c0, c1)
        const int nc = c1 - c0;
        if (nc <= 0) return;
        const double total = cost(lo, hi);
        int c = 0, start = lo;
        for (int i = lo; i < hi && c + 1 < nc; ++i)
          while (c + 1 < nc && cost(lo, i + 1) >= total * (c + 1) / nc) {
            row_lo[c0 + c] = start;
            row_hi[c0 + c] = i + 1;
            start = i + 1;
            ++c;
          }
        row_lo[c0 + c] = start;
        row_hi[c0 + c] = hi;
        for (++c; c < nc; ++c) row_lo[c0 + c] = row_hi[c0 + c] = hi;
      };
      split(own_u0, own_u1, 0, Gu);
      split(P.n_u + own_p0, P.n_u + own_p1, Gu, G);
    }
    // the arena: sized for everything sub-allocated from it below
    {
      auto up = [](size_t b) { return (b + 255) / 256 * 256 + 256; };
      size_t bytes = up(sizeof(double) * P.n) + up(sizeof(double) * 2 * kMaxWorld * NSLOT) + up(sizeof(unsigned) * 2 * kMaxWorld);
      for (int b = 0; b < 2; ++b)
        bytes += 2 * up(sizeof(double) * P.blk[b].n) + up(sizeof(uint4) * (static_cast<size_t>(P.blk[b].n) + 1));
      h->arena = reinterpret_cast<char*>(h->alloc<char>(bytes));
      h->arena_size = bytes;
      h->arena_used = 0;
      cudaMemset(h->arena, 0, bytes);
    }
    Args& a = h->args;
    a = Args{};
    a.n = P.n;
    a.n_u = P.n_u;
    a.n_p = P.n_p;
    a.k_rp = h->upload(P.k_rp);
    a.k_ci = h->upload(P.k_ci);
    a.k_v = h->upload(P.k_v);
    a.row_lo = h->upload(row_lo);
    a.row_hi = h->upload(row_hi);
    // lanes per row: 16 (64 entries per pass) for the long 3D rows (C4, ~500 entries: saddle
    // 164.7 us vs 172.2 with 8 or 32 lanes, tools/spmv_ab.py); 8 below 256 entries per row
    // (2D): equal in the stand-alone kernel (C3 72.0 vs 71.5 us) but faster inside the
    // persistent kernel, where 16 warps per SM want more rows in flight (C3 saddle phase
    // 153 -> 120 us, inner A phase 116 -> 96 us; profiles/r02_phases_spmv.md)
    auto lanes_for = [](double mean_row) {
      if (const char* env = std::getenv("DSGPU_SPMV_LANES")) {
        const int L = std::atoi(env);
        if (L == 8 || L == 16 || L == 32) return L;
      }
      return mean_row >= 256.0 ? 16 : 8;
    };
    a.k_lanes = lanes_for(static_cast<double>(P.k_rp[P.n]) / P.n);
    const int32_t* d_na = h->upload(P.k_na);
    for (int b = 0; b < 2; ++b) {
      HostBlock& hb = P.blk[b];
      DBlock& d = a.blk[b];
      d.kind = hb.kind;
      d.n = hb.n;
      d.off = hb.off;
      d.ic_cta = b;
      if (b == 0) {
        d.rp = a.k_rp;
        d.ci = a.k_ci;
        d.v = a.k_v;
        d.na = d_na;
        {
          double sum = 0.0;
          for (int i = 0; i < P.n_u; ++i) sum += P.k_na[i];
          d.lanes = lanes_for(sum / std::max(1, P.n_u));
        }
      } else if (hb.kind != DSGPU_BLOCK_JACOBI) {
        d.rp = h->upload(hb.rp);
        d.ci = h->upload(hb.ci);
        d.v = h->upload(hb.v);
        d.na = nullptr;
        d.lanes = lanes_for(static_cast<double>(hb.rp[hb.n]) / std::max(1, hb.n));
      }
      if (!hb.dinv.empty()) d.dinv = h->upload(hb.dinv);
      d.exact = h->exact ? 1 : 0;
      if (hb.kind == DSGPU_BLOCK_PCG_IC0 && h->pi) {
        const PiPlan& pp = h->pip[b];
        d.pi = 1;
        d.pim.nb = pp.nb;
        d.pim.bsz = pp.bsz;
        d.pim.n = pp.n;
        d.pim.wmax = pp.wmax;
        d.pim.cbase = h->pi_cbase;
        d.pim.cslot = h->pi_cslot;
        d.pim.blk = h->upload(pp.blk);
        double* coef = h->alloc<double>(static_cast<size_t>(pp.n_coef));
        d.pim.coef = coef;
        d.pim.set[0] = h->alloc<double>(static_cast<size_t>(4) * pp.n);
        d.pim.set[1] = h->alloc<double>(static_cast<size_t>(4) * pp.n);
        const std::string e = pi_fill(pp, hb.lrp.data(), hb.lci.data(), hb.lv.data(), coef, h->stream);
        if (!e.empty()) throw std::runtime_error("partitioned-inverse setup: " + e);
      } else if (hb.kind == DSGPU_BLOCK_PCG_IC0 && h->bs) {
        d.bs = 1;
        d.bs_ns = h->bs_ns;
        const int G_max = std::max(hb.bfwd.G, hb.bbwd.G);
        h->levels[2 * b] = hb.bfwd.G;
        h->levels[2 * b + 1] = hb.bbwd.G;
        d.bfwd = upload_bsweep(h, hb.bfwd);
        d.bbwd = upload_bsweep(h, hb.bbwd);
        d.y = h->alloc<double>(hb.n + 1);
        d.bb = h->alloc<double>(hb.n + 1);
        cudaMemset(d.y, 0, sizeof(double) * (hb.n + 1));
        cudaMemset(d.bb, 0, sizeof(double) * (hb.n + 1));
        // tag 0 is never a sweep's tag (launch ids start at 1): zeroed = "not written"
        d.bs_bt = h->arena_alloc<uint4>(static_cast<size_t>(hb.n) + 1);
        d.bs_gt = h->alloc<uint4>(static_cast<size_t>(hb.n) + 1);
        d.bs_fps = h->alloc<uint4>(static_cast<size_t>(G_max) * kBsB);
        cudaMemset(d.bs_gt, 0, sizeof(uint4) * (static_cast<size_t>(hb.n) + 1));
        cudaMemset(d.bs_fps, 0, sizeof(uint4) * static_cast<size_t>(G_max) * kBsB);
        d.n_remote = h->far_ctas[b];
        d.remote_cta0 = 1 + (b == 1 ? h->far_ctas[0] : 0);  // worker units (Ctx::remote_rank)
      } else if (hb.kind == DSGPU_BLOCK_PCG_IC0) {
        if (h->exact) {
          d.fwd = upload_sweep(h, hb.fwd);
          d.bwd = upload_sweep(h, hb.bwd);
        } else {
          d.ffwd = upload_flow(h, hb.ffwd);
          d.fbwd = upload_flow(h, hb.fbwd);
        }
        d.y = h->alloc<double>(hb.n + 1);
        d.bb = h->alloc<double>(hb.n + 1);
        cudaMemset(d.y, 0, sizeof(double) * (hb.n + 1));
        cudaMemset(d.bb, 0, sizeof(double) * (hb.n + 1));
      }
      if (hb.kind == DSGPU_BLOCK_PCG_IC0 && !h->exact && hb.ffwd.ring) {
        // remote helpers: CTAs [2 + b R, 2 + (b+1) R) of the persistent kernel
        const int G_max = std::max(hb.ffwd.G, hb.fbwd.G);
        d.rpsum = h->alloc<double>(static_cast<size_t>(G_max) * kRSplit * 32);
        d.rflag = h->alloc<unsigned>(static_cast<size_t>(G_max) * kRSplit);
        d.gprog = h->alloc<unsigned long long>(1);
        cudaMemset(d.rflag, 0, sizeof(unsigned) * G_max * kRSplit);
        cudaMemset(d.gprog, 0, sizeof(unsigned long long));
        const int R = std::min(h->remote_max, (G - 1) / 2);
        d.n_remote = R > 0 ? R : 0;
        d.remote_cta0 = 1 + b * d.n_remote;  // worker units (Ctx::remote_rank), after the lead worker
      }
      d.r = h->alloc<double>(hb.n);
      d.z = h->alloc<double>(hb.n + 1);  // z[n] = 0: the padding column of the far lists
      cudaMemset(d.z, 0, sizeof(double) * (hb.n + 1));
      d.q = h->alloc<double>(hb.n);
      d.p0 = h->arena_alloc<double>(hb.n);
      d.p1 = h->arena_alloc<double>(hb.n);
    }
    if (!h->bs) {
      h->levels[0] = P.blk[0].fwd.n_levels;
      h->levels[1] = P.blk[0].bwd.n_levels;
      h->levels[2] = P.blk[1].fwd.n_levels;
      h->levels[3] = P.blk[1].bwd.n_levels;
    }
    h->nnz_k = nnz;
    h->nnz_a = P.nnz_a;
    for (int b = 0; b < 2; ++b)
      h->nnz_l[b] = P.blk[b].kind == DSGPU_BLOCK_PCG_IC0 ? L_nnz[b] : 0;
    h->nnz_q = P.blk[1].rp.empty() ? 0 : P.nnz_q;
    a.perm_u = h->upload(P.blk[0].perm);
    a.perm_p = h->upload(P.blk[1].perm);
    a.x = h->alloc<double>(P.n);
    a.y = h->arena_alloc<double>(P.n);
    a.v = h->alloc<double>(P.n);
    a.av = h->alloc<double>(P.n);
    a.res = h->alloc<double>(P.n);
    for (int i = 0; i < 4; ++i) a.rbuf[i] = h->alloc<double>(P.n);
    for (int i = 0; i < 3; ++i) {
      a.w[i] = h->alloc<double>(P.n);
      a.aw[i] = h->alloc<double>(P.n);
    }
    a.smem_half = nmax;
    a.filter = P.filter ? 1 : 0;
    a.qk = P.filter ? h->upload(P.qk) : nullptr;
    a.filter_den = P.filter_den;
    a.partial = h->alloc<double>(static_cast<size_t>(2) * NSLOT * G);
    a.bar = h->alloc<unsigned>(128);
    a.n_srv = n_srv;
    a.bs_pair = h->bs_pair ? 1 : 0;
    a.mbox = h->alloc<Mailbox>(2);
    rc = cuda_check(h, cudaMemset(a.bar, 0, 128 * sizeof(unsigned)), "cudaMemset");
    if (rc) return rc;
    h->d_rep = h->alloc<DevReport>(1);
    a.rep = h->d_rep;
    h->d_f = h->alloc<double>(P.n_u);
    h->d_u = h->alloc<double>(P.n_u);
    h->d_p = h->alloc<double>(P.n_p);
    for (int i = 0; i < 3; ++i) h->d_tmp[i] = h->alloc<double>(P.n);
    // multi-GPU state (world == 1: no peers, no halos)
    MultiGpu& m = a.mg;
    m = MultiGpu{};
    m.world = h->world;
    m.rank = h->rank;
    m.arena[h->rank] = h->arena;
    m.xsum = h->arena_alloc<double>(2 * kMaxWorld * NSLOT);
    m.xflag = h->arena_alloc<unsigned>(2 * kMaxWorld);
    if (h->world > 1) {
      const RankPart& R = part.rank[h->rank];
      std::vector<int2> hy, hp[2];
      for (int s2 = 0; s2 < h->world; ++s2)
        for (int k = R.src_ptr[s2]; k < R.src_ptr[s2 + 1]; ++k) {
          hy.push_back(make_int2(R.halo[k], s2));
          if (k - R.src_ptr[s2] < R.a_cnt[s2]) hp[0].push_back(make_int2(R.halo[k], s2));  // A' part: velocity columns
        }
      if (P.blk[1].kind == DSGPU_BLOCK_PCG_IC0) {  // Q' columns of the own pressure rows
        const HostBlock& hb = P.blk[1];
        std::vector<int32_t> cols;
        for (int i = R.p0; i < R.p1; ++i)
          for (int64_t k = hb.rp[i]; k < hb.rp[i + 1]; ++k)
            if (hb.ci[k] < R.p0 || hb.ci[k] >= R.p1) cols.push_back(hb.ci[k]);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        for (const int32_t c : cols) hp[1].push_back(make_int2(c, part.owner_of(P.n_u + c)));
      }
      m.halo_y = h->upload(hy);
      m.n_halo_y = static_cast<int>(hy.size());
      for (int b = 0; b < 2; ++b) {
        m.halo_p[b] = h->upload(hp[b]);
        m.n_halo_p[b] = static_cast<int>(hp[b].size());
      }
    }
  } catch (const std::exception& e) {
    h->free_all();
    return fail(h, DSGPU_E_CUDA, e.what());
  }
  h->ready = true;
  return DSGPU_OK;
}

// The argument block of one solve launch (and the reset of the launch's
// barrier / mailbox words on the handle's stream).
static int solve_args(dsgpu_handle* h, const double* d_f, const dsgpu_opts* o, double* d_u, double* d_p,
                      double* d_hm, double* d_he, int hist_cap, Args& a) {
  a = h->args;
  a.f_in = d_f;
  a.u0_in = h->warm ? h->d_u0 : nullptr;  // one solve only
  a.p0_in = h->warm ? h->d_p0 : nullptr;
  h->warm = false;
  a.u_out = d_u;
  a.p_out = d_p;
  dsgpu_opts def;
  dsgpu_default_opts(&def);
  if (!o) o = &def;
  if (!(o->outer_tol > 0.0) || o->max_iter < 0 || o->inner_cap < 1)
    return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_solve: bad options");
  a.outer_tol = o->outer_tol;
  a.inner_tol = o->inner_tol;
  a.max_iter = o->max_iter;
  a.stop_euclid = o->stop == DSGPU_STOP_EUCLIDEAN ? 1 : 0;
  a.inner_cap = o->inner_cap;
  a.hist_m = d_hm;
  a.hist_e = d_he;
  a.hist_cap = (d_hm && d_he) ? hist_cap : 0;
  a.launch_id = h->next_solve_id();
  int rc = cuda_check(h, cudaMemsetAsync(a.bar, 0, 128 * sizeof(unsigned), h->stream), "memset");
  if (!rc) rc = cuda_check(h, cudaMemsetAsync(a.mbox, 0, 2 * sizeof(Mailbox), h->stream), "memset");
  return rc;
}

// Device report -> dsgpu_report (+ the error the status stands for).
static int solve_report(dsgpu_handle* h, const DevReport& R, float ms, dsgpu_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  rep->iterations = R.iterations;
  rep->converged = R.converged;
  rep->status = R.status;
  rep->failed_block = R.failed_block;
  rep->wall_seconds = ms * 1e-3;
  rep->relres_m = R.relres_m;
  rep->relres_e = R.relres_e;
  rep->inner_top = R.inner[0];
  rep->inner_bottom = R.inner[1];
  rep->apps_top = R.apps[0];
  rep->apps_bottom = R.apps[1];
  rep->mean_inner_top = (h->plan.blk[0].kind != DSGPU_BLOCK_JACOBI && R.apps[0] > 0)
                            ? static_cast<double>(R.inner[0]) / R.apps[0]
                            : 0.0;
  rep->mean_inner_bottom = (h->plan.blk[1].kind != DSGPU_BLOCK_JACOBI && R.apps[1] > 0)
                               ? static_cast<double>(R.inner[1]) / R.apps[1]
                               : 0.0;
  rep->hist_len = R.hist_len;
  rep->gpu_launches = 1;
  if (R.status == DSGPU_E_TIMEOUT)
    return fail(h, DSGPU_E_TIMEOUT, "a device-side wait exceeded DSGPU_TIMEOUT_S (solve aborted)");
  if (R.status == DSGPU_E_CUDA) return fail(h, DSGPU_E_CUDA, "device-side abort");
  if (R.status != DSGPU_OK)
    return fail(h, R.status,
                R.status == DSGPU_E_NEG_CURVATURE
                    ? "pcg: operator is not positive definite"
                    : std::string("preconditioner: ") + (R.failed_block == 1 ? "pressure" : "velocity") +
                          " block produced a negative inner product");
  return DSGPU_OK;
}

// Launch of a persistent solve kernel (all CTAs must be co-resident: they wait
// on one another). Without clusters: a cooperative launch. `pair`: as 2-CTA
// thread-block clusters (the IC(0) server pairs exchange data through
// distributed shared memory) WITHOUT the cooperative attribute -- Nsight
// Compute 2025.2 fails cluster + cooperative launches ("LaunchFailed"), and a
// kernel that cannot be profiled cannot be judged; co-residency is established
// at setup instead (one CTA per SM by shared memory, grid <= SM count, and
// cudaOccupancyMaxActiveClusters >= grid / 2). DSGPU_COOP=1 adds the attribute.
static cudaError_t launch_solve_kernel(const void* fn, int grid, void** params, size_t smem, cudaStream_t stream,
                                       bool pair) {
  if (!pair) return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), params, smem, stream);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  static const bool coop = std::getenv("DSGPU_COOP") && std::atoi(std::getenv("DSGPU_COOP")) != 0;
  cfg.numAttrs = coop ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, fn, params);
}

static int run_solve(dsgpu_handle* h, const double* d_f, const dsgpu_opts* o, double* d_u,
                     double* d_p, dsgpu_report* rep, double* d_hm, double* d_he, int hist_cap) {
  Args a;
  int rc = solve_args(h, d_f, o, d_u, d_p, d_hm, d_he, hist_cap, a);
  if (rc) return rc;
  dsgpu_report rep_local;
  if (!rep) rep = &rep_local;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h->stream);
  void* params[] = {&a};
  const bool warm = a.u0_in != nullptr;
  const void* fn = reinterpret_cast<const void*>(minres_for(h->tb, h->ring, h->pi, warm));
  if (warm) {  // the warm-start instantiation: its shared-memory limit is raised on first use
    if (!fn) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return fail(h, DSGPU_E_UNSUPPORTED, "initial guess: blocked-sweep and partitioned-inverse modes only");
    }
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    raise_smem_limit(fn, optin);
  }
  rc = cuda_check(h, launch_solve_kernel(fn, h->grid, params, h->smem, h->stream, h->bs_pair), "cooperative launch");
  cudaEventRecord(e1, h->stream);
  if (rc) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc;
  }
  DevReport R{};
  rc = cuda_check(h, cudaMemcpyAsync(&R, h->d_rep, sizeof(R), cudaMemcpyDeviceToHost, h->stream),
                  "report D2H");
  if (!rc) rc = cuda_check(h, cudaStreamSynchronize(h->stream), "solve");
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  return solve_report(h, R, ms, rep);
}

// Multi-rank emulation (tests; see minres_emul_kernel): `world` handles made by
// dsgpu_create_multi(r, world, device) on ONE device in this process and set up
// with the same system solve it as `world` ranks inside a single cooperative
// launch. f, u_out, p_out are host vectors of the whole system; reps[r] is
// rank r's report.
int dsgpu_debug_emulate_ranks(dsgpu_handle** hs, int world, const double* f, const dsgpu_opts* o,
                              double* u_out, double* p_out, dsgpu_report* reps) {
  if (!hs || world < 1 || world > kMaxWorld || !f || !u_out || !p_out || !reps) return DSGPU_E_BAD_INPUT;
  dsgpu_handle* h0 = hs[0];
  for (int r = 0; r < world; ++r) {
    dsgpu_handle* h = hs[r];
    if (!h || !h->ready || h->world != world || h->rank != r || h->device != h0->device || h->grid != h0->grid ||
        h->tb != 0 || h->pi || !h->ring || h->bs_pair != h0->bs_pair)
      return fail(h0, DSGPU_E_BAD_INPUT, "dsgpu_debug_emulate_ranks: handles must be ranks 0..world-1 of one device, "
                                          "blocked sweeps, equal grids");
  }
  cudaSetDevice(h0->device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h0->device);
  if (world * h0->grid > sms)
    return fail(h0, DSGPU_E_BAD_INPUT, "dsgpu_debug_emulate_ranks: world x grid exceeds the SM count (set DSGPU_GRID)");
  const HostPlan& P = h0->plan;
  std::vector<Args> all(world);
  size_t smem = 0;
  for (int r = 0; r < world; ++r) {
    dsgpu_handle* h = hs[r];
    for (int q = 0; q < world; ++q) {  // peers: the other handles' arenas, same address space
      h->peer_arena[q] = hs[q]->arena;
      h->args.mg.arena[q] = hs[q]->arena;
    }
    int rc = cuda_check(h, cudaMemcpyAsync(h->d_f, f, sizeof(double) * P.n_u, cudaMemcpyHostToDevice, h->stream), "f H2D");
    if (!rc) rc = cuda_check(h, cudaMemsetAsync(h->d_u, 0, sizeof(double) * P.n_u, h->stream), "memset");
    if (!rc) rc = cuda_check(h, cudaMemsetAsync(h->d_p, 0, sizeof(double) * P.n_p, h->stream), "memset");
    if (!rc) rc = solve_args(h, h->d_f, o, h->d_u, h->d_p, nullptr, nullptr, 0, all[r]);
    if (!rc) rc = cuda_check(h, cudaStreamSynchronize(h->stream), "sync");
    if (rc) return rc;
    all[r].launch_id = all[0].launch_id;  // one launch: the ranks' tags and epochs must agree
    smem = std::max(smem, h->smem);
  }
  Args* d_all = nullptr;
  int rc = cuda_check(h0, cudaMalloc(&d_all, sizeof(Args) * world), "cudaMalloc");
  if (rc) return rc;
  cudaMemcpy(d_all, all.data(), sizeof(Args) * world, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(minres_emul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int per_rank = h0->grid;
  void* params[] = {&d_all, &per_rank};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h0->stream);
  // (with CTA pairs every rank's share of the grid is even, so the 2-CTA clusters never straddle two ranks)
  rc = cuda_check(h0,
                  launch_solve_kernel(reinterpret_cast<const void*>(minres_emul_kernel), world * per_rank, params, smem,
                                      h0->stream, h0->bs_pair),
                  "launch (emulated ranks)");
  cudaEventRecord(e1, h0->stream);
  if (!rc) rc = cuda_check(h0, cudaStreamSynchronize(h0->stream), "emulated solve");
  float ms = 0.0f;
  if (!rc) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_all);
  if (rc) return rc;
  std::vector<double> u(P.n_u), p(P.n_p);
  std::fill(u_out, u_out + P.n_u, 0.0);
  std::fill(p_out, p_out + P.n_p, 0.0);
  int first_err = DSGPU_OK;
  for (int r = 0; r < world; ++r) {
    dsgpu_handle* h = hs[r];
    DevReport R{};
    cudaMemcpy(&R, h->d_rep, sizeof(R), cudaMemcpyDeviceToHost);
    cudaMemcpy(u.data(), h->d_u, sizeof(double) * P.n_u, cudaMemcpyDeviceToHost);
    cudaMemcpy(p.data(), h->d_p, sizeof(double) * P.n_p, cudaMemcpyDeviceToHost);
    for (int i = 0; i < P.n_u; ++i) u_out[i] += u[i];  // every row is written by exactly one rank
    for (int i = 0; i < P.n_p; ++i) p_out[i] += p[i];
    const int src = solve_report(h, R, ms, reps + r);
    if (src && !first_err) first_err = src;
  }
  return first_err;
}

int dsgpu_set_initial_guess(dsgpu_handle* h, const double* u0, const double* p0) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_set_initial_guess: not set up");
  if (!u0 || !p0) {  // back to x0 = 0
    h->warm = false;
    return DSGPU_OK;
  }
  if (h->world > 1) return fail(h, DSGPU_E_UNSUPPORTED, "dsgpu_set_initial_guess: single-GPU handles only");
  cudaSetDevice(h->device);
  const HostPlan& P = h->plan;
  try {
    if (!h->d_u0) {
      h->d_u0 = h->alloc<double>(P.n_u);
      h->d_p0 = h->alloc<double>(P.n_p);
    }
  } catch (const std::exception& e) {
    return fail(h, DSGPU_E_CUDA, e.what());
  }
  int rc = cuda_check(h, cudaMemcpyAsync(h->d_u0, u0, sizeof(double) * P.n_u, cudaMemcpyHostToDevice, h->stream), "x0 H2D");
  if (!rc) rc = cuda_check(h, cudaMemcpyAsync(h->d_p0, p0, sizeof(double) * P.n_p, cudaMemcpyHostToDevice, h->stream), "x0 H2D");
  if (!rc) rc = cuda_check(h, cudaStreamSynchronize(h->stream), "x0 H2D");
  if (rc) return rc;
  h->warm = true;
  return DSGPU_OK;
}

int dsgpu_solve_device(dsgpu_handle* h, const double* d_f, const dsgpu_opts* o, double* d_u_out,
                       double* d_p_out, dsgpu_report* rep) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_solve_device: not set up");
  cudaSetDevice(h->device);
  return run_solve(h, d_f, o, d_u_out, d_p_out, rep, nullptr, nullptr, 0);
}

int dsgpu_solve(dsgpu_handle* h, const double* f, const dsgpu_opts* o, double* u_out,
                double* p_out, dsgpu_report* rep, double* hist_m, double* hist_e,
                int32_t hist_cap) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "dsgpu_solve: not set up");
  cudaSetDevice(h->device);
  const HostPlan& P = h->plan;
  int rc = cuda_check(h,
                      cudaMemcpyAsync(h->d_f, f, sizeof(double) * P.n_u, cudaMemcpyHostToDevice,
                                      h->stream),
                      "f H2D");
  if (rc) return rc;
  double* d_hm = nullptr;
  double* d_he = nullptr;
  if (hist_m && hist_e && hist_cap > 0) {
    if (cudaMallocAsync(&d_hm, sizeof(double) * hist_cap, h->stream) != cudaSuccess ||
        cudaMallocAsync(&d_he, sizeof(double) * hist_cap, h->stream) != cudaSuccess)
      return fail(h, DSGPU_E_CUDA, "history alloc failed");
  }
  const int src = run_solve(h, h->d_f, o, h->d_u, h->d_p, rep, d_hm, d_he, hist_cap);
  if (src == DSGPU_OK || src == DSGPU_E_INDEFINITE_PRECOND || src == DSGPU_E_NEG_CURVATURE) {
    cudaMemcpyAsync(u_out, h->d_u, sizeof(double) * P.n_u, cudaMemcpyDeviceToHost, h->stream);
    cudaMemcpyAsync(p_out, h->d_p, sizeof(double) * P.n_p, cudaMemcpyDeviceToHost, h->stream);
    if (d_hm) {
      const int len = std::min(rep->hist_len, hist_cap);
      cudaMemcpyAsync(hist_m, d_hm, sizeof(double) * len, cudaMemcpyDeviceToHost, h->stream);
      cudaMemcpyAsync(hist_e, d_he, sizeof(double) * len, cudaMemcpyDeviceToHost, h->stream);
    }
  }
  if (d_hm) {
    cudaFreeAsync(d_hm, h->stream);
    cudaFreeAsync(d_he, h->stream);
  }
  rc = cuda_check(h, cudaStreamSynchronize(h->stream), "solve D2H");
  return src ? src : rc;
}

int dsgpu_apply_saddle(dsgpu_handle* h, const double* x, double* y) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "not set up");
  cudaSetDevice(h->device);
  const HostPlan& P = h->plan;
  const Args& a = h->args;
  double *d0 = h->d_tmp[0], *d1 = h->d_tmp[1], *d2 = h->d_tmp[2];
  cudaMemcpyAsync(d0, x, sizeof(double) * P.n, cudaMemcpyHostToDevice, h->stream);
  // to RCM basis: x'[i] = x[perm_u[i]] / x'[n_u+i] = x[n_u + perm_p[i]]
  gather_kernel<<<(P.n_u + 255) / 256, 256, 0, h->stream>>>(P.n_u, a.perm_u, d0, d1);
  gather_kernel<<<(P.n_p + 255) / 256, 256, 0, h->stream>>>(P.n_p, a.perm_p, d0 + P.n_u, d1 + P.n_u);
  spmv_kernel<<<spmv_grid(P.n, a.k_lanes), 256, 0, h->stream>>>(P.n, a.k_rp, a.k_ci, a.k_v, nullptr, d1, d2, a.k_lanes);
  scatter_kernel<<<(P.n_u + 255) / 256, 256, 0, h->stream>>>(P.n_u, a.perm_u, d2, d0);
  scatter_kernel<<<(P.n_p + 255) / 256, 256, 0, h->stream>>>(P.n_p, a.perm_p, d2 + P.n_u, d0 + P.n_u);
  cudaMemcpyAsync(y, d0, sizeof(double) * P.n, cudaMemcpyDeviceToHost, h->stream);
  return cuda_check(h, cudaStreamSynchronize(h->stream), "apply_saddle");
}

// One standalone IC(0) apply of block B (r -> B.z). Ring mode adds the remote
// helper CTAs (co-resident: cooperative launch).
static cudaError_t launch_ic(dsgpu_handle* h, DBlock B, const double* r) {
  unsigned* abort_flag = h->args.bar + 64;
  if (B.pi) {
    fill_sentinel<<<h->sms, 256, 0, h->stream>>>(B.pim.set[0], 4ll * B.pim.n);
    DPi P = B.pim;
    double* z = B.z;
    unsigned par = 0;
    void* params[] = {&P, &r, &z, &par, &abort_flag};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(pi_apply_kernel), dim3(h->grid), dim3(kThreads),
                                       params, h->smem, h->stream);
  }
  unsigned id = h->next_launch_id();
  const int R = B.bs ? std::min(h->sms - 1, B.n_remote)
                     : (B.n_remote > 0 ? std::min(h->sms - 1, std::max(B.n_remote, 2 * h->remote_max)) : 0);
  int pair = (B.bs && h->bs_pair && !B.exact) ? 1 : 0;  // the sweep CTA pair of the solve (2-CTA cluster)
  int Rr = R;
  if (pair) Rr = std::min(R, h->sms - 2) & ~1;  // an even grid
  B.remote_cta0 = 1;
  B.n_remote = Rr;
  if (Rr == 0 && !pair) {
    ic_for(h->tb, h->ring)<<<1, kThreads, h->smem, h->stream>>>(B, r, abort_flag, id, 0);
    return cudaGetLastError();
  }
  void* params[] = {&B, &r, &abort_flag, &id, &pair};
  return launch_solve_kernel(reinterpret_cast<const void*>(ic_for(h->tb, h->ring)), (pair ? 2 : 1) + Rr, params,
                             h->smem, h->stream, pair != 0);
}

int dsgpu_apply_ic0(dsgpu_handle* h, int block, const double* r, double* z) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "not set up");
  if (block < 0 || block > 1 || h->plan.blk[block].kind != DSGPU_BLOCK_PCG_IC0)
    return fail(h, DSGPU_E_BAD_INPUT, "block has no IC(0) factor");
  cudaSetDevice(h->device);
  const int n = h->plan.blk[block].n;
  double *d0 = h->d_tmp[0], *d1 = h->d_tmp[1];
  cudaMemcpyAsync(d0, r, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream);
  cudaMemsetAsync(h->args.bar, 0, 128 * sizeof(unsigned), h->stream);
  DBlock B = h->args.blk[block];
  B.r = d0;
  B.z = d1;
  const int rc = cuda_check(h, launch_ic(h, B, d0), "apply_ic0 launch");
  if (rc) return rc;
  cudaMemcpyAsync(z, d1, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream);
  return cuda_check(h, cudaStreamSynchronize(h->stream), "apply_ic0");
}

int dsgpu_apply_block_matrix(dsgpu_handle* h, int block, const double* x, double* y) {
  if (!h || !h->ready) return fail(h, DSGPU_E_BAD_INPUT, "not set up");
  if (block < 0 || block > 1 || !h->args.blk[block].rp)
    return fail(h, DSGPU_E_BAD_INPUT, "block has no device operator");
  cudaSetDevice(h->device);
  const DBlock& B = h->args.blk[block];
  double *d0 = h->d_tmp[0], *d1 = h->d_tmp[1];
  cudaMemcpyAsync(d0, x, sizeof(double) * B.n, cudaMemcpyHostToDevice, h->stream);
  spmv_kernel<<<spmv_grid(B.n, B.lanes), 256, 0, h->stream>>>(B.n, B.rp, B.ci, B.v, B.na, d0, d1, B.lanes);
  cudaMemcpyAsync(y, d1, sizeof(double) * B.n, cudaMemcpyDeviceToHost, h->stream);
  return cuda_check(h, cudaStreamSynchronize(h->stream), "apply_block_matrix");
}

int dsgpu_time_kernel(dsgpu_handle* h, int which, int reps, double* ms) {
  if (!h || !h->ready || reps < 1) return fail(h, DSGPU_E_BAD_INPUT, "not set up");
  cudaSetDevice(h->device);
  const HostPlan& P = h->plan;
  const Args& a = h->args;
  double *d0 = h->d_tmp[0], *d1 = h->d_tmp[1];
  cudaMemsetAsync(d0, 0, sizeof(double) * P.n, h->stream);
  cudaMemsetAsync(a.bar, 0, 128 * sizeof(unsigned), h->stream);
  auto launch = [&]() {
    if (which == 0) {
      spmv_kernel<<<spmv_grid(P.n, a.k_lanes), 256, 0, h->stream>>>(P.n, a.k_rp, a.k_ci, a.k_v, nullptr, d0, d1, a.k_lanes);
    } else if (which == 1 || which == 2) {
      DBlock B = a.blk[which - 1];
      B.r = d0;
      B.z = d1;
      launch_ic(h, B, d0);
    } else {
      const DBlock& B = a.blk[0];
      spmv_kernel<<<spmv_grid(B.n, B.lanes), 256, 0, h->stream>>>(B.n, B.rp, B.ci, B.v, B.na, d0, d1, B.lanes);
    }
  };
  if ((which == 1 || which == 2) && a.blk[which - 1].kind != DSGPU_BLOCK_PCG_IC0)
    return fail(h, DSGPU_E_BAD_INPUT, "block has no IC(0) factor");
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h->stream);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1, h->stream);
  const int rc = cuda_check(h, cudaEventSynchronize(e1), "time_kernel");
  float t = 0.0f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = t / reps;
  return rc;
}

namespace {
__global__ void vec_init_kernel(int n, double* v, double* av, double* w1, double* w2, double* aw1, double* aw2,
                                double* x, double* res) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    v[i] = (i % 97) / 100.0;
    av[i] = (i % 89) / 50.0 - 0.5;
    w1[i] = (i % 83) * 3e-3;
    w2[i] = (i % 79) * 4e-3;
    aw1[i] = (i % 73) * 5e-3;
    aw2[i] = (i % 71) * 6e-3;
    x[i] = (i % 67) * 7e-3;
    res[i] = (i % 61) * 8e-3 - 0.2;
  }
}
}  // namespace

int dsgpu_time_vector_update(int device, int64_t n64, int reps, double* ms, double* res2) {
  if (n64 < 1 || n64 > (1ll << 30) || reps < 1 || !ms || !res2) {
    g_err = "dsgpu_time_vector_update: bad arguments";
    return DSGPU_E_BAD_INPUT;
  }
  const int n = static_cast<int>(n64);
  if (cudaSetDevice(device) != cudaSuccess) {
    g_err = "dsgpu_time_vector_update: cudaSetDevice failed";
    return DSGPU_E_CUDA;
  }
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, minres_vec_kernel, kThreads, 0);
  const int grid = std::max(1, sms * std::max(1, per_sm));
  double* buf = nullptr;
  const size_t nn = static_cast<size_t>(n);
  if (cudaMalloc(&buf, sizeof(double) * (10 * nn + grid)) != cudaSuccess) {
    g_err = "dsgpu_time_vector_update: cudaMalloc failed";
    return DSGPU_E_CUDA;
  }
  double *v = buf, *av = v + nn, *w1 = av + nn, *w2 = w1 + nn, *aw1 = w2 + nn, *aw2 = aw1 + nn, *wn = aw2 + nn,
         *awn = wn + nn, *x = awn + nn, *res = x + nn, *partial = res + nn;
  vec_init_kernel<<<grid, 256>>>(n, v, av, w1, w2, aw1, aw2, x, res);
  minres_vec_kernel<<<grid, kThreads>>>(n, v, av, w1, w2, aw1, aw2, wn, awn, x, res, partial);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    minres_vec_kernel<<<grid, kThreads>>>(n, v, av, w1, w2, aw1, aw2, wn, awn, x, res, partial);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float t = 0.0f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::vector<double> hp(grid);
  if (e == cudaSuccess) e = cudaMemcpy(hp.data(), partial, sizeof(double) * grid, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) {
    g_err = std::string("dsgpu_time_vector_update: ") + cudaGetErrorString(e);
    return DSGPU_E_CUDA;
  }
  double sum = 0.0;
  for (const double p : hp) sum += p;
  *ms = t / reps;
  *res2 = sum;
  return DSGPU_OK;
}

int dsgpu_debug_counters(int reset, int64_t* out32) {
  unsigned long long v[32] = {};
  cudaMemcpyFromSymbol(v, g_flow_dbg, sizeof(v));
  for (int i = 0; i < 32; ++i) out32[i] = static_cast<int64_t>(v[i]);
  if (reset) {
    const unsigned long long z[32] = {};
    cudaMemcpyToSymbol(g_flow_dbg, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? DSGPU_OK : DSGPU_E_CUDA;
}

int dsgpu_debug_bs_counters(int reset, int64_t* out16) {
#ifdef DSGPU_DIAG
  unsigned long long v[16] = {};
  cudaMemcpyFromSymbol(v, g_bs_dbg, sizeof(v));
  for (int i = 0; i < 16; ++i) out16[i] = static_cast<int64_t>(v[i]);
  if (reset) {
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_bs_dbg, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? DSGPU_OK : DSGPU_E_CUDA;
#else
  (void)reset;
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  return DSGPU_OK;
#endif
}

int dsgpu_debug_phases(int reset, int64_t* out8) {
  unsigned long long v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_phase_dbg, sizeof(v));
  for (int i = 0; i < 8; ++i) out8[i] = static_cast<int64_t>(v[i]);
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_dbg, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? DSGPU_OK : DSGPU_E_CUDA;
}

int dsgpu_debug_spmv_phases(int reset, int64_t* out8) {
  unsigned long long v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyFromSymbol(v, g_spmv_dbg, sizeof(v));
  for (int i = 0; i < 8; ++i) out8[i] = static_cast<int64_t>(v[i]);
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_spmv_dbg, z, sizeof(z));
  }
  return cudaGetLastError() == cudaSuccess ? DSGPU_OK : DSGPU_E_CUDA;
}

int dsgpu_debug_pi_trace(int arm, int64_t* out1024) {
  if (arm) {
    const unsigned long long z[2][512] = {};
    const int on[2] = {1, 1};
    cudaMemcpyToSymbol(g_pi_trace, z, sizeof(z));
    cudaMemcpyToSymbol(g_pi_trace_arm, on, sizeof(on));
  } else {
    static unsigned long long v[2][512];
    cudaMemcpyFromSymbol(v, g_pi_trace, sizeof(v));
    for (int i = 0; i < 1024; ++i) out1024[i] = static_cast<int64_t>(v[i / 512][i % 512]);
  }
  return cudaGetLastError() == cudaSuccess ? DSGPU_OK : DSGPU_E_CUDA;
}

int dsgpu_info(const dsgpu_handle* h, int64_t* info) {
  if (!h || !h->ready) return DSGPU_E_BAD_INPUT;
  info[0] = h->plan.n_u;
  info[1] = h->plan.n_p;
  info[2] = h->nnz_k;
  info[3] = h->nnz_a;
  info[4] = h->nnz_l[0];
  info[5] = h->nnz_l[1];
  info[6] = h->nnz_q;
  for (int i = 0; i < 4; ++i) info[7 + i] = h->levels[i];
  info[11] = h->grid;
  info[12] = h->exact ? 0 : h->bs ? 3 : h->pi ? 2 : 1;
  info[13] = h->bs ? h->levels[0] + h->levels[1] : h->pi ? h->pi_steps : h->levels[0] + h->levels[1];
  info[14] = h->far_ctas[0];
  info[15] = h->far_ctas[1];
  return DSGPU_OK;
}

}  // extern "C"
