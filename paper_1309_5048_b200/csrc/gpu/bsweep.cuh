// Device side of the blocked triangular sweep (see bsweep.hpp for the method
// and the roles). Included by solver.cu after its mbarrier / bulk-copy helpers.
#pragma once

#include "bsweep.hpp"
#include <type_traits>

#include "kernels.cuh"

namespace dsgpu {
namespace dev {

struct DBSweep {
  int n, G, dir;
  const uint8_t* slots;
  const uint8_t* tblk;
  const int32_t *mw, *ms;
  const int64_t* mptr;
  const int32_t* mcols;
  const double* mvals;
  const int32_t* fw;
  const int64_t* fptr;
  const int32_t* fcols;
  const double* fvals;
  const int32_t *fcptr, *fneed;
};

// Global hand-off state of one sweep (shared by a block's two sweeps: tags
// differ). Cross-SM hand-offs carry NO fence and NO flag: every double travels
// as one 16-byte unit {low word, tag, high word, tag} (two self-validating
// 8-byte halves, like NCCL's LL protocol), and the consumer polls the data
// itself until both tags are the sweep's. Measured on B200 (tools/bs_lab.cu):
// 175 cycles per hop, against 2,260 for data + __threadfence + release flag.
struct BsFar {
  uint4* gt;       // [n + 1] tagged copy of the result vector (what the far workers gather)
  uint4* fps;      // [G][16] tagged far partial sum of every row
  unsigned tag;    // unique per sweep (launch id | sweep number)
  int workers;     // far-worker warps outside the sweep CTA (0: its spare warps)
};

__device__ __forceinline__ uint4 bs_pack(double v, unsigned tag) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return make_uint4(static_cast<unsigned>(b), tag, static_cast<unsigned>(b >> 32), tag);
}
__device__ __forceinline__ bool bs_valid(const uint4& w, unsigned tag) { return w.y == tag && w.w == tag; }
// Re-read of a tagged unit inside a polling loop: volatile, so the compiler can
// neither hoist it out of the loop nor merge it with the first read (__ldcg is
// a plain asm the optimizer treats as a pure function of its address).
__device__ __forceinline__ uint4 bs_poll(const uint4* p) {
  uint4 w;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(p)
               : "memory");
  return w;
}
__device__ __forceinline__ double bs_value(const uint4& w) {
  return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(w.z) << 32) | w.x));
}

// Tag of group g's units inside one sweep (shared-memory hand-offs reuse their
// slots every kBsRC groups, so the tag names the group as well as the sweep).
__device__ __forceinline__ unsigned bs_gtag(unsigned sweep_tag, int g) {
  return ((sweep_tag & 0x3FFFu) << 18) + static_cast<unsigned>(g + 1);  // linear in g: the main warp just increments it
}
__device__ __forceinline__ uint4 bs_lds_poll(const uint4* p) {  // volatile 16-byte shared-memory load
  uint4 w;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "r"(smem_u32(p))
               : "memory");
  return w;
}
__device__ __forceinline__ void bs_sts_unit(uint4* p, const uint4& w) {
  asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(w.x), "r"(w.y), "r"(w.z),
               "r"(w.w)
               : "memory");
}
// The same address in the shared memory of CTA `rank` of this cluster (DSMEM).
__device__ __forceinline__ unsigned bs_peer_addr(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
// ... as a 64-bit generic pointer (computed once: a st.shared::cluster through a
// 32-bit address makes the compiler rebuild the generic address -- S2R SR_SWINHI,
// ~50 cycles -- at every store)
__device__ __forceinline__ unsigned long long bs_peer_generic(const void* p, unsigned rank) {
  unsigned long long g;
  asm volatile("cvta.shared::cluster.u64 %0, %1;" : "=l"(g) : "l"(static_cast<unsigned long long>(bs_peer_addr(p, rank))));
  return g;
}
__device__ __forceinline__ void bs_st_generic(unsigned long long addr, const uint4& w) {
  asm volatile("st.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
}
__device__ __forceinline__ void bs_st_peer(unsigned addr, const uint4& w) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
               : "memory");
}
__device__ __forceinline__ void bs_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Diagnostics exist only in the -DDSGPU_DIAG build (make diag): the production
// kernels carry no counters, clocks or atomics on their paths.
#ifdef DSGPU_DIAG
// [0] main cycles, [1] main cycles waiting for c, [2] for slots, [3] for the
// publisher, [4] groups, [5] co-main cycles waiting for progress, [6] for far
// sums, [7] co-main cycles, [8] far-worker cycles waiting, [9] far-worker cycles,
// [10..13] co-main cycles by stage: prefetch + staging wait, mid lists (incl.
// waits), T product, hand-off, [14] main cycles waiting for q, [15] second-main
// cycles waiting for y
__device__ unsigned long long g_bs_dbg[16];
#define BS_DIAG(...) __VA_ARGS__
#else
#define BS_DIAG(...)
#endif

__device__ __forceinline__ double bs_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double bs_shfl_xor16(double v) { return __shfl_xor_sync(0xffffffffu, v, 16); }

// Co-main warps: the warps 0, 1, 2, 4, 5, 6, 8, 9, 10 (never 3 mod 4: that SM
// sub-partition belongs to the main warp).
__device__ __forceinline__ int bs_comain_warp(int i) { return i + i / 3; }

// Shared-memory workspace of the sweep CTA.
struct BsSmem {
  double* ring;             // kBsR groups x 16 results, then the zero slot
  uint4* land;              // kBsRC x 16 tagged units at the SAME offset in every part: c (co-main -> main) in
                            //   the whole / chain CTA, y (main -> relay) in the list CTA
  double* qbuf;             // kBsRQ x 32 lane partials (second main -> main)
  uint8_t* slots;           // ns x kBsSlotBytes
  uint8_t* stage;           // kBsNC x 2 x kBsStageBytes: co-main mid-list staging
  uint64_t* mbar;           // ns
  volatile int* sready;     // ns: group whose blocks have landed in the slot
  int* base_use;            // ns: completed mbarrier phases before this sweep
  volatile int* qready;     // kBsRQ: group whose q is staged
  volatile int* progress;   // groups finished by the main warp
  volatile int* pubdone;    // groups copied to global memory by the publisher
  int ns;                   // slots of THIS part (0 in the list CTA)
  __device__ BsSmem(double* base, int ns_, int part) : ns(part == kBsLists ? 0 : ns_) {
    static_assert(kBsRL == kBsRC, "the landing rings share one region");
    const int nc = part == kBsLists ? kBsNC2 : (part == kBsChain ? 0 : kBsNC);
    uint8_t* p = reinterpret_cast<uint8_t*>(base);
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    p += (128u - (a & 127u)) & 127u;
    ring = reinterpret_cast<double*>(p);
    p += kBsZero + 128;
    land = reinterpret_cast<uint4*>(p);
    p += kBsRC * kBsB * 16;
    qbuf = reinterpret_cast<double*>(p);
    p += kBsRQ * 32 * 8;
    slots = p;
    p += static_cast<size_t>(ns) * kBsSlotBytes;
    stage = p;
    p += static_cast<size_t>(nc) * 2 * kBsStageBytes;
    mbar = reinterpret_cast<uint64_t*>(p);
    p += static_cast<size_t>(ns) * 8;
    sready = reinterpret_cast<volatile int*>(p);
    base_use = reinterpret_cast<int*>(p) + ns;
    qready = reinterpret_cast<volatile int*>(p) + 2 * ns;
    progress = qready + kBsRQ;
    pubdone = progress + 1;
  }
};

// Once per kernel launch and sweep CTA: the slot ring's mbarriers are
// initialized once and only ever advance afterwards.
__device__ void bs_setup(double* smem, int ns, int part) {
  BsSmem S(smem, ns, part);
  for (int i = threadIdx.x; i < S.ns; i += blockDim.x) {
    mbar_init(S.mbar + i, 1);
    S.base_use[i] = 0;
  }
  for (int i = threadIdx.x; i < kBsRC * kBsB; i += blockDim.x) S.land[i] = make_uint4(0u, 0u, 0u, 0u);  // tag 0: never valid
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (part != kBsWhole) bs_cluster_sync();  // the peer's landing ring is clean before anything is sent to it
}

// Far workers: for every group the partial sums of its far entries, gathered
// from the tagged result vector F.gt as the publisher fills it. A gathered
// entry that does not carry this sweep's tag yet is simply read again (lists
// are oldest-first, so only the last chunk of a list ever waits). wid / W: this
// warp among the far-worker warps.
__device__ void bs_far(const DBSweep& s, BsFar F, int wid, int W, unsigned* abort_flag) {
  const int lane = threadIdx.x & 31;
  const uint4* __restrict__ gt = F.gt;
  const unsigned tag = F.tag;
  BS_DIAG(long long t_begin = clock64(); long long t_wait = 0;)
  for (int g = wid; g < s.G; g += W) {
    const int fw = __ldg(s.fw + g);
    if (fw == 0) continue;
    const int64_t base = __ldg(s.fptr + g);
    const int4* cp = reinterpret_cast<const int4*>(s.fcols + base) + lane;
    const double2* vp = reinterpret_cast<const double2*>(s.fvals + base) + lane;
    const int nch = fw / kBsFC;
    double acc = 0.0;
    int4 ca = __ldcs(cp), cb = __ldcs(cp + 32);
    double2 v0 = __ldcs(vp), v1 = __ldcs(vp + 32), v2 = __ldcs(vp + 64), v3 = __ldcs(vp + 96);
    for (int c = 0; c < nch; ++c) {
      // next chunk's lists first: independent of the dependency wait
      int4 na = ca, nb = cb;
      double2 n0 = v0, n1 = v1, n2 = v2, n3 = v3;
      if (c + 1 < nch) {
        na = __ldcs(cp + (2 * c + 2) * 32);
        nb = __ldcs(cp + (2 * c + 3) * 32);
        n0 = __ldcs(vp + (4 * c + 4) * 32);
        n1 = __ldcs(vp + (4 * c + 5) * 32);
        n2 = __ldcs(vp + (4 * c + 6) * 32);
        n3 = __ldcs(vp + (4 * c + 7) * 32);
      }
      uint4 w0 = __ldcg(gt + ca.x), w1 = __ldcg(gt + ca.y), w2 = __ldcg(gt + ca.z), w3 = __ldcg(gt + ca.w);
      uint4 w4 = __ldcg(gt + cb.x), w5 = __ldcg(gt + cb.y), w6 = __ldcg(gt + cb.z), w7 = __ldcg(gt + cb.w);
      auto all_valid = [&]() {
        return bs_valid(w0, tag) && bs_valid(w1, tag) && bs_valid(w2, tag) && bs_valid(w3, tag) &&
               bs_valid(w4, tag) && bs_valid(w5, tag) && bs_valid(w6, tag) && bs_valid(w7, tag);
      };
      if (!all_valid()) {
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        unsigned ns_sleep = 100;
        do {
          __nanosleep(ns_sleep);
          ns_sleep = min(2000u, ns_sleep * 2);
          w0 = bs_poll(gt + ca.x);
          w1 = bs_poll(gt + ca.y);
          w2 = bs_poll(gt + ca.z);
          w3 = bs_poll(gt + ca.w);
          w4 = bs_poll(gt + cb.x);
          w5 = bs_poll(gt + cb.y);
          w6 = bs_poll(gt + cb.z);
          w7 = bs_poll(gt + cb.w);
        } while (!all_valid() && !sg.expired());
        BS_DIAG(t_wait += clock64() - tw;)
      }
      double p0 = v0.x * bs_value(w0), p1 = v1.x * bs_value(w2), p2 = v2.x * bs_value(w4), p3 = v3.x * bs_value(w6);
      p0 = fma(v0.y, bs_value(w1), p0);
      p1 = fma(v1.y, bs_value(w3), p1);
      p2 = fma(v2.y, bs_value(w5), p2);
      p3 = fma(v3.y, bs_value(w7), p3);
      acc += (p0 + p1) + (p2 + p3);
      ca = na;
      cb = nb;
      v0 = n0;
      v1 = n1;
      v2 = n2;
      v3 = n3;
    }
    acc += bs_shfl_xor16(acc);
    if (lane < kBsB) __stcg(F.fps + static_cast<int64_t>(g) * kBsB + lane, bs_pack(acc, tag));
  }
  BS_DIAG(if (lane == 0) {
    atomicAdd(&g_bs_dbg[8], static_cast<unsigned long long>(t_wait));
    atomicAdd(&g_bs_dbg[9], static_cast<unsigned long long>(clock64() - t_begin));
  })
}

// The main warp's waits, out of line (see the step in bsweep): after step g
// (g = -1: before the first) make sure that the dense blocks of group g + 3 have
// landed, that c_{g+1} (tagged unit, re-polled into cw) and q_{g+1} are there and
// that the publisher is not lapped on the y ring.
struct BsMainWait {
  uint4 cw;
  int pd;
};
__device__ __noinline__ BsMainWait bs_main_wait(volatile int* sready_s3, const uint4* land, volatile int* qready,
                                                volatile int* pubdone, unsigned sweep_tag, int g, int G, int r,
                                                uint4 cw, int pd, unsigned* abort_flag) {
  const int gn = g + 1;
  BsMainWait out{cw, pd};
  SpinGuard sg(abort_flag);
  BS_DIAG(long long t0 = clock64(); const bool rec = (threadIdx.x & 31) == 0;)
  // diag: cycles by what was waited for ([2] slots, [1] c, [14] q, [3] publisher)
#define BS_WAIT_MARK(slot)                                                               \
  BS_DIAG({                                                                              \
    const long long t1 = clock64();                                                      \
    if (rec) atomicAdd(&g_bs_dbg[slot], static_cast<unsigned long long>(t1 - t0));       \
    t0 = t1;                                                                             \
  })
  if (g >= 0)
    while (*sready_s3 != g + 3)
      if (sg.expired()) return out;
  BS_WAIT_MARK(2)
  if (gn >= G) return out;
  const unsigned tg = bs_gtag(sweep_tag, gn);
  const uint4* q = land + (gn & (kBsRC - 1)) * kBsB + r;
  while (!bs_valid(out.cw, tg)) {
    if (sg.expired()) return out;
    out.cw = bs_lds_poll(q);
  }
  BS_WAIT_MARK(1)
  if (gn >= 3)
    while (*(qready + (gn & (kBsRQ - 1))) != gn)
      if (sg.expired()) return out;
  BS_WAIT_MARK(14)
  if (gn - out.pd >= kBsR - 2)
    while ((out.pd = *pubdone) < gn - (kBsR - 3))
      if (sg.expired()) return out;
  BS_WAIT_MARK(3)
#undef BS_WAIT_MARK
  return out;
}

// One blocked sweep by every thread of the sweep CTA: gx = T^{-1} rhs (both in
// the factor's ordering). Returns after a CTA barrier with the result complete
// in global memory (plain in gx, tagged in F.gt).
template <int K>
// Right-hand side: rt (tagged units carrying rtag, written by the rows' owners --
// possibly other GPUs -- and polled here) or, when rt is null, the plain vector rhs.
__device__ void bsweep(const DBSweep& s_in, double* smem, int ns_in, const uint4* __restrict__ rt, unsigned rtag,
                       const double* __restrict__ rhs, double* gx, BsFar F, unsigned* abort_flag,
                       int part = kBsWhole) {
  static_assert(K >= 3 && K <= 8 && K == kBsK, "dense coupling depth (F_1, F_2: main warp; F_3..F_K: second main warp)");
  const DBSweep s = s_in;
  const int G = s.G, n = s.n;
  BsSmem S(smem, ns_in, part);
  const int ns = S.ns;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane & 15, hf = lane >> 4;
  // the partner CTA's landing ring (same offset in its shared memory)
  const unsigned peer_land = part == kBsWhole ? 0u : bs_peer_addr(S.land, part == kBsChain ? 1u : 0u);
  for (int i = threadIdx.x; i <= kBsR * kBsB; i += blockDim.x) S.ring[i] = 0.0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) S.sready[i] = -1;
  for (int i = threadIdx.x; i < kBsRQ; i += blockDim.x) S.qready[i] = -1;
  if (threadIdx.x == 0) {
    *S.progress = 0;
    *S.pubdone = 0;
  }
  __syncthreads();
  // roles (warp w runs on SM sub-partition w % 4; the main warp keeps its own)
  const bool chain = part != kBsLists, lists = part != kBsChain;
  const int mainw = chain ? nw - 1 : -1, pubw = chain ? nw - 2 : -1, prodw = chain ? nw - 3 : -1,
            main2w = chain ? nw - 6 : -1;
  const int NCv = part == kBsLists ? kBsNC2 : kBsNC;  // co-main warps of this CTA (round-robin stride)
  const int relayw = part == kBsLists ? kBsNC2 : -1;
  int cid = -1;
  if (part == kBsLists) {
    static_assert(kBsNC2 <= 14, "list CTA: co-mains, one relay warp, spare warps");
    if (warp < kBsNC2) cid = warp;
  } else if (part == kBsWhole) {
    static_assert(kBsNC <= 9, "co-main warps are taken off the main warp's sub-partition");
    for (int i = 0; i < kBsNC; ++i)
      if (warp == bs_comain_warp(i)) cid = i;
  }
  auto orig = [&](int p) { return s.dir ? n - 1 - p : p; };
  // this lane's half row (8 doubles) of dense block `block` of a slot
  auto ld_block = [&](const uint8_t* slot, int block, double* out) {
    const double2* p = reinterpret_cast<const double2*>(slot + block * kBsBlock) + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 t = p[q * 32];
      out[2 * q] = t.x;
      out[2 * q + 1] = t.y;
    }
  };
  auto wait_eq = [&](volatile int* p, int want) {
    SpinGuard sg(abort_flag);
    while (*p != want)
      if (sg.expired()) break;
  };

  if (warp == mainw && G > 0) {
    // ---- main: y_g = c_g - q_g - F_1^g y_{g-1} - F_2^g y_{g-2} -----------------------
    // One step per group; only F_1 y_{g-1} (+ one shuffle) is on the dependent
    // chain. F_2 of group g+1 is applied to y_{g-1} beside it; the next step's
    // rows, c, q and flags are loaded under the chain's tail. The slot array has
    // K + 1 zero groups behind the last one, so no look-ahead index is clamped.
    BS_DIAG(const long long t0 = clock64(); long long w_c = 0, w_s = 0, w_p = 0, w_q = 0;)
    uint8_t* const ringb = reinterpret_cast<uint8_t*>(S.ring);
    for (int k = 0; k <= 2; ++k) wait_eq(S.sready + k % ns, k);
    // c_g arrives as a tagged unit in the landing ring (from this CTA's co-mains or
    // the list CTA's): the load is the poll. The step below is straight-line
    // code: everything it may have to wait for is tested by ONE predicate, and
    // the waiting itself lives out of line (bs_main_wait) -- with a single warp
    // on its sub-partition every taken branch costs an instruction-fetch
    // bubble (ncu: 32 % of the step was no_inst / branch_resolving when each
    // wait had its own inline block).
    asm volatile("" ::: "memory");
    auto slot_at = [&](int slot) { return S.slots + static_cast<size_t>(slot) * kBsSlotBytes; };
    auto next_slot = [&](int slot) { return slot + 1 == ns ? 0 : slot + 1; };
    int s3 = 2 % ns;  // slot of group g+2; o1, o2: byte offsets of the slots of groups g, g+1
    int o1 = 0, o2 = (1 % ns) * kBsSlotBytes, o3 = (2 % ns) * kBsSlotBytes;
    const int oend = ns * kBsSlotBytes;
    const uint8_t* const slot_l = S.slots + lane * 16;  // this lane's unit inside every block
    // this lane's half row (4 units, 512 bytes apart) of one block
    auto ld_row = [&](const uint8_t* p, double* out) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 t = *reinterpret_cast<const double2*>(p + q * 512);
        out[2 * q] = t.x;
        out[2 * q + 1] = t.y;
      }
    };
    (void)slot_at;
    (void)next_slot;
    double f1[8], f2[8];
    ld_row(slot_l + o1, f1);             // F_1 of group 0
    ld_row(slot_l + o2 + kBsBlock, f2);  // F_2 of group 1
    // running addresses and tags of the step: the c unit of group g+1, the tag of
    // group g, the partner's y landing unit of group g
    int coff = (1 & (kBsRC - 1)) * kBsB * 16 + r * 16;
    unsigned tg = bs_gtag(F.tag, 0);
    const uint8_t* const landb = reinterpret_cast<const uint8_t*>(S.land);
    const unsigned long long peer_y = part == kBsChain ? bs_peer_generic(S.land, 1u) + r * 16 : 0ull;
    int poff = 0;
    int pd = 0;
    double c, q2 = 0.0, Q0 = 0.0;
    {
      uint4 cw0 = bs_lds_poll(S.land + r);
      const BsMainWait mw = bs_main_wait(S.sready + s3, S.land, S.qready, S.pubdone, F.tag, -1, G, r, cw0, pd, abort_flag);
      c = bs_value(mw.cw);
    }
    int yoff = (kBsR - 1) * 128 + hf * 64;  // ring bytes of y_{g-1}, this lane's half
    int woff = r * 8;                       // ring bytes of y_g, this lane's row
    // invariant at the top of step g: the slots of groups <= g + 2 have landed
    // One step. (fa, fb) hold F_1 of group g and F_2 of group g+1; the next step's
    // blocks are loaded into the OTHER register set (na, nb): the loop below is
    // unrolled by two with the sets swapped, so no loaded value is copied and
    // nothing on the chain's tail waits for a load.
    auto step = [&](const int g, const double (&fa)[8], const double (&fb)[8], double (&na)[8], double (&nb)[8]) {
      const double2* yp = reinterpret_cast<const double2*>(ringb + yoff);
      const double2 y0 = yp[0], y1 = yp[1], y2 = yp[2], y3 = yp[3];
      double pa = fa[0] * y0.x, pb = fa[4] * y2.x, ua = fb[0] * y0.x, ub = fb[4] * y2.x;
      pa = fma(fa[1], y0.y, pa);
      pb = fma(fa[5], y2.y, pb);
      ua = fma(fb[1], y0.y, ua);
      ub = fma(fb[5], y2.y, ub);
      pa = fma(fa[2], y1.x, pa);
      pb = fma(fa[6], y3.x, pb);
      ua = fma(fb[2], y1.x, ua);
      ub = fma(fb[6], y3.x, ub);
      pa = fma(fa[3], y1.y, pa);
      pb = fma(fa[7], y3.y, pb);
      ua = fma(fb[3], y1.y, ua);
      ub = fma(fb[7], y3.y, ub);
      // next step's operands (slots g+1, g+2: landed) and the flags behind them
      o1 = o2;
      o2 = o3;
      o3 = o3 + kBsSlotBytes == oend ? 0 : o3 + kBsSlotBytes;
      s3 = s3 + 1 == ns ? 0 : s3 + 1;
      ld_row(slot_l + o1, na);
      ld_row(slot_l + o2 + kBsBlock, nb);
      const int gn = g + 1;
      // the chain's tail
      double t = (pa + pb) + (Q0 + q2);
      t += bs_shfl_xor16(t);
      // the flags and c of the next step, as late as their latency allows (issued
      // under the shuffle): a c that lands during the tail is still seen
      uint4 cw = bs_lds_poll(reinterpret_cast<const uint4*>(landb + coff));
      const int fq = S.qready[gn & (kBsRQ - 1)];
      const int fs = S.sready[s3];
      const double y = c - t;
      if (hf == 0) {
        *reinterpret_cast<double*>(ringb + woff) = y;
        if (part == kBsChain)  // the list CTA's copy, through distributed shared memory
          bs_st_generic(peer_y + poff, bs_pack(y, tg));
      }
      poff = (poff + kBsB * 16) & (kBsRL * kBsB * 16 - 1);
      coff = (coff + kBsB * 16) & (kBsRC * kBsB * 16 - 1);
      tg += 1u;  // = bs_gtag(F.tag, g + 1)
      Q0 = ua + ub;
      __syncwarp();
      if (lane == 0) *S.progress = gn;
      yoff = woff - r * 8 + hf * 64;
      woff = woff + 128 == kBsZero + r * 8 ? r * 8 : woff + 128;
      // anything to wait for? (slot of group g+3, c and q of group g+1, the publisher)
      const bool slow = (fs != g + 3) | !bs_valid(cw, tg) | (gn >= 3 && fq != gn) |
                        (gn - pd >= kBsR - 2) | (gn >= G);
      if (__builtin_expect(slow, 0)) {
        const BsMainWait mw = bs_main_wait(S.sready + s3, S.land, S.qready, S.pubdone, F.tag, g, G, r, cw, pd, abort_flag);
        cw = mw.cw;
        pd = mw.pd;
      }
      asm volatile("" ::: "memory");
      c = bs_value(cw);
      q2 = gn >= 3 ? S.qbuf[(gn & (kBsRQ - 1)) * 32 + lane] : 0.0;
    };
    double f1b[8], f2b[8];
    int g = 0;
    for (; g + 1 < G; g += 2) {
      step(g, f1, f2, f1b, f2b);
      step(g + 1, f1b, f2b, f1, f2);
    }
    if (g < G) step(g, f1, f2, f1b, f2b);
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[0], static_cast<unsigned long long>(clock64() - t0));
      atomicAdd(&g_bs_dbg[1], static_cast<unsigned long long>(w_c));
      atomicAdd(&g_bs_dbg[2], static_cast<unsigned long long>(w_s));
      atomicAdd(&g_bs_dbg[3], static_cast<unsigned long long>(w_p));
      atomicAdd(&g_bs_dbg[4], static_cast<unsigned long long>(G));
      atomicAdd(&g_bs_dbg[14], static_cast<unsigned long long>(w_q));
    })
  } else if (warp == main2w && G > 3) {
    // ---- second main: q_t = sum_{k=3..K} F_k^t y_{t-k} --------------------------------
    // Step j consumes y_j as soon as the main warp has published it: the k = 3 term
    // completes q_{j+3} (handed to the main warp two steps before it is needed), the
    // terms k = 4..K go into the running sums of the groups behind it.
    BS_DIAG(long long w_y = 0;)
    const uint8_t* const ringb = reinterpret_cast<const uint8_t*>(S.ring);
    auto slot_at = [&](int slot) { return S.slots + static_cast<size_t>(slot) * kBsSlotBytes; };
    auto next_slot = [&](int slot) { return slot + 1 == ns ? 0 : slot + 1; };
    int sl[K - 2];  // slots of groups j+3 .. j+K
#pragma unroll
    for (int i = 0; i < K - 2; ++i) sl[i] = (3 + i) % ns;
    double A[K - 2];
#pragma unroll
    for (int i = 0; i < K - 2; ++i) A[i] = 0.0;
    int prog = 0, yoff = hf * 64;
    for (int j = 0; j + 3 < G; ++j) {
      if (S.sready[sl[K - 3]] != j + K) wait_eq(S.sready + sl[K - 3], j + K);
      if (prog < j + 1) {
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        while ((prog = *S.progress) < j + 1)
          if (sg.expired()) break;
        BS_DIAG(w_y += clock64() - tw;)
      }
      asm volatile("" ::: "memory");
      const double2* yp = reinterpret_cast<const double2*>(ringb + yoff);
      const double2 y0 = yp[0], y1 = yp[1], y2 = yp[2], y3 = yp[3];
      double pk[K - 2];
#pragma unroll
      for (int i = 0; i < K - 2; ++i) {
        double fk[8];
        ld_block(slot_at(sl[i]), 2 + i, fk);  // F_{3+i} of group j+3+i
        double ua = fk[0] * y0.x, ub = fk[4] * y2.x;
        ua = fma(fk[1], y0.y, ua);
        ub = fma(fk[5], y2.y, ub);
        ua = fma(fk[2], y1.x, ua);
        ub = fma(fk[6], y3.x, ub);
        ua = fma(fk[3], y1.y, ua);
        ub = fma(fk[7], y3.y, ub);
        pk[i] = ua + ub;
      }
      const int t = j + 3;
      S.qbuf[(t & (kBsRQ - 1)) * 32 + lane] = A[0] + pk[0];
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        S.qready[t & (kBsRQ - 1)] = t;
      }
#pragma unroll
      for (int i = 0; i + 1 < K - 2; ++i) A[i] = A[i + 1] + pk[i + 1];
      A[K - 3] = 0.0;
#pragma unroll
      for (int i = 0; i < K - 2; ++i) sl[i] = next_slot(sl[i]);
      yoff = yoff + 128 >= kBsZero ? hf * 64 : yoff + 128;
    }
    BS_DIAG(if (lane == 0) atomicAdd(&g_bs_dbg[15], static_cast<unsigned long long>(w_y));)
  } else if (cid >= 0) {
    // ---- co-main: c_h = T_h (rhs_h - far_h - mid_h) ---------------------------
    // A three-deep pipeline over this warp's groups h, h + NC, h + 2 NC: list
    // sizes two groups ahead, mid-list staging (cp.async) and the right-hand
    // side one group ahead, so no global-memory latency sits on a group's path.
    BS_DIAG(const long long t0 = clock64(); long long w_p = 0, w_f = 0, d_a = 0, d_b = 0, d_c = 0, d_d = 0;)
    const uint8_t* ringb = reinterpret_cast<const uint8_t*>(S.ring);
    uint8_t* const stage0 = S.stage + static_cast<size_t>(cid) * 2 * kBsStageBytes;
    struct Meta {
      int mw, ms, fw;
      int64_t mb;
    };
    auto load_meta = [&](int h) {
      Meta m{0, 0, 0, 0};
      if (h < G) {
        m.mw = __ldg(s.mw + h);
        m.ms = __ldg(s.ms + h);
        m.fw = __ldg(s.fw + h);
        m.mb = __ldg(s.mptr + h);
      }
      return m;
    };
    // stage the first min(mw, kBsStage) mid entries of a group (lane-private units)
    auto stage_group = [&](const Meta& m, int buf) {
      const int mw = min(m.mw, kBsStage);
      const int4* cp = reinterpret_cast<const int4*>(s.mcols + m.mb) + lane;
      const double2* vp = reinterpret_cast<const double2*>(s.mvals + m.mb) + lane;
      const unsigned dst = smem_u32(stage0 + static_cast<size_t>(buf) * kBsStageBytes) + lane * 16;
      for (int c = 0; c < mw / kBsMC; ++c) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536), "l"(cp + c * 32) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536 + 512), "l"(vp + 2 * c * 32)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536 + 1024),
                     "l"(vp + (2 * c + 1) * 32)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // right-hand side of group h, this lane's row: issued one group ahead; a
    // tagged unit that has not arrived yet is polled when it is needed
    auto load_rhs = [&](int h) {
      const int p = h * kBsB + r;
      uint4 w = make_uint4(0u, rtag, 0u, rtag);  // rows without a right-hand side: 0.0, valid
      if (hf == 0 && p < n) w = rt ? __ldcg(rt + orig(p)) : bs_pack(__ldcg(rhs + orig(p)), rtag);
      return w;
    };
    auto take_rhs = [&](uint4 w, int h) {
      if (!bs_valid(w, rtag)) {
        SpinGuard sg(abort_flag);
        const uint4* q = rt + orig(h * kBsB + r);
        do {
          w = bs_poll(q);
        } while (!bs_valid(w, rtag) && !sg.expired());
      }
      return bs_value(w);
    };
    // this lane's half row of T_h, straight from global memory (one group ahead)
    struct TRow {
      double2 a, b, c, d;
    };
    auto load_t = [&](int h) {
      TRow t{};
      if (h < G) {
        const double2* tp = reinterpret_cast<const double2*>(s.tblk + static_cast<size_t>(h) * kBsBlock) + lane;
        t.a = __ldg(tp);
        t.b = __ldg(tp + 32);
        t.c = __ldg(tp + 64);
        t.d = __ldg(tp + 96);
      }
      return t;
    };
    int prog = 0;  // last progress value seen
    Meta m0 = load_meta(cid), m1 = load_meta(cid + NCv);
    stage_group(m0, 0);
    uint4 rhs0 = load_rhs(cid);
    TRow tr0 = load_t(cid);
    int buf = 0;
    for (int h = cid; h < G; h += NCv, buf ^= 1) {
      BS_DIAG(const long long ta = clock64();)
      const Meta m2 = load_meta(h + 2 * NCv);
      stage_group(m1, buf ^ 1);
      const uint4 rhs1 = load_rhs(h + NCv);
      const TRow tr1 = load_t(h + NCv);
      // the far partial sum of this lane's row: the load is the poll
      const uint4* fp = F.fps + static_cast<int64_t>(h) * kBsB + r;
      uint4 fw0 = make_uint4(0u, 0u, 0u, 0u);
      if (m0.fw > 0 && hf == 0) fw0 = __ldcg(fp);
      double acc = take_rhs(rhs0, h);
      const int mw = m0.mw, ms = m0.ms;
      const int4* cp = reinterpret_cast<const int4*>(s.mcols + m0.mb) + lane;
      const double2* vp = reinterpret_cast<const double2*>(s.mvals + m0.mb) + lane;
      const uint8_t* sbuf = stage0 + static_cast<size_t>(buf) * kBsStageBytes + lane * 16;
      auto wait_progress = [&](int need) {
        if (prog >= need) return;
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        // Polling shared memory is not free for the other warps of the SM (every
        // poll is a load on the shared LSU): only the waiter whose turn is next
        // spins; the others sleep in proportion to their distance.
        while ((prog = *S.progress) < need) {
          const int d = need - prog;
          if (part == kBsLists) {  // the list CTA's pipe is its own: short naps only when far away
            if (d > 3) __nanosleep(100);
          } else if (d > 1) {
            __nanosleep(d > 4 ? 400 : 80 * (d - 1));
          }
          if (sg.expired()) break;
        }
        asm volatile("" ::: "memory");
        BS_DIAG(w_p += clock64() - tw;)
      };
      auto use = [&](const int4 cc, const double2 va, const double2 vb) {
        const double x0 = *reinterpret_cast<const double*>(ringb + cc.x);
        const double x1 = *reinterpret_cast<const double*>(ringb + cc.y);
        const double x2 = *reinterpret_cast<const double*>(ringb + cc.z);
        const double x3 = *reinterpret_cast<const double*>(ringb + cc.w);
        double pa = va.x * x0, pb = vb.x * x2;
        pa = fma(va.y, x1, pa);
        pb = fma(vb.y, x3, pb);
        acc -= pa + pb;
      };
      auto chunks = [&](int k0, int k1) {  // mid entries [k0, k1), whole chunks
        int k = k0;
        for (; k < k1 && k < kBsStage; k += kBsMC) {  // staged part
          const uint8_t* q = sbuf + (k / kBsMC) * 1536;
          use(*reinterpret_cast<const int4*>(q), *reinterpret_cast<const double2*>(q + 512),
              *reinterpret_cast<const double2*>(q + 1024));
        }
        if (k >= k1) return;
        // lists wider than the staging buffer (the few groups at the ends of the ordering)
        int4 cc = __ldcs(cp + (k / 4) * 32);
        double2 va = __ldcs(vp + (k / 2) * 32), vb = __ldcs(vp + (k / 2 + 1) * 32);
        for (; k < k1; k += kBsMC) {
          int4 nc = cc;
          double2 na = va, nb = vb;
          if (k + kBsMC < k1) {
            nc = __ldcs(cp + (k / 4 + 1) * 32);
            na = __ldcs(vp + (k / 2 + 2) * 32);
            nb = __ldcs(vp + (k / 2 + 3) * 32);
          }
          use(cc, va, vb);
          cc = nc;
          va = na;
          vb = nb;
        }
      };
      // this group's staged list has landed (all but the newest commit group)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      BS_DIAG(const long long tb = clock64(); d_a += tb - ta;)
      // entries that only need groups <= h-K-3
      wait_progress(h - K - 2);
      chunks(0, ms);
      if (m0.fw > 0 && hf == 0) {
        if (!bs_valid(fw0, F.tag)) {
          BS_DIAG(const long long tw = clock64();)
          SpinGuard sg(abort_flag);
          do {
            fw0 = bs_poll(fp);
          } while (!bs_valid(fw0, F.tag) && !sg.expired());
          BS_DIAG(w_f += clock64() - tw;)
        }
        acc -= bs_value(fw0);
      }
      // the newest mid entries need group h-K-1
      wait_progress(h - K);
      chunks(ms, mw);
      const double t = acc + bs_shfl_xor16(acc);
      BS_DIAG(const long long tc = clock64(); d_b += tc - tb;)
      // c = T t: this lane's half of row r; t_m lives in lane m
      const int src = hf * 8;
      double ca = tr0.a.x * bs_shfl(t, src), cb = tr0.c.x * bs_shfl(t, src + 4);
      ca = fma(tr0.a.y, bs_shfl(t, src + 1), ca);
      cb = fma(tr0.c.y, bs_shfl(t, src + 5), cb);
      ca = fma(tr0.b.x, bs_shfl(t, src + 2), ca);
      cb = fma(tr0.d.x, bs_shfl(t, src + 6), cb);
      ca = fma(tr0.b.y, bs_shfl(t, src + 3), ca);
      cb = fma(tr0.d.y, bs_shfl(t, src + 7), cb);
      double cv = ca + cb;
      cv += bs_shfl_xor16(cv);
      BS_DIAG(const long long td = clock64(); d_c += td - tc;)
      wait_progress(h - kBsRC + 1);  // the c ring slot is free
      if (hf == 0) {  // one self-validating unit: no flag, no fence
        const uint4 u = bs_pack(cv, bs_gtag(F.tag, h));
        const int at = (h & (kBsRC - 1)) * kBsB + r;
        if (part == kBsLists)
          bs_st_peer(peer_land + at * 16, u);
        else
          bs_sts_unit(S.land + at, u);
      }

      m0 = m1;
      m1 = m2;
      rhs0 = rhs1;
      tr0 = tr1;
      BS_DIAG(d_d += clock64() - td;)
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[5], static_cast<unsigned long long>(w_p));
      atomicAdd(&g_bs_dbg[6], static_cast<unsigned long long>(w_f));
      atomicAdd(&g_bs_dbg[7], static_cast<unsigned long long>(clock64() - t0));
      atomicAdd(&g_bs_dbg[10], static_cast<unsigned long long>(d_a));
      atomicAdd(&g_bs_dbg[11], static_cast<unsigned long long>(d_b));
      atomicAdd(&g_bs_dbg[12], static_cast<unsigned long long>(d_c));
      atomicAdd(&g_bs_dbg[13], static_cast<unsigned long long>(d_d));
    })
  } else if (warp == prodw) {
    if (lane == 0) {
      int issued = 0, done = 0, isl = 0, dsl = 0;
      const int Gs = G + K + 1;  // incl. the zero groups behind the last one
      SpinGuard sg(abort_flag);
      while (done < Gs) {
        bool idle = true;
        if (issued < Gs && *S.progress >= issued - ns + 1) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(S.mbar + isl, kBsSlotBytes);
          bulk_g2s(S.slots + static_cast<size_t>(isl) * kBsSlotBytes,
                   s.slots + static_cast<size_t>(issued) * kBsSlotBytes, kBsSlotBytes, S.mbar + isl);
          ++issued;
          isl = isl + 1 == ns ? 0 : isl + 1;
          idle = false;
        }
        if (done < issued) {
          if (mbar_poll(S.mbar + dsl, (S.base_use[dsl] + done / ns) & 1)) {
            S.sready[dsl] = done;
            ++done;
            dsl = dsl + 1 == ns ? 0 : dsl + 1;
            idle = false;
          }
        }
        if (idle) {
          __nanosleep(100);
          if (sg.expired()) break;
        } else {
          sg.t0 = clock64();
        }
      }
    }
  } else if (warp == pubw) {
    // ---- publisher: y ring -> the result vector (plain and tagged) -------------
    int done = 0;
    SpinGuard sg(abort_flag);
    while (done < G) {
      const int pnow = *S.progress;
      if (pnow > done) {
        asm volatile("" ::: "memory");
        for (int g = done + hf; g < pnow; g += 2) {
          const int p = g * kBsB + r;
          if (p < n) {
            const double v = S.ring[(g & (kBsR - 1)) * kBsB + r];
            const int o = orig(p);
            __stcg(F.gt + o, bs_pack(v, F.tag));
            __stcg(gx + o, v);
          }
        }
        __syncwarp();
        if (lane == 0) *S.pubdone = pnow;
        done = pnow;
        sg.t0 = clock64();
      } else {
        __nanosleep(200);
        if (sg.expired()) break;
      }
    }
  } else if (warp == relayw) {
    // ---- relay (list CTA): the chain CTA's results, landed as tagged units through
    // DSMEM, into this CTA's y ring; `progress` is what the co-mains here wait on.
    // It cannot be lapped: the main warp needs c_g, c_g needs progress >= g - K here.
    SpinGuard sg(abort_flag);
    for (int g = 0; g < G; ++g) {
      const unsigned tg = bs_gtag(F.tag, g);
      bool ok = true;
      if (lane < kBsB) {
        const uint4* q = S.land + (g & (kBsRL - 1)) * kBsB + lane;
        uint4 w = bs_lds_poll(q);
        while (!bs_valid(w, tg)) {
          if (sg.expired()) {
            ok = false;
            break;
          }
          w = bs_lds_poll(q);
        }
        S.ring[(g & (kBsR - 1)) * kBsB + lane] = bs_value(w);
      }
      if (!__all_sync(0xffffffffu, ok)) break;  // aborted
      if (lane == 0) {
        __threadfence_block();
        *S.progress = g + 1;
      }
      sg.t0 = clock64();
      sg.w0 = 0;
    }
  } else if (lists && F.workers == 0 && (part == kBsLists ? warp > relayw : true)) {
    // no far-worker CTAs (small grids): the spare warps of this CTA
    int idx = 0, cnt = 0;
    for (int w = 0; w < nw; ++w) {
      bool spare;
      if (part == kBsLists) {
        spare = w > relayw;
      } else {
        bool role = w == mainw || w == pubw || w == prodw || w == main2w;
        for (int i = 0; i < kBsNC; ++i) role = role || w == bs_comain_warp(i);
        spare = !role;
      }
      if (spare) {
        if (w == warp) idx = cnt;
        ++cnt;
      }
    }
    bs_far(s, F, idx, cnt, abort_flag);
  }
  __syncthreads();
  if (threadIdx.x < ns) {
    const int sl = threadIdx.x;
    if (G + K + 1 > sl) S.base_use[sl] += (G + K - sl) / ns + 1;
  }
  __syncthreads();
}

}  // namespace dev
}  // namespace dsgpu
