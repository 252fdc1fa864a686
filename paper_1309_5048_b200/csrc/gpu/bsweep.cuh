// Device side of the blocked triangular sweep (see bsweep.hpp for the method
// and the roles).
#pragma once

#include "bsweep.hpp"
#include "kernels.cuh"

namespace dsgpu {
namespace dev {

struct DBSweep {
  int n, G, dir;
  const uint8_t* slots;  // (G + K + 1) x kBsSlotBytes
  const uint8_t* tblk;   // G x kBsBlock
  const int32_t* lw;
  const int64_t* lptr;
  const int32_t* lcols;
  const double* lvals;
};

// Global hand-off state of one sweep. Cross-SM hand-offs carry NO fence and NO
// flag: every double travels as one 16-byte unit {low word, tag, high word,
// tag} (two self-validating 8-byte halves, like NCCL's LL protocol), and the
// consumer polls the data itself until both tags are right.
struct BsLink {
  const uint4* rt;            // tagged right-hand side (factor ordering), tag rtag
  unsigned rtag;
  uint4* gt;                  // tagged result vector (what the workers gather), tag `tag`
  uint4* ct;                  // [G][16] tagged c of every group (worker -> main warp)
  unsigned long long* hint;   // (tag << 32) | groups finished: a progress HINT for sleeping workers
  unsigned tag;               // unique per sweep (launch id | sweep number)
  int workers;                // worker warps outside the sweep CTA (0: its spare warps)
};

__device__ __forceinline__ uint4 bs_pack(double v, unsigned tag) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return make_uint4(static_cast<unsigned>(b), tag, static_cast<unsigned>(b >> 32), tag);
}
__device__ __forceinline__ bool bs_valid(const uint4& w, unsigned tag) { return w.y == tag && w.w == tag; }
__device__ __forceinline__ double bs_value(const uint4& w) {
  return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(w.z) << 32) | w.x));
}
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
__device__ __forceinline__ unsigned long long bs_poll64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Diagnostics exist only in the -DDSGPU_DIAG build (make diag): the production
// kernels carry no counters, clocks or atomics on their paths.
#ifdef DSGPU_DIAG
// [0] main cycles, [1] main cycles waiting for c, [2] for slots, [3] for the
// publisher, [4] groups, [5] main cycles waiting for q, [6] second-main cycles
// waiting for y, [7] second-main cycles, [8] worker cycles waiting for y, [9]
// worker cycles, [10] worker cycles waiting for the right-hand side
__device__ unsigned long long g_bs_dbg[16];
#define BS_DIAG(...) __VA_ARGS__
#else
#define BS_DIAG(...)
#endif

__device__ __forceinline__ double bs_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double bs_shfl_xor16(double v) { return __shfl_xor_sync(0xffffffffu, v, 16); }

// Shared-memory workspace of the sweep CTA.
struct BsSmem {
  double* ring;             // kBsR groups x 16 results
  double* qbuf;             // kBsRQ x 32 lane partials (second main -> main)
  uint8_t* slots;           // ns x kBsSlotBytes
  uint64_t* mbar;           // ns
  volatile int* sready;     // ns: group whose blocks have landed in the slot
  int* base_use;            // ns: completed mbarrier phases before this sweep
  volatile int* qready;     // kBsRQ: group whose q is staged
  volatile int* progress;   // groups finished by the main warp
  volatile int* pubdone;    // groups copied to global memory by the publisher
  int ns;
  __device__ BsSmem(double* base, int ns_) : ns(ns_) {
    uint8_t* p = reinterpret_cast<uint8_t*>(base);
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    p += (128u - (a & 127u)) & 127u;
    ring = reinterpret_cast<double*>(p);
    p += kBsR * kBsB * 8;
    qbuf = reinterpret_cast<double*>(p);
    p += kBsRQ * 32 * 8;
    slots = p;
    p += static_cast<size_t>(ns) * kBsSlotBytes;
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
__device__ void bs_setup(double* smem, int ns) {
  BsSmem S(smem, ns);
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    mbar_init(S.mbar + i, 1);
    S.base_use[i] = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

// Workers: c_g = T_g ( r_g - sum of the group's list entries times y ) for the
// groups g = wid, wid + W, ... The list (every factor entry older than K
// groups) streams from HBM in chunks of 8 entries per lane; y is gathered from
// the tagged result vector as the main warp fills it -- a unit that does not
// carry this sweep's tag yet is read again (lists are oldest-first, so only
// the last chunk ever waits; the progress hint tells a worker that is far
// ahead how long it may sleep).
__device__ void bs_worker(const DBSweep& s, BsLink L, int wid, int W, unsigned* abort_flag) {
  const int lane = threadIdx.x & 31, r = lane & 15, hf = lane >> 4;
  const uint4* __restrict__ gt = L.gt;
  const unsigned tag = L.tag;
  const int n = s.n;
  BS_DIAG(long long t_begin = clock64(); long long t_wait = 0, t_rhs = 0;)
  for (int g = wid; g < s.G; g += W) {
    const int p = g * kBsB + r;
    const int o = s.dir ? n - 1 - p : p;
    // this lane's half row of T_g and its right-hand side: issued first, used last
    const double2* tp = reinterpret_cast<const double2*>(s.tblk + static_cast<size_t>(g) * kBsBlock) + lane;
    const double2 t0 = __ldg(tp), t1 = __ldg(tp + 32), t2 = __ldg(tp + 64), t3 = __ldg(tp + 96);
    uint4 rw = make_uint4(0u, 0u, 0u, 0u);
    const bool has_rhs = hf == 0 && p < n;
    if (has_rhs) rw = __ldcg(L.rt + o);
    const int lw = __ldg(s.lw + g);
    double acc = 0.0;
    if (lw > 0) {
      const int64_t base = __ldg(s.lptr + g);
      const int4* cp = reinterpret_cast<const int4*>(s.lcols + base) + lane;
      const double2* vp = reinterpret_cast<const double2*>(s.lvals + base) + lane;
      const int nch = lw / kBsLC;
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
          do {
            // far ahead of the main warp: sleep by the hint; close: poll the data
            const unsigned long long hv = bs_poll64(L.hint);
            w0 = bs_poll(gt + ca.x);
            w1 = bs_poll(gt + ca.y);
            w2 = bs_poll(gt + ca.z);
            w3 = bs_poll(gt + ca.w);
            w4 = bs_poll(gt + cb.x);
            w5 = bs_poll(gt + cb.y);
            w6 = bs_poll(gt + cb.z);
            w7 = bs_poll(gt + cb.w);
            const int done = static_cast<unsigned>(hv >> 32) == tag ? static_cast<int>(static_cast<unsigned>(hv)) : -64;
            const int dist = g - kBsK - done;  // groups the main warp still had to finish
            if (dist > 6 && !all_valid()) __nanosleep(min(8000, dist * 60));
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
    }
    double rhs = 0.0;
    if (has_rhs) {
      if (!bs_valid(rw, L.rtag)) {
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        do {
          rw = bs_poll(L.rt + o);
        } while (!bs_valid(rw, L.rtag) && !sg.expired());
        BS_DIAG(t_rhs += clock64() - tw;)
      }
      rhs = bs_value(rw);
    }
    double t = rhs - acc;
    t += bs_shfl_xor16(t);
    // c = T t: this lane's half of row r; t_m lives in lanes m and m + 16
    const int src = hf * 8;
    double ca2 = t0.x * bs_shfl(t, src), cb2 = t2.x * bs_shfl(t, src + 4);
    ca2 = fma(t0.y, bs_shfl(t, src + 1), ca2);
    cb2 = fma(t2.y, bs_shfl(t, src + 5), cb2);
    ca2 = fma(t1.x, bs_shfl(t, src + 2), ca2);
    cb2 = fma(t3.x, bs_shfl(t, src + 6), cb2);
    ca2 = fma(t1.y, bs_shfl(t, src + 3), ca2);
    cb2 = fma(t3.y, bs_shfl(t, src + 7), cb2);
    double cv = ca2 + cb2;
    cv += bs_shfl_xor16(cv);
    if (lane < kBsB) __stcg(L.ct + static_cast<int64_t>(g) * kBsB + lane, bs_pack(cv, tag));
  }
  BS_DIAG(if (lane == 0) {
    atomicAdd(&g_bs_dbg[8], static_cast<unsigned long long>(t_wait));
    atomicAdd(&g_bs_dbg[9], static_cast<unsigned long long>(clock64() - t_begin));
    atomicAdd(&g_bs_dbg[10], static_cast<unsigned long long>(t_rhs));
  })
}

// One blocked sweep by every thread of the sweep CTA. The result goes to L.gt
// (tagged) and, when gx is not null, to gx (plain, factor ordering). Returns
// after a CTA barrier with the result complete.
template <int K>
__device__ void bsweep(const DBSweep& s_in, double* smem, int ns, double* gx, BsLink L, unsigned* abort_flag) {
  static_assert(K >= 3 && K <= 8 && K == kBsK, "dense coupling depth (F_1, F_2: main warp; F_3..F_K: second main warp)");
  const DBSweep s = s_in;
  const int G = s.G, n = s.n;
  BsSmem S(smem, ns);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane & 15, hf = lane >> 4;
  for (int i = threadIdx.x; i < kBsR * kBsB; i += blockDim.x) S.ring[i] = 0.0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) S.sready[i] = -1;
  for (int i = threadIdx.x; i < kBsRQ; i += blockDim.x) S.qready[i] = -1;
  if (threadIdx.x == 0) {
    *S.progress = 0;
    *S.pubdone = gx ? 0 : (1 << 30);  // no plain copy wanted: nobody to wait for
  }
  __syncthreads();
  // roles (warp w runs on SM sub-partition w % 4; the main warp keeps its own)
  const int mainw = nw - 1, pubw = nw - 2, prodw = nw - 3, main2w = nw - 6;
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
  auto slot_at = [&](int slot) { return S.slots + static_cast<size_t>(slot) * kBsSlotBytes; };
  auto next_slot = [&](int slot) { return slot + 1 == ns ? 0 : slot + 1; };

  if (warp == mainw && G > 0) {
    // ---- main: y_g = c_g - q_g - F_1^g y_{g-1} - F_2^g y_{g-2} -----------------------
    // One step per group; only F_1 y_{g-1} (+ one shuffle) is on the dependent
    // chain. F_2 of group g+1 is applied to y_{g-1} beside it; the next step's
    // rows, c, q and flags are loaded under the chain's tail. The slot array has
    // K + 1 zero groups behind the last one, so no look-ahead index is clamped.
    BS_DIAG(const long long t0 = clock64(); long long w_c = 0, w_s = 0, w_p = 0, w_q = 0;)
    uint8_t* const ringb = reinterpret_cast<uint8_t*>(S.ring);
    for (int k = 0; k <= 2; ++k) wait_eq(S.sready + k % ns, k);
    asm volatile("" ::: "memory");
    int s1 = 0, s2 = 1 % ns, s3 = 2 % ns;  // slots of groups g, g+1, g+2
    double f1[8], f2[8];
    ld_block(slot_at(s1), 0, f1);  // F_1 of group 0
    ld_block(slot_at(s2), 1, f2);  // F_2 of group 1
    const uint4* cp = L.ct + r;    // c of group g: cp[16 g]
    uint4 cw = __ldcg(cp);
    {
      BS_DIAG(const long long tw = clock64();)
      SpinGuard sg(abort_flag);
      while (!bs_valid(cw, L.tag) && !sg.expired()) cw = bs_poll(cp);
      BS_DIAG(w_c += clock64() - tw;)
    }
    double c = bs_value(cw), q2 = 0.0, Q0 = 0.0;
    int pd = 0;
    int yoff = (kBsR - 1) * 128 + hf * 64;  // ring bytes of y_{g-1}, this lane's half
    int woff = r * 8;                       // ring bytes of y_g, this lane's row
    int po = s.dir ? n - 1 - r : r, pstep = s.dir ? -kBsB : kBsB;  // this lane's row of the result vector
    int prow = r;
    // invariant at the top of step g: the slots of groups <= g + 2 have landed
    for (int g = 0; g < G; ++g) {
      const int gn = g + 1;
      // c of the next group: the load is issued a whole step before its use
      if (gn < G) cw = __ldcg(cp + static_cast<int64_t>(gn) * kBsB);
      const double2* yp = reinterpret_cast<const double2*>(ringb + yoff);
      const double2 y0 = yp[0], y1 = yp[1], y2 = yp[2], y3 = yp[3];
      double pa = f1[0] * y0.x, pb = f1[4] * y2.x, ua = f2[0] * y0.x, ub = f2[4] * y2.x;
      pa = fma(f1[1], y0.y, pa);
      pb = fma(f1[5], y2.y, pb);
      ua = fma(f2[1], y0.y, ua);
      ub = fma(f2[5], y2.y, ub);
      pa = fma(f1[2], y1.x, pa);
      pb = fma(f1[6], y3.x, pb);
      ua = fma(f2[2], y1.x, ua);
      ub = fma(f2[6], y3.x, ub);
      pa = fma(f1[3], y1.y, pa);
      pb = fma(f1[7], y3.y, pb);
      ua = fma(f2[3], y1.y, ua);
      ub = fma(f2[7], y3.y, ub);
      // next step's operands (slots g+1, g+2: landed) and the flags behind them
      s1 = s2;
      s2 = s3;
      s3 = next_slot(s3);
      ld_block(slot_at(s1), 0, f1);
      ld_block(slot_at(s2), 1, f2);
      const int fq = S.qready[gn & (kBsRQ - 1)];
      const int fs = S.sready[s3];
      // the chain's tail
      double t = (pa + pb) + (Q0 + q2);
      t += bs_shfl_xor16(t);
      const double y = c - t;
      if (hf == 0) {
        *reinterpret_cast<double*>(ringb + woff) = y;
        if (prow < n) __stcg(L.gt + po, bs_pack(y, L.tag));  // to the workers: no fence, no flag
      }
      Q0 = ua + ub;
      __syncwarp();
      if (lane == 0) {
        *S.progress = gn;
        __stcg(L.hint, (static_cast<unsigned long long>(L.tag) << 32) | static_cast<unsigned>(gn));
      }
      yoff = woff - r * 8 + hf * 64;
      woff = woff + 128 == kBsR * 128 + r * 8 ? r * 8 : woff + 128;
      po += pstep;
      prow += kBsB;
      if (fs != g + 3) {
        BS_DIAG(const long long tw = clock64();)
        wait_eq(S.sready + s3, g + 3);
        BS_DIAG(w_s += clock64() - tw;)
      }
      if (gn < G) {
        if (gn >= 3 && fq != gn) {
          BS_DIAG(const long long tw = clock64();)
          wait_eq(S.qready + (gn & (kBsRQ - 1)), gn);
          BS_DIAG(w_q += clock64() - tw;)
        }
        asm volatile("" ::: "memory");
        q2 = gn >= 3 ? S.qbuf[(gn & (kBsRQ - 1)) * 32 + lane] : 0.0;
        if (!bs_valid(cw, L.tag)) {
          BS_DIAG(const long long tw = clock64();)
          SpinGuard sg(abort_flag);
          do {
            cw = bs_poll(cp + static_cast<int64_t>(gn) * kBsB);
          } while (!bs_valid(cw, L.tag) && !sg.expired());
          BS_DIAG(w_c += clock64() - tw;)
        }
        c = bs_value(cw);
      }
      if (gn - pd >= kBsR - 2) {  // never lap the publisher on the y ring
        pd = *S.pubdone;
        if (gn - pd >= kBsR - 2) {
          BS_DIAG(const long long tw = clock64();)
          SpinGuard sg(abort_flag);
          while ((pd = *S.pubdone) < gn - (kBsR - 3))
            if (sg.expired()) break;
          BS_DIAG(w_p += clock64() - tw;)
        }
      }
    }
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[0], static_cast<unsigned long long>(clock64() - t0));
      atomicAdd(&g_bs_dbg[1], static_cast<unsigned long long>(w_c));
      atomicAdd(&g_bs_dbg[2], static_cast<unsigned long long>(w_s));
      atomicAdd(&g_bs_dbg[3], static_cast<unsigned long long>(w_p));
      atomicAdd(&g_bs_dbg[4], static_cast<unsigned long long>(G));
      atomicAdd(&g_bs_dbg[5], static_cast<unsigned long long>(w_q));
    })
  } else if (warp == main2w && G > 3) {
    // ---- second main: q_t = sum_{k=3..K} F_k^t y_{t-k} --------------------------------
    // Step j consumes y_j as soon as the main warp has published it: the k = 3 term
    // completes q_{j+3} (handed to the main warp two steps before it is needed), the
    // terms k = 4..K go into the running sums of the groups behind it.
    BS_DIAG(const long long t0 = clock64(); long long w_y = 0;)
    const uint8_t* const ringb = reinterpret_cast<const uint8_t*>(S.ring);
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
      yoff = yoff + 128 >= kBsR * 128 ? hf * 64 : yoff + 128;
    }
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[6], static_cast<unsigned long long>(w_y));
      atomicAdd(&g_bs_dbg[7], static_cast<unsigned long long>(clock64() - t0));
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
          isl = next_slot(isl);
          idle = false;
        }
        if (done < issued) {
          if (mbar_poll(S.mbar + dsl, (S.base_use[dsl] + done / ns) & 1)) {
            S.sready[dsl] = done;
            ++done;
            dsl = next_slot(dsl);
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
  } else if (warp == pubw && gx) {
    // ---- publisher: y ring -> the plain result vector ---------------------------------
    int done = 0;
    SpinGuard sg(abort_flag);
    while (done < G) {
      const int pnow = *S.progress;
      if (pnow > done) {
        asm volatile("" ::: "memory");
        for (int g = done + hf; g < pnow; g += 2) {
          const int p = g * kBsB + r;
          if (p < n) __stcg(gx + (s.dir ? n - 1 - p : p), S.ring[(g & (kBsR - 1)) * kBsB + r]);
        }
        __syncwarp();
        if (lane == 0) *S.pubdone = pnow;
        done = pnow;
        sg.t0 = clock64();
      } else {
        __nanosleep(100);
        if (sg.expired()) break;
      }
    }
  } else if (L.workers == 0 && warp < nw - 6 && (warp & 3) != (mainw & 3)) {
    // no worker CTAs (tiny grids): the spare warps off the main warp's sub-partition
    int idx = 0, cnt = 0;
    for (int w = 0; w < nw - 6; ++w)
      if ((w & 3) != (mainw & 3)) {
        if (w == warp) idx = cnt;
        ++cnt;
      }
    bs_worker(s, L, idx, cnt, abort_flag);
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
