// Device side of the blocked triangular sweep (see bsweep.hpp for the method
// and the roles). Included by solver.cu after its mbarrier / bulk-copy helpers.
#pragma once

#include "bsweep.hpp"
#include "kernels.cuh"

namespace dsgpu {
namespace dev {

struct DBSweep {
  int n, G, dir;
  const uint8_t* slots;
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

// Global hand-off state of one sweep (shared by a block's two sweeps: tags differ).
struct BsFar {
  double* fpsum;               // [G][16] far partial sum of every row
  unsigned* fflag;             // [G] sweep tag once fpsum[g] is final
  unsigned long long* gprog;   // (sweep tag << 32) | groups published in the result vector
  unsigned tag;
  int workers;                 // far-worker warps outside the sweep CTA (0: its spare warps)
};

// Diagnostics exist only in the -DDSGPU_DIAG build (make diag): the production
// kernels carry no counters, clocks or atomics on their paths.
#ifdef DSGPU_DIAG
// [0] main cycles, [1] main cycles waiting for c, [2] for slots, [3] for the
// publisher, [4] groups, [5] co-main cycles waiting for progress, [6] for far
// sums, [7] co-main cycles, [8] far-worker cycles waiting, [9] far-worker cycles
__device__ unsigned long long g_bs_dbg[16];
#define BS_DIAG(...) __VA_ARGS__
#else
#define BS_DIAG(...)
#endif

__device__ __forceinline__ unsigned long long bs_ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bs_st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double bs_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double bs_shfl_xor16(double v) { return __shfl_xor_sync(0xffffffffu, v, 16); }

// Shared-memory workspace of the sweep CTA.
struct BsSmem {
  double* ring;             // kBsR groups x 16 results, then the zero slot
  double* cbuf;             // kBsRC x 16 (co-main -> main)
  uint8_t* slots;           // ns x kBsSlotBytes
  uint8_t* stage;           // kBsNC x 2 x kBsStageBytes: co-main mid-list staging
  uint64_t* mbar;           // ns
  volatile int* sready;     // ns: group whose blocks have landed in the slot
  int* base_use;            // ns: completed mbarrier phases before this sweep
  volatile int* aready;     // kBsRC: group whose c is staged
  volatile int* progress;   // groups finished by the main warp
  volatile int* pubdone;    // groups copied to global memory by the publisher
  int ns;
  __device__ BsSmem(double* base, int ns_) : ns(ns_) {
    uint8_t* p = reinterpret_cast<uint8_t*>(base);
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    p += (128u - (a & 127u)) & 127u;
    ring = reinterpret_cast<double*>(p);
    p += kBsZero + 128;
    cbuf = reinterpret_cast<double*>(p);
    p += kBsRC * kBsB * 8;
    slots = p;
    p += static_cast<size_t>(ns) * kBsSlotBytes;
    stage = p;
    p += static_cast<size_t>(kBsNC) * 2 * kBsStageBytes;
    mbar = reinterpret_cast<uint64_t*>(p);
    p += static_cast<size_t>(ns) * 8;
    sready = reinterpret_cast<volatile int*>(p);
    base_use = reinterpret_cast<int*>(p) + ns;
    aready = reinterpret_cast<volatile int*>(p) + 2 * ns;
    progress = aready + kBsRC;
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

// Far workers: for every group the partial sums of its far entries, gathered
// from the published part of the result vector gx. wid / W: this warp among
// the far-worker warps.
__device__ void bs_far(const DBSweep& s, const double* __restrict__ gx, BsFar F, int wid, int W,
                       unsigned* abort_flag) {
  const int lane = threadIdx.x & 31;
  unsigned seen = 0;
  BS_DIAG(long long t_begin = clock64(); long long t_wait = 0;)
  for (int g = wid; g < s.G; g += W) {
    const int fw = __ldg(s.fw + g);
    if (fw == 0) continue;
    const int64_t base = __ldg(s.fptr + g);
    const int32_t* need = s.fneed + __ldg(s.fcptr + g);
    const int4* cp = reinterpret_cast<const int4*>(s.fcols + base) + lane;
    const double2* vp = reinterpret_cast<const double2*>(s.fvals + base) + lane;
    const int nch = fw / kBsFC;
    double acc = 0.0;
    SpinGuard sg(abort_flag);
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
      const unsigned nd = static_cast<unsigned>(__ldg(need + c) + 1);
      if (seen < nd) {
        BS_DIAG(const long long tw = clock64();)
        for (;;) {  // the tag must match: progress words of other sweeps never count
          const unsigned long long v = bs_ld_acquire_u64(F.gprog);
          unsigned ns_sleep = 500;
          if (static_cast<unsigned>(v >> 32) == F.tag) {
            seen = static_cast<unsigned>(v);
            if (seen >= nd) break;
            ns_sleep = min(4000u, (nd - seen) * 48u);  // ~half the expected wait
          }
          __nanosleep(ns_sleep);
          if (sg.expired()) break;
        }
        BS_DIAG(t_wait += clock64() - tw;)
      }
      const double x0 = __ldcg(gx + ca.x), x1 = __ldcg(gx + ca.y), x2 = __ldcg(gx + ca.z), x3 = __ldcg(gx + ca.w);
      const double x4 = __ldcg(gx + cb.x), x5 = __ldcg(gx + cb.y), x6 = __ldcg(gx + cb.z), x7 = __ldcg(gx + cb.w);
      double p0 = v0.x * x0, p1 = v1.x * x2, p2 = v2.x * x4, p3 = v3.x * x6;
      p0 = fma(v0.y, x1, p0);
      p1 = fma(v1.y, x3, p1);
      p2 = fma(v2.y, x5, p2);
      p3 = fma(v3.y, x7, p3);
      acc += (p0 + p1) + (p2 + p3);
      ca = na;
      cb = nb;
      v0 = n0;
      v1 = n1;
      v2 = n2;
      v3 = n3;
    }
    acc += bs_shfl_xor16(acc);
    if (lane < kBsB) __stcg(F.fpsum + static_cast<int64_t>(g) * kBsB + lane, acc);
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(F.fflag + g, F.tag);
  }
  BS_DIAG(if (lane == 0) {
    atomicAdd(&g_bs_dbg[8], static_cast<unsigned long long>(t_wait));
    atomicAdd(&g_bs_dbg[9], static_cast<unsigned long long>(clock64() - t_begin));
  })
}

// One blocked sweep by every thread of the sweep CTA: gx = T^{-1} rhs (both in
// the factor's ordering; gx has n + 1 entries, gx[n] = 0). Returns after a CTA
// barrier with the result complete in global memory.
template <int K>
__device__ void bsweep(const DBSweep& s_in, double* smem, int ns, const double* __restrict__ rhs, double* gx,
                       BsFar F, unsigned* abort_flag) {
  static_assert(K >= 1 && K <= 4 && K == kBsK, "dense coupling depth");
  const DBSweep s = s_in;
  const int G = s.G, n = s.n;
  BsSmem S(smem, ns);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane & 15, hf = lane >> 4;
  for (int i = threadIdx.x; i <= kBsR * kBsB; i += blockDim.x) S.ring[i] = 0.0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) S.sready[i] = -1;
  for (int i = threadIdx.x; i < kBsRC; i += blockDim.x) S.aready[i] = -1;
  if (threadIdx.x == 0) {
    *S.progress = 0;
    *S.pubdone = 0;
  }
  __syncthreads();
  // roles (warp w runs on SM sub-partition w % 4; the main warp keeps its own)
  const int mainw = nw - 1, pubw = nw - 2, prodw = nw - 8;
  int cid = -1;
  {
    const int cw[kBsNC] = {0, 1, 2, 4};
    for (int i = 0; i < kBsNC; ++i)
      if (warp == cw[i]) cid = i;
  }
  auto slot_of = [&](int g) { return S.slots + static_cast<size_t>(g % ns) * kBsSlotBytes; };
  auto orig = [&](int p) { return s.dir ? n - 1 - p : p; };
  // row `row` (this lane's half) of dense block `block` of the slot
  auto ld_block = [&](const uint8_t* slot, int block, double* out) {
    const double2* p = reinterpret_cast<const double2*>(slot + block * kBsBlock) + lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 t = p[q * 32];
      out[2 * q] = t.x;
      out[2 * q + 1] = t.y;
    }
  };
  auto wait_int = [&](volatile int* p, int want_ge, bool exact) {
    SpinGuard sg(abort_flag);
    for (;;) {
      const int v = *p;
      if (exact ? v == want_ge : v >= want_ge) break;
      if (sg.expired()) break;
    }
    asm volatile("" ::: "memory");  // data reads stay behind the flag
  };

  if (warp == mainw && G > 0) {
    BS_DIAG(const long long t0 = clock64(); long long w_c = 0, w_s = 0, w_p = 0;)
    double Q[K > 1 ? K - 1 : 1];
#pragma unroll
    for (int k = 0; k < (K > 1 ? K - 1 : 1); ++k) Q[k] = 0.0;
    for (int k = 0; k < K; ++k) wait_int(S.sready + (k < G ? k : G - 1) % ns, k < G ? k : G - 1, true);
    double f1[8];
    ld_block(slot_of(0), 0, f1);
    wait_int(S.aready + 0, 0, true);
    double c = S.cbuf[r];
    int pd = 0;
    for (int g = 0; g < G; ++g) {
      // ---- the critical chain: y_g = c_g - (Q + F_1 y_{g-1}) ----------------
      const double2* yp =
          reinterpret_cast<const double2*>(reinterpret_cast<const uint8_t*>(S.ring) + ((g + kBsR - 1) % kBsR) * 128 + hf * 64);
      const double2 y0 = yp[0], y1 = yp[1], y2 = yp[2], y3 = yp[3];
      double pa = f1[0] * y0.x, pb = f1[4] * y2.x;
      pa = fma(f1[1], y0.y, pa);
      pb = fma(f1[5], y2.y, pb);
      pa = fma(f1[2], y1.x, pa);
      pb = fma(f1[6], y3.x, pb);
      pa = fma(f1[3], y1.y, pa);
      pb = fma(f1[7], y3.y, pb);
      double t = pa + pb;
      if (K > 1) t += Q[0];
      t += bs_shfl_xor16(t);
      const double y = c - t;
      if (hf == 0) S.ring[(g % kBsR) * kBsB + r] = y;
      __syncwarp();
      if (lane == 0) *S.progress = g + 1;
      // ---- off the chain: flags of the next step, future partial sums -------
      const int gn = g + 1 < G ? g + 1 : G - 1;
      const int gs = g + K < G ? g + K : G - 1;
      const int fa = S.aready[gn % kBsRC];
      const int fs = S.sready[gs % ns];
      if (g + 1 - pd >= kBsR - 2) pd = *S.pubdone;
#pragma unroll
      for (int k = 2; k <= K; ++k) {
        const int gk = g + k - 1 < G ? g + k - 1 : G - 1;
        double fk[8];
        ld_block(slot_of(gk), k - 1, fk);
        double qa = fk[0] * y0.x, qb = fk[4] * y2.x;
        qa = fma(fk[1], y0.y, qa);
        qb = fma(fk[5], y2.y, qb);
        qa = fma(fk[2], y1.x, qa);
        qb = fma(fk[6], y3.x, qb);
        qa = fma(fk[3], y1.y, qa);
        qb = fma(fk[7], y3.y, qb);
        Q[k - 2] = (k < K ? Q[k - 1] : 0.0) + (qa + qb);
      }
      if (fs != gs) {
        BS_DIAG(const long long tw = clock64();)
        wait_int(S.sready + gs % ns, gs, true);
        BS_DIAG(w_s += clock64() - tw;)
      }
      ld_block(slot_of(gn), 0, f1);
      if (fa != gn) {
        BS_DIAG(const long long tw = clock64();)
        wait_int(S.aready + gn % kBsRC, gn, true);
        BS_DIAG(w_c += clock64() - tw;)
      }
      asm volatile("" ::: "memory");
      c = S.cbuf[(gn % kBsRC) * kBsB + r];
      if (g + 1 - pd >= kBsR - 2) {  // never lap the publisher on the y ring
        BS_DIAG(const long long tw = clock64();)
        wait_int(S.pubdone, g + 1 - (kBsR - 3), false);
        pd = *S.pubdone;
        BS_DIAG(w_p += clock64() - tw;)
      }
    }
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[0], static_cast<unsigned long long>(clock64() - t0));
      atomicAdd(&g_bs_dbg[1], static_cast<unsigned long long>(w_c));
      atomicAdd(&g_bs_dbg[2], static_cast<unsigned long long>(w_s));
      atomicAdd(&g_bs_dbg[3], static_cast<unsigned long long>(w_p));
      atomicAdd(&g_bs_dbg[4], static_cast<unsigned long long>(G));
    })
  } else if (cid >= 0) {
    // ---- co-main: c_h = T_h (rhs_h - far_h - mid_h) ---------------------------
    BS_DIAG(const long long t0 = clock64(); long long w_p = 0, w_f = 0;)
    const uint8_t* ringb = reinterpret_cast<const uint8_t*>(S.ring);
    uint8_t* const stage0 = S.stage + static_cast<size_t>(cid) * 2 * kBsStageBytes;
    // stage the first min(mw, kBsStage) mid entries of group h (this lane's
    // 16-byte units, lane-private: no cross-lane synchronization needed)
    auto stage_group = [&](int h, int buf) {
      if (h < G) {
        const int mw = min(__ldg(s.mw + h), kBsStage);
        const int64_t mb = __ldg(s.mptr + h);
        const int4* cp = reinterpret_cast<const int4*>(s.mcols + mb) + lane;
        const double2* vp = reinterpret_cast<const double2*>(s.mvals + mb) + lane;
        const unsigned dst = smem_u32(stage0 + static_cast<size_t>(buf) * kBsStageBytes) + lane * 16;
        for (int c = 0; c < mw / kBsMC; ++c) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536), "l"(cp + c * 32) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536 + 512), "l"(vp + 2 * c * 32)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + c * 1536 + 1024),
                       "l"(vp + (2 * c + 1) * 32)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int prog = 0;  // last progress value seen
    stage_group(cid, 0);
    int buf = 0;
    for (int h = cid; h < G; h += kBsNC, buf ^= 1) {
      stage_group(h + kBsNC, buf ^ 1);
      const int p = h * kBsB + r;
      double acc = (hf == 0 && p < n) ? __ldcg(rhs + orig(p)) : 0.0;
      const int mw = __ldg(s.mw + h), ms = __ldg(s.ms + h), fw = __ldg(s.fw + h);
      const int64_t mb = __ldg(s.mptr + h);
      const int4* cp = reinterpret_cast<const int4*>(s.mcols + mb) + lane;
      const double2* vp = reinterpret_cast<const double2*>(s.mvals + mb) + lane;
      const uint8_t* sbuf = stage0 + static_cast<size_t>(buf) * kBsStageBytes + lane * 16;
      auto wait_progress = [&](int need) {
        if (prog >= need) return;
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        while ((prog = *S.progress) < need)
          if (sg.expired()) break;
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
      // entries that only need groups <= h-K-3
      wait_progress(h - K - 2);
      chunks(0, ms);
      if (fw > 0) {  // far partial sum of this lane's row
        BS_DIAG(const long long tw = clock64();)
        SpinGuard sg(abort_flag);
        while (ld_acquire(F.fflag + h) != F.tag) {
          __nanosleep(40);
          if (sg.expired()) break;
        }
        BS_DIAG(w_f += clock64() - tw;)
        if (hf == 0) acc -= __ldcg(F.fpsum + static_cast<int64_t>(h) * kBsB + r);
      }
      // the newest mid entries need group h-K-1
      wait_progress(h - K);
      chunks(ms, mw);
      const double t = acc + bs_shfl_xor16(acc);
      // c = T t: this lane's half of row r; t_m lives in lane m
      if (S.sready[h % ns] != h) wait_int(S.sready + h % ns, h, true);
      double tr[8];
      ld_block(slot_of(h), K, tr);
      double ca = 0.0, cb = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ca = fma(tr[j], bs_shfl(t, hf * 8 + j), ca);
        cb = fma(tr[4 + j], bs_shfl(t, hf * 8 + 4 + j), cb);
      }
      double cv = ca + cb;
      cv += bs_shfl_xor16(cv);
      wait_progress(h - kBsRC + 1);  // the c ring slot is free
      if (hf == 0) S.cbuf[(h % kBsRC) * kBsB + r] = cv;
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        S.aready[h % kBsRC] = h;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    BS_DIAG(if (lane == 0) {
      atomicAdd(&g_bs_dbg[5], static_cast<unsigned long long>(w_p));
      atomicAdd(&g_bs_dbg[6], static_cast<unsigned long long>(w_f));
      atomicAdd(&g_bs_dbg[7], static_cast<unsigned long long>(clock64() - t0));
    })
  } else if (warp == prodw) {
    if (lane == 0) {
      int issued = 0, done = 0;
      SpinGuard sg(abort_flag);
      while (done < G) {
        bool idle = true;
        if (issued < G && *S.progress >= issued - ns + 1) {
          const int sl = issued % ns;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(S.mbar + sl, kBsSlotBytes);
          bulk_g2s(S.slots + static_cast<size_t>(sl) * kBsSlotBytes,
                   s.slots + static_cast<size_t>(issued) * kBsSlotBytes, kBsSlotBytes, S.mbar + sl);
          ++issued;
          idle = false;
        }
        if (done < issued) {
          const int sl = done % ns;
          if (mbar_poll(S.mbar + sl, (S.base_use[sl] + done / ns) & 1)) {
            S.sready[sl] = done;
            ++done;
            idle = false;
          }
        }
        if (idle) {
          if (sg.expired()) break;
        } else {
          sg.t0 = clock64();
        }
      }
    }
  } else if (warp == pubw) {
    // ---- publisher: y ring -> result vector, then the progress word ----------
    int done = 0;
    SpinGuard sg(abort_flag);
    while (done < G) {
      const int pnow = *S.progress;
      if (pnow > done) {
        asm volatile("" ::: "memory");
        for (int g = done + hf; g < pnow; g += 2) {
          const int p = g * kBsB + r;
          if (p < n) __stcg(gx + orig(p), S.ring[(g % kBsR) * kBsB + r]);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          bs_st_release_u64(F.gprog, (static_cast<unsigned long long>(F.tag) << 32) | static_cast<unsigned>(pnow));
          *S.pubdone = pnow;
        }
        done = pnow;
        sg.t0 = clock64();
      } else if (sg.expired()) {
        break;
      }
    }
  } else if (F.workers == 0 && (warp & 3) != (mainw & 3)) {
    // no far-worker CTAs: the spare warps off the main warp's sub-partition
    int idx = 0, cnt = 0;
    for (int w = 0; w < nw; ++w) {
      bool role = w == mainw || w == pubw || w == prodw;
      for (int i = 0; i < kBsNC; ++i) role = role || w == (i < 3 ? i : 4);
      if (!role && (w & 3) != (mainw & 3)) {
        if (w == warp) idx = cnt;
        ++cnt;
      }
    }
    bs_far(s, gx, F, idx, cnt, abort_flag);
  }
  __syncthreads();
  if (threadIdx.x < ns) {
    const int sl = threadIdx.x;
    if (G > sl) S.base_use[sl] += (G - 1 - sl) / ns + 1;
  }
  __syncthreads();
}

}  // namespace dev
}  // namespace dsgpu
