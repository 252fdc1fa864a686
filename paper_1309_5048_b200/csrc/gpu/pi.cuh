// Device side of the partitioned-inverse IC(0) apply (layout: pi.hpp).
//
// Executed by every CTA of the persistent kernel (or of the standalone apply
// kernel) for one or both IC(0) blocks at once:
//   G  g = blockdiag(D^{-1}) r          rows interleaved over all warps
//   Y  y_i = g_i + F_i y[c_i, s_i)      chain over blocks; every CTA owns a
//                                       slice of each block's rows
//   H  h = blockdiag(D^{-T}) y          rows interleaved over all warps
//   Z  z_i = h_i + H_i z[e_i, v_i)      chain, descending
// There are no barriers: g, y, h, z live in "sentinel" buffers (a NaN payload
// marks a value not yet written) and consumers poll the values themselves.
// Each chain step a CTA stages its window in shared memory (all threads poll
// in parallel) while its warps already hold the step's F/H rows in registers.
// Two buffer sets alternate between consecutive applies; an apply resets the
// set of the next one (its last readers finished before the grid barrier that
// separates consecutive applies).
#pragma once
#include "kernels.cuh"
#include "pi.hpp"

namespace dsgpu {
namespace dev {

struct DPi {
  int nb = 0, bsz = 0, n = 0, wmax = 0;
  int cbase = 0, cslot = 0;  // chain coefficient prefetch in shared memory: per-warp slot
                             // of cslot doubles at ws + cbase + warp * cslot (0: none)
  const PiBlk* blk = nullptr;
  const double* coef = nullptr;
  double* set[2] = {nullptr, nullptr};  // 4 n each: g | y | h | z
};

// r of block-local row k for the apply: preconditioner input (src0 + coef src1
// at global index off + k) or the PCG residual update r - alpha q.
struct PiRhs {
  const double* src0 = nullptr;
  const double* src1 = nullptr;
  double coef = 0.0;
  int off = 0;
  const double* r = nullptr;
  const double* q = nullptr;
  double na = 0.0;
  __device__ __forceinline__ double at(int k) const {
    if (r) return add_rn(r[k], mul_rn(na, q[k]));
    const int i = off + k;
    return src1 ? add_rn(src0[i], mul_rn(coef, src1[i])) : src0[i];
  }
};

// Timeline diagnostics (dsgpu_debug_pi_trace): when armed, CTA 0 and the last
// CTA record %globaltimer at every phase boundary of their next apply.
__device__ unsigned long long g_pi_trace[2][512];
__device__ int g_pi_trace_arm[2];
struct PiTrace {
  int slot = -1, k = 0;
  __device__ __forceinline__ void init(int cta, int G) {
    slot = cta == 0 ? 0 : (cta == G - 1 ? 1 : -1);
    if (slot >= 0 && !*reinterpret_cast<volatile int*>(&g_pi_trace_arm[slot])) slot = -1;
  }
  __device__ __forceinline__ void mark() {
    if (slot >= 0 && threadIdx.x == 0 && k < 511) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_pi_trace[slot][++k] = t;
      g_pi_trace[slot][0] = k;
    }
  }
  __device__ __forceinline__ void done() {
    if (slot >= 0 && threadIdx.x == 0) g_pi_trace_arm[slot] = 0;
  }
};

// Per-warp mbarriers for the chain rows' bulk copies (initialized once per
// kernel launch by pi_prologue; parity tracked in pi_mb_phase).
__shared__ __align__(8) uint64_t pi_mb[16];
__shared__ unsigned pi_mb_phase[16];
__device__ __forceinline__ unsigned pi_s32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// every thread of the CTA, once per launch before any apply
__device__ __forceinline__ void pi_prologue() {
  if (threadIdx.x < 16) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pi_s32(&pi_mb[threadIdx.x])) : "memory");
    pi_mb_phase[threadIdx.x] = 0u;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
}

__device__ __forceinline__ unsigned long long pi_ld(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pi_st(double* p, double x) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  if (b == kSentinel) b = kCanonNaN;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}
__device__ __forceinline__ double pi_wait(const double* p, unsigned* ab) {
  unsigned long long v = pi_ld(p);
  if (v != kSentinel) return __longlong_as_double(static_cast<long long>(v));
  SpinGuard g(ab);
  do {
    v = pi_ld(p);
    if (g.expired()) return __longlong_as_double(static_cast<long long>(kCanonNaN));
  } while (v == kSentinel);
  return __longlong_as_double(static_cast<long long>(v));
}

// every thread of the CTA: ws[0, len) = src[0, len), polling for sentinels
__device__ __forceinline__ void pi_stage(double* ws, const double* src, int len, unsigned* ab) {
  constexpr int U = 8;
  const int T = blockDim.x;
  for (int base = 0; base < len; base += U * T) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u * T + threadIdx.x;
      v[u] = k < len ? pi_ld(src + k) : 0ull;
    }
    bool miss = false;
#pragma unroll
    for (int u = 0; u < U; ++u) miss |= v[u] == kSentinel;
    if (miss) {
      SpinGuard g(ab);
      while (miss) {
        miss = false;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (v[u] == kSentinel) {
            v[u] = pi_ld(src + base + u * T + threadIdx.x);
            miss |= v[u] == kSentinel;
          }
        if (miss && g.expired()) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (v[u] == kSentinel) v[u] = kCanonNaN;
          miss = false;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u * T + threadIdx.x;
      if (k < len) ws[k] = __longlong_as_double(static_cast<long long>(v[u]));
    }
  }
}

// ---- G and H: dense block-diagonal products, warp per row ------------------
// g[row] = sum_{k <= rr} Dinv[rr][k] r(s + k)
__device__ __forceinline__ double pi_g_row(const DPi& P, const PiRhs& rhs, int row, int lane) {
  const int i = row / P.bsz;
  const PiBlk& B = P.blk[i];
  const int b = B.e - B.s, rr = row - B.s;
  const double* c = P.coef + B.dinv + static_cast<int64_t>(rr) * b;
  double acc = 0.0;
  constexpr int U = 8;
  for (int k0 = 0; k0 <= rr; k0 += 32 * U) {
    double cv[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * 32 + lane;
      cv[u] = k <= rr ? __ldg(c + k) : 0.0;
      xv[u] = k <= rr ? rhs.at(B.s + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(cv[u], xv[u], acc);
  }
  return warp_sum(acc);
}
// h[row] = sum_{k >= rr} DinvT[rr][k] y(s + k), y polled
__device__ __forceinline__ double pi_h_row(const DPi& P, const double* y, int row, int lane, unsigned* ab) {
  const int i = row / P.bsz;
  const PiBlk& B = P.blk[i];
  const int b = B.e - B.s, rr = row - B.s;
  const double* c = P.coef + B.dinvt + static_cast<int64_t>(rr) * b;
  double acc = 0.0;
  constexpr int U = 8;
  for (int k0 = rr; k0 < b; k0 += 32 * U) {
    double cv[U];
    unsigned long long xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * 32 + lane;
      cv[u] = k < b ? __ldg(c + k) : 0.0;
      xv[u] = k < b ? pi_ld(y + B.s + k) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * 32 + lane;
      double x = __longlong_as_double(static_cast<long long>(xv[u]));
      if (xv[u] == kSentinel) x = pi_wait(y + B.s + k, ab);
      acc = fma(cv[u], x, acc);
    }
  }
  return warp_sum(acc);
}

// window part of a chain row: sum_k c[k] ws[k], four independent accumulators
// (the fp64 FMA dependency chain is the row's latency)
__device__ __forceinline__ double pi_win(const double* c, const double* ws, int w, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = lane;
  for (; k + 96 < w; k += 128) {
    a0 = fma(c[k], ws[k], a0);
    a1 = fma(c[k + 32], ws[k + 32], a1);
    a2 = fma(c[k + 64], ws[k + 64], a2);
    a3 = fma(c[k + 96], ws[k + 96], a3);
  }
  for (; k < w; k += 32) a0 = fma(c[k], ws[k], a0);
  return (a0 + a1) + (a2 + a3);
}
__device__ __forceinline__ double pi_win_g(const double* __restrict__ c, const double* ws, int w, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = lane;
  for (; k + 96 < w; k += 128) {
    a0 = fma(__ldg(c + k), ws[k], a0);
    a1 = fma(__ldg(c + k + 32), ws[k + 32], a1);
    a2 = fma(__ldg(c + k + 64), ws[k + 64], a2);
    a3 = fma(__ldg(c + k + 96), ws[k + 96], a3);
  }
  for (; k < w; k += 32) a0 = fma(__ldg(c + k), ws[k], a0);
  return (a0 + a1) + (a2 + a3);
}

// ---- chain ------------------------------------------------------------------
// Per-block view of one chain step for this CTA (scalars only: no arrays
// indexed at run time, which would live in local memory).
struct PiStep {
  int i = 0, lo = 0, hi = 0, wlo = 0, wl = 0;
};
template <bool FWD>
__device__ __forceinline__ PiStep pi_step(const DPi& P, bool act, int t, int cta, int G) {
  PiStep S;
  if (!act || t >= P.nb) return S;
  S.i = FWD ? t : P.nb - 1 - t;
  const PiBlk& B = P.blk[S.i];
  const int b = B.e - B.s;
  S.lo = B.s + static_cast<int>(static_cast<int64_t>(b) * cta / G);
  S.hi = B.s + static_cast<int>(static_cast<int64_t>(b) * (cta + 1) / G);
  S.wlo = FWD ? B.c : B.e;
  S.wl = FWD ? B.s - B.c : B.v - B.e;
  return S;
}

// One chain (FWD: y from g; else z from h) of the active blocks. Backward:
// rho0/rho1 accumulate rhs(row) * z(row) over the rows this CTA produced (lane
// 0 of each warp), zc0/zc1 receive a plain copy of z.
template <bool FWD>
__device__ void pi_chain(const DPi& P0, const DPi& P1, bool act0, bool act1, const PiRhs& rhs0,
                         const PiRhs& rhs1, double* zc0, double* zc1, unsigned par, int cta, int G, double* ws,
                         unsigned* ab, double& rho0, double& rho1, PiTrace& tr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nsteps = max(act0 ? P0.nb : 0, act1 ? P1.nb : 0);
  constexpr int kIn = FWD ? 1 : 3, kBase = FWD ? 0 : 2;
  for (int t = 0; t < nsteps; ++t) {
    const PiStep S0 = pi_step<FWD>(P0, act0, t, cta, G);
    const PiStep S1 = pi_step<FWD>(P1, act1, t, cta, G);
    const int nj0 = S0.hi - S0.lo, nj = nj0 + S1.hi - S1.lo;
    // prefetch this warp's first row, before waiting for the window: its
    // coefficients (one bulk copy into the warp's shared-memory slot) and
    // its base value
    unsigned long long bse_raw = 0ull;
    double* cs = ws + P0.cbase + warp * P0.cslot;
    const bool pre = warp < nj && P0.cslot > 0;
    if (warp < nj) {
      const bool q = warp >= nj0;
      const DPi& P = q ? P1 : P0;
      const int row = q ? S1.lo + warp - nj0 : S0.lo + warp;
      const int w = q ? S1.wl : S0.wl;
      const PiBlk& B = P.blk[q ? S1.i : S0.i];
      if (lane == 0) {
        if (pre && w > 0) {
          const unsigned bytes = static_cast<unsigned>(pi_ldw(w)) * 8u;
          const double* cr = P.coef + (FWD ? B.f : B.h) + static_cast<int64_t>(row - B.s) * pi_ldw(w);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pi_s32(&pi_mb[warp])),
                       "r"(bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  pi_s32(cs)),
              "l"(cr), "r"(bytes), "r"(pi_s32(&pi_mb[warp]))
              : "memory");
        }
        bse_raw = pi_ld(P.set[par] + kBase * P.n + row);  // checked after the stage
      }
    }
    // stage the windows: block 0 at ws[0, wl0), block 1 at ws[wl0, wl0 + wl1)
    __syncthreads();  // the previous step's readers of ws are done
    if (S0.wl > 0) pi_stage(ws, P0.set[par] + kIn * P0.n + S0.wlo, S0.wl, ab);
    if (S1.wl > 0) pi_stage(ws + S0.wl, P1.set[par] + kIn * P1.n + S1.wlo, S1.wl, ab);
    __syncthreads();
    tr.mark();
    for (int j = warp; j < nj; j += nw) {
      const bool q = j >= nj0;
      const DPi& P = q ? P1 : P0;
      const int row = q ? S1.lo + j - nj0 : S0.lo + j;
      const int w = q ? S1.wl : S0.wl;
      const PiBlk& B = P.blk[q ? S1.i : S0.i];
      const double* wsb = ws + (q ? S0.wl : 0);
      double acc;
      if (j == warp && pre) {
        if (w > 0) {  // wait for the bulk copy of the row
          const unsigned ph = pi_mb_phase[warp];
          unsigned ok = 0;
          while (!ok)
            asm volatile(
                "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                : "=r"(ok)
                : "r"(pi_s32(&pi_mb[warp])), "r"(ph)
                : "memory");
          __syncwarp();
          if (lane == 0) pi_mb_phase[warp] = ph ^ 1u;
        }
        acc = pi_win(cs, wsb, w, lane);
      } else {
        acc = pi_win_g(P.coef + (FWD ? B.f : B.h) + static_cast<int64_t>(row - B.s) * pi_ldw(w), wsb, w, lane);
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        const double base = (j == warp && bse_raw != kSentinel)
                                ? __longlong_as_double(static_cast<long long>(bse_raw))
                                : pi_wait(P.set[par] + kBase * P.n + row, ab);
        const double v = add_rn(base, acc);
        pi_st(P.set[par] + kIn * P.n + row, v);
        if (!FWD) {
          if (q) {
            zc1[row] = v;
            rho1 += rhs1.at(row) * v;
          } else {
            zc0[row] = v;
            rho0 += rhs0.at(row) * v;
          }
        }
      }
    }
    tr.mark();
  }
}

__device__ __forceinline__ void pi_reset(const DPi& P, unsigned set, int cta, int G) {
  unsigned long long* o = reinterpret_cast<unsigned long long*>(P.set[set]);
  for (int k = cta * blockDim.x + threadIdx.x; k < 4 * P.n; k += G * blockDim.x) o[k] = kSentinel;
}

// Full apply for the active blocks (every thread of every CTA). rho0/rho1:
// this warp's partial <r, z> (lane 0), to be reduced by the caller.
__device__ __forceinline__ void pi_apply(const DPi& P0, const DPi& P1, bool act0, bool act1, const PiRhs& rhs0,
                         const PiRhs& rhs1, double* zc0, double* zc1, unsigned par, int cta, int G, double* ws,
                         unsigned* ab, double& rho0, double& rho1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gw = cta * nw + warp, gws = G * nw;
  PiTrace tr;
  tr.init(cta, G);
  tr.mark();
  // reset the other buffer set (the next apply's) of every PI block, active
  // or not: the parity advances for both blocks on every apply
  if (P0.n) pi_reset(P0, par ^ 1u, cta, G);
  if (P1.n) pi_reset(P1, par ^ 1u, cta, G);
  if (act0)
    for (int row = gw; row < P0.n; row += gws) {
      const double v = pi_g_row(P0, rhs0, row, lane);
      if (lane == 0) pi_st(P0.set[par] + row, v);
    }
  if (act1)
    for (int row = gw; row < P1.n; row += gws) {
      const double v = pi_g_row(P1, rhs1, row, lane);
      if (lane == 0) pi_st(P1.set[par] + row, v);
    }
  tr.mark();
  pi_chain<true>(P0, P1, act0, act1, rhs0, rhs1, zc0, zc1, par, cta, G, ws, ab, rho0, rho1, tr);
  if (act0)
    for (int row = gw; row < P0.n; row += gws) {
      const double v = pi_h_row(P0, P0.set[par] + P0.n, row, lane, ab);
      if (lane == 0) pi_st(P0.set[par] + 2 * P0.n + row, v);
    }
  if (act1)
    for (int row = gw; row < P1.n; row += gws) {
      const double v = pi_h_row(P1, P1.set[par] + P1.n, row, lane, ab);
      if (lane == 0) pi_st(P1.set[par] + 2 * P1.n + row, v);
    }
  tr.mark();
  pi_chain<false>(P0, P1, act0, act1, rhs0, rhs1, zc0, zc1, par, cta, G, ws, ab, rho0, rho1, tr);
  tr.done();
}

}  // namespace dev
}  // namespace dsgpu
