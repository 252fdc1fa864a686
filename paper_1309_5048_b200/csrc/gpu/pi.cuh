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
                         unsigned* ab, double& rho0, double& rho1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nsteps = max(act0 ? P0.nb : 0, act1 ? P1.nb : 0);
  constexpr int kIn = FWD ? 1 : 3, kBase = FWD ? 0 : 2;
  for (int t = 0; t < nsteps; ++t) {
    const PiStep S0 = pi_step<FWD>(P0, act0, t, cta, G);
    const PiStep S1 = pi_step<FWD>(P1, act1, t, cta, G);
    const int nj0 = S0.hi - S0.lo, nj = nj0 + S1.hi - S1.lo;
    // prefetch this warp's first row: coefficients (cp.async into its shared-
    // memory slot) and base value, both before waiting for the window
    double bse = 0.0;
    double* cs = ws + P0.cbase + warp * P0.cslot;
    const bool pre = warp < nj && P0.cslot > 0;
    if (warp < nj) {
      const bool q = warp >= nj0;
      const DPi& P = q ? P1 : P0;
      const int row = q ? S1.lo + warp - nj0 : S0.lo + warp;
      const int w = q ? S1.wl : S0.wl;
      const PiBlk& B = P.blk[q ? S1.i : S0.i];
      const double* cr = P.coef + (FWD ? B.f : B.h) + static_cast<int64_t>(row - B.s) * w;
      if (pre) {
        for (int k = lane; k < w; k += 32) {
          const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(cs + k));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(cr + k) : "memory");
        }
      }
      if (lane == 0) bse = pi_wait(P.set[par] + kBase * P.n + row, ab);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // stage the windows: block 0 at ws[0, wl0), block 1 at ws[wl0, wl0 + wl1)
    __syncthreads();  // the previous step's readers of ws are done
    if (S0.wl > 0) pi_stage(ws, P0.set[par] + kIn * P0.n + S0.wlo, S0.wl, ab);
    if (S1.wl > 0) pi_stage(ws + S0.wl, P1.set[par] + kIn * P1.n + S1.wlo, S1.wl, ab);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int j = warp; j < nj; j += nw) {
      const bool q = j >= nj0;
      const DPi& P = q ? P1 : P0;
      const int row = q ? S1.lo + j - nj0 : S0.lo + j;
      const int w = q ? S1.wl : S0.wl;
      const PiBlk& B = P.blk[q ? S1.i : S0.i];
      const double* wsb = ws + (q ? S0.wl : 0);
      double acc = 0.0;
      if (j == warp && pre) {
        for (int k = lane; k < w; k += 32) acc = fma(cs[k], wsb[k], acc);
      } else {
        const double* cr = P.coef + (FWD ? B.f : B.h) + static_cast<int64_t>(row - B.s) * w;
        for (int k = lane; k < w; k += 32) acc = fma(__ldg(cr + k), wsb[k], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        const double base = j == warp ? bse : pi_wait(P.set[par] + kBase * P.n + row, ab);
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
  }
}

__device__ __forceinline__ void pi_reset(const DPi& P, unsigned set, int cta, int G) {
  unsigned long long* o = reinterpret_cast<unsigned long long*>(P.set[set]);
  for (int k = cta * blockDim.x + threadIdx.x; k < 4 * P.n; k += G * blockDim.x) o[k] = kSentinel;
}

// Full apply for the active blocks (every thread of every CTA). rho0/rho1:
// this warp's partial <r, z> (lane 0), to be reduced by the caller.
__device__ void pi_apply(const DPi& P0, const DPi& P1, bool act0, bool act1, const PiRhs& rhs0,
                         const PiRhs& rhs1, double* zc0, double* zc1, unsigned par, int cta, int G, double* ws,
                         unsigned* ab, double& rho0, double& rho1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gw = cta * nw + warp, gws = G * nw;
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
  pi_chain<true>(P0, P1, act0, act1, rhs0, rhs1, zc0, zc1, par, cta, G, ws, ab, rho0, rho1);
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
  pi_chain<false>(P0, P1, act0, act1, rhs0, rhs1, zc0, zc1, par, cta, G, ws, ab, rho0, rho1);
}

}  // namespace dev
}  // namespace dsgpu
