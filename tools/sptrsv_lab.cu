// Exploration harness for the single-CTA dataflow triangular sweep (not part of
// the product). Builds the BASELINE C2 IC(0) factor through the native host
// library, then times sweep variants with CUDA events and reports the SM clock
// seen inside the kernel (clock64 vs globaltimer).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <type_traits>
#include "dshost.h"
#include "../paper_1309_5048_b200/csrc/gpu/dsgpu_internal.hpp"
#include "../paper_1309_5048_b200/csrc/gpu/kernels.cuh"
using namespace dsgpu;
using namespace dsgpu::dev;

struct S { int n_groups; const int64_t* gptr; const int32_t* gwidth; const int32_t* grows; const int32_t* cols; const double* vals; const double* diag; };

__device__ __forceinline__ unsigned long long gtimer() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <int MODE>
__device__ __forceinline__ double waitv(const double* xs, int c, unsigned* ab) {
  const volatile unsigned long long* p = reinterpret_cast<const volatile unsigned long long*>(xs);
  unsigned long long b = p[c];
  if (MODE == 0) { while (b == kSentinel) b = p[c]; }
  else if (MODE == 1) { while (b == kSentinel) { __nanosleep(20); b = p[c]; } }
  else { return slot_wait(xs, c, ab); }
  return __longlong_as_double((long long)b);
}

template <int MODE>
__global__ void __launch_bounds__(1024,1) sweep_k(S s, int n, const double* r, double* out, unsigned* ab, unsigned long long* t) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  unsigned long long c0 = clock64(), g0 = gtimer();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    const int row = s.grows[(int64_t)g * 32 + lane];
    double acc = row >= 0 ? r[row] : 0.0;
    const int width = s.gwidth[g];
    const int32_t* cp = s.cols + s.gptr[g] + lane;
    const double* vp = s.vals + s.gptr[g] + lane;
    int k = 0;
    for (; k + 4 <= width; k += 4) {
      const int a0 = cp[0], a1 = cp[32], a2 = cp[64], a3 = cp[96];
      const double v0 = vp[0], v1 = vp[32], v2 = vp[64], v3 = vp[96];
      cp += 128; vp += 128;
      if (a0 >= 0) acc = sub_rn(acc, mul_rn(v0, waitv<MODE>(xs, a0, ab)));
      if (a1 >= 0) acc = sub_rn(acc, mul_rn(v1, waitv<MODE>(xs, a1, ab)));
      if (a2 >= 0) acc = sub_rn(acc, mul_rn(v2, waitv<MODE>(xs, a2, ab)));
      if (a3 >= 0) acc = sub_rn(acc, mul_rn(v3, waitv<MODE>(xs, a3, ab)));
    }
    for (; k < width; ++k) { const int a0 = cp[0]; const double v0 = vp[0]; cp += 32; vp += 32;
      if (a0 >= 0) acc = sub_rn(acc, mul_rn(v0, waitv<MODE>(xs, a0, ab))); }
    if (row >= 0) { const double xi = div_rn(acc, s.diag[row]); slot_publish(xs, row, xi); out[row] = xi; }
  }
  __syncthreads();
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}

// no-dependency variant: measures pure streaming of the group data (throughput bound)
__global__ void __launch_bounds__(1024,1) stream_k(S s, int n, const double* r, double* out, unsigned long long* t) {
  unsigned long long c0 = clock64(), g0 = gtimer();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    const int row = s.grows[(int64_t)g * 32 + lane];
    double acc = row >= 0 ? r[row] : 0.0;
    const int width = s.gwidth[g];
    const int32_t* cp = s.cols + s.gptr[g] + lane;
    const double* vp = s.vals + s.gptr[g] + lane;
    for (int k = 0; k < width; ++k) { const int a0 = cp[0]; const double v0 = vp[0]; cp += 32; vp += 32;
      if (a0 >= 0) acc = sub_rn(acc, mul_rn(v0, r[a0])); }
    if (row >= 0) out[row] = div_rn(acc, s.diag[row]);
  }
  __syncthreads();
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v2: compact group layout + register-preloaded tail --------------------
constexpr int TAIL = 4;
struct S2 { int n_groups; const int64_t* gptr; const int32_t* gnrow; const int32_t* gpw; const int32_t* grows; const int32_t* cols; const double* vals; const double* diag; const double* dinv; };
struct H2 { std::vector<int64_t> gptr; std::vector<int32_t> gnrow, gpw, grows, cols; std::vector<double> vals; };
H2 build2(const HostSweep& s) {
  // rebuild from the SELL-32 arrays of HostSweep (rows' entries in order)
  H2 h; h.gptr.push_back(0);
  for (int g = 0; g < s.n_groups; ++g) {
    int nrow = 0; for (int l = 0; l < 32; ++l) if (s.grows[g*32+l] >= 0) nrow = l + 1;
    std::vector<std::vector<std::pair<int,double>>> rows(nrow);
    for (int l = 0; l < nrow; ++l) for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) rows[l].push_back({s.cols[e], s.vals[e]}); }
    int pw = 0; for (auto& r : rows) pw = std::max<int>(pw, (int)r.size() - TAIL);
    h.gnrow.push_back(nrow); h.gpw.push_back(pw);
    for (int l = 0; l < 32; ++l) h.grows.push_back(s.grows[g*32+l]);
    int64_t base = h.gptr.back(); int64_t sz = (int64_t)(pw + TAIL) * nrow;
    h.cols.resize(base + sz, -1); h.vals.resize(base + sz, 0.0);
    for (int l = 0; l < nrow; ++l) { auto& r = rows[l]; int len = r.size(); int tl = std::min(len, TAIL); int pl = len - tl;
      for (int k = 0; k < pl; ++k) { h.cols[base + (int64_t)k*nrow + l] = r[k].first; h.vals[base + (int64_t)k*nrow + l] = r[k].second; }
      for (int t = 0; t < tl; ++t) { int slot = TAIL - tl + t; h.cols[base + (int64_t)(pw+slot)*nrow + l] = r[pl+t].first; h.vals[base + (int64_t)(pw+slot)*nrow + l] = r[pl+t].second; } }
    h.gptr.push_back(base + sz);
  }
  return h;
}
template <bool RECIP, int CH>
__global__ void __launch_bounds__(1024,1) sweep2(S2 s, int n, const double* __restrict__ r, double* out, unsigned* ab, unsigned long long* t) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  unsigned long long c0 = clock64(), g0 = gtimer();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
    const bool act = lane < nrow;
    const int64_t base = __ldg(s.gptr + g);
    int row = -1; double acc = 0.0, d = 1.0;
    int tc[TAIL]; double tv[TAIL];
    if (act) {
      row = __ldg(s.grows + (int64_t)g*32 + lane); acc = r[row]; d = RECIP ? __ldg(s.dinv + row) : __ldg(s.diag + row);
#pragma unroll
      for (int q = 0; q < TAIL; ++q) { tc[q] = __ldg(s.cols + base + (int64_t)(pw+q)*nrow + lane); tv[q] = __ldg(s.vals + base + (int64_t)(pw+q)*nrow + lane); }
      const int32_t* cp = s.cols + base + lane; const double* vp = s.vals + base + lane;
      int k = 0;
      for (; k + CH <= pw; k += CH) {
        int c[CH]; double v[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) { c[q] = __ldg(cp + (int64_t)q*nrow); v[q] = __ldg(vp + (int64_t)q*nrow); }
        cp += (int64_t)CH*nrow; vp += (int64_t)CH*nrow;
#pragma unroll
        for (int q = 0; q < CH; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], waitv<0>(xs, c[q], ab)));
      }
      for (; k < pw; ++k) { const int c0_ = __ldg(cp); const double v0 = __ldg(vp); cp += nrow; vp += nrow; if (c0_ >= 0) acc = sub_rn(acc, mul_rn(v0, waitv<0>(xs, c0_, ab))); }
#pragma unroll
      for (int q = 0; q < TAIL; ++q) if (tc[q] >= 0) acc = sub_rn(acc, mul_rn(tv[q], waitv<0>(xs, tc[q], ab)));
      const double xi = RECIP ? mul_rn(acc, d) : div_rn(acc, d);
      slot_publish(xs, row, xi); out[row] = xi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v3: mbarrier hardware-sleep waits (one barrier per row) --------------
__device__ __forceinline__ void mb_init(uint64_t* mb, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(mb)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* mb) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" :: "r"((unsigned)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, unsigned parity) {
  asm volatile("{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1; @!P bra WAIT_%=; }"
               :: "r"((unsigned)__cvta_generic_to_shared(mb)), "r"(parity) : "memory");
}
template <int SLEEPNS>
__device__ __forceinline__ double wait3(const double* xs, uint64_t* mb, int c, unsigned par) {
  const volatile unsigned long long* p = reinterpret_cast<const volatile unsigned long long*>(xs);
  unsigned long long b = p[c];
  if (b != kSentinel) return __longlong_as_double((long long)b);
  if (SLEEPNS < 0) { mb_wait(mb + c, par); b = p[c]; }
  else { while (b == kSentinel) { if (SLEEPNS) __nanosleep(SLEEPNS); b = p[c]; } }
  return __longlong_as_double((long long)b);
}
template <int SLEEPNS>
__global__ void __launch_bounds__(1024,1) sweep3(S2 s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps) {
  extern __shared__ double xs[];
  uint64_t* mb = reinterpret_cast<uint64_t*>(xs + n);
  if (SLEEPNS < 0) for (int i = threadIdx.x; i < n; i += blockDim.x) mb_init(mb + i, 1);
  __syncthreads();
  unsigned long long c0 = 0, g0 = 0;
  for (int sw = 0; sw < nsweeps; ++sw) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
  const unsigned par = sw & 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
    const bool act = lane < nrow;
    const int64_t base = __ldg(s.gptr + g);
    if (act) {
      const int row = __ldg(s.grows + (int64_t)g*32 + lane); double acc = r[row]; const double d = __ldg(s.diag + row);
      int tc[TAIL]; double tv[TAIL];
#pragma unroll
      for (int q = 0; q < TAIL; ++q) { tc[q] = __ldg(s.cols + base + (int64_t)(pw+q)*nrow + lane); tv[q] = __ldg(s.vals + base + (int64_t)(pw+q)*nrow + lane); }
      const int32_t* cp = s.cols + base + lane; const double* vp = s.vals + base + lane;
      int k = 0;
      for (; k + 4 <= pw; k += 4) {
        int c[4]; double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q] = __ldg(cp + (int64_t)q*nrow); v[q] = __ldg(vp + (int64_t)q*nrow); }
        cp += (int64_t)4*nrow; vp += (int64_t)4*nrow;
#pragma unroll
        for (int q = 0; q < 4; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], wait3<SLEEPNS>(xs, mb, c[q], par)));
      }
      for (; k < pw; ++k) { const int c0_ = __ldg(cp); const double v0 = __ldg(vp); cp += nrow; vp += nrow; if (c0_ >= 0) acc = sub_rn(acc, mul_rn(v0, wait3<SLEEPNS>(xs, mb, c0_, par))); }
#pragma unroll
      for (int q = 0; q < TAIL; ++q) if (tc[q] >= 0) acc = sub_rn(acc, mul_rn(tv[q], wait3<SLEEPNS>(xs, mb, tc[q], par)));
      const double xi = div_rn(acc, d);
      slot_publish(xs, row, xi);
      if (SLEEPNS < 0) mb_arrive(mb + row);
      out[row] = xi;
    }
  }
  __syncthreads();
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v4: instrumented v3-spin (timestamps per group) -----------------------
__global__ void __launch_bounds__(1024,1) sweep4(S2 s, int n, const double* __restrict__ r, double* out, long long* ts, int nsweeps) {
  extern __shared__ double xs[];
  for (int sw = 0; sw < nsweeps; ++sw) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  const long long T0 = clock64();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    long long tA = clock64() - T0;
    const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
    const bool act = lane < nrow;
    const int64_t base = __ldg(s.gptr + g);
    long long tB = 0, tC = 0;
    if (act) {
      const int row = __ldg(s.grows + (int64_t)g*32 + lane); double acc = r[row]; const double d = __ldg(s.diag + row);
      int tc[TAIL]; double tv[TAIL];
#pragma unroll
      for (int q = 0; q < TAIL; ++q) { tc[q] = __ldg(s.cols + base + (int64_t)(pw+q)*nrow + lane); tv[q] = __ldg(s.vals + base + (int64_t)(pw+q)*nrow + lane); }
      const int32_t* cp = s.cols + base + lane; const double* vp = s.vals + base + lane;
      int k = 0;
      for (; k + 4 <= pw; k += 4) {
        int c[4]; double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q] = __ldg(cp + (int64_t)q*nrow); v[q] = __ldg(vp + (int64_t)q*nrow); }
        cp += (int64_t)4*nrow; vp += (int64_t)4*nrow;
#pragma unroll
        for (int q = 0; q < 4; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], wait3<0>(xs, nullptr, c[q], 0)));
      }
      for (; k < pw; ++k) { const int c0_ = __ldg(cp); const double v0 = __ldg(vp); cp += nrow; vp += nrow; if (c0_ >= 0) acc = sub_rn(acc, mul_rn(v0, wait3<0>(xs, nullptr, c0_, 0))); }
      tB = clock64() - T0;
#pragma unroll
      for (int q = 0; q < TAIL; ++q) if (tc[q] >= 0) acc = sub_rn(acc, mul_rn(tv[q], wait3<0>(xs, nullptr, tc[q], 0)));
      tC = clock64() - T0;
      const double xi = div_rn(acc, d);
      slot_publish(xs, row, xi);
      out[row] = xi;
    }
    long long tD = clock64() - T0;
    if (sw == nsweeps - 1 && lane == 0) { ts[g*4+0] = tA; ts[g*4+1] = tB; ts[g*4+2] = tC; ts[g*4+3] = tD; }
  }
  __syncthreads();
  }
}
__global__ void chase(const int32_t* nxt, int steps, long long* out) {
  int j = 0; long long t0 = clock64();
  for (int i = 0; i < steps; ++i) j = __ldg(nxt + j);
  out[0] = clock64() - t0; out[1] = j;
}


// ---- v5: v3-spin + L1 prefetch of the whole group (and optionally the next) ----
__device__ __forceinline__ void pf_l1(const void* a) { asm volatile("prefetch.global.L1 [%0];" :: "l"(a)); }
__device__ __forceinline__ void prefetch_group(const S2& s, int g, int lane) {
  const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
  const int64_t base = __ldg(s.gptr + g);
  const int64_t cnt = (int64_t)(pw + TAIL) * nrow;
  const char* c0 = reinterpret_cast<const char*>(s.cols + base);
  const char* v0 = reinterpret_cast<const char*>(s.vals + base);
  for (int64_t b = (int64_t)lane * 128; b < cnt * 4 + 128; b += 32 * 128) pf_l1(c0 + b);
  for (int64_t b = (int64_t)lane * 128; b < cnt * 8 + 128; b += 32 * 128) pf_l1(v0 + b);
}
template <int NEXT>
__global__ void __launch_bounds__(1024,1) sweep5(S2 s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps) {
  extern __shared__ double xs[];
  unsigned long long c0 = 0, g0 = 0;
  for (int sw = 0; sw < nsweeps; ++sw) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (NEXT) prefetch_group(s, warp, lane);
  for (int g = warp; g < s.n_groups; g += nw) {
    if (NEXT) { if (g + nw < s.n_groups) prefetch_group(s, g + nw, lane); }
    else prefetch_group(s, g, lane);
    const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
    const bool act = lane < nrow;
    const int64_t base = __ldg(s.gptr + g);
    if (act) {
      const int row = __ldg(s.grows + (int64_t)g*32 + lane); double acc = r[row]; const double d = __ldg(s.diag + row);
      int tc[TAIL]; double tv[TAIL];
#pragma unroll
      for (int q = 0; q < TAIL; ++q) { tc[q] = s.cols[base + (int64_t)(pw+q)*nrow + lane]; tv[q] = s.vals[base + (int64_t)(pw+q)*nrow + lane]; }
      const int32_t* cp = s.cols + base + lane; const double* vp = s.vals + base + lane;
      int k = 0;
      for (; k + 4 <= pw; k += 4) {
        int c[4]; double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q] = cp[(int64_t)q*nrow]; v[q] = vp[(int64_t)q*nrow]; }
        cp += (int64_t)4*nrow; vp += (int64_t)4*nrow;
#pragma unroll
        for (int q = 0; q < 4; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], wait3<0>(xs, nullptr, c[q], 0)));
      }
      for (; k < pw; ++k) { const int c0_ = *cp; const double v0 = *vp; cp += nrow; vp += nrow; if (c0_ >= 0) acc = sub_rn(acc, mul_rn(v0, wait3<0>(xs, nullptr, c0_, 0))); }
#pragma unroll
      for (int q = 0; q < TAIL; ++q) if (tc[q] >= 0) acc = sub_rn(acc, mul_rn(tv[q], wait3<0>(xs, nullptr, tc[q], 0)));
      const double xi = div_rn(acc, d);
      slot_publish(xs, row, xi);
      out[row] = xi;
    }
  }
  __syncthreads();
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v6: entries in dependency-level order (not bit-exact), 8-entry register tail ----
constexpr int TAIL6 = 8;
H2 build6(const HostSweep& s, std::vector<int>& lev_out) {
  // level of each row from the group order
  int n = s.n; std::vector<int> lev(n, 0);
  for (int g = 0; g < s.n_groups; ++g) for (int l = 0; l < 32; ++l) { int r = s.grows[g*32+l]; if (r >= 0) {
      int lv = 0; for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) lv = std::max(lv, lev[s.cols[e]] + 1); } lev[r] = lv; } }
  lev_out = lev;
  H2 h; h.gptr.push_back(0);
  for (int g = 0; g < s.n_groups; ++g) {
    int nrow = 0; for (int l = 0; l < 32; ++l) if (s.grows[g*32+l] >= 0) nrow = l + 1;
    std::vector<std::vector<std::pair<int,double>>> rows(nrow);
    for (int l = 0; l < nrow; ++l) { for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) rows[l].push_back({s.cols[e], s.vals[e]}); }
      std::stable_sort(rows[l].begin(), rows[l].end(), [&](auto& a, auto& b) { return lev[a.first] < lev[b.first]; }); }
    int pw = 0; for (auto& r : rows) pw = std::max<int>(pw, (int)r.size() - TAIL6);
    h.gnrow.push_back(nrow); h.gpw.push_back(pw);
    for (int l = 0; l < 32; ++l) h.grows.push_back(s.grows[g*32+l]);
    int64_t base = h.gptr.back(); int64_t sz = (int64_t)(pw + TAIL6) * nrow;
    h.cols.resize(base + sz, -1); h.vals.resize(base + sz, 0.0);
    for (int l = 0; l < nrow; ++l) { auto& r = rows[l]; int len = r.size(); int tl = std::min(len, TAIL6); int pl = len - tl;
      for (int k = 0; k < pl; ++k) { h.cols[base + (int64_t)k*nrow + l] = r[k].first; h.vals[base + (int64_t)k*nrow + l] = r[k].second; }
      for (int t = 0; t < tl; ++t) { int slot = TAIL6 - tl + t; h.cols[base + (int64_t)(pw+slot)*nrow + l] = r[pl+t].first; h.vals[base + (int64_t)(pw+slot)*nrow + l] = r[pl+t].second; } }
    h.gptr.push_back(base + sz);
  }
  return h;
}
template <bool RECIP, bool PF>
__global__ void __launch_bounds__(1024,1) sweep6(S2 s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* ts) {
  extern __shared__ double xs[];
  unsigned long long c0 = 0, g0 = 0;
  for (int sw = 0; sw < nsweeps; ++sw) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
  const long long T0 = clock64();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < s.n_groups; g += nw) {
    if (PF && g + nw < s.n_groups) prefetch_group(s, g + nw, lane);
    long long tA = clock64() - T0, tB = 0, tC = 0;
    const int nrow = __ldg(s.gnrow + g), pw = __ldg(s.gpw + g);
    const bool act = lane < nrow;
    const int64_t base = __ldg(s.gptr + g);
    if (act) {
      const int row = __ldg(s.grows + (int64_t)g*32 + lane); double acc = r[row]; const double d = RECIP ? __ldg(s.dinv + row) : __ldg(s.diag + row);
      int tc[TAIL6]; double tv[TAIL6];
#pragma unroll
      for (int q = 0; q < TAIL6; ++q) { tc[q] = s.cols[base + (int64_t)(pw+q)*nrow + lane]; tv[q] = s.vals[base + (int64_t)(pw+q)*nrow + lane]; }
      const int32_t* cp = s.cols + base + lane; const double* vp = s.vals + base + lane;
      int k = 0;
      for (; k + 4 <= pw; k += 4) {
        int c[4]; double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q] = cp[(int64_t)q*nrow]; v[q] = vp[(int64_t)q*nrow]; }
        cp += (int64_t)4*nrow; vp += (int64_t)4*nrow;
#pragma unroll
        for (int q = 0; q < 4; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], wait3<0>(xs, nullptr, c[q], 0)));
      }
      for (; k < pw; ++k) { const int c0_ = *cp; const double v0 = *vp; cp += nrow; vp += nrow; if (c0_ >= 0) acc = sub_rn(acc, mul_rn(v0, wait3<0>(xs, nullptr, c0_, 0))); }
      tB = clock64() - T0;
#pragma unroll
      for (int q = 0; q < TAIL6; ++q) if (tc[q] >= 0) acc = sub_rn(acc, mul_rn(tv[q], wait3<0>(xs, nullptr, tc[q], 0)));
      tC = clock64() - T0;
      const double xi = RECIP ? mul_rn(acc, d) : div_rn(acc, d);
      slot_publish(xs, row, xi);
      out[row] = xi;
    }
    long long tD = clock64() - T0;
    if (ts && sw == nsweeps - 1 && lane == 0) { ts[g*4+0] = tA; ts[g*4+1] = tB; ts[g*4+2] = tC; ts[g*4+3] = tD; }
  }
  __syncthreads();
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}
// pure chain: level l has one row (warp l%32, lane 0) depending on row l-1; register data
__global__ void __launch_bounds__(1024,1) chain7(int levels, unsigned long long* t, double* out) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < levels; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  unsigned long long c0 = clock64();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = warp; l < levels; l += nw) {
    if (lane < 8) {
      double acc = 1.0;
      if (l > 0) acc = sub_rn(acc, mul_rn(0.5, wait3<0>(xs, nullptr, l - 1, 0)));
      const double xi = div_rn(acc, 1.0001);
      if (lane == 0) slot_publish(xs, l, xi);
      out[l] = xi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) t[0] = clock64() - c0;
}


template <bool RECIP, int SLEEP>
__global__ void chain8(int levels, unsigned long long* t, double* out) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < levels; i += blockDim.x) slot_reset(xs, i);
  __syncthreads();
  unsigned long long c0 = clock64();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = warp; l < levels; l += nw) {
    if (lane == 0) {
      double acc = 1.0;
      if (l > 0) {
        const volatile unsigned long long* p = reinterpret_cast<const volatile unsigned long long*>(xs);
        unsigned long long b = p[l-1];
        while (b == kSentinel) { if (SLEEP) __nanosleep(SLEEP); b = p[l-1]; }
        acc = sub_rn(acc, mul_rn(0.5, __longlong_as_double((long long)b)));
      }
      const double xi = RECIP ? mul_rn(acc, 0.9999) : div_rn(acc, 1.0001);
      slot_publish(xs, l, xi);
      out[l] = xi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) t[0] = clock64() - c0;
}
// single warp, sequential levels, value passed in registers (floor of the math chain)
template <bool RECIP>
__global__ void chain9(int levels, unsigned long long* t, double* out) {
  unsigned long long c0 = clock64();
  double x = 0.0;
  for (int l = 0; l < levels; ++l) { double acc = sub_rn(1.0, mul_rn(0.5, x)); x = RECIP ? mul_rn(acc, 0.9999) : div_rn(acc, 1.0001); }
  out[threadIdx.x] = x;
  t[0] = clock64() - c0;
}


// ---- v8: serial main warp + helper warps (prefix sums + staging) ------------
constexpr int R8 = 16;
struct H8 { int G, TW; std::vector<int32_t> nr, need, grows; std::vector<int64_t> pptr, tptr; std::vector<int32_t> pw, tw, pcols, tcols; std::vector<double> pvals, tvals; };
H8 build8(const HostSweep& s, int D) {
  int n = s.n; std::vector<int> lev(n, 0);
  // rows with their entries in stored (column) order, from the SELL-32 arrays
  std::vector<std::vector<std::pair<int,double>>> rows(n);
  std::vector<int> order;
  for (int g = 0; g < s.n_groups; ++g) for (int l = 0; l < 32; ++l) { int r = s.grows[g*32+l]; if (r < 0) continue;
      order.push_back(r);
      for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) rows[r].push_back({s.cols[e], s.vals[e]}); } }
  for (int r : order) { int lv = 0; for (auto& e : rows[r]) lv = std::max(lv, lev[e.first] + 1); lev[r] = lv; }
  // groups = HostSweep groups (<=32 rows of one level, level-ordered)
  H8 h; h.G = s.n_groups; std::vector<int> gof(n);
  for (int g = 0; g < s.n_groups; ++g) for (int l = 0; l < 32; ++l) { int r = s.grows[g*32+l]; if (r >= 0) gof[r] = g; }
  h.pptr.push_back(0); h.tptr.push_back(0); h.TW = 0;
  for (int g = 0; g < s.n_groups; ++g) {
    int nr = 0; for (int l = 0; l < 32; ++l) if (s.grows[g*32+l] >= 0) nr = l + 1;
    int pw = 0, tw = 0, need = -1;
    std::vector<int> split(nr);
    for (int l = 0; l < nr; ++l) { int r = s.grows[g*32+l]; auto& e = rows[r]; int L = lev[r]; int p = e.size();
      for (int k = 0; k < (int)e.size(); ++k) if (lev[e[k].first] > L - D) { p = k; break; }
      split[l] = p; pw = std::max(pw, p); tw = std::max(tw, (int)e.size() - p);
      for (int k = 0; k < p; ++k) need = std::max(need, gof[e[k].first]); }
    h.nr.push_back(nr); h.need.push_back(need); h.pw.push_back(pw); h.tw.push_back(tw); h.TW = std::max(h.TW, tw);
    for (int l = 0; l < 32; ++l) h.grows.push_back(s.grows[g*32+l]);
    int64_t pb = h.pptr.back(), tb = h.tptr.back();
    h.pcols.resize(pb + (int64_t)pw*nr, -1); h.pvals.resize(pb + (int64_t)pw*nr, 0.0);
    h.tcols.resize(tb + (int64_t)tw*nr, -1); h.tvals.resize(tb + (int64_t)tw*nr, 0.0);
    for (int l = 0; l < nr; ++l) { int r = s.grows[g*32+l]; auto& e = rows[r];
      for (int k = 0; k < split[l]; ++k) { h.pcols[pb + (int64_t)k*nr + l] = e[k].first; h.pvals[pb + (int64_t)k*nr + l] = e[k].second; }
      for (int k = split[l]; k < (int)e.size(); ++k) { h.tcols[tb + (int64_t)(k-split[l])*nr + l] = e[k].first; h.tvals[tb + (int64_t)(k-split[l])*nr + l] = e[k].second; } }
    h.pptr.push_back(pb + (int64_t)pw*nr); h.tptr.push_back(tb + (int64_t)tw*nr);
  }
  return h;
}
struct S8 { int G; const int32_t *nr, *need, *grows, *pw, *tw, *pcols, *tcols; const int64_t *pptr, *tptr; const double *pvals, *tvals, *diag; };
template <int TWMAX, bool RECIP8>
__global__ void __launch_bounds__(1024,1) sweep8(S8 s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg = nullptr) {
  extern __shared__ double sm[];
  double* xs = sm;                                   // n
  double* psum = xs + n;                             // R8*32
  double* dg = psum + R8*32;                         // R8*32
  double* tv = dg + R8*32;                           // R8*TWMAX*32
  int* tc = reinterpret_cast<int*>(tv + R8*TWMAX*32);// R8*TWMAX*32
  int* rows = tc + R8*TWMAX*32;                      // R8*32
  volatile int* ready = rows + R8*32;                // R8
  volatile int* progress = ready + R8;               // 1
  int* snr = const_cast<int*>(progress) + 4;         // R8
  int* stw = snr + R8;                               // R8
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R8; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) *progress = 0;
    __syncthreads();
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    long long waitc = 0;
    if (warp == 0) {
      // ---- main: serial over groups
      for (int g = 0; g < s.G; ++g) {
        const int sl = g % R8;
        long long w0 = clock64();
        while (ready[sl] != g) {}
        const long long w1 = clock64();
        waitc += w1 - w0;
        const int nr = snr[sl], tw = stw[sl];
        double x = 0.0; int orow = -1;
        if (lane < nr) {
          double acc = psum[sl*32 + lane];
          const int row = rows[sl*32 + lane];
#pragma unroll 4
          for (int k = 0; k < tw; ++k) { const int c = tc[(sl*TWMAX + k)*32 + lane]; if (c >= 0) acc = sub_rn(acc, mul_rn(tv[(sl*TWMAX + k)*32 + lane], xs[c])); }
          x = RECIP8 ? mul_rn(acc, dg[sl*32 + lane]) : div_rn(acc, dg[sl*32 + lane]);
          xs[row] = x; orow = row;
        }
        __syncwarp();
        const long long w2 = clock64();
        if (lane == 0) { __threadfence_block(); *progress = g + 1; }
        (void)orow;
        const long long w3 = clock64();
        if (lane == 0 && sw == nsweeps - 1 && tsg) { tsg[g*3+0] = w1 - w0; tsg[g*3+1] = w2 - w1; tsg[g*3+2] = w3 - w2; }
      }
      if (lane == 0 && sw == nsweeps - 1) t[2] = waitc;
    } else {
      // ---- helpers
      for (int g = warp - 1; g < s.G; g += nw - 1) {
        const int sl = g % R8;
        const int nr = __ldg(s.nr + g), pw = __ldg(s.pw + g), tw = __ldg(s.tw + g), need = __ldg(s.need + g);
        const int64_t pb = __ldg(s.pptr + g), tb = __ldg(s.tptr + g);
        int row = -1; double acc = 0.0, d = 1.0;
        int tcr[TWMAX]; double tvr[TWMAX];
        if (lane < nr) {
          row = __ldg(s.grows + g*32 + lane); acc = r[row]; d = RECIP8 ? 1.0 / __ldg(s.diag + row) : __ldg(s.diag + row);
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) { tcr[k] = k < tw ? __ldg(s.tcols + tb + (int64_t)k*nr + lane) : -1; tvr[k] = k < tw ? __ldg(s.tvals + tb + (int64_t)k*nr + lane) : 0.0; }
        }
        // prefix needs groups <= need done by main
        while (*progress <= need) { __nanosleep(64); }
        if (lane < nr) {
          const int32_t* cp = s.pcols + pb + lane; const double* vp = s.pvals + pb + lane;
          int k = 0;
          for (; k + 4 <= pw; k += 4) {
            int c[4]; double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { c[q] = __ldg(cp + (int64_t)q*nr); v[q] = __ldg(vp + (int64_t)q*nr); }
            cp += 4*nr; vp += 4*nr;
#pragma unroll
            for (int q = 0; q < 4; ++q) if (c[q] >= 0) acc = sub_rn(acc, mul_rn(v[q], xs[c[q]]));
          }
          for (; k < pw; ++k) { const int c = __ldg(cp); const double v = __ldg(vp); cp += nr; vp += nr; if (c >= 0) acc = sub_rn(acc, mul_rn(v, xs[c])); }
        }
        // slot free? (group g - R8 consumed)
        while (*progress < g - R8 + 1) { __nanosleep(64); }
        if (lane < nr) {
          psum[sl*32 + lane] = acc; dg[sl*32 + lane] = d; rows[sl*32 + lane] = row;
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) { tc[(sl*TWMAX + k)*32 + lane] = tcr[k]; tv[(sl*TWMAX + k)*32 + lane] = tvr[k]; }
        }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; stw[sl] = tw; __threadfence_block(); ready[sl] = g; }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v9: v8 with register-batched main tail and helper prefix chunks of 8; <=256 threads
template <int TWMAX, bool RECIP8, int MODE9 = 0>
__global__ void __launch_bounds__(256,1) sweep9(S8 s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg = nullptr) {
  extern __shared__ double sm[];
  double* xs = sm;
  double* psum = xs + n + 1;
  double* dg = psum + R8*32;
  double* tv = dg + R8*32;
  int* tc = reinterpret_cast<int*>(tv + R8*TWMAX*32);
  int* rows = tc + R8*TWMAX*32;
  volatile int* ready = rows + R8*32;
  volatile int* progress = ready + R8;
  int* snr = const_cast<int*>(progress) + 4;
  int* stw = snr + R8;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R8; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    if (warp == 0) {
      for (int g = 0; g < s.G; ++g) {
        const int sl = g % R8;
        const long long w0 = clock64();
        while (ready[sl] != g) {}
        const long long w1 = clock64();
        const int nr = snr[sl], tw = stw[sl];
        if (lane < nr) {
          double acc = psum[sl*32 + lane];
          const int row = rows[sl*32 + lane];
          const double d = dg[sl*32 + lane];
          int c[TWMAX]; double v[TWMAX], xv[TWMAX];
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) { c[k] = k < tw ? tc[(sl*TWMAX + k)*32 + lane] : -1; v[k] = k < tw ? tv[(sl*TWMAX + k)*32 + lane] : 0.0; }
          if (MODE9 == 0) {
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) xv[k] = c[k] >= 0 ? xs[c[k]] : 0.0;
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) if (c[k] >= 0) acc = sub_rn(acc, mul_rn(v[k], xv[k]));
          } else {
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) xv[k] = MODE9 == 1 ? xs[c[k] < 0 ? n : c[k]] : 0.5;
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) acc = sub_rn(acc, mul_rn(v[k], xv[k]));
          }
          xs[row] = RECIP8 ? mul_rn(acc, d) : div_rn(acc, d);
        }
        __syncwarp();
        const long long w2 = clock64();
        if (lane == 0) { __threadfence_block(); *progress = g + 1; }
        const long long w3 = clock64();
        if (lane == 0 && sw == nsweeps - 1 && tsg) { tsg[g*3+0] = w1 - w0; tsg[g*3+1] = w2 - w1; tsg[g*3+2] = w3 - w2; }
      }
    } else {
      for (int g = warp - 1; g < s.G; g += nw - 1) {
        const int sl = g % R8;
        const int nr = __ldg(s.nr + g), pw = __ldg(s.pw + g), tw = __ldg(s.tw + g), need = __ldg(s.need + g);
        const int64_t pb = __ldg(s.pptr + g), tb = __ldg(s.tptr + g);
        int row = -1; double acc = 0.0, d = 1.0;
        int tcr[TWMAX]; double tvr[TWMAX];
        if (lane < nr) {
          row = __ldg(s.grows + g*32 + lane); acc = r[row]; d = RECIP8 ? 1.0 / __ldg(s.diag + row) : __ldg(s.diag + row);
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) { tcr[k] = k < tw ? __ldg(s.tcols + tb + (int64_t)k*nr + lane) : -1; tvr[k] = k < tw ? __ldg(s.tvals + tb + (int64_t)k*nr + lane) : 0.0; }
        }
        // preload prefix chunk 0 before waiting
        constexpr int CH = 8;
        int pc[CH]; double pv[CH];
        const int32_t* cp = s.pcols + pb + lane; const double* vp = s.pvals + pb + lane;
        if (lane < nr) {
#pragma unroll
          for (int q = 0; q < CH; ++q) { pc[q] = q < pw ? __ldg(cp + (int64_t)q*nr) : -1; pv[q] = q < pw ? __ldg(vp + (int64_t)q*nr) : 0.0; }
        }
        while (*progress <= need) { __nanosleep(32); }
        if (lane < nr) {
          for (int k = 0; k < pw; k += CH) {
            int nc[CH]; double nv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) { const int kk = k + CH + q; nc[q] = kk < pw ? __ldg(cp + (int64_t)kk*nr) : -1; nv[q] = kk < pw ? __ldg(vp + (int64_t)kk*nr) : 0.0; }
            double xv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = pc[q] >= 0 ? xs[pc[q]] : 0.0;
#pragma unroll
            for (int q = 0; q < CH; ++q) if (pc[q] >= 0) acc = sub_rn(acc, mul_rn(pv[q], xv[q]));
#pragma unroll
            for (int q = 0; q < CH; ++q) { pc[q] = nc[q]; pv[q] = nv[q]; }
          }
        }
        while (*progress < g - R8 + 1) { __nanosleep(32); }
        if (lane < nr) {
          psum[sl*32 + lane] = acc; dg[sl*32 + lane] = d; rows[sl*32 + lane] = row;
#pragma unroll
          for (int k = 0; k < TWMAX; ++k) { tc[(sl*TWMAX + k)*32 + lane] = tcr[k]; tv[(sl*TWMAX + k)*32 + lane] = tvr[k]; }
        }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; stw[sl] = tw; __threadfence_block(); ready[sl] = g; }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v10: software-pipelined serial main warp (A(g+1) || B(g)), shuffles for
// deps on the previous group, helpers stage slots and far prefix sums ---------
constexpr int R10 = 16;
struct H10 { int G, TAm, TBm; std::vector<int32_t> nr, need, amax, bmax, grows, pw; std::vector<int64_t> pptr; std::vector<int32_t> pcols; std::vector<double> pvals;
             std::vector<int32_t> acol, bcol; std::vector<int8_t> bsrc; std::vector<double> aval, bval; };
template <int TA, int TB>
H10 build10(const HostSweep& s, int D, bool level_order) {
  int n = s.n; std::vector<int> lev(n, 0), gof(n), lof(n);
  std::vector<std::vector<std::pair<int,double>>> rows(n);
  for (int g = 0; g < s.n_groups; ++g) for (int l = 0; l < 32; ++l) { int r = s.grows[g*32+l]; if (r < 0) continue; gof[r] = g; lof[r] = l;
      for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) rows[r].push_back({s.cols[e], s.vals[e]}); } }
  if (level_order) for (int r = 0; r < n; ++r) std::stable_sort(rows[r].begin(), rows[r].end(), [&](auto& a, auto& b) { return gof[a.first] < gof[b.first]; });
  H10 h; h.G = s.n_groups; h.TAm = 0; h.TBm = 0; h.pptr.push_back(0);
  for (int g = 0; g < s.n_groups; ++g) {
    int nr = 0; for (int l = 0; l < 32; ++l) if (s.grows[g*32+l] >= 0) nr = l + 1;
    int pw = 0, need = -1, am = 0, bm = 0;
    std::vector<int> ps(nr), as(nr), bs(nr);
    for (int l = 0; l < nr; ++l) { int r = s.grows[g*32+l]; auto& e = rows[r]; int len = e.size();
      int cb = len; for (int k = 0; k < len; ++k) if (gof[e[k].first] == g - 1) { cb = k; break; }   // crit-tail start
      if (len - cb > TB) { printf("row %d crit tail %d > TB\n", r, len - cb); exit(1); }
      int ca = cb; for (int k = 0; k < cb; ++k) if (gof[e[k].first] > g - D) { ca = k; break; }     // pre-tail start
      if (cb - ca > TA) ca = cb - TA;
      ps[l] = ca; as[l] = cb - ca; bs[l] = len - cb;
      pw = std::max(pw, ca); am = std::max(am, cb - ca); bm = std::max(bm, len - cb);
      for (int k = 0; k < ca; ++k) need = std::max(need, gof[e[k].first]); }
    h.nr.push_back(nr); h.need.push_back(need); h.pw.push_back(pw); h.amax.push_back(am); h.bmax.push_back(bm);
    h.TAm = std::max(h.TAm, am); h.TBm = std::max(h.TBm, bm);
    for (int l = 0; l < 32; ++l) h.grows.push_back(s.grows[g*32+l]);
    int64_t pb = h.pptr.back(); h.pcols.resize(pb + (int64_t)pw*nr, -1); h.pvals.resize(pb + (int64_t)pw*nr, 0.0);
    size_t a0 = h.acol.size(); h.acol.resize(a0 + TA*32, n); h.aval.resize(a0 + TA*32, 0.0);   // pad: col n (xs[n] = 0), val 0
    size_t b0 = h.bcol.size(); h.bcol.resize(b0 + TB*32, n); h.bval.resize(b0 + TB*32, 0.0); h.bsrc.resize(b0 + TB*32, -1);
    for (int l = 0; l < nr; ++l) { int r = s.grows[g*32+l]; auto& e = rows[r];
      for (int k = 0; k < ps[l]; ++k) { h.pcols[pb + (int64_t)k*nr + l] = e[k].first; h.pvals[pb + (int64_t)k*nr + l] = e[k].second; }
      for (int k = 0; k < as[l]; ++k) { auto& x = e[ps[l] + k]; h.acol[a0 + k*32 + l] = x.first; h.aval[a0 + k*32 + l] = x.second; }
      for (int k = 0; k < bs[l]; ++k) { auto& x = e[ps[l] + as[l] + k]; h.bval[b0 + k*32 + l] = x.second;
        if (gof[x.first] == g - 1) { h.bsrc[b0 + k*32 + l] = (int8_t)lof[x.first]; h.bcol[b0 + k*32 + l] = n; } else h.bcol[b0 + k*32 + l] = x.first; } }
    h.pptr.push_back(pb + (int64_t)pw*nr);
  }
  return h;
}
struct S10d { int G; const int32_t *nr, *need, *amax, *bmax, *grows, *pw, *pcols, *acol, *bcol; const int8_t* bsrc; const int64_t* pptr; const double *pvals, *aval, *bval, *diag; };
template <int TA, int TB, bool MARK, int EXCL = 0>
__global__ void __launch_bounds__(512,1) sweep10(S10d s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg) {
  extern __shared__ double sm[];
  double* xs = sm;                                    // n + 1 (xs[n] = 0 pad)
  double* psum = xs + n + 1;                          // R*32
  double* dg = psum + R10*32;                         // R*32 (diag)
  double* av = dg + R10*32;                           // R*TA*32
  double* bv = av + R10*TA*32;                        // R*TB*32
  int* ac = reinterpret_cast<int*>(bv + R10*TB*32);   // R*TA*32
  int* bc = ac + R10*TA*32;                           // R*TB*32
  int* rows = bc + R10*TB*32;                         // R*32
  int8_t* bsr = reinterpret_cast<int8_t*>(rows + R10*32); // R*TB*32
  volatile int* meta = reinterpret_cast<volatile int*>(bsr + R10*TB*32); // ready[R], nr[R], amax[R], bmax[R], progress
  volatile int* ready = meta; int* snr = const_cast<int*>(meta) + R10; int* sam = snr + R10; int* sbm = sam + R10;
  volatile int* progress = meta + 4*R10;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R10; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    const int mainw = EXCL ? nw - 1 : 0;
    int hid = -1, nh = 0;   // helper index among helper warps
    for (int w = 0; w < nw; ++w) { const bool isH = (w != mainw) && !(EXCL == 2 && (w & 3) == (mainw & 3)); if (isH) { if (w == warp) hid = nh; ++nh; } }
    if (warp == mainw) {
      double xprev = 0.0;
      // state for group g (prepared by A)
      double acc_pre = 0.0, d = 1.0; int row = -1, nr = 0, bm = 0;
      double bvl[TB], bx[TB]; int bsl[TB];
      auto prep = [&](int g) {   // A(g): needs x of groups <= g-2 (already in xs)
        const int sl = g % R10;
        while (ready[sl] != g) {}
        nr = snr[sl]; const int am = sam[sl]; bm = sbm[sl];
        double acc = psum[sl*32 + lane];
        d = dg[sl*32 + lane]; row = rows[sl*32 + lane];
        int acl[TA]; double avl[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = ac[(sl*TA + k)*32 + lane]; avl[k] = av[(sl*TA + k)*32 + lane]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsr[(sl*TB + k)*32 + lane]; bvl[k] = bv[(sl*TB + k)*32 + lane]; bx[k] = xs[bc[(sl*TB + k)*32 + lane]]; }
        double axv[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) axv[k] = xs[acl[k]];
#pragma unroll
        for (int k = 0; k < TA; ++k) if (k < am) acc = sub_rn(acc, mul_rn(avl[k], axv[k]));
        acc_pre = acc;
      };
      prep(0);
      for (int g = 0; g < s.G; ++g) {
        const long long w0 = clock64();
        // B(g)
        double acc = acc_pre;
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          if (k < bm) {
            const double sx = __shfl_sync(0xffffffffu, xprev, bsl[k] < 0 ? 0 : bsl[k]);
            const double X = bsl[k] >= 0 ? sx : bx[k];
            acc = sub_rn(acc, mul_rn(bvl[k], X));
          }
        }
        double x;
        if (MARK) { const double q0 = mul_rn(acc, 1.0 / d); const double rr = fma(-q0, d, acc); x = fma(rr, 1.0 / d, q0); }
        else x = div_rn(acc, d);
        if (lane < nr) xs[row] = x;
        xprev = x;
        __syncwarp();
        if (lane == 0) *progress = g + 1;
        const long long w1 = clock64();
        if (g + 1 < s.G) prep(g + 1);
        const long long w2 = clock64();
        if (tsg && lane == 0 && sw == nsweeps - 1) { tsg[g*2] = w1 - w0; tsg[g*2+1] = w2 - w1; }
      }
    } else if (hid >= 0) {
      for (int g = hid; g < s.G; g += nh) {
        const int sl = g % R10;
        const int nr = __ldg(s.nr + g), pw = __ldg(s.pw + g), need = __ldg(s.need + g);
        const int64_t pb = __ldg(s.pptr + g);
        int row = -1; double acc = 0.0, dd = 1.0;
        if (lane < nr) { row = __ldg(s.grows + g*32 + lane); acc = r[row]; dd = __ldg(s.diag + row); }
        int acl[TA]; double avl[TA]; int bcl[TB]; double bvl[TB]; int8_t bsl[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = __ldg(s.acol + (int64_t)(g*TA + k)*32 + lane); avl[k] = __ldg(s.aval + (int64_t)(g*TA + k)*32 + lane); }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bcl[k] = __ldg(s.bcol + (int64_t)(g*TB + k)*32 + lane); bvl[k] = __ldg(s.bval + (int64_t)(g*TB + k)*32 + lane); bsl[k] = s.bsrc[(int64_t)(g*TB + k)*32 + lane]; }
        constexpr int CH = 8;
        int pc[CH]; double pv[CH];
        const int32_t* cp = s.pcols + pb + lane; const double* vp = s.pvals + pb + lane;
        if (lane < nr) {
#pragma unroll
          for (int q = 0; q < CH; ++q) { pc[q] = q < pw ? __ldg(cp + (int64_t)q*nr) : -1; pv[q] = q < pw ? __ldg(vp + (int64_t)q*nr) : 0.0; }
        }
        while (*progress <= need) { __nanosleep(32); }
        if (lane < nr) {
          for (int k = 0; k < pw; k += CH) {
            int nc[CH]; double nv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) { const int kk = k + CH + q; nc[q] = kk < pw ? __ldg(cp + (int64_t)kk*nr) : -1; nv[q] = kk < pw ? __ldg(vp + (int64_t)kk*nr) : 0.0; }
            double xv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = xs[pc[q] < 0 ? n : pc[q]];
#pragma unroll
            for (int q = 0; q < CH; ++q) if (pc[q] >= 0) acc = sub_rn(acc, mul_rn(pv[q], xv[q]));
#pragma unroll
            for (int q = 0; q < CH; ++q) { pc[q] = nc[q]; pv[q] = nv[q]; }
          }
        }
        while (*progress < g - R10 + 2) { __nanosleep(32); }
        psum[sl*32 + lane] = acc; dg[sl*32 + lane] = dd; rows[sl*32 + lane] = row;
#pragma unroll
        for (int k = 0; k < TA; ++k) { ac[(sl*TA + k)*32 + lane] = acl[k]; av[(sl*TA + k)*32 + lane] = avl[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bc[(sl*TB + k)*32 + lane] = bcl[k]; bv[(sl*TB + k)*32 + lane] = bvl[k]; bsr[(sl*TB + k)*32 + lane] = bsl[k]; }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; sam[sl] = __ldg(s.amax + g); sbm[sl] = __ldg(s.bmax + g); __threadfence_block(); ready[sl] = g; }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v11: branch-free software-pipelined main (loads(g+1) | B(g) | A(g+1)), dinv staged
template <int TA, int TB, bool MARK>
__global__ void __launch_bounds__(512,1) sweep11(S10d s, const double* __restrict__ dinv, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg) {
  extern __shared__ double sm[];
  double* xs = sm;                                    // n + 1
  double* psum = xs + n + 1;                          // R*32
  double* dg = psum + R10*32;                         // R*32
  double* di = dg + R10*32;                           // R*32
  double* av = di + R10*32;                           // R*TA*32
  double* bv = av + R10*TA*32;                        // R*TB*32
  int* ac = reinterpret_cast<int*>(bv + R10*TB*32);   // R*TA*32
  int* bc = ac + R10*TA*32;                           // R*TB*32
  int* rows = bc + R10*TB*32;                         // R*32
  int* bsr = rows + R10*32;                           // R*TB*32 (int)
  volatile int* meta = reinterpret_cast<volatile int*>(bsr + R10*TB*32);
  volatile int* ready = meta; int* snr = const_cast<int*>(meta) + R10;
  volatile int* progress = meta + 2*R10;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mainw = nw - 1;
  int hid = -1, nh = 0;
  for (int w = 0; w < nw; ++w) { const bool isH = (w != mainw) && ((w & 3) != (mainw & 3)); if (isH) { if (w == warp) hid = nh; ++nh; } }
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R10; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    if (warp == mainw) {
      double xprev = 0.0;
      // registers of group g
      double acc_pre, d, dv; int row, nr; double bvl[TB], bx[TB]; int bsl[TB];
      // prologue: A(0)
      {
        while (ready[0] != 0) {}
        nr = snr[0]; acc_pre = psum[lane]; d = dg[lane]; dv = di[lane]; row = rows[lane];
        double avl[TA]; int acl[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = ac[k*32 + lane]; avl[k] = av[k*32 + lane]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsr[k*32 + lane]; bvl[k] = bv[k*32 + lane]; bx[k] = xs[bc[k*32 + lane]]; }
#pragma unroll
        for (int k = 0; k < TA; ++k) acc_pre = sub_rn(acc_pre, mul_rn(avl[k], xs[acl[k]]));
      }
      for (int g = 0; g < s.G; ++g) {
        const long long w0 = clock64();
        const int g1 = g + 1 < s.G ? g + 1 : g;   // last iteration: dummy reload of g
        const int sl = g1 % R10;
        const long long wr0 = clock64();
        while (ready[sl] != g1) {}
        const long long wr1 = clock64();
        if (tsg && lane == 0 && sw == nsweeps - 1) tsg[g*2+1] = wr1 - wr0;
        // loads for g+1 (independent of x_g)
        const int nr1 = snr[sl];
        double acc1 = psum[sl*32 + lane];
        const double d1 = dg[sl*32 + lane], dv1 = di[sl*32 + lane]; const int row1 = rows[sl*32 + lane];
        double avl[TA]; int acl[TA]; double bvl1[TB], bx1[TB]; int bsl1[TB], bcl1[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = ac[(sl*TA + k)*32 + lane]; avl[k] = av[(sl*TA + k)*32 + lane]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl1[k] = bsr[(sl*TB + k)*32 + lane]; bvl1[k] = bv[(sl*TB + k)*32 + lane]; bcl1[k] = bc[(sl*TB + k)*32 + lane]; }
        double axv[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) axv[k] = xs[acl[k]];
#pragma unroll
        for (int k = 0; k < TB; ++k) bx1[k] = xs[bcl1[k]];
        // B(g): critical
        double acc = acc_pre;
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const double sx = __shfl_sync(0xffffffffu, xprev, bsl[k] & 31);
          const double X = bsl[k] >= 0 ? sx : bx[k];
          acc = sub_rn(acc, mul_rn(bvl[k], X));
        }
        double x;
        if (MARK) { const double q0 = mul_rn(acc, dv); const double rr = fma(-q0, d, acc); x = fma(rr, dv, q0); }
        else x = div_rn(acc, d);
        if (lane < nr) xs[row] = x;
        xprev = x;
        // A(g+1): pre-tail chain (deps on groups <= g-1)
#pragma unroll
        for (int k = 0; k < TA; ++k) acc1 = sub_rn(acc1, mul_rn(avl[k], axv[k]));
        __syncwarp();
        if (lane == 0) *progress = g + 1;
        acc_pre = acc1; d = d1; dv = dv1; row = row1; nr = nr1;
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsl1[k]; bvl[k] = bvl1[k]; bx[k] = bx1[k]; }
        if (tsg && lane == 0 && sw == nsweeps - 1) tsg[g*2] = clock64() - w0;
      }
    } else if (hid >= 0) {
      for (int g = hid; g < s.G; g += nh) {
        const int sl = g % R10;
        const int nr = __ldg(s.nr + g), pw = __ldg(s.pw + g), need = __ldg(s.need + g);
        const int64_t pb = __ldg(s.pptr + g);
        int row = -1; double acc = 0.0, dd = 1.0, ddi = 1.0;
        if (lane < nr) { row = __ldg(s.grows + g*32 + lane); acc = r[row]; dd = __ldg(s.diag + row); ddi = __ldg(dinv + row); }
        int acl[TA]; double avl[TA]; int bcl[TB]; double bvl[TB]; int bsl[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = __ldg(s.acol + (int64_t)(g*TA + k)*32 + lane); avl[k] = __ldg(s.aval + (int64_t)(g*TA + k)*32 + lane); }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bcl[k] = __ldg(s.bcol + (int64_t)(g*TB + k)*32 + lane); bvl[k] = __ldg(s.bval + (int64_t)(g*TB + k)*32 + lane); bsl[k] = s.bsrc[(int64_t)(g*TB + k)*32 + lane]; }
        constexpr int CH = 8;
        int pc[CH]; double pv[CH];
        const int32_t* cp = s.pcols + pb + lane; const double* vp = s.pvals + pb + lane;
        if (lane < nr) {
#pragma unroll
          for (int q = 0; q < CH; ++q) { pc[q] = q < pw ? __ldg(cp + (int64_t)q*nr) : -1; pv[q] = q < pw ? __ldg(vp + (int64_t)q*nr) : 0.0; }
        }
        while (*progress <= need) { __nanosleep(20); }
        if (lane < nr) {
          for (int k = 0; k < pw; k += CH) {
            int nc[CH]; double nv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) { const int kk = k + CH + q; nc[q] = kk < pw ? __ldg(cp + (int64_t)kk*nr) : -1; nv[q] = kk < pw ? __ldg(vp + (int64_t)kk*nr) : 0.0; }
            double xv[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = xs[pc[q] < 0 ? n : pc[q]];
#pragma unroll
            for (int q = 0; q < CH; ++q) if (pc[q] >= 0) acc = sub_rn(acc, mul_rn(pv[q], xv[q]));
#pragma unroll
            for (int q = 0; q < CH; ++q) { pc[q] = nc[q]; pv[q] = nv[q]; }
          }
        }
        while (*progress < g - R10 + 2) { __nanosleep(20); }
        psum[sl*32 + lane] = acc; dg[sl*32 + lane] = dd; di[sl*32 + lane] = ddi; rows[sl*32 + lane] = row;
#pragma unroll
        for (int k = 0; k < TA; ++k) { ac[(sl*TA + k)*32 + lane] = acl[k]; av[(sl*TA + k)*32 + lane] = avl[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bc[(sl*TB + k)*32 + lane] = bcl[k]; bv[(sl*TB + k)*32 + lane] = bvl[k]; bsr[(sl*TB + k)*32 + lane] = bsl[k]; }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; __threadfence_block(); ready[sl] = g; }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v12: FAST (reassociated) sums: tree reductions in main A/B and helper prefix; helper prefetch
template <int N>
__device__ __forceinline__ double tree_sum(double* p) {
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int k = 0; k + w < N; k += 2 * w) p[k] = add_rn(p[k], p[k + w]);
  return p[0];
}
template <int TA, int TB, int PW, bool ISO = false>
__global__ void __launch_bounds__(512,1) sweep12(S10d s, const double* __restrict__ dinv, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg) {
  extern __shared__ double sm[];
  double* xs = sm;
  double* psum = xs + n + 1;
  double* dg = psum + R10*32;
  double* di = dg + R10*32;
  double* av = di + R10*32;
  double* bv = av + R10*TA*32;
  int* ac = reinterpret_cast<int*>(bv + R10*TB*32);
  int* bc = ac + R10*TA*32;
  int* rows = bc + R10*TB*32;
  int* bsr = rows + R10*32;
  volatile int* meta = reinterpret_cast<volatile int*>(bsr + R10*TB*32);
  volatile int* ready = meta; int* snr = const_cast<int*>(meta) + R10;
  volatile int* progress = meta + 2*R10;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mainw = nw - 1;
  int hid = -1, nh = 0;
  for (int w = 0; w < nw; ++w) { const bool isH = (w != mainw) && ((w & 3) != (mainw & 3)); if (isH) { if (w == warp) hid = nh; ++nh; } }
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R10; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (ISO) {
      // prefill all ring slots with group 0's layout pattern (valid indices), mark ready
      for (int i = threadIdx.x; i < R10*32; i += blockDim.x) { psum[i] = 1.0; dg[i] = 2.0; di[i] = 0.5; rows[i] = (i % 32) + 32 * ((i / 32) % 8); }
      for (int i = threadIdx.x; i < R10*TA*32; i += blockDim.x) { ac[i] = (i * 7) % n; av[i] = 0.25; }
      for (int i = threadIdx.x; i < R10*TB*32; i += blockDim.x) { bc[i] = (i * 13) % n; bv[i] = 0.125; bsr[i] = (i % 3 == 0) ? (i % 32) : -1; }
      for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = 1.0;
      for (int i = threadIdx.x; i < R10; i += blockDim.x) { snr[i] = 8; }
      __syncthreads();
    }
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    if (warp == mainw) {
      double xprev = 0.0;
      double acc_pre, d, dv; int row, nr; double bvl[TB], bx[TB]; int bsl[TB];
      {
        if (!ISO) while (ready[0] != 0) {}
        nr = snr[0]; d = dg[lane]; dv = di[lane]; row = rows[lane];
        double pa[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(av[k*32 + lane], xs[ac[k*32 + lane]]);
        acc_pre = sub_rn(psum[lane], tree_sum<TA>(pa));
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsr[k*32 + lane]; bvl[k] = bv[k*32 + lane]; bx[k] = xs[bc[k*32 + lane]]; }
      }
      for (int g = 0; g < s.G; ++g) {
        const long long w0 = clock64();
        const int g1 = g + 1 < s.G ? g + 1 : g;
        const int sl = g1 % R10;
        const long long wr0 = clock64();
        if (!ISO) while (ready[sl] != g1) {}
        const long long wr1 = clock64();
        const int nr1 = snr[sl];
        const double ps1 = psum[sl*32 + lane];
        const double d1 = dg[sl*32 + lane], dv1 = di[sl*32 + lane]; const int row1 = rows[sl*32 + lane];
        double pa[TA]; double bvl1[TB], bx1[TB]; int bsl1[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(av[(sl*TA + k)*32 + lane], xs[ac[(sl*TA + k)*32 + lane]]);
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl1[k] = bsr[(sl*TB + k)*32 + lane]; bvl1[k] = bv[(sl*TB + k)*32 + lane]; bx1[k] = xs[bc[(sl*TB + k)*32 + lane]]; }
        // B(g)
        double pb[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const double sx = __shfl_sync(0xffffffffu, xprev, bsl[k] & 31);
          pb[k] = mul_rn(bvl[k], bsl[k] >= 0 ? sx : bx[k]);
        }
        const double acc = sub_rn(acc_pre, tree_sum<TB>(pb));
        const double q0 = mul_rn(acc, dv); const double rr = fma(-q0, d, acc); const double x = fma(rr, dv, q0);
        if (lane < nr) xs[row] = x;
        xprev = x;
        const double acc1 = sub_rn(ps1, tree_sum<TA>(pa));
        __syncwarp();
        if (lane == 0) *progress = g + 1;
        acc_pre = acc1; d = d1; dv = dv1; row = row1; nr = nr1;
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsl1[k]; bvl[k] = bvl1[k]; bx[k] = bx1[k]; }
        if (tsg && lane == 0 && sw == nsweeps - 1) { tsg[g*2] = clock64() - w0; tsg[g*2+1] = wr1 - wr0; }
      }
    } else if (hid >= 0 && !ISO) {
      int g = hid;
      // prefetched header of the current group
      int nr = 0, pw = 0, need = 0; int64_t pb0 = 0;
      if (g < s.G) { nr = __ldg(s.nr + g); pw = __ldg(s.pw + g); need = __ldg(s.need + g); pb0 = __ldg(s.pptr + g); }
      for (; g < s.G; g += nh) {
        const int sl = g % R10;
        const int gn = g + nh;
        int nrn = 0, pwn = 0, needn = 0; int64_t pbn = 0;
        if (gn < s.G) { nrn = __ldg(s.nr + gn); pwn = __ldg(s.pw + gn); needn = __ldg(s.need + gn); pbn = __ldg(s.pptr + gn); }
        int row = -1; double acc = 0.0, dd = 1.0, ddi = 1.0;
        if (lane < nr) { row = __ldg(s.grows + g*32 + lane); dd = __ldg(s.diag + row); ddi = __ldg(dinv + row); }
        int acl[TA]; double avl[TA]; int bcl[TB]; double bvl[TB]; int bsl[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = __ldg(s.acol + (int64_t)(g*TA + k)*32 + lane); avl[k] = __ldg(s.aval + (int64_t)(g*TA + k)*32 + lane); }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bcl[k] = __ldg(s.bcol + (int64_t)(g*TB + k)*32 + lane); bvl[k] = __ldg(s.bval + (int64_t)(g*TB + k)*32 + lane); bsl[k] = s.bsrc[(int64_t)(g*TB + k)*32 + lane]; }
        const int32_t* cp = s.pcols + pb0 + lane; const double* vp = s.pvals + pb0 + lane;
        double part = 0.0;
        for (int k0 = 0; k0 < pw; k0 += PW) {
          int pc[PW]; double pv[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) { const bool ok = lane < nr && k0 + q < pw; pc[q] = ok ? __ldg(cp + (int64_t)(k0+q)*nr) : n; pv[q] = ok ? __ldg(vp + (int64_t)(k0+q)*nr) : 0.0; }
          if (k0 == 0) while (*progress <= need) { __nanosleep(20); }
          double pp[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) pp[q] = mul_rn(pv[q], xs[pc[q]]);
          part = add_rn(part, tree_sum<PW>(pp));
        }
        if (pw == 0) while (*progress <= need) { __nanosleep(20); }
        if (lane < nr) acc = sub_rn(r[row], part);
        while (*progress < g - R10 + 2) { __nanosleep(20); }
        psum[sl*32 + lane] = acc; dg[sl*32 + lane] = dd; di[sl*32 + lane] = ddi; rows[sl*32 + lane] = row;
#pragma unroll
        for (int k = 0; k < TA; ++k) { ac[(sl*TA + k)*32 + lane] = acl[k]; av[(sl*TA + k)*32 + lane] = avl[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bc[(sl*TB + k)*32 + lane] = bcl[k]; bv[(sl*TB + k)*32 + lane] = bvl[k]; bsr[(sl*TB + k)*32 + lane] = bsl[k]; }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; __threadfence_block(); ready[sl] = g; }
        nr = nrn; pw = pwn; need = needn; pb0 = pbn;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v13: v12 with explicit ordering: SHFL(B(g)) -> loads(g+1) -> B math -> STS -> A(g+1) math
__device__ __forceinline__ double shfl_d(double v, int src) {
  unsigned lo, hi, rlo, rhi;
  asm volatile("mov.b64 {%0,%1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rlo) : "r"(lo), "r"(src));
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(rhi) : "r"(hi), "r"(src));
  double out;
  asm volatile("mov.b64 %0, {%1,%2};" : "=d"(out) : "r"(rlo), "r"(rhi));
  return out;
}
template <int TA, int TB, int PW, bool ISO = false>
__global__ void __launch_bounds__(512,1) sweep13(S10d s, const double* __restrict__ dinv, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg) {
  extern __shared__ double sm[];
  double* xs = sm;
  double* psum = xs + n + 1;
  double* dg = psum + R10*32;
  double* di = dg + R10*32;
  double* av = di + R10*32;
  double* bv = av + R10*TA*32;
  int* ac = reinterpret_cast<int*>(bv + R10*TB*32);
  int* bc = ac + R10*TA*32;
  int* rows = bc + R10*TB*32;
  int* bsr = rows + R10*32;
  volatile int* meta = reinterpret_cast<volatile int*>(bsr + R10*TB*32);
  volatile int* ready = meta; int* snr = const_cast<int*>(meta) + R10;
  volatile int* progress = meta + 2*R10;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mainw = nw - 1;
  int hid = -1, nh = 0;
  for (int w = 0; w < nw; ++w) { const bool isH = (w != mainw) && ((w & 3) != (mainw & 3)); if (isH) { if (w == warp) hid = nh; ++nh; } }
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R10; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (ISO) {
      for (int i = threadIdx.x; i < R10*32; i += blockDim.x) { psum[i] = 1.0; dg[i] = 2.0; di[i] = 0.5; rows[i] = (i % 32) + 32 * ((i / 32) % 8); }
      for (int i = threadIdx.x; i < R10*TA*32; i += blockDim.x) { ac[i] = (i * 7) % n; av[i] = 0.25; }
      for (int i = threadIdx.x; i < R10*TB*32; i += blockDim.x) { bc[i] = (i * 13) % n; bv[i] = 0.125; bsr[i] = (i % 3 == 0) ? (i % 32) : -1; }
      for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = 1.0;
      for (int i = threadIdx.x; i < R10; i += blockDim.x) { snr[i] = 8; }
      __syncthreads();
    }
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    if (warp == mainw) {
      double xprev = 0.0;
      double acc_pre, d, dv; int row, nr; double bvl[TB], bx[TB]; int bsl[TB];
      {
        if (!ISO) while (ready[0] != 0) {}
        nr = snr[0]; d = dg[lane]; dv = di[lane]; row = rows[lane];
        double pa[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(av[k*32 + lane], xs[ac[k*32 + lane]]);
        acc_pre = sub_rn(psum[lane], tree_sum<TA>(pa));
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsr[k*32 + lane]; bvl[k] = bv[k*32 + lane]; bx[k] = xs[bc[k*32 + lane]]; }
      }
      for (int g = 0; g < s.G; ++g) {
        const long long w0 = clock64();
        // (1) shuffles for B(g): x_{g-1} lives in xprev
        double sx[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) sx[k] = shfl_d(xprev, bsl[k] & 31);
        asm volatile("" ::: "memory");
        // (2) next group's slot
        const int g1 = g + 1 < s.G ? g + 1 : g;
        const int sl = g1 % R10;
        if (!ISO) while (ready[sl] != g1) {}
        const int nr1 = snr[sl];
        const double ps1 = psum[sl*32 + lane];
        const double d1 = dg[sl*32 + lane], dv1 = di[sl*32 + lane]; const int row1 = rows[sl*32 + lane];
        double avl[TA], axv[TA]; double bvl1[TB], bx1[TB]; int bsl1[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { avl[k] = av[(sl*TA + k)*32 + lane]; axv[k] = xs[ac[(sl*TA + k)*32 + lane]]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl1[k] = bsr[(sl*TB + k)*32 + lane]; bvl1[k] = bv[(sl*TB + k)*32 + lane]; bx1[k] = xs[bc[(sl*TB + k)*32 + lane]]; }
        // (3) B(g) math
        double pb[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) pb[k] = mul_rn(bvl[k], bsl[k] >= 0 ? sx[k] : bx[k]);
        const double acc = sub_rn(acc_pre, tree_sum<TB>(pb));
        const double q0 = mul_rn(acc, dv); const double rr = fma(-q0, d, acc); const double x = fma(rr, dv, q0);
        xprev = x;
        if (lane < nr) xs[row] = x;
        __syncwarp();
        if (lane == 0) *progress = g + 1;
        // (4) A(g+1)
        double pa[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(avl[k], axv[k]);
        acc_pre = sub_rn(ps1, tree_sum<TA>(pa)); d = d1; dv = dv1; row = row1; nr = nr1;
#pragma unroll
        for (int k = 0; k < TB; ++k) { bsl[k] = bsl1[k]; bvl[k] = bvl1[k]; bx[k] = bx1[k]; }
        if (tsg && lane == 0 && sw == nsweeps - 1) { tsg[g*2] = clock64() - w0; tsg[g*2+1] = 0; }
      }
    } else if (hid >= 0 && !ISO) {
      int g = hid;
      int nr = 0, pw = 0, need = 0; int64_t pb0 = 0;
      if (g < s.G) { nr = __ldg(s.nr + g); pw = __ldg(s.pw + g); need = __ldg(s.need + g); pb0 = __ldg(s.pptr + g); }
      for (; g < s.G; g += nh) {
        const int sl = g % R10;
        const int gn = g + nh;
        int nrn = 0, pwn = 0, needn = 0; int64_t pbn = 0;
        if (gn < s.G) { nrn = __ldg(s.nr + gn); pwn = __ldg(s.pw + gn); needn = __ldg(s.need + gn); pbn = __ldg(s.pptr + gn); }
        int row = -1; double acc = 0.0, dd = 1.0, ddi = 1.0;
        if (lane < nr) { row = __ldg(s.grows + g*32 + lane); dd = __ldg(s.diag + row); ddi = __ldg(dinv + row); }
        int acl[TA]; double avl[TA]; int bcl[TB]; double bvl[TB]; int bsl[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = __ldg(s.acol + (int64_t)(g*TA + k)*32 + lane); avl[k] = __ldg(s.aval + (int64_t)(g*TA + k)*32 + lane); }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bcl[k] = __ldg(s.bcol + (int64_t)(g*TB + k)*32 + lane); bvl[k] = __ldg(s.bval + (int64_t)(g*TB + k)*32 + lane); bsl[k] = s.bsrc[(int64_t)(g*TB + k)*32 + lane]; }
        const int32_t* cp = s.pcols + pb0 + lane; const double* vp = s.pvals + pb0 + lane;
        double part = 0.0;
        for (int k0 = 0; k0 < pw; k0 += PW) {
          int pc[PW]; double pv[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) { const bool ok = lane < nr && k0 + q < pw; pc[q] = ok ? __ldg(cp + (int64_t)(k0+q)*nr) : n; pv[q] = ok ? __ldg(vp + (int64_t)(k0+q)*nr) : 0.0; }
          if (k0 == 0) while (*progress <= need) { __nanosleep(20); }
          double pp[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) pp[q] = mul_rn(pv[q], xs[pc[q]]);
          part = add_rn(part, tree_sum<PW>(pp));
        }
        if (pw == 0) while (*progress <= need) { __nanosleep(20); }
        if (lane < nr) acc = sub_rn(r[row], part);
        while (*progress < g - R10 + 2) { __nanosleep(20); }
        psum[sl*32 + lane] = acc; dg[sl*32 + lane] = dd; di[sl*32 + lane] = ddi; rows[sl*32 + lane] = row;
#pragma unroll
        for (int k = 0; k < TA; ++k) { ac[(sl*TA + k)*32 + lane] = acl[k]; av[(sl*TA + k)*32 + lane] = avl[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bc[(sl*TB + k)*32 + lane] = bcl[k]; bv[(sl*TB + k)*32 + lane] = bvl[k]; bsr[(sl*TB + k)*32 + lane] = bsl[k]; }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; __threadfence_block(); ready[sl] = g; }
        nr = nrn; pw = pwn; need = needn; pb0 = pbn;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}


// ---- v14: deeper pipeline. Group G entries: prefix (dep <= G-D, helpers), A (G-D < dep <= G-3,
// main gathers one iteration ahead), B (dep in {G-2, G-1}: two register shuffles).
struct H14 { int G; std::vector<int32_t> nr, need, grows, pw; std::vector<int64_t> pptr; std::vector<int32_t> pcols, acol; std::vector<double> pvals, aval, bval; std::vector<int32_t> bsrc; };
template <int TA, int TB>
H14 build14(const HostSweep& s, int D) {
  int n = s.n; std::vector<int> gof(n), lof(n);
  std::vector<std::vector<std::pair<int,double>>> rows(n);
  for (int g = 0; g < s.n_groups; ++g) for (int l = 0; l < 32; ++l) { int r = s.grows[g*32+l]; if (r < 0) continue; gof[r] = g; lof[r] = l;
      for (int k = 0; k < s.gwidth[g]; ++k) { int64_t e = s.gptr[g] + (int64_t)k*32 + l; if (s.cols[e] >= 0) rows[r].push_back({s.cols[e], s.vals[e]}); } }
  H14 h; h.G = s.n_groups; h.pptr.push_back(0);
  int ta_max = 0, tb_max = 0;
  for (int g = 0; g < s.n_groups; ++g) {
    int nr = 0; for (int l = 0; l < 32; ++l) if (s.grows[g*32+l] >= 0) nr = l + 1;
    std::vector<std::vector<std::pair<int,double>>> P(nr), A(nr), B(nr);
    int need = -1, pw = 0;
    for (int l = 0; l < nr; ++l) for (auto& e : rows[s.grows[g*32+l]]) {
      int dg = gof[e.first];
      if (dg >= g - 2) B[l].push_back(e); else if (dg > g - D) A[l].push_back(e); else P[l].push_back(e);
    }
    for (int l = 0; l < nr; ++l) {
      while ((int)A[l].size() > TA) { P[l].push_back(A[l].front()); A[l].erase(A[l].begin()); }  // oldest to prefix
      if ((int)B[l].size() > TB) { printf("B overflow %zu\n", B[l].size()); exit(1); }
      for (auto& e : P[l]) need = std::max(need, gof[e.first]);
      pw = std::max(pw, (int)P[l].size()); ta_max = std::max(ta_max, (int)A[l].size()); tb_max = std::max(tb_max, (int)B[l].size()); }
    h.nr.push_back(nr); h.need.push_back(need); h.pw.push_back(pw);
    for (int l = 0; l < 32; ++l) h.grows.push_back(s.grows[g*32+l]);
    int64_t pb = h.pptr.back(); h.pcols.resize(pb + (int64_t)pw*nr, n); h.pvals.resize(pb + (int64_t)pw*nr, 0.0);
    size_t a0 = h.acol.size(); h.acol.resize(a0 + TA*32, n); h.aval.resize(a0 + TA*32, 0.0);
    size_t b0 = h.bval.size(); h.bval.resize(b0 + TB*32, 0.0); h.bsrc.resize(b0 + TB*32, 0);
    for (int l = 0; l < nr; ++l) {
      for (size_t k = 0; k < P[l].size(); ++k) { h.pcols[pb + (int64_t)k*nr + l] = P[l][k].first; h.pvals[pb + (int64_t)k*nr + l] = P[l][k].second; }
      for (size_t k = 0; k < A[l].size(); ++k) { h.acol[a0 + k*32 + l] = A[l][k].first; h.aval[a0 + k*32 + l] = A[l][k].second; }
      for (size_t k = 0; k < B[l].size(); ++k) { int dg = gof[B[l][k].first]; h.bval[b0 + k*32 + l] = B[l][k].second; h.bsrc[b0 + k*32 + l] = lof[B[l][k].first] | (dg == g - 2 ? 32 : 0); } }
    h.pptr.push_back(pb + (int64_t)pw*nr);
  }
  printf("build14 D=%d: max A %d, max B %d\n", D, ta_max, tb_max);
  return h;
}
struct S14d { int G; const int32_t *nr, *need, *grows, *pw, *pcols, *acol, *bsrc; const int64_t* pptr; const double *pvals, *aval, *bval, *diag, *dinv; };
template <int TA, int TB, int PW, bool ISO = false>
__global__ void __launch_bounds__(512,1) sweep14(S14d s, int n, const double* __restrict__ r, double* out, unsigned long long* t, int nsweeps, long long* tsg) {
  extern __shared__ double sm[];
  double* xs = sm;                                  // n+1
  double* psum = xs + n + 1;                        // R*32
  double* dg = psum + R10*32;
  double* di = dg + R10*32;
  double* av = di + R10*32;                         // R*TA*32
  double* bv = av + R10*TA*32;                      // R*TB*32
  int* ac = reinterpret_cast<int*>(bv + R10*TB*32); // R*TA*32
  int* rows = ac + R10*TA*32;                       // R*32
  int* bsr = rows + R10*32;                         // R*TB*32
  volatile int* meta = reinterpret_cast<volatile int*>(bsr + R10*TB*32);
  volatile int* ready = meta; int* snr = const_cast<int*>(meta) + R10;
  volatile int* progress = meta + 2*R10;
  unsigned long long c0 = 0, g0 = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mainw = nw - 1;
  int hid = -1, nh = 0;
  for (int w = 0; w < nw; ++w) { const bool isH = (w != mainw) && ((w & 3) != (mainw & 3)); if (isH) { if (w == warp) hid = nh; ++nh; } }
  for (int sw = 0; sw < nsweeps; ++sw) {
    for (int i = threadIdx.x; i < R10; i += blockDim.x) ready[i] = -1;
    if (threadIdx.x == 0) { *progress = 0; xs[n] = 0.0; }
    __syncthreads();
    if (ISO) {
      for (int i = threadIdx.x; i < R10*32; i += blockDim.x) { psum[i] = 1.0; dg[i] = 2.0; di[i] = 0.5; rows[i] = (i % 32) + 32 * ((i / 32) % 8); }
      for (int i = threadIdx.x; i < R10*TA*32; i += blockDim.x) { ac[i] = (i * 7) % n; av[i] = 0.25; }
      for (int i = threadIdx.x; i < R10*TB*32; i += blockDim.x) { bv[i] = 0.125; bsr[i] = i % 64; }
      for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = 1.0;
      for (int i = threadIdx.x; i < R10; i += blockDim.x) { snr[i] = 8; }
      __syncthreads();
    }
    if (sw == nsweeps - 1) { c0 = clock64(); g0 = gtimer(); }
    if (warp == mainw) {
      double x1 = 0.0, x2 = 0.0;          // x of groups g-1, g-2 (per lane)
      // group g state (B pending): acc_pre, d, dv, row, nr, bvl, bsl
      // group g+1 state (A pending): ps1, avl1, axv1, d1, dv1, row1, nr1, bvl1, bsl1
      double acc_pre = 0.0, d = 1.0, dv = 1.0; int row = -1, nr = 0; double bvl[TB]; int bsl[TB];
      double ps1 = 0.0, d1 = 1.0, dv1 = 1.0; int row1 = -1, nr1 = 0; double avl1[TA], axv1[TA], bvl1[TB]; int bsl1[TB];
      auto load = [&](int gg, double& ps, double& dd, double& ddv, int& rr, int& nn, double* avl, double* axv, double* bvl_, int* bsl_) {
        const int sl = gg % R10;
        if (!ISO) while (ready[sl] != gg) {}
        nn = snr[sl]; ps = psum[sl*32 + lane]; dd = dg[sl*32 + lane]; ddv = di[sl*32 + lane]; rr = rows[sl*32 + lane];
#pragma unroll
        for (int k = 0; k < TA; ++k) { avl[k] = av[(sl*TA + k)*32 + lane]; axv[k] = xs[ac[(sl*TA + k)*32 + lane]]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bvl_[k] = bv[(sl*TB + k)*32 + lane]; bsl_[k] = bsr[(sl*TB + k)*32 + lane]; }
      };
      // prologue: group 0 (A done now), group 1 loaded
      {
        double avl[TA], axv[TA];
        load(0, acc_pre, d, dv, row, nr, avl, axv, bvl, bsl);
        double pa[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(avl[k], axv[k]);
        acc_pre = sub_rn(acc_pre, tree_sum<TA>(pa));
        if (s.G > 1) load(1, ps1, d1, dv1, row1, nr1, avl1, axv1, bvl1, bsl1);
      }
      for (int g = 0; g < s.G; ++g) {
        const long long w0 = clock64();
        // (1) B(g) shuffles
        double X[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const int src = bsl[k] & 31;
          const double a1 = shfl_d(x1, src), a2 = shfl_d(x2, src);
          X[k] = (bsl[k] & 32) ? a2 : a1;
        }
        asm volatile("" ::: "memory");
        // (2) loads for g+2 (deps <= g-1 for its A part: available)
        double ps2 = 0.0, d2 = 1.0, dv2 = 1.0; int row2 = -1, nr2 = 0; double avl2[TA], axv2[TA], bvl2[TB]; int bsl2[TB];
        if (g + 2 < s.G) load(g + 2, ps2, d2, dv2, row2, nr2, avl2, axv2, bvl2, bsl2);
        // (3) B(g) math
        double pb[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) pb[k] = mul_rn(bvl[k], X[k]);
        const double acc = sub_rn(acc_pre, tree_sum<TB>(pb));
        const double q0 = mul_rn(acc, dv); const double rr = fma(-q0, d, acc); const double x = fma(rr, dv, q0);
        if (lane < nr) xs[row] = x;
        __syncwarp();
        if (lane == 0) *progress = g + 1;
        x2 = x1; x1 = x;
        // (4) A(g+1) with registers loaded one iteration ago
        double pa[TA];
#pragma unroll
        for (int k = 0; k < TA; ++k) pa[k] = mul_rn(avl1[k], axv1[k]);
        acc_pre = sub_rn(ps1, tree_sum<TA>(pa)); d = d1; dv = dv1; row = row1; nr = nr1;
#pragma unroll
        for (int k = 0; k < TB; ++k) { bvl[k] = bvl1[k]; bsl[k] = bsl1[k]; }
        ps1 = ps2; d1 = d2; dv1 = dv2; row1 = row2; nr1 = nr2;
#pragma unroll
        for (int k = 0; k < TA; ++k) { avl1[k] = avl2[k]; axv1[k] = axv2[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bvl1[k] = bvl2[k]; bsl1[k] = bsl2[k]; }
        if (tsg && lane == 0 && sw == nsweeps - 1) tsg[g] = clock64() - w0;
      }
    } else if (hid >= 0 && !ISO) {
      int g = hid;
      int nr = 0, pw = 0, need = 0; int64_t pb0 = 0;
      if (g < s.G) { nr = __ldg(s.nr + g); pw = __ldg(s.pw + g); need = __ldg(s.need + g); pb0 = __ldg(s.pptr + g); }
      for (; g < s.G; g += nh) {
        const int sl = g % R10;
        const int gn = g + nh;
        int nrn = 0, pwn = 0, needn = 0; int64_t pbn = 0;
        if (gn < s.G) { nrn = __ldg(s.nr + gn); pwn = __ldg(s.pw + gn); needn = __ldg(s.need + gn); pbn = __ldg(s.pptr + gn); }
        int row = -1; double acc = 0.0, dd = 1.0, ddi = 1.0;
        if (lane < nr) { row = __ldg(s.grows + g*32 + lane); dd = __ldg(s.diag + row); ddi = __ldg(s.dinv + row); }
        int acl[TA]; double avl[TA]; double bvl[TB]; int bsl[TB];
#pragma unroll
        for (int k = 0; k < TA; ++k) { acl[k] = __ldg(s.acol + (int64_t)(g*TA + k)*32 + lane); avl[k] = __ldg(s.aval + (int64_t)(g*TA + k)*32 + lane); }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bvl[k] = __ldg(s.bval + (int64_t)(g*TB + k)*32 + lane); bsl[k] = __ldg(s.bsrc + (int64_t)(g*TB + k)*32 + lane); }
        const int32_t* cp = s.pcols + pb0 + lane; const double* vp = s.pvals + pb0 + lane;
        double part = 0.0;
        for (int k0 = 0; k0 < pw; k0 += PW) {
          int pc[PW]; double pv[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) { const bool ok = lane < nr && k0 + q < pw; pc[q] = ok ? __ldg(cp + (int64_t)(k0+q)*nr) : n; pv[q] = ok ? __ldg(vp + (int64_t)(k0+q)*nr) : 0.0; }
          if (k0 == 0) while (*progress <= need) { __nanosleep(20); }
          double pp[PW];
#pragma unroll
          for (int q = 0; q < PW; ++q) pp[q] = mul_rn(pv[q], xs[pc[q]]);
          part = add_rn(part, tree_sum<PW>(pp));
        }
        if (pw == 0) while (*progress <= need) { __nanosleep(20); }
        if (lane < nr) acc = sub_rn(r[row], part);
        while (*progress < g - R10 + 3) { __nanosleep(20); }
        psum[sl*32 + lane] = acc; dg[sl*32 + lane] = dd; di[sl*32 + lane] = ddi; rows[sl*32 + lane] = row;
#pragma unroll
        for (int k = 0; k < TA; ++k) { ac[(sl*TA + k)*32 + lane] = acl[k]; av[(sl*TA + k)*32 + lane] = avl[k]; }
#pragma unroll
        for (int k = 0; k < TB; ++k) { bv[(sl*TB + k)*32 + lane] = bvl[k]; bsr[(sl*TB + k)*32 + lane] = bsl[k]; }
        __syncwarp();
        if (lane == 0) { snr[sl] = nr; __threadfence_block(); ready[sl] = g; }
        nr = nrn; pw = pwn; need = needn; pb0 = pbn;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
  }
  if (threadIdx.x == 0) { t[0] = clock64() - c0; t[1] = gtimer() - g0; }
}

template <class T> T* up(const std::vector<T>& v) { T* d; cudaMalloc(&d, v.size()*sizeof(T)+8); cudaMemcpy(d, v.data(), v.size()*sizeof(T), cudaMemcpyHostToDevice); return d; }

int main(int argc, char** argv) {
  int k = argc > 1 ? atoi(argv[1]) : 2, N = argc > 2 ? atoi(argv[2]) : 64;
  dshost_system* sys; if (dshost_assemble(2, k, N, 0, 1.0, 0, &sys)) { printf("asm fail\n"); return 1; }
  int nr, nc; const int64_t* rp; const int32_t* ci; const double* v;
  dshost_block(sys, DSHOST_A, &nr, &nc, &rp, &ci, &v);
  int n = nr; std::vector<int32_t> perm(n); dshost_rcm(n, rp, ci, perm.data());
  int64_t nnz = rp[n]; std::vector<int64_t> prp(n+1); std::vector<int32_t> pci(nnz); std::vector<double> pv(nnz);
  dshost_permute(n, rp, ci, v, perm.data(), prp.data(), pci.data(), pv.data());
  int64_t ln = dshost_lower_nnz(n, prp.data(), pci.data()); std::vector<int64_t> lrp(n+1); std::vector<int32_t> lci(ln); std::vector<double> lv(ln); int bad;
  dshost_ic0(n, prp.data(), pci.data(), pv.data(), lrp.data(), lci.data(), lv.data(), &bad);
  dsgpu_csr L{n, n, lrp.data(), lci.data(), lv.data()};
  HostSweep f, b; build_sweeps(L, f, b);
  const bool only11 = argc > 3 && strcmp(argv[3], "v11") == 0;
  printf("n=%d nnzL=%ld levels=%d groups=%d sell_entries=%ld\n", n, (long)ln, f.n_levels, f.n_groups, (long)f.gptr.back());
  S s{f.n_groups, up(f.gptr), up(f.gwidth), up(f.grows), up(f.cols), up(f.vals), up(f.diag)};
  std::vector<double> rh(n, 1.0); double* r = up(rh); double* out; cudaMalloc(&out, n*8);
  unsigned* ab; cudaMalloc(&ab, 64); cudaMemset(ab, 0, 64);
  unsigned long long* t; cudaMalloc(&t, 32);
  size_t smem = n * 8;
  cudaFuncSetAttribute(sweep_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sweep_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(sweep_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (!only11) for (int threads : {1024}) {
    for (int mode = 0; mode < 4; ++mode) {
      unsigned long long th[2]; float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (mode == 0) sweep_k<0><<<1, threads, smem>>>(s, n, r, out, ab, t);
        if (mode == 1) sweep_k<1><<<1, threads, smem>>>(s, n, r, out, ab, t);
        if (mode == 2) sweep_k<2><<<1, threads, smem>>>(s, n, r, out, ab, t);
        if (mode == 3) stream_k<<<1, threads>>>(s, n, r, out, t);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) { best = ms; cudaMemcpy(th, t, 16, cudaMemcpyDeviceToHost); }
      }
      printf("threads=%4d mode=%d (%s): %.1f us  cycles=%llu  ns=%llu  eff_MHz=%.0f  cyc/level=%.0f  err=%s\n", threads, mode,
             mode==0?"spin":mode==1?"spin+nanosleep":mode==2?"spin+clock":"stream-nodep", best*1e3, th[0], th[1], th[0]*1e3/(double)th[1], th[0]/(double)f.n_levels, cudaGetErrorString(cudaGetLastError()));
    }
  }

  {
    H2 h2 = build2(f);
    std::vector<double> dinv(n); for (int i = 0; i < n; ++i) dinv[i] = 1.0 / f.diag[i];
    printf("compact entries=%ld (SELL-32 had %ld)\n", (long)h2.gptr.back(), (long)f.gptr.back());
    S2 s2{f.n_groups, up(h2.gptr), up(h2.gnrow), up(h2.gpw), up(h2.grows), up(h2.cols), up(h2.vals), up(f.diag), up(dinv)};
    double* out_ref; cudaMalloc(&out_ref, n*8);
    cudaFuncSetAttribute(sweep2<false,4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sweep2<false,8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sweep2<true,8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweep_k<0><<<1, 1024, smem>>>(s, n, r, out_ref, ab, t);
    std::vector<double> o1(n), o2(n); cudaMemcpy(o1.data(), out_ref, n*8, cudaMemcpyDeviceToHost);
    if (!only11) for (int var = 0; var < 3; ++var) for (int threads : {1024, 512}) {
      unsigned long long th[2]; float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        if (var == 0) sweep2<false,4><<<1, threads, smem>>>(s2, n, r, out, ab, t);
        if (var == 1) sweep2<false,8><<<1, threads, smem>>>(s2, n, r, out, ab, t);
        if (var == 2) sweep2<true,8><<<1, threads, smem>>>(s2, n, r, out, ab, t);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) { best = ms; cudaMemcpy(th, t, 16, cudaMemcpyDeviceToHost); }
      }
      cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
      double md = 0; bool eq = true; for (int i = 0; i < n; ++i) { md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i]))); eq &= o1[i]==o2[i]; }
      printf("v2 var=%d (%s) threads=%d: %.1f us cyc/level=%.0f bitexact=%d maxrel=%.2e err=%s\n", var, var==0?"div,ch4":var==1?"div,ch8":"recip,ch8", threads, best*1e3, th[0]/(double)f.n_levels, (int)eq, md, cudaGetErrorString(cudaGetLastError()));
    }

    if (!only11) {
      size_t smem3 = n * 16;
      cudaFuncSetAttribute(sweep3<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      cudaFuncSetAttribute(sweep3<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      cudaFuncSetAttribute(sweep3<100>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      cudaFuncSetAttribute(sweep3<400>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      for (int var = 0; var < 4; ++var) for (int threads : {1024, 512, 256}) {
        unsigned long long th[2]; float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          if (var == 0) sweep3<-1><<<1, threads, smem3>>>(s2, n, r, out, t, 4);
          if (var == 1) sweep3<0><<<1, threads, smem3>>>(s2, n, r, out, t, 4);
          if (var == 2) sweep3<100><<<1, threads, smem3>>>(s2, n, r, out, t, 4);
          if (var == 3) sweep3<400><<<1, threads, smem3>>>(s2, n, r, out, t, 4);
          cudaDeviceSynchronize(); unsigned long long tt[2]; cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; th[0]=tt[0]; th[1]=tt[1]; }
        }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        bool eq = true; for (int i = 0; i < n; ++i) eq &= o1[i]==o2[i];
        printf("v3 var=%d (%s) threads=%d: %.1f us/sweep cyc/level=%.0f bitexact=%d err=%s\n", var, var==0?"mbarrier":var==1?"spin":var==2?"sleep100":"sleep400", threads, best, th[0]/(double)f.n_levels, (int)eq, cudaGetErrorString(cudaGetLastError()));
      }
    }

    if (!only11) {
      size_t smem3 = n * 8;
      cudaFuncSetAttribute(sweep4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      long long* ts; cudaMalloc(&ts, f.n_groups * 32);
      sweep4<<<1, 1024, smem3>>>(s2, n, r, out, ts, 3);
      cudaDeviceSynchronize();
      std::vector<long long> h(f.n_groups * 4); cudaMemcpy(h.data(), ts, h.size()*8, cudaMemcpyDeviceToHost);
      printf("v4 err=%s\n", cudaGetErrorString(cudaGetLastError()));
      // per-group: start, prefix-done, tail-done, publish
      double sA=0,sB=0,sC=0,sD=0; int cnt=0;
      for (int g = 64; g < f.n_groups - 64; ++g) { sA += h[g*4+1]-h[g*4+0]; sB += h[g*4+2]-h[g*4+1]; sC += h[g*4+3]-h[g*4+2]; sD += h[g*4+3]-h[(g-1)*4+3]; cnt++; }
      printf("v4 mean cycles: start->prefixdone %.0f, tail wait %.0f, div+publish %.0f, publish-to-publish(prev group) %.0f\n", sA/cnt, sB/cnt, sC/cnt, sD/cnt);
      for (int g = 500; g < 510; ++g) printf("  g=%d start=%lld prefix=%lld tail=%lld pub=%lld\n", g, h[g*4], h[g*4+1], h[g*4+2], h[g*4+3]);
      // pointer chase latency over a 16 MB buffer (L2-resident)
      int M = 4 << 20; std::vector<int32_t> nx(M); for (int i = 0; i < M; ++i) nx[i] = (int)((i + 1000003ll * 7) % M);
      int32_t* dn = up(nx); long long* lo; cudaMalloc(&lo, 16);
      chase<<<1,1>>>(dn, 1000, lo); chase<<<1,1>>>(dn, 10000, lo); cudaDeviceSynchronize();
      long long hl[2]; cudaMemcpy(hl, lo, 16, cudaMemcpyDeviceToHost);
      printf("L2 pointer-chase latency: %.0f cycles\n", hl[0] / 10000.0);
    }

    if (!only11) {
      size_t smem3 = n * 8;
      for (int extra : {0, 69000}) {
      cudaFuncSetAttribute(sweep5<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem3+extra));
      cudaFuncSetAttribute(sweep5<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem3+extra));
      for (int var = 0; var < 2; ++var) for (int threads : {1024, 512}) {
        unsigned long long th[2]; float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          if (var == 0) sweep5<0><<<1, threads, smem3+extra>>>(s2, n, r, out, t, 4);
          if (var == 1) sweep5<1><<<1, threads, smem3+extra>>>(s2, n, r, out, t, 4);
          cudaDeviceSynchronize(); unsigned long long tt[2]; cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; th[0]=tt[0]; th[1]=tt[1]; }
        }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        bool eq = true; for (int i = 0; i < n; ++i) eq &= o1[i]==o2[i];
        printf("v5 var=%d (%s) smem_extra=%d threads=%d: %.1f us/sweep cyc/level=%.0f bitexact=%d err=%s\n", var, var==0?"pf-cur":"pf-next", extra, threads, best, th[0]/(double)f.n_levels, (int)eq, cudaGetErrorString(cudaGetLastError()));
      }
      }
    }

    if (!only11) {
      std::vector<int> lev; H2 h6 = build6(f, lev);
      S2 s6{f.n_groups, up(h6.gptr), up(h6.gnrow), up(h6.gpw), up(h6.grows), up(h6.cols), up(h6.vals), up(f.diag), up(dinv)};
      size_t smem3 = n * 8;
      cudaFuncSetAttribute(sweep6<false,false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      cudaFuncSetAttribute(sweep6<false,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      cudaFuncSetAttribute(sweep6<true,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
      for (int var = 0; var < 3; ++var) for (int threads : {1024, 512}) {
        unsigned long long th[2]; float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          if (var == 0) sweep6<false,false><<<1, threads, smem3>>>(s6, n, r, out, t, 4, nullptr);
          if (var == 1) sweep6<false,true><<<1, threads, smem3>>>(s6, n, r, out, t, 4, nullptr);
          if (var == 2) sweep6<true,true><<<1, threads, smem3>>>(s6, n, r, out, t, 4, nullptr);
          cudaDeviceSynchronize(); unsigned long long tt[2]; cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; th[0]=tt[0]; th[1]=tt[1]; }
        }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        double md = 0; for (int i = 0; i < n; ++i) md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i])));
        printf("v6 var=%d (%s) threads=%d: %.1f us/sweep cyc/level=%.0f maxrel=%.2e err=%s\n", var, var==0?"levelorder,div":var==1?"levelorder,div,pf":"levelorder,recip,pf", threads, best, th[0]/(double)f.n_levels, md, cudaGetErrorString(cudaGetLastError()));
      }
      long long* ts; cudaMalloc(&ts, f.n_groups * 32);
      sweep6<false,true><<<1, 1024, smem3>>>(s6, n, r, out, t, 3, ts); cudaDeviceSynchronize();
      std::vector<long long> h(f.n_groups * 4); cudaMemcpy(h.data(), ts, h.size()*8, cudaMemcpyDeviceToHost);
      double sA=0,sB=0,sC=0,sD=0; int cnt=0;
      for (int g = 64; g < f.n_groups - 64; ++g) { sA += h[g*4+1]-h[g*4+0]; sB += h[g*4+2]-h[g*4+1]; sC += h[g*4+3]-h[g*4+2]; sD += h[g*4+3]-h[(g-1)*4+3]; cnt++; }
      printf("v6 mean cycles: start->prefixdone %.0f, tail wait %.0f, div+publish %.0f, publish-to-publish %.0f\n", sA/cnt, sB/cnt, sC/cnt, sD/cnt);
      for (int g = 500; g < 506; ++g) printf("  g=%d start=%lld prefix=%lld tail=%lld pub=%lld\n", g, h[g*4], h[g*4+1], h[g*4+2], h[g*4+3]);
      // how many tail entries are at lev-1 / lev-2 and prefix max level
      long long pref_bad = 0, rows_cnt = 0;
      for (int g = 0; g < f.n_groups; ++g) for (int l = 0; l < h6.gnrow[g]; ++l) { int row = h6.grows[g*32+l]; rows_cnt++;
        for (int k = 0; k < h6.gpw[g]; ++k) { int c = h6.cols[h6.gptr[g] + (int64_t)k*h6.gnrow[g] + l]; if (c >= 0 && lev[c] >= lev[row]-2) { pref_bad++; break; } } }
      printf("rows with prefix deps at level >= l-2: %lld of %lld\n", pref_bad, rows_cnt);
      cudaFuncSetAttribute(chain7, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024*8);
      chain7<<<1,1024,1024*8>>>(1024, t, out); cudaDeviceSynchronize();
      unsigned long long tt[2]; cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
      printf("pure chain: %.0f cycles/level err=%s\n", tt[0]/1024.0, cudaGetErrorString(cudaGetLastError()));
    }

    if (!only11) {
      unsigned long long tt[2];
      cudaFuncSetAttribute(chain8<false,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
      cudaFuncSetAttribute(chain8<true,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
      cudaFuncSetAttribute(chain8<false,32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
      for (int threads : {64, 128, 256, 512, 1024}) {
        chain8<false,0><<<1,threads,8192>>>(1024, t, out); cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost); double a = tt[0]/1024.0;
        chain8<true,0><<<1,threads,8192>>>(1024, t, out); cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost); double b = tt[0]/1024.0;
        chain8<false,32><<<1,threads,8192>>>(1024, t, out); cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost); double c = tt[0]/1024.0;
        printf("chain8 threads=%d: div %.0f  recip %.0f  div+sleep32 %.0f cycles/level\n", threads, a, b, c);
      }
      chain9<false><<<1,1>>>(1024, t, out); cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost); printf("chain9 div: %.1f cycles/level\n", tt[0]/1024.0);
      chain9<true><<<1,1>>>(1024, t, out); cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost); printf("chain9 recip: %.1f cycles/level\n", tt[0]/1024.0);
    }

    if (!only11) for (int D : {2, 3, 4, 6, 8}) {
      H8 h8 = build8(f, D);
      if (h8.TW > 16) { printf("v8 D=%d TW=%d too big\n", D, h8.TW); continue; }
      S8 s8{h8.G, up(h8.nr), up(h8.need), up(h8.grows), up(h8.pw), up(h8.tw), up(h8.pcols), up(h8.tcols), up(h8.pptr), up(h8.tptr), up(h8.pvals), up(h8.tvals), up(f.diag)};
      const int TWM = 16;
      size_t smem8 = n*8 + R8*32*8*2 + R8*TWM*32*12 + R8*32*4 + R8*4 + 16 + R8*8;
      cudaFuncSetAttribute(sweep8<16,false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      cudaFuncSetAttribute(sweep8<16,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      for (int rc = 0; rc < 2; ++rc)
      for (int threads : {1024, 512, 256}) {
        unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0; double waitfrac = 0;
        for (int rep = 0; rep < 3; ++rep) {
          if (rc) sweep8<16,true><<<1, threads, smem8>>>(s8, n, r, out, t, 4); else sweep8<16,false><<<1, threads, smem8>>>(s8, n, r, out, t, 4);
          cudaDeviceSynchronize(); unsigned long long t3[3]; cudaMemcpy(t3, t, 24, cudaMemcpyDeviceToHost); tt[0]=t3[0]; tt[1]=t3[1];
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; waitfrac = t3[2]/(double)t3[0]; }
        }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        bool eq = true; for (int i = 0; i < n; ++i) eq &= o1[i]==o2[i];
        printf("v8 %s D=%d TW=%d threads=%d smem=%zu: %.1f us/sweep cyc/level=%.0f main-wait-frac=%.2f bitexact=%d err=%s\n", rc?"recip":"div", D, h8.TW, threads, smem8, best, bc/(double)f.n_levels, waitfrac, (int)eq, cudaGetErrorString(cudaGetLastError()));
      }
    }

    if (!only11) {
      H8 h8 = build8(f, 6);
      S8 s8{h8.G, up(h8.nr), up(h8.need), up(h8.grows), up(h8.pw), up(h8.tw), up(h8.pcols), up(h8.tcols), up(h8.pptr), up(h8.tptr), up(h8.pvals), up(h8.tvals), up(f.diag)};
      const int TWM = 16;
      size_t smem8 = n*8 + R8*32*8*2 + R8*TWM*32*12 + R8*32*4 + R8*4 + 16 + R8*8;
      long long* tsg; cudaMalloc(&tsg, h8.G * 24);
      sweep8<16,true><<<1, 256, smem8>>>(s8, n, r, out, t, 2, tsg); cudaDeviceSynchronize();
      std::vector<long long> hh(h8.G*3); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
      double a=0,b=0,c=0; for (int g = 0; g < h8.G; ++g) { a += hh[g*3]; b += hh[g*3+1]; c += hh[g*3+2]; }
      printf("v8 main breakdown (cycles/group): wait-ready %.0f, compute %.0f, fence+progress %.0f ; tw mean %.1f\n", a/h8.G, b/h8.G, c/h8.G, [&]{double s=0; for (int x : h8.tw) s+=x; return s/h8.G;}());
    }

    if (!only11) for (int D : {6}) {
      H8 h8 = build8(f, D);
      S8 s8{h8.G, up(h8.nr), up(h8.need), up(h8.grows), up(h8.pw), up(h8.tw), up(h8.pcols), up(h8.tcols), up(h8.pptr), up(h8.tptr), up(h8.pvals), up(h8.tvals), up(f.diag)};
      const int TWM = 16;
      size_t smem8 = n*8 + 8 + R8*32*8*2 + R8*TWM*32*12 + R8*32*4 + R8*4 + 16 + R8*8;
      cudaFuncSetAttribute(sweep9<16,false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      cudaFuncSetAttribute(sweep9<16,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      cudaFuncSetAttribute(sweep9<16,false,1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      cudaFuncSetAttribute(sweep9<16,false,2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8);
      long long* tsg; cudaMalloc(&tsg, h8.G * 24);
      for (int rc = 0; rc < 4; ++rc) for (int threads : {256}) {
        unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
        for (int rep = 0; rep < 3; ++rep) {
          if (rc == 1) sweep9<16,true><<<1, threads, smem8>>>(s8, n, r, out, t, 4, tsg); else if (rc == 0) sweep9<16,false><<<1, threads, smem8>>>(s8, n, r, out, t, 4, tsg);
          else if (rc == 2) sweep9<16,false,1><<<1, threads, smem8>>>(s8, n, r, out, t, 4, tsg); else sweep9<16,false,2><<<1, threads, smem8>>>(s8, n, r, out, t, 4, tsg);
          cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
        }
        std::vector<long long> hh(h8.G*3); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
        double a=0,b=0,c=0; for (int g = 0; g < h8.G; ++g) { a += hh[g*3]; b += hh[g*3+1]; c += hh[g*3+2]; }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        bool eq = true; for (int i = 0; i < n; ++i) eq &= o1[i]==o2[i];
        printf("v9 mode=%d %s D=%d threads=%d: %.1f us/sweep cyc/level=%.0f [main: wait %.0f compute %.0f fence %.0f] bitexact=%d err=%s\n", rc, rc==1?"recip":"div", D, threads, best, bc/(double)f.n_levels, a/h8.G, b/h8.G, c/h8.G, (int)eq, cudaGetErrorString(cudaGetLastError()));
      }
    }

    if (!only11) for (int lo = 0; lo < 2; ++lo) for (int D : {6}) {
      constexpr int TA = 8, TB = 10;
      H10 h = build10<TA, TB>(f, D, lo == 1);
      S10d sd{h.G, up(h.nr), up(h.need), up(h.amax), up(h.bmax), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bcol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag)};
      size_t smem10 = (n + 1) * 8 + R10*32*8*2 + R10*TA*32*12 + R10*TB*32*13 + R10*32*4 + 4*R10*4 + 64;
      cudaFuncSetAttribute(sweep10<TA,TB,false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem10);
      cudaFuncSetAttribute(sweep10<TA,TB,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem10);
      cudaFuncSetAttribute(sweep10<TA,TB,true,1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem10);
      cudaFuncSetAttribute(sweep10<TA,TB,true,2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem10);
      long long* tsg; cudaMalloc(&tsg, h.G * 16);
      for (int mk = 1; mk < 4; ++mk) for (int threads : {512, 256}) {
        unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
        for (int rep = 0; rep < 3; ++rep) {
          if (mk == 1) sweep10<TA,TB,true><<<1, threads, smem10>>>(sd, n, r, out, t, 4, tsg);
          else if (mk == 2) sweep10<TA,TB,true,1><<<1, threads, smem10>>>(sd, n, r, out, t, 4, tsg);
          else sweep10<TA,TB,true,2><<<1, threads, smem10>>>(sd, n, r, out, t, 4, tsg);
          cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
          if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
        }
        std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
        double a=0,b=0; for (int g = 0; g < h.G; ++g) { a += hh[g*2]; b += hh[g*2+1]; }
        cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
        bool eq = true; double md = 0; for (int i = 0; i < n; ++i) { eq &= o1[i]==o2[i]; md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i]))); }
        printf("v10 excl=%d %s %s D=%d TAm=%d TBm=%d threads=%d: %.1f us/sweep cyc/level=%.0f [B %.0f, A %.0f] bitexact=%d maxrel=%.1e err=%s\n", mk-1, lo?"levelord":"colord", mk?"markstein":"div", D, h.TAm, h.TBm, threads, best, bc/(double)f.n_levels, a/h.G, b/h.G, (int)eq, md, cudaGetErrorString(cudaGetLastError()));
      }
    }

    {
      std::vector<double> dinvh(n); for (int i = 0; i < n; ++i) dinvh[i] = 1.0 / f.diag[i];
      double* ddinv = up(dinvh);
      auto runv11 = [&](auto TAc, auto TBc, int D, bool lo) {
        constexpr int TA = decltype(TAc)::value, TB = decltype(TBc)::value;
        H10 h = build10<TA, TB>(f, D, lo);
        S10d sd{h.G, up(h.nr), up(h.need), up(h.amax), up(h.bmax), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bcol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag)};
        size_t smem = (n + 1) * 8 + R10*32*8*3 + R10*TA*32*12 + R10*TB*32*16 + R10*32*4 + 2*R10*4 + 64;
        cudaFuncSetAttribute(sweep11<TA,TB,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long* tsg; cudaMalloc(&tsg, h.G * 16);
        for (int threads : {512, 256}) {
          unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
          for (int rep = 0; rep < 3; ++rep) {
            sweep11<TA,TB,true><<<1, threads, smem>>>(sd, ddinv, n, r, out, t, 4, tsg);
            cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
            if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
          }
          std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0, wsum=0; for (int g = 0; g < h.G; ++g) { a += hh[g*2]; wsum += hh[g*2+1]; }
          cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
          bool eq = true; double md = 0; for (int i = 0; i < n; ++i) { eq &= o1[i]==o2[i]; md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i]))); }
          printf("v11 %s TA=%d TB=%d D=%d (TAm=%d TBm=%d) threads=%d: %.1f us/sweep cyc/level=%.0f [main iter %.0f, ready-wait %.0f] bitexact=%d maxrel=%.1e err=%s\n", lo?"levelord":"colord", TA, TB, D, h.TAm, h.TBm, threads, best, bc/(double)f.n_levels, a/h.G, wsum/h.G, (int)eq, md, cudaGetErrorString(cudaGetLastError()));
        }
      };
      runv11(std::integral_constant<int,8>(), std::integral_constant<int,8>(), 6, false);
      runv11(std::integral_constant<int,8>(), std::integral_constant<int,3>(), 6, true);
      runv11(std::integral_constant<int,12>(), std::integral_constant<int,3>(), 10, true);
      runv11(std::integral_constant<int,4>(), std::integral_constant<int,2>(), 4, true);
    }

    {
      std::vector<double> dinvh(n); for (int i = 0; i < n; ++i) dinvh[i] = 1.0 / f.diag[i];
      double* ddinv = up(dinvh);
      auto runv12 = [&](auto TAc, auto TBc, int D) {
        constexpr int TA = decltype(TAc)::value, TB = decltype(TBc)::value;
        H10 h = build10<TA, TB>(f, D, true);
        S10d sd{h.G, up(h.nr), up(h.need), up(h.amax), up(h.bmax), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bcol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag)};
        size_t smem = (n + 1) * 8 + R10*32*8*3 + R10*TA*32*12 + R10*TB*32*16 + R10*32*4 + 2*R10*4 + 64;
        cudaFuncSetAttribute(sweep12<TA,TB,16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long* tsg; cudaMalloc(&tsg, h.G * 16);
        for (int threads : {512, 256}) {
          unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
          for (int rep = 0; rep < 3; ++rep) {
            sweep12<TA,TB,16><<<1, threads, smem>>>(sd, ddinv, n, r, out, t, 4, tsg);
            cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
            if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
          }
          std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0, wsum=0; for (int g = 0; g < h.G; ++g) { a += hh[g*2]; wsum += hh[g*2+1]; }
          cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
          double md = 0; for (int i = 0; i < n; ++i) md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i])));
          printf("v12 TA=%d TB=%d D=%d (TAm=%d TBm=%d) threads=%d: %.1f us/sweep cyc/level=%.0f [main iter %.0f, ready-wait %.0f] maxrel=%.1e err=%s\n", TA, TB, D, h.TAm, h.TBm, threads, best, bc/(double)f.n_levels, a/h.G, wsum/h.G, md, cudaGetErrorString(cudaGetLastError()));
        }
      };
      runv12(std::integral_constant<int,8>(), std::integral_constant<int,4>(), 6);
      runv12(std::integral_constant<int,16>(), std::integral_constant<int,4>(), 10);
      runv12(std::integral_constant<int,4>(), std::integral_constant<int,4>(), 4);
    }

    {
      std::vector<double> dinvh(n); for (int i = 0; i < n; ++i) dinvh[i] = 1.0 / f.diag[i];
      double* ddinv = up(dinvh);
      H10 h = build10<8, 4>(f, 6, true);
      S10d sd{h.G, up(h.nr), up(h.need), up(h.amax), up(h.bmax), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bcol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag)};
      size_t smem = (n + 1) * 8 + R10*32*8*3 + R10*8*32*12 + R10*4*32*16 + R10*32*4 + 2*R10*4 + 64;
      cudaFuncSetAttribute(sweep12<8,4,16,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      long long* tsg; cudaMalloc(&tsg, h.G * 16);
      for (int threads : {512, 32}) {
        sweep12<8,4,16,true><<<1, threads, smem>>>(sd, ddinv, n, r, out, t, 2, tsg); cudaDeviceSynchronize();
        std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
        double a=0; for (int g = 0; g < h.G; ++g) a += hh[g*2];
        printf("v12-ISO threads=%d main iter %.0f cycles err=%s\n", threads, a/h.G, cudaGetErrorString(cudaGetLastError()));
      }
    }

    {
      std::vector<double> dinvh(n); for (int i = 0; i < n; ++i) dinvh[i] = 1.0 / f.diag[i];
      double* ddinv = up(dinvh);
      auto runv13 = [&](auto TAc, auto TBc, int D) {
        constexpr int TA = decltype(TAc)::value, TB = decltype(TBc)::value;
        H10 h = build10<TA, TB>(f, D, true);
        S10d sd{h.G, up(h.nr), up(h.need), up(h.amax), up(h.bmax), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bcol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag)};
        size_t smem = (n + 1) * 8 + R10*32*8*3 + R10*TA*32*12 + R10*TB*32*16 + R10*32*4 + 2*R10*4 + 64;
        cudaFuncSetAttribute(sweep13<TA,TB,16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep13<TA,TB,16,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long* tsg; cudaMalloc(&tsg, h.G * 16);
        sweep13<TA,TB,16,true><<<1, 512, smem>>>(sd, ddinv, n, r, out, t, 2, tsg); cudaDeviceSynchronize();
        { std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0; for (int g = 0; g < h.G; ++g) a += hh[g*2]; printf("v13-ISO TA=%d TB=%d main iter %.0f\n", TA, TB, a/h.G); }
        for (int threads : {512, 256}) {
          unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
          for (int rep = 0; rep < 3; ++rep) {
            sweep13<TA,TB,16><<<1, threads, smem>>>(sd, ddinv, n, r, out, t, 4, tsg);
            cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
            if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
          }
          std::vector<long long> hh(h.G*2); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0; for (int g = 0; g < h.G; ++g) a += hh[g*2];
          cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
          double md = 0; for (int i = 0; i < n; ++i) md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i])));
          printf("v13 TA=%d TB=%d D=%d (TAm=%d TBm=%d) threads=%d: %.1f us/sweep cyc/level=%.0f [main iter %.0f] maxrel=%.1e err=%s\n", TA, TB, D, h.TAm, h.TBm, threads, best, bc/(double)f.n_levels, a/h.G, md, cudaGetErrorString(cudaGetLastError()));
        }
      };
      runv13(std::integral_constant<int,8>(), std::integral_constant<int,4>(), 6);
      runv13(std::integral_constant<int,16>(), std::integral_constant<int,4>(), 10);
      runv13(std::integral_constant<int,8>(), std::integral_constant<int,2>(), 6);
    }

    {
      std::vector<double> dinvh(n); for (int i = 0; i < n; ++i) dinvh[i] = 1.0 / f.diag[i];
      double* ddinv = up(dinvh);
      auto runv14 = [&](auto TAc, auto TBc, int D) {
        constexpr int TA = decltype(TAc)::value, TB = decltype(TBc)::value;
        H14 h = build14<TA, TB>(f, D);
        S14d sd{h.G, up(h.nr), up(h.need), up(h.grows), up(h.pw), up(h.pcols), up(h.acol), up(h.bsrc), up(h.pptr), up(h.pvals), up(h.aval), up(h.bval), up(f.diag), ddinv};
        size_t smem = (n + 1) * 8 + R10*32*8*3 + R10*TA*32*12 + R10*TB*32*12 + R10*32*4 + 2*R10*4 + 64;
        cudaFuncSetAttribute(sweep14<TA,TB,16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(sweep14<TA,TB,16,true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long* tsg; cudaMalloc(&tsg, h.G * 8);
        sweep14<TA,TB,16,true><<<1, 512, smem>>>(sd, n, r, out, t, 2, tsg); cudaDeviceSynchronize();
        { std::vector<long long> hh(h.G); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0; for (int g = 0; g < h.G; ++g) a += hh[g]; printf("v14-ISO TA=%d TB=%d main iter %.0f\n", TA, TB, a/h.G); }
        for (int threads : {512, 256}) {
          unsigned long long tt[2]; float best = 1e9; unsigned long long bc = 0;
          for (int rep = 0; rep < 3; ++rep) {
            sweep14<TA,TB,16><<<1, threads, smem>>>(sd, n, r, out, t, 4, tsg);
            cudaDeviceSynchronize(); cudaMemcpy(tt, t, 16, cudaMemcpyDeviceToHost);
            if (tt[1]*1e-3 < best) { best = tt[1]*1e-3; bc = tt[0]; }
          }
          std::vector<long long> hh(h.G); cudaMemcpy(hh.data(), tsg, hh.size()*8, cudaMemcpyDeviceToHost);
          double a=0; for (int g = 0; g < h.G; ++g) a += hh[g];
          cudaMemcpy(o2.data(), out, n*8, cudaMemcpyDeviceToHost);
          double md = 0; for (int i = 0; i < n; ++i) md = std::max(md, std::abs(o1[i]-o2[i])/std::max(1e-300,std::abs(o1[i])));
          printf("v14 TA=%d TB=%d D=%d threads=%d: %.1f us/sweep cyc/level=%.0f [main iter %.0f] maxrel=%.1e err=%s\n", TA, TB, D, threads, best, bc/(double)f.n_levels, a/h.G, md, cudaGetErrorString(cudaGetLastError()));
        }
      };
      runv14(std::integral_constant<int,8>(), std::integral_constant<int,4>(), 7);
      runv14(std::integral_constant<int,12>(), std::integral_constant<int,4>(), 10);
      runv14(std::integral_constant<int,6>(), std::integral_constant<int,4>(), 5);
    }
  }
  return 0;
}
