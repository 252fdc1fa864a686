// Device building blocks for the B200 MINRES + IC(0) solve (sm_100a, fp64).
//
// Arithmetic convention: every element-wise update uses explicitly rounded
// mul/add/sub/div (__dmul_rn etc.), i.e. no FMA contraction, so each update
// rounds exactly like the reference's scalar C++ (x86-64 baseline, no FMA).
// Reductions (dot products, SpMV row sums) use a fixed warp-shuffle tree and a
// fixed CTA/grid order: deterministic run to run, different summation order
// from the reference (round-off level).
#pragma once

#include <cstdint>

namespace dsgpu {
namespace dev {

constexpr unsigned long long kSentinel = 0xFFF4A11C0DEDBEEFull;  // "not yet computed" (a NaN payload)
constexpr unsigned long long kCanonNaN = 0x7FF8000000000000ull;
constexpr long long kSpinTimeoutCycles = 2000000000ll;  // grid barrier / mailbox waits (cycles)
// Abort flag values: a device spin that gives up sets the flag so every other
// spin ends too (the solve returns an error instead of hanging the GPU).
constexpr unsigned kAbortSet = 1u, kAbortTimeout = 2u;
// Wall-clock limit of one device spin in ns (%globaltimer: independent of the
// SM clock, so throttling or a profiler's replay do not shorten it);
// DSGPU_TIMEOUT_S sets it at dsgpu_setup (default 10 s).
__device__ unsigned long long g_spin_timeout_ns = 10000000000ull;
__device__ __forceinline__ unsigned long long wall_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA sum; result valid in every thread of warp 0.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// ---- CSR SpMV with 128-bit loads --------------------------------------------
// Device operators are stored with every row (the velocity rows of K': each of
// the two parts [A' | Bt']) padded to a multiple of 4 entries (pad: the row's
// own column, value 0), so a row starts on a 16-byte boundary of both the
// int32 column array and the f64 value array. L lanes (8, 16 or 32, chosen per
// operator from its mean row length) cooperate on a row: lane `sub` reads
// entries 4 sub .. 4 sub + 3 as one int4 + two double2 and strides 4 L. The
// matrix is streamed (evict-first); the gathered vector stays cached.
template <class X>
__device__ __forceinline__ double row_partial(const int32_t* ci, const double* v, int len, int sub, int L, X xf) {
  const int4* cp = reinterpret_cast<const int4*>(ci) + sub;
  const double2* vp = reinterpret_cast<const double2*>(v) + 2 * sub;
  double a0 = 0.0, a1 = 0.0;
  for (int k = 4 * sub; k < len; k += 4 * L, cp += L, vp += 2 * L) {
#ifdef DSGPU_SPMV_LDG
    const int4 c = __ldg(cp);
    const double2 p = __ldg(vp), q = __ldg(vp + 1);
#else
    const int4 c = __ldcs(cp);
    const double2 p = __ldcs(vp), q = __ldcs(vp + 1);
#endif
    a0 = fma(p.x, xf(c.x), a0);
    a1 = fma(p.y, xf(c.y), a1);
    a0 = fma(q.x, xf(c.z), a0);
    a1 = fma(q.y, xf(c.w), a1);
  }
  return a0 + a1;
}
// sum over the L lanes of a row group (L a power of two <= 32); all 32 lanes call it
__device__ __forceinline__ double group_sum(double v, int L) {
  for (int o = L >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row loop of the SpMV phases INSIDE the persistent kernel, software-pipelined.
// A persistent CTA is alone on its SM (16 warps), so with one 48-byte trip per
// lane in flight the phase is latency-bound (measured in the diag build:
// 25 GB/s per CTA, 3.5 TB/s over the grid, against 6.2 TB/s for spmv_kernel
// at full occupancy). Here every lane issues the NEXT trip of its row -- or,
// on the row's last trip, the first trip of its next row -- before the
// current trip's gathers, and reads the next row's extent one row ahead: two
// trips per lane in flight and no row-pointer latency on the path. The
// per-lane order of the products is that of row_partial, so the results are
// bit-identical to it.
//   info(i, s, len): first stored entry and entry count of row i (lo <= i < hi)
//   xf(j): the gathered operand; done(i, ok, sum): called by every lane after
//   the row group's shuffle sum (ok: the lane's row exists)
struct SpmvTrip {
  int4 c;
  double2 p, q;
};
__device__ __forceinline__ SpmvTrip spmv_trip(const int32_t* ci, const double* v, int64_t at) {
  SpmvTrip t;
  const double2* vp = reinterpret_cast<const double2*>(v + at);
  t.c = __ldcs(reinterpret_cast<const int4*>(ci + at));
  t.p = __ldcs(vp);
  t.q = __ldcs(vp + 1);
  return t;
}
template <class Info, class X, class Done>
__device__ __forceinline__ void spmv_rows(int lo, int hi, int L, const int32_t* ci, const double* v, Info info,
                                          X xf, Done done) {
  const int lane = threadIdx.x & 31, sub = lane & (L - 1), per = 32 / L;
  const int ng = static_cast<int>(blockDim.x >> 5) * per;
  int i = lo + static_cast<int>(threadIdx.x >> 5) * per + lane / L;
  bool ok = i < hi;
  int64_t s = 0;
  int len = 0;
  if (ok) info(i, s, len);
  bool have = ok && 4 * sub < len;
  SpmvTrip t = {};
  if (have) t = spmv_trip(ci, v, s + 4 * sub);
  for (int base = lo; base < hi; base += ng) {
    const int in = i + ng;
    const bool okn = in < hi;
    int64_t sn = 0;
    int lenn = 0;
    if (okn) info(in, sn, lenn);
    const bool first_n = okn && 4 * sub < lenn;
    double a0 = 0.0, a1 = 0.0;
    bool ahead = false;  // the next row's first trip is already in flight
    int k = 4 * sub;
    while (have) {
      const int kn = k + 4 * L;
      const bool more = kn < len;
      SpmvTrip n = {};
      if (more) {
        n = spmv_trip(ci, v, s + kn);
      } else {
        if (first_n) n = spmv_trip(ci, v, sn + 4 * sub);
        ahead = true;
      }
      a0 = fma(t.p.x, xf(t.c.x), a0);
      a1 = fma(t.p.y, xf(t.c.y), a1);
      a0 = fma(t.q.x, xf(t.c.z), a0);
      a1 = fma(t.q.y, xf(t.c.w), a1);
      t = n;
      k = kn;
      have = more;
    }
    if (!ahead && first_n) t = spmv_trip(ci, v, sn + 4 * sub);
    done(i, ok, group_sum(a0 + a1, L));
    i = in;
    ok = okn;
    s = sn;
    len = lenn;
    have = first_n;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).
// Fences on both sides make every write before the barrier visible to every
// read after it (and invalidate this SM's L1 on the way out). Returns false
// on timeout (abort flag set) instead of hanging the GPU.
// Barrier over `expected` CTAs (the participating ones; default: the grid).
__device__ __forceinline__ bool grid_sync(unsigned* count, unsigned* gen, unsigned* abort_flag,
                                          unsigned expected = 0) {
  if (expected == 0) expected = gridDim.x;
  __shared__ int ok_sh;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
    const unsigned g = ld_acquire(gen);
    __threadfence();
    const unsigned prev = atomicAdd(count, 1u);
    if (prev == expected - 1) {
      atomicExch(count, 0u);
      __threadfence();
      st_release(gen, g + 1);
    } else {
      const long long t0 = clock64();
      const unsigned long long w0 = wall_ns();
      while (ld_acquire(gen) == g) {
        if (*reinterpret_cast<volatile unsigned*>(abort_flag)) {
          ok = 0;
          break;
        }
        if (clock64() - t0 > kSpinTimeoutCycles && wall_ns() - w0 > g_spin_timeout_ns) {
          atomicCAS(abort_flag, 0u, kAbortTimeout);
          ok = 0;
          break;
        }
      }
    }
    __threadfence();
    ok_sh = ok;
  }
  __syncthreads();
  return ok_sh != 0;
}

// Bounded spin: expires after kSpinTimeoutCycles (sets the abort flag) or as
// soon as another thread has aborted; the flag is only read after a short
// grace period so the fast path stays free of global loads.
struct SpinGuard {
  long long t0;              // cycles: the cheap test of the fast path
  unsigned long long w0 = 0; // wall clock, taken once the grace period is over
  unsigned* ab;
  __device__ __forceinline__ explicit SpinGuard(unsigned* a) {
#ifdef __CUDA_ARCH__
    t0 = clock64();
#else
    t0 = 0;
#endif
    ab = a;
  }
  __device__ __forceinline__ bool expired() {
#ifdef __CUDA_ARCH__
    const long long dt = clock64() - t0;
    if (dt < (1ll << 16)) return false;
    if (*reinterpret_cast<volatile unsigned*>(ab)) return true;
    const unsigned long long now = wall_ns();
    if (w0 == 0) w0 = now;
    if (now - w0 > g_spin_timeout_ns) {
      atomicCAS(ab, 0u, kAbortTimeout);
      return true;
    }
#endif
    return false;
  }
};

// ---- shared-memory dataflow slots for the triangular sweeps --------------
__device__ __forceinline__ void slot_reset(double* xs, int i) {
  reinterpret_cast<volatile unsigned long long*>(xs)[i] = kSentinel;
}
__device__ __forceinline__ void slot_publish(double* xs, int i, double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  if (b == kSentinel) b = kCanonNaN;
  reinterpret_cast<volatile unsigned long long*>(xs)[i] = b;
}
// Spin until slot c holds a value. On timeout sets *abort_flag and returns NaN.
__device__ __forceinline__ double slot_wait(const double* xs, int c, unsigned* abort_flag) {
  const volatile unsigned long long* p = reinterpret_cast<const volatile unsigned long long*>(xs);
  unsigned long long b = p[c];
  if (b != kSentinel) return __longlong_as_double(static_cast<long long>(b));
  const long long t0 = clock64();
  do {
    b = p[c];
    const long long dt = clock64() - t0;
    // slow path only after ~0.5 ms of waiting: a global abort-flag load costs
    // an L2 round trip and must stay off the per-level critical path
    if (dt > (1ll << 20) &&
        (dt > kSpinTimeoutCycles || *reinterpret_cast<volatile unsigned*>(abort_flag))) {
      atomicExch(abort_flag, 1u);
      return __longlong_as_double(static_cast<long long>(kCanonNaN));
    }
  } while (b == kSentinel);
  return __longlong_as_double(static_cast<long long>(b));
}

// ---- mbarrier / bulk-copy (TMA) helpers -----------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* mb, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
      : "=r"(ok)
      : "r"(smem_u32(mb)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mb))
      : "memory");
}
// non-blocking poll (try_wait may suspend the thread for a while)
__device__ __forceinline__ bool mbar_poll(uint64_t* mb, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
      : "=r"(ok)
      : "r"(smem_u32(mb)), "r"(parity)
      : "memory");
  return ok != 0;
}

}  // namespace dev
}  // namespace dsgpu
