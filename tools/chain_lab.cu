// Lab: IC(0) apply z = (L L^T)^{-1} r as a block-partitioned-inverse chain
// with warp-level dataflow (no barriers). Each output row is one warp task:
//   out = segB . srcB[jB..jB+lB) + segA . srcA[jA..jA+lA)
// forward  (block i, row r): segB = Dinv_i[r, 0..r]   on r,  segA = -F_i[r,:] on y tail
// backward (block i, row r): segB = Dinv_i^T[r, r..b) on y,  segA = -H_i[r,:] on z head
// y / z hold a sentinel NaN until written; consumers poll the values themselves.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace {
constexpr unsigned long long kSent = 0xFFF4A11C0DEDBEEFull;
#ifndef SLEEPNS
#define SLEEPNS 64
#endif
constexpr int kSleepNs = SLEEPNS;

struct Task {
  int out, flags;  // flags: bits 0-2 out vector, 3-5 base vector (7 = none), 6-8 src vector, bit 9 poll src
  int jB, lB, pad0, pad1;  // segment: src[jB .. jB + lB) . coef[off ..]
  long long off;
};

__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(x)) : "memory");
}

template <int U>
__device__ __forceinline__ double seg_dot(const double* __restrict__ c, const double* src, int len,
                                          bool poll, int lane, double acc) {
  for (int base = 0; base < len; base += 32 * U) {
    double cv[U];
    unsigned long long sv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u * 32 + lane;
      cv[u] = k < len ? __ldg(c + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = base + u * 32 + lane;
      sv[u] = k < len ? (poll ? ld_relaxed(src + k) : __double_as_longlong(src[k])) : 0ull;
    }
    if (poll) {
      bool miss = false;
#pragma unroll
      for (int u = 0; u < U; ++u) miss |= sv[u] == kSent;
      while (miss) {
        __nanosleep(16);
        miss = false;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (sv[u] == kSent) sv[u] = ld_relaxed(src + base + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < U; ++u) miss |= sv[u] == kSent;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(cv[u], __longlong_as_double(sv[u]), acc);
  }
  return acc;
}

// all loads of a segment issued before any use; poll only what is missing
template <int UA, class W>
__device__ __forceinline__ double seg_regs(const double* __restrict__ c, const double* src, int len,
                                           bool poll, int lane, double acc, W wait) {
  double cv[UA];
  unsigned long long sv[UA];
#pragma unroll
  for (int u = 0; u < UA; ++u) {
    const int k = u * 32 + lane;
    cv[u] = k < len ? __ldg(c + k) : 0.0;
  }
  wait();
#pragma unroll
  for (int u = 0; u < UA; ++u) {
    const int k = u * 32 + lane;
    sv[u] = k < len ? (poll ? ld_relaxed(src + k) : __double_as_longlong(src[k])) : 0ull;
  }
  if (poll) {
    // waiting costs one load per lane per round; a round that made progress
    // is followed by a batch reload of everything still missing
    bool batch = false;
    for (;;) {
      bool miss = false;
#pragma unroll
      for (int u = 0; u < UA; ++u) miss |= sv[u] == kSent;
      if (!__any_sync(0xffffffffu, miss)) break;
      if (!batch) __nanosleep(kSleepNs);
      bool got = false, first = true;
#pragma unroll
      for (int u = 0; u < UA; ++u)
        if (sv[u] == kSent && (batch || first)) {
          first = false;
          sv[u] = ld_relaxed(src + u * 32 + lane);
          got |= sv[u] != kSent;
        }
      batch = __any_sync(0xffffffffu, got);
    }
  }
#pragma unroll
  for (int u = 0; u < UA; ++u) acc = fma(cv[u], __longlong_as_double(sv[u]), acc);
  return acc;
}

template <class W>
__device__ __forceinline__ double seg_any(const double* __restrict__ c, const double* src, int len,
                                          bool poll, int lane, double acc, W wait) {
  if (len <= 8 * 32) return seg_regs<8>(c, src, len, poll, lane, acc, wait);
  if (len <= 16 * 32) return seg_regs<16>(c, src, len, poll, lane, acc, wait);
  if (len <= 24 * 32) return seg_regs<24>(c, src, len, poll, lane, acc, wait);
  wait();
  return seg_dot<8>(c, src, len, poll, lane, acc);
}

__device__ __forceinline__ double poll1(const double* p) {
  unsigned long long v = ld_relaxed(p);
  while (v == kSent) {
    __nanosleep(kSleepNs);
    v = ld_relaxed(p);
  }
  return __longlong_as_double(v);
}

// vectors: 0 r, 1 g, 2 y, 3 h, 4 z
// Task.pad0 = chain block of the output (-1: bulk task), pad1 = chain block the
// segment depends on (-1: none). Warp 15 of every CTA is the watcher: it polls
// the per-chain-block completion counters in order and publishes progress in
// shared memory, so chain warps wait on shared memory instead of polling L2.
constexpr int kMaxChain = 256;
__global__ void __launch_bounds__(512, 1)
chain_kernel(const Task* __restrict__ T, const int* __restrict__ wptr, const double* __restrict__ coef,
             double* vec0, int n, unsigned long long* trace, unsigned* cnt, const int* __restrict__ total,
             const int* __restrict__ quota, int nc) {
  __shared__ unsigned sc[kMaxChain];
  __shared__ int q_sh[kMaxChain];
  __shared__ volatile int ready;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    sc[c] = 0;
    q_sh[c] = quota[blockIdx.x * nc + c];
  }
  if (threadIdx.x == 0) ready = 0;
  __syncthreads();
  if (warp == 15) {
    if (lane == 0) {
      for (int c = 0; c < nc; ++c) {
        const unsigned tot = total[c];
        while (true) {
          unsigned v;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + c) : "memory");
          if (v >= tot) break;
        }
        ready = c + 1;
      }
    }
    return;
  }
  const int gw = blockIdx.x * 15 + warp;
  const int t1 = wptr[gw + 1];
  for (int t = wptr[gw]; t < t1; ++t) {
    unsigned long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const Task tk = T[t];
    const int ov = tk.flags & 7, bv = (tk.flags >> 3) & 7, sv = (tk.flags >> 6) & 7;
    const bool pl = (tk.flags >> 9) & 1;
    double base = 0.0;
    if (bv != 7 && lane == 0) base = poll1(vec0 + (size_t)bv * n + tk.out);
    const int dep = tk.pad1;
    double acc = seg_any(coef + tk.off, vec0 + (size_t)sv * n + tk.jB, tk.lB, pl, lane, 0.0, [&] {
      if (dep >= 0)
        while (ready <= dep) {
        }
    });
    unsigned long long gr;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gr));
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      acc += base;
      st_relaxed(vec0 + (size_t)ov * n + tk.out, acc);
      if (tk.pad0 >= 0) {
        const unsigned old = atomicAdd(&sc[tk.pad0], 1u);
        if (old + 1 == (unsigned)q_sh[tk.pad0])
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(cnt + tk.pad0), "r"(q_sh[tk.pad0]) : "memory");
      }
      if (trace) {
        unsigned long long g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        trace[3 * t] = g0;
        trace[3 * t + 1] = gr;
        trace[3 * t + 2] = g1;
      }
    }
  }
}

__global__ void fill_sent(double* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    reinterpret_cast<unsigned long long*>(p)[i] = kSent;
}
}  // namespace

extern "C" int chain_run(int n, int n_tasks, const void* tasks, int n_warps_total, const int* wptr,
                         long long n_coef, const double* coef, const double* r, double* z_out,
                         int grid, int reps, double* ms_out, unsigned long long* trace_out,
                         int nc, const int* total, const int* quota) {
  Task* dT;
  int *dW, *dtot, *dq;
  unsigned* dcnt;
  double *dc, *dv;
  cudaMalloc(&dT, sizeof(Task) * n_tasks);
  cudaMalloc(&dW, sizeof(int) * (n_warps_total + 1));
  cudaMalloc(&dc, sizeof(double) * n_coef);
  cudaMalloc(&dtot, sizeof(int) * nc);
  cudaMalloc(&dq, sizeof(int) * nc * grid);
  cudaMalloc(&dcnt, sizeof(unsigned) * nc * (reps + 2));
  cudaMemset(dcnt, 0, sizeof(unsigned) * nc * (reps + 2));
  const size_t per = 5ull * n;
  cudaMalloc(&dv, sizeof(double) * per * (reps + 2));
  cudaMemcpy(dT, tasks, sizeof(Task) * n_tasks, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, wptr, sizeof(int) * (n_warps_total + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dc, coef, sizeof(double) * n_coef, cudaMemcpyHostToDevice);
  cudaMemcpy(dtot, total, sizeof(int) * nc, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, quota, sizeof(int) * nc * grid, cudaMemcpyHostToDevice);
  fill_sent<<<148, 512>>>(dv, per * (reps + 2));
  for (int k = 0; k < reps + 2; ++k) cudaMemcpy(dv + per * k, r, sizeof(double) * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chain_kernel<<<grid, 512>>>(dT, dW, dc, dv + per * reps, n, nullptr, dcnt + nc * reps, dtot, dq, nc);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int k = 0; k < reps; ++k)
    chain_kernel<<<grid, 512>>>(dT, dW, dc, dv + per * k, n, nullptr, dcnt + nc * k, dtot, dq, nc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / reps;
  cudaMemcpy(z_out, dv + 4ull * n, sizeof(double) * n, cudaMemcpyDeviceToHost);
  if (trace_out) {
    unsigned long long* dtr;
    cudaMalloc(&dtr, 24ull * n_tasks);
    chain_kernel<<<grid, 512>>>(dT, dW, dc, dv + per * (reps + 1), n, dtr, dcnt + nc * (reps + 1), dtot, dq, nc);
    cudaMemcpy(trace_out, dtr, 24ull * n_tasks, cudaMemcpyDeviceToHost);
    cudaFree(dtr);
  }
  const cudaError_t err = cudaDeviceSynchronize();
  cudaFree(dT); cudaFree(dW); cudaFree(dc); cudaFree(dv); cudaFree(dtot); cudaFree(dq); cudaFree(dcnt);
  if (err != cudaSuccess) {
    fprintf(stderr, "cuda: %s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
