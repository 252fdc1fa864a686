// Lab: the hardware numbers the blocked IC(0) sweep is designed around (B200).
//   1. how many bytes per cycle ONE SM can pull from L2 / HBM (LDG.128 stream,
//      and TMA bulk copies into a shared-memory ring), alone and with peers;
//   2. fp64 FMA dependent latency, LDS latency, same-warp STS -> LDS round
//      trip, 64-bit shuffle latency;
//   3. cross-SM publish -> observe latency (st + fence + flag / acquire poll).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bs_lab bs_lab.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---- 1a. LDG stream: each CTA reads its own `bytes` region `reps` times ----
__global__ void __launch_bounds__(512, 1) ldg_stream(const int4* src, size_t bytes_per_cta, int reps,
                                                      unsigned long long* out) {
  const int4* p = src + static_cast<size_t>(blockIdx.x) * (bytes_per_cta / 16);
  const size_t n = bytes_per_cta / 16;
  int4 acc = make_int4(0, 0, 0, 0);
  __syncthreads();
  const long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (size_t i = threadIdx.x; i + 3 * blockDim.x < n; i += 4 * blockDim.x) {
      const int4 a = __ldcg(p + i), b = __ldcg(p + i + blockDim.x), c = __ldcg(p + i + 2 * blockDim.x),
                 d = __ldcg(p + i + 3 * blockDim.x);
      acc.x ^= a.x ^ b.x ^ c.x ^ d.x;
      acc.y ^= a.y ^ b.y ^ c.y ^ d.y;
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
  if (acc.x == 0x12345 && acc.y == 0x777) out[1000] = 1;
}

// ---- 1b. TMA bulk stream into a ring of `NS` slots of `slot` bytes ---------
__global__ void __launch_bounds__(64, 1) tma_stream(const uint8_t* src, size_t bytes_per_cta, int slot, int NS,
                                                     unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm);
  uint8_t* ring = sm + 1024;
  const uint8_t* p = src + static_cast<size_t>(blockIdx.x) * bytes_per_cta;
  const int n = static_cast<int>(bytes_per_cta / slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar + i)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const long long c0 = clock64();
  if (threadIdx.x == 0) {
    int issued = 0, done = 0;
    while (done < n) {
      if (issued < n && issued - done < NS) {
        const int sl = issued % NS;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar + sl)),
                     "r"(slot)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(ring + static_cast<size_t>(sl) * slot)),
            "l"(p + static_cast<size_t>(issued) * slot), "r"(slot), "r"(smem_u32(mbar + sl))
            : "memory");
        ++issued;
      }
      if (done < issued && (issued == n || issued - done == NS)) {
        const int sl = done % NS;
        unsigned ok;
        asm volatile(
            "{ .reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
            : "=r"(ok)
            : "r"(smem_u32(mbar + sl)), "r"((done / NS) & 1)
            : "memory");
        if (ok) ++done;
      }
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
}

// ---- 2. latencies ---------------------------------------------------------
__global__ void lat(unsigned long long* out, double seed) {
  __shared__ double sh[64];
  __shared__ int idx[64];
  const int lane = threadIdx.x;
  sh[lane] = seed + lane;
  sh[lane + 32] = seed;
  idx[lane] = (lane + 1) & 31;
  __syncwarp();
  const int N = 4096;
  // DFMA dependent chain
  double a = seed, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0);
  // DADD dependent chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, c);
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0);
  // LDS dependent chain (pointer chase in shared)
  int j = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) j = *reinterpret_cast<volatile int*>(&idx[j]);
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0);
  // same-warp STS -> syncwarp -> LDS round trip (value dependent)
  double v = a;
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) {
    *reinterpret_cast<volatile double*>(&sh[lane]) = v;
    __syncwarp();
    v = *reinterpret_cast<volatile double*>(&sh[(lane + 1) & 31]);
    __syncwarp();
  }
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0);
  // 64-bit shuffle dependent chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 16);
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0);
  // DFMA throughput: 8 independent chains
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) {
    x0 = fma(x0, b, c);
    x1 = fma(x1, b, c);
    x2 = fma(x2, b, c);
    x3 = fma(x3, b, c);
    x4 = fma(x4, b, c);
    x5 = fma(x5, b, c);
    x6 = fma(x6, b, c);
    x7 = fma(x7, b, c);
  }
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0);
  if (a + v + j + x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[20] = 1;
  if (lane == 0) out[6] = N;
}

// ---- 3. publish -> observe: CTA 0 stores 16 doubles + fence + release flag;
// CTA `peer` polls with ld.acquire and reads the data; it answers through its
// own flag. Round trip / 2 = one publish hop.
// MODE 0: every lane fences (__threadfence), syncwarp, release flag.
// MODE 1: syncwarp, then lane 0's st.release alone (cumulative release).
// MODE 2: no flag: each double travels as two 8-byte {half, tag} words
//         (LL-style, self-validating); the consumer polls the data itself.
template <int MODE>
__global__ void hop(double* data, unsigned* flags, int iters, int peer, unsigned long long* out) {
  if (blockIdx.x != 0 && blockIdx.x != peer) return;
  const bool a = blockIdx.x == 0;
  const int lane = threadIdx.x;
  unsigned* mine = flags + (a ? 0 : 64);
  unsigned* theirs = flags + (a ? 64 : 0);
  double* dout = data + (a ? 0 : 128);
  const double* din = data + (a ? 128 : 0);
  double v = lane;
  const long long c0 = clock64();
  for (int k = 1; k <= iters; ++k) {
    auto send = [&]() {
      if (MODE == 2) {
        if (lane < 16) {
          const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
          uint4 w;
          w.x = static_cast<unsigned>(b);
          w.y = k;
          w.z = static_cast<unsigned>(b >> 32);
          w.w = k;
          __stcg(reinterpret_cast<uint4*>(dout) + lane, w);
        }
        return;
      }
      if (lane < 16) __stcg(dout + lane, v);
      if (MODE == 0) __threadfence();
      __syncwarp();
      if (lane == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(theirs), "r"(k) : "memory");
    };
    auto recv = [&]() {
      if (MODE == 2) {
        uint4 w;
        do {
          w = __ldcg(reinterpret_cast<const uint4*>(din) + (lane & 15));
        } while (w.y != static_cast<unsigned>(k) || w.w != static_cast<unsigned>(k));
        v = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(w.z) << 32) | w.x)) + 1.0;
        return;
      }
      unsigned f;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(mine) : "memory");
      } while (f != static_cast<unsigned>(k));
      v = __ldcg(din + (lane & 15)) + 1.0;
    };
    if (a) send();
    recv();
    if (!a) send();
  }
  if (a && lane == 0) {
    out[0] = clock64() - c0;
    out[1] = static_cast<unsigned long long>(v);
  }
}

int main(int argc, char** argv) {
  const bool only_lat = argc > 1;
  unsigned long long* out;
  CK(cudaMalloc(&out, 8192 * 8));
  std::vector<unsigned long long> h(2048);
  const size_t big = size_t(1) << 30;  // 1 GiB source
  uint8_t* src;
  CK(cudaMalloc(&src, big));
  CK(cudaMemset(src, 1, big));
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int ctas : {1, 2, 8, 32, 148}) {
    if (only_lat) break;
    for (size_t per : {size_t(4) << 20, size_t(1) << 20}) {  // 4 MiB (x reps) and L2-resident 1 MiB
      const int reps = per == (size_t(1) << 20) ? 16 : 4;
      ldg_stream<<<ctas, 512>>>(reinterpret_cast<const int4*>(src), per, 1, out);  // warm
      ldg_stream<<<ctas, 512>>>(reinterpret_cast<const int4*>(src), per, reps, out);
      CK(cudaMemcpy(h.data(), out, 8 * ctas, cudaMemcpyDeviceToHost));
      unsigned long long mx = 0;
      for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("LDG.128 stream   ctas %3d  %4zu KiB/CTA x%2d: %.1f B/clk/SM\n", ctas, per >> 10, reps,
             double(per) * reps / mx);
    }
    for (int slot : {8192, 16384}) {
      for (int NS : {4, 8}) {
        const size_t per = size_t(4) << 20;
        tma_stream<<<ctas, 64, 1024 + slot * NS>>>(src, per, slot, NS, out);
        tma_stream<<<ctas, 64, 1024 + slot * NS>>>(src, per, slot, NS, out);
        CK(cudaMemcpy(h.data(), out, 8 * ctas, cudaMemcpyDeviceToHost));
        unsigned long long mx = 0;
        for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("TMA bulk stream  ctas %3d  slot %5d ring %d (L2-warm 4 MiB/CTA): %.1f B/clk/SM\n", ctas, slot, NS,
               double(per) / mx);
      }
    }
  }
  if (!only_lat) {  // cold (HBM) single-CTA TMA: a fresh 64 MiB region
    tma_stream<<<1, 64, 1024 + 8192 * 8>>>(src + (size_t(512) << 20), size_t(64) << 20, 8192, 8, out);
    CK(cudaMemcpy(h.data(), out, 8, cudaMemcpyDeviceToHost));
    printf("TMA bulk stream  1 CTA 64 MiB cold (HBM): %.1f B/clk\n", double(size_t(64) << 20) / h[0]);
    ldg_stream<<<1, 512>>>(reinterpret_cast<const int4*>(src + (size_t(256) << 20)), size_t(64) << 20, 1, out);
    CK(cudaMemcpy(h.data(), out, 8, cudaMemcpyDeviceToHost));
    printf("LDG.128 stream   1 CTA 64 MiB cold (HBM): %.1f B/clk\n", double(size_t(64) << 20) / h[0]);
  }
  lat<<<1, 32>>>(out, 1.0);
  CK(cudaMemcpy(h.data(), out, 8 * 8, cudaMemcpyDeviceToHost));
  const double N = double(h[6]);
  printf("DFMA dependent %.1f cyc | DADD dependent %.1f | LDS chase %.1f | STS->syncwarp->LDS->syncwarp %.1f | "
         "shfl64 %.1f | DFMA x8 indep %.1f cyc per 8 (warp)\n",
         h[0] / N, h[1] / N, h[2] / N, h[3] / N, h[4] / N, h[5] / N);
  double* data;
  unsigned* flags;
  CK(cudaMalloc(&data, 8192));
  CK(cudaMalloc(&flags, 4096));
  for (int mode = 0; mode < 3; ++mode)
    for (int peer : {1, 74, 147}) {
      CK(cudaMemset(flags, 0, 4096));
      CK(cudaMemset(data, 0, 4096));
      if (mode == 0) hop<0><<<148, 32>>>(data, flags, 2000, peer, out);
      if (mode == 1) hop<1><<<148, 32>>>(data, flags, 2000, peer, out);
      if (mode == 2) hop<2><<<148, 32>>>(data, flags, 2000, peer, out);
      CK(cudaMemcpy(h.data(), out, 16, cudaMemcpyDeviceToHost));
      printf("publish hop mode %d (0: all-lane fence + release flag, 1: syncwarp + release flag, 2: {half,tag} words), "
             "peer CTA %3d: %.0f cycles one way\n", mode, peer, double(h[0]) / 2000 / 2);
    }
  CK(cudaDeviceSynchronize());
  printf("ok\n");
  return 0;
}
