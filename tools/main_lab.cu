// Lab: the blocked sweep's main-warp step in isolation (one warp of a 512-thread
// CTA, everything it reads resident in shared memory, every flag always ready).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o main_lab tools/main_lab.cu && ./main_lab
// Variants: V0 the production step (F_1, F_2 from a slot ring, c / q / flags
// loaded, y through the shared ring), V1 without the flag / c / q loads, V2 F
// blocks kept in registers (no slot loads), V3 only the dependent chain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kSteps = 20000, kNs = 8, kSlot = 5 * 2048, kRing = 32;

__device__ __forceinline__ double shfl_xor16(double v) { return __shfl_xor_sync(0xffffffffu, v, 16); }

template <int V>
__global__ void __launch_bounds__(512, 1) lab(double* out, long long* cyc, int busy_warps, const uint8_t* gsrc) {
  extern __shared__ __align__(128) uint8_t smem[];
  double* ring = reinterpret_cast<double*>(smem);               // 32 groups x 16 + zero slot
  uint8_t* slots = smem + 4352;                                 // kNs x kSlot
  volatile int* flags = reinterpret_cast<volatile int*>(slots + kNs * kSlot);  // 64 ints
  double* cbuf = reinterpret_cast<double*>(slots + kNs * kSlot + 256);         // 16 x 16
  double* qbuf = cbuf + 256;                                                  // 8 x 32
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane & 15, hf = lane >> 4;
  for (int i = threadIdx.x; i < (4352 + kNs * kSlot + 256 + 2048 + 2048) / 8; i += blockDim.x)
    reinterpret_cast<double*>(smem)[i] = 1e-3 * ((i * 37) % 101 - 50);
  __syncthreads();
  if (warp == 15) {
    uint8_t* const ringb = smem;
    auto ld_block = [&](const uint8_t* slot, int block, double* o) {
      const double2* p = reinterpret_cast<const double2*>(slot + block * 2048) + lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 t = p[q * 32];
        o[2 * q] = t.x;
        o[2 * q + 1] = t.y;
      }
    };
    double f1[8], f2[8], f1b[8], f2b[8];
    ld_block(slots, 0, f1);
    ld_block(slots + kSlot, 1, f2);
    double c = cbuf[r], q2 = 0.0, Q0 = 0.0;
    int yoff = (kRing - 1) * 128 + hf * 64, woff = r * 8, s1 = 0, s2 = 1, s3 = 2;
    int sink = 0;
    auto step = [&](int g, const double (&fa)[8], const double (&fb)[8], double (&na)[8], double (&nb)[8]) {
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
      const int gn = g + 1;
      if (V <= 1) {
        s1 = s2;
        s2 = s3;
        s3 = s3 + 1 == kNs ? 0 : s3 + 1;
        ld_block(slots + s1 * kSlot, 0, na);
        ld_block(slots + s2 * kSlot, 1, nb);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          na[i] = fa[i];
          nb[i] = fb[i];
        }
      }
      int fa_ = 0, fq_ = 0, fs_ = 0;
      if (V == 0) {
        fa_ = flags[gn & 15];
        fq_ = flags[16 + (gn & 7)];
        fs_ = flags[32 + s3];
      }
      double t = (pa + pb) + (Q0 + q2);
      t += shfl_xor16(t);
      const double y = c - t;
      if (hf == 0) *reinterpret_cast<double*>(ringb + woff) = y * 1e-3;
      Q0 = ua + ub;
      __syncwarp();
      if (V <= 2 && lane == 0) flags[48] = gn;
      yoff = woff - r * 8 + hf * 64;
      woff = woff + 128 == kRing * 128 + r * 8 ? r * 8 : woff + 128;
      if (V == 0) {
        sink += fa_ + fq_ + fs_;
        c = cbuf[(gn & 15) * 16 + r];
        q2 = qbuf[(gn & 7) * 32 + lane];
      }
    };
    const long long t0 = clock64();
    for (int g = 0; g < kSteps; g += 2) {
      step(g, f1, f2, f1b, f2b);
      step(g + 1, f1b, f2b, f1, f2);
    }
    const long long t1 = clock64();
    if (lane == 0) cyc[V] = t1 - t0;
    out[lane] = c + q2 + Q0 + sink + f1[0];
  } else if (busy_warps < 100 && warp < busy_warps) {
    // background shared-memory traffic on the other sub-partitions (gathers)
    double acc = 0.0;
    const double* ringd = reinterpret_cast<const double*>(smem);
    for (int i = 0; i < kSteps * 40; ++i) acc += ringd[(lane * 17 + i * 5 + warp) & 511];
    out[32 + threadIdx.x] = acc;
  } else if ((busy_warps == 101 || busy_warps == 110) && warp == 10) {
    // a second-main-like warp: 12 LDS.128 + 24 FMA per iteration, polling the progress word
    double acc = 0.0;
    for (int i = 0; i < kSteps; ++i) {
      while (flags[48] < i - 2 && flags[48] < kSteps - 4) {
      }
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double2* p = reinterpret_cast<const double2*>(slots + ((i + b) % kNs) * kSlot + (2 + b) * 2048) + lane;
        const double2 a0 = p[0], a1 = p[32], a2 = p[64], a3 = p[96];
        acc = fma(a0.x, a1.y, acc);
        acc = fma(a2.x, a3.y, acc);
      }
    }
    out[32 + threadIdx.x] = acc;
  } else if ((busy_warps == 102 || busy_warps == 110) && (warp == 13 || warp == 14) && lane == 0) {
    // pollers: producer / publisher style spinning on the progress word
    int v = 0, n = 0;
    while ((v = flags[48]) < kSteps - 4) {
      ++n;
      if (warp == 14) __nanosleep(200);
    }
    out[32 + threadIdx.x] = n;
  } else if ((busy_warps == 103 || busy_warps == 110) && warp == 12 && lane == 0) {
    // TMA producer: 10 KB bulk copies global -> the slot ring, back to back
    uint64_t* mbar = reinterpret_cast<uint64_t*>(const_cast<int*>(flags) + 56);
    const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned phase = 0;
    int i = 0;
    while (flags[48] < kSteps - 4) {
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(slots + ((i + 3) % kNs) * kSlot));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(kSlot) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(gsrc + (i % 64) * kSlot), "r"(kSlot), "r"(mb)
                   : "memory");
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(mb), "r"(phase)
                     : "memory");
      phase ^= 1;
      ++i;
    }
    out[32 + threadIdx.x] = i;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8192);
  cudaMallocManaged(&cyc, 64);
  const int smem = 4352 + kNs * kSlot + 256 + 2048 + 2048 + 128;
  cudaFuncSetAttribute(lab<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(lab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(lab<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(lab<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint8_t* gsrc;
  cudaMalloc(&gsrc, 64 * kSlot);
  cudaMemset(gsrc, 0, 64 * kSlot);
  for (int busy : {0, 4, 10, 101, 102, 103, 110}) {
    for (int rep = 0; rep < 2; ++rep) {
      lab<0><<<1, 512, smem>>>(out, cyc, busy, gsrc);
      lab<1><<<1, 512, smem>>>(out, cyc, busy, gsrc);
      lab<2><<<1, 512, smem>>>(out, cyc, busy, gsrc);
      lab<3><<<1, 512, smem>>>(out, cyc, busy, gsrc);
      cudaDeviceSynchronize();
    }
    printf("background %3d (101 second-main-like, 102 pollers, 103 TMA producer, 110 all three): cycles/step  V0 production %.1f | V1 no flag/c/q loads %.1f | V2 F in registers %.1f | V3 chain only %.1f\n",
           busy, double(cyc[0]) / kSteps, double(cyc[1]) / kSteps, double(cyc[2]) / kSteps, double(cyc[3]) / kSteps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
