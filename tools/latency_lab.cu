// Lab: cross-SM hand-off latency on B200 (ping-pong through global memory)
// and __nanosleep granularity. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_lab latency_lab.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// CTA 0 and CTA `peer` ping-pong `iters` times; sleep_ns in the poll loop
__global__ void pingpong(unsigned long long* buf, int iters, int sleep_ns, int peer, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  if (blockIdx.x != 0 && blockIdx.x != peer) return;
  const bool a = blockIdx.x == 0;
  unsigned long long* mine = buf + (a ? 0 : 32);
  unsigned long long* theirs = buf + (a ? 32 : 0);
  const long long c0 = clock64();
  const unsigned long long t0 = gtime();
  for (int k = 1; k <= iters; ++k) {
    if (a) {
      st_relaxed(theirs, k);
      while (ld_relaxed(mine) != (unsigned long long)k)
        if (sleep_ns) __nanosleep(sleep_ns);
    } else {
      while (ld_relaxed(mine) != (unsigned long long)k)
        if (sleep_ns) __nanosleep(sleep_ns);
      st_relaxed(theirs, k);
    }
  }
  if (a) {
    out[0] = gtime() - t0;
    out[1] = clock64() - c0;
  }
}

__global__ void sleeper(int ns, int iters, unsigned long long* out) {
  const unsigned long long t0 = gtime();
  for (int k = 0; k < iters; ++k) __nanosleep(ns);
  if (threadIdx.x == 0) out[0] = gtime() - t0;
}

// load latency: dependent chain of global loads (L2 hits)
__global__ void chase(const unsigned* p, int iters, unsigned long long* out) {
  unsigned j = 0;
  const long long c0 = clock64();
  for (int k = 0; k < iters; ++k) j = __ldcg(p + j);
  out[0] = clock64() - c0;
  out[1] = j;
}

int main() {
  unsigned long long *buf, *out;
  cudaMalloc(&buf, 4096);
  cudaMalloc(&out, 64);
  unsigned long long h[2];
  const int iters = 2000;
  for (int peer : {1, 2, 74, 147}) {
    for (int s : {0, 32, 100}) {
      cudaMemset(buf, 0, 4096);
      pingpong<<<148, 32>>>(buf, iters, s, peer, out);
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("pingpong peer CTA %3d sleep %3d ns: round trip %.0f ns (%.0f cycles)\n", peer, s,
             (double)h[0] / iters, (double)h[1] / iters);
    }
  }
  for (int s : {0, 16, 32, 64, 100, 200, 500, 1000}) {
    sleeper<<<1, 32>>>(s, 1000, out);
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("nanosleep(%d): %.0f ns each\n", s, (double)h[0] / 1000);
  }
  unsigned* p;
  const int n = 1 << 20;
  cudaMalloc(&p, n * 4);
  unsigned* hp = new unsigned[n];
  for (int i = 0; i < n; ++i) hp[i] = (i * 7919u + 104729u) % n;
  cudaMemcpy(p, hp, n * 4, cudaMemcpyHostToDevice);
  chase<<<1, 1>>>(p, 1000, out);
  chase<<<1, 1>>>(p, 10000, out);
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("L2 dependent load latency: %.0f cycles\n", (double)h[0] / 10000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
