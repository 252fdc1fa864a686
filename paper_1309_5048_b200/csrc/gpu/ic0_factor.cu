// IC(0) factorization on the device, bit-identical
// to the reference's ic0 (proj/src/cholesky.cpp:84-134). Two schedules of the
// same per-row work: a barrier-free dataflow kernel (default, below) and
// level-scheduled launches (DSGPU_IC0_FLOW=0).
//
// The reference walks rows in order; inside row i, entry (i, j) is
//   s = A_ij - sum_{c < j, c in row i and row j} L_ic L_jc   (merge order = c ascending)
//   L_ij = s / L_jj
// and the diagonal is sqrt(A_ii - sum_k L_ik^2) (FactorBreakdown when not > 0).
// Row i reads only rows j < i of its own pattern, so rows of one level of
// L's dependency DAG are independent: one launch per level, one warp per row.
// Within a row the entries stay sequential (entry ku uses the finished
// entries before it) and every subtraction is applied in the reference's
// order with explicitly rounded mul / sub / div / sqrt (no FMA), so the result
// is the reference's factor bit for bit. The 32 lanes parallelize the merge:
// each lane takes one entry of row j and finds its column's position in row i
// through a per-warp column -> position map in global memory (n ints per row
// of the widest level, set at the row's start, cleared at its end); the
// matched products are compacted into shared memory and subtracted in column
// order by one sequential chain.
// Row j's entries and their map lookups do not depend on row i's results, so
// the next two entries' are loaded while the current one is reduced.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/dsgpu.h"

namespace {

thread_local std::string g_ic0_err;

constexpr int kWarpsPerBlock = 4;

// Row j's entries (without its diagonal) of one pass: U chunks of 32, the
// column's position in row i (pos map), the value. Prefetched one entry ahead.
struct RowChunk {
  static constexpr int U = 8;
  int col[U], pos[U];
  double val[U];
};

__device__ __forceinline__ void load_chunk(RowChunk& r, const int32_t* __restrict__ ci, const double* v,
                                           const int* __restrict__ pos, int64_t b, int64_t e, int pmax, int lane) {
#pragma unroll
  for (int u = 0; u < RowChunk::U; ++u) {
    const int64_t q = b + u * 32 + lane;
    r.col[u] = q < e ? __ldg(ci + q) : -1;
    r.val[u] = q < e ? v[q] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < RowChunk::U; ++u)
    r.pos[u] = (r.col[u] >= 0 && r.col[u] <= pmax) ? pos[r.col[u]] : -1;
}

// s - p[0] - p[1] - ... in order; the loads are batched ahead of the
// dependent subtractions.
__device__ __forceinline__ double sub_chain(double s, const double* p, int cnt) {
  int k = 0;
  for (; k + 8 <= cnt; k += 8) {
    double b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) b[q] = p[k + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dsub_rn(s, b[q]);
  }
  for (; k < cnt; ++k) s = __dsub_rn(s, p[k]);
  return s;
}

// s -= the matched products of one pass, in column (= chunk, then lane)
// order: the hits are compacted into the warp's shared buffer (ballot + popc
// rank), then every lane runs the same sequential subtraction chain from it
// (loads independent of s, one dependent fp64 subtract per product).
// Returns true when the pass reached past row i's prefix (nothing more can match).
__device__ __forceinline__ bool apply_chunk(const RowChunk& r, const double* sval, int t, int pmax, double& s,
                                            double* buf, int lane) {
  int cnt = 0;
  bool done = false;
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < RowChunk::U; ++u) {
    const bool hit = r.pos[u] >= 0 && r.pos[u] < t;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) buf[cnt + __popc(m & below)] = __dmul_rn(sval[r.pos[u]], r.val[u]);
    cnt += __popc(m);
    const int last = __shfl_sync(0xffffffffu, r.col[u], 31);
    if (last < 0 || last >= pmax) {
      done = true;
      break;
    }
  }
  __syncwarp();
  s = sub_chain(s, buf, cnt);
  __syncwarp();  // buf is reused by the next pass
  return done;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    ic0_level_kernel(const int32_t* __restrict__ rows, int nrows, const int64_t* __restrict__ rp,
                     const int32_t* __restrict__ ci, double* v, int maxlen, int* pos_maps, int64_t map_len,
                     int* bad) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int w = blockIdx.x * kWarpsPerBlock + wl;
  if (w >= nrows) return;
  int32_t* scol = reinterpret_cast<int32_t*>(smem) + static_cast<size_t>(wl) * maxlen;
  double* sval = reinterpret_cast<double*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 4 +
                                           static_cast<size_t>(wl) * maxlen * 8);
  // per entry of row i: row j's range and its final diagonal L_jj
  int64_t* sjb = reinterpret_cast<int64_t*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 12) +
                 static_cast<size_t>(wl) * maxlen * 3;
  int64_t* sje = sjb + maxlen;
  double* sdg = reinterpret_cast<double*>(sje + maxlen);
  double* buf = reinterpret_cast<double*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 36) +
                static_cast<size_t>(wl) * RowChunk::U * 32;
  int* pos = pos_maps + static_cast<int64_t>(w) * map_len;  // this warp's column -> position map (all -1)
  const int i = rows[w];
  const int64_t ib = rp[i], ie = rp[i + 1];
  const int len = static_cast<int>(ie - ib);
  for (int k = lane; k < len; k += 32) {
    const int c = ci[ib + k];
    scol[k] = c;
    sval[k] = v[ib + k];
    if (k < len - 1) {
      pos[c] = k;
      const int64_t b = rp[c], e = rp[c + 1] - 1;
      sjb[k] = b;
      sje[k] = e;
      sdg[k] = v[e];  // row c is at an earlier level: final
    }
  }
  __syncwarp();
  const int pfull = len >= 2 ? scol[len - 2] : -1;  // largest off-diagonal column of row i
  RowChunk cur, nxt, nx2;  // entries t, t+1, t+2 (two-deep prefetch of static data)
  if (len >= 2) load_chunk(cur, ci, v, pos, sjb[0], sje[0], pfull, lane);
  if (len >= 3) load_chunk(nxt, ci, v, pos, sjb[1], sje[1], pfull, lane);
  for (int t = 0; t < len - 1; ++t) {  // entry ku = ib + t, column j < i
    const int64_t jb = sjb[t], je = sje[t];  // row j = scol[t] without its diagonal
    if (t + 2 < len - 1) load_chunk(nx2, ci, v, pos, sjb[t + 2], sje[t + 2], pfull, lane);
    double s = sval[t];
    const int pmax = t > 0 ? scol[t - 1] : -1;  // largest column of row i's finished prefix
    if (t > 0 && !apply_chunk(cur, sval, t, pmax, s, buf, lane)) {
      // rows longer than one pass: the rest, synchronously
      for (int64_t b = jb + RowChunk::U * 32; b < je; b += RowChunk::U * 32) {
        RowChunk more;
        load_chunk(more, ci, v, pos, b, je, pfull, lane);
        if (apply_chunk(more, sval, t, pmax, s, buf, lane)) break;
      }
    }
    const double lij = __ddiv_rn(s, sdg[t]);  // L_jj is final (earlier level)
    if (lane == 0) {
      sval[t] = lij;
      v[ib + t] = lij;
    }
    __syncwarp();
    cur = nxt;
    nxt = nx2;
  }
  for (int k = lane; k < len - 1; k += 32) sjb[k] = __double_as_longlong(__dmul_rn(sval[k], sval[k]));
  __syncwarp();
  const double d = sub_chain(sval[len - 1], reinterpret_cast<const double*>(sjb), len - 1);
  for (int k = lane; k < len - 1; k += 32) pos[scol[k]] = -1;  // leave the map clean
  if (lane == 0) {
    if (!(d > 0.0)) atomicMin(bad, i);
    v[ie - 1] = __dsqrt_rn(d);
  }
}

// ---- dataflow variant: no level barriers ----------------------------------
// A persistent grid of warps walks the rows in order (warp w: rows w, w + W,
// ...). Entry (i, j) waits only for row j's completion flag (st.release by
// the warp that finished it, ld.acquire here), so a row processes its entries
// on old rows at once and stalls only on its most recent dependencies. All
// warps are co-resident and each walks its rows in increasing order, so the
// smallest unfinished row can always progress.
__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int x;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
  return x;
}
__device__ __forceinline__ void st_release_i32(int* p, int x) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

__device__ __forceinline__ void load_chunk_cg(RowChunk& r, const int32_t* __restrict__ ci, const double* v,
                                              const int* __restrict__ pos, int64_t b, int64_t e, int pmax,
                                              int lane) {
#pragma unroll
  for (int u = 0; u < RowChunk::U; ++u) {
    const int64_t q = b + u * 32 + lane;
    r.col[u] = q < e ? __ldg(ci + q) : -1;
    r.val[u] = q < e ? __ldcg(v + q) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < RowChunk::U; ++u)
    r.pos[u] = (r.col[u] >= 0 && r.col[u] <= pmax) ? pos[r.col[u]] : -1;
}

// spin until row j is final; false on timeout (abort flag set)
__device__ __forceinline__ bool wait_row(const int* done, int j, int* abort_flag) {
  if (ld_acquire_i32(done + j)) return true;
  const long long t0 = clock64();
  while (!ld_acquire_i32(done + j)) {
    __nanosleep(32);
    if (*reinterpret_cast<volatile int*>(abort_flag)) return false;
    if (clock64() - t0 > 20000000000ll) {  // ~10 s: report instead of hanging the GPU
      atomicExch(abort_flag, 1);
      return false;
    }
  }
  return true;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    ic0_flow_kernel(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, double* v, int maxlen,
                    int* pos_maps, int* done, int* bad, int* abort_flag) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int w = blockIdx.x * kWarpsPerBlock + wl, W = gridDim.x * kWarpsPerBlock;
  int32_t* scol = reinterpret_cast<int32_t*>(smem) + static_cast<size_t>(wl) * maxlen;
  double* sval = reinterpret_cast<double*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 4 +
                                           static_cast<size_t>(wl) * maxlen * 8);
  int64_t* sjb = reinterpret_cast<int64_t*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 12) +
                 static_cast<size_t>(wl) * maxlen * 3;
  int64_t* sje = sjb + maxlen;
  double* buf = reinterpret_cast<double*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 36) +
                static_cast<size_t>(wl) * RowChunk::U * 32;
  int* pos = pos_maps + static_cast<int64_t>(w) * n;
  for (int i = w; i < n; i += W) {
    const int64_t ib = rp[i], ie = rp[i + 1];
    const int len = static_cast<int>(ie - ib);
    for (int k = lane; k < len; k += 32) {
      const int c = ci[ib + k];
      scol[k] = c;
      sval[k] = v[ib + k];  // A's values: only this warp writes row i
      if (k < len - 1) {
        pos[c] = k;
        sjb[k] = rp[c];
        sje[k] = rp[c + 1] - 1;
      }
    }
    __syncwarp();
    const int pfull = len >= 2 ? scol[len - 2] : -1;
    bool ok = true;
    RowChunk cur, nxt;
    bool cur_ok = false, nxt_ok = false;  // chunk loaded after its row was seen final
    if (len >= 2 && ld_acquire_i32(done + scol[0])) {
      load_chunk_cg(cur, ci, v, pos, sjb[0], sje[0], pfull, lane);
      cur_ok = true;
    }
    for (int t = 0; t < len - 1; ++t) {
      const int j = scol[t];
      if (t + 1 < len - 1) {
        nxt_ok = ld_acquire_i32(done + scol[t + 1]) != 0;
        if (nxt_ok) load_chunk_cg(nxt, ci, v, pos, sjb[t + 1], sje[t + 1], pfull, lane);
      }
      ok = ok && wait_row(done, j, abort_flag);
      if (!cur_ok) load_chunk_cg(cur, ci, v, pos, sjb[t], sje[t], pfull, lane);
      const int64_t jb = sjb[t], je = sje[t];
      double s = sval[t];
      const int pmax = t > 0 ? scol[t - 1] : -1;
      if (t > 0 && !apply_chunk(cur, sval, t, pmax, s, buf, lane)) {
        for (int64_t b = jb + RowChunk::U * 32; b < je; b += RowChunk::U * 32) {
          RowChunk more;
          load_chunk_cg(more, ci, v, pos, b, je, pfull, lane);
          if (apply_chunk(more, sval, t, pmax, s, buf, lane)) break;
        }
      }
      const double lij = __ddiv_rn(s, __ldcg(v + je));  // L_jj: row j is final
      if (lane == 0) {
        sval[t] = lij;
        v[ib + t] = lij;
      }
      __syncwarp();
      cur = nxt;
      cur_ok = nxt_ok;
    }
    for (int k = lane; k < len - 1; k += 32) sjb[k] = __double_as_longlong(__dmul_rn(sval[k], sval[k]));
    __syncwarp();
    const double d = sub_chain(sval[len - 1], reinterpret_cast<const double*>(sjb), len - 1);
    for (int k = lane; k < len - 1; k += 32) pos[scol[k]] = -1;
    if (lane == 0) {
      if (!(d > 0.0) || !ok) atomicMin(bad, i);
      v[ie - 1] = __dsqrt_rn(d);
      __threadfence();
      st_release_i32(done + i, 1);
    }
    __syncwarp();
  }
}

int fail(int code, const std::string& msg) {
  g_ic0_err = msg;
  return code;
}

}  // namespace

extern "C" {

const char* dsgpu_ic0_last_error(void) { return g_ic0_err.c_str(); }

int dsgpu_ic0_factor(int device, int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                     int64_t* l_row_ptr, int32_t* l_cols, double* l_vals, int* bad_row, int* n_levels,
                     double* device_ms) {
  if (bad_row) *bad_row = -1;
  if (n < 0 || !row_ptr || (n > 0 && (!cols || !vals || !l_row_ptr || !l_cols || !l_vals)))
    return fail(DSGPU_E_BAD_INPUT, "ic0: bad arguments");
  // lower pattern incl. the diagonal, values of A (cholesky.cpp:88-105)
  l_row_ptr[0] = 0;
  for (int i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) c += cols[k] <= i;
    l_row_ptr[i + 1] = l_row_ptr[i] + c;
  }
  {
    int64_t pos = 0;
    for (int i = 0; i < n; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
        if (cols[k] <= i) {
          l_cols[pos] = cols[k];
          l_vals[pos] = vals[k];
          ++pos;
        }
  }
  // structural checks (cholesky.cpp:109-111) and dependency levels
  std::vector<int32_t> level(n, 0);
  int maxlen = 1, nlev = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t b = l_row_ptr[i], e = l_row_ptr[i + 1];
    if (e == b || l_cols[e - 1] != i)
      return fail(DSGPU_E_BAD_INPUT, "ic0: structurally missing diagonal at row " + std::to_string(i));
    int lv = 0;
    for (int64_t k = b; k < e - 1; ++k) {
      if (l_cols[k] < 0 || l_cols[k] >= i)
        return fail(DSGPU_E_BAD_INPUT, "ic0: row " + std::to_string(i) + " has a column outside [0, row)");
      lv = std::max(lv, level[l_cols[k]] + 1);
    }
    level[i] = lv;
    nlev = std::max(nlev, lv + 1);
    maxlen = std::max(maxlen, static_cast<int>(e - b));
  }
  if (n_levels) *n_levels = nlev;
  if (n == 0) return DSGPU_OK;
  std::vector<int64_t> lstart(nlev + 1, 0);
  for (int i = 0; i < n; ++i) ++lstart[level[i] + 1];
  for (int l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
  int maxw = 1;  // widest level: one column-position map (n ints) per row of it
  for (int l = 0; l < nlev; ++l) maxw = std::max(maxw, static_cast<int>(lstart[l + 1] - lstart[l]));
  // dataflow grid: up to 2,368 warps (whole CTAs), maps capped at 8 GB;
  // DSGPU_IC0_MAX_WARPS lowers the cap (tests)
  int64_t cap_w = std::min<int64_t>(2368, (8ll << 30) / (4ll * std::max(n, 1)));
  if (const char* env = std::getenv("DSGPU_IC0_MAX_WARPS")) cap_w = std::min<int64_t>(cap_w, std::atoll(env));
  const int maxw_flow = static_cast<int>(std::max<int64_t>(kWarpsPerBlock, cap_w / kWarpsPerBlock * kWarpsPerBlock));
  // the barrier-free dataflow kernel by default; DSGPU_IC0_FLOW=0: level-scheduled launches.
  // Column-position maps: one per warp of the dataflow grid, or one per row of the
  // widest level for the level schedule -- never both (the widest level of a large
  // 3D block would ask for tens of GB the dataflow kernel never touches).
  const bool flow = !(std::getenv("DSGPU_IC0_FLOW") && std::atoi(std::getenv("DSGPU_IC0_FLOW")) == 0);
  maxw = flow ? maxw_flow : maxw;
  std::vector<int32_t> order(n);
  {
    std::vector<int64_t> fill(lstart.begin(), lstart.end() - 1);
    for (int i = 0; i < n; ++i) order[fill[level[i]]++] = i;
  }
  // 4-byte columns and 8-byte values of maxlen entries per warp: keep the
  // product buffers behind them 8-byte aligned
  maxlen = (maxlen + 1) / 2 * 2;
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * (maxlen * 36 + RowChunk::U * 32 * 8);
  if (cudaSetDevice(device) != cudaSuccess) return fail(DSGPU_E_CUDA, "ic0: cudaSetDevice failed");
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (smem > static_cast<size_t>(optin)) return fail(DSGPU_E_UNSUPPORTED, "ic0: row too long for this build");
  if (cudaFuncSetAttribute(ic0_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
      cudaSuccess)
    return fail(DSGPU_E_CUDA, "ic0: cudaFuncSetAttribute failed");
  const int64_t nnz = l_row_ptr[n];
  int64_t* d_rp = nullptr;
  int32_t *d_ci = nullptr, *d_rows = nullptr;
  double* d_v = nullptr;
  int* d_bad = nullptr;
  int* d_pos = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaFree(d_rows);
    cudaFree(d_v);
    cudaFree(d_bad);
    cudaFree(d_pos);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  };
  const int big = 0x7fffffff;
  if (cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1)) != cudaSuccess ||
      cudaMalloc(&d_ci, sizeof(int32_t) * nnz) != cudaSuccess ||
      cudaMalloc(&d_rows, sizeof(int32_t) * n) != cudaSuccess || cudaMalloc(&d_v, sizeof(double) * nnz) != cudaSuccess ||
      cudaMalloc(&d_bad, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&d_pos, sizeof(int) * static_cast<size_t>(maxw) * n) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cleanup();
    return fail(DSGPU_E_CUDA, "ic0: device allocation failed");
  }
  cudaMemcpyAsync(d_rp, l_row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_ci, l_cols, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_v, l_vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_rows, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d_pos, 0xFF, sizeof(int) * static_cast<size_t>(maxw) * n, st);  // all -1
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int flow_grid = 0;
  int* d_done = nullptr;
  int* d_abort = nullptr;
  if (flow) {
    int per_sm = 0, sms = 0;
    cudaFuncSetAttribute(ic0_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ic0_flow_kernel, kWarpsPerBlock * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    flow_grid = std::max(1, std::min(per_sm * sms, maxw_flow / kWarpsPerBlock));  // W <= maps allocated
    if (cudaMalloc(&d_done, sizeof(int) * n) != cudaSuccess || cudaMalloc(&d_abort, sizeof(int)) != cudaSuccess) {
      cudaFree(d_done);
      cudaFree(d_abort);
      cleanup();
      return fail(DSGPU_E_CUDA, "ic0: device allocation failed");
    }
    cudaMemsetAsync(d_done, 0, sizeof(int) * n, st);
    cudaMemsetAsync(d_abort, 0, sizeof(int), st);
  }
  cudaEventRecord(e0, st);
  cudaError_t le = cudaSuccess;
  if (flow) {
    // its warps wait on one another's rows: a cooperative launch (every CTA co-resident)
    int n_arg = n, maxlen_arg = maxlen;
    void* params[] = {&n_arg, &d_rp, &d_ci, &d_v, &maxlen_arg, &d_pos, &d_done, &d_bad, &d_abort};
    le = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ic0_flow_kernel), dim3(flow_grid),
                                     dim3(kWarpsPerBlock * 32), params, smem, st);
  }
  for (int l = 0; !flow && l < nlev; ++l) {
    const int cnt = static_cast<int>(lstart[l + 1] - lstart[l]);
    const int grid = (cnt + kWarpsPerBlock - 1) / kWarpsPerBlock;
    ic0_level_kernel<<<grid, kWarpsPerBlock * 32, smem, st>>>(d_rows + lstart[l], cnt, d_rp, d_ci, d_v, maxlen,
                                                              d_pos, static_cast<int64_t>(n), d_bad);
  }
  cudaEventRecord(e1, st);
  int bad = big, aborted = 0;
  if (flow) cudaMemcpyAsync(&aborted, d_abort, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(l_vals, d_v, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (le != cudaSuccess) e = le;
  float ms = 0.0f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(d_done);
  cudaFree(d_abort);
  cleanup();
  if (e != cudaSuccess) return fail(DSGPU_E_CUDA, std::string("ic0: ") + cudaGetErrorString(e));
  if (aborted) return fail(DSGPU_E_CUDA, "ic0: dataflow wait timed out");
  if (device_ms) *device_ms = ms;
  if (bad != big) {
    if (bad_row) *bad_row = bad;
    return fail(DSGPU_E_FACTOR_BREAKDOWN, "factorization breakdown: nonpositive pivot at row " + std::to_string(bad));
  }
  return DSGPU_OK;
}

}  // extern "C"
