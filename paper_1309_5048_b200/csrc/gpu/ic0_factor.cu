// IC(0) factorization on the device, bit-identical
// to the reference's ic0 (proj/src/cholesky.cpp:84-134).
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
// each lane takes one entry of row j and binary-searches its column among the
// finished entries of row i (staged in shared memory); the matched products
// are then subtracted in column order through warp shuffles.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/dsgpu.h"

namespace {

thread_local std::string g_ic0_err;

constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    ic0_level_kernel(const int32_t* __restrict__ rows, int nrows, const int64_t* __restrict__ rp,
                     const int32_t* __restrict__ ci, double* v, int maxlen, int* bad) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int w = blockIdx.x * kWarpsPerBlock + wl;
  if (w >= nrows) return;
  int32_t* scol = reinterpret_cast<int32_t*>(smem) + static_cast<size_t>(wl) * maxlen;
  double* sval = reinterpret_cast<double*>(smem + static_cast<size_t>(kWarpsPerBlock) * maxlen * 4 +
                                           static_cast<size_t>(wl) * maxlen * 8);
  const int i = rows[w];
  const int64_t ib = rp[i], ie = rp[i + 1];
  const int len = static_cast<int>(ie - ib);
  for (int k = lane; k < len; k += 32) {
    scol[k] = ci[ib + k];
    sval[k] = v[ib + k];
  }
  __syncwarp();
  for (int t = 0; t < len - 1; ++t) {  // entry ku = ib + t, column j < i
    const int j = scol[t];
    double s = sval[t];
    const int64_t jb = rp[j], je = rp[j + 1] - 1;  // row j without its diagonal
    const int pmax = t > 0 ? scol[t - 1] : -1;     // largest column of row i's finished prefix
    for (int64_t c0 = jb; t > 0 && c0 < je; c0 += 32) {
      const int64_t q = c0 + lane;
      int col = -1;
      double vj = 0.0;
      if (q < je) {
        col = ci[q];
        vj = v[q];
      }
      // col among row i's finished entries [0, t) (sorted ascending)
      int lo = 0, hi = t;
      if (col >= 0)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (scol[mid] < col)
            lo = mid + 1;
          else
            hi = mid;
        }
      const bool hit = col >= 0 && lo < t && scol[lo] == col;
      const double prod = hit ? __dmul_rn(sval[lo], vj) : 0.0;
      unsigned m = __ballot_sync(0xffffffffu, hit);
      while (m) {  // the merge's order: ascending column = lane order
        const int l = __ffs(m) - 1;
        m &= m - 1;
        s = __dsub_rn(s, __shfl_sync(0xffffffffu, prod, l));
      }
      // row j's columns ascend: once past row i's prefix nothing can match
      const int last = __shfl_sync(0xffffffffu, col, 31);
      if (last < 0 || last >= pmax) break;
    }
    const double lij = __ddiv_rn(s, v[rp[j + 1] - 1]);  // L_jj is final (earlier level)
    if (lane == 0) {
      sval[t] = lij;
      v[ib + t] = lij;
    }
    __syncwarp();
  }
  double d = sval[len - 1];
  for (int k = 0; k < len - 1; ++k) d = __dsub_rn(d, __dmul_rn(sval[k], sval[k]));
  if (lane == 0) {
    if (!(d > 0.0)) atomicMin(bad, i);
    v[ie - 1] = __dsqrt_rn(d);
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
    for (int64_t k = b; k < e - 1; ++k) lv = std::max(lv, level[l_cols[k]] + 1);
    level[i] = lv;
    nlev = std::max(nlev, lv + 1);
    maxlen = std::max(maxlen, static_cast<int>(e - b));
  }
  if (n_levels) *n_levels = nlev;
  if (n == 0) return DSGPU_OK;
  std::vector<int64_t> lstart(nlev + 1, 0);
  for (int i = 0; i < n; ++i) ++lstart[level[i] + 1];
  for (int l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
  std::vector<int32_t> order(n);
  {
    std::vector<int64_t> fill(lstart.begin(), lstart.end() - 1);
    for (int i = 0; i < n; ++i) order[fill[level[i]]++] = i;
  }
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * maxlen * 12;
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
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaFree(d_rows);
    cudaFree(d_v);
    cudaFree(d_bad);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  };
  const int big = 0x7fffffff;
  if (cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1)) != cudaSuccess ||
      cudaMalloc(&d_ci, sizeof(int32_t) * nnz) != cudaSuccess ||
      cudaMalloc(&d_rows, sizeof(int32_t) * n) != cudaSuccess || cudaMalloc(&d_v, sizeof(double) * nnz) != cudaSuccess ||
      cudaMalloc(&d_bad, sizeof(int)) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cleanup();
    return fail(DSGPU_E_CUDA, "ic0: device allocation failed");
  }
  cudaMemcpyAsync(d_rp, l_row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_ci, l_cols, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_v, l_vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_rows, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int l = 0; l < nlev; ++l) {
    const int cnt = static_cast<int>(lstart[l + 1] - lstart[l]);
    const int grid = (cnt + kWarpsPerBlock - 1) / kWarpsPerBlock;
    ic0_level_kernel<<<grid, kWarpsPerBlock * 32, smem, st>>>(d_rows + lstart[l], cnt, d_rp, d_ci, d_v, maxlen,
                                                              d_bad);
  }
  cudaEventRecord(e1, st);
  int bad = big;
  cudaMemcpyAsync(l_vals, d_v, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  float ms = 0.0f;
  if (e == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
  cleanup();
  if (e != cudaSuccess) return fail(DSGPU_E_CUDA, std::string("ic0: ") + cudaGetErrorString(e));
  if (device_ms) *device_ms = ms;
  if (bad != big) {
    if (bad_row) *bad_row = bad;
    return fail(DSGPU_E_FACTOR_BREAKDOWN, "factorization breakdown: nonpositive pivot at row " + std::to_string(bad));
  }
  return DSGPU_OK;
}

}  // extern "C"
