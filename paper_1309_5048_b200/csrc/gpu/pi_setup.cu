// Setup of the partitioned-inverse IC(0) apply (see pi.hpp): block plan on
// the host, block inverses on the device (cuBLAS dtrsm per block; setup only,
// not on the solve path).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "pi.hpp"

namespace dsgpu {

int pi_bandwidth(int n, const int64_t* lrp, const int32_t* lci) {
  int bw = 0;
  for (int i = 0; i < n; ++i)
    if (lrp[i + 1] > lrp[i]) bw = std::max(bw, i - lci[lrp[i]]);
  return bw;
}

PiPlan pi_plan(int n, const int64_t* lrp, const int32_t* lci, int bsz) {
  PiPlan P;
  P.n = n;
  P.bsz = std::max(1, std::min(bsz, n));
  P.nb = (n + P.bsz - 1) / P.bsz;
  const int bw = pi_bandwidth(n, lrp, lci);
  std::vector<int32_t> rowmin(n);
  for (int i = 0; i < n; ++i) rowmin[i] = lrp[i + 1] > lrp[i] ? lci[lrp[i]] : i;
  int64_t off = 0;
  P.blk.resize(P.nb);
  for (int i = 0; i < P.nb; ++i) {
    PiBlk& B = P.blk[i];
    B.s = i * P.bsz;
    B.e = std::min(n, B.s + P.bsz);
    int c = B.s;
    for (int r = B.s; r < B.e; ++r) c = std::min(c, rowmin[r]);
    B.c = c;
    int v = B.e;
    for (int r = B.e; r < std::min(n, B.e + bw + 1); ++r)
      if (rowmin[r] < B.e) v = r + 1;
    B.v = v;
    const int64_t b = B.e - B.s;
    auto even = [](int64_t x) { return (x + 1) & ~int64_t{1}; };
    B.dinv = off;
    off = even(off + b * b);
    B.dinvt = off;
    off = even(off + b * b);
    B.f = off;
    off = even(off + b * pi_ldw(B.s - B.c));
    B.h = off;
    off = even(off + b * pi_ldw(B.v - B.e));
    P.wmax = std::max(P.wmax, std::max(B.s - B.c, B.v - B.e));
  }
  P.n_coef = off;
  return P;
}

namespace {

// dense D (b x b), E (b x wf), Gt (b x wv), all column-major, from L's CSR
__global__ void scatter_block(const int64_t* rp, const int32_t* ci, const double* v, int s, int e,
                              int c, int vend, double* D, double* E, double* Gt) {
  const int b = e - s;
  for (int r = s + blockIdx.x; r < vend; r += gridDim.x)
    for (int64_t k = rp[r] + threadIdx.x; k < rp[r + 1]; k += blockDim.x) {
      const int col = ci[k];
      const double x = v[k];
      if (r < e) {
        if (col >= s)
          D[(r - s) + static_cast<int64_t>(col - s) * b] = x;
        else if (col >= c)
          E[(r - s) + static_cast<int64_t>(col - c) * b] = x;
      } else if (col >= s && col < e) {
        Gt[(col - s) + static_cast<int64_t>(r - e) * b] = x;
      }
    }
}

__global__ void set_identity(double* X, int b) {
  const int64_t nn = static_cast<int64_t>(b) * b;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nn;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    X[i] = (i % b) == (i / b) ? 1.0 : 0.0;
}

struct Scratch {
  void* p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  cublasHandle_t cb = nullptr;
  ~Scratch() {
    for (void* q : p) cudaFree(q);
    if (cb) cublasDestroy(cb);
  }
};

}  // namespace

std::string pi_fill(const PiPlan& P, const int64_t* lrp, const int32_t* lci, const double* lv,
                    double* d_coef, void* stream_v) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_v);
  Scratch S;
  const int n = P.n;
  const int64_t nnz = lrp[n];
  const int64_t b = P.bsz;
  auto ck = [](cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  };
  auto cbk = [](cublasStatus_t e, const char* what) {
    if (e != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string(what) + ": cuBLAS status " + std::to_string(e));
  };
  try {
    int64_t wf = 1, wv = 1;
    for (const PiBlk& B : P.blk) {
      wf = std::max<int64_t>(wf, B.s - B.c);
      wv = std::max<int64_t>(wv, B.v - B.e);
    }
    ck(cudaMalloc(&S.p[0], sizeof(int64_t) * (n + 1)), "pi: alloc");
    ck(cudaMalloc(&S.p[1], sizeof(int32_t) * std::max<int64_t>(nnz, 1)), "pi: alloc");
    ck(cudaMalloc(&S.p[2], sizeof(double) * std::max<int64_t>(nnz, 1)), "pi: alloc");
    ck(cudaMalloc(&S.p[3], sizeof(double) * b * b * 2), "pi: alloc");  // D | X
    ck(cudaMalloc(&S.p[4], sizeof(double) * b * wf), "pi: alloc");     // E
    ck(cudaMalloc(&S.p[5], sizeof(double) * b * wv), "pi: alloc");     // Gt
    auto* d_rp = static_cast<int64_t*>(S.p[0]);
    auto* d_ci = static_cast<int32_t*>(S.p[1]);
    auto* d_v = static_cast<double*>(S.p[2]);
    double* D = static_cast<double*>(S.p[3]);
    double* X = D + b * b;
    double* E = static_cast<double*>(S.p[4]);
    double* Gt = static_cast<double*>(S.p[5]);
    ck(cudaMemcpyAsync(d_rp, lrp, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st), "pi: H2D");
    ck(cudaMemcpyAsync(d_ci, lci, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st), "pi: H2D");
    ck(cudaMemcpyAsync(d_v, lv, sizeof(double) * nnz, cudaMemcpyHostToDevice, st), "pi: H2D");
    ck(cudaMemsetAsync(d_coef, 0, sizeof(double) * P.n_coef, st), "pi: memset");
    cbk(cublasCreate(&S.cb), "cublasCreate");
    cbk(cublasSetStream(S.cb, st), "cublasSetStream");
    cbk(cublasSetMathMode(S.cb, CUBLAS_PEDANTIC_MATH), "cublasSetMathMode");
    const double one = 1.0, mone = -1.0, zero = 0.0;
    for (const PiBlk& B : P.blk) {
      const int bi = B.e - B.s, w1 = B.s - B.c, w2 = B.v - B.e;
      ck(cudaMemsetAsync(D, 0, sizeof(double) * bi * bi, st), "pi: memset");
      if (w1) ck(cudaMemsetAsync(E, 0, sizeof(double) * bi * w1, st), "pi: memset");
      if (w2) ck(cudaMemsetAsync(Gt, 0, sizeof(double) * bi * w2, st), "pi: memset");
      scatter_block<<<std::min(B.v - B.s, 4096), 128, 0, st>>>(d_rp, d_ci, d_v, B.s, B.e, B.c, B.v, D, E, Gt);
      set_identity<<<256, 256, 0, st>>>(X, bi);
      ck(cudaGetLastError(), "pi: scatter");
      // X = D^{-1} (column-major) == row-major D^{-T}
      cbk(cublasDtrsm(S.cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, bi, bi,
                      &one, D, bi, X, bi),
          "trsm Dinv");
      ck(cudaMemcpyAsync(d_coef + B.dinvt, X, sizeof(double) * bi * bi, cudaMemcpyDeviceToDevice, st), "pi: copy");
      // row-major D^{-1} = column-major X^T
      cbk(cublasDgeam(S.cb, CUBLAS_OP_T, CUBLAS_OP_N, bi, bi, &one, X, bi, &zero, X, bi, d_coef + B.dinv, bi),
          "geam Dinv");
      if (w1) {
        cbk(cublasDtrsm(S.cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, bi, w1,
                        &mone, D, bi, E, bi),
            "trsm F");
        cbk(cublasDgeam(S.cb, CUBLAS_OP_T, CUBLAS_OP_N, w1, bi, &one, E, bi, &zero, E, w1, d_coef + B.f, pi_ldw(w1)),
            "geam F");
      }
      if (w2) {
        cbk(cublasDtrsm(S.cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, bi, w2,
                        &mone, D, bi, Gt, bi),
            "trsm H");
        cbk(cublasDgeam(S.cb, CUBLAS_OP_T, CUBLAS_OP_N, w2, bi, &one, Gt, bi, &zero, Gt, w2, d_coef + B.h, pi_ldw(w2)),
            "geam H");
      }
    }
    ck(cudaStreamSynchronize(st), "pi: setup");
  } catch (const std::exception& e) {
    cudaStreamSynchronize(st);
    return e.what();
  }
  (void)b;
  return std::string();
}

}  // namespace dsgpu
