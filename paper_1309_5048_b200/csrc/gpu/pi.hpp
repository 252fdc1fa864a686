// Partitioned-inverse ("PI") IC(0) apply: data layout shared by the setup
// (pi_setup.cu, host + cuBLAS) and the device code (pi.cuh).
//
// z = (L L^T)^{-1} r with L the IC(0) factor in RCM order (Ic0Factor::solve,
// reference proj/src/cholesky.cpp:136-152). Rows are cut into consecutive
// blocks i = [s_i, e_i) of size b >= the lower bandwidth of L, so block i
// couples only to the window [c_i, s_i) of earlier rows (forward) and the
// window [e_i, v_i) of later rows (backward). With D_i the diagonal block of L,
//   forward : y_i = D_i^{-1} r_i  - D_i^{-1} E_i y[c_i, s_i)      (= g_i + F_i y_win)
//   backward: z_i = D_i^{-T} y_i  - D_i^{-T} G_i^T z[e_i, v_i)    (= h_i + H_i z_win)
// The block inverses are formed once at setup; the apply is then four dense
// phases (g, forward chain, h, backward chain) whose only sequential part is
// the chain over blocks: 2 * ceil(n / b) dependent steps instead of the
// 2 * (RCM depth) levels of a level-scheduled sweep.
#ifndef DSGPU_PI_HPP
#define DSGPU_PI_HPP
#include <cstdint>
#include <string>
#include <vector>

namespace dsgpu {

struct PiBlk {
  int32_t s, e;    // rows [s, e)
  int32_t c, v;    // forward window [c, s); backward window [e, v)
  int64_t dinv;    // D_i^{-1}, row-major b_i x b_i (lower triangle used), offset in doubles
  int64_t dinvt;   // D_i^{-T}, row-major b_i x b_i (upper triangle used)
  int64_t f;       // F_i = -D_i^{-1} E_i, row-major b_i x (s - c), row stride pi_ld(s - c)
  int64_t h;       // H_i = -D_i^{-T} G_i^T, row-major b_i x (v - e), row stride pi_ld(v - e)
};

// F/H row stride: even, so every row starts 16-byte aligned (one bulk copy)
inline constexpr int pi_ldw(int w) { return (w + 1) & ~1; }

struct PiPlan {
  int n = 0, bsz = 0, nb = 0;
  int wmax = 0;          // largest window (forward or backward)
  int64_t n_coef = 0;    // doubles of coefficient storage
  std::vector<PiBlk> blk;
};

// Blocks of size bsz (>= 1) over the factor L (CSR, lower triangle incl. the
// diagonal, diagonal last in each row).
PiPlan pi_plan(int n, const int64_t* lrp, const int32_t* lci, int bsz);
// Lower bandwidth max_i (i - min col of row i).
int pi_bandwidth(int n, const int64_t* lrp, const int32_t* lci);
// Fill d_coef (plan.n_coef doubles, device) on `stream` (cuBLAS trsm per
// block). Returns an empty string on success, else the error.
std::string pi_fill(const PiPlan& plan, const int64_t* lrp, const int32_t* lci, const double* lv,
                    double* d_coef, void* stream);

}  // namespace dsgpu
#endif
