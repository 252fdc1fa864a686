/* dsgpu — C ABI of the B200 (sm_100a) MINRES + IC(0) block-preconditioned
 * Stokes solve. Drop-in for the reference's solve call:
 *
 *   StokesSolution solve_stokes(const StokesSystem&, BlockDiagPreconditioner&,
 *                               const SolverOptions&)        proj/src/precond.cpp:245-293
 *   (strategy menu make_strategy, proj/src/precond.cpp:161-193)
 *
 * The reference's host code keeps assembling the system and building the
 * preconditioner factor exactly as PcgBlock does (rcm_permutation ->
 * permute_symmetric -> ic0, proj/src/precond.cpp:61-64) and hands the
 * resulting CSR arrays to dsgpu_setup; dsgpu_solve then runs the whole
 * MINRES loop (proj/src/solvers.cpp:24-123) with its inner PCG
 * (proj/src/solvers.cpp:125-159) and IC(0) applies (proj/src/cholesky.cpp:
 * 136-152) on the device — one cooperative persistent kernel, no host round
 * trip per iteration. See INTEGRATION.md for the reference-side shim.
 *
 * Layout: every CSR is the reference CsrMatrix layout (proj/include/divstokes/
 * csr.hpp:12-16): int64 row_ptr[n_rows+1], int32 cols (sorted, unique), f64
 * vals. All host arrays are borrowed for the duration of the call only.
 *
 * Errors mirror the reference's exception taxonomy (precond.cpp:141-147,
 * solvers.cpp:46,74-75,133,142,148): non-convergence is NOT an error
 * (report.converged = 0). A handle is not thread-safe (like BlockSolver);
 * distinct handles may be used from different threads, but their solves
 * serialize on the device: a solve is one cooperative kernel that occupies
 * every SM.
 */
#ifndef DSGPU_H
#define DSGPU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DSGPU_OK = 0,
  DSGPU_E_INDEFINITE_PRECOND = 1, /* <z,r> < 0 (block in report.failed_block) */
  DSGPU_E_NEG_CURVATURE = 2,      /* inner PCG: <p,Ap> <= 0 */
  DSGPU_E_BAD_INPUT = 3,          /* std::invalid_argument */
  DSGPU_E_CUDA = 4,               /* CUDA failure: dsgpu_last_error() */
  DSGPU_E_NONPOS_DIAG = 5,        /* Jacobi block: nonpositive diagonal (std::domain_error) */
  DSGPU_E_FACTOR_BREAKDOWN = 6,   /* IC(0): nonpositive pivot (FactorBreakdown, cholesky.hpp:13-19) */
  DSGPU_E_UNSUPPORTED = 7,        /* size beyond this build's limits */
  DSGPU_E_TIMEOUT = 8             /* a device-side wait exceeded DSGPU_TIMEOUT_S (default 10 s wall
                                     clock): the solve was aborted instead of hanging the GPU */
};

/* preconditioner block kinds (precond.cpp:14-118) */
enum {
  DSGPU_BLOCK_JACOBI = 0,     /* JacobiBlock: z = r / diag */
  DSGPU_BLOCK_PCG_JACOBI = 1, /* PcgBlock(Inner::jacobi) */
  DSGPU_BLOCK_PCG_IC0 = 2     /* PcgBlock(Inner::ic0): RCM + IC(0) preconditioned CG */
};

enum { DSGPU_STOP_PRECONDITIONED = 0, DSGPU_STOP_EUCLIDEAN = 1 }; /* MinresStop */

typedef struct {
  int32_t n_rows, n_cols;
  const int64_t* row_ptr;
  const int32_t* cols;
  const double* vals;
} dsgpu_csr;

/* SolverOptions (precond.hpp:52-59) + the inner cap make_strategy uses */
typedef struct {
  double outer_tol;  /* default 1e-12 */
  double inner_tol;  /* PCG tolerance; must match the factor's strategy */
  int32_t max_iter;  /* default 20000 */
  int32_t stop;      /* DSGPU_STOP_*; reference solve_stokes default: EUCLIDEAN */
  int32_t inner_cap; /* default 100000 (precond.cpp:167) */
} dsgpu_opts;

/* SolveReport (solvers.hpp:15-23) plus diagnostics */
typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t status;       /* DSGPU_* */
  int32_t failed_block; /* 0 velocity, 1 pressure, -1 none */
  double wall_seconds;  /* MINRES kernel time (CUDA events), excl. H2D/D2H */
  double mean_inner_top, mean_inner_bottom;
  double relres_m, relres_e; /* final M^-1-norm and Euclidean relative residuals */
  int64_t inner_top, apps_top, inner_bottom, apps_bottom;
  int32_t hist_len;     /* entries written to the history buffers */
  int32_t gpu_launches; /* kernels launched by this solve */
} dsgpu_report;

typedef struct dsgpu_handle dsgpu_handle;

const char* dsgpu_last_error(const dsgpu_handle* h); /* h may be NULL */
void dsgpu_default_opts(dsgpu_opts* o);

int dsgpu_create(int device, dsgpu_handle** out);
void dsgpu_destroy(dsgpu_handle* h);

/* ---- one solve across the GPUs of one NVLink box ----------
 * One process per GPU (rank r of `world` <= 8). Every rank calls
 * dsgpu_create_multi, then dsgpu_setup with the SAME system (each rank keeps
 * the operator rows it owns -- one contiguous velocity range and one pressure
 * range, balanced by nonzeros -- and the whole IC(0) plan: the sweeps are
 * replicated so the preconditioner is the single-GPU one), then exchanges one
 * 64-byte CUDA IPC handle with the other ranks (dsgpu_multi_ipc_export; the
 * host layer all-gathers them, e.g. torch.distributed; dsgpu_multi_ipc_import
 * takes the world x 64 bytes in rank order). After that dsgpu_solve /
 * dsgpu_solve_device run ONE partitioned solve: all ranks call them together
 * with the same arguments; SpMV halos are read from the owners' memory over
 * NVLink, dot products are exchanged through peer mailboxes and summed in rank
 * order (every rank computes identical scalars), and each rank returns the
 * entries of u and p it owns (all other entries of u_out / p_out untouched:
 * sum the ranks' zero-initialized outputs). world == 1 is dsgpu_create.
 * Blocked-sweep IC(0) velocity block required; Jacobi-PCG blocks unsupported. */
int dsgpu_create_multi(int rank, int world, int device, dsgpu_handle** out);
int dsgpu_multi_ipc_export(dsgpu_handle* h, void* handle64);
int dsgpu_multi_ipc_import(dsgpu_handle* h, const void* handles_world_x_64);

/* Upload the saddle system and the two preconditioner blocks.
 *   A (n_u x n_u), B (n_p x n_u), Bt (n_u x n_p), Q_nu (n_p x n_p): the
 *     StokesSystem blocks (assembly.hpp:31-49), original DOF order.
 *   top_kind / bottom_kind: DSGPU_BLOCK_*.
 *   perm_A, L_A: for PCG_IC0 tops, the RCM permutation of A and the IC(0)
 *     factor of permute_symmetric(A, perm_A) (Ic0Factor::lower: lower
 *     triangle incl. diagonal). NULL otherwise. Same for perm_Q, L_Q.
 *   Q_filter: the unscaled pressure mass Q when the constant pressure spans
 *     Ker(B^T) and solve_stokes's zero-mean filter applies (precond.cpp:
 *     266-284, kernel = all ones on the identity map); NULL disables it.
 * Everything is kept on the device in the RCM basis diag(P_A, P_Q), so the
 * inner PCG needs no per-apply gather/scatter. */
int dsgpu_setup(dsgpu_handle* h, const dsgpu_csr* A, const dsgpu_csr* B, const dsgpu_csr* Bt,
                const dsgpu_csr* Q_nu, int top_kind, const int32_t* perm_A, const dsgpu_csr* L_A,
                int bottom_kind, const int32_t* perm_Q, const dsgpu_csr* L_Q,
                const dsgpu_csr* Q_filter);

/* solve_stokes: b = [f; 0], x0 = 0, MINRES, zero-mean filter. HOST buffers
 * (f: n_u; u_out: n_u; p_out: n_p; histories nullable, capacity hist_cap:
 * residual_history / euclid_history as in SolveReport). */
int dsgpu_solve(dsgpu_handle* h, const double* f, const dsgpu_opts* opts, double* u_out,
                double* p_out, dsgpu_report* rep, double* hist_m, double* hist_e,
                int32_t hist_cap);

/* Initial guess of the NEXT solve on this handle (MinresOptions::x0,
 * solvers.hpp:34, solvers.cpp:35-42: x = x0, r1 = b - K x0, relative residuals
 * against ||b - K x0||): host vectors u0 (n_u), p0 (n_p) in the original
 * ordering, copied at once; the solve after it consumes the guess, later solves
 * start from 0 again. NULL, NULL cancels. Single-GPU handles. */
int dsgpu_set_initial_guess(dsgpu_handle* h, const double* u0, const double* p0);

/* Same, DEVICE buffers (cudaMalloc'd by the caller), on the handle's stream;
 * histories stay device-side and are not returned. Synchronizes at the end. */
int dsgpu_solve_device(dsgpu_handle* h, const double* d_f, const dsgpu_opts* opts,
                       double* d_u_out, double* d_p_out, dsgpu_report* rep);

/* ---- kernel-level entry points (parity tests, benchmarks) -------------- */
/* y = [A Bt; B 0] x in the ORIGINAL ordering (StokesSystem::apply,
 * assembly.cpp:363-372); host buffers of length n_u + n_p. */
int dsgpu_apply_saddle(dsgpu_handle* h, const double* x, double* y);
/* z = (L L^T)^{-1} r for block 0 (top) / 1 (bottom), in the block's RCM
 * ordering (Ic0Factor::solve, cholesky.cpp:136-152): the same operator, i.e.
 * mathematically identical to the reference's preconditioner. Bitwise identical
 * to the reference only in DSGPU_EXACT=1 mode (column-order sweeps, no FMA);
 * the default blocked sweeps re-associate each row's sum (dense 16 x 16 blocks
 * next to the diagonal, formed in long double) and agree with the reference
 * to round-off: <= 1e-13 relative in the tests, ~1e-15 measured. */
int dsgpu_apply_ic0(dsgpu_handle* h, int block, const double* r, double* z);
/* y = M x with M = permuted A (block 0) or permuted Q_nu (block 1). */
int dsgpu_apply_block_matrix(dsgpu_handle* h, int block, const double* x, double* y);
/* Time `reps` back-to-back launches of one kernel on device-resident data:
 * which = 0 saddle SpMV, 1 IC(0) apply (top), 2 IC(0) apply (bottom),
 * 3 block-0 SpMV. Returns mean ms per launch in *ms. */
int dsgpu_time_kernel(dsgpu_handle* h, int which, int reps, double* ms);
/* Roofline probe of the fused MINRES vector pass (the persistent kernel's
 * minres_update_row + ||res||^2 block reduction, solvers.cpp:93-101) as a
 * stand-alone kernel on `device` over n rows of synthetic data (no handle):
 * v[i] = (i%97)/100, av = (i%89)/50 - 1/2, w1 = (i%83) 3e-3, w2 = (i%79) 4e-3,
 * aw1 = (i%73) 5e-3, aw2 = (i%71) 6e-3, x = (i%67) 7e-3,
 * res = (i%61) 8e-3 - 1/5; oldeps = 1/4, delta = 1/2, gamma = 3/2, phi = 1e-3.
 * Runs 1 + reps launches (x, res updated in place each launch), returns the
 * mean ms of the last reps in *ms and ||res||^2 after the last launch in
 * *res2 (sum of the per-CTA partials). 96 bytes per row per launch. */
int dsgpu_time_vector_update(int device, int64_t n, int reps, double* ms, double* res2);

/* ---- host-setup on the device --------------- */
/* IC(0) factor of a symmetric CSR matrix on `device`, bit-identical to the
 * reference's ic0 (proj/src/cholesky.cpp:84-134): one warp per row, each
 * row's entries in the reference's order with explicitly rounded arithmetic;
 * a persistent dataflow kernel where entry (i, j) waits only for row j's
 * completion flag (DSGPU_IC0_FLOW=0: one launch per level of L's DAG).
 * Outputs (host, caller-allocated): l_row_ptr[n+1], l_cols / l_vals sized
 * nnz(lower(A)) incl. the diagonal. Errors: DSGPU_E_BAD_INPUT (structurally
 * missing diagonal, std::invalid_argument), DSGPU_E_FACTOR_BREAKDOWN with the
 * first failing row in *bad_row. *n_levels = DAG depth, *device_ms = time of
 * the level launches (CUDA events). Message: dsgpu_ic0_last_error(). */
int dsgpu_ic0_factor(int device, int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                     int64_t* l_row_ptr, int32_t* l_cols, double* l_vals, int* bad_row, int* n_levels,
                     double* device_ms);
const char* dsgpu_ic0_last_error(void);

/* Sizes of the device-resident problem (for roofline accounting):
 * info[0..15] = n_u, n_p, nnz_K, nnz_Aperm, nnz_L_A, nnz_L_Q, nnz_Qperm,
 * dependent steps of the forward / backward sweep of A, of Q (16-row groups
 * with the blocked sweeps, dependency levels otherwise), grid_ctas, IC(0)
 * apply mode (0 exact column order, 1 staged level sweeps, 2 partitioned
 * inverse, 3 blocked sweeps), dependent steps of one velocity IC(0) apply,
 * far-worker CTAs of the A and Q block. */
int dsgpu_info(const dsgpu_handle* h, int64_t* info);

/* Blocked-sweep plan check (no device): builds the blocked-sweep plan of the
 * factor L (as dsgpu_setup does) and evaluates it on the host in the plan's own
 * arithmetic order, z = (L L^T)^{-1} r. A test hook for the plan's structure
 * and coefficients, never used by a solve. stats8 (nullable): groups, factor
 * entries in dense blocks / mid lists / far lists (forward sweep), widest mid
 * and far list, padded mid and far list entries. */
int dsgpu_debug_bsweep_host(int n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                            const double* r, double* z, int64_t* stats8);

/* Multi-GPU row partition check (no device): partitions a square operator
 * (n rows; the first n_u are velocity rows whose first na[i] entries are the A
 * part, na nullable) over `world` ranks as dsgpu_setup_multi does -- one
 * contiguous velocity range and one pressure range per rank, each balanced by
 * nonzeros -- and evaluates y = K x rank by rank: halo gather from the owners'
 * slices, then the local rows. bounds: 2 (world + 1) ints; halo_counts:
 * world x world entries (row r: what rank r reads from each source rank). */
int dsgpu_debug_partition_spmv(int n, int n_u, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                               const int32_t* na, int world, int32_t* bounds, int64_t* halo_counts,
                               const double* x, double* y);

/* Multi-rank emulation on ONE GPU (tests of the multi-GPU data plane on a
 * single-GPU box): `world` handles made by dsgpu_create_multi(r, world, device)
 * on the same device in this process and set up with the same system (their
 * grids equal and world x grid <= SM count: DSGPU_GRID) solve it as `world`
 * ranks inside ONE cooperative launch whose CTAs are split into `world` groups;
 * group r runs rank r's solve and reaches the other ranks' arenas exactly as it
 * would reach peer GPUs (halo gathers, reduction mailboxes, pushed residuals).
 * f / u_out / p_out: host vectors of the whole system; reps: world reports. */
int dsgpu_debug_emulate_ranks(dsgpu_handle** handles, int world, const double* f, const dsgpu_opts* o,
                              double* u_out, double* p_out, dsgpu_report* reps);

/* Process-wide sweep diagnostics (summed since the last reset), out32:
 * [0] main-warp cycles, [1] main cycles waiting, [2] groups, [3] abort code,
 * [4] main cycles waiting for static slot data, [5] helper cycles waiting for
 * dependencies, [6] helper cycles waiting for remote partial sums, [7] helper
 * cycles; [8..11] groups by the main warp's distance when their prefix sum was
 * published (<=1, 2-3, 4-6, >=7 groups ahead), [12..15] the same when the
 * helper started them (<=3, 4-7, 8-11, >=12); [16] helper cycles from the last
 * dependency wait to publication, [17] groups whose last wait spun, [18]
 * co-main cycles waiting, [19..22] helper publication phases (last chunk,
 * slot reuse, store, fence + flag), [23] co-main cycles from its last wait to
 * publication, [24..27] co-main publications by the main warp's distance
 * (<=0, 1, 2, >=3 groups ahead), [28..29] co-main waits that found the
 * prefix sum / the dependencies not ready, [30..31] 0. */
int dsgpu_debug_counters(int reset, int64_t* out32);
/* Blocked-sweep diagnostics, summed since the last reset; all zero unless the
 * library was built with -DDSGPU_DIAG (make diag; the production kernels carry
 * no counters). out16: [0] main-warp cycles, [1] main cycles waiting for c,
 * [2] for dense-block slots, [3] for the publisher, [4] groups, [5] co-main
 * cycles waiting for progress, [6] for far sums, [7] co-main cycles, [8]
 * far-worker cycles waiting for progress, [9] far-worker cycles. */
int dsgpu_debug_bs_counters(int reset, int64_t* out16);
/* Persistent-kernel phase diagnostics (cycles; -DDSGPU_DIAG build only): out8 = CTA0 grid-barrier
 * wait, CTA0 IC(0) apply, CTA2 grid-barrier wait, barriers, CTA0 kernel,
 * CTA1 IC(0) apply, 0, 0. */
int dsgpu_debug_phases(int reset, int64_t* out8);
/* SpMV phases inside the persistent kernel as worker CTA 0 times them (cycles;
 * -DDSGPU_DIAG build only). Outer saddle SpMV (the reference's
 * StokesSystem::apply inside minres, solvers.cpp:66): out8[0] cycles over its own
 * rows, [1] phases, [2] stored entries of its rows, [3] cycles through the
 * phase's grid barrier. Inner A-block SpMV (pcg, solvers.cpp:139): [4] own
 * cycles, [5] phases, [6] stored entries of its rows, [7] cycles through the
 * barrier (the pressure block's SpMV included). */
int dsgpu_debug_spmv_phases(int reset, int64_t* out8);
/* Partitioned-inverse IC(0) apply timeline: arm != 0 arms the recorder (CTA 0
 * and the last CTA record %globaltimer at every phase boundary of their next
 * apply); arm == 0 reads it: out1024[s*512] = marks recorded by slot s,
 * out1024[s*512 + 1 ..] = timestamps (ns): start, g done, per forward step
 * (window staged, rows stored), h done, per backward step (same). */
int dsgpu_debug_pi_trace(int arm, int64_t* out1024);

#ifdef __cplusplus
}
#endif
#endif
