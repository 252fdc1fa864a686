"""GPU parity: the sm_100a solve through the C ABI against the CPU oracle
(the reference itself when oracle/_ref is built, else the C restatement) on
identical inputs. Bar (BASELINE north_star): solution rel-L2 <= 1e-8, outer
iterations within +-2, final relative residual <= tol. Kernel-level checks:
saddle SpMV to 1e-14 (fp64, different summation order), IC(0) apply
bit-identical (same per-row operation order as Ic0Factor::solve)."""
import numpy as np
import pytest

from conftest import golden_csr, load_golden, to_oracle

pytestmark = pytest.mark.gpu

STRATS = ["IC0-PCG(A,Q)", "IC0-PCG(A)+Diag(Q)", "PCG(A,Q)", "PCG(A)+Diag(Q)", "Diag(A,Q)"]


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_5048_b200 import host, solver
    return host, solver


def reference_solve(port, system, strategy, outer, inner, max_iter=20000):
    """CPU oracle solve on the identical system (reference-exact restatement)."""
    o = port.solve_stokes(to_oracle(system.A), to_oracle(system.B), to_oracle(system.Bt),
                          to_oracle(system.Q_nu), system.f, strategy, outer, inner,
                          max_iter=max_iter, Q_filter=to_oracle(system.Q))
    assert o["status"] == 0
    return o


def check_parity(sol, o, tol):
    x = np.concatenate([sol.u, sol.p])
    xr = np.concatenate([o["u"], o["p"]])
    rel = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    assert rel <= 1e-8, rel
    assert abs(sol.report.iterations - o["iterations"]) <= 2
    assert sol.report.converged and o["converged"]
    assert sol.report.relres_e <= tol
    return rel


def test_saddle_apply_matches_reference(gpu, port):
    host, solver = gpu
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    y = g.apply(d["apply_x"])
    ref = d["apply_y"]
    assert np.abs(y - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("pi_b", [None, "0.5", "1.7", "3.0"])
def test_ic0_apply_partitioned_inverse_matches_reference(gpu, port, monkeypatch, pi_b):
    """Legacy partitioned-inverse IC(0) apply (DSGPU_PI=1; block inverses of
    the same factor; agreement to round-off). pi_b scales the block size (0.5:
    windows spanning two earlier blocks; 1.7: ragged last block; 3.0: windows
    shorter than the block)."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_PI", "1")
    if pi_b:
        monkeypatch.setenv("DSGPU_PI_B", pi_b)
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    for b, tag in ((0, "A"), (1, "Q")):
        z = g.apply_ic0(b, d["ic_r_" + tag])
        ref = d["ic_z_" + tag]  # the reference's own Ic0Factor::solve output
        assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()
    s = host.assemble("psi-mms", 2, 64)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    for b, fac in ((0, g.top.factor), (1, g.bottom.factor)):
        r = np.random.default_rng(3 + b).standard_normal(fac.n_rows)
        z = g.apply_ic0(b, r)
        ref = port.ic0_solve(to_oracle(fac), r)
        assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)


@pytest.mark.parametrize("knobs", [{}, {"DSGPU_FAR_A": "0", "DSGPU_FAR_Q": "0"}, {"DSGPU_GRID": "5"},
                                   {"DSGPU_FAR_A": "3", "DSGPU_FAR_Q": "1", "DSGPU_BS_SLOTS": "10"},
                                   {"DSGPU_BS_PAIR": "0"}, {"DSGPU_BS_PAIR": "0", "DSGPU_FAR_A": "0", "DSGPU_FAR_Q": "0"}])
def test_ic0_apply_blocked_matches_reference(gpu, port, monkeypatch, knobs):
    """Blocked sweeps (bsweep.hpp; the IC(0) apply of the large 3D systems,
    forced here with DSGPU_SWEEP=bs) -- dense 16x16 blocks next to the diagonal
    on the two main warps, mid entries on the co-main warps, far entries on
    far-worker CTAs -- against the reference's own Ic0Factor::solve output
    (fixture), the CPU oracle on 2D and 3D factors, and through a whole solve.
    knobs: no far-worker CTAs (the sweep CTAs' spare warps do the far lists), a
    5-CTA grid, few far CTAs with a different slot ring depth; by default every
    sweep runs on a CTA pair (2-CTA cluster: chain + lists over DSMEM),
    DSGPU_BS_PAIR=0 is the single-CTA form."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_SWEEP", "bs")
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    assert g.info()["ic0_mode"] == "blocked"
    for b, tag in ((0, "A"), (1, "Q")):
        z = g.apply_ic0(b, d["ic_r_" + tag])
        ref = d["ic_z_" + tag]  # the reference's own Ic0Factor::solve output
        assert np.abs(z - ref).max() <= 1e-13 * np.abs(ref).max()
    g.close()
    for case, k, n, dim in (("psi-mms", 2, 64, 2), ("random", 3, 32, 2), ("psi-mms", 2, 12, 3)):
        s = host.assemble(case, k, n, dim=dim, seed=7)
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
        for b, fac in ((0, g.top.factor), (1, g.bottom.factor)):
            r = np.random.default_rng(3 + b).standard_normal(fac.n_rows)
            ref = port.ic0_solve(to_oracle(fac), r)
            for _ in range(2):  # a second apply reuses the slot ring, flags and tags
                z = g.apply_ic0(b, r)
                assert np.linalg.norm(z - ref) <= 1e-13 * np.linalg.norm(ref)
        sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
        check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)
        g.close()


def test_ic0_mode_policy(gpu):
    """Setup's choice of the IC(0) apply: the partitioned inverse where its
    model wins (small-bandwidth 2D factors), the exact sweeps on request."""
    host, solver = gpu
    g = solver.GpuStokesSolver(host.assemble("psi-mms", 2, 32), "IC0-PCG(A,Q)")
    assert g.info()["ic0_mode"] == "partitioned-inverse"
    g.close()


def test_multi_gpu_entry_point_world1(gpu, port):
    """dsgpu_create_multi with world = 1 is the single-GPU solver (the multi-GPU
    data plane -- per-rank row ranges, owner-written tagged right-hand sides,
    the arena -- is one code path; with one rank it has no peers and no halos)."""
    import ctypes as C
    host, solver = gpu
    s = host.assemble("psi-mms", 2, 10, dim=3)
    monkey = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    L = monkey.L
    h = C.c_void_p()
    assert L.dsgpu_create_multi(0, 1, 0, C.byref(h)) == 0
    L.dsgpu_destroy(h)
    assert L.dsgpu_create_multi(1, 1, 0, C.byref(h)) != 0  # rank out of range
    assert L.dsgpu_create_multi(0, 9, 0, C.byref(h)) != 0  # more than one box's GPUs
    sol = monkey.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)
    monkey.close()


@pytest.mark.parametrize("world,dim,n", [(2, 2, 16), (3, 2, 24), (4, 3, 8), (2, 3, 12)])
def test_multi_gpu_data_plane_emulated(gpu, port, monkeypatch, world, dim, n):
    """The multi-GPU solve (row-partitioned operators, halo gathers, cross-rank
    reductions, pushed tagged residuals, replicated sweeps) run as `world` ranks
    inside ONE cooperative launch on one GPU (dsgpu_debug_emulate_ranks): every
    rank must report the reference's iteration counts and the assembled
    solution must match the reference like the single-GPU solve does."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_SWEEP", "bs")
    monkeypatch.setenv("DSGPU_GRID", str((148 // world - 4) & ~1))   # worker CTAs per rank (+ 2 server CTA pairs each)
    monkeypatch.setenv("DSGPU_TIMEOUT_S", "60")
    s = host.assemble("psi-mms", 2, n, dim=dim)
    o = solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1)
    sol, reps = solver.emulate_ranks(s, "IC0-PCG(A,Q)", world, o)
    ref = reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1)
    check_parity(sol, ref, 1e-8)
    for r in reps:
        assert (r.iterations, r.inner_top, r.inner_bottom) == (reps[0].iterations, reps[0].inner_top,
                                                               reps[0].inner_bottom)
        assert r.relres_e == reps[0].relres_e  # identical scalars on every rank


def test_two_handles_of_different_sizes(gpu, port):
    """Distinct handles: a smaller system set up after a larger one must not
    disturb the first handle's launches (shared-memory limits are per kernel
    function, raised once, never lowered)."""
    host, solver = gpu
    s1 = host.assemble("psi-mms", 2, 32)
    s2 = host.assemble("psi-mms", 2, 8)
    g1 = solver.GpuStokesSolver(s1, "IC0-PCG(A,Q)")
    g2 = solver.GpuStokesSolver(s2, "IC0-PCG(A)+Diag(Q)")
    o = solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1)
    check_parity(g1.solve(options=o), reference_solve(port, s1, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)
    check_parity(g2.solve(options=o), reference_solve(port, s2, "IC0-PCG(A)+Diag(Q)", 1e-8, 1e-1), 1e-8)
    check_parity(g1.solve(options=o), reference_solve(port, s1, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)
    g1.close()
    g2.close()


def test_ic0_apply_staged_matches_reference(gpu, port, monkeypatch):
    """Staged dataflow sweeps (DSGPU_PI=0; the mode for systems whose block
    inverses do not fit): same factor and operation, summation reassociated
    inside each row -> agreement to round-off."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_PI", "0")
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    for b, tag in ((0, "A"), (1, "Q")):
        z = g.apply_ic0(b, d["ic_r_" + tag])
        ref = d["ic_z_" + tag]  # the reference's own Ic0Factor::solve output
        assert np.abs(z - ref).max() <= 1e-13 * np.abs(ref).max()
    s = host.assemble("psi-mms", 2, 64)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    r = np.random.default_rng(3).standard_normal(s.n_u)
    z = g.apply_ic0(0, r)
    ref = port.ic0_solve(to_oracle(g.top.factor), r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()


def test_ic0_apply_exact_mode_bit_identical(gpu, port, monkeypatch):
    """DSGPU_EXACT=1 selects column-order sweeps with separately rounded
    mul/sub and IEEE division: bit-identical to Ic0Factor::solve."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_EXACT", "1")
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    for b, tag in ((0, "A"), (1, "Q")):
        assert np.array_equal(g.apply_ic0(b, d["ic_r_" + tag]), d["ic_z_" + tag])
    s = host.assemble("psi-mms", 2, 64)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    r = np.random.default_rng(3).standard_normal(s.n_u)
    assert np.array_equal(g.apply_ic0(0, r), port.ic0_solve(to_oracle(g.top.factor), r))
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    assert sol.report.converged and sol.report.iterations == 57


def test_block_matrix_apply(gpu, port):
    host, solver = gpu
    s = host.assemble("cavity", 2, 16)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    P = port.permute(to_oracle(s.A), g.top.perm)
    x = np.random.default_rng(4).standard_normal(s.n_u)
    y = g.apply_block_matrix(0, x)
    yr = port.spmv(P, x)
    assert np.abs(y - yr).max() <= 1e-14 * np.abs(yr).max()


@pytest.mark.parametrize("strategy", STRATS)
def test_small_system_all_strategies_vs_golden(gpu, strategy):
    """Reference solutions committed by make_golden.py (reference run)."""
    host, solver = gpu
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    for itol in (1e-1, 1e-6):
        key = f"{strategy}|{itol:g}"
        sol = solver.solve_stokes(s, strategy, solver.SolverOptions(outer_tol=1e-8, inner_tol=itol))
        meta = d["sol_meta|" + key]
        x = np.concatenate([sol.u, sol.p])
        xr = np.concatenate([d["sol_u|" + key], d["sol_p|" + key]])
        assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
        assert abs(sol.report.iterations - int(meta[0])) <= 2
        assert sol.report.converged
        hm = sol.report.residual_history
        assert hm[0] == 1.0 and len(hm) == sol.report.iterations + 1
        assert np.all(hm[1:] <= hm[:-1] * (1 + 1e-10))  # M^-1-norm nonincreasing


def test_config1_vs_golden(gpu):
    """BASELINE config 1: 16x16, IC0-PCG(A)+Diag(Q), outer 1e-8, inner 1e-1."""
    host, solver = gpu
    g = load_golden("c1_psi_k2_n16.npz")
    s = host.assemble("psi-mms", 2, 16)
    sol = solver.solve_stokes(s, "IC0-PCG(A)+Diag(Q)",
                              solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    x = np.concatenate([sol.u, sol.p])
    xr = np.concatenate([g["u"], g["p"]])
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
    assert abs(sol.report.iterations - int(g["meta"][0])) <= 2
    assert abs(sol.report.mean_inner_top - g["meta"][2]) < 0.1
    assert sol.report.relres_e <= 1e-8


@pytest.mark.parametrize("inner", [1e-1, 1e-8])
def test_config2_both_variants(gpu, port, inner):
    """BASELINE config 2: 64x64 k'=2, IC0-PCG(A,Q), exact-ish and relaxed inner CG."""
    host, solver = gpu
    s = host.assemble("psi-mms", 2, 64)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-8, inner_tol=inner))
    o = reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, inner)
    check_parity(sol, o, 1e-8)
    assert abs(sol.report.mean_inner_top - o["mean_inner_top"]) < 0.2


def test_random_rhs_k3(gpu, port):
    """Config-3 data (k'=3, U[-1,1] RHS, seed 1234) at a CI-sized mesh."""
    host, solver = gpu
    s = host.assemble("random", 3, 16, seed=1234)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)


def test_3d_small(gpu, port):
    """Config-4 data (3D psi-MMS, k'=2) at 4^3: no reference 3D code exists, the
    oracle is the reference's solver layer restated."""
    host, solver = gpu
    s = host.assemble("psi-mms", 2, 4, dim=3)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)


def test_cavity_ic0_windows(gpu):
    """test_system.cpp:178-197: cavity k'=2 h=1/32, default options."""
    host, solver = gpu
    s = host.assemble("cavity", 2, 32)
    for tol, lo, hi in ((1e-3, 4.0, 9.0), (1e-6, 9.0, 17.0)):
        sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(inner_tol=tol))
        r = sol.report
        assert r.converged and 34 <= r.iterations <= 44
        assert r.mean_inner_bottom <= 2.0 and lo <= r.mean_inner_top <= hi


def test_nu_rescaling_identical(gpu):
    """test_system.cpp:199-215 (with the GPU strategy): nu = 1 vs 4."""
    host, solver = gpu
    a = host.assemble("cavity", 2, 8, nu=1.0)
    b = host.assemble("cavity", 2, 8, nu=4.0)
    ra = solver.solve_stokes(a, "IC0-PCG(A,Q)", solver.SolverOptions()).report
    rb = solver.solve_stokes(b, "IC0-PCG(A,Q)", solver.SolverOptions()).report
    assert ra.iterations == rb.iterations
    np.testing.assert_allclose(ra.residual_history, rb.residual_history, rtol=1e-13)


def test_bit_deterministic(gpu):
    host, solver = gpu
    s = host.assemble("cavity", 2, 8)
    g = solver.GpuStokesSolver(s, "PCG(A,Q)")
    a = g.solve()
    b = g.solve()
    assert a.report.iterations == b.report.iterations
    assert np.array_equal(a.u, b.u) and np.array_equal(a.p, b.p)
    assert np.array_equal(a.report.euclid_history, b.report.euclid_history)


def test_blocked_sweeps_bitwise_reproducible(gpu, monkeypatch):
    """The blocked sweeps fix the order of every sum (dense blocks, mid lists,
    far partial sums per worker), so repeated solves -- on one handle and on a
    fresh one -- must agree BIT FOR BIT; a lost hand-off or a race between the
    chain CTA, the list CTA and the far workers would show as a differing bit
    (tools/soak.py is the long form: 20 C4 solves, 6 at 48^3)."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_SWEEP", "bs")
    s = host.assemble("random", 2, 14, dim=3, seed=42)
    o = solver.SolverOptions(outer_tol=1e-6, inner_tol=1e-1)
    ref = None
    for _ in range(2):
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
        assert g.info()["ic0_mode"] == "blocked"
        for _ in range(4):
            sol = g.solve(options=o)
            x = np.concatenate([sol.u, sol.p])
            ref = x if ref is None else ref
            assert np.array_equal(ref, x)
        g.close()


def test_max_iter_and_errors(gpu):
    host, solver = gpu
    s = host.assemble("psi-mms", 2, 8)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1, max_iter=3))
    assert not sol.report.converged and sol.report.iterations == 3
    # max_iter = 0: the reference returns x0 = 0 after one preconditioner apply (solvers.cpp:36-62)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1, max_iter=0))
    assert not sol.report.converged and sol.report.iterations == 0
    assert not sol.u.any() and not sol.p.any() and len(sol.report.euclid_history) == 1
    from paper_1309_5048_b200.host import CsrMatrix, StokesSystem
    negQ = CsrMatrix(s.Q_nu.n_rows, s.Q_nu.n_cols, s.Q_nu.row_ptr, s.Q_nu.cols, -s.Q_nu.vals)
    bad = StokesSystem(s.A, s.B, s.Bt, s.Q, negQ, s.f)
    with pytest.raises(ArithmeticError):
        solver.solve_stokes(bad, "IC0-PCG(A)+Diag(Q)")
    # indefinite A: PCG(A) hits negative curvature
    negA = CsrMatrix(s.A.n_rows, s.A.n_cols, s.A.row_ptr, s.A.cols, s.A.vals.copy())
    diag = negA.cols == np.repeat(np.arange(negA.n_rows), np.diff(negA.row_ptr))
    negA.vals[~diag] *= 40.0
    bad = StokesSystem(negA, s.B, s.Bt, s.Q, s.Q_nu, s.f)
    with pytest.raises(solver.PreconditionerError):
        solver.solve_stokes(bad, "PCG(A)+Diag(Q)", solver.SolverOptions(inner_tol=1e-6))


def test_ring_mode_forced_small(gpu, port, monkeypatch):
    """Ring mode (results beyond the shared-memory ring published in global
    memory) forced on a small system: same answers as the full-vector mode."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_PI", "0")
    monkeypatch.setenv("DSGPU_RING_N", "1")
    s = host.assemble("psi-mms", 2, 16)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    r = np.random.default_rng(5).standard_normal(s.n_u)
    z = g.apply_ic0(0, r)
    ref = port.ic0_solve(to_oracle(g.top.factor), r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)


@pytest.mark.parametrize("pi", ["0", "1"])
def test_large_system_ring_mode(gpu, port, monkeypatch, pi):
    """k'=3, 96x96 (n_u = 19,404 > shared memory): ring mode chosen by setup
    when the partitioned inverse is off; the partitioned inverse otherwise."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_PI", pi)
    s = host.assemble("random", 3, 96, seed=1234)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)


# C3 stagnates near 4e-7 in the reference (relaxed inner CG makes the block
# preconditioner vary between applications), so both sides run to the same
# iteration cap and parity is parity of the iterates at that count.
FULL = {
    "c3": ("c3_rand_k3_n256.npz",
           dict(case="random", k_prime=3, n_elem=256, dim=2, seed=1234, max_iter=150)),
    "c4": ("c4_psi3d_k2_n32.npz",
           dict(case="psi-mms", k_prime=2, n_elem=32, dim=3, seed=0, max_iter=400)),
}


@pytest.mark.parametrize("cfg", sorted(FULL))
def test_full_size_config_vs_reference(gpu, cfg):
    """BASELINE configs 3 (2D k'=3 256^2, U[-1,1] seed 1234) and 4 (3D 32^3
    psi-MMS) at FULL size against the reference's own solve of the identical
    system (tests/golden/make_golden_large.py): rel-L2 <= 1e-8, outer
    iterations +-2, inner means close, the Euclidean residual history within
    1e-8 relative, convergence (C4: final residual <= 1e-8) or the same capped
    non-convergence (C3), and the true residual ||b - K x|| / ||b|| through the
    device saddle apply agreeing with the recurrence."""
    host, solver = gpu
    name, kw = FULL[cfg]
    g = load_golden(name)
    s = host.assemble(kw["case"], kw["k_prime"], kw["n_elem"], dim=kw["dim"], seed=kw["seed"])
    assert [s.n_u, s.n_p, s.A.nnz, s.B.nnz, s.Q.nnz] == g["sizes"].tolist()
    gs = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    assert gs.info()["ic0_mode"] == ("blocked" if cfg == "c4" else "partitioned-inverse")
    sol = gs.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1,
                                                max_iter=kw["max_iter"]))
    x = np.concatenate([sol.u, sol.p])
    xr = np.concatenate([g["u"], g["p"]])
    rel = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    assert rel <= 1e-8, rel
    assert abs(sol.report.iterations - int(g["meta"][0])) <= 2, (sol.report.iterations, g["meta"])
    assert abs(sol.report.mean_inner_top - g["meta"][2]) < 0.2
    assert abs(sol.report.mean_inner_bottom - g["meta"][3]) < 0.2
    he, hr = sol.report.euclid_history, g["he"]
    m = min(len(he), len(hr))
    assert np.all(np.abs(he[:m] - hr[:m]) <= 1e-8 * hr[:m])
    assert sol.report.converged == bool(g["meta"][1])
    if sol.report.converged:
        assert sol.report.relres_e <= 1e-8
    b = np.concatenate([s.f, np.zeros(s.n_p)])
    true = np.linalg.norm(b - gs.apply(x)) / np.linalg.norm(b)
    assert abs(true - sol.report.relres_e) <= 1e-3 * sol.report.relres_e + 1e-12
    gs.close()


def test_c5_data_small_vs_reference(gpu, port):
    """Config-5 data (3D k'=2, f_u ~ U[-1,1] seed 42, outer 1e-6) at 8^3 against
    the CPU oracle on the identical system."""
    host, solver = gpu
    s = host.assemble("random", 2, 8, dim=3, seed=42)
    sol = solver.solve_stokes(s, "IC0-PCG(A,Q)", solver.SolverOptions(outer_tol=1e-6, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-6, 1e-1), 1e-6)


def test_c5_data_48_vs_reference(gpu):
    """BASELINE config 5's data (3D k'=2, f_u ~ U[-1,1] seed 42, outer 1e-6,
    inner 1e-1) at 48^3 (492,500 unknowns, nnz(L_A) 90.5M, ring-mode sweeps with
    remote helpers) against the reference's own solve of the identical system
    (tests/golden/make_golden_large.py c5_48): rel-L2 <= 1e-8, outer iterations
    +-2, inner means, the Euclidean residual history, convergence to 1e-6, and
    the true residual through the device saddle apply. The preconditioner setup
    uses the device IC(0) factor (bit-identical to the reference's)."""
    host, solver = gpu
    g = load_golden("c5data_rand3d_k2_n48.npz")
    s = host.assemble("random", 2, 48, dim=3, seed=42)
    assert [s.n_u, s.n_p, s.A.nnz, s.B.nnz, s.Q.nnz] == g["sizes"].tolist()
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    gs = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
    sol = gs.solve(options=solver.SolverOptions(outer_tol=1e-6, inner_tol=1e-1, max_iter=400))
    x = np.concatenate([sol.u, sol.p])
    xr = np.concatenate([g["u"], g["p"]])
    rel = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    assert rel <= 1e-8, rel
    assert abs(sol.report.iterations - int(g["meta"][0])) <= 2, (sol.report.iterations, g["meta"])
    assert abs(sol.report.mean_inner_top - g["meta"][2]) < 0.2
    assert abs(sol.report.mean_inner_bottom - g["meta"][3]) < 0.2
    he, hr = sol.report.euclid_history, g["he"]
    m = min(len(he), len(hr))
    assert np.all(np.abs(he[:m] - hr[:m]) <= 1e-8 * hr[:m])
    assert sol.report.converged and sol.report.relres_e <= 1e-6
    b = np.concatenate([s.f, np.zeros(s.n_p)])
    true = np.linalg.norm(b - gs.apply(x)) / np.linalg.norm(b)
    assert abs(true - sol.report.relres_e) <= 1e-3 * sol.report.relres_e + 1e-12
    gs.close()


@pytest.mark.skipif(not __import__("os").environ.get("DSGPU_TEST_C5"),
                    reason="C5 at full size: ~12 min of host assembly/setup and ~100 GB host RAM; "
                           "set DSGPU_TEST_C5=1 (last recorded run: profiles/r02_c5_pin.md)")
def test_c5_full_size_vs_reference(gpu):
    """BASELINE config 5 (3D k'=2 96^3, 3.7M unknowns, nnz(K) 2.24e9 > 2^31) at
    full size against the reference's own solve of the identical system, run
    once on the GPU box's host (tests/golden/make_golden_c5.py; 1,077 s of
    MINRES on one core): outer iterations +-2, inner means, the Euclidean
    residual history, ||u|| and ||p||, a strided 4,096-entry sample of the
    solution, samples of one saddle apply and one IC(0) apply -- plus the
    size-independent properties (true residual = recurrence residual, the
    M^-1-norm history non-increasing) and the structural sizes of SURVEY.md §8(d)."""
    host, solver = gpu
    g = load_golden("c5_rand3d_k2_n96_full.npz")
    gb = load_golden("c5_rand3d_k2_n96_bounded.npz")
    s = host.assemble("random", 2, 96, dim=3, seed=42)
    assert [s.n_u, s.n_p, s.A.nnz, s.B.nnz, s.Q.nnz] == g["sizes"].tolist() == [
        2794764, 941192, 1432223760, 404794368, 113379904]
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    gs = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
    sample = g["sample"]
    rng = np.random.default_rng(int(g["probe_seed"][0]))
    xv = rng.uniform(-1.0, 1.0, s.n_u + s.n_p)
    rv = rng.uniform(-1.0, 1.0, s.n_u)
    ya = gs.apply(xv)[sample]
    assert np.linalg.norm(ya - g["apply_sample"]) <= 1e-13 * np.linalg.norm(g["apply_sample"])
    zi = gs.apply_ic0(0, rv)[sample[sample < s.n_u]]
    assert np.linalg.norm(zi - g["ic_sample"]) <= 1e-12 * np.linalg.norm(g["ic_sample"])
    for gold, mi in ((gb, 5), (g, 20000)):
        sol = gs.solve(options=solver.SolverOptions(outer_tol=1e-6, inner_tol=1e-1, max_iter=mi))
        r = sol.report
        x = np.concatenate([sol.u, sol.p])
        assert abs(r.iterations - int(gold["meta"][0])) <= 2
        assert abs(r.mean_inner_top - gold["meta"][2]) < 0.2 and abs(r.mean_inner_bottom - gold["meta"][3]) < 0.2
        he, hr = r.euclid_history, gold["he"]
        m = min(len(he), len(hr))
        assert np.all(np.abs(he[:m] - hr[:m]) <= 1e-8 * hr[:m])
        assert np.linalg.norm(x[sample] - gold["x_sample"]) <= 1e-8 * np.linalg.norm(gold["x_sample"])
        assert abs(np.linalg.norm(sol.u) - gold["norms"][0]) <= 1e-9 * gold["norms"][0]
        assert abs(np.linalg.norm(sol.p) - gold["norms"][1]) <= 1e-9 * gold["norms"][1]
    assert r.converged and r.relres_e <= 1e-6
    b = np.concatenate([s.f, np.zeros(s.n_p)])
    true = np.linalg.norm(b - gs.apply(x)) / np.linalg.norm(b)
    assert abs(true - r.relres_e) <= 1e-3 * r.relres_e
    hm = r.residual_history
    assert np.all(hm[1:] <= hm[:-1] * (1 + 1e-10))
    gs.close()


def vector_update_reference(n, launches):
    """numpy restatement of minres_update_row (solvers.cpp:93-101) on the
    probe's synthetic data (include/dsgpu.h, dsgpu_time_vector_update)."""
    i = np.arange(n)
    v, av = (i % 97) / 100.0, (i % 89) / 50.0 - 0.5
    w1, w2, aw1, aw2 = (i % 83) * 3e-3, (i % 79) * 4e-3, (i % 73) * 5e-3, (i % 71) * 6e-3
    res = (i % 61) * 8e-3 - 0.2
    oldeps, delta, gamma, phi = 0.25, 0.5, 1.5, 1e-3
    aw = ((av - oldeps * aw1) - delta * aw2) / gamma
    for _ in range(launches):
        res = res + (-phi) * aw
    return float(np.dot(res, res))


@pytest.mark.parametrize("n", [1, 1000, 300007])
def test_fused_vector_update_kernel(gpu, n):
    """The stand-alone fused MINRES vector pass (same device function as the
    persistent kernel) and its ||res||^2 reduction against numpy."""
    _, solver = gpu
    ms, res2 = solver.time_vector_update(n, reps=3)
    ref = vector_update_reference(n, 4)
    assert ms > 0.0
    assert abs(res2 - ref) <= 1e-12 * abs(ref)


def test_solve_from_reference_matrix_market_dump(gpu, port):
    """Drop-in path for a system the reference dumped (--dump-matrices,
    runner.cpp:223-229): A/B/Q read from its Matrix Market files, solved on the
    GPU, against the oracle on the same blocks."""
    import os
    from conftest import GOLDEN
    host, solver = gpu
    mm = os.path.join(GOLDEN, "mm")
    s = host.system_from_matrix_market(os.path.join(mm, "A_psi_k2_h3.mtx"), os.path.join(mm, "B_psi_k2_h3.mtx"),
                                       os.path.join(mm, "Q_psi_k2_h3.mtx"),
                                       np.load(os.path.join(mm, "f_psi_k2_h3.npy")))
    for strategy in ("IC0-PCG(A,Q)", "IC0-PCG(A)+Diag(Q)"):
        sol = solver.solve_stokes(s, strategy, solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
        check_parity(sol, reference_solve(port, s, strategy, 1e-8, 1e-1), 1e-8)


# ---- IC(0) factorization on the device -----------

def _same_csr(a, rp, ci, v):
    return (np.array_equal(a.row_ptr, rp) and np.array_equal(a.cols, ci)
            and np.array_equal(a.vals.view(np.int64), np.asarray(v).view(np.int64)))


def test_ic0_factor_gpu_bit_identical_to_reference_fixture(gpu):
    """The device factor of RCM(A) / RCM(Q_nu) equals the reference's own
    ic0 output stored in the golden fixture, bit for bit."""
    host, solver = gpu
    d = load_golden("c1_psi_k2_n8.npz")
    s = host.assemble("psi-mms", 2, 8)
    for m, tag in ((s.A, "A"), (s.Q_nu, "Q")):
        perm = host.rcm_permutation(m)
        L, info = solver.ic0_factor_gpu(host.permute_symmetric(m, perm))
        ref = golden_csr(d, "L_" + tag)
        assert _same_csr(L, ref.rp, ref.ci, ref.v), tag
        assert info["levels"] > 1


@pytest.mark.parametrize("flow", ["0", "1"])
@pytest.mark.parametrize("case,k,n,dim", [("psi-mms", 2, 64, 2), ("random", 3, 16, 2), ("cavity", 2, 16, 2),
                                          ("psi-mms", 2, 6, 3)])
def test_ic0_factor_gpu_bit_identical_to_host(gpu, monkeypatch, case, k, n, dim, flow):
    """Against the native host ic0 (itself bit-identical to the reference,
    tests/test_host.py) on BASELINE-shaped systems, 2D and 3D; flow = 1 runs
    the barrier-free dataflow kernel instead of level-scheduled launches."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_IC0_FLOW", flow)
    s = host.assemble(case, k, n, dim=dim, seed=1234)
    for m in (s.A, s.Q_nu):
        pm = host.permute_symmetric(m, host.rcm_permutation(m))
        L, _ = solver.ic0_factor_gpu(pm)
        H = host.ic0(pm)
        assert _same_csr(L, H.row_ptr, H.cols, H.vals)


@pytest.mark.parametrize("max_warps", ["4", "37", "101"])
def test_ic0_factor_gpu_dataflow_small_grids(gpu, monkeypatch, max_warps):
    """The dataflow schedule with few warps (each walks many rows; the cap is
    rounded down to whole CTAs so every warp owns a position map)."""
    host, solver = gpu
    monkeypatch.setenv("DSGPU_IC0_MAX_WARPS", max_warps)
    s = host.assemble("psi-mms", 2, 6, dim=3)
    for m in (s.A, s.Q_nu):
        pm = host.permute_symmetric(m, host.rcm_permutation(m))
        L, _ = solver.ic0_factor_gpu(pm)
        H = host.ic0(pm)
        assert _same_csr(L, H.row_ptr, H.cols, H.vals)


def test_ic0_factor_gpu_errors(gpu):
    """FactorBreakdown at the reference's first failing row; a structurally
    missing diagonal is std::invalid_argument (cholesky.cpp:109-111,128)."""
    host, solver = gpu
    d = np.array([[4.0, 1.0, 0.0, 0.0], [1.0, 4.0, 3.0, 0.0], [0.0, 3.0, 1.0, 1.0], [0.0, 0.0, 1.0, 4.0]])
    rows, cols = np.nonzero(d)
    rp = np.zeros(5, np.int64)
    np.cumsum(np.bincount(rows, minlength=4), out=rp[1:])
    m = host.CsrMatrix(4, 4, rp, cols.astype(np.int32), d[rows, cols])
    with pytest.raises(host.FactorBreakdown) as e_host:
        host.ic0(m)
    with pytest.raises(host.FactorBreakdown) as e_gpu:
        solver.ic0_factor_gpu(m)
    assert e_gpu.value.row == e_host.value.row == 2
    nodiag = host.CsrMatrix(2, 2, np.array([0, 1, 2], np.int64), np.array([0, 0], np.int32), np.array([1.0, 0.5]))
    with pytest.raises(ValueError, match="missing diagonal"):
        solver.ic0_factor_gpu(nodiag)


def test_solve_with_device_factor_matches_reference(gpu, port):
    """The whole preconditioner setup with the device factor feeds the same
    solve (prepare_block(ic0_on_gpu=True))."""
    host, solver = gpu
    s = host.assemble("psi-mms", 2, 16)
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    check_parity(sol, reference_solve(port, s, "IC0-PCG(A,Q)", 1e-8, 1e-1), 1e-8)
