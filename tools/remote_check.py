"""Ring-mode sweeps with 0..R remote helper CTAs: correctness vs the oracle,
IC(0) apply time, main-warp counters, and a full solve."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import PortLib, CSR
from paper_1309_5048_b200 import host, solver
P = PortLib()
c = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)
cases = [("psi-mms", 2, 64, "1"), ("random", 3, 128, None)]
if len(sys.argv) > 1:
    cases = [(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), None)]
for (case, k, n, ringn) in cases:
    s = host.assemble(case, k, n, seed=1234)
    if ringn is None: os.environ.pop("DSGPU_RING_N", None)
    else: os.environ["DSGPU_RING_N"] = ringn
    r = np.random.default_rng(0).standard_normal(s.n_u)
    zr = None
    for R in [int(x) for x in os.environ.get('REMOTES', '0,4,16').split(',')]:
        os.environ["DSGPU_REMOTE"] = str(R)
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
        if zr is None: zr = P.ic0_solve(c(g.top.factor), r)
        z = g.apply_ic0(0, r)
        err = np.abs(z - zr).max() / np.abs(zr).max()
        cnt = np.zeros(32, np.int64)
        g.L.dsgpu_debug_counters.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
        g.L.dsgpu_debug_counters(1, cnt)
        ms = g.time_kernel(1, 5)
        g.L.dsgpu_debug_counters(1, cnt)
        sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1), history=False)
        print(f"{case} k={k} N={n} ring_n={ringn} R={R}: IC apply {ms*1e3:.0f} us maxrel {err:.1e} "
              f"main/group {cnt[0]/max(cnt[2],1):.0f} wait {cnt[1]/max(cnt[2],1):.0f} (static {cnt[4]/max(cnt[2],1):.0f}) "
              f"helper/group: need-wait {cnt[5]/max(cnt[2],1):.0f} remote-wait {cnt[6]/max(cnt[2],1):.0f} total {cnt[7]/max(cnt[2],1):.0f} abort {cnt[3]} | "
              f"solve it={sol.report.iterations} {sol.report.wall_seconds*1e3:.1f} ms grid {g.info()['grid_ctas']}",
              flush=True)
        del g
