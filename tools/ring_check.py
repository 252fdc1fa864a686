"""Ring-mode vs full-mode staged sweeps (forced with DSGPU_RING_N) and large systems."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import PortLib, CSR
from paper_1309_5048_b200 import host, solver
P = PortLib()
c = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)
for (case, k, n, ringn) in [("psi-mms", 2, 64, None), ("psi-mms", 2, 64, 1), ("random", 3, 128, None)]:
    if ringn is None: os.environ.pop("DSGPU_RING_N", None)
    else: os.environ["DSGPU_RING_N"] = str(ringn)
    s = host.assemble(case, k, n, seed=1234)
    t0 = time.time(); g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)"); ts = time.time() - t0
    r = np.random.default_rng(0).standard_normal(s.n_u)
    z = g.apply_ic0(0, r)
    zr = P.ic0_solve(c(g.top.factor), r)
    err = np.abs(z - zr).max() / np.abs(zr).max()
    ms = g.time_kernel(1, 5)
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1), history=False)
    print(f"{case} k={k} N={n} ring_n={ringn}: setup {ts:.1f}s IC apply {ms*1e3:.0f} us maxrel {err:.1e} levels {g.info()['levels_fwd_A']} solve it={sol.report.iterations} inner={sol.report.mean_inner_top:.2f}/{sol.report.mean_inner_bottom:.2f} {sol.report.wall_seconds*1e3:.1f} ms", flush=True)
