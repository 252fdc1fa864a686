"""GPU check of the partitioned-inverse IC(0) mode on BASELINE C2 (and optional
other sizes): IC(0) apply parity vs the oracle, apply timing, and the full C2
solves (relaxed / exact-ish inner CG) against the oracle, PI on vs off.

python tools/pi_check.py [k n case]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import CSR, PortLib  # noqa: E402
from paper_1309_5048_b200 import host, solver  # noqa: E402


def main():
    k, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 64)
    case = sys.argv[3] if len(sys.argv) > 3 else ("psi-mms" if k == 2 else "random")
    s = host.assemble(case, k, n, seed=1234)
    port = PortLib()
    c = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)  # noqa: E731
    t0 = time.time()
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    print(f"setup {time.time() - t0:.2f}s info {g.info()}", flush=True)
    for blk, fac in ((0, g.top.factor), (1, g.bottom.factor)):
        r = np.random.default_rng(5).standard_normal(fac.n_rows)
        z = g.apply_ic0(blk, r)
        ref = port.ic0_solve(c(fac), r)
        print(f"block {blk}: IC apply rel err {np.abs(z - ref).max() / np.abs(ref).max():.2e}, "
              f"{g.time_kernel(1 + blk, 50) * 1e3:.1f} us/apply", flush=True)
    for inner in (1e-1, 1e-8):
        o = solver.SolverOptions(outer_tol=1e-8, inner_tol=inner)
        sol = g.solve(options=o)
        sol = g.solve(options=o)
        ref = port.solve_stokes(c(s.A), c(s.B), c(s.Bt), c(s.Q_nu), s.f, "IC0-PCG(A,Q)", 1e-8, inner,
                                Q_filter=c(s.Q))
        x = np.concatenate([sol.u, sol.p])
        xr = np.concatenate([ref["u"], ref["p"]])
        rel = np.linalg.norm(x - xr) / np.linalg.norm(xr)
        r = sol.report
        print(f"inner {inner:g}: iters {r.iterations} (oracle {ref['iterations']}), rel L2 {rel:.2e}, "
              f"relres {r.relres_e:.2e}, mean inner {r.mean_inner_top:.2f}/{r.mean_inner_bottom:.2f} "
              f"(oracle {ref['mean_inner_top']:.2f}/{ref['mean_inner_bottom']:.2f}), "
              f"solve {r.wall_seconds * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
