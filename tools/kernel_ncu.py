"""Launch the stand-alone hot kernels of one config once each (for ncu).

  ncu ... python tools/kernel_ncu.py c4

Saddle SpMV (spmv_kernel over K), block-A SpMV (spmv_kernel, A part of K's
velocity rows), and one velocity IC(0) apply (ic_apply_kernel / pi_apply_kernel).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    c = CFG[sys.argv[1]]
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    for which in (0, 3, 1):
        print(which, g.time_kernel(which, 1), flush=True)
    g.close()


if __name__ == "__main__":
    main()
