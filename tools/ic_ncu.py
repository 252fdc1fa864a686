"""One velocity IC(0) apply of a config through the stand-alone apply kernel
(ic_apply_kernel for staged sweeps, pi_apply_kernel for the partitioned
inverse), preceded by one warm-up apply — for ncu -k regex:apply_kernel -s 1 -c 1.

  python tools/ic_ncu.py c4
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    c = CFG[sys.argv[1]]
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    r = np.random.default_rng(0).standard_normal(s.n_u)
    for _ in range(2):
        g.apply_ic0(0, r)
    print("info", g.info(), flush=True)
    g.close()


if __name__ == "__main__":
    main()
