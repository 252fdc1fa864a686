"""Drive the standalone IC(0) apply kernel on BASELINE C2 (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1309_5048_b200 import host, solver
k, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 64)
s = host.assemble("psi-mms", k, n)
g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
r = np.random.default_rng(0).standard_normal(s.n_u)
for _ in range(3):
    z = g.apply_ic0(0, r)
print("ic apply ms", g.time_kernel(1, 10), "info", g.info())
