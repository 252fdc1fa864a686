import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1309_5048_b200 import host, solver
case, k, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = host.assemble(case, k, n, seed=1234)
g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
cnt = np.zeros(32, np.int64)
g.L.dsgpu_debug_counters.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
g.apply_ic0(0, np.ones(s.n_u))
g.L.dsgpu_debug_counters(1, cnt)
ms = g.time_kernel(1, 4)
g.L.dsgpu_debug_counters(1, cnt)
print(f"{case} k={k} N={n}: IC apply {ms*1e3:.0f} us, groups/sweep {cnt[2]/10:.0f}, main cycles/group {cnt[0]/cnt[2]:.0f}, waiting {cnt[1]/cnt[2]:.0f}, info {g.info()}", flush=True)
