import os, sys, ctypes as C, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1309_5048_b200 import host, solver
s = host.assemble("psi-mms", 2, int(sys.argv[1]) if len(sys.argv) > 1 else 8)
g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
cnt = np.zeros(4, np.int64)
g.L.dsgpu_debug_counters.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
g.L.dsgpu_debug_counters(1, cnt)
print("ic", g.time_kernel(1, 2), flush=True)
g.L.dsgpu_debug_counters(1, cnt); print("after ic", cnt, flush=True)
try:
    sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
    print("solve", sol.report.iterations, sol.report.converged, flush=True)
except Exception as e:
    print("ERR", e, flush=True)
g.L.dsgpu_debug_counters(1, cnt); print("after solve", cnt, flush=True)
