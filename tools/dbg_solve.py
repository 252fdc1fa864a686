import os, sys, ctypes as C, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1309_5048_b200 import host, solver
s = host.assemble("psi-mms", 2, int(sys.argv[1]) if len(sys.argv) > 1 else 8)
g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
cnt = np.zeros(32, np.int64)
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
ph = np.zeros(8, np.int64)
g.L.dsgpu_debug_phases.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
g.L.dsgpu_debug_phases(1, ph)
sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1))
g.L.dsgpu_debug_phases(1, ph)
print("phases: kernel %.1f ms, CTA0 barrier-wait %.1f ms, CTA0 IC %.1f ms, CTA1 IC %.1f ms, CTA2 barrier-wait %.1f ms, barriers %d, solve %.1f ms" % (ph[4]/1.96e6, ph[0]/1.96e6, ph[1]/1.96e6, ph[5]/1.96e6, ph[2]/1.96e6, ph[3], sol.report.wall_seconds*1e3))
