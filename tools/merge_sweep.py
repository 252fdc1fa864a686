"""IC(0) apply time and solve time vs level-merge factor (DSGPU_MERGE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import PortLib, CSR
from paper_1309_5048_b200 import host, solver
P = PortLib()
k, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 64)
s = host.assemble("psi-mms", k, n)
c = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)
for M in (1, 2, 4, 8):
    os.environ["DSGPU_MERGE"] = str(M)
    t0 = time.time()
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    ts = time.time() - t0
    r = np.random.default_rng(0).standard_normal(s.n_u)
    z = g.apply_ic0(0, r)
    zr = P.ic0_solve(c(g.top.factor), r)
    err = np.abs(z - zr).max() / np.abs(zr).max()
    import ctypes as C
    cnt = np.zeros(32, np.int64)
    g.L.dsgpu_debug_counters.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
    g.L.dsgpu_debug_counters(1, cnt)
    ms = g.time_kernel(1, 10)
    g.L.dsgpu_debug_counters(1, cnt)
    G = max(cnt[2], 1)
    print(f"   main cycles/group {cnt[0]/G:.0f}, waiting {cnt[1]/G:.0f} (static {cnt[4]/G:.0f}), helper need-wait {cnt[5]/G:.0f} total {cnt[7]/G:.0f}, groups/sweep {cnt[2]/20:.0f}")
    print(f"   publish distance <=1/2-3/4-6/>=7: {cnt[8:12].tolist()}  start distance <=3/4-7/8-11/>=12: {cnt[12:16].tolist()}"
          f"  post-wait latency {cnt[16]/G:.0f}/group, last wait spun {cnt[17]/G:.2f}, co-main wait {cnt[18]/G:.0f}/group"
          f"  publication phases {(cnt[19:23]/G).round().tolist()}")
    print(f"   co-main: work after wait {cnt[23]/G:.0f}/group, publish distance <=0/1/2/>=3 {cnt[24:28].tolist()}, waits on psum {cnt[28]} on deps {cnt[29]}")
    out = []
    for itol in (1e-1, 1e-8):
        sol = g.solve(options=solver.SolverOptions(outer_tol=1e-8, inner_tol=itol), history=False)
        out.append((sol.report.iterations, round(sol.report.mean_inner_top, 3), round(sol.report.wall_seconds * 1e3, 2)))
    print(f"M={M}: setup {ts:.2f}s  IC apply {ms*1e3:.1f} us  maxrel {err:.1e}  solves (it, inner, ms) {out}", flush=True)
