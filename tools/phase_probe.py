"""In-kernel phase table of one solve (diag build: make -C paper_1309_5048_b200/csrc diag;
DSGPU_LIB_DIR=paper_1309_5048_b200/lib_diag python tools/phase_probe.py c4 [c3 ...]).

Per workload: cycles of the persistent kernel (worker CTA 0), of its grid-barrier
waits, of the two IC(0) servers' applies, and the blocked sweeps' own counters
(main-warp cycles per group and what it waited for; co-main and far-worker
waits). One JSON line per workload. The counters exist only in the diag build;
the production kernels carry none."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    for tag in sys.argv[1:]:
        c = CFG[tag]
        s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
        o = solver.SolverOptions(outer_tol=c["outer"], inner_tol=c["inner"], max_iter=c.get("max_iter", 20000))
        g.solve(options=o)  # warm-up
        ph, bs, sp = np.zeros(8, np.int64), np.zeros(16, np.int64), np.zeros(8, np.int64)
        vp = C.c_void_p
        g.L.dsgpu_debug_phases(1, ph.ctypes.data_as(vp))
        g.L.dsgpu_debug_bs_counters(1, bs.ctypes.data_as(vp))
        g.L.dsgpu_debug_spmv_phases(1, sp.ctypes.data_as(vp))
        sol = g.solve(options=o)
        g.L.dsgpu_debug_phases(1, ph.ctypes.data_as(vp))
        g.L.dsgpu_debug_bs_counters(1, bs.ctypes.data_as(vp))
        g.L.dsgpu_debug_spmv_phases(1, sp.ctypes.data_as(vp))
        r = sol.report
        k = float(ph[4]) or 1.0
        out = dict(cfg=tag, ic0_mode=g.info()["ic0_mode"], iterations=r.iterations, kernel_ms=round(r.wall_seconds * 1e3, 2),
                   applies_A=int(r.apps_top + r.inner_top), applies_Q=int(r.apps_bottom + r.inner_bottom),
                   kernel_cycles=int(ph[4]), grid_barriers=int(ph[3]),
                   frac_cta0_barrier_wait=round(ph[0] / k, 4), frac_cta2_barrier_wait=round(ph[2] / k, 4),
                   frac_server_A_busy=round(ph[1] / k, 4), frac_server_Q_busy=round(ph[5] / k, 4))
        # SpMV phases inside the persistent kernel (worker CTA 0's clock; 12 bytes per stored
        # entry = int32 column + f64 value; cycles -> ns through kernel_ms / kernel_cycles)
        info = g.info()
        ns = r.wall_seconds * 1e9 / k
        for name, j, nnz in (("saddle_spmv_M1", 0, info["nnz_K"]), ("A_spmv_L1", 4, info["nnz_A"])):
            if sp[j + 1]:
                own = sp[j] / sp[j + 1] * ns
                thru = sp[j + 3] / sp[j + 1] * ns
                out[name] = dict(phases=int(sp[j + 1]), cta0_entries=int(sp[j + 2]), cta0_own_us=round(own / 1e3, 2),
                                 cta0_GBps=round(sp[j + 2] * 12 / own, 2),
                                 ctas_sharing_rows=round(nnz / max(1, int(sp[j + 2])), 1),
                                 GBps_own=round(nnz * 12 / own, 1),
                                 through_barrier_us=round(thru / 1e3, 2), GBps_through_barrier=round(nnz * 12 / thru, 1))
        if bs[4]:
            G = float(bs[4])
            out["bsweep"] = dict(groups=int(bs[4]), main_cycles_per_group=round(bs[0] / G, 1),
                                 main_wait_c=round(bs[1] / G, 1), main_wait_slots=round(bs[2] / G, 1),
                                 main_wait_publisher=round(bs[3] / G, 1),
                                 comain_cycles_per_group=round(bs[7] / G, 1),
                                 comain_wait_progress=round(bs[5] / G, 1), comain_wait_far=round(bs[6] / G, 1),
                                 far_worker_wait_frac=round(bs[8] / max(1.0, float(bs[9])), 4),
                                 main_wait_q=round(bs[14] / G, 1), main2_wait_y=round(bs[15] / G, 1),
                                 comain_stage_cycles=dict(prefetch_and_staging_wait=round(bs[10] / G, 1),
                                                          mid_lists_incl_waits=round(bs[11] / G, 1),
                                                          t_product=round(bs[12] / G, 1),
                                                          hand_off=round(bs[13] / G, 1)))
        print(json.dumps(out), flush=True)
        g.close()


if __name__ == "__main__":
    main()
