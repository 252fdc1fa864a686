"""IC(0) apply time of one config under setup knobs (env read by dsgpu_setup).

  python tools/knob_sweep.py c4 "DSGPU_PI=0" "DSGPU_PI=0 DSGPU_REMOTE=16" ... [--solve]

--solve adds, per knob set, two whole solves (the second timed: kernel time,
iterations) and the persistent kernel's phase counters of the timed one.

One host assembly + RCM/IC(0); then per knob set a fresh device handle and
time_kernel of the velocity (1) and pressure (2) IC(0) applies, plus the sweep
diagnostics counters of one velocity apply. One JSON line per knob set.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402

KNOBS = ("DSGPU_PI", "DSGPU_PI_B", "DSGPU_REMOTE", "DSGPU_MERGE", "DSGPU_HSLEEP", "DSGPU_FLOWD",
         "DSGPU_GRID", "DSGPU_NOWAIT", "DSGPU_RING_N", "DSGPU_PI_G", "DSGPU_PI_DIRECT")


def main():
    from paper_1309_5048_b200 import host, solver
    do_solve = "--solve" in sys.argv
    argv = [a for a in sys.argv if a != "--solve"]
    tag = argv[1]
    c = CFG[tag]
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0)
    r = np.random.default_rng(0).standard_normal(s.n_u)
    z_ref = None
    for spec in argv[2:]:
        for k in KNOBS:
            os.environ.pop(k, None)
        for kv in spec.split():
            k, v = kv.split("=")
            os.environ[k] = v
        out = dict(cfg=tag, knobs=spec)
        try:
            t0 = time.time()
            g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
            out["setup_s"] = round(time.time() - t0, 2)
            z = g.apply_ic0(0, r)
            if z_ref is None:
                z_ref = z
            out["z_rel_diff"] = float(np.linalg.norm(z - z_ref) / np.linalg.norm(z_ref))
            cnt = np.zeros(32, np.int64)
            g.L.dsgpu_debug_counters.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
            g.L.dsgpu_debug_counters(1, cnt)
            g.apply_ic0(0, r)
            g.L.dsgpu_debug_counters(1, cnt)
            out["counters"] = cnt.tolist()
            out["us_ic0_A"] = round(g.time_kernel(1, 10) * 1e3, 1)
            out["us_ic0_Q"] = round(g.time_kernel(2, 10) * 1e3, 1)
            if do_solve:
                o = solver.SolverOptions(outer_tol=c["outer"], inner_tol=c["inner"],
                                         max_iter=c.get("max_iter", 20000))
                g.solve(options=o)
                ph = np.zeros(8, np.int64)
                g.L.dsgpu_debug_phases.argtypes = [C.c_int, np.ctypeslib.ndpointer(dtype=np.int64)]
                g.L.dsgpu_debug_phases(1, ph)
                sol = g.solve(options=o)
                g.L.dsgpu_debug_phases(1, ph)
                rep = sol.report
                out.update(iterations=rep.iterations, converged=rep.converged,
                           kernel_s=round(rep.wall_seconds, 4),
                           inner=[round(rep.mean_inner_top, 3), round(rep.mean_inner_bottom, 3)],
                           relres_e=rep.relres_e,
                           phases_ms=dict(kernel=round(ph[4] / 1.965e6, 2), cta0_barrier=round(ph[0] / 1.965e6, 2),
                                          cta0_ic=round(ph[1] / 1.965e6, 2), cta1_ic=round(ph[5] / 1.965e6, 2),
                                          cta2_barrier=round(ph[2] / 1.965e6, 2), barriers=int(ph[3])))
            g.close()
        except Exception as e:
            out["error"] = f"{type(e).__name__}: {e}"[:300]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
