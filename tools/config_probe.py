"""Solve BASELINE configs C3 / C4 on the GPU and record timings + parity.

  python tools/config_probe.py c3 [c4 ...]  [--modes=bs,legacy,1,0] [--ic0-gpu] [--check-ic0]

Per config and IC(0) apply mode (bs: blocked sweeps, the default; legacy: the
round-1 cost model; DSGPU_PI=1 partitioned inverse / 0 staged level sweeps): native assembly + host setup time, device setup time, two solves
(first = warm-up), outer iterations, inner means, kernel time, per-kernel
microbenchmarks, and — when tests/golden/<cfg>.npz exists — rel-L2 against the
reference's solution and the iteration difference. One JSON line per run.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFG = {
    # C3 stagnates near 4e-7 in the reference (variable relaxed preconditioner):
    # capped like tests/golden/make_golden_large.py
    "c3": dict(case="random", k=3, n=256, dim=2, seed=1234, outer=1e-8, inner=1e-1,
               golden="c3_rand_k3_n256.npz", max_iter=150),
    "c4": dict(case="psi-mms", k=2, n=32, dim=3, seed=0, outer=1e-8, inner=1e-1,
               golden="c4_psi3d_k2_n32.npz", max_iter=400),
    "c2": dict(case="psi-mms", k=2, n=64, dim=2, seed=0, outer=1e-8, inner=1e-1, golden=None),
    "c2x": dict(case="psi-mms", k=2, n=64, dim=2, seed=0, outer=1e-8, inner=1e-8, golden=None),
    "k3n128": dict(case="random", k=3, n=128, dim=2, seed=1234, outer=1e-8, inner=1e-1,
                   golden=None),
    "3d16": dict(case="psi-mms", k=2, n=16, dim=3, seed=0, outer=1e-8, inner=1e-1, golden=None),
    # C5 data (U[-1,1] seed 42, outer 1e-6) at growing 3D sizes, and C5 itself
    "c5_48": dict(case="random", k=2, n=48, dim=3, seed=42, outer=1e-6, inner=1e-1, golden=None),
    "c5_64": dict(case="random", k=2, n=64, dim=3, seed=42, outer=1e-6, inner=1e-1, golden=None),
    "c5": dict(case="random", k=2, n=96, dim=3, seed=42, outer=1e-6, inner=1e-1, golden=None),
}


T0 = time.time()


def log(msg):
    import resource
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
    print(f"[{time.time() - T0:7.1f}s rss {rss:6.1f} GB] {msg}", file=sys.stderr, flush=True)


def memguard(min_avail_gb: float):
    """Exit the process (not the box) before the host runs out of memory: poll
    MemAvailable and _exit(3) below the threshold (C5-size setups)."""
    import threading

    def watch():
        while True:
            with open("/proc/meminfo") as fh:
                for line in fh:
                    if line.startswith("MemAvailable:"):
                        avail = int(line.split()[1]) / 2**20
                        break
            if avail < min_avail_gb:
                log(f"memguard: MemAvailable {avail:.1f} GB < {min_avail_gb} GB, exiting")
                os._exit(3)
            time.sleep(0.1)

    threading.Thread(target=watch, daemon=True).start()


def main():
    if os.environ.get("PROBE_MEMGUARD_GB"):
        memguard(float(os.environ["PROBE_MEMGUARD_GB"]))
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    modes = ["bs"]
    for a in sys.argv[1:]:
        if a.startswith("--modes="):
            modes = a.split("=", 1)[1].split(",")
    from paper_1309_5048_b200 import host, solver
    for tag in args:
        c = CFG[tag]
        t0 = time.time()
        s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
        t_asm = time.time() - t0
        log(f"{tag}: assembled n_u={s.n_u} n_p={s.n_p}")
        t0 = time.time()
        ic0_gpu = "--ic0-gpu" in sys.argv  # factor on the device (dsgpu_ic0_factor, bit-identical)
        top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=ic0_gpu)
        bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=ic0_gpu)
        t_host = time.time() - t0
        log(f"{tag}: host setup (RCM, permute, IC0) {t_host:.1f}s")
        gold = None
        if c["golden"] and os.path.exists(os.path.join(ROOT, "tests", "golden", c["golden"])):
            gold = np.load(os.path.join(ROOT, "tests", "golden", c["golden"]))
        for mode in modes:
            os.environ.pop("DSGPU_PI", None)
            os.environ.pop("DSGPU_SWEEP", None)
            if mode in ("bs", "legacy"):
                os.environ["DSGPU_SWEEP"] = mode
            elif mode != "auto":
                os.environ["DSGPU_SWEEP"] = "legacy"
                os.environ["DSGPU_PI"] = mode
            out = dict(cfg=tag, pi=mode, n_u=s.n_u, n_p=s.n_p, assemble_s=round(t_asm, 2),
                       host_setup_s=round(t_host, 2), ic0_on_gpu=ic0_gpu)
            try:
                t0 = time.time()
                g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
                out["device_setup_s"] = round(time.time() - t0, 2)
                out["info"] = g.info()
                log(f"{tag} pi={mode}: device setup {out['device_setup_s']}s")
                if "--check-ic0" in sys.argv:  # one velocity apply against the CPU oracle
                    from oracle import CSR, PortLib
                    F = top.factor
                    rv = np.random.default_rng(5).uniform(-1.0, 1.0, F.n_rows)
                    zr = PortLib().ic0_solve(CSR(F.n_rows, F.n_cols, F.row_ptr, F.cols, F.vals), rv)
                    zg = g.apply_ic0(0, rv)
                    out["ic0_apply_rel"] = float(np.linalg.norm(zg - zr) / np.linalg.norm(zr))
                    log(f"{tag} {mode}: IC(0) apply rel {out['ic0_apply_rel']:.2e}")
                bs_cnt = np.zeros(16, np.int64)
                g.L.dsgpu_debug_bs_counters(1, bs_cnt.ctypes.data_as(__import__("ctypes").c_void_p))
                o = solver.SolverOptions(outer_tol=c["outer"], inner_tol=c["inner"],
                                         max_iter=c.get("max_iter", 20000))
                sol = g.solve(options=o)
                log(f"{tag} pi={mode}: first solve {sol.report.iterations} it "
                    f"{sol.report.wall_seconds:.3f}s relres {sol.report.relres_e:.2e}")
                t0 = time.time()
                sol = g.solve(options=o)
                out["wall_s"] = round(time.time() - t0, 4)
                r = sol.report
                out.update(iterations=r.iterations, converged=r.converged,
                           inner=[round(r.mean_inner_top, 3), round(r.mean_inner_bottom, 3)],
                           kernel_s=round(r.wall_seconds, 4),
                           iter_per_s=round(r.iterations / r.wall_seconds, 2),
                           relres_e=r.relres_e)
                x = np.concatenate([sol.u, sol.p])
                if os.environ.get("PROBE_SAVE"):
                    np.savez(os.path.join(os.environ["PROBE_SAVE"], f"{tag}_pi{mode}.npz"), x=x,
                             hm=r.residual_history, he=r.euclid_history)
                # true residual through the device saddle apply
                b = np.concatenate([s.f, np.zeros(s.n_p)])
                out["true_relres"] = float(np.linalg.norm(b - g.apply(x)) / np.linalg.norm(b))
                g.L.dsgpu_debug_bs_counters(1, bs_cnt.ctypes.data_as(__import__("ctypes").c_void_p))
                if bs_cnt.any():
                    out["bs_counters_solves"] = bs_cnt.tolist()
                for w, nm in [(0, "saddle_spmv"), (1, "ic0_A"), (2, "ic0_Q"), (3, "spmv_A")]:
                    out["us_" + nm] = round(g.time_kernel(w, 20) * 1e3, 2)
                    if w == 1:
                        g.L.dsgpu_debug_bs_counters(1, bs_cnt.ctypes.data_as(__import__("ctypes").c_void_p))
                        if bs_cnt.any():
                            out["bs_counters_21_applies_A"] = bs_cnt.tolist()
                if gold is not None:
                    xr = np.concatenate([gold["u"], gold["p"]])
                    out["relL2_vs_ref"] = float(np.linalg.norm(x - xr) / np.linalg.norm(xr))
                    out["ref_iterations"] = int(gold["meta"][0])
                    out["ref_inner"] = [round(float(gold["meta"][2]), 3),
                                        round(float(gold["meta"][3]), 3)]
                    out["ref_minres_s"] = round(float(gold["meta"][4]), 2)
                g.close()
            except Exception as e:  # record and continue with the next mode
                out["error"] = f"{type(e).__name__}: {e}"[:300]
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
