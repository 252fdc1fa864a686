"""Pin BASELINE config 5 (3D k'=2 96^3, f_u ~ U[-1,1] seed 42, outer 1e-6, inner
1e-1) to the UNMODIFIED reference, at full size.

Runs on the GPU box (196 GB host, one B200), where the prebuilt
oracle/_ref/libdivstokes_ref.so travels with the repo snapshot:

  gpurun --timeout 6600 -- 'python tests/golden/make_golden_c5.py --n 96 \
      --out gpurun_out/c5_pin'

Stages (each writes its result before the next starts):
  1. native assembly of the 96^3 blocks (paper_1309_5048_b200.host);
  2. GPU: preconditioner setup (RCM, permute, device IC(0)), the full solve,
     a bounded solve (max_iter = K_BOUNDED), one saddle apply and one IC(0)
     apply of seeded vectors;
  3. reference: the same blocks through ref_from_csr; StokesSystem::apply
     (assembly.cpp:363-372) and Ic0Factor::solve (cholesky.cpp:136-152) of the
     same seeded vectors; make_strategy("IC0-PCG(A,Q)") once
     (precond.cpp:161-193), then solve_stokes (precond.cpp:245-290) bounded
     and full;
  4. the comparison (north_star bar: rel-L2 <= 1e-8, iterations +-2, final
     relres <= tol) and a compact golden: both residual histories, iteration
     counts, inner means, ||u||, ||p||, a strided sample of x, samples of the
     two kernel outputs.

--n 8 / 16 run the identical flow at small size (dry runs; --no-gpu skips
stage 2 on a CPU-only machine).
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

K_BOUNDED = 5
T0 = time.time()


def log(msg):
    import resource
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
    print(f"[{time.time() - T0:7.1f}s peak-rss {rss:6.1f} GB] {msg}", file=sys.stderr, flush=True)


def memguard(min_avail_gb):
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


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=96)
    ap.add_argument("--out", default="gpurun_out/c5_pin")
    ap.add_argument("--no-gpu", action="store_true")
    ap.add_argument("--ref-max-iter", type=int, default=200)
    ap.add_argument("--skip-full-ref", action="store_true")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    memguard(6.0)
    rec = dict(n_elem=a.n, case="random", seed=42, outer_tol=1e-6, inner_tol=1e-1,
               strategy="IC0-PCG(A,Q)", k_bounded=K_BOUNDED)

    def dump():
        with open(os.path.join(a.out, f"c5_pin_n{a.n}.json"), "w") as fh:
            json.dump(rec, fh, indent=1)

    from oracle import CSR, RefLib
    from oracle.oracle import RefPrecond
    from paper_1309_5048_b200 import host

    t0 = time.time()
    s = host.assemble("random", 2, a.n, dim=3, seed=42)
    rec["assemble_s"] = round(time.time() - t0, 1)
    rec["sizes"] = [s.n_u, s.n_p, s.A.nnz, s.B.nnz, s.Q.nnz]
    log(f"assembled n_u={s.n_u} n_p={s.n_p} nnzA={s.A.nnz}")
    n_u, n_p = s.n_u, s.n_p
    f = s.f.copy()
    cv = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)  # noqa: E731
    bt1 = cv(s.Bt).matvec(np.ones(n_p))
    filt = bool(np.abs(bt1).max() <= 1e-10 * np.abs(s.B.vals).max())
    one = np.ones(n_p)
    qk = cv(s.Q).matvec(one)
    rec["filter"] = filt
    rng = np.random.default_rng(96)
    xv = rng.uniform(-1.0, 1.0, n_u + n_p)     # saddle-apply probe
    rv = rng.uniform(-1.0, 1.0, n_u)           # IC(0)-apply probe (RCM ordering of A)
    sample = np.unique(np.linspace(0, n_u + n_p - 1, 4096).astype(np.int64))
    gpu = {}
    L_A = None
    if not a.no_gpu:
        from paper_1309_5048_b200 import solver
        t0 = time.time()
        top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
        bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
        rec["gpu_host_setup_s"] = round(time.time() - t0, 1)
        log(f"GPU-side preconditioner setup {rec['gpu_host_setup_s']} s")
        t0 = time.time()
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
        rec["gpu_device_setup_s"] = round(time.time() - t0, 1)
        rec["gpu_info"] = g.info()
        log(f"device setup {rec['gpu_device_setup_s']} s")
        for tag, mi in (("bounded", K_BOUNDED), ("full", 20000)):
            sol = g.solve(options=solver.SolverOptions(outer_tol=1e-6, inner_tol=1e-1, max_iter=mi))
            r = sol.report
            gpu[tag] = dict(x=np.concatenate([sol.u, sol.p]), hm=r.residual_history,
                            he=r.euclid_history)
            rec["gpu_" + tag] = dict(iterations=r.iterations, converged=r.converged,
                                     inner=[r.mean_inner_top, r.mean_inner_bottom],
                                     kernel_s=r.wall_seconds, relres_e=r.relres_e)
            log(f"GPU {tag}: {r.iterations} it, {r.wall_seconds:.2f} s, relres {r.relres_e:.3e}")
        b = np.concatenate([f, np.zeros(n_p)])
        rec["gpu_full"]["true_relres"] = float(
            np.linalg.norm(b - g.apply(gpu["full"]["x"])) / np.linalg.norm(b))
        gpu["apply_y"] = g.apply(xv)
        gpu["ic_z"] = g.apply_ic0(0, rv)
        g.close()
        L_A = top.factor
        del g, top, bot
        np.savez_compressed(os.path.join(a.out, f"c5_pin_gpu_n{a.n}.npz"),
                            he=gpu["full"]["he"], hm=gpu["full"]["hm"],
                            he_b=gpu["bounded"]["he"], x_sample=gpu["full"]["x"][sample],
                            sample=sample)
        dump()
    # ---- reference ---------------------------------------------------------
    R = RefLib()
    rs = R.from_csr(cv(s.A), cv(s.B), cv(s.Q), f, nu=s.nu)
    log("reference system built (ref_from_csr)")
    t0 = time.time()
    y_ref = rs.apply(xv)
    rec["ref_apply_s"] = round(time.time() - t0, 2)
    if L_A is None:  # --no-gpu: factor on the host (bit-identical to the reference's)
        pa = host.permute_symmetric(s.A, host.rcm_permutation(s.A))
        L_A = host.ic0(pa)
        del pa
    del s
    t0 = time.time()
    z_ref = R.ic0_solve(cv(L_A), rv)
    rec["ref_ic0_solve_s"] = round(time.time() - t0, 2)
    del L_A
    if gpu:
        rec["apply_relL2"] = rel(gpu["apply_y"], y_ref)
        rec["ic0_apply_relL2"] = rel(gpu["ic_z"], z_ref)
        log(f"saddle apply rel-L2 {rec['apply_relL2']:.2e}; IC(0) apply rel-L2 "
            f"{rec['ic0_apply_relL2']:.2e}")
    dump()
    pre = RefPrecond(rs, "IC0-PCG(A,Q)", 1e-1)
    rec["ref_setup_s"] = round(pre.setup_seconds, 1)
    log(f"reference make_strategy {pre.setup_seconds:.1f} s")
    runs = [("bounded", K_BOUNDED)] + ([] if a.skip_full_ref else [("full", a.ref_max_iter)])
    ref = {}
    for tag, mi in runs:
        res = pre.solve(1e-6, max_iter=mi)
        p = res["p"]
        if filt:  # precond.cpp:266-284 with k = ones (ref_from_csr carries no geometry pair)
            p = p - (qk @ p) / (qk @ one) * one
        x = np.concatenate([res["u"], p])
        ref[tag] = dict(x=x, he=res["euclid_history"], hm=res["residual_history"])
        rec["ref_" + tag] = dict(iterations=res["iterations"], converged=res["converged"],
                                 inner=[res["mean_inner_top"], res["mean_inner_bottom"]],
                                 minres_s=res["wall_seconds"], norm_u=float(np.linalg.norm(res["u"])),
                                 norm_p=float(np.linalg.norm(p)),
                                 relres_e=float(res["euclid_history"][-1]))
        log(f"reference {tag}: {res['iterations']} it, MINRES {res['wall_seconds']:.1f} s")
        if gpu:
            gx = gpu[tag]
            m = min(len(gx["he"]), len(res["euclid_history"]))
            rec["cmp_" + tag] = dict(
                relL2=rel(gx["x"], x),
                iter_diff=rec["gpu_" + tag]["iterations"] - res["iterations"],
                hist_max_rel=float(np.max(np.abs(gx["he"][:m] - res["euclid_history"][:m])
                                          / res["euclid_history"][:m])))
            log(f"parity {tag}: {rec['cmp_' + tag]}")
        np.savez_compressed(
            os.path.join(a.out, f"c5_rand3d_k2_n{a.n}_{tag}.npz"),
            he=res["euclid_history"], hm=res["residual_history"],
            meta=np.array([res["iterations"], res["converged"], res["mean_inner_top"],
                           res["mean_inner_bottom"], res["wall_seconds"], pre.setup_seconds]),
            norms=np.array([np.linalg.norm(res["u"]), np.linalg.norm(p)]),
            sample=sample, x_sample=x[sample], sizes=np.array(rec["sizes"], np.int64),
            apply_sample=y_ref[sample], ic_sample=z_ref[sample[sample < n_u]],
            probe_seed=np.array([96]))
        dump()
    pre.close()
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
