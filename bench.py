"""Benchmark: MINRES + IC(0) block-preconditioned Stokes solve on B200.

Headline workload (BASELINE.json configs[3], "C4"): 3D unit-cube Stokes, k'=2
divergence-conforming B-splines on 32^3 elements (153,748 unknowns, nnz(K) =
84.9M: 1.0 GB per saddle SpMV, HBM-resident), psi-MMS forcing, IC0-PCG(A,Q)
(RCM + IC(0) preconditioned inner CG on A and on Q_nu), outer 1e-8, inner
1e-1. One bench step = one solve. It is the largest BASELINE configuration
whose GPU arm AND bounded reference arm fit the default run's few minutes
(C5, 96^3, needs ~20 min of host assembly/setup: --workload c5). BASELINE
configs[1] (C2: 2D 64x64, the relaxed + exact-ish solve pair, L2-resident) is
measured in the same run and reported under "extra".

metric  : MINRES outer iterations per second (whole job, all ranks)
value   : device-resident solves (inputs already in HBM), CUDA-event time of
          the solve kernels
e2e     : the same solves through the C-ABI with HOST buffers (H2D of f and
          D2H of u, p inside the timed region), wall clock
roofline: dominant kernel = the persistent MINRES kernel; algorithmic bytes
          per SURVEY.md §8(d) with the counted inner iterations
--impl reference: the unmodified reference (oracle/_ref, built from
          /root/reference/proj/src) on the host CPU, same workload.
Multi-GPU (--gpus N under torchrun, one rank per GPU): the ranks solve ONE
row-partitioned system together (dsgpu_create_multi: halo gathers and
reduction mailboxes over NVLink peer memory, replicated sweeps; "strong"
scaling, max-over-ranks device time; NCCL carries the IPC-handle exchange,
the timing reduction and the assembly of the owned solution entries in the
e2e leg). --replicas runs N independent copies instead ("weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c2": dict(case="psi-mms", k=2, n=64, dim=2, seed=0, strategy="IC0-PCG(A,Q)",
               outer=1e-8, inners=(1e-1, 1e-8),
               label="C2: 2D k'=2 64x64 psi-MMS, IC0-PCG(A,Q), outer 1e-8, inner {1e-1, 1e-8}"),
    "c1": dict(case="psi-mms", k=2, n=16, dim=2, seed=0, strategy="IC0-PCG(A)+Diag(Q)",
               outer=1e-8, inners=(1e-1,),
               label="C1: 2D k'=2 16x16 psi-MMS, IC0-PCG(A)+Diag(Q), outer 1e-8, inner 1e-1"),
    # C3 stagnates near 4e-7 in the reference too (variable relaxed preconditioner):
    # capped at 150 outer iterations (tests/golden/make_golden_large.py)
    "c3": dict(case="random", k=3, n=256, dim=2, seed=1234, strategy="IC0-PCG(A,Q)",
               outer=1e-8, inners=(1e-1,), max_iter=150, cpu_max_iter=20,
               label="C3: 2D k'=3 256x256 U[-1,1] seed 1234, IC0-PCG(A,Q), outer 1e-8 (cap 150), "
                     "inner 1e-1"),
    "c4": dict(case="psi-mms", k=2, n=32, dim=3, seed=0, strategy="IC0-PCG(A,Q)",
               outer=1e-8, inners=(1e-1,), cpu_max_iter=12,
               label="C4: 3D k'=2 32^3 psi-MMS, IC0-PCG(A,Q), outer 1e-8, inner 1e-1"),
    # C5's data at 48^3 (the reference-pinned -m gpu test size) and C5 itself
    # (96^3: ~10 min of native assembly + ~5 min of setup before the first step)
    "c5_48": dict(case="random", k=2, n=48, dim=3, seed=42, strategy="IC0-PCG(A,Q)",
                  outer=1e-6, inners=(1e-1,), cpu_max_iter=4,
                  label="C5 data at 48^3: 3D k'=2 U[-1,1] seed 42, IC0-PCG(A,Q), outer 1e-6, inner 1e-1"),
    "c5": dict(case="random", k=2, n=96, dim=3, seed=42, strategy="IC0-PCG(A,Q)",
               outer=1e-6, inners=(1e-1,), cpu_max_iter=1,
               label="C5: 3D k'=2 96^3 U[-1,1] seed 42, IC0-PCG(A,Q), outer 1e-6, inner 1e-1"),
}
DEFAULT_WORKLOAD = "c4"
_SYSTEMS = {}  # workload tag -> assembled system (the GPU arm and the cpu_baseline leg share it)


def assembled(W):
    from paper_1309_5048_b200 import host
    key = (W["case"], W["k"], W["n"], W["dim"], W["seed"])
    if key not in _SYSTEMS:
        _SYSTEMS[key] = host.assemble(W["case"], W["k"], W["n"], dim=W["dim"], seed=W["seed"])
    return _SYSTEMS[key]
EXTRA_WORKLOADS = ("c2",)  # measured after the headline, reported under "extra"


def metric_for(workload: str) -> str:
    name = {"c2": "C2 solve pair", "c5_48": "C5-data 48^3 solve"}.get(workload, f"{workload.upper()} solve")
    return f"MINRES outer iterations/s (time-to-solution of the BASELINE {name})"


def workload_config(W) -> dict:
    """What the workload IS (identical in the GPU and the reference arm)."""
    return {"workload": W["label"], "case": W["case"], "dim": W["dim"], "k_prime": W["k"],
            "n_elem": W["n"], "strategy": W["strategy"], "outer_tol": W["outer"],
            "inner_tols": list(W["inners"]), "max_iter": W.get("max_iter", 20000)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(label: str, ic0_mode: str):
    """(DRAM bytes read + written by the dominant kernel per step, source) from
    the committed ncu capture of this workload AND this IC(0) apply mode
    (profiles/r02_minres_traffic*.json, written by tools/minres_profile.py with
    the commit it was captured on), else (None, None): ncu cannot run inside
    the timed bench, and a capture of another kernel variant is not this run's
    traffic."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_minres_traffic*.json"))):
        try:
            with open(path) as fh:
                t = json.load(fh)
            if t.get("workload") == label and t.get("ic0_mode") == ic0_mode:
                return float(t["dram_bytes_per_step"]), f"{os.path.basename(path)} @ {t.get('commit', '?')}"
        except Exception:
            continue
    return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
            sm = [float(r[0]) for r in rows]
            mx = max(float(r[1]) for r in rows)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = sorted({names[i] for r in rows for i in range(4)
                              if r[2 + i].strip().lower() in ("active", "1")})
            loaded = [s for s in sm if s > 0.5 * mx] or sm
            return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(sm)}
        except Exception as e:  # no nvidia-smi
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)[:80]}


def reduce_over_ranks(dist, device, ms: float, units: float):
    """Whole-job timing of one replica per rank: (max over ranks of the
    device-timed ms, sum over ranks of the units processed). With no process
    group (N = 1) the inputs pass through. Collective: every rank calls it."""
    if dist is None:
        return ms, units
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def algorithmic_bytes(info: dict, rep, outer_iters: int) -> float:
    """SURVEY.md §8(d) algorithmic bytes of one solve with the counted work:
    outer_iters saddle SpMVs + MINRES vector passes, and for each block
    apps x (IC apply + PCG init) + inner x (block SpMV + IC apply + PCG vectors)."""
    n_u, n_p = info["n_u"], info["n_p"]
    n = n_u + n_p
    S_K = 12 * info["nnz_K"] + 4 * n + 16 * n
    S_A = 12 * info["nnz_A"] + 20 * n_u
    S_ICA = 24 * info["nnz_L_A"] + 40 * n_u
    S_ICQ = 24 * info["nnz_L_Q"] + 40 * n_p
    S_Q = 12 * info["nnz_Q"] + 20 * n_p
    return (outer_iters * (S_K + 160 * n)
            + rep.apps_top * (S_ICA + 48 * n_u) + rep.inner_top * (S_A + S_ICA + 72 * n_u)
            + rep.apps_bottom * (S_ICQ + 48 * n_p) + rep.inner_bottom * (S_Q + S_ICQ + 72 * n_p))


def measure(tag, args, world, rank, local, dist, full: bool):
    """Device-timed and end-to-end runs of one workload; `full` adds the
    per-kernel microbenchmarks and the roofline of the headline workload."""
    import torch
    from paper_1309_5048_b200 import host, solver
    partitioned = world > 1 and not args.replicas  # one system across the ranks

    W = WORKLOADS[tag]
    t0 = time.perf_counter()
    s = assembled(W)
    assemble_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    tk, bk = solver.STRATEGIES[W["strategy"]]
    top = solver.prepare_block(s.A, tk, ic0_on_gpu=True)       # RCM, permute (host) + IC(0) (device)
    bot = solver.prepare_block(s.Q_nu, bk, ic0_on_gpu=True)
    precond_setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    fallback = None
    g = None
    if partitioned:
        os.environ["DSGPU_SWEEP"] = "bs"  # the multi-GPU data plane runs the replicated blocked sweeps
        err = ""
        try:
            g = solver.GpuStokesSolver(s, W["strategy"], device=local, top=top, bottom=bot, rank=rank,
                                       world=world, process_group=None)
        except Exception as e:  # e.g. no peer access between these GPUs
            err = f"{type(e).__name__}: {e}"[:160]
        ok = torch.tensor([0 if g is None else 1], device=torch.device("cuda", local))
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same branch
        if int(ok.item()) == 0:
            if g is not None:
                g.close()
                g = None
            partitioned = False
            fallback = "partitioned setup failed on a rank (" + (err or "another rank") + "): independent replicas"
            os.environ.pop("DSGPU_SWEEP", None)
    if g is None:
        g = solver.GpuStokesSolver(s, W["strategy"], device=local, top=top, bottom=bot)
    device_setup_s = time.perf_counter() - t0
    info = g.info()
    opts = [solver.SolverOptions(outer_tol=W["outer"], inner_tol=t,
                                 max_iter=W.get("max_iter", 20000)) for t in W["inners"]]
    dev = torch.device("cuda", local)
    d_f = torch.from_numpy(s.f).to(dev)
    d_u = torch.empty(s.n_u, dtype=torch.float64, device=dev)
    d_p = torch.empty(s.n_p, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_device():
        return [g.solve_device(d_f.data_ptr(), d_u.data_ptr(), d_p.data_ptr(), o) for o in opts]

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    dev_ms, iters, launches, last = 0.0, 0, 0, None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between steps (256 MiB write > 126 MB L2)
            torch.cuda.synchronize()
            reps = step_device()
            torch.cuda.synchronize()
            dev_ms += sum(r.wall_seconds for r in reps) * 1e3
            iters += sum(r.iterations for r in reps)
            launches += sum(r.gpu_launches for r in reps)
            last = reps
    # partitioned: every rank counts the same iterations of the one solve
    dev_ms, job_iters = reduce_over_ranks(dist, dev, dev_ms, iters if (not partitioned or rank == 0) else 0)
    if dist:
        dist.barrier()
    # ---- e2e: host buffers through the C ABI (pinned), wall clock ---------
    f_pin = torch.from_numpy(s.f.copy()).pin_memory()
    f_np = f_pin.numpy()
    e2e_s, e2e_iters = 0.0, 0
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for o in opts:
            sol = g.solve(f_np, o, history=False)
            e2e_iters += sol.report.iterations
        torch.cuda.synchronize()
        e2e_s += time.perf_counter() - t1
    e2e_ms, job_e2e_iters = reduce_over_ranks(dist, dev, e2e_s * 1e3,
                                              e2e_iters if (not partitioned or rank == 0) else 0)
    out = {
        "metric": metric_for(tag),
        "value": job_iters / (dev_ms * 1e-3),
        "unit": "iter/s",
        "ms_per_step": dev_ms / args.steps,
        "config": workload_config(W),
        "run": {"n_u": info["n_u"], "n_p": info["n_p"], "nnz_K": info["nnz_K"], "nnz_L_A": info["nnz_L_A"],
                "outer_iterations_per_step": iters // args.steps,
                "mean_inner_A": [round(r.mean_inner_top, 3) for r in last],
                "mean_inner_Q": [round(r.mean_inner_bottom, 3) for r in last],
                "time_to_solution_ms": [round(r.wall_seconds * 1e3, 3) for r in last],
                "converged": [bool(r.converged) for r in last],
                "setup_s": {"assemble_host": round(assemble_s, 2),
                            "rcm_permute_host_ic0_device": round(precond_setup_s, 2),
                            "plan_and_upload": round(device_setup_s, 2)},
                "time_to_solution_incl_precond_setup_s": round(
                    precond_setup_s + device_setup_s + sum(r.wall_seconds for r in last), 3),
                "grid_ctas": info["grid_ctas"], "ic0_apply": info["ic0_mode"],
                "far_ctas": [info["far_ctas_A"], info["far_ctas_Q"]],
                "l2": "flushed between steps (256 MiB write)", "parallelism": (f"one system row-partitioned over {world} GPUs" if partitioned
                                else f"replicas x{world}")},
        "e2e": {"value": job_e2e_iters / (e2e_ms * 1e-3), "unit": "iter/s",
                "h2d_bytes_per_step": 8 * s.n_u * len(opts),
                "d2h_bytes_per_step": 8 * (s.n_u + s.n_p) * len(opts)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    out["scaling"] = "strong" if partitioned else "weak"
    if fallback:
        out["run"]["multi_gpu_fallback"] = fallback
    if full:
        # ---- roofline of the dominant kernel (the persistent MINRES kernel) ----
        peak, peak_kind = measured_peak()
        if partitioned:
            peak *= world  # the one solve streams from every rank's HBM
        bytes_step = sum(algorithmic_bytes(info, r, r.iterations) for r in last)
        kern_ms = sum(r.wall_seconds for r in last) * 1e3
        achieved = bytes_step / (kern_ms * 1e-3) / 1e9
        traffic, traffic_src = measured_traffic(W["label"], info["ic0_mode"])
        out["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                           "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                           "peak_kind": peak_kind, "kernel": "minres_kernel (persistent, cooperative)",
                           "algorithmic_bytes_per_step": bytes_step}
        # per-kernel microbenchmarks on device-resident data (same launch path)
        try:
            if partitioned:
                raise RuntimeError("stand-alone kernels are timed in the single-GPU run")
            n = info["n_u"] + info["n_p"]
            spmv_ms, spmva_ms = g.time_kernel(0, 50), g.time_kernel(3, 50)
            ic_ms, icq_ms = g.time_kernel(1, 10), g.time_kernel(2, 10)
            ic_bytes = 24 * info["nnz_L_A"] + 40 * info["n_u"]
            out["kernels"] = {
                "saddle_spmv": {"ms": spmv_ms, "GB/s": (12 * info["nnz_K"] + 20 * n) / (spmv_ms * 1e-3) / 1e9},
                "A_spmv": {"ms": spmva_ms,
                           "GB/s": (12 * info["nnz_A"] + 20 * info["n_u"]) / (spmva_ms * 1e-3) / 1e9},
                "ic0_apply_A": {"ms": ic_ms, "GB/s": ic_bytes / (ic_ms * 1e-3) / 1e9,
                                "frac_of_peak": ic_bytes / (ic_ms * 1e-3) / 1e9 / peak,
                                "mode": info["ic0_mode"], "dependent_steps": info["ic0_steps_A"],
                                "us_per_step": ic_ms * 1e3 / max(1, info["ic0_steps_A"])},
                "ic0_apply_Q": {"ms": icq_ms},
            }
            # fused MINRES vector pass + ||res|| reduction, stand-alone at C5's n
            # (3,735,956 rows, 359 MB per pass: HBM-resident)
            n5 = 3735956
            vec_ms, _ = solver.time_vector_update(n5, reps=20, device=local)
            out["kernels"]["minres_vector_pass_c5_n"] = {"ms": vec_ms, "rows": n5,
                                                         "GB/s": 96.0 * n5 / (vec_ms * 1e-3) / 1e9}
        except Exception as e:
            out["kernels"] = {"error": str(e)[:100]}
    g.close()
    del g, top, bot, s, flush
    torch.cuda.empty_cache()
    return out


def run_ours(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    head = measure(args.workload, args, world, rank, local, dist, full=True)
    extra = {}
    if not args.no_extra and args.workload == DEFAULT_WORKLOAD and (world == 1 or args.replicas):
        for tag in EXTRA_WORKLOADS:
            e = measure(tag, args, world, rank, local, dist, full=False)
            extra[tag] = {k: e[k] for k in ("metric", "value", "unit", "ms_per_step", "config", "run", "e2e")}
    result = None
    if rank == 0:
        W = WORKLOADS[args.workload]
        cpu = cpu_baseline(args, W) if (world == 1 and not args.no_cpu_baseline) else None
        result = {
            "metric": head["metric"], "value": head["value"], "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE forcing / seeded RHS, native assembly; the 2D assembly is "
                    "bit-identical to the reference's, the 3D blocks follow the same rule)",
            "config": head["config"], "run": head["run"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "roofline": head["roofline"],
            "kernels": head["kernels"], "clocks": head["clocks"], "cpu_baseline": cpu, "extra": extra,
        }
        print(json.dumps(result), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


def cpu_runner(W):
    """run(inner_tol, max_iter) -> result dict of the reference solve of the
    workload on this host: oracle/_ref (the unmodified reference; its own
    assembly in 2D, the native 3D blocks through ref_from_csr since the
    reference has no 3D code) or, when it is not built, the C restatement. The
    reference's make_strategy (RCM, permute, IC(0): precond.cpp:161-193) runs
    once per inner tolerance and is reused by every timed solve."""
    from oracle import CSR, RefLib, ref_available
    from paper_1309_5048_b200 import host
    c = lambda m: CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)  # noqa: E731
    if ref_available():
        from oracle.oracle import RefPrecond
        R = RefLib()
        if W["dim"] == 2:
            rs = R.assemble(W["case"], W["k"], W["n"], seed=W["seed"])
        else:
            s = assembled(W)
            rs = R.from_csr(c(s.A), c(s.B), c(s.Q), s.f, nu=s.nu)
        if W["strategy"] not in ("IC0-PCG(A)+Diag(Q)",) and hasattr(R.L, "ref_precond_make"):
            pre = {}

            def run(t, mi):
                if t not in pre:
                    pre[t] = RefPrecond(rs, W["strategy"], t)
                return pre[t].solve(W["outer"], max_iter=mi)
            return run, "reference"
        return (lambda t, mi: rs.solve(W["strategy"], W["outer"], t, max_iter=mi)), "reference"
    from oracle import PortLib
    P = PortLib()
    s = assembled(W)
    return (lambda t, mi: P.solve_stokes(c(s.A), c(s.B), c(s.Bt), c(s.Q_nu), s.f, W["strategy"],
                                         W["outer"], t, max_iter=mi, Q_filter=c(s.Q))), "port"


def cpu_sample_note(W, reps):
    cap = W.get("cpu_max_iter")
    what = (f"the first {cap} outer iterations of each solve" if cap else
            f"the {len(W['inners'])}-solve step")
    return (f"{reps} x {what} (MINRES time only, preconditioner setup excluded; the reference "
            "solver is single-threaded)")


def cpu_baseline(args, W):
    """The reference (oracle/_ref) on this host's cores, bounded sample."""
    try:
        run, kind = cpu_runner(W)
        cap = W.get("cpu_max_iter", W.get("max_iter", 20000))
        iters, secs, reps = 0, 0.0, 0
        t_start = time.perf_counter()
        while reps < 3 and (reps == 0 or time.perf_counter() - t_start < args.cpu_budget_s):
            for t in W["inners"]:
                r = run(t, cap)
                iters += r["iterations"]
                secs += r["wall_seconds"]
            reps += 1
        return {"value": iters / secs, "unit": "iter/s", "cores": 1, "kind": kind,
                "sample": cpu_sample_note(W, reps)}
    except Exception as e:
        return {"value": None, "unit": "iter/s", "cores": 1, "kind": "reference",
                "sample": f"unavailable: {str(e)[:100]}"}


def run_reference(args, world, rank):
    if rank != 0:
        return None
    W = WORKLOADS[args.workload]
    run, kind = cpu_runner(W)
    cap = W.get("cpu_max_iter", W.get("max_iter", 20000))
    for _ in range(min(args.warmup, 1)):  # one warm-up solve builds the preconditioner
        for t in W["inners"]:
            run(t, cap)
    iters, secs = 0, 0.0
    for _ in range(args.steps):
        for t in W["inners"]:
            r = run(t, cap)
            iters += r["iterations"]
            secs += r["wall_seconds"]
    value = iters / secs
    out = {"impl": "reference", "metric": metric_for(args.workload), "value": value, "unit": "iter/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(W),
           "run": {"parallelism": "1 host core (serial reference)", "kind": kind},
           "cpu_baseline": {"value": value, "unit": "iter/s", "cores": 1, "kind": kind,
                            "sample": cpu_sample_note(W, args.steps)},
           "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas (weak scaling) instead of one partitioned solve")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
