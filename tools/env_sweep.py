"""A/B of run-time knobs on one config: assemble once, one solver per knob set.
  python tools/env_sweep.py c4 'DSGPU_BS_SLOTS=12' 'DSGPU_FAR_A=48' ...   (a bare '-' = defaults)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    c = CFG[sys.argv[1]]
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    o = solver.SolverOptions(outer_tol=c["outer"], inner_tol=c["inner"], max_iter=c.get("max_iter", 20000))
    for spec in sys.argv[2:]:
        kv = dict(x.split("=", 1) for x in spec.split(",") if "=" in x)
        for k, v in kv.items():
            os.environ[k] = v
        try:
            g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
            g.solve(options=o)
            best = min(g.solve(options=o).report.wall_seconds for _ in range(2))
            out = dict(knobs=spec, kernel_s=round(best, 4), us_ic0_A=round(g.time_kernel(1, 10) * 1e3, 1))
            g.close()
        except Exception as e:
            out = dict(knobs=spec, error=str(e)[:200])
        for k in kv:
            os.environ.pop(k, None)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
