"""Drive one bench step (the C2 solve pair) for ncu captures of the persistent
MINRES kernel: 1 warm-up step, then the profiled step (launches 3 and 4 with
--launch-skip 2 --launch-count 2 -k regex:minres_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1309_5048_b200 import host, solver

W = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
s = host.assemble(W["case"], W["k"], W["n"], dim=W["dim"], seed=W["seed"])
g = solver.GpuStokesSolver(s, W["strategy"])
opts = [solver.SolverOptions(outer_tol=W["outer"], inner_tol=t, max_iter=W.get("max_iter", 20000))
        for t in W["inners"]]
for step in range(2):
    for o in opts:
        sol = g.solve(s.f, o, history=False)
        print(f"step {step} inner {o.inner_tol:g}: it={sol.report.iterations} "
              f"{sol.report.wall_seconds * 1e3:.2f} ms", flush=True)
