"""Determinism soak: the same solve N times on one handle and on a fresh handle; every result must be
bit-identical (the blocked sweeps fix the order of every sum; a race would show as a differing bit).
  python tools/soak.py c4 10"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from config_probe import CFG  # noqa: E402


def main():
    from paper_1309_5048_b200 import host, solver
    c = CFG[sys.argv[1]]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    s = host.assemble(c["case"], c["k"], c["n"], dim=c["dim"], seed=c["seed"])
    top = solver.prepare_block(s.A, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    bot = solver.prepare_block(s.Q_nu, solver.BLOCK_PCG_IC0, ic0_on_gpu=True)
    o = solver.SolverOptions(outer_tol=c["outer"], inner_tol=c["inner"], max_iter=c.get("max_iter", 20000))
    ref = None
    bad = 0
    for h in range(2):
        g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)", top=top, bottom=bot)
        for i in range(n):
            sol = g.solve(options=o)
            x = np.concatenate([sol.u, sol.p])
            if ref is None:
                ref = x
            same = np.array_equal(ref, x)
            bad += not same
            print(f"handle {h} solve {i}: it {sol.report.iterations} {sol.report.wall_seconds:.3f}s "
                  f"{'identical' if same else 'DIFFERS max ' + str(np.abs(ref - x).max())}", flush=True)
        g.close()
    print("soak", "ok" if bad == 0 else f"FAILED ({bad} differing results)")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
