"""Timeline of one partitioned-inverse IC(0) apply (dsgpu_debug_pi_trace):
standalone (block 0) and the first apply inside a C2 solve (both blocks).
python tools/pi_trace.py [k n]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1309_5048_b200 import host, solver  # noqa: E402


def show(L, tag):
    out = np.zeros(1024, np.int64)
    L.dsgpu_debug_pi_trace(0, out.ctypes.data_as(C.c_void_p))
    for slot in range(2):
        k = int(out[slot * 512])
        t = out[slot * 512 + 1: slot * 512 + 1 + k]
        if k == 0:
            continue
        d = np.diff(t)
        print(f"{tag} cta{'0' if slot == 0 else '-1'}: total {t[-1] - t[0]} ns; deltas " + " ".join(str(x) for x in d))


def main():
    k, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2, 64)
    s = host.assemble("psi-mms" if k == 2 else "random", k, n, seed=1234)
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    L = g.L
    L.dsgpu_debug_pi_trace.argtypes = [C.c_int, C.c_void_p]
    r = np.random.default_rng(0).standard_normal(s.n_u)
    g.apply_ic0(0, r)
    L.dsgpu_debug_pi_trace(1, None)
    g.apply_ic0(0, r)
    show(L, "standalone A")
    o = solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1)
    g.solve(options=o)
    L.dsgpu_debug_pi_trace(1, None)
    g.solve(options=o)
    show(L, "in-solve A+Q")


if __name__ == "__main__":
    main()
