"""Lab driver for tools/chain2_lab.cu (CTA-stepped block-inverse IC(0) apply).

python tools/chain2_lab.py [k n b_mult grid]
"""
import ctypes as C
import os
import subprocess
import sys
import time

import numpy as np
import scipy.linalg as sla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BLK = np.dtype([("s", "<i4"), ("e", "<i4"), ("c", "<i4"), ("v", "<i4"), ("dinv", "<i8"), ("dinvt", "<i8"),
                ("f", "<i8"), ("h", "<i8")])


def dense_rows(L, lo, hi, clo, chi):
    d = np.zeros((hi - lo, chi - clo))
    for i in range(lo, hi):
        s, e = L.row_ptr[i], L.row_ptr[i + 1]
        c = L.cols[s:e]
        m = (c >= clo) & (c < chi)
        d[i - lo, c[m] - clo] = L.vals[s:e][m]
    return d


def build(L, b, grid):
    n = L.n_rows
    starts = list(range(0, n, b)) + [n]
    nb = len(starts) - 1
    rowmin = np.array([L.cols[L.row_ptr[i]] for i in range(n)])
    blks = np.zeros(nb, dtype=BLK)
    parts = []
    off = 0

    def put(a):
        nonlocal off
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        o = off
        parts.append(a)
        off += len(a)
        return o

    for i in range(nb):
        s, e = starts[i], starts[i + 1]
        D = dense_rows(L, s, e, s, e)
        Dinv = sla.solve_triangular(D, np.eye(e - s), lower=True)
        c = min(int(rowmin[s:e].min()), s)
        F = Dinv @ dense_rows(L, s, e, c, s) if c < s else np.zeros((e - s, 0))
        below = np.nonzero(rowmin[e:] < e)[0]
        v = e + int(below.max()) + 1 if len(below) else e
        Hm = Dinv.T @ dense_rows(L, e, v, s, e).T if v > e else np.zeros((e - s, 0))
        blks[i] = (s, e, c, v, put(Dinv), put(Dinv.T), put(-F), put(-Hm))
    coef = np.concatenate(parts)
    # G/H row split: balanced by row length (~ b/2 avg), contiguous
    grow = np.linspace(0, n, grid + 1).round().astype(np.int32)
    return blks, coef, grow, nb


def main():
    k, n_el, bmul, grid = 2, 64, 1.0, 148
    if len(sys.argv) > 2:
        k, n_el = int(sys.argv[1]), int(sys.argv[2])
    if len(sys.argv) > 3:
        bmul = float(sys.argv[3])
    if len(sys.argv) > 4:
        grid = int(sys.argv[4])
    from paper_1309_5048_b200 import host
    from oracle import CSR, PortLib
    s = host.assemble("psi-mms" if k == 2 else "random", k, n_el)
    port = PortLib()
    so = os.path.join(ROOT, "tools", "libchain2lab.so")
    if not os.path.exists(so):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-shared", "-Xcompiler", "-fPIC", "-o", so,
                               os.path.join(ROOT, "tools", "chain2_lab.cu")])
    lib = C.CDLL(so)
    for name, M in (("A", s.A), ("Q", s.Q_nu)):
        p = host.rcm_permutation(M)
        L = host.ic0(host.permute_symmetric(M, p))
        n = L.n_rows
        rows = np.repeat(np.arange(n), np.diff(L.row_ptr))
        w = int((rows - L.cols).max())
        b = max(32, int(w * bmul))
        t0 = time.time()
        blks, coef, grow, nb = build(L, b, grid)
        tb = time.time() - t0
        r = np.random.default_rng(0).standard_normal(n)
        ref = port.ic0_solve(CSR(n, n, L.row_ptr, L.cols, L.vals), r)
        z = np.zeros(n)
        tl = np.zeros(1024, dtype=np.uint64)
        ms = C.c_double()
        rc = lib.chain2_run(C.c_int(n), C.c_int(nb), blks.ctypes.data_as(C.c_void_p), C.c_longlong(len(coef)),
                            coef.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                            grow.ctypes.data_as(C.c_void_p), C.c_int(grid), C.c_int(20),
                            z.ctypes.data_as(C.c_void_p), C.byref(ms), tl.ctypes.data_as(C.c_void_p))
        err = np.abs(z - ref).max() / np.abs(ref).max()
        print(f"{name}: n={n} w={w} b={b} steps={2 * nb} coef={len(coef) * 8 / 1e6:.1f} MB "
              f"build={tb:.1f}s rc={rc} apply={ms.value * 1e3:.1f} us  rel.err={err:.2e}", flush=True)
        for c in range(2):
            t = tl[c * 512: c * 512 + 4 + 4 * nb].astype(np.int64)
            t = t - t[0]
            # marks: start, G done, [stage, rows] x nb, H start (after sync), [stage, rows] x nb
            g = t[1]
            fw = t[2:2 + 2 * nb].reshape(nb, 2)
            h0 = t[2 + 2 * nb]
            bw = t[3 + 2 * nb: 3 + 4 * nb].reshape(nb, 2)
            print(f"  cta{'0' if c == 0 else '-1'}: G {g} ns | fwd stage-done " + " ".join(str(x) for x in fw[:, 0])
                  + f" | H done {h0} | bwd stage-done " + " ".join(str(x) for x in bw[:, 0]) + f" | end {bw[-1, 1]}")


if __name__ == "__main__":
    main()
