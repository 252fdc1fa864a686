"""Lab driver for tools/chain_lab.cu: block-partitioned-inverse IC(0) apply.

python tools/chain_lab.py [k n b_mult grid]
Builds RCM + IC(0) of A for the 2D psi-MMS system, the block inverse data and
warp task lists, runs the chain kernel on the GPU, checks against the oracle.
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

TASK = np.dtype([("out", "<i4"), ("flags", "<i4"), ("jB", "<i4"), ("lB", "<i4"), ("jA", "<i4"),
                 ("lA", "<i4"), ("off", "<i8")])


def dense_rows(L, lo, hi, clo, chi):
    d = np.zeros((hi - lo, chi - clo))
    for i in range(lo, hi):
        s, e = L.row_ptr[i], L.row_ptr[i + 1]
        c = L.cols[s:e]
        m = (c >= clo) & (c < chi)
        d[i - lo, c[m] - clo] = L.vals[s:e][m]
    return d


R, G_, Y, H_, Z, NONE = 0, 1, 2, 3, 4, 7


def task(out_v, out, base_v, src_v, j, l, off, poll, chain=-1, dep=-1):
    return (out, out_v | (base_v << 3) | (src_v << 6) | (int(poll) << 9), j, l, chain, dep, off)


def build_tasks(L, b, n_warps, h_lag=1):
    """Task slots: G (g = Dinv r) slot 0; F_i slot 1 + i; H_i slot 2 + i + h_lag;
    B_i (descending) after the forward chain."""
    n = L.n_rows
    starts = list(range(0, n, b)) + [n]
    nb = len(starts) - 1
    rowmin = np.array([L.cols[L.row_ptr[i]] for i in range(n)])
    tasks, coefs = [], []
    off = 0
    slots = {}

    def add(slot, t, c):
        nonlocal off
        tasks.append(t)
        coefs.append(c)
        off += len(c)
        slots.setdefault(slot, []).append(len(tasks) - 1)

    dinvs = []
    for i in range(nb):
        s, e = starts[i], starts[i + 1]
        D = dense_rows(L, s, e, s, e)
        Dinv = sla.solve_triangular(D, np.eye(e - s), lower=True)
        dinvs.append(Dinv)
        for r in range(e - s):
            add(0, task(G_, s + r, NONE, R, s, r + 1, off, False), Dinv[r, : r + 1])
    for i in range(nb):
        s, e = starts[i], starts[i + 1]
        c = min(int(rowmin[s:e].min()), s)
        F = dinvs[i] @ dense_rows(L, s, e, c, s) if c < s else np.zeros((e - s, 0))
        for r in range(e - s):
            add(1 + i, task(Y, s + r, G_, Y, c, s - c, off, True, i, i - 1), -F[r])
        for r in range(e - s):
            add(2 + i + h_lag, task(H_, s + r, NONE, Y, s + r, e - s - r, off, True), dinvs[i].T[r, r:])
    base = 2 + nb + h_lag
    for k, i in enumerate(reversed(range(nb))):
        s, e = starts[i], starts[i + 1]
        below = np.nonzero(rowmin[e:] < e)[0]
        vend = e + int(below.max()) + 1 if len(below) else e
        H = dinvs[i].T @ dense_rows(L, e, vend, s, e).T if vend > e else np.zeros((e - s, 0))
        for r in range(e - s):
            add(base + k, task(Z, s + r, H_, Z, e, vend - e, off, True, nb + k, nb + k - 1), -H[r])
    # roles: per CTA the first CHAIN_W warps run the Y/Z chain, the others G/H
    per_warp = [[] for _ in range(n_warps)]
    cw = int(os.environ.get("CHAIN_W", "12"))
    chain_ws = [w for w in range(n_warps) if w % 15 < cw]
    bulk_ws = [w for w in range(n_warps) if w % 15 >= cw]
    kc = kb = 0
    all_ws = list(range(n_warps))
    ka = 0
    for sl in sorted(slots):
        for t in slots[sl]:
            kind = tasks[t][1] & 7
            if kind == G_ and os.environ.get("G_ALL", "1") == "1":
                per_warp[all_ws[ka % n_warps]].append(t)
                ka += 1
            elif kind in (Y, Z):
                per_warp[chain_ws[kc % len(chain_ws)]].append(t)
                kc += 1
            else:
                per_warp[bulk_ws[kb % len(bulk_ws)]].append(t)
                kb += 1
    order = [t for lst in per_warp for t in lst]
    wptr = np.zeros(n_warps + 1, dtype=np.int32)
    wptr[1:] = np.cumsum([len(l) for l in per_warp])
    T = np.array([tasks[t] for t in order], dtype=TASK)
    coef = np.concatenate(coefs)
    nc = 2 * nb
    total = np.zeros(nc, dtype=np.int32)
    quota = np.zeros((n_warps // 15, nc), dtype=np.int32)
    for w, lst in enumerate(per_warp):
        for t in lst:
            c = tasks[t][4]
            if c >= 0:
                total[c] += 1
                quota[w // 15, c] += 1
    return T, wptr, coef, nb, total, quota


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
    so = os.path.join(ROOT, "tools", "libchainlab.so")
    if not os.path.exists(so):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-shared", "-Xcompiler", "-fPIC", "-o", so,
                               os.path.join(ROOT, "tools", "chain_lab.cu")])
    lib = C.CDLL(so)
    for name, M in (("A", s.A), ("Q", s.Q_nu)):
        p = host.rcm_permutation(M)
        L = host.ic0(host.permute_symmetric(M, p))
        n = L.n_rows
        rows = np.repeat(np.arange(n), np.diff(L.row_ptr))
        w = int((rows - L.cols).max())
        b = max(32, int(w * bmul))
        t0 = time.time()
        T, wptr, coef, nb, total, quota = build_tasks(L, b, grid * 15)
        tb = time.time() - t0
        r = np.random.default_rng(0).standard_normal(n)
        ref = port.ic0_solve(CSR(n, n, L.row_ptr, L.cols, L.vals), r)
        z = np.zeros(n)
        trace = np.zeros(3 * len(T), dtype=np.uint64)
        ms = C.c_double()
        rc = lib.chain_run(C.c_int(n), C.c_int(len(T)), T.ctypes.data_as(C.c_void_p), C.c_int(grid * 15),
                           wptr.ctypes.data_as(C.c_void_p), C.c_longlong(len(coef)),
                           coef.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                           z.ctypes.data_as(C.c_void_p), C.c_int(grid), C.c_int(20), C.byref(ms),
                           trace.ctypes.data_as(C.c_void_p), C.c_int(len(total)),
                           total.ctypes.data_as(C.c_void_p), quota.ctypes.data_as(C.c_void_p))
        err = np.abs(z - ref).max() / np.abs(ref).max()
        print(f"{name}: n={n} w={w} b={b} steps={2 * nb} coef={len(coef) * 8 / 1e6:.1f} MB "
              f"build={tb:.1f}s rc={rc} apply={ms.value * 1e3:.1f} us  rel.err={err:.2e}", flush=True)
        tr = trace.reshape(-1, 3).astype(np.int64)
        tr -= tr[:, 0].min()
        kinds = (T["flags"] & 7)
        for kd, nm in ((1, "G"), (2, "Y"), (3, "H"), (4, "Z")):
            m = kinds == kd
            print(f"  {nm}: tasks {m.sum()} start {tr[m,0].min()}..{tr[m,0].max()} end {tr[m,2].min()}..{tr[m,2].max()} "
                  f"fetch+wait mean {np.mean(tr[m,1]-tr[m,0]):.0f} finish mean {np.mean(tr[m,2]-tr[m,1]):.0f}")
        for kd, nm in ((2, "Y"), (4, "Z")):
            m = kinds == kd
            outs = T["out"][m]
            t = tr[m]
            blocks = outs // b
            prev_end = None
            rows = []
            order = range(blocks.max() + 1) if kd == 2 else reversed(range(blocks.max() + 1))
            for i in order:
                q = t[blocks == i]
                if prev_end is not None:
                    late = np.maximum(q[:, 0] - prev_end, 0)
                    rows.append(f"blk{i}: end {q[:,2].max()} (+{q[:,2].max()-prev_end}) late-start max {late.max()} "
                                f"mean {late.mean():.0f}; ready-after-dep max {np.max(q[:,1]-np.maximum(q[:,0],prev_end))}")
                prev_end = q[:, 2].max()
            print(f"  {nm} chain: " + " | ".join(r.split(";")[0].split(" late")[0] for r in rows))


if __name__ == "__main__":
    main()
