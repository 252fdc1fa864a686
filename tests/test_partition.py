"""Multi-GPU data plane, host side (paper_1309_5048_b200/csrc/gpu/partition.cpp;
SURVEY.md §8(e)): the contiguous row partition of the saddle operator, its
halo index sets, and the partitioned SpMV / dot-product pipeline, checked on
the CPU — the partitioned product against the full product (bit for bit: a
row's entries keep their order), and one preconditioned MINRES iteration
(solvers.cpp:63-105) run by two gloo ranks on their slices against the
single-rank iteration."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def saddle_csr(s):
    """K = [A Bt; B 0] row by row, A's entries first in the velocity rows (the
    layout of the device operator K')."""
    n_u, n_p = s.n_u, s.n_p
    la, lb = np.diff(s.A.row_ptr), np.diff(s.Bt.row_ptr)
    rp = np.zeros(n_u + n_p + 1, np.int64)
    rp[1:n_u + 1] = np.cumsum(la + lb)
    rp[n_u + 1:] = rp[n_u] + np.cumsum(np.diff(s.B.row_ptr))
    ci = np.zeros(rp[-1], np.int32)
    v = np.zeros(rp[-1])
    for i in range(n_u):
        a0, a1 = s.A.row_ptr[i], s.A.row_ptr[i + 1]
        b0, b1 = s.Bt.row_ptr[i], s.Bt.row_ptr[i + 1]
        o = rp[i]
        ci[o:o + a1 - a0] = s.A.cols[a0:a1]
        v[o:o + a1 - a0] = s.A.vals[a0:a1]
        o += a1 - a0
        ci[o:o + b1 - b0] = s.Bt.cols[b0:b1] + n_u
        v[o:o + b1 - b0] = s.Bt.vals[b0:b1]
    ci[rp[n_u]:] = s.B.cols
    v[rp[n_u]:] = s.B.vals
    return rp, ci, v, la.astype(np.int32)


def hook():
    from paper_1309_5048_b200._lib import load_gpu
    L = load_gpu()
    L.dsgpu_debug_partition_spmv.argtypes = [C.c_int, C.c_int, _i64, _i32, _dp, _i32, C.c_int, _i32, _i64,
                                             _dp, _dp]
    return L.dsgpu_debug_partition_spmv


def partition(rp, ci, v, na, n_u, world, x):
    n = len(rp) - 1
    bounds = np.zeros(2 * (world + 1), np.int32)
    halo = np.zeros(world * world, np.int64)
    y = np.zeros(n)
    rc = hook()(n, n_u, rp, ci, v, na, world, bounds, halo, np.ascontiguousarray(x), y)
    assert rc == 0
    return bounds[:world + 1], bounds[world + 1:], halo.reshape(world, world), y


def full_spmv(rp, ci, v, x):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    y = np.zeros(len(rp) - 1)
    # same left-to-right accumulation as the device row loop
    for i in range(len(rp) - 1):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc += v[k] * x[ci[k]]
        y[i] = acc
    del rows
    return y


@pytest.mark.parametrize("case,k,n,dim", [("psi-mms", 2, 16, 2), ("random", 2, 4, 3)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partitioned_spmv_equals_full(case, k, n, dim, world):
    from paper_1309_5048_b200 import host
    s = host.assemble(case, k, n, dim=dim, seed=42)
    rp, ci, v, na = saddle_csr(s)
    x = np.random.default_rng(1).uniform(-1, 1, s.n_u + s.n_p)
    ub, pb, halo, y = partition(rp, ci, v, na, s.n_u, world, x)
    assert np.array_equal(y.view(np.int64), full_spmv(rp, ci, v, x).view(np.int64))
    # contiguous, complete, balanced by nonzeros within 2x of the mean
    assert ub[0] == 0 and ub[-1] == s.n_u and np.all(np.diff(ub) >= 0)
    assert pb[0] == 0 and pb[-1] == s.n_p and np.all(np.diff(pb) >= 0)
    if world > 1:
        nnz_u = np.array([rp[ub[r + 1]] - rp[ub[r]] for r in range(world)])
        assert nnz_u.max() <= 2.0 * nnz_u.mean() + rp[1:].max()
        assert np.all(np.diag(halo) == 0)  # nobody reads its own slice as halo
        assert halo.sum() > 0


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _minres_iteration(K_apply, dots, b, dinv, its):
    """its preconditioned MINRES iterations (solvers.cpp:36-105) with a Jacobi
    preconditioner on vectors whose dot products go through `dots`; returns x."""
    x = np.zeros_like(b)
    r1 = b.copy()
    y = dinv * r1
    beta1 = np.sqrt(dots(r1, y))
    r2 = r1.copy()
    oldb, beta, dbar, epsln, phibar = 0.0, beta1, 0.0, 0.0, beta1
    cs, sn = -1.0, 0.0
    w = np.zeros_like(b)
    w2 = np.zeros_like(b)
    for it in range(1, its + 1):
        v = y / beta
        y = K_apply(v)
        if it >= 2:
            y = y - (beta / oldb) * r1
        alfa = dots(v, y)
        y = y - (alfa / beta) * r2
        r1, r2 = r2, y
        y = dinv * r2
        oldb = beta
        beta = np.sqrt(dots(r2, y))
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        gamma = max(np.sqrt(gbar * gbar + beta * beta), 2.220446049250313e-16)
        cs, sn = gbar / gamma, beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1, w2 = w2, w
        w = (v - oldeps * w1 - delta * w2) / gamma
        x = x + phi * w
    return x


def _worker(rank, world, port, out):
    import scipy.sparse as sp
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1309_5048_b200 import host
    s = host.assemble("psi-mms", 2, 8)
    rp, ci, v, na = saddle_csr(s)
    n, n_u = s.n_u + s.n_p, s.n_u
    ub, pb, _, _ = partition(rp, ci, v, na, n_u, world, np.zeros(n))
    own = np.concatenate([np.arange(ub[rank], ub[rank + 1]), n_u + np.arange(pb[rank], pb[rank + 1])])
    K = sp.csr_matrix((v, ci, rp), shape=(n, n))
    K_own = K[own]                       # this rank's rows
    d = np.abs(K.diagonal())
    d[d == 0.0] = 1.0
    b = np.concatenate([s.f, np.zeros(s.n_p)])
    owners = [np.concatenate([np.arange(ub[r], ub[r + 1]), n_u + np.arange(pb[r], pb[r + 1])])
              for r in range(world)]

    def apply_own(v_own):                # halo exchange: every rank publishes its slice
        parts = [None] * world
        dist.all_gather_object(parts, v_own)
        full = np.zeros(n)
        for r in range(world):
            full[owners[r]] = parts[r]
        return K_own @ full

    def dots(a, c):                      # partial + all-reduce
        t = torch.tensor([float(a @ c)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    x_own = _minres_iteration(apply_own, dots, b[own], 1.0 / d[own], 5)
    parts = [None] * world
    dist.all_gather_object(parts, x_own)
    if rank == 0:
        x = np.zeros(n)
        for r in range(world):
            x[owners[r]] = parts[r]
        xs = _minres_iteration(lambda q: K @ q, lambda a, c: float(a @ c), b, 1.0 / d, 5)
        out["rel"] = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_minres_iterations_gloo_world2():
    import torch.multiprocessing as mp
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        rel = out["rel"]
    assert rel <= 1e-12, rel
