"""Host-side mirror of the reference's solver/preconditioner plugin API over the
B200 C-ABI (include/dsgpu.h).

Reference interface mirrored (proj/include/divstokes/precond.hpp):
  * ``strategy_names()`` / strategy menu        precond.cpp:154-193
  * ``SolverOptions``                           precond.hpp:52-59
  * ``SolveReport`` / ``StokesSolution``         solvers.hpp:15-23, precond.hpp:61-64
  * ``solve_stokes(system, strategy, options)``  precond.cpp:245-299

The setup is the one ``make_strategy`` performs for a PcgBlock with IC(0)
(precond.cpp:61-64): rcm_permutation -> permute_symmetric -> ic0, done by the
native host library (bit-identical to the reference), then uploaded once.
Everything inside the MINRES loop runs in one sm_100a cooperative kernel.
There is no CPU fallback: a missing libdsgpu.so or CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import host
from ._lib import load_gpu

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

BLOCK_JACOBI, BLOCK_PCG_JACOBI, BLOCK_PCG_IC0 = 0, 1, 2
STOP_PRECONDITIONED, STOP_EUCLIDEAN = 0, 1
DSGPU_OK, E_INDEFINITE, E_NEG_CURVATURE, E_BAD_INPUT, E_CUDA, E_NONPOS_DIAG, E_UNSUPPORTED = (
    0, 1, 2, 3, 4, 5, 7)
E_FACTOR_BREAKDOWN = 6
E_TIMEOUT = 8

# strategy -> (top block, bottom block); precond.cpp:161-193 plus the
# "IC0-PCG(A)+Diag(Q)" composition BASELINE config 1 asks for
STRATEGIES = {
    "PCG(A,Q)": (BLOCK_PCG_JACOBI, BLOCK_PCG_JACOBI),
    "PCG(A)+Diag(Q)": (BLOCK_PCG_JACOBI, BLOCK_JACOBI),
    "Diag(A,Q)": (BLOCK_JACOBI, BLOCK_JACOBI),
    "IC0-PCG(A,Q)": (BLOCK_PCG_IC0, BLOCK_PCG_IC0),
    "IC0-PCG(A)+Diag(Q)": (BLOCK_PCG_IC0, BLOCK_JACOBI),
}
# exact sparse-Cholesky blocks: out of scope on the GPU
UNSUPPORTED = ("Ideal(A,Q)", "Ideal(A)+Diag(Q)")


def strategy_names() -> list[str]:
    return list(STRATEGIES)


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_cols", C.c_int32), ("row_ptr", C.c_void_p),
                ("cols", C.c_void_p), ("vals", C.c_void_p)]


class _Opts(C.Structure):
    _fields_ = [("outer_tol", C.c_double), ("inner_tol", C.c_double), ("max_iter", C.c_int32),
                ("stop", C.c_int32), ("inner_cap", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("failed_block", C.c_int32), ("wall_seconds", C.c_double),
                ("mean_inner_top", C.c_double), ("mean_inner_bottom", C.c_double),
                ("relres_m", C.c_double), ("relres_e", C.c_double), ("inner_top", C.c_int64),
                ("apps_top", C.c_int64), ("inner_bottom", C.c_int64),
                ("apps_bottom", C.c_int64), ("hist_len", C.c_int32),
                ("gpu_launches", C.c_int32)]


def _lib():
    L = load_gpu()
    if not getattr(L, "_typed", False):
        vp, ip = C.c_void_p, C.c_int
        L.dsgpu_last_error.restype = C.c_char_p
        L.dsgpu_last_error.argtypes = [vp]
        L.dsgpu_create.argtypes = [ip, C.POINTER(vp)]
        L.dsgpu_destroy.argtypes = [vp]
        L.dsgpu_create_multi.argtypes = [ip, ip, ip, C.POINTER(vp)]
        L.dsgpu_multi_ipc_export.argtypes = [vp, vp]
        L.dsgpu_multi_ipc_import.argtypes = [vp, vp]
        L.dsgpu_debug_emulate_ranks.argtypes = [C.POINTER(vp), ip, _dp, C.POINTER(_Opts), _dp, _dp,
                                                C.POINTER(_Report)]
        L.dsgpu_setup.argtypes = [vp, C.POINTER(_Csr), C.POINTER(_Csr), C.POINTER(_Csr),
                                  C.POINTER(_Csr), ip, vp, C.POINTER(_Csr), ip, vp,
                                  C.POINTER(_Csr), C.POINTER(_Csr)]
        L.dsgpu_solve.argtypes = [vp, _dp, C.POINTER(_Opts), _dp, _dp, C.POINTER(_Report), vp, vp,
                                  C.c_int32]
        L.dsgpu_set_initial_guess.argtypes = [vp, vp, vp]
        L.dsgpu_solve_device.argtypes = [vp, vp, C.POINTER(_Opts), vp, vp, C.POINTER(_Report)]
        L.dsgpu_apply_saddle.argtypes = [vp, _dp, _dp]
        L.dsgpu_apply_ic0.argtypes = [vp, ip, _dp, _dp]
        L.dsgpu_apply_block_matrix.argtypes = [vp, ip, _dp, _dp]
        L.dsgpu_time_kernel.argtypes = [vp, ip, ip, C.POINTER(C.c_double)]
        L.dsgpu_time_vector_update.argtypes = [ip, C.c_int64, ip, C.POINTER(C.c_double),
                                               C.POINTER(C.c_double)]
        L.dsgpu_ic0_factor.argtypes = [ip, ip, _i64, _i32, _dp, _i64, _i32, _dp, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.dsgpu_ic0_last_error.restype = C.c_char_p
        L.dsgpu_info.argtypes = [vp, np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")]
        L._typed = True
    return L


def _csr(m: host.CsrMatrix) -> _Csr:
    return _Csr(m.n_rows, m.n_cols, m.row_ptr.ctypes.data, m.cols.ctypes.data,
                m.vals.ctypes.data)


@dataclass
class SolverOptions:
    """precond.hpp:52-59 (stop defaults to the Euclidean benchmark convention)."""

    outer_tol: float = 1e-12
    inner_tol: float = 1e-6
    max_iter: int = 20000
    stop: int = STOP_EUCLIDEAN
    inner_cap: int = 100000


@dataclass
class SolveReport:
    iterations: int = 0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    euclid_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    wall_seconds: float = 0.0
    mean_inner_top: float = 0.0
    mean_inner_bottom: float = 0.0
    relres_m: float = 1.0
    relres_e: float = 1.0
    inner_top: int = 0
    apps_top: int = 0
    inner_bottom: int = 0
    apps_bottom: int = 0
    gpu_launches: int = 0


@dataclass
class StokesSolution:
    u: np.ndarray
    p: np.ndarray
    report: SolveReport


class PreconditionerError(RuntimeError):
    """Indefinite preconditioner / negative curvature (reference std::runtime_error)."""


class DeviceTimeout(RuntimeError):
    """A device-side wait exceeded DSGPU_TIMEOUT_S; the solve was aborted."""


def _raise(code: int, msg: str):
    if code in (E_INDEFINITE, E_NEG_CURVATURE):
        raise PreconditionerError(msg)
    if code == E_TIMEOUT:
        raise DeviceTimeout(msg)
    if code == E_NONPOS_DIAG:
        raise ArithmeticError(msg)  # std::domain_error
    if code in (E_BAD_INPUT, E_UNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(msg)


@dataclass
class BlockSetup:
    kind: int
    perm: np.ndarray | None = None
    factor: host.CsrMatrix | None = None


def prepare_block(m: host.CsrMatrix, kind: int, ic0_on_gpu: bool = False) -> BlockSetup:
    """PcgBlock ctor, precond.cpp:59-73: for IC(0) blocks rcm -> permute -> ic0
    (ic0_on_gpu: the factor from ic0_factor_gpu, bit-identical)."""
    if kind != BLOCK_PCG_IC0:
        return BlockSetup(kind)
    perm = host.rcm_permutation(m)
    pm = host.permute_symmetric(m, perm)
    factor = ic0_factor_gpu(pm)[0] if ic0_on_gpu else host.ic0(pm)
    return BlockSetup(kind, perm, factor)


def ic0_factor_gpu(a: host.CsrMatrix, device: int = 0):
    """IC(0) factor of a symmetric CSR matrix on the device, bit-identical to
    the reference's ic0 (cholesky.cpp:84-134; dsgpu_ic0_factor). Returns
    (L, {"levels": DAG depth, "device_ms": level-launch time}). Raises
    host.FactorBreakdown (first failing row) or ValueError like host.ic0."""
    L = _lib()
    n = a.n_rows
    rows = np.repeat(np.arange(n), np.diff(a.row_ptr))
    lnnz = int(np.count_nonzero(a.cols <= rows))
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(max(lnnz, 1), np.int32)
    v = np.zeros(max(lnnz, 1))
    bad, lev, ms = C.c_int(-1), C.c_int(0), C.c_double(0.0)
    rc = L.dsgpu_ic0_factor(device, n, np.ascontiguousarray(a.row_ptr, np.int64),
                            np.ascontiguousarray(a.cols, np.int32), np.ascontiguousarray(a.vals, np.float64),
                            rp, ci, v, C.byref(bad), C.byref(lev), C.byref(ms))
    msg = L.dsgpu_ic0_last_error().decode()
    if rc == E_FACTOR_BREAKDOWN:
        raise host.FactorBreakdown(msg, bad.value)
    if rc in (E_BAD_INPUT, E_UNSUPPORTED):
        raise ValueError(msg)
    if rc:
        raise RuntimeError(f"dsgpu_ic0_factor failed ({rc}): {msg}")
    return (host.CsrMatrix(n, n, rp, ci[:lnnz].copy(), v[:lnnz].copy()),
            {"levels": lev.value, "device_ms": ms.value})


class GpuStokesSolver:
    """One device-resident system + preconditioner (the C-ABI handle)."""

    def __init__(self, system: host.StokesSystem, strategy: str = "IC0-PCG(A,Q)",
                 device: int = 0, top: BlockSetup | None = None,
                 bottom: BlockSetup | None = None, rank: int = 0, world: int = 1,
                 process_group=None, exchange: bool = True):
        """rank / world / process_group: one partitioned solve across the GPUs of
        one box (one process per GPU, torch.distributed group for the exchange of
        the CUDA IPC handles and of the owned solution entries); see dsgpu.h."""
        if strategy in UNSUPPORTED:
            raise ValueError(f"strategy {strategy} (exact Cholesky blocks) is not provided on GPU")
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown preconditioning strategy: {strategy}")
        self.L = _lib()
        self.system = system
        self.strategy = strategy
        tk, bk = STRATEGIES[strategy]
        self.top = top or prepare_block(system.A, tk)
        self.bottom = bottom or prepare_block(system.Q_nu, bk)
        h = C.c_void_p()
        self.rank, self.world, self.group = rank, world, process_group
        rc = (self.L.dsgpu_create_multi(rank, world, device, C.byref(h)) if world > 1
              else self.L.dsgpu_create(device, C.byref(h)))
        if rc:
            _raise(rc, self.L.dsgpu_last_error(None).decode())
        self.h = h
        s = system
        keep = [_csr(s.A), _csr(s.B), _csr(s.Bt), _csr(s.Q_nu)]
        la = _csr(self.top.factor) if self.top.factor is not None else None
        lq = _csr(self.bottom.factor) if self.bottom.factor is not None else None
        qf = _csr(s.Q) if s.has_constant_pressure_kernel else None
        pa = self.top.perm.ctypes.data if self.top.perm is not None else None
        pq = self.bottom.perm.ctypes.data if self.bottom.perm is not None else None
        rc = self.L.dsgpu_setup(h, C.byref(keep[0]), C.byref(keep[1]), C.byref(keep[2]),
                                C.byref(keep[3]), tk, pa, C.byref(la) if la else None, bk, pq,
                                C.byref(lq) if lq else None, C.byref(qf) if qf else None)
        if rc:
            msg = self.L.dsgpu_last_error(h).decode()
            self.close()
            _raise(rc, msg)
        if world > 1 and exchange:
            self._exchange_ipc_handles()

    def _exchange_ipc_handles(self):
        """All-gather the ranks' arena handles (64 bytes each) and map the peers."""
        import torch
        import torch.distributed as dist
        mine = np.zeros(64, np.uint8)
        rc = self.L.dsgpu_multi_ipc_export(self.h, mine.ctypes.data)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        t = torch.from_numpy(mine)
        cuda = dist.get_backend(self.group) == "nccl"
        if cuda:
            t = t.cuda()
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        allh = np.concatenate([p.cpu().numpy() for p in parts])
        rc = self.L.dsgpu_multi_ipc_import(self.h, allh.ctypes.data)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())

    def _sum_over_ranks(self, *arrays):
        """Owned entries -> full vectors (every rank returned zeros elsewhere)."""
        import torch
        import torch.distributed as dist
        cuda = dist.get_backend(self.group) == "nccl"
        for a in arrays:
            t = torch.from_numpy(a)
            tt = t.cuda() if cuda else t
            dist.all_reduce(tt, group=self.group)
            if cuda:
                t.copy_(tt.cpu())

    def close(self):
        if getattr(self, "h", None):
            self.L.dsgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _opts(self, o: SolverOptions) -> _Opts:
        return _Opts(o.outer_tol, o.inner_tol, o.max_iter, o.stop, o.inner_cap)

    def solve(self, f: np.ndarray | None = None, options: SolverOptions | None = None,
              history: bool = True, x0: tuple[np.ndarray, np.ndarray] | None = None) -> StokesSolution:
        """x0 = (u0, p0): MINRES initial guess (MinresOptions::x0, solvers.hpp:34)."""
        o = options or SolverOptions()
        s = self.system
        if x0 is not None:
            u0 = np.ascontiguousarray(x0[0], np.float64)
            p0 = np.ascontiguousarray(x0[1], np.float64)
            assert u0.shape == (s.n_u,) and p0.shape == (s.n_p,)
            rc = self.L.dsgpu_set_initial_guess(self.h, u0.ctypes.data, p0.ctypes.data)
            if rc:
                _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        f = np.ascontiguousarray(s.f if f is None else f, np.float64)
        u = np.zeros(s.n_u)
        p = np.zeros(s.n_p)
        rep = _Report()
        cap = o.max_iter + 1 if history else 0
        hm = np.zeros(max(cap, 1))
        he = np.zeros(max(cap, 1))
        opts = self._opts(o)
        rc = self.L.dsgpu_solve(self.h, f, C.byref(opts), u, p, C.byref(rep),
                                hm.ctypes.data if cap else None,
                                he.ctypes.data if cap else None, cap)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        if self.world > 1:
            self._sum_over_ranks(u, p)
        n = min(rep.hist_len, cap)
        r = SolveReport(rep.iterations, bool(rep.converged), hm[:n].copy(), he[:n].copy(),
                        rep.wall_seconds, rep.mean_inner_top, rep.mean_inner_bottom,
                        rep.relres_m, rep.relres_e, rep.inner_top, rep.apps_top,
                        rep.inner_bottom, rep.apps_bottom, rep.gpu_launches)
        return StokesSolution(u, p, r)

    def solve_device(self, d_f: int, d_u: int, d_p: int,
                     options: SolverOptions | None = None) -> SolveReport:
        """Device-pointer variant (torch tensors' data_ptr()); no H2D/D2H."""
        o = options or SolverOptions()
        rep = _Report()
        opts = self._opts(o)
        rc = self.L.dsgpu_solve_device(self.h, d_f, C.byref(opts), d_u, d_p, C.byref(rep))
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        return SolveReport(rep.iterations, bool(rep.converged), np.zeros(0), np.zeros(0),
                           rep.wall_seconds, rep.mean_inner_top, rep.mean_inner_bottom,
                           rep.relres_m, rep.relres_e, rep.inner_top, rep.apps_top,
                           rep.inner_bottom, rep.apps_bottom, rep.gpu_launches)

    # ---- kernel-level entry points ------------------------------------
    def apply(self, x: np.ndarray) -> np.ndarray:
        """StokesSystem::apply (assembly.cpp:363-372) on the device."""
        y = np.zeros(self.system.size)
        rc = self.L.dsgpu_apply_saddle(self.h, np.ascontiguousarray(x, np.float64), y)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        return y

    def apply_ic0(self, block: int, r: np.ndarray) -> np.ndarray:
        """Ic0Factor::solve (cholesky.cpp:136-152) in the block's RCM ordering."""
        z = np.zeros(len(r))
        rc = self.L.dsgpu_apply_ic0(self.h, block, np.ascontiguousarray(r, np.float64), z)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        return z

    def apply_block_matrix(self, block: int, x: np.ndarray) -> np.ndarray:
        y = np.zeros(len(x))
        rc = self.L.dsgpu_apply_block_matrix(self.h, block, np.ascontiguousarray(x, np.float64), y)
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        return y

    def time_kernel(self, which: int, reps: int = 20) -> float:
        ms = C.c_double()
        rc = self.L.dsgpu_time_kernel(self.h, which, reps, C.byref(ms))
        if rc:
            _raise(rc, self.L.dsgpu_last_error(self.h).decode())
        return ms.value

    def info(self) -> dict:
        a = np.zeros(16, np.int64)
        self.L.dsgpu_info(self.h, a)
        keys = ["n_u", "n_p", "nnz_K", "nnz_A", "nnz_L_A", "nnz_L_Q", "nnz_Q", "levels_fwd_A",
                "levels_bwd_A", "levels_fwd_Q", "levels_bwd_Q", "grid_ctas", "ic0_mode",
                "ic0_steps_A", "far_ctas_A", "far_ctas_Q"]
        d = dict(zip(keys, a.tolist()))
        d["ic0_mode"] = ("exact", "staged", "partitioned-inverse", "blocked")[d["ic0_mode"]]
        return d


def emulate_ranks(system: host.StokesSystem, strategy: str, world: int,
                  options: SolverOptions | None = None, device: int = 0,
                  top: BlockSetup | None = None, bottom: BlockSetup | None = None):
    """The multi-GPU solve of `world` ranks emulated on ONE GPU
    (dsgpu_debug_emulate_ranks: one cooperative launch, one CTA group per rank;
    set DSGPU_GRID so that world x grid fits the SM count). Returns
    (StokesSolution of rank 0's report, [SolveReport per rank])."""
    o = options or SolverOptions()
    tk, bk = STRATEGIES[strategy]
    top = top or prepare_block(system.A, tk)
    bottom = bottom or prepare_block(system.Q_nu, bk)
    ranks = [GpuStokesSolver(system, strategy, device, top, bottom, rank=r, world=world, exchange=False)
             for r in range(world)]
    try:
        L = ranks[0].L
        hs = (C.c_void_p * world)(*[g.h for g in ranks])
        reps = (_Report * world)()
        u, p = np.zeros(system.n_u), np.zeros(system.n_p)
        opts = ranks[0]._opts(o)
        rc = L.dsgpu_debug_emulate_ranks(hs, world, np.ascontiguousarray(system.f, np.float64), C.byref(opts),
                                         u, p, reps)
        if rc:
            _raise(rc, L.dsgpu_last_error(ranks[0].h).decode())
        out = [SolveReport(r.iterations, bool(r.converged), np.zeros(0), np.zeros(0), r.wall_seconds,
                           r.mean_inner_top, r.mean_inner_bottom, r.relres_m, r.relres_e, r.inner_top,
                           r.apps_top, r.inner_bottom, r.apps_bottom, r.gpu_launches) for r in reps]
        return StokesSolution(u, p, out[0]), out
    finally:
        for g in ranks:
            g.close()


def solve_stokes(system: host.StokesSystem, strategy: str,
                 options: SolverOptions | None = None, device: int = 0) -> StokesSolution:
    """Mirror of ``solve_stokes(system, strategy, options)`` (precond.cpp:295-299)."""
    o = options or SolverOptions()
    solver = GpuStokesSolver(system, strategy, device)
    try:
        return solver.solve(options=o)
    finally:
        solver.close()


__all__ = ["SolverOptions", "SolveReport", "StokesSolution", "GpuStokesSolver", "solve_stokes",
           "strategy_names", "STRATEGIES", "PreconditionerError", "prepare_block", "BlockSetup"]


def time_vector_update(n: int, reps: int = 20, device: int = 0):
    """Stand-alone roofline probe of the fused MINRES vector pass
    (dsgpu_time_vector_update): (mean ms per launch, ||res||^2 after 1 + reps
    launches). 96 bytes per row per launch."""
    L = _lib()
    ms, res2 = C.c_double(0.0), C.c_double(0.0)
    rc = L.dsgpu_time_vector_update(device, n, reps, C.byref(ms), C.byref(res2))
    if rc != 0:
        raise RuntimeError(f"dsgpu_time_vector_update failed ({rc}): {L.dsgpu_last_error(None).decode()}")
    return ms.value, res2.value
