"""TEST INFRASTRUCTURE — ctypes bindings to oracle/_ref/*.so (see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_SO = os.path.join(REF_DIR, "libdivstokes_ref.so")
PORT_SO = os.path.join(REF_DIR, "libdsoracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

STRATEGIES = ("PCG(A,Q)", "PCG(A)+Diag(Q)", "Diag(A,Q)", "IC0-PCG(A,Q)", "IC0-PCG(A)+Diag(Q)")
# block kinds per strategy (top, bottom): 0 Jacobi, 1 Jacobi-PCG, 2 IC0-PCG
STRATEGY_BLOCKS = {
    "PCG(A,Q)": (1, 1),
    "PCG(A)+Diag(Q)": (1, 0),
    "Diag(A,Q)": (0, 0),
    "IC0-PCG(A,Q)": (2, 2),
    "IC0-PCG(A)+Diag(Q)": (2, 0),
}
CASES = {"psi-mms": 0, "cavity": 1, "square": 2, "random": 3}


@dataclass
class CSR:
    n_rows: int
    n_cols: int
    rp: np.ndarray  # int64
    ci: np.ndarray  # int32
    v: np.ndarray  # float64

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            s, e = self.rp[i], self.rp[i + 1]
            d[i, self.ci[s:e]] = self.v[s:e]
        return d

    def matvec(self, x: np.ndarray) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.rp))
        return np.bincount(rows, weights=self.v * x[self.ci], minlength=self.n_rows)

    @staticmethod
    def from_dense(d: np.ndarray) -> "CSR":
        d = np.asarray(d, dtype=np.float64)
        rp = [0]
        ci, v = [], []
        for i in range(d.shape[0]):
            nz = np.nonzero(d[i])[0]
            ci.extend(nz.tolist())
            v.extend(d[i, nz].tolist())
            rp.append(len(ci))
        return CSR(d.shape[0], d.shape[1], np.array(rp, np.int64), np.array(ci, np.int32),
                   np.array(v, np.float64))


def build(quiet: bool = True) -> None:
    """Build oracle/_ref (C restatement always; reference when present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefLib:
    """The unmodified reference (oracle/_ref/libdivstokes_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_assemble.restype = C.c_void_p
        L.ref_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_ulonglong,
                                   C.c_char_p, C.c_int]
        L.ref_from_csr.restype = C.c_void_p
        L.ref_from_csr.argtypes = [C.c_int, C.c_int, _i64p, _i32p, _dp, _i64p, _i32p, _dp,
                                   _i64p, _i32p, _dp, C.c_double, _dp]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _i64p]
        L.ref_export.argtypes = [C.c_void_p, C.c_int, _i64p, _i32p, _dp]
        L.ref_rhs.argtypes = [C.c_void_p, _dp]
        L.ref_set_rhs.argtypes = [C.c_void_p, _dp]
        L.ref_apply.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_force_scalar.argtypes = [C.c_int]
        L.ref_force_scalar.restype = C.c_int
        L.ref_solve.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double, C.c_int,
                                C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_char_p, C.c_int]
        L.ref_spmv.argtypes = [C.c_int, C.c_int, _i64p, _i32p, _dp, _dp, _dp]
        if hasattr(L, "ref_precond_make"):
            L.ref_precond_make.restype = C.c_void_p
            L.ref_precond_make.argtypes = [C.c_void_p, C.c_char_p, C.c_double,
                                           C.POINTER(C.c_double), C.c_char_p, C.c_int]
            L.ref_precond_free.argtypes = [C.c_void_p]
            L.ref_solve_with.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int,
                                         C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_char_p,
                                         C.c_int]
        L.ref_rcm.argtypes = [C.c_int, _i64p, _i32p, _i32p, C.c_char_p, C.c_int]
        L.ref_write_mm.argtypes = [C.c_int, C.c_int, _i64p, _i32p, _dp, C.c_char_p, C.c_int,
                                   C.c_char_p, C.c_int]
        L.ref_read_mm.restype = C.c_void_p
        L.ref_read_mm.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int64), C.c_char_p, C.c_int]
        L.ref_mm_take.argtypes = [C.c_void_p, _i64p, _i32p, _dp]
        L.ref_bandwidth.argtypes = [C.c_int, _i64p, _i32p]
        L.ref_bandwidth.restype = C.c_int
        L.ref_permute.argtypes = [C.c_int, _i64p, _i32p, _dp, _i32p, _i64p, _i32p, _dp,
                                  C.c_char_p, C.c_int]
        L.ref_ic0.argtypes = [C.c_int, _i64p, _i32p, _dp, _i64p, _i32p, _dp,
                              C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_ic0_solve.argtypes = [C.c_int, _i64p, _i32p, _dp, _dp, _dp]
        L.ref_pcg_csr.argtypes = [C.c_int, _i64p, _i32p, _dp, _dp, C.c_int, C.c_double,
                                  C.c_int, _dp, _dp, C.c_char_p, C.c_int]
        L.ref_minres_csr.argtypes = [C.c_int, _i64p, _i32p, _dp, _dp, C.c_int, C.c_double,
                                     C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_int,
                                     C.c_char_p, C.c_int]

    # -- systems ---------------------------------------------------------
    def assemble(self, case: str, k_prime: int, n_elem: int, nu: float = 1.0,
                 seed: int = 0) -> "RefSystem":
        err = C.create_string_buffer(512)
        h = self.L.ref_assemble(CASES[case], k_prime, n_elem, nu, seed, err, 512)
        if not h:
            raise RuntimeError(err.value.decode())
        return RefSystem(self, h)

    def from_csr(self, A: CSR, B: CSR, Q: CSR, f: np.ndarray, nu: float = 1.0) -> "RefSystem":
        h = self.L.ref_from_csr(A.n_rows, B.n_rows, A.rp, A.ci, A.v, B.rp, B.ci, B.v, Q.rp,
                                Q.ci, Q.v, nu, np.ascontiguousarray(f, np.float64))
        return RefSystem(self, h)

    def force_scalar(self, on: bool) -> int:
        return self.L.ref_force_scalar(1 if on else 0)

    # -- primitives ------------------------------------------------------
    def spmv(self, A: CSR, x: np.ndarray) -> np.ndarray:
        y = np.zeros(A.n_rows)
        self.L.ref_spmv(A.n_rows, A.n_cols, A.rp, A.ci, A.v, np.ascontiguousarray(x), y)
        return y

    def rcm(self, A: CSR) -> np.ndarray:
        perm = np.zeros(A.n_rows, np.int32)
        err = C.create_string_buffer(256)
        rc = self.L.ref_rcm(A.n_rows, A.rp, A.ci, perm, err, 256)
        if rc:
            raise ValueError(err.value.decode())
        return perm

    def write_matrix_market(self, A: CSR, path: str, symmetric: bool = False) -> None:
        """The reference's write_matrix_market (csr.cpp:126-142)."""
        err = C.create_string_buffer(256)
        rc = self.L.ref_write_mm(A.n_rows, A.n_cols, A.rp, A.ci, A.v, path.encode(), int(symmetric),
                                 err, 256)
        if rc:
            raise RuntimeError(err.value.decode())

    def read_matrix_market(self, path: str) -> CSR:
        """The reference's read_matrix_market (csr.cpp:144-175)."""
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int64()
        err = C.create_string_buffer(256)
        h = self.L.ref_read_mm(path.encode(), C.byref(nr), C.byref(nc), C.byref(nnz), err, 256)
        if not h:
            raise RuntimeError(err.value.decode())
        rp = np.zeros(nr.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int32)
        v = np.zeros(nnz.value)
        self.L.ref_mm_take(h, rp, ci, v)
        return CSR(nr.value, nc.value, rp, ci, v)

    def bandwidth(self, A: CSR) -> int:
        return self.L.ref_bandwidth(A.n_rows, A.rp, A.ci)

    def permute(self, A: CSR, perm: np.ndarray) -> CSR:
        rp = np.zeros(A.n_rows + 1, np.int64)
        ci = np.zeros(A.nnz, np.int32)
        v = np.zeros(A.nnz)
        err = C.create_string_buffer(256)
        rc = self.L.ref_permute(A.n_rows, A.rp, A.ci, A.v, np.ascontiguousarray(perm, np.int32),
                                rp, ci, v, err, 256)
        if rc:
            raise ValueError(err.value.decode())
        return CSR(A.n_rows, A.n_cols, rp, ci, v)

    def ic0(self, A: CSR) -> CSR:
        rows = np.repeat(np.arange(A.n_rows), np.diff(A.rp))
        lnnz = int(np.count_nonzero(A.ci <= rows))
        rp = np.zeros(A.n_rows + 1, np.int64)
        ci = np.zeros(lnnz, np.int32)
        v = np.zeros(lnnz)
        bad = C.c_int(-1)
        err = C.create_string_buffer(256)
        rc = self.L.ref_ic0(A.n_rows, A.rp, A.ci, A.v, rp, ci, v, C.byref(bad), err, 256)
        if rc:
            e = RuntimeError(err.value.decode())
            e.row = bad.value  # type: ignore[attr-defined]
            e.code = rc  # type: ignore[attr-defined]
            raise e
        return CSR(A.n_rows, A.n_cols, rp, ci, v)

    def ic0_solve(self, L: CSR, r: np.ndarray) -> np.ndarray:
        z = np.zeros(L.n_rows)
        self.L.ref_ic0_solve(L.n_rows, L.rp, L.ci, L.v, np.ascontiguousarray(r), z)
        return z

    def pcg(self, A: CSR, b: np.ndarray, pre_kind: int, tol: float, max_iter: int):
        x = np.zeros(A.n_rows)
        rep = np.zeros(3)
        err = C.create_string_buffer(256)
        rc = self.L.ref_pcg_csr(A.n_rows, A.rp, A.ci, A.v, np.ascontiguousarray(b), pre_kind,
                                tol, max_iter, x, rep, err, 256)
        if rc:
            raise RuntimeError(err.value.decode())
        return x, int(rep[0]), bool(rep[1])

    def minres(self, A: CSR, b: np.ndarray, pre_kind: int, tol: float, max_iter: int,
               euclid: bool = False):
        x = np.zeros(A.n_rows)
        rep = np.zeros(3)
        hm = np.zeros(max_iter + 1)
        he = np.zeros(max_iter + 1)
        err = C.create_string_buffer(256)
        rc = self.L.ref_minres_csr(A.n_rows, A.rp, A.ci, A.v, np.ascontiguousarray(b), pre_kind,
                                   tol, max_iter, int(euclid), x, rep, hm, he, max_iter + 1,
                                   err, 256)
        if rc:
            raise RuntimeError(err.value.decode())
        n = int(rep[2])
        return x, int(rep[0]), bool(rep[1]), hm[:n], he[:n]


class RefSystem:
    def __init__(self, lib: RefLib, handle: int):
        self.lib, self.h = lib, handle
        nu_, np_ = C.c_int(), C.c_int()
        nnz = np.zeros(5, np.int64)
        lib.L.ref_dims(C.c_void_p(handle), C.byref(nu_), C.byref(np_), nnz)
        self.n_u, self.n_p = nu_.value, np_.value
        self._nnz = nnz

    def __del__(self):
        try:
            self.lib.L.ref_free(C.c_void_p(self.h))
        except Exception:
            pass

    def block(self, which: str) -> CSR:
        idx = {"A": 0, "B": 1, "Bt": 2, "Q": 3, "Q_nu": 4}[which]
        shapes = {"A": (self.n_u, self.n_u), "B": (self.n_p, self.n_u),
                  "Bt": (self.n_u, self.n_p), "Q": (self.n_p, self.n_p),
                  "Q_nu": (self.n_p, self.n_p)}[which]
        nnz = int(self._nnz[idx])
        rp = np.zeros(shapes[0] + 1, np.int64)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz)
        self.lib.L.ref_export(C.c_void_p(self.h), idx, rp, ci, v)
        return CSR(shapes[0], shapes[1], rp, ci, v)

    def rhs(self) -> np.ndarray:
        f = np.zeros(self.n_u)
        self.lib.L.ref_rhs(C.c_void_p(self.h), f)
        return f

    def set_rhs(self, f: np.ndarray) -> None:
        self.lib.L.ref_set_rhs(C.c_void_p(self.h), np.ascontiguousarray(f, np.float64))

    def apply(self, x: np.ndarray) -> np.ndarray:
        y = np.zeros(self.n_u + self.n_p)
        self.lib.L.ref_apply(C.c_void_p(self.h), np.ascontiguousarray(x, np.float64), y)
        return y

    def solve(self, strategy: str, outer_tol: float, inner_tol: float, max_iter: int = 20000,
              euclid: bool = True, hist_cap: int = 0):
        u = np.zeros(self.n_u)
        p = np.zeros(self.n_p)
        rep = np.zeros(7)
        cap = hist_cap or (max_iter + 1)
        hm = np.zeros(cap)
        he = np.zeros(cap)
        err = C.create_string_buffer(512)
        rc = self.lib.L.ref_solve(C.c_void_p(self.h), strategy.encode(), outer_tol, inner_tol,
                                  max_iter, int(euclid), u, p, rep, hm, he, cap, err, 512)
        if rc:
            e = RuntimeError(err.value.decode())
            e.code = rc  # type: ignore[attr-defined]
            raise e
        n = min(int(rep[6]), cap)
        return dict(u=u, p=p, iterations=int(rep[0]), converged=bool(rep[1]),
                    wall_seconds=rep[2], mean_inner_top=rep[3], mean_inner_bottom=rep[4],
                    setup_seconds=rep[5], residual_history=hm[:n], euclid_history=he[:n])


class RefPrecond:
    """make_strategy once (precond.cpp:161-193), many solve_stokes(system, precond, options)."""

    def __init__(self, system: RefSystem, strategy: str, inner_tol: float):
        self.system, self.inner_tol = system, inner_tol
        err = C.create_string_buffer(512)
        t = C.c_double(0.0)
        self.h = system.lib.L.ref_precond_make(C.c_void_p(system.h), strategy.encode(), inner_tol,
                                               C.byref(t), err, 512)
        if not self.h:
            raise RuntimeError(err.value.decode())
        self.setup_seconds = t.value

    def close(self):
        if self.h:
            self.system.lib.L.ref_precond_free(C.c_void_p(self.h))
            self.h = None

    def solve(self, outer_tol: float, max_iter: int = 20000, euclid: bool = True):
        s = self.system
        u = np.zeros(s.n_u)
        p = np.zeros(s.n_p)
        rep = np.zeros(7)
        cap = max_iter + 1
        hm = np.zeros(cap)
        he = np.zeros(cap)
        err = C.create_string_buffer(512)
        rc = s.lib.L.ref_solve_with(C.c_void_p(s.h), C.c_void_p(self.h), outer_tol, self.inner_tol,
                                    max_iter, int(euclid), u, p, rep, hm, he, cap, err, 512)
        if rc:
            e = RuntimeError(err.value.decode())
            e.code = rc  # type: ignore[attr-defined]
            raise e
        n = min(int(rep[6]), cap)
        return dict(u=u, p=p, iterations=int(rep[0]), converged=bool(rep[1]),
                    wall_seconds=rep[2], mean_inner_top=rep[3], mean_inner_bottom=rep[4],
                    setup_seconds=self.setup_seconds, residual_history=hm[:n],
                    euclid_history=he[:n])


def ref_minres_x0(pre: "RefPrecond", x0: np.ndarray, outer_tol: float, max_iter: int = 20000,
                  euclid: bool = True):
    """The reference's minres with MinresOptions::x0 on pre.system (no pressure filter)."""
    s = pre.system
    n = s.n_u + s.n_p
    x = np.zeros(n)
    rep = np.zeros(3)
    he = np.zeros(max_iter + 1)
    err = C.create_string_buffer(512)
    fn = s.lib.L.ref_minres_x0
    fn.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int,
                   C.c_char_p, C.c_int]
    rc = fn(C.c_void_p(s.h), C.c_void_p(pre.h), np.ascontiguousarray(x0, np.float64), outer_tol, max_iter,
            int(euclid), x, rep, he, max_iter + 1, err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    k = min(int(rep[2]), max_iter + 1)
    return dict(x=x, iterations=int(rep[0]), converged=bool(rep[1]), euclid_history=he[:k])


class _OrCsr(C.Structure):
    _fields_ = [("n_rows", C.c_int), ("n_cols", C.c_int), ("rp", C.c_void_p),
                ("ci", C.c_void_p), ("v", C.c_void_p)]


class _OrReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("wall_seconds", C.c_double),
                ("setup_seconds", C.c_double), ("mean_inner_top", C.c_double),
                ("mean_inner_bottom", C.c_double), ("hist_len", C.c_int), ("status", C.c_int),
                ("failed_block", C.c_int), ("breakdown_row", C.c_int),
                ("inner_top", C.c_long), ("apps_top", C.c_long), ("inner_bottom", C.c_long),
                ("apps_bottom", C.c_long)]


def _orcsr(a: CSR) -> _OrCsr:
    return _OrCsr(a.n_rows, a.n_cols, a.rp.ctypes.data, a.ci.ctypes.data, a.v.ctypes.data)


class PortLib:
    """The plain-C restatement (oracle/_ref/libdsoracle.so)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.or_spmv.argtypes = [C.POINTER(_OrCsr), _dp, _dp]
        L.or_rcm.argtypes = [C.c_int, _i64p, _i32p, _i32p]
        L.or_permute.argtypes = [C.c_int, _i64p, _i32p, _dp, _i32p, _i64p, _i32p, _dp]
        L.or_lower_nnz.argtypes = [C.c_int, _i64p, _i32p]
        L.or_lower_nnz.restype = C.c_int64
        L.or_ic0.argtypes = [C.c_int, _i64p, _i32p, _dp, _i64p, _i32p, _dp, C.POINTER(C.c_int)]
        L.or_ic0_solve.argtypes = [C.c_int, _i64p, _i32p, _dp, _dp, _dp]
        L.or_pcg.argtypes = [C.POINTER(_OrCsr), _dp, C.c_int, C.POINTER(_OrCsr), C.c_double,
                             C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_solve_stokes.argtypes = [C.POINTER(_OrCsr)] * 5 + [
            _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, _dp, _dp,
            C.POINTER(_OrReport), _dp, _dp, C.c_int]

    def spmv(self, A: CSR, x: np.ndarray) -> np.ndarray:
        y = np.zeros(A.n_rows)
        a = _orcsr(A)
        self.L.or_spmv(C.byref(a), np.ascontiguousarray(x, np.float64), y)
        return y

    def rcm(self, A: CSR) -> np.ndarray:
        perm = np.zeros(A.n_rows, np.int32)
        if self.L.or_rcm(A.n_rows, A.rp, A.ci, perm) != 0:
            raise ValueError("rcm_permutation: pattern is not symmetric")
        return perm

    def permute(self, A: CSR, perm: np.ndarray) -> CSR:
        rp = np.zeros(A.n_rows + 1, np.int64)
        ci = np.zeros(A.nnz, np.int32)
        v = np.zeros(A.nnz)
        self.L.or_permute(A.n_rows, A.rp, A.ci, A.v, np.ascontiguousarray(perm, np.int32), rp,
                          ci, v)
        return CSR(A.n_rows, A.n_cols, rp, ci, v)

    def ic0(self, A: CSR) -> CSR:
        lnnz = self.L.or_lower_nnz(A.n_rows, A.rp, A.ci)
        rp = np.zeros(A.n_rows + 1, np.int64)
        ci = np.zeros(lnnz, np.int32)
        v = np.zeros(lnnz)
        bad = C.c_int(-1)
        rc = self.L.or_ic0(A.n_rows, A.rp, A.ci, A.v, rp, ci, v, C.byref(bad))
        if rc:
            e = RuntimeError(f"ic0 failed (code {rc}) at row {bad.value}")
            e.row = bad.value  # type: ignore[attr-defined]
            e.code = rc  # type: ignore[attr-defined]
            raise e
        return CSR(A.n_rows, A.n_cols, rp, ci, v)

    def ic0_solve(self, L: CSR, r: np.ndarray) -> np.ndarray:
        z = np.zeros(L.n_rows)
        self.L.or_ic0_solve(L.n_rows, L.rp, L.ci, L.v, np.ascontiguousarray(r, np.float64), z)
        return z

    def pcg(self, A: CSR, b: np.ndarray, pre_kind: int, tol: float, max_iter: int,
            L: CSR | None = None):
        x = np.zeros(A.n_rows)
        it, conv = C.c_int(), C.c_int()
        a = _orcsr(A)
        lf = _orcsr(L) if L is not None else _orcsr(A)
        rc = self.L.or_pcg(C.byref(a), np.ascontiguousarray(b, np.float64), pre_kind,
                           C.byref(lf), tol, max_iter, x, C.byref(it), C.byref(conv))
        if rc:
            raise RuntimeError(f"pcg failed with code {rc}")
        return x, it.value, bool(conv.value)

    def solve_stokes(self, A: CSR, B: CSR, Bt: CSR, Q_nu: CSR, f: np.ndarray, strategy: str,
                     outer_tol: float, inner_tol: float, max_iter: int = 20000,
                     euclid: bool = True, inner_cap: int = 100000, Q_filter: CSR | None = None):
        top, bottom = STRATEGY_BLOCKS[strategy]
        u = np.zeros(A.n_rows)
        p = np.zeros(Q_nu.n_rows)
        hm = np.zeros(max_iter + 1)
        he = np.zeros(max_iter + 1)
        rep = _OrReport()
        mats = [_orcsr(A), _orcsr(B), _orcsr(Bt), _orcsr(Q_nu)]
        qf = _orcsr(Q_filter) if Q_filter is not None else None
        rc = self.L.or_solve_stokes(C.byref(mats[0]), C.byref(mats[1]), C.byref(mats[2]),
                                    C.byref(mats[3]), C.byref(qf) if qf is not None else None,
                                    np.ascontiguousarray(f, np.float64), top, bottom, outer_tol,
                                    inner_tol, max_iter, int(euclid), inner_cap, u, p,
                                    C.byref(rep), hm, he, max_iter + 1)
        n = min(rep.hist_len, max_iter + 1)
        return dict(status=rc, u=u, p=p, iterations=rep.iterations,
                    converged=bool(rep.converged), wall_seconds=rep.wall_seconds,
                    setup_seconds=rep.setup_seconds, mean_inner_top=rep.mean_inner_top,
                    mean_inner_bottom=rep.mean_inner_bottom, residual_history=hm[:n],
                    euclid_history=he[:n], failed_block=rep.failed_block,
                    inner_top=rep.inner_top, apps_top=rep.apps_top,
                    inner_bottom=rep.inner_bottom, apps_bottom=rep.apps_bottom)
