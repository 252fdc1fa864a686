"""ctypes binding of the native host library (include/dshost.h).

Builds BASELINE's Stokes systems and the preconditioner setup (RCM, symmetric
permutation, IC(0)) natively; mirrors the reference's host steps
(``build_pair`` + ``assemble_stokes``, ``rcm_permutation``,
``permute_symmetric``, ``ic0``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import load_host

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

CASES = {"psi-mms": 0, "cavity": 1, "random": 3}


class FactorBreakdown(RuntimeError):
    """Nonpositive IC(0) pivot (reference ``FactorBreakdown``, cholesky.hpp:13-19)."""

    def __init__(self, msg: str, row: int):
        super().__init__(msg)
        self.row = row


@dataclass
class CsrMatrix:
    """Reference ``CsrMatrix`` layout (csr.hpp:12-16): int64 row_ptr, int32 cols, f64 vals."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def diagonal(self) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        d = np.zeros(min(self.n_rows, self.n_cols))
        m = self.cols == rows
        d[rows[m]] = self.vals[m]
        return d


@dataclass
class StokesSystem:
    """Mirror of the reference ``StokesSystem`` (assembly.hpp:31-49)."""

    A: CsrMatrix
    B: CsrMatrix
    Bt: CsrMatrix
    Q: CsrMatrix
    Q_nu: CsrMatrix
    f: np.ndarray
    nu: float = 1.0
    dim: int = 2
    # identity-map systems built here: the constant pressure spans Ker(B^T),
    # so solve_stokes applies the reference's zero-mean filter
    has_constant_pressure_kernel: bool = True

    @property
    def n_u(self) -> int:
        return self.A.n_rows

    @property
    def n_p(self) -> int:
        return self.Q.n_rows

    @property
    def size(self) -> int:
        return self.n_u + self.n_p


def _err(lib) -> str:
    return lib.dshost_last_error().decode()


def _host():
    L = load_host()
    if not getattr(L, "_typed", False):
        L.dshost_last_error.restype = C.c_char_p
        L.dshost_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_uint64, C.POINTER(C.c_void_p)]
        L.dshost_free.argtypes = [C.c_void_p]
        L.dshost_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), _i64p]
        L.dshost_block.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_void_p)]
        L.dshost_rhs.restype = C.c_void_p
        L.dshost_rhs.argtypes = [C.c_void_p]
        L.dshost_rcm.argtypes = [C.c_int, _i64p, _i32p, _i32p]
        L.dshost_permute.argtypes = [C.c_int, _i64p, _i32p, _dp, _i32p, _i64p, _i32p, _dp]
        L.dshost_lower_nnz.argtypes = [C.c_int, _i64p, _i32p]
        L.dshost_lower_nnz.restype = C.c_int64
        L.dshost_ic0.argtypes = [C.c_int, _i64p, _i32p, _dp, _i64p, _i32p, _dp,
                                 C.POINTER(C.c_int)]
        L.dshost_write_matrix_market.argtypes = [C.c_char_p, C.c_int, C.c_int, _i64p, _i32p, _dp,
                                                 C.c_int]
        L.dshost_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.dshost_csr_view.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_void_p)]
        L.dshost_csr_free.argtypes = [C.c_void_p]
        L._typed = True
    return L


def assemble(case: str = "psi-mms", k_prime: int = 2, n_elem: int = 16, dim: int = 2,
             nu: float = 1.0, seed: int = 0) -> StokesSystem:
    """Assemble one of BASELINE's systems natively (copies out of the C++ handle)."""
    L = _host()
    h = C.c_void_p()
    rc = L.dshost_assemble(dim, k_prime, n_elem, CASES[case], nu, seed, C.byref(h))
    if rc:
        raise ValueError(_err(L))
    try:
        nu_, np_ = C.c_int(), C.c_int()
        nnz = np.zeros(5, np.int64)
        L.dshost_dims(h, C.byref(nu_), C.byref(np_), nnz)
        blocks = []
        for which in range(5):
            nr, nc = C.c_int(), C.c_int()
            rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
            L.dshost_block(h, which, C.byref(nr), C.byref(nc), C.byref(rp), C.byref(ci),
                           C.byref(v))
            k = int(nnz[which])
            blocks.append(CsrMatrix(
                nr.value, nc.value,
                np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_int64)), (nr.value + 1,)).copy(),
                np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_int32)), (max(k, 1),))[:k].copy(),
                np.ctypeslib.as_array(C.cast(v, C.POINTER(C.c_double)), (max(k, 1),))[:k].copy()))
        f = np.ctypeslib.as_array(C.cast(L.dshost_rhs(h), C.POINTER(C.c_double)),
                                  (nu_.value,)).copy()
    finally:
        L.dshost_free(h)
    return StokesSystem(*blocks, f=f, nu=nu, dim=dim)


def rcm_permutation(a: CsrMatrix) -> np.ndarray:
    L = _host()
    perm = np.zeros(a.n_rows, np.int32)
    if L.dshost_rcm(a.n_rows, a.row_ptr, a.cols, perm):
        raise ValueError(_err(L))
    return perm


def permute_symmetric(a: CsrMatrix, perm: np.ndarray) -> CsrMatrix:
    L = _host()
    rp = np.zeros(a.n_rows + 1, np.int64)
    ci = np.zeros(a.nnz, np.int32)
    v = np.zeros(a.nnz)
    if L.dshost_permute(a.n_rows, a.row_ptr, a.cols, a.vals,
                        np.ascontiguousarray(perm, np.int32), rp, ci, v):
        raise ValueError(_err(L))
    return CsrMatrix(a.n_rows, a.n_cols, rp, ci, v)


def ic0(a: CsrMatrix) -> CsrMatrix:
    L = _host()
    lnnz = L.dshost_lower_nnz(a.n_rows, a.row_ptr, a.cols)
    rp = np.zeros(a.n_rows + 1, np.int64)
    ci = np.zeros(lnnz, np.int32)
    v = np.zeros(lnnz)
    bad = C.c_int(-1)
    rc = L.dshost_ic0(a.n_rows, a.row_ptr, a.cols, a.vals, rp, ci, v, C.byref(bad))
    if rc == 6:
        raise FactorBreakdown(_err(L), bad.value)
    if rc:
        raise ValueError(_err(L))
    return CsrMatrix(a.n_rows, a.n_cols, rp, ci, v)


__all__ = ["CsrMatrix", "StokesSystem", "FactorBreakdown", "assemble", "rcm_permutation",
           "permute_symmetric", "ic0", "CASES"]
_ = os


# ---- Matrix Market wire format (proj/src/csr.cpp:126-175) -----------------
DSHOST_E_INVALID, DSHOST_E_RUNTIME = 3, 8


def _raise(L, rc: int):
    msg = _err(L)
    if rc == DSHOST_E_INVALID:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise RuntimeError(msg)    # std::runtime_error (I/O, file format)


def write_matrix_market(a: CsrMatrix, path: str, symmetric: bool = False) -> None:
    """The reference's dump format (write_matrix_market, csr.cpp:126-142),
    byte for byte; symmetric writes the lower triangle only."""
    L = _host()
    rc = L.dshost_write_matrix_market(str(path).encode(), a.n_rows, a.n_cols,
                                      np.ascontiguousarray(a.row_ptr, np.int64),
                                      np.ascontiguousarray(a.cols, np.int32),
                                      np.ascontiguousarray(a.vals, np.float64), int(symmetric))
    if rc:
        _raise(L, rc)


def read_matrix_market(path: str) -> CsrMatrix:
    """The CSR the reference's read_matrix_market (csr.cpp:144-175) builds."""
    L = _host()
    h = C.c_void_p()
    rc = L.dshost_read_matrix_market(str(path).encode(), C.byref(h))
    if rc:
        _raise(L, rc)
    try:
        nr, nc = C.c_int(), C.c_int()
        rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.dshost_csr_view(h, C.byref(nr), C.byref(nc), C.byref(rp), C.byref(ci), C.byref(v))
        row_ptr = np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_int64)), (nr.value + 1,)).copy()
        k = int(row_ptr[-1])
        cols = np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_int32)), (max(k, 1),))[:k].copy()
        vals = np.ctypeslib.as_array(C.cast(v, C.POINTER(C.c_double)), (max(k, 1),))[:k].copy()
    finally:
        L.dshost_csr_free(h)
    return CsrMatrix(nr.value, nc.value, row_ptr, cols, vals)


def transpose(a: CsrMatrix) -> CsrMatrix:
    """CsrMatrix::transposed: rows of the result keep the source row order."""
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int32), np.diff(a.row_ptr))
    order = np.argsort(a.cols, kind="stable")
    rp = np.zeros(a.n_cols + 1, np.int64)
    np.cumsum(np.bincount(a.cols, minlength=a.n_cols), out=rp[1:])
    return CsrMatrix(a.n_cols, a.n_rows, rp, rows[order].astype(np.int32), a.vals[order].copy())


def system_from_matrix_market(a_path: str, b_path: str, q_path: str, f: np.ndarray,
                              nu: float = 1.0, dim: int = 2,
                              has_constant_pressure_kernel: bool = True) -> StokesSystem:
    """A StokesSystem from the reference's --dump-matrices files
    (runner.cpp:223-229: A, B, Q) and a velocity right-hand side, completed
    like assemble_stokes (assembly.cpp:350-355): Bt = B^T, Q_nu = Q / (2 nu)."""
    A, B, Q = read_matrix_market(a_path), read_matrix_market(b_path), read_matrix_market(q_path)
    if A.n_rows != A.n_cols or Q.n_rows != Q.n_cols or B.n_rows != Q.n_rows or B.n_cols != A.n_rows:
        raise ValueError("system_from_matrix_market: inconsistent block dimensions")
    f = np.ascontiguousarray(f, np.float64)
    if f.shape != (A.n_rows,):
        raise ValueError("system_from_matrix_market: f must have n_u entries")
    scale = 1.0 / (2.0 * nu)
    Q_nu = CsrMatrix(Q.n_rows, Q.n_cols, Q.row_ptr.copy(), Q.cols.copy(), Q.vals * scale)
    return StokesSystem(A, B, transpose(B), Q, Q_nu, f=f.copy(), nu=nu, dim=dim,
                        has_constant_pressure_kernel=has_constant_pressure_kernel)
