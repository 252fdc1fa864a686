"""Blocked-sweep plan (paper_1309_5048_b200/csrc/gpu/bsweep_plan.cpp) on the
host, without a GPU: the plan dsgpu_setup builds from an IC(0) factor (dense
16x16 blocks next to the diagonal, mid / far lane-interleaved lists), evaluated
in the plan's own arithmetic order by the library's test hook
dsgpu_debug_bsweep_host, must reproduce Ic0Factor::solve
(proj/src/cholesky.cpp:136-152, restated in oracle/ds_oracle.c) to round-off."""
import ctypes as C

import numpy as np
import pytest

from conftest import to_oracle

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


@pytest.fixture(scope="module")
def hook():
    from paper_1309_5048_b200._lib import load_gpu
    L = load_gpu()
    L.dsgpu_debug_bsweep_host.argtypes = [C.c_int, _i64, _i32, _dp, _dp, _dp, _i64]
    return L.dsgpu_debug_bsweep_host


def plan_apply(hook, F, r):
    z = np.zeros(F.n_rows)
    st = np.zeros(8, np.int64)
    rc = hook(F.n_rows, F.row_ptr, F.cols, F.vals, np.ascontiguousarray(r), z, st)
    return rc, z, st


@pytest.mark.parametrize("case,k,n,dim", [("psi-mms", 2, 8, 2), ("psi-mms", 2, 64, 2), ("random", 3, 16, 2),
                                          ("cavity", 2, 16, 2), ("psi-mms", 2, 6, 3), ("random", 2, 12, 3)])
def test_plan_matches_reference_substitution(hook, port, case, k, n, dim):
    from paper_1309_5048_b200 import host
    s = host.assemble(case, k, n, dim=dim, seed=42)
    rng = np.random.default_rng(7)
    for m in (s.A, s.Q_nu):
        F = host.ic0(host.permute_symmetric(m, host.rcm_permutation(m)))
        r = rng.uniform(-1.0, 1.0, F.n_rows)
        rc, z, st = plan_apply(hook, F, r)
        assert rc == 0
        zr = port.ic0_solve(to_oracle(F), r)
        assert np.linalg.norm(z - zr) <= 1e-13 * np.linalg.norm(zr)
        # every strictly-lower factor entry is in exactly one class
        assert st[1] + st[2] + st[3] == F.nnz - F.n_rows
        assert st[0] == (F.n_rows + 15) // 16


def test_plan_sizes_not_multiple_of_group(hook, port):
    """n not a multiple of 16 (padding rows), n smaller than one group, a
    diagonal factor, and a dense lower-triangular factor."""
    from paper_1309_5048_b200.host import CsrMatrix
    rng = np.random.default_rng(3)
    for n in (1, 5, 16, 17, 33, 100):
        d = np.tril(rng.uniform(-0.2, 0.2, (n, n)), -1)
        if n == 5:
            d[:] = 0.0
        d += np.diag(rng.uniform(1.0, 2.0, n))
        rows, cols = np.nonzero(d)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
        F = CsrMatrix(n, n, rp, cols.astype(np.int32), d[rows, cols])
        r = rng.uniform(-1.0, 1.0, n)
        rc, z, _ = plan_apply(hook, F, r)
        assert rc == 0
        zr = np.linalg.solve(d.T, np.linalg.solve(d, r))
        assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)


def test_plan_rejects_bad_factor(hook):
    from paper_1309_5048_b200.host import CsrMatrix
    # upper entry / unsorted / missing diagonal
    for rp, ci, v in (([0, 2, 3], [0, 1, 1], [1.0, 0.5, 1.0]), ([0, 1, 1], [0], [1.0]),
                      ([0, 1, 4], [0, 1, 0, 1], [1.0, 0.3, 0.2, 1.0])):
        F = CsrMatrix(2, 2, np.array(rp, np.int64), np.array(ci, np.int32), np.array(v))
        rc, _, _ = plan_apply(hook, F, np.ones(2))
        assert rc != 0
