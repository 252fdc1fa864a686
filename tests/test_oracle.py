"""The CPU oracle (oracle/ds_oracle.c) pinned against the unmodified reference
and the reference's own known-answer tests (proj/tests/test_solvers.cpp,
test_sparse.cpp). CPU only."""
import numpy as np
import pytest

from conftest import golden_csr, load_golden
from oracle import CSR
from oracle.oracle import STRATEGIES


def tri(n):
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 1.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = 1.0
    return CSR.from_dense(d)


def bandwidth(m):
    rows = np.repeat(np.arange(m.n_rows), np.diff(m.rp))
    return int(np.abs(rows - m.ci).max()) if m.nnz else 0


def test_rcm_known_answers(port):
    # test_sparse.cpp:173-210: tridiagonal stays 1, arrowhead 5 -> 4, star <= 3
    t = tri(8)
    assert bandwidth(port.permute(t, port.rcm(t))) == 1
    a = np.eye(6)
    a[0, 1:] = a[1:, 0] = 1.0
    a = CSR.from_dense(a)
    assert bandwidth(a) == 5
    assert bandwidth(port.permute(a, port.rcm(a))) == 4
    s = np.eye(5)
    s[0, 1:] = s[1:, 0] = 1.0
    s = CSR.from_dense(s)
    assert bandwidth(port.permute(s, port.rcm(s))) <= 3


def test_rcm_bijection_and_nonsymmetric(port):
    rng = np.random.default_rng(13)
    d = (rng.random((40, 40)) < 0.1) * 1.0
    d = d + d.T + np.eye(40)
    perm = port.rcm(CSR.from_dense(d))
    assert sorted(perm.tolist()) == list(range(40))
    bad = CSR.from_dense(np.array([[1.0, 1.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        port.rcm(bad)


def test_ic0_known_answers(port):
    # test_sparse.cpp:222-264
    f = port.ic0(CSR.from_dense(np.diag([4.0, 9.0, 16.0])))
    assert np.array_equal(f.to_dense().diagonal(), [2.0, 3.0, 4.0])
    a = np.array([[4.0, 1.0, 0.5], [1.0, 3.0, 0.25], [0.5, 0.25, 5.0]])
    L = port.ic0(CSR.from_dense(a)).to_dense()
    np.testing.assert_allclose(L @ L.T, a, rtol=1e-14)
    rng = np.random.default_rng(77)
    m = (rng.random((60, 60)) < 0.08) * rng.uniform(-1, 1, (60, 60))
    m = np.tril(m, -1)
    m = m + m.T
    np.fill_diagonal(m, np.abs(m).sum(1) + 1.0)
    Ld = port.ic0(CSR.from_dense(m)).to_dense()
    LLt = Ld @ Ld.T
    mask = np.tril(m != 0)
    assert np.all(np.abs(LLt - m)[mask] < 1e-12 * (1 + np.abs(m[mask])))
    with pytest.raises(RuntimeError) as e:
        port.ic0(CSR.from_dense(np.diag([1.0, -1.0])))
    assert e.value.row == 1 and e.value.code == 6
    with pytest.raises(RuntimeError) as e:
        port.ic0(CSR.from_dense(np.array([[1.0, 1.0], [1.0, 0.0]])))
    assert e.value.code == 3


def test_pcg_known_answers(port):
    # test_solvers.cpp:110-136
    d = CSR.from_dense(np.diag([2.0, 5.0, 1.0, 9.0]))
    x, it, conv = port.pcg(d, np.array([1.0, 2.0, 3.0, 4.0]), 1, 1e-12, 10)
    assert conv and it == 1 and abs(x[1] - 0.4) < 1e-14
    m2 = CSR.from_dense(np.array([[4.0, 1.0], [1.0, 3.0]]))
    x, it, conv = port.pcg(m2, np.array([1.0, 2.0]), 0, 1e-12, 10)
    assert conv and it <= 2
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=1e-10)
    with pytest.raises(RuntimeError):
        port.pcg(CSR.from_dense(np.diag([-1.0, -2.0])), np.ones(2), 0, 1e-10, 10)


def test_restatement_bitexact_vs_reference_scalar(ref, port):
    """With the reference forced onto its scalar kernels the C restatement
    reproduces every reference solve bit for bit."""
    s = ref.assemble("psi-mms", 2, 8)
    A, B, Bt, Q, Qn = (s.block(w) for w in ("A", "B", "Bt", "Q", "Q_nu"))
    f = s.rhs()
    ref.force_scalar(True)
    try:
        for strat in STRATEGIES:
            r = s.solve(strat, 1e-8, 1e-1)
            o = port.solve_stokes(A, B, Bt, Qn, f, strat, 1e-8, 1e-1, Q_filter=Q)
            assert o["status"] == 0
            assert r["iterations"] == o["iterations"]
            assert np.array_equal(r["u"], o["u"]) and np.array_equal(r["p"], o["p"])
            assert np.array_equal(r["euclid_history"], o["euclid_history"])
            assert np.array_equal(r["residual_history"], o["residual_history"])
    finally:
        ref.force_scalar(False)


def test_restatement_primitives_bitexact(ref, port):
    s = ref.assemble("cavity", 3, 8)
    A = s.block("A")
    perm = ref.rcm(A)
    assert np.array_equal(perm, port.rcm(A))
    Ar, Ap = ref.permute(A, perm), port.permute(A, perm)
    assert np.array_equal(Ar.v, Ap.v) and np.array_equal(Ar.ci, Ap.ci)
    Lr, Lp = ref.ic0(Ar), port.ic0(Ap)
    assert np.array_equal(Lr.v, Lp.v)
    r = np.random.default_rng(1).standard_normal(A.n_rows)
    assert np.array_equal(ref.ic0_solve(Lr, r), port.ic0_solve(Lp, r))


def test_oracle_against_golden_fixtures(port):
    """The committed fixtures were produced by the reference (make_golden.py)."""
    d = load_golden("c1_psi_k2_n8.npz")
    A, B, Bt, Q, Qn = (golden_csr(d, w) for w in ("A", "B", "Bt", "Q", "Q_nu"))
    for tag, M in (("A", A), ("Q", Qn)):
        perm = port.rcm(M)
        assert np.array_equal(perm, d["perm_" + tag])
        L = port.ic0(port.permute(M, perm))
        assert np.array_equal(L.v, d["L_" + tag + "_v"])
        z = port.ic0_solve(L, d["ic_r_" + tag])
        np.testing.assert_array_equal(z, d["ic_z_" + tag])
    for strat in STRATEGIES:
        key = f"{strat}|0.1"
        o = port.solve_stokes(A, B, Bt, Qn, d["f"], strat, 1e-8, 1e-1, Q_filter=Q)
        meta = d["sol_meta|" + key]
        assert abs(o["iterations"] - meta[0]) <= 2
        x_ref = np.concatenate([d["sol_u|" + key], d["sol_p|" + key]])
        x = np.concatenate([o["u"], o["p"]])
        assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
    g = load_golden("c1_psi_k2_n16.npz")
    A, B, Bt, Q, Qn = (golden_csr(g, w) for w in ("A", "B", "Bt", "Q", "Q_nu"))
    o = port.solve_stokes(A, B, Bt, Qn, g["f"], "IC0-PCG(A)+Diag(Q)", 1e-8, 1e-1, Q_filter=Q)
    assert o["iterations"] == int(g["meta"][0])
    x_ref = np.concatenate([g["u"], g["p"]])
    x = np.concatenate([o["u"], o["p"]])
    assert np.linalg.norm(x - x_ref) <= 1e-12 * np.linalg.norm(x_ref)


def test_oracle_errors(port):
    d = load_golden("c1_psi_k2_n8.npz")
    A, B, Bt, Q, Qn = (golden_csr(d, w) for w in ("A", "B", "Bt", "Q", "Q_nu"))
    neg = CSR(Qn.n_rows, Qn.n_cols, Qn.rp, Qn.ci, -Qn.v)
    o = port.solve_stokes(A, B, Bt, neg, d["f"], "IC0-PCG(A)+Diag(Q)", 1e-8, 1e-1)
    assert o["status"] == 5  # JacobiBlock: nonpositive diagonal
    o = port.solve_stokes(A, B, Bt, Qn, d["f"], "IC0-PCG(A,Q)", 1e-8, 1e-1, max_iter=3)
    assert o["status"] == 0 and not o["converged"] and o["iterations"] == 3
