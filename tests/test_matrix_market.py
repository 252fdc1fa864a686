"""Matrix Market wire format (libdshost: dshost_write/read_matrix_market)
against the reference's write_matrix_market / read_matrix_market
(proj/src/csr.cpp:126-175) and its own round-trip test
(tests/test_sparse.cpp:147-169). The writer must be byte-identical, the reader
must build bit-identical CSR arrays (symmetric mirroring, duplicate summation,
csr_from_triplets ordering), and the error paths must raise the reference's
exception classes. CPU only; the fixtures under tests/golden/mm/ were written
by the reference (tests/golden/make_golden_mm.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, to_oracle
from paper_1309_5048_b200 import host

MM = os.path.join(GOLDEN, "mm")


def same(a, b):
    return (a.n_rows == b.n_rows and a.n_cols == b.n_cols and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.cols, b.cols) and np.array_equal(a.vals.view(np.int64), b.vals.view(np.int64)))


def random_sparse(n, density, seed, symmetric):
    """A random n x n CSR (the reference test's random_sparse shape)."""
    rng = np.random.default_rng(seed)
    d = (rng.random((n, n)) < density) * rng.standard_normal((n, n))
    if symmetric:
        d = np.tril(d) + np.tril(d, -1).T
    np.fill_diagonal(d, np.abs(np.diag(d)) + 1.0)
    rows, cols = np.nonzero(d)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return host.CsrMatrix(n, n, rp, cols.astype(np.int32), d[rows, cols].astype(np.float64))


def test_reader_on_reference_dumps_matches_assembly():
    """The reference's dump of psi-MMS k'=2 3x3 reads back into exactly the
    blocks our native assembly builds; the completed system (Bt, Q_nu) too."""
    s = host.assemble("psi-mms", 2, 3)
    f = np.load(os.path.join(MM, "f_psi_k2_h3.npy"))
    m = host.system_from_matrix_market(os.path.join(MM, "A_psi_k2_h3.mtx"),
                                       os.path.join(MM, "B_psi_k2_h3.mtx"),
                                       os.path.join(MM, "Q_psi_k2_h3.mtx"), f)
    for w in ("A", "B", "Bt", "Q", "Q_nu"):
        a, b = getattr(m, w), getattr(s, w)
        assert a.n_rows == b.n_rows and np.array_equal(a.row_ptr, b.row_ptr), w
        assert np.array_equal(a.cols, b.cols), w
        # text at 17 significant digits round-trips every double exactly
        assert np.array_equal(a.vals, b.vals), w
    assert np.array_equal(m.f, s.f)


@pytest.mark.parametrize("name,symmetric", [("A", True), ("B", False), ("Q", True)])
def test_writer_byte_identical_to_reference_dump(tmp_path, name, symmetric):
    s = host.assemble("psi-mms", 2, 3)
    out = tmp_path / f"{name}.mtx"
    host.write_matrix_market(getattr(s, name), str(out), symmetric)
    ref = open(os.path.join(MM, f"{name}_psi_k2_h3.mtx"), "rb").read()
    assert out.read_bytes() == ref


def test_rectangular_round_trip(tmp_path):
    """test_sparse.cpp:149-158: 3x5 general."""
    b = host.read_matrix_market(os.path.join(MM, "rect_3x5.mtx"))
    assert (b.n_rows, b.n_cols) == (3, 5)
    assert b.row_ptr.tolist() == [0, 1, 2, 3] and b.cols.tolist() == [4, 0, 2]
    assert b.vals.tolist() == [1.5, -2.0, 0.25]
    p = tmp_path / "r.mtx"
    host.write_matrix_market(b, str(p))
    assert p.read_bytes() == open(os.path.join(MM, "rect_3x5.mtx"), "rb").read()


@pytest.mark.parametrize("symmetric", [False, True])
def test_random_round_trip(tmp_path, symmetric):
    """test_sparse.cpp:159-168 (pattern exact, values to 1e-15 there; exact here)."""
    m = random_sparse(30, 0.15, 5 if symmetric else 6, symmetric)
    p = tmp_path / "rt.mtx"
    host.write_matrix_market(m, str(p), symmetric)
    assert same(host.read_matrix_market(str(p)), m)


def test_duplicates_summed_in_file_order_and_mirrored(tmp_path):
    """csr_from_triplets (csr.cpp:88-111): stable (row, col) order, duplicates
    summed from 0.0 in file order; symmetric off-diagonals mirrored."""
    p = tmp_path / "dup.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n"
                 "3 3 6\n2 1 0.1\n1 1 1e-17\n2 1 0.2\n1 1 1.0\n3 3 -0.0\n3 2 7\n")
    m = host.read_matrix_market(str(p))
    assert m.row_ptr.tolist() == [0, 2, 4, 6]
    assert m.cols.tolist() == [0, 1, 0, 2, 1, 2]
    assert m.vals[0] == (0.0 + 1e-17) + 1.0
    assert m.vals[1] == (0.0 + 0.1) + 0.2 and m.vals[2] == (0.0 + 0.1) + 0.2
    assert m.vals[3] == 7.0 and m.vals[4] == 7.0
    assert m.vals[5] == 0.0 and not np.signbit(m.vals[5])  # 0.0 + -0.0


BAD = {
    "nohead.mtx": ("1 1 1\n1 1 1\n", "missing MatrixMarket header"),
    "array.mtx": ("%%MatrixMarket matrix array real general\n1 1\n1\n", "unsupported MatrixMarket type"),
    "herm.mtx": ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
                 "unsupported qualifier hermitian"),
    "size.mtx": ("%%MatrixMarket matrix coordinate real general\n2 x 1\n", "bad size line"),
    "trunc.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2\n", "truncated entry list"),
    "nan.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n", "truncated entry list"),
}


@pytest.mark.parametrize("fname", sorted(BAD))
def test_format_errors_raise_runtime_error(tmp_path, fname):
    text, msg = BAD[fname]
    p = tmp_path / fname
    p.write_text(text)
    with pytest.raises(RuntimeError, match=msg):
        host.read_matrix_market(str(p))


def test_missing_file_and_out_of_range(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        host.read_matrix_market(str(tmp_path / "nope.mtx"))
    p = tmp_path / "oor.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    with pytest.raises(ValueError, match="index out of range"):
        host.read_matrix_market(str(p))


# ---- against the reference library itself (where oracle/_ref is built) ----

@pytest.mark.parametrize("symmetric", [False, True])
def test_writer_and_reader_match_reference_library(ref, tmp_path, symmetric):
    s = host.assemble("cavity", 2, 8)
    for w in ("A", "B", "Q"):
        sym = symmetric and w != "B"
        mine, theirs = tmp_path / f"m_{w}.mtx", tmp_path / f"r_{w}.mtx"
        host.write_matrix_market(getattr(s, w), str(mine), sym)
        ref.write_matrix_market(to_oracle(getattr(s, w)), str(theirs), sym)
        assert mine.read_bytes() == theirs.read_bytes(), w
        a, r = host.read_matrix_market(str(theirs)), ref.read_matrix_market(str(theirs))
        assert same(a, host.CsrMatrix(r.n_rows, r.n_cols, r.rp, r.ci, r.v)), w


def test_reader_matches_reference_on_messy_input(ref, tmp_path):
    """Duplicates, unsorted entries, entries split across lines, comments."""
    rng = np.random.default_rng(7)
    n, k = 40, 600
    i, j = rng.integers(1, n + 1, k), rng.integers(1, n + 1, k)
    v = rng.standard_normal(k)
    body = "".join(f"{a} {b}\n{float(x)!r}\n" for a, b, x in zip(i, j, v))
    for qual in ("general", "symmetric"):
        if qual == "symmetric":
            keep = i >= j
            body = "".join(f"{a} {b} {float(x)!r}\n" for a, b, x in zip(i[keep], j[keep], v[keep]))
            cnt = int(keep.sum())
        else:
            cnt = k
        p = tmp_path / f"messy_{qual}.mtx"
        p.write_text(f"%%MatrixMarket matrix coordinate real {qual}\n%c\n{n} {n} {cnt}\n{body}")
        a, r = host.read_matrix_market(str(p)), ref.read_matrix_market(str(p))
        assert same(a, host.CsrMatrix(r.n_rows, r.n_cols, r.rp, r.ci, r.v)), qual
