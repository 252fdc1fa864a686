"""Matrix Market fixtures written by the UNMODIFIED reference's
write_matrix_market (proj/src/csr.cpp:126-142), the way its runner dumps a
system (--dump-matrices, runner.cpp:223-229: A and Q symmetric, B general).

Run here (where oracle/_ref/libdivstokes_ref.so is built):
``python tests/golden/make_golden_mm.py``. Writes tests/golden/mm/:
  A_psi_k2_h3.mtx, B_psi_k2_h3.mtx, Q_psi_k2_h3.mtx  psi-MMS, k'=2, 3x3 elements
  f_psi_k2_h3.npy                                      its velocity right-hand side
  rect_3x5.mtx                                         the reference test's 3x5 case
                                                       (test_sparse.cpp:149-152)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import CSR, RefLib  # noqa: E402


def main():
    R = RefLib()
    out = os.path.join(HERE, "mm")
    os.makedirs(out, exist_ok=True)
    s = R.assemble("psi-mms", 2, 3)
    R.write_matrix_market(s.block("A"), os.path.join(out, "A_psi_k2_h3.mtx"), True)
    R.write_matrix_market(s.block("B"), os.path.join(out, "B_psi_k2_h3.mtx"), False)
    R.write_matrix_market(s.block("Q"), os.path.join(out, "Q_psi_k2_h3.mtx"), True)
    np.save(os.path.join(out, "f_psi_k2_h3.npy"), s.rhs())
    rect = CSR(3, 5, np.array([0, 1, 2, 3], np.int64), np.array([4, 0, 2], np.int32),
               np.array([1.5, -2.0, 0.25]))
    R.write_matrix_market(rect, os.path.join(out, "rect_3x5.mtx"), False)


if __name__ == "__main__":
    main()
