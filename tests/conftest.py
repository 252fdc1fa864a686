import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def port():
    from oracle import PortLib
    from oracle.oracle import PORT_SO, build
    if not os.path.exists(PORT_SO):
        build()
    return PortLib()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("reference library (oracle/_ref/libdivstokes_ref.so) not built")
    return RefLib()


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def golden_csr(d, name):
    from oracle import CSR
    shape = d[name + "_shape"]
    return CSR(int(shape[0]), int(shape[1]), d[name + "_rp"], d[name + "_ci"], d[name + "_v"])


def to_oracle(m):
    from oracle import CSR
    return CSR(m.n_rows, m.n_cols, m.row_ptr, m.cols, m.vals)


def to_host(m):
    from paper_1309_5048_b200.host import CsrMatrix
    return CsrMatrix(m.n_rows, m.n_cols, m.rp, m.ci, m.v)
