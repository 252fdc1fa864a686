"""Drop-in check: the reference's own StokesSystem (assembled by the
unmodified reference) solved through integration/divstokes_gpu.cpp (a
reference-side shim over include/dsgpu.h) against the reference's own
solve_stokes on the same object."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SHIM = os.path.join(ROOT, "oracle", "_ref", "libdivstokes_gpu_shim.so")


@pytest.fixture(scope="module")
def shim(ref):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SHIM):
        pytest.skip("integration shim not built (needs the reference tree)")
    L = C.CDLL(SHIM)
    L.divstokes_gpu_solve.argtypes = [C.c_void_p, C.c_char_p, C.c_double, C.c_double, C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
    return L


@pytest.mark.parametrize("case,k,n,strategy,inner", [
    ("psi-mms", 2, 16, "IC0-PCG(A)+Diag(Q)", 1e-1),
    ("psi-mms", 2, 32, "IC0-PCG(A,Q)", 1e-1),
    ("cavity", 2, 16, "IC0-PCG(A,Q)", 1e-6),
    ("random", 3, 16, "IC0-PCG(A,Q)", 1e-1),
])
def test_shim_matches_reference_solve(ref, shim, case, k, n, strategy, inner):
    s = ref.assemble(case, k, n, seed=1234)
    r = s.solve(strategy, 1e-8, inner)
    u = np.zeros(s.n_u)
    p = np.zeros(s.n_p)
    rep = np.zeros(4)
    err = C.create_string_buffer(256)
    rc = shim.divstokes_gpu_solve(C.c_void_p(s.h), strategy.encode(), 1e-8, inner, 20000,
                                  u.ctypes.data, p.ctypes.data, rep.ctypes.data, err, 256)
    assert rc == 0, err.value
    x, xr = np.concatenate([u, p]), np.concatenate([r["u"], r["p"]])
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
    assert abs(int(rep[0]) - r["iterations"]) <= 2 and rep[1] == 1.0
    assert abs(rep[2] - r["mean_inner_top"]) < 0.2


def test_initial_guess_matches_reference_minres(ref):
    """MinresOptions::x0 (solvers.hpp:34, solvers.cpp:35-42) through
    dsgpu_set_initial_guess: the GPU solve started from a perturbed solution
    against the reference's own minres started from the same vector on the same
    system and preconditioner (no zero-mean filter on either side: that is
    solve_stokes's, not minres's). The guess is consumed by one solve."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.oracle import RefPrecond, ref_minres_x0
    from paper_1309_5048_b200 import host, solver
    rs = ref.assemble("psi-mms", 2, 16, seed=0)
    pre = RefPrecond(rs, "IC0-PCG(A,Q)", 1e-1)
    s = host.assemble("psi-mms", 2, 16)
    s.has_constant_pressure_kernel = False
    g = solver.GpuStokesSolver(s, "IC0-PCG(A,Q)")
    o = solver.SolverOptions(outer_tol=1e-8, inner_tol=1e-1)
    cold = g.solve(options=o)
    rng = np.random.default_rng(3)
    x0 = np.concatenate([cold.u, cold.p]) * (1.0 + 1e-3 * rng.standard_normal(s.size))
    r = ref_minres_x0(pre, x0, 1e-8)
    warm = g.solve(options=o, x0=(x0[:s.n_u], x0[s.n_u:]))
    x = np.concatenate([warm.u, warm.p])
    assert np.linalg.norm(x - r["x"]) <= 1e-8 * np.linalg.norm(r["x"])
    assert abs(warm.report.iterations - r["iterations"]) <= 2 and warm.report.converged == r["converged"]
    he, hr = warm.report.euclid_history, r["euclid_history"]
    m = min(len(he), len(hr))
    assert m > 1 and np.all(np.abs(he[:m] - hr[:m]) <= 1e-6 * np.maximum(hr[:m], 1e-12))
    again = g.solve(options=o)  # the guess was for one solve only
    assert again.report.iterations == cold.report.iterations
    assert np.array_equal(again.u, cold.u)
    g.close()
