"""B200-native MINRES + IC(0) block-preconditioned Stokes solve (arXiv 1309.5048).

Drop-in for the reference's ``solve_stokes`` (proj/src/precond.cpp:245-299):
``host`` builds BASELINE's systems and the RCM/IC(0) setup natively,
``solver`` runs the whole preconditioned MINRES on one sm_100a cooperative
kernel through the C ABI in ``include/dsgpu.h``.
"""
from . import host  # noqa: F401
from .host import StokesSystem, assemble  # noqa: F401
from .solver import (GpuStokesSolver, SolverOptions, StokesSolution, solve_stokes,  # noqa: F401
                     strategy_names)

__all__ = ["host", "assemble", "StokesSystem", "GpuStokesSolver", "SolverOptions",
           "StokesSolution", "solve_stokes", "strategy_names"]
