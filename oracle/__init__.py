"""TEST INFRASTRUCTURE — CPU checkers for the MINRES + IC(0) Stokes solve.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package. The product package
(``paper_1309_5048_b200``) never imports it and has no CPU fallback.

Two checkers, both built by ``oracle/Makefile`` into ``oracle/_ref/``:

* ``RefLib`` — the unmodified reference library (``/root/reference/proj/src``)
  behind ``ref_driver.cpp``'s extern "C" entry points;
* ``PortLib`` — the plain-C restatement ``ds_oracle.c``.
"""
from .oracle import CSR, PortLib, RefLib, build, ref_available  # noqa: F401
