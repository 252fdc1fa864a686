"""The C-ABI libraries load and export every symbol include/*.h declares; the
GPU library refuses to run without a device (no CPU fallback). CPU only."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADERS = {"dsgpu.h": "libdsgpu.so", "dshost.h": "libdshost.so"}


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:dsgpu|dshost)_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", sorted(HEADERS.items()))
def test_exports_every_declared_symbol(header, lib):
    path = os.path.join(ROOT, "paper_1309_5048_b200", "lib", lib)
    L = C.CDLL(path)
    names = declared(header)
    assert len(names) >= 6
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_gpu_library_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = C.CDLL(os.path.join(ROOT, "paper_1309_5048_b200", "lib", "libdsgpu.so"))
    h = C.c_void_p()
    rc = L.dsgpu_create(0, C.byref(h))
    assert rc == 4 and not h.value  # DSGPU_E_CUDA


def test_python_mirror_has_no_fallback(monkeypatch):
    from paper_1309_5048_b200 import _lib
    monkeypatch.setattr(_lib, "GPU_SO", "/nonexistent/libdsgpu.so")
    _lib._cache.pop("/nonexistent/libdsgpu.so", None)
    with pytest.raises(_lib.NativeLibraryMissing):
        _lib.load_gpu()


def test_strategy_menu():
    from paper_1309_5048_b200 import solver
    assert "IC0-PCG(A,Q)" in solver.strategy_names()
    assert "IC0-PCG(A)+Diag(Q)" in solver.strategy_names()
