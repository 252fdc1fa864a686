"""Locate and load the in-tree native libraries. No fallback: a missing or
unloadable library raises, so nothing silently runs a non-native path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.environ.get("DSGPU_LIB_DIR", os.path.join(HERE, "lib"))
HOST_SO = os.path.join(LIB_DIR, "libdshost.so")
GPU_SO = os.path.join(LIB_DIR, "libdsgpu.so")

_cache: dict[str, C.CDLL] = {}


class NativeLibraryMissing(RuntimeError):
    pass


def _load(path: str) -> C.CDLL:
    if path not in _cache:
        if not os.path.exists(path):
            raise NativeLibraryMissing(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_1309_5048_b200/csrc`")
        _cache[path] = C.CDLL(path)
    return _cache[path]


def load_host() -> C.CDLL:
    return _load(HOST_SO)


def load_gpu() -> C.CDLL:
    return _load(GPU_SO)


def build(verbose: bool = False) -> None:
    import subprocess

    out = subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j8"], capture_output=True,
                         text=True)
    if verbose or out.returncode != 0:
        print(out.stdout[-4000:], out.stderr[-4000:])
    if out.returncode != 0:
        raise RuntimeError("native build failed")
