"""ORACLE (test infrastructure only): loaders for the C oracle and for the
reference's own compiled ``_atomics`` (oracle/_ref/, built by oracle/Makefile
from /root/reference/pkg/src/asyncsgd/_atomics.c)."""

from __future__ import annotations

import ctypes
import importlib.machinery
import importlib.util
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True, capture_output=True)


def _lib() -> ctypes.CDLL:
    if not LIB.exists():
        build()
    lib = ctypes.CDLL(str(LIB))
    f, vp, sz = ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t
    lib.oracle_apply_sgd.argtypes = [vp, vp, vp, sz, f, f, f]
    lib.oracle_apply_sgd.restype = None
    lib.oracle_accum.argtypes = [vp, sz, sz, vp, sz, f]
    lib.oracle_accum.restype = ctypes.c_int
    lib.oracle_snapshot.argtypes = [vp, vp, sz]
    lib.oracle_snapshot.restype = None
    lib.oracle_average.argtypes = [ctypes.POINTER(vp), ctypes.c_int, sz, sz, vp]
    lib.oracle_average.restype = ctypes.c_int
    return lib


_L = None


def lib() -> ctypes.CDLL:
    global _L
    if _L is None:
        _L = _lib()
    return _L


def _f32(a: np.ndarray) -> np.ndarray:
    if a.dtype != np.float32 or not a.flags.c_contiguous:
        raise ValueError("oracle buffers must be C-contiguous float32")
    return a


def apply_sgd(x: np.ndarray, g: np.ndarray, m: np.ndarray | None, lr: float, mu: float = 0.0,
              wd: float = 0.0) -> None:
    _f32(x), _f32(g)
    mp = _f32(m).ctypes.data if m is not None else None
    lib().oracle_apply_sgd(x.ctypes.data, g.ctypes.data, mp, x.size, lr, mu, wd)


def accum(dst: np.ndarray, start: int, delta: np.ndarray, scale: float) -> None:
    _f32(dst), _f32(delta)
    if lib().oracle_accum(dst.ctypes.data, dst.size, start, delta.ctypes.data, delta.size, scale):
        raise IndexError("update range out of bounds")


def average(arenas: list[np.ndarray], lo: int, hi: int, mean_out: np.ndarray | None = None) -> None:
    ptrs = (ctypes.c_void_p * len(arenas))(*[_f32(a).ctypes.data for a in arenas])
    mp = _f32(mean_out).ctypes.data if mean_out is not None else None
    lib().oracle_average(ptrs, len(arenas), lo, hi, mp)


def reference_atomics():
    """The reference's compiled ``_atomics`` module, or None if not built."""
    cands = sorted((HERE / "_ref").glob("_atomics*.so"))
    if not cands:
        try:
            build()
        except Exception:
            return None
        cands = sorted((HERE / "_ref").glob("_atomics*.so"))
        if not cands:
            return None
    loader = importlib.machinery.ExtensionFileLoader("_atomics", str(cands[0]))
    spec = importlib.util.spec_from_file_location("_atomics", str(cands[0]), loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod
