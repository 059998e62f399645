"""TEST INFRASTRUCTURE ONLY: ctypes binding of the C oracle (oracle/oracle.c).

Bit-identical to :mod:`oracle.np_oracle` (same per-term rounding, canonical
order); parallel over rows with OpenMP.  Used by the tests for full-size
parity and by ``bench.py`` as the timed CPU baseline (``kind: "port"``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (outputs only under oracle/_build)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        for name, ptr in (("sbo_sweep_f64", ctypes.c_double), ("sbo_sweep_f32", ctypes.c_float)):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                           ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ptr),
                           ctypes.c_int64, ctypes.c_int]
        lib.sbo_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().sbo_max_threads())


def sweep(box: np.ndarray, r: int, offsets, weights, steps: int,
          threads: int | None = None, inplace: bool = False) -> np.ndarray:
    """``steps`` oracle steps on a compact halo-inclusive box.

    ``box.dtype`` float64 runs the fp64 restatement; float32 runs the same
    arithmetic in fp32 (weights rounded to fp32).
    """
    lib = _load()
    d = box.ndim
    dims = np.array([s - 2 * r for s in box.shape], dtype=np.int64)
    offs = np.ascontiguousarray(np.array(offsets, dtype=np.int32).reshape(-1))
    w = np.ascontiguousarray(np.array(weights, dtype=np.float64))
    if box.dtype == np.float64:
        fn, ctype = lib.sbo_sweep_f64, ctypes.c_double
    elif box.dtype == np.float32:
        fn, ctype = lib.sbo_sweep_f32, ctypes.c_float
    else:
        raise TypeError(f"unsupported dtype {box.dtype}")
    out = box if inplace else np.array(box, copy=True, order="C")
    if not out.flags.c_contiguous:
        raise ValueError("box must be C-contiguous")
    rc = fn(d, r, len(w), offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            out.ctypes.data_as(ctypes.POINTER(ctype)), int(steps),
            int(threads or max_threads()))
    if rc != 0:
        raise RuntimeError(f"oracle sweep failed with status {rc}")
    return out
