"""ctypes binding of the C ABI (include/sb200.h), loaded from the in-tree
``lib/libsb200.so``.  There is no fallback: if the library is missing or no
CUDA device is present, calls fail loudly."""

from __future__ import annotations

import ctypes
import os

from .core import GridError, SpecError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SB200_LIB") or os.path.join(_PKG, "lib", "libsb200.so")  # override: dev only

SB_OK, SB_ERR_SPEC, SB_ERR_GRID, SB_ERR_ARG, SB_ERR_CUDA, SB_ERR_NOMEM, SB_ERR_STATE = 0, -1, -2, -3, -4, -5, -6
SB_F64, SB_F32 = 0, 1
SB_ARITH_EXACT, SB_ARITH_FMA = 0, 1
SB_STAR, SB_BOX = 0, 1
SB_KERNEL_AUTO, SB_KERNEL_GENERIC, SB_KERNEL_FUSED = 0, 1, 2
SB_LAYOUT_NATURAL, SB_LAYOUT_BLOCK_TRANSPOSE, SB_LAYOUT_DLT = 0, 1, 2

#: every symbol include/sb200.h declares (checked by tests/test_abi.py)
EXPORTS = ("sb_plan_create", "sb_plan_destroy", "sb_host_elems", "sb_upload",
           "sb_download", "sb_run", "sb_launch", "sb_set_stream", "sb_device_view",
           "sb_plan_k", "sb_kernel_count", "sb_last_error", "sb_abi_version", "sb_device_count",
           "sb_upload_async", "sb_download_async", "sb_synchronize", "sb_step_box",
           "sb_upload_storage", "sb_download_storage", "sb_layout_convert", "sb_launch_range",
           "sb_multi_create", "sb_multi_destroy", "sb_multi_upload", "sb_multi_download", "sb_multi_run",
           "sb_multi_info", "sb_multi_slab", "sb_problem_k", "sb_launch_repeat", "sb_repeat_times",
           "sb_upload_pitched", "sb_download_pitched", "sb_sweep_host")


class SbProblem(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("r", ctypes.c_int32), ("shape", ctypes.c_int32),
                ("nw", ctypes.c_int32),
                ("offsets", ctypes.POINTER(ctypes.c_int32)),
                ("weights", ctypes.POINTER(ctypes.c_double)),
                ("dims", ctypes.c_int64 * 3),
                ("dtype", ctypes.c_int32), ("arith", ctypes.c_int32), ("k", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("device", ctypes.c_int32),
                ("ghost_lo", ctypes.c_int32), ("ghost_hi", ctypes.c_int32)]


class SbTiming(ctypes.Structure):
    _fields_ = [("device_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("launches", ctypes.c_int64), ("point_updates", ctypes.c_int64),
                ("k_used", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("kernel_name", ctypes.c_char * 64)]


class SbStorage(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int32), ("vl", ctypes.c_int32), ("unit_n", ctypes.c_int64),
                ("unit_np", ctypes.c_int64), ("halo_unit", ctypes.c_int64)]


class CudaError(RuntimeError):
    """CUDA runtime failure (or no device) reported by the C ABI."""


_lib = None


def load():
    """Load libsb200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`python -m paper_2103_08825_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.sb_plan_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(SbProblem)]
    lib.sb_plan_destroy.argtypes = [P]
    lib.sb_plan_destroy.restype = None
    lib.sb_host_elems.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    lib.sb_upload.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_download.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_upload_async.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_upload_pitched.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_download_pitched.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_sweep_host.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64]
    lib.sb_download_async.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_synchronize.argtypes = [P]
    lib.sb_step_box.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.sb_run.argtypes = [P, ctypes.c_int64, ctypes.POINTER(SbTiming)]
    lib.sb_launch.argtypes = [P, ctypes.c_int64]
    lib.sb_launch_range.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
    lib.sb_set_stream.argtypes = [P, ctypes.c_void_p]
    lib.sb_device_view.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_int64), ctypes.c_int64 * 3]
    lib.sb_plan_k.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.sb_kernel_count.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    SP = ctypes.POINTER(SbStorage)
    lib.sb_upload_storage.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t, SP]
    lib.sb_download_storage.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t, SP]
    lib.sb_layout_convert.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, SP, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_void_p]
    lib.sb_multi_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(SbProblem), ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32)]
    lib.sb_multi_destroy.argtypes = [P]
    lib.sb_multi_destroy.restype = None
    lib.sb_multi_upload.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_multi_download.argtypes = [P, ctypes.c_void_p, ctypes.c_size_t]
    lib.sb_multi_run.argtypes = [P, ctypes.c_int64, ctypes.POINTER(SbTiming)]
    lib.sb_multi_info.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    lib.sb_multi_slab.argtypes = [P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int32)]
    lib.sb_problem_k.argtypes = [ctypes.POINTER(SbProblem), ctypes.POINTER(ctypes.c_int32)]
    lib.sb_launch_repeat.argtypes = [P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
    lib.sb_repeat_times.argtypes = [P, ctypes.POINTER(ctypes.c_float), ctypes.c_int32]
    lib.sb_last_error.restype = ctypes.c_char_p
    lib.sb_last_error.argtypes = []
    lib.sb_abi_version.restype = ctypes.c_int
    lib.sb_device_count.restype = ctypes.c_int
    for name in ("sb_plan_create", "sb_host_elems", "sb_upload", "sb_download", "sb_run",
                 "sb_launch", "sb_set_stream", "sb_device_view", "sb_plan_k", "sb_kernel_count",
                 "sb_upload_async", "sb_download_async", "sb_synchronize", "sb_step_box",
                 "sb_upload_storage", "sb_download_storage", "sb_layout_convert", "sb_launch_range",
                 "sb_multi_create", "sb_multi_upload", "sb_multi_download", "sb_multi_run",
                 "sb_multi_info", "sb_multi_slab", "sb_problem_k", "sb_launch_repeat", "sb_repeat_times",
           "sb_upload_pitched", "sb_download_pitched", "sb_sweep_host"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C status to the reference's exception types (core.py:38-43)."""
    if rc == SB_OK:
        return
    msg = (load().sb_last_error() or b"").decode(errors="replace")
    if rc == SB_ERR_SPEC:
        raise SpecError(msg)
    if rc == SB_ERR_GRID:
        raise GridError(msg)
    if rc == SB_ERR_ARG:
        raise ValueError(msg)
    if rc == SB_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == SB_ERR_STATE:
        raise RuntimeError(msg)
    raise CudaError(msg)


def device_count() -> int:
    return int(load().sb_device_count())
