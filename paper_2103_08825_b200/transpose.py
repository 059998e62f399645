"""Layout conversions on the GPU: drop-ins for ``stencilbench.transpose``.

``to_block_transpose`` / ``from_block_transpose`` / ``to_dlt`` / ``from_dlt``
keep the reference's signatures, checks and in-place semantics
(transpose.py:286-357: the grid's storage is permuted and the grid retagged;
unit-axis halo cells stay where they are), but the permutation runs on the
device through ``sb_layout_convert`` (csrc/layout.cuh: shared-memory staged
tiles, coalesced on both sides).  :func:`convert_device` is the
device-resident form for torch CUDA tensors (no host copies).

PyTorch only provides device memory and the stream here; there is no CPU
path -- without the library or a GPU the calls raise.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from .core import GridError
from .grid import Layout, layout_value
from .plan import storage_descriptor


def _retag(grid, value: str) -> None:
    enum = type(grid.layout)
    grid.layout = enum(value) if hasattr(enum, "NATURAL") else Layout(value)


def convert_device(src, dst, grid_like, to_layout: bool, layout: str | None = None, vl: int | None = None) -> None:
    """Convert device storage ``src`` -> ``dst`` (torch CUDA tensors shaped like
    ``grid_like.data``, float64 or float32) on torch's current stream.

    ``to_layout`` True: NATURAL ``src`` -> ``layout`` (default: grid_like's) in
    ``dst``; False: the inverse.
    """
    import torch

    if not (src.is_cuda and dst.is_cuda) or src.shape != dst.shape or src.dtype != dst.dtype:
        raise GridError("convert_device needs two CUDA tensors of the same shape and dtype")
    if not (src.is_contiguous() and dst.is_contiguous()):
        raise GridError("storage tensors must be contiguous")
    st = storage_descriptor(grid_like)
    if layout is not None:
        st.layout = {"natural": 0, "block_transpose": 1, "dlt": 2}[layout]
    if vl is not None:
        st.vl = int(vl)
    dtype = {torch.float64: _abi.SB_F64, torch.float32: _abi.SB_F32}.get(src.dtype)
    if dtype is None:
        raise GridError(f"unsupported dtype {src.dtype}")
    rows = src.numel() // src.shape[-1] if src.dim() else 0
    stream = torch.cuda.current_stream(src.device).cuda_stream
    with torch.cuda.device(src.device):
        _abi.check(_abi.load().sb_layout_convert(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                                 rows, ctypes.byref(st), 1 if to_layout else 0, dtype,
                                                 ctypes.c_void_p(stream)))


def _convert_inplace(grid, target: str, to_layout: bool, vl: int) -> None:
    import torch

    data = grid.data
    if data.dtype not in (np.float64, np.float32):
        raise GridError(f"unsupported storage dtype {data.dtype}")
    src = torch.from_numpy(np.ascontiguousarray(data)).cuda()
    dst = torch.empty_like(src)
    convert_device(src, dst, grid, to_layout, layout=target, vl=vl)
    grid.data[...] = dst.cpu().numpy().reshape(data.shape)


def to_block_transpose(grid, vl: int):
    """NATURAL -> BLOCK_TRANSPOSE in place, retagged (transpose.py:286-301)."""
    if layout_value(grid) != "natural":
        raise GridError(f"expected NATURAL grid, got {grid.layout}")
    if vl != grid.vl:
        raise GridError(f"grid was allocated for vl={grid.vl}, got {vl}")
    if grid.unit_np % (vl * vl):
        raise GridError(f"unit extent {grid.unit_np} not padded to a multiple of {vl * vl}")
    _convert_inplace(grid, "block_transpose", True, vl)
    _retag(grid, "block_transpose")
    return grid


def from_block_transpose(grid):
    """Inverse of :func:`to_block_transpose` (transpose.py:303-311)."""
    if layout_value(grid) != "block_transpose":
        raise GridError(f"expected BLOCK_TRANSPOSE grid, got {grid.layout}")
    _convert_inplace(grid, "block_transpose", False, grid.vl)
    _retag(grid, "natural")
    return grid


def to_dlt(grid, vl: int):
    """NATURAL -> DLT in place, retagged (transpose.py:314-336)."""
    if layout_value(grid) != "natural":
        raise GridError(f"expected NATURAL grid, got {grid.layout}")
    if vl != grid.vl:
        raise GridError(f"grid was allocated for vl={grid.vl}, got {vl}")
    if grid.unit_np % vl:
        raise GridError(f"unit extent {grid.unit_np} not divisible by {vl}")
    _convert_inplace(grid, "dlt", True, vl)
    _retag(grid, "dlt")
    return grid


def from_dlt(grid):
    """Inverse of :func:`to_dlt` (transpose.py:339-357)."""
    if layout_value(grid) != "dlt":
        raise GridError(f"expected DLT grid, got {grid.layout}")
    _convert_inplace(grid, "dlt", False, grid.vl)
    _retag(grid, "natural")
    return grid


__all__ = ["to_block_transpose", "from_block_transpose", "to_dlt", "from_dlt", "convert_device"]
