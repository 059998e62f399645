"""Grid buffers: the host mirror of ``stencilbench.core.GridBuffer``.

Restates the storage contract of ``core.py:232-373`` -- halo r on outer
axes, 2r on the unit axis (``UNIT_HALO_FACTOR``, ``core.py:35``), the unit
extent padded to the layout's block multiple (``core.py:191-203``),
zero-initialised, halo and padding read-only -- so drop-in callers and the
parity tests can hand the same objects to the reference and to sb200.
Reference ``GridBuffer`` instances are accepted anywhere a grid is taken
(duck-typed on ``data``, ``dims``, ``r``, ``halo_unit``, ``unit_n``,
``unit_np``, ``layout``, ``vl``).

The sm_100a kernels always sweep the NATURAL order; BLOCK_TRANSPOSE and DLT
grids are permuted to and from it on the device (``csrc/layout.cuh``,
``sb_upload_storage`` / ``sb_download_storage``).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from functools import lru_cache

import numpy as np

from .core import GridError

UNIT_HALO_FACTOR = 2
SUPPORTED_VL = (4, 8)   # core.py:31


class Layout(Enum):
    """Storage order of the unit-stride dimension (values of ``core.Layout``, core.py:46-51)."""

    NATURAL = "natural"
    BLOCK_TRANSPOSE = "block_transpose"
    DLT = "dlt"


def layout_value(grid_or_layout) -> str:
    """'natural' | 'block_transpose' | 'dlt' for a grid or a layout member of
    either this module's enum or the reference's."""
    lay = getattr(grid_or_layout, "layout", grid_or_layout)
    val = getattr(lay, "value", None)
    if val not in ("natural", "block_transpose", "dlt"):
        raise GridError(f"unsupported layout {lay!r}")
    return val


def _pad_multiple(layout: str, vl: int) -> int:
    # core.py:198-203
    return {"block_transpose": vl * vl, "dlt": vl}.get(layout, 1)


@lru_cache(maxsize=64)
def unit_permutation(layout: str, unit_np: int, vl: int) -> np.ndarray:
    """Natural unit index -> storage offset in the padded region (core.py:206-229).

    BLOCK_TRANSPOSE moves block offset o to (o mod vl)*vl + o//vl; DLT moves
    q*(N/vl)+c to c*vl+q; NATURAL is the identity.  Host-side index map used by
    the grid accessors; the device applies the same map in csrc/layout.cuh.
    """
    if not isinstance(layout, str):
        layout = layout_value(layout)
    idx = np.arange(unit_np, dtype=np.int64)
    if layout == "natural":
        return idx
    if layout == "block_transpose":
        if unit_np % (vl * vl):
            raise GridError(f"extent {unit_np} not a multiple of {vl * vl}")
        o = idx % (vl * vl)
        return idx - o + (o % vl) * vl + o // vl
    if unit_np % vl:
        raise GridError(f"extent {unit_np} not a multiple of {vl}")
    sub = unit_np // vl
    return (idx % sub) * vl + idx // sub


@dataclass
class GridBuffer:
    data: np.ndarray
    dims: tuple[int, ...]
    r: int
    unit_n: int
    unit_np: int
    layout: Layout = Layout.NATURAL
    vl: int = 4

    @property
    def d(self) -> int:
        return len(self.dims)

    @property
    def halo_unit(self) -> int:
        return UNIT_HALO_FACTOR * self.r

    @property
    def halo_outer(self) -> int:
        return self.r

    @property
    def interior_points(self) -> int:
        return int(np.prod(self.dims))

    def natural_interior(self) -> np.ndarray:
        """Interior values in natural order (core.py:308-316)."""
        return interior_natural(self)

    def set_interior(self, values) -> None:
        """Write natural-order interior values through the layout map (core.py:318-327)."""
        values = np.asarray(values, dtype=np.float64)
        if values.shape != tuple(self.dims):
            raise GridError(f"expected shape {self.dims}, got {values.shape}")
        perm = unit_permutation(layout_value(self), self.unit_np, self.vl)
        region = _outer_interior(self)[..., self.halo_unit:self.halo_unit + self.unit_np]
        region[..., perm[:self.unit_n]] = values

    def clone(self) -> "GridBuffer":
        g = alloc_like(self)
        g.data[...] = self.data
        return g


def alloc_grid(spec, dims, layout: Layout = Layout.NATURAL, vl: int = 4, pad_for=None) -> GridBuffer:
    """Zeroed grid for ``spec`` (core.py:335-362): halo r on outer axes, 2r on
    the unit axis, unit extent padded to the (pad_for) layout's block multiple."""
    if vl not in SUPPORTED_VL:
        raise GridError(f"vl must be one of {SUPPORTED_VL}, got {vl}")
    dims = (dims,) if isinstance(dims, (int, np.integer)) else tuple(int(n) for n in dims)
    if len(dims) != spec.d:
        raise GridError(f"{getattr(spec, 'name', 'spec')} needs {spec.d} extents, got {len(dims)}")
    if any(n <= 0 for n in dims):
        raise GridError(f"extents must be positive, got {dims}")
    lay = Layout(layout_value(layout))
    pad_layout = layout_value(pad_for) if (lay is Layout.NATURAL and pad_for is not None) else lay.value
    mult = _pad_multiple(pad_layout, vl)
    unit_n = dims[-1]
    unit_np = -(-unit_n // mult) * mult
    hu = UNIT_HALO_FACTOR * spec.r
    shape = tuple(n + 2 * spec.r for n in dims[:-1]) + (unit_np + 2 * hu,)
    return GridBuffer(np.zeros(shape), dims, spec.r, unit_n, unit_np, lay, vl)


def alloc_like(grid) -> GridBuffer:
    lay = Layout(layout_value(grid))
    return GridBuffer(np.zeros_like(grid.data), tuple(grid.dims), grid.r, grid.unit_n,
                      grid.unit_np, lay, getattr(grid, "vl", 4))


def is_natural(grid) -> bool:
    layout = getattr(grid, "layout", None)
    return getattr(layout, "value", None) == "natural"


def storage_rows(grid) -> int:
    """Number of unit-stride rows of the storage (outer halo rows included)."""
    return int(np.prod(grid.data.shape[:-1])) if grid.data.ndim > 1 else 1


def compact_view(grid, r: int | None = None) -> np.ndarray:
    """Halo-inclusive compact box view (C-ABI host convention) of a NATURAL grid.

    ``r`` is the stencil order of the sweep (default: the order the grid was
    allocated for).  A grid sized for a larger order than the stencil's is
    legal in the reference (``_region`` offsets by the grid's own halo,
    kernels.py:88-100): the view keeps the r cells next to the interior on
    every axis -- the only ones a NATURAL sweep of order r reads.
    """
    g_r, hu = grid.r, grid.halo_unit
    r = g_r if r is None else int(r)
    if r > g_r:
        raise GridError(f"grid halo sized for order {g_r} cannot serve a stencil of order {r}")
    outer = tuple(slice(g_r - r, g_r + n + r) for n in grid.dims[:-1])
    return grid.data[outer + (slice(hu - r, hu + grid.unit_n + r),)]


def _outer_interior(grid) -> np.ndarray:
    r = grid.r
    return grid.data[tuple(slice(r, r + n) for n in grid.dims[:-1])]


def interior_view(grid) -> np.ndarray:
    """View of the interior of a NATURAL grid."""
    hu = grid.halo_unit
    return _outer_interior(grid)[..., hu:hu + grid.unit_n]


def interior_natural(grid) -> np.ndarray:
    """Interior values of a grid in any layout, natural order, as a fresh array."""
    hu = grid.halo_unit
    perm = unit_permutation(layout_value(grid), grid.unit_np, getattr(grid, "vl", 4))
    region = _outer_interior(grid)[..., hu:hu + grid.unit_np]
    return region[..., perm[:grid.unit_n]].copy()
