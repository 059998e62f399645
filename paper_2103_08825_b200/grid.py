"""NATURAL-layout grid buffers: the host mirror of ``stencilbench.core.GridBuffer``.

Restates the storage contract of ``core.py:232-373`` for the natural layout
-- halo r on outer axes, 2r on the unit axis (``UNIT_HALO_FACTOR``,
``core.py:35``), zero-initialised, halo read-only -- so drop-in callers and
the parity tests can hand the same objects to the reference and to sb200.
Reference ``GridBuffer`` instances are accepted anywhere a grid is taken
(duck-typed on ``data``, ``dims``, ``r``, ``halo_unit``, ``unit_n``, ``layout``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import GridError

UNIT_HALO_FACTOR = 2


class Layout:
    """Stand-in for ``stencilbench.core.Layout`` (only NATURAL is native here)."""

    class _Tag:
        def __init__(self, value):
            self.value = value

        def __repr__(self):
            return f"Layout.{self.value.upper()}"

    NATURAL = _Tag("natural")


@dataclass
class GridBuffer:
    data: np.ndarray
    dims: tuple[int, ...]
    r: int
    unit_n: int
    unit_np: int
    layout: object = Layout.NATURAL
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

    def natural_interior(self) -> np.ndarray:
        return interior_view(self).copy()

    def set_interior(self, values) -> None:
        values = np.asarray(values, dtype=np.float64)
        if values.shape != tuple(self.dims):
            raise GridError(f"expected shape {self.dims}, got {values.shape}")
        interior_view(self)[...] = values

    def clone(self) -> "GridBuffer":
        g = alloc_like(self)
        g.data[...] = self.data
        return g


def alloc_grid(spec, dims) -> GridBuffer:
    """Zeroed NATURAL grid for ``spec`` (core.py:335-362, natural layout)."""
    dims = (dims,) if isinstance(dims, int) else tuple(int(n) for n in dims)
    if len(dims) != spec.d:
        raise GridError(f"{getattr(spec, 'name', 'spec')} needs {spec.d} extents, got {len(dims)}")
    if any(n <= 0 for n in dims):
        raise GridError(f"extents must be positive, got {dims}")
    hu = UNIT_HALO_FACTOR * spec.r
    shape = tuple(n + 2 * spec.r for n in dims[:-1]) + (dims[-1] + 2 * hu,)
    return GridBuffer(np.zeros(shape), dims, spec.r, dims[-1], dims[-1])


def alloc_like(grid) -> GridBuffer:
    return GridBuffer(np.zeros_like(grid.data), tuple(grid.dims), grid.r, grid.unit_n,
                      grid.unit_np, grid.layout, getattr(grid, "vl", 4))


def is_natural(grid) -> bool:
    layout = getattr(grid, "layout", None)
    return getattr(layout, "value", None) == "natural"


def compact_view(grid) -> np.ndarray:
    """Halo-inclusive compact box view (C-ABI host convention) of a grid.

    Outer axes keep their r halo; on the unit axis the r cells adjacent to the
    interior (the only ones NATURAL sweeps read, kernels.py:89-100).
    """
    r, hu = grid.r, grid.halo_unit
    return grid.data[..., hu - r:hu + grid.unit_n + r]


def interior_view(grid) -> np.ndarray:
    r, hu = grid.r, grid.halo_unit
    outer = tuple(slice(r, r + n) for n in grid.dims[:-1])
    return grid.data[outer + (slice(hu, hu + grid.unit_n),)]
