"""Drop-in method entry points for the reference's plugin interface.

The reference dispatches sweeps through ``METHODS: dict[str, (Layout,
step_fn)]`` (``stencilbench/kernels.py:538-544``) with the single-step
signature ``step(src, dst, spec, counters=None, ranges=None)`` and through
the multi-step in-place ``jam_sweep(grid, spec, k, T, counters=None)``
(``timejam.py:288-304``).  This module provides both, backed by the sm_100a
kernels:

* :func:`b200_step` -- METHODS-compatible single step (out-of-place, halo
  read-only, EXACT arithmetic: bit-identical to ``scalar_step``);
* :func:`b200_sweep` -- jam_sweep-compatible T-step in-place sweep with k
  fused steps per HBM round trip (any k the fused kernel supports);
* :func:`register` -- adds ``"b200"`` to a reference ``METHODS`` registry.
"""

from __future__ import annotations

import numpy as np

from .core import GridError, validate
from .grid import compact_view, interior_view, is_natural
from .plan import Plan


def _check_pair(src, dst) -> None:
    # kernels.py:111-117
    if src is dst:
        raise GridError("single steps are out-of-place: src and dst must differ")
    if not (is_natural(src) and is_natural(dst)):
        raise GridError("method requires natural layout on both grids")
    if tuple(src.dims) != tuple(dst.dims) or src.unit_np != dst.unit_np:
        raise GridError("src and dst grids have mismatched geometry")


def _points(grid) -> int:
    n = 1
    for x in grid.dims:
        n *= int(x)
    return n


def b200_step(src, dst, spec, counters=None, ranges=None, *, arith="exact") -> None:
    """One sweep ``dst = S(src)`` on the GPU (signature of kernels.py:120-134).

    ``ranges`` = [(lo, hi)] per axis restricts the step to that interior
    sub-box, as the reference's tiled runner drives it (tiling.py:353-354):
    the device computes only the box (sb_step_box) and only the box of
    ``dst`` is written; counters count the box's points (kernels.py:127-134).
    """
    _check_pair(src, dst)
    validate(spec)
    r = spec.r
    box = np.ascontiguousarray(compact_view(src), dtype=np.float64)
    if ranges is not None:
        ranges = [(int(lo), int(hi)) for lo, hi in ranges]
        if len(ranges) != len(src.dims):
            raise GridError(f"ranges has {len(ranges)} axes, grid has {len(src.dims)}")
        for (lo, hi), n in zip(ranges, src.dims):
            if lo < 0 or hi > n:
                raise GridError(f"range ({lo}, {hi}) outside an axis of extent {n}")
        if any(hi <= lo for lo, hi in ranges):
            return                                   # empty box: nothing computed or counted
        with Plan(spec, tuple(src.dims), arith=arith, k=1, kernel="generic") as p:
            p.upload(box)
            p.step_box(ranges)
            out = p.download()
        sel = tuple(slice(lo, hi) for lo, hi in ranges)
        sel_box = tuple(slice(r + lo, r + hi) for lo, hi in ranges)
        interior_view(dst)[sel] = out[sel_box]
        pts = int(np.prod([hi - lo for lo, hi in ranges]))
    else:
        with Plan(spec, tuple(src.dims), arith=arith, k=1) as p:
            p.upload(box)
            p.run(1)
            out = p.download()
        interior_view(dst)[...] = out[tuple(slice(r, s - r) for s in out.shape)]
        pts = _points(src)
    if counters is not None:
        counters.point_updates += pts
        counters.scalar_loads += len(spec.weights) * pts
        counters.scalar_stores += pts


def b200_sweep(grid, spec, k, T, counters=None, *, arith="exact") -> None:
    """Advance ``grid`` T steps in place, k fused steps per launch (timejam.py:288-304).

    Unlike the reference register pipeline (k in {1, 2}, 1D, r <= 2), any
    dimension and any k in {1, 2, 4, 8, 16} is accepted; T need not be a
    multiple of k (the tail runs at smaller k).
    """
    if not is_natural(grid):
        raise GridError("b200 sweep runs on natural-layout grids")
    validate(spec)
    if T < 0:
        raise GridError(f"total steps T={T} must be >= 0")
    box = np.ascontiguousarray(compact_view(grid), dtype=np.float64)
    with Plan(spec, tuple(grid.dims), arith=arith, k=k) as p:
        p.upload(box)
        p.run(T)
        out = p.download()
    interior_view(grid)[...] = out[tuple(slice(spec.r, s - spec.r) for s in out.shape)]
    if counters is not None:
        counters.point_updates += _points(grid) * T


def register(methods: dict, natural_layout) -> None:
    """Register ``"b200"`` in a reference METHODS dict (kernels.py:538-544)."""
    methods["b200"] = (natural_layout, b200_step)
