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
* :func:`register` -- adds ``"b200"`` (NATURAL) and, when the registry's
  Layout enum has them, ``"b200_transpose"`` (BLOCK_TRANSPOSE, the layout of
  the reference's ``"transpose"`` method and of ``jam_sweep``) and
  ``"b200_dlt"`` (DLT) to a reference ``METHODS`` registry.

Grids in BLOCK_TRANSPOSE or DLT layout travel as whole storage arrays and are
permuted to and from the natural order on the device (``sb_upload_storage``
/ ``sb_download_storage``, ``csrc/layout.cuh``); the sweep itself always runs
the natural-order kernels, so results are bit-identical to the reference's
``transpose_layout_step`` / ``dlt_step`` / ``jam_sweep`` (which are
bit-identical to ``scalar_step``, test_kernels.py:82, test_timejam.py:94).
"""

from __future__ import annotations

import numpy as np

from .core import GridError, validate
from .grid import compact_view, interior_view, is_natural, layout_value, unit_permutation
from .plan import cached_plan


def _check_pair(src, dst) -> None:
    # kernels.py:111-117
    if src is dst:
        raise GridError("single steps are out-of-place: src and dst must differ")
    if layout_value(src) != layout_value(dst):
        raise GridError("src and dst grids have different layouts")
    if tuple(src.dims) != tuple(dst.dims) or src.unit_np != dst.unit_np or \
            getattr(src, "vl", 4) != getattr(dst, "vl", 4):
        raise GridError("src and dst grids have mismatched geometry")


def _points(grid) -> int:
    n = 1
    for x in grid.dims:
        n *= int(x)
    return n


def _check_ranges(ranges, dims):
    ranges = [(int(lo), int(hi)) for lo, hi in ranges]
    if len(ranges) != len(dims):
        raise GridError(f"ranges has {len(ranges)} axes, grid has {len(dims)}")
    for (lo, hi), n in zip(ranges, dims):
        if lo < 0 or hi > n:
            raise GridError(f"range ({lo}, {hi}) outside an axis of extent {n}")
    return ranges


def _store_interior(dst, storage: np.ndarray, ranges=None) -> None:
    """Copy the interior (or the ``ranges`` box) of a storage array in dst's
    layout into ``dst.data``; everything else of dst stays as it was."""
    hu = dst.halo_unit
    perm = unit_permutation(layout_value(dst), dst.unit_np, getattr(dst, "vl", 4))
    if ranges is None:
        ranges = [(0, n) for n in dst.dims]
    outer = tuple(slice(dst.r + lo, dst.r + hi) for lo, hi in ranges[:-1])
    cols = hu + perm[ranges[-1][0]:ranges[-1][1]]
    dst.data[outer + (cols,)] = storage[outer + (cols,)]


def b200_step(src, dst, spec, counters=None, ranges=None, *, arith="exact") -> None:
    """One sweep ``dst = S(src)`` on the GPU (signature of kernels.py:120-134).

    ``ranges`` = [(lo, hi)] per axis restricts the step to that interior
    sub-box, as the reference's tiled runner drives it (tiling.py:353-354):
    the device computes only the box and only the box of ``dst`` is written;
    counters count the box's points (kernels.py:127-134).  NATURAL grids move
    only the box plus its r-deep neighbourhood host<->device; BLOCK_TRANSPOSE
    / DLT grids are un-permuted whole on the device and stepped with
    sb_step_box.
    Grids may be NATURAL, BLOCK_TRANSPOSE or DLT (both in the same layout).
    """
    _check_pair(src, dst)
    validate(spec)
    r = spec.r
    natural = is_natural(src)
    if ranges is not None:
        ranges = _check_ranges(ranges, src.dims)
        if any(hi <= lo for lo, hi in ranges):
            return                                   # empty box: nothing computed or counted
    if ranges is not None and natural:
        # Only the box and its r-deep neighbourhood travel: the box is swept as
        # a grid of its own whose halo is src's values around it (the cells the
        # step reads, kernels.py:103-108), so each point sums the same terms in
        # the same order as in a whole-grid step.
        sub = compact_view(src, r)[tuple(slice(lo, hi + 2 * r) for lo, hi in ranges)]
        p = cached_plan(spec, tuple(hi - lo for lo, hi in ranges), arith=arith, k=1, kernel="generic")
        p.upload(np.ascontiguousarray(sub, dtype=np.float64))
        p.run(1)
        out = p.download()
        interior_view(dst)[tuple(slice(lo, hi) for lo, hi in ranges)] = \
            out[tuple(slice(r, s - r) for s in out.shape)]
        _count(counters, spec, int(np.prod([hi - lo for lo, hi in ranges])))
        return
    if not natural and src.r != r:
        raise GridError(f"{layout_value(src)} grid sized for order {src.r}, stencil order {r}")
    kernel = "generic" if ranges is not None else "auto"
    p = cached_plan(spec, tuple(src.dims), arith=arith, k=1, kernel=kernel)
    sd = src.data
    if (natural and src.r == r and sd.dtype == np.float64 and sd.flags.c_contiguous and sd.ndim >= 2):
        # the storage array is the host box with a row pitch: no compacting copy (see b200_sweep);
        # dst takes only its interior below (its own halo stays, kernels.py:120-134)
        p.upload_pitched(sd.ctypes.data + (src.halo_unit - r) * sd.itemsize, sd.shape[-1] * sd.itemsize)
    elif natural:
        p.upload(np.ascontiguousarray(compact_view(src, r), dtype=np.float64))
    else:
        p.upload_storage(src)
    if ranges is not None:
        p.step_box(ranges)
    else:
        p.run(1)
    out = p.download() if natural else p.download_storage(src)
    if natural:
        if ranges is None:
            interior_view(dst)[...] = out[tuple(slice(r, s - r) for s in out.shape)]
        else:
            sel = tuple(slice(lo, hi) for lo, hi in ranges)
            sel_box = tuple(slice(r + lo, r + hi) for lo, hi in ranges)
            interior_view(dst)[sel] = out[sel_box]
    else:
        _store_interior(dst, out, ranges)
    _count(counters, spec, _points(src) if ranges is None else int(np.prod([hi - lo for lo, hi in ranges])))


def _count(counters, spec, pts: int) -> None:
    """Meter one step over ``pts`` points as scalar_step does (kernels.py:127-134)."""
    if counters is not None:
        counters.point_updates += pts
        counters.scalar_loads += len(spec.weights) * pts
        counters.scalar_stores += pts


def b200_sweep(grid, spec, k, T, counters=None, *, arith="exact") -> None:
    """Advance ``grid`` T steps in place, k fused steps per launch (timejam.py:288-304).

    Unlike the reference register pipeline (k in {1, 2}, 1D, r <= 2,
    BLOCK_TRANSPOSE only), any dimension, layout (NATURAL, BLOCK_TRANSPOSE,
    DLT) and any k the fused kernels support is accepted; T need not be a
    multiple of k (the tail runs at smaller k).
    """
    validate(spec)
    if T < 0:
        raise GridError(f"total steps T={T} must be >= 0")
    natural = is_natural(grid)
    if not natural and grid.r != spec.r:
        raise GridError(f"{layout_value(grid)} grid sized for order {grid.r}, stencil order {spec.r}")
    p = cached_plan(spec, tuple(grid.dims), arith=arith, k=k)
    data = grid.data
    # a NATURAL grid whose halo is the stencil's order is the C-ABI host box with a row
    # pitch (only the unit axis carries extra halo, core.py:335-362): moved in place, no
    # compacting host copies (768^3: ~2 s of numpy strided copies around a 0.1 s sweep)
    in_place = (natural and grid.r == spec.r and data.dtype == np.float64 and data.flags.c_contiguous
                and data.flags.writeable and data.ndim >= 2)
    if in_place:
        first = data.ctypes.data + (grid.halo_unit - spec.r) * data.itemsize
        pitch = data.shape[-1] * data.itemsize
        p.sweep_host_pitched(first, pitch, first, pitch, T)      # upload, T steps, write back
        if counters is not None:
            counters.point_updates += _points(grid) * T
        return
    if natural:
        p.upload(np.ascontiguousarray(compact_view(grid, spec.r), dtype=np.float64))
    else:
        p.upload_storage(grid)
    p.run(T)
    if natural:
        out = p.download()
        interior_view(grid)[...] = out[tuple(slice(spec.r, s - spec.r) for s in out.shape)]
    else:
        out = p.download_storage(grid)
        _store_interior(grid, out)
    if counters is not None:
        counters.point_updates += _points(grid) * T


def register(methods: dict, layout) -> None:
    """Register the b200 methods in a reference METHODS dict (kernels.py:538-544).

    ``layout`` is the registry's Layout enum (or any of its members, e.g.
    ``Layout.NATURAL`` as in ``register(METHODS, Layout.NATURAL)``).
    """
    enum = layout if isinstance(layout, type) else type(layout)
    methods["b200"] = (getattr(enum, "NATURAL", layout), b200_step)
    if hasattr(enum, "BLOCK_TRANSPOSE"):
        methods["b200_transpose"] = (enum.BLOCK_TRANSPOSE, b200_step)
    if hasattr(enum, "DLT"):
        methods["b200_dlt"] = (enum.DLT, b200_step)


__all__ = ["b200_step", "b200_sweep", "register"]
