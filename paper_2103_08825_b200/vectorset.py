"""Device drop-in for the reference's vector-set step (kernels.py:404-511).

``vs_step(vs, left_deps, right_deps, cross_deps, spec)`` advances one vl x vl
block held as vl row vectors (``rows[j][l]`` = natural element
``base + l*vl + j``, core.py:167-182) by one time step, with its dependency
vectors at distances 1..r on each side (assembled by ``assemble_left/right``,
kernels.py:404-420) and, for d > 1, the co-located bands of the vertically
adjacent blocks (``Band``, kernels.py:423-445).  Lane l of output row j is

    sum over canonical offsets o of  w_o * band[o[:-1]].row(j + o[-1])[l]

with one rounded multiply and one rounded add per term (``fma`` of simd.py:129-131
rounds in between; ``_vs_step_1d`` nests the same products, kernels.py:448-475).

On the device every lane is an independent stencil evaluation, so the block
becomes one small grid: lane l's dependency rows -r .. vl+r-1 form a segment of
vl + 2r cells along the unit axis, the lanes' segments are laid end to end, and
for d > 1 the bands are stacked along the outer axes (band offset + r).  One
EXACT step of the generic kernel over that grid (canonical order, bit-identical
to the reference's arithmetic) produces every lane's outputs in place; cells
computed across segment joins or outside the centre band are discarded (each
kept output reads only its own segment and the stacked bands).  Plans are
cached per thread (``plan.cached_plan``).

This is the reference's per-block interface on a GPU -- correct, not fast: a
block is 16-64 values, so each call is dominated by two tiny host<->device
copies.  The fast path for whole grids is ``kernels.b200_sweep`` /
``b200_step``, which sweep the natural order directly.
"""

from __future__ import annotations

import itertools

import numpy as np

from .core import GridError, canonical, validate
from .plan import cached_plan


def _band_rows(rows, left, right, r, need_deps):
    """Rows -r .. vl+r-1 of a band (Band.row, kernels.py:436-445); dependency
    rows no kept output reads (star stencils' cross bands) may be absent."""
    vl = len(rows)
    if len(left) < r or len(right) < r:
        if need_deps:
            raise GridError(f"need {r} dependency vectors per side")
        zero = (0.0,) * vl
        left = tuple(left) + (zero,) * (r - len(left))
        right = tuple(right) + (zero,) * (r - len(right))
    return [left[m - 1] for m in range(r, 0, -1)] + list(rows) + [right[m] for m in range(r)]


def _lanes(v, vl):
    lanes = getattr(v, "lanes", v)
    if len(lanes) != vl:
        raise GridError(f"dependency vector has {len(lanes)} lanes, block has {vl}")
    return [float(x) for x in lanes]


def vs_step(vs, left_deps, right_deps, cross_deps, spec):
    """One time step of a vector set on the device (kernels.py:478-511 semantics)."""
    validate(spec)
    rows = tuple(vs.rows)
    vl = len(rows)
    r, d = spec.r, spec.d
    if len(left_deps) < r or len(right_deps) < r:
        raise GridError(f"need {r} dependency vectors per side")
    centre = (0,) * (d - 1)
    bands = {centre: (rows, tuple(left_deps), tuple(right_deps))}
    if d > 1 or cross_deps:
        for key, band in (cross_deps or {}).items():
            bands[tuple(key)] = (tuple(band.rows), tuple(getattr(band, "left", ())), tuple(getattr(band, "right", ())))
        for off in canonical(spec)[0]:
            if tuple(off[:-1]) not in bands:
                raise GridError(f"missing dependency band for outer offset {tuple(off[:-1])}")
    S = vl + 2 * r                      # cells per lane segment
    N = vl * S                          # unit-axis interior
    outer = (2 * r + 1,) * (d - 1)      # stacked bands, offset + r
    box = np.zeros(tuple(n + 2 * r for n in outer) + (N + 2 * r,))
    for key in itertools.product(range(-r, r + 1), repeat=d - 1):
        if key not in bands:
            continue                    # not read by any kept output (star stencils)
        b_rows, b_left, b_right = bands[key]
        if len(b_rows) != vl:
            raise GridError(f"band {key} has {len(b_rows)} rows, block has {vl}")
        need = any(tuple(o[:-1]) == key and o[-1] != 0 for o in canonical(spec)[0])
        ext = _band_rows(b_rows, b_left, b_right, r, need)   # S vectors of vl lanes
        seg = np.array([_lanes(v, vl) for v in ext]).T       # [lane][cell]
        idx = tuple(k + r + r for k in key)                  # box index of the stacked band
        box[idx + (slice(r, r + N),)] = seg.reshape(-1)
    p = cached_plan(spec, outer + (N,), arith="exact", k=1, kernel="generic")
    p.upload(box)
    p.run(1)
    out = p.download()
    line = out[tuple(r + r for _ in outer)] if d > 1 else out    # centre band
    vals = line[r: r + N].reshape(vl, S)[:, r: r + vl]           # [lane][row j]
    vtype = type(rows[0]) if rows and hasattr(rows[0], "lanes") else tuple
    new_rows = tuple(vtype(float(vals[l, j]) for l in range(vl)) for j in range(vl))
    try:
        return type(vs)(new_rows, getattr(vs, "base", 0))
    except TypeError:
        return new_rows


__all__ = ["vs_step"]
