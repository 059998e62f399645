"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference scalar oracle.

Follows ``stencilbench/kernels.py:89-108`` (``_region`` +
``_natural_accumulate``) and ``stencilbench/harness.py:149-157``
(``run_oracle``): per step, ``out[...] = 0.0`` then, for each offset in
canonical (lexicographic, ``core.py:96-103``) order,
``out += w * shifted_view`` -- one rounded multiply into a temporary and one
rounded add per term.  The halo is read and never written.

Grids use the C-ABI host convention: a compact C-order box of shape
``(n_0+2r, ..., n_{d-1}+2r)`` (interior plus an r-deep halo).
"""

from __future__ import annotations

import numpy as np


def canonical(weights: dict) -> tuple[list[tuple[int, ...]], list[float]]:
    """Offsets sorted lexicographically with their weights (core.py:96-103)."""
    offs = sorted(weights)
    return offs, [float(weights[o]) for o in offs]


def _interior(box: np.ndarray, r: int, shift=None) -> np.ndarray:
    d = box.ndim
    shift = shift or (0,) * d
    return box[tuple(slice(r + s, box.shape[a] - r + s) for a, s in enumerate(shift))]


def step(src: np.ndarray, dst: np.ndarray, r: int, offsets, weights) -> None:
    """One out-of-place oracle step (kernels.py:120-134)."""
    if src is dst:
        raise ValueError("single steps are out-of-place: src and dst must differ")
    out = _interior(dst, r)
    out[...] = 0.0
    for off, w in zip(offsets, weights):
        out += src.dtype.type(w) * _interior(src, r, off)


def sweep(box: np.ndarray, r: int, offsets, weights, steps: int) -> np.ndarray:
    """``steps`` oracle steps from ``box`` (not modified); returns the final box."""
    a = np.array(box, copy=True)
    b = np.array(box, copy=True)           # halo present in both buffers
    for _ in range(steps):
        step(a, b, r, offsets, weights)
        a, b = b, a
    return a


def max_rel_error(got: np.ndarray, want: np.ndarray) -> float:
    """``stencilbench/harness.py:214-216``: max |got-want| / max(|want|, tiny)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    denom = np.maximum(np.abs(want), np.finfo(np.float64).tiny)
    return float(np.max(np.abs(got - want) / denom)) if want.size else 0.0
