"""Generate the golden fixtures by running the REFERENCE itself.

Run once in the build container (the reference is not present on the GPU
box):  ``python tests/golden/make_golden.py``.  It imports ``stencilbench``
from /root/reference/pkg/src, builds each StencilSpec with the exact
weights (reference presets, or the BASELINE config weights via the
reference's own ``StencilSpec`` constructor, validated at
``stencilbench/core.py:71-94``), seeds the grid, and iterates
``stencilbench.kernels.scalar_step`` exactly like the reference test helper
``tests/conftest.py:33-40`` / ``harness.run_oracle`` (``harness.py:149-157``).

Two halo conventions per case:
  * ``zero`` -- interior from ``default_rng(seed).random(dims)``, halo 0,
    identical to ``harness.seed_grid`` (``harness.py:139-146``);
  * ``full`` -- the whole halo-inclusive box from
    ``default_rng(seed).random(dims + 2r)``.

Fixtures hold compact halo-inclusive boxes (C-ABI host convention): the
outer axes' r-deep halo and the inner r cells of the reference's 2r-wide
unit-axis halo (``core.py:260-266``; only those r are read in NATURAL layout).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from stencilbench import core as ref_core            # noqa: E402
from stencilbench.kernels import scalar_step          # noqa: E402

from paper_2103_08825_b200 import core as sb_core     # noqa: E402

SEED = 12345

# name -> (spec source, dims, output steps)
CASES = {
    "c1_1d3p": ("cfg:c1", (1000,), (1, 7, 64)),
    "c2_1d5p": ("cfg:c2", (4099,), (1, 8, 40)),
    "c3a_2d9p_avg": ("cfg:c3a", (37, 131), (1, 5, 20)),
    "c3b_2d9p_rand": ("cfg:c3b", (37, 131), (1, 5, 20)),
    "c4_3d7p": ("cfg:c4", (11, 13, 37), (1, 4, 12)),
    "c5_3d27p": ("cfg:c5", (9, 11, 29), (1, 3, 8)),
    "p_1d3p": ("preset:1d3p", (300,), (1, 5)),
    "p_1d5p": ("preset:1d5p", (301,), (1, 5)),
    "p_2d5p": ("preset:2d5p", (21, 45), (1, 5)),
    "p_2d9p": ("preset:2d9p", (21, 45), (1, 5)),
    "p_3d7p": ("preset:3d7p", (7, 9, 33), (1, 5)),
    "p_3d27p": ("preset:3d27p", (7, 9, 33), (1, 5)),
    "x_2d13p_r2_star": ("rand:2:2:star:7", (19, 40), (1, 4)),
    "x_3d125p_r2_box": ("rand:3:2:box:8", (6, 7, 20), (1, 3)),
    "x_1d7p_r3_star": ("rand:1:3:star:9", (257,), (1, 6)),
}


def ref_spec(source: str):
    kind, _, rest = source.partition(":")
    if kind == "preset":
        return ref_core.make_stencil_spec(rest)
    if kind == "cfg":
        mine = sb_core.config_spec(rest)
        return ref_core.StencilSpec(mine.name, mine.d, mine.r, mine.shape, dict(mine.weights))
    d, r, shape, seed = rest.split(":")
    d, r, seed = int(d), int(r), int(seed)
    if shape == "box":
        w = sb_core.random_box_weights(d, r, seed)
    else:
        n = 2 * d * r + 1
        vals = np.random.default_rng(seed).random(n)
        w = sb_core.weights_from_list(d, r, "star", vals / vals.sum())
    return ref_core.StencilSpec(f"x_{d}d_r{r}_{shape}", d, r, shape, w)


def compact_view(grid, r):
    """Halo-inclusive compact box view of a reference NATURAL GridBuffer."""
    hu = grid.halo_unit
    return grid.data[..., hu - r:hu + grid.unit_n + r]


def run_case(name, source, dims, out_steps):
    spec = ref_spec(source)
    r = spec.r
    offs = spec.offsets
    arrays = {
        "d": np.int64(spec.d), "r": np.int64(r),
        "shape": np.array(spec.shape),
        "offsets": np.array(offs, dtype=np.int32).reshape(len(offs), spec.d),
        "weights": np.array([spec.weights[o] for o in offs], dtype=np.float64),
        "dims": np.array(dims, dtype=np.int64),
        "steps": np.array(out_steps, dtype=np.int64),
    }
    for halo in ("zero", "full"):
        a = ref_core.alloc_grid(spec, dims, ref_core.Layout.NATURAL, 4)
        rng = np.random.default_rng(SEED)
        if halo == "zero":
            a.set_interior(rng.random(dims))
        else:
            compact_view(a, r)[...] = rng.random(tuple(n + 2 * r for n in dims))
        arrays[f"in_{halo}"] = compact_view(a, r).copy()
        b = ref_core.alloc_like(a)
        b.data[...] = a.data
        t = 0
        for T in out_steps:
            while t < T:
                scalar_step(a, b, spec)
                a, b = b, a
                t += 1
            arrays[f"out_{halo}_T{T}"] = compact_view(a, r).copy()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    return sum(v.nbytes for v in arrays.values())


def main():
    total = 0
    for name, (source, dims, steps) in CASES.items():
        total += run_case(name, source, dims, steps)
        print(f"{name}: ok")
    print(f"total bytes {total}")


if __name__ == "__main__":
    main()
