"""Generate the layout golden fixtures (l_*.npz) by running the REFERENCE.

Run once in the build container (the reference is not present on the GPU
box):  ``python tests/golden/make_golden_layouts.py``.  For each case it
allocates a reference ``GridBuffer`` (``core.alloc_grid`` with ``pad_for``,
core.py:335-362), seeds every storage cell except the Dirichlet padding
``[unit_n, unit_np)`` of each row (which stays 0), converts it with the
reference's own ``transpose.to_block_transpose`` / ``to_dlt``
(transpose.py:286-336), and advances it with the layout's own method
(``transpose_layout_step`` kernels.py:257-340, ``dlt_step`` kernels.py:352-399,
and for 1D BLOCK_TRANSPOSE also ``timejam.jam_sweep`` timejam.py:288-304),
storing the full storage arrays.

Fixture keys: d, r, offsets, weights (canonical order), dims, vl, layout,
unit_np, halo_unit, nat (NATURAL storage), lay (converted storage),
step_T{t} (storage after t method steps, still in the layout), and jam_k2_T{t}.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from stencilbench import core as ref_core                        # noqa: E402
from stencilbench import transpose as ref_tr                     # noqa: E402
from stencilbench.kernels import dlt_step, transpose_layout_step  # noqa: E402
from stencilbench.timejam import jam_sweep                       # noqa: E402

from make_golden import ref_spec                                 # noqa: E402

SEED = 777

# name -> (spec source, dims, layout, vl, steps, jam steps)
CASES = {
    "l_1d3p_bt4": ("cfg:c1", (70,), "block_transpose", 4, (1, 3), (2, 4)),
    "l_1d5p_bt8": ("cfg:c2", (150,), "block_transpose", 8, (1, 2), (2, 4)),
    "l_1d3p_dlt4": ("cfg:c1", (70,), "dlt", 4, (1, 3), ()),
    "l_1d5p_dlt8": ("cfg:c2", (203,), "dlt", 8, (1, 2), ()),
    "l_2d9p_bt4": ("cfg:c3b", (9, 45), "block_transpose", 4, (1, 3), ()),
    "l_2d9p_dlt4": ("cfg:c3a", (7, 50), "dlt", 4, (1, 2), ()),
    "l_3d7p_dlt8": ("cfg:c4", (5, 6, 50), "dlt", 8, (1, 2), ()),
    "l_3d27p_bt4": ("cfg:c5", (4, 5, 33), "block_transpose", 4, (1, 2), ()),
}


def seeded_grid(spec, dims, layout, vl):
    g = ref_core.alloc_grid(spec, dims, ref_core.Layout.NATURAL, vl, pad_for=layout)
    g.data[...] = np.random.default_rng(SEED).random(g.data.shape)
    hu = g.halo_unit
    g.data[..., hu + g.unit_n:hu + g.unit_np] = 0.0          # Dirichlet padding
    return g


def run_case(name, source, dims, layout_name, vl, steps, jam_steps):
    spec = ref_spec(source)
    layout = ref_core.Layout(layout_name)
    offs = spec.offsets
    g = seeded_grid(spec, dims, layout, vl)
    arrays = {
        "d": np.int64(spec.d), "r": np.int64(spec.r), "shape": np.array(spec.shape),
        "offsets": np.array(offs, dtype=np.int32).reshape(len(offs), spec.d),
        "weights": np.array([spec.weights[o] for o in offs], dtype=np.float64),
        "dims": np.array(dims, dtype=np.int64), "vl": np.int64(vl), "layout": np.array(layout_name),
        "unit_np": np.int64(g.unit_np), "halo_unit": np.int64(g.halo_unit),
        "nat": g.data.copy(),
    }
    if layout is ref_core.Layout.BLOCK_TRANSPOSE:
        ref_tr.to_block_transpose(g, vl)
        step = transpose_layout_step
    else:
        ref_tr.to_dlt(g, vl)
        step = dlt_step
    arrays["lay"] = g.data.copy()
    a = g.clone()
    b = ref_core.alloc_like(a)
    b.data[...] = a.data                                      # fixed halo in both buffers
    t = 0
    for T in steps:
        while t < T:
            step(a, b, spec)
            a, b = b, a
            t += 1
        arrays[f"step_T{T}"] = a.data.copy()
    for T in jam_steps:
        j = g.clone()
        jam_sweep(j, spec, 2, T)
        arrays[f"jam_k2_T{T}"] = j.data.copy()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    return sum(v.nbytes for v in arrays.values())


def main():
    total = 0
    for name, args in CASES.items():
        total += run_case(name, *args)
        print(f"{name}: ok")
    print(f"total bytes {total}")


if __name__ == "__main__":
    main()
