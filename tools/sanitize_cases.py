"""Small fused 1D/2D/3D sweeps incl. slab (ghost) plans, composed paths and ranges steps, for
compute-sanitizer memcheck (closed on the current GPU pool: run plainly there as an exit-0 smoke)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08825_b200.core import config_spec  # noqa: E402
from paper_2103_08825_b200.plan import sweep  # noqa: E402
from paper_2103_08825_b200.slab import SlabSweep, run_local  # noqa: E402

rng = np.random.default_rng(0)
for cfg, dims, ks in (("c2", (5000,), (2, 16)), ("c1", (777,), (8,)), ("c3b", (70, 300), (1, 8)),
                      ("c4", (9, 40, 70), (1, 4)), ("c5", (7, 35, 66), (2, 3))):
    spec = config_spec(cfg)
    box = rng.random(tuple(n + 2 * spec.r for n in dims))
    for k in ks:
        sweep(spec, box, 2 * k + 1, k=k, kernel="fused")
        sweep(spec, box.astype(np.float32), k, k=k, kernel="fused")
    sweep(spec, box, 2, kernel="generic")
    g = 2
    k = ks[-1]
    sw = [SlabSweep(spec, (dims[0] * 0 + max(dims[0], 2 * k * spec.r * g + 2),) + dims[1:], rank=r, world=g, k=k)
          for r in range(g)]
    gbox = rng.random((sw[0].global_dims[0] + 2 * spec.r,) + tuple(n + 2 * spec.r for n in dims[1:]))
    for s in sw:
        s.upload(s.local_box(gbox))
    run_local(sw, 2 * k + 1)
# composed 3D star (FMA, k=2: main + shell kernels), incl. z slabs
spec = config_spec("c4")
for dims in ((4, 4, 4), (9, 37, 70), (12, 21, 131)):
    box = rng.random(tuple(n + 2 for n in dims))
    sweep(spec, box, 5, k=2, arith="fma")
sw = [SlabSweep(spec, (24, 21, 70), rank=r, world=3, k=2, arith="fma") for r in range(3)]
gbox = rng.random((26, 23, 72))
for s in sw:
    s.upload(s.local_box(gbox))
run_local(sw, 6)
# fp32 box, paired FFMA2 path (k=1, 2)
spec = config_spec("c5")
box = rng.random((9, 37, 70)).astype(np.float32)
for k in (1, 2):
    sweep(spec, box, 2 * k + 1, k=k, arith="fma")
# layout conversions and storage upload/download
from paper_2103_08825_b200.grid import Layout, alloc_grid  # noqa: E402
from paper_2103_08825_b200 import transpose as tr  # noqa: E402
from paper_2103_08825_b200.kernels import b200_sweep  # noqa: E402
for cfg, dims, lay, vl in (("c1", (70,), "block_transpose", 4), ("c2", (203,), "dlt", 8),
                           ("c3b", (9, 45), "block_transpose", 4), ("c4", (5, 6, 50), "dlt", 8)):
    spec = config_spec(cfg)
    g = alloc_grid(spec, dims, Layout.NATURAL, vl, pad_for=Layout(lay))
    g.data[...] = rng.random(g.data.shape)
    (tr.to_block_transpose if lay == "block_transpose" else tr.to_dlt)(g, vl)
    b200_sweep(g, spec, 2, 3)
    (tr.from_block_transpose if lay == "block_transpose" else tr.from_dlt)(g)
# composed 1D (FMA, k=32/64, boundary windows in the launch) and separable composed 2D (c3a, k=16/32)
for cfg, dims, ks in (("c2", (20000,), (32,)), ("c1", (13001,), (64,)), ("c3a", (70, 300), (16, 32)),
                      ("c3a", (131, 97), (32,))):
    spec = config_spec(cfg)
    box = rng.random(tuple(n + 2 * spec.r for n in dims))
    for k in ks:
        sweep(spec, box, 2 * k + 3, k=k, arith="fma")
spec = config_spec("c3a")
sw = [SlabSweep(spec, (140, 300), rank=r, world=2, k=32, arith="fma") for r in range(2)]
gbox = rng.random((142, 302))
for s in sw:
    s.upload(s.local_box(gbox))
run_local(sw, 64)
# ranges-restricted steps (box swept as its own grid; BLOCK_TRANSPOSE via sb_step_box)
from paper_2103_08825_b200.kernels import b200_step  # noqa: E402
from paper_2103_08825_b200.grid import alloc_like  # noqa: E402
for cfg, dims, rg in (("c5", (9, 20, 33), [(2, 7), (5, 6), (1, 32)]), ("c3b", (41, 66), [(40, 41), (0, 66)])):
    spec = config_spec(cfg)
    g = alloc_grid(spec, dims)
    g.set_interior(rng.random(dims))
    b200_step(g, alloc_like(g), spec, ranges=rg)
print("sanitize cases done")
