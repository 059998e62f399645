"""Small fused 1D/2D/3D sweeps incl. slab (ghost) plans, for compute-sanitizer memcheck."""
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
print("sanitize cases done")
