"""Single-GPU slab emulation vs oracle: where do mismatches land? (debug aid)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import c_oracle  # noqa: E402
from paper_2103_08825_b200.core import canonical, config_spec  # noqa: E402
from paper_2103_08825_b200.slab import SlabSweep, run_local  # noqa: E402

for cfg, dims, k, g, steps in (("c3b", (400, 300), 8, 4, 8), ("c3b", (400, 300), 8, 2, 8), ("c3b", (400, 300), 1, 2, 1),
                               ("c3b", (400, 300), 2, 2, 2), ("c3b", (40, 300), 8, 2, 8)):
    spec = config_spec(cfg)
    gbox = np.random.default_rng(3).random(tuple(n + 2 for n in dims))
    sweeps = [SlabSweep(spec, dims, rank=r, world=g, k=k, arith="exact", device=0) for r in range(g)]
    for s in sweeps:
        s.upload(s.local_box(gbox))
    run_local(sweeps, steps)
    got = np.concatenate([s.download()[s.geom.interior_slice()] for s in sweeps], axis=0)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(gbox, 1, offs, ws, steps)[1:1 + dims[0]]
    bad = np.argwhere(got != want)
    print(cfg, dims, "k", k, "g", g, "mismatch", len(bad), "rows", sorted(set(bad[:, 0].tolist()))[:20],
          "cols", sorted(set(bad[:, 1].tolist()))[:8] if len(bad) else "")
