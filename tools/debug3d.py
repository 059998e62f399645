"""Small 3D fused-vs-oracle comparisons with mismatch locations (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import c_oracle  # noqa: E402
from paper_2103_08825_b200.core import canonical, config_spec  # noqa: E402
from paper_2103_08825_b200.plan import sweep  # noqa: E402

cases = [("c4", (3, 5, 7), 1, 1), ("c4", (9, 40, 70), 1, 1), ("c5", (9, 40, 70), 1, 1),
         ("c5", (9, 40, 70), 2, 2), ("c4", (9, 40, 70), 2, 3), ("c5", (37, 33, 130), 2, 7)]
for cfg, dims, k, T in cases:
    spec = config_spec(cfg)
    box = np.random.default_rng(1).random(tuple(n + 2 for n in dims))
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box, 1, offs, ws, T)
    try:
        got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
    except Exception as e:  # noqa: BLE001
        print(cfg, dims, k, T, "ERROR", e)
        break
    bad = np.argwhere(got != want)
    print(cfg, dims, "k", k, "T", T, "mismatches", len(bad), "of", got.size,
          "max abs err %.3g" % np.max(np.abs(got - want)))
    if len(bad):
        print("   first:", bad[:6].tolist(), "got", got[tuple(bad[0])], "want", want[tuple(bad[0])])
        zs = sorted(set(bad[:, 0].tolist()))
        print("   planes:", zs[:12], "rows:", sorted(set(bad[:, 1].tolist()))[:12], "cols:", sorted(set(bad[:, 2].tolist()))[:12])
