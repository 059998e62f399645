#!/usr/bin/env python
"""Time 2D sweeps (16384^2, T) for config/k list (development tool)."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
T = int(sys.argv[1]) if len(sys.argv) > 1 else 48
for cfg, k in [("c3b", 4), ("c3b", 8), ("c3b", 2), ("c3a", 4), ("c3a", 8)]:
    dims = (16384, 16384)
    box = np.random.default_rng(1).random(tuple(n + 2 for n in dims))
    with Plan(config_spec(cfg), dims, k=k, arith="fma") as p:
        p.upload(box)
        p.run(T)
        best = min(p.run(T).device_ms for _ in range(3))
    print(json.dumps({"cfg": cfg, "k": k, "gstencil": round(np.prod(dims) * T / best / 1e6, 1)}), flush=True)
