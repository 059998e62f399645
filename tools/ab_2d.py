#!/usr/bin/env python
"""Time 2D sweeps (16384^2) for a list of cfg:k pairs (development tool).
usage: ab_2d.py T cfg:k [cfg:k ...]   (environment knobs select the variant)"""
import json, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
T = int(sys.argv[1])
for arg in sys.argv[2:]:
    cfg, k = arg.split(":")[:2]
    arith = arg.split(":")[2] if arg.count(":") > 1 else "fma"
    dims = (16384, 16384)
    box = np.random.default_rng(1).random(tuple(n + 2 for n in dims))
    with Plan(config_spec(cfg), dims, k=int(k), arith=arith, kernel="fused") as p:
        p.upload(box)
        p.run(T)
        best = min(p.run(T).device_ms for _ in range(3))
    print(json.dumps({"cfg": cfg, "k": int(k), "arith": arith, "gstencil": round(np.prod(dims) * T / best / 1e6, 1)}), flush=True)
