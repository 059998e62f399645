#!/usr/bin/env python
"""Time the user-facing call (sweep(spec, box, T) on a pageable numpy box) phase by phase
(development tool): plan creation, upload, run, download."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec, CONFIGS
from paper_2103_08825_b200.plan import Plan, sweep
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
spec = config_spec(cfg)
wl = {"c5": ((768, 768, 768), 100), "c4": ((512, 512, 512), 200), "c3b": ((16384, 16384), 500), "c2": ((1 << 26,), 1000)}[cfg]
dims, T = wl
box = np.random.default_rng(1).random(tuple(n + 2 * spec.r for n in dims))
for rep in range(3):
    t0 = time.perf_counter()
    p = Plan(spec, dims)
    t1 = time.perf_counter()
    p.upload(box)
    p.synchronize()
    t2 = time.perf_counter()
    p.run(T)
    t3 = time.perf_counter()
    out = p.download()
    t4 = time.perf_counter()
    p.close()
    t5 = time.perf_counter()
    n = float(np.prod(dims)) * T
    print(json.dumps({"cfg": cfg, "rep": rep, "plan_ms": (t1 - t0) * 1e3, "upload_ms": (t2 - t1) * 1e3, "run_ms": (t3 - t2) * 1e3,
                      "download_ms": (t4 - t3) * 1e3, "close_ms": (t5 - t4) * 1e3, "call_gstencil": n / (t5 - t0) / 1e9,
                      "box_GB": box.nbytes / 1e9}), flush=True)
t0 = time.perf_counter()
out2 = sweep(spec, box, T)
t1 = time.perf_counter()
print(json.dumps({"sweep_call_ms": (t1 - t0) * 1e3, "gstencil": float(np.prod(dims)) * T / (t1 - t0) / 1e9, "same": bool(np.array_equal(out, out2))}))
