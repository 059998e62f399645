#!/usr/bin/env python
"""Time Plan.sweep_host on PINNED host buffers (development tool): the streamed form
(default for pinned memory) against upload + run + download (SB200_STREAM_SWEEP=0)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
dims, T = {"c5": ((768, 768, 768), 100), "c4": ((512, 512, 512), 200), "c5f32": ((768, 768, 768), 100)}[cfg]
dt = torch.float32 if cfg == "c5f32" else torch.float64
shape = tuple(n + 2 for n in dims)
a = torch.empty(shape, dtype=dt, pin_memory=True)
a.numpy()[...] = np.random.default_rng(1).random(shape)
b = torch.empty_like(a, pin_memory=True)
with Plan(config_spec("c5" if cfg == "c5f32" else cfg), dims, dtype="f32" if cfg == "c5f32" else "f64") as p:
    for mode in ("0", "", "0", ""):
        if mode:
            os.environ["SB200_STREAM_SWEEP"] = mode
        else:
            os.environ.pop("SB200_STREAM_SWEEP", None)
        p.sweep_host(a.numpy(), T, out=b.numpy())
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            p.sweep_host(a.numpy(), T, out=b.numpy())
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"cfg": cfg, "stream": mode or "default(pinned: on)", "ms": best * 1e3,
                          "gstencil": float(np.prod(dims)) * T / best / 1e9}), flush=True)
