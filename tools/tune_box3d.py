#!/usr/bin/env python
"""Time the C5 sweep (768^3, T=100, k=2) for the kernel-variant env knobs
given on the command line, each in a fresh process: NAME=VAL,NAME=VAL ...
(development tool; prints GStencil/s per variant)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
wl, dtype, T, k = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
dims = {"c5": (768, 768, 768), "c4": (512, 512, 512)}[wl]
spec = config_spec(wl)
box = np.random.default_rng(1).random(tuple(n + 2 for n in dims)).astype(np.float32 if dtype == "f32" else np.float64)
with Plan(spec, dims, k=k, arith="fma", dtype=dtype) as p:
    p.upload(box)
    p.run(T)
    best = 1e9
    for _ in range(4):
        t = p.run(T)
        best = min(best, t.device_ms)
    print(json.dumps({"gstencil": np.prod(dims) * T / best / 1e6, "ms": best, "kernel": t.kernel_name}))
''' % REPO

def main():
    wl = os.environ.get("WL", "c5")
    dtype = os.environ.get("DT", "f64")
    T = int(os.environ.get("T", "100"))
    k = int(os.environ.get("K", "2"))
    for variant in sys.argv[1:]:
        env = dict(os.environ)
        if variant != "-":
            for kv in variant.split(","):
                n, v = kv.split("=")
                env[n] = v
        out = subprocess.run([sys.executable, "-c", CHILD, wl, dtype, str(T), str(k)], env=env,
                             capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        print(f"{wl} {dtype} k={k} {variant:40s}", line[-1] if line else out.stderr[-500:], flush=True)

if __name__ == "__main__":
    main()
