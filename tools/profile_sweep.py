"""Tiny driver for ncu: one config, a few fused launches (no timing claims)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08825_b200.core import config_spec  # noqa: E402
from paper_2103_08825_b200.plan import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2")
ap.add_argument("--dims", default="67108864")
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--steps", type=int, default=24)
ap.add_argument("--arith", default="fma")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--kernel", default="auto")
a = ap.parse_args()
spec = config_spec(a.cfg)
dims = tuple(int(x) for x in a.dims.split("x"))
box = np.random.default_rng(1).random(tuple(n + 2 * spec.r for n in dims))
if a.dtype == "f32":
    box = box.astype(np.float32)
with Plan(spec, dims, k=a.k, arith=a.arith, dtype=a.dtype, kernel=a.kernel) as p:
    p.upload(box)
    t = p.run(a.steps)
    print(t)
