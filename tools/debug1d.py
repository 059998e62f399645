"""1D fused-vs-oracle diagnostics over sizes around the schedule regimes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import c_oracle  # noqa: E402
from paper_2103_08825_b200.core import canonical, config_spec  # noqa: E402
from paper_2103_08825_b200.plan import sweep  # noqa: E402

spec = config_spec("c2")
offs, ws = canonical(spec)
for n in (1000, 3072, 3073, 4096, 6144, 9216, 9217, 70001):
    for halo in ("zero", "full"):
        rng = np.random.default_rng(99)
        box = np.zeros(n + 4)
        if halo == "zero":
            box[2:-2] = rng.random(n)
        else:
            box[:] = rng.random(n + 4)
        for k, T in ((2, 2), (2, 100), (16, 100)):
            got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
            want = c_oracle.sweep(box, 2, offs, ws, T)
            bad = np.flatnonzero(got != want)
            if len(bad):
                print(n, halo, k, T, "mismatch", len(bad), "first", bad[:5], "last", bad[-3:])
print("done")
