"""Shared test helpers: golden fixtures, seeded inputs, markers.

``gpu``-marked tests need a B200 (run by the driver with ``-m gpu``); all
others run on the CPU build container.
"""

from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")

# The reference package (stencilbench) for the integration tests: the per-pod
# install under baseline/_ref (travels to the GPU box with the repo), else the
# read-only source tree of this build container.  Tests that need it skip
# when neither exists.
for _ref in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(_ref, "stencilbench")):
        if _ref not in sys.path:
            sys.path.append(_ref)
        break


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names():
    """Natural-layout sweep fixtures (make_golden.py); the l_* layout fixtures
    (make_golden_layouts.py) have their own tests (test_layouts.py)."""
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith("l_"))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = {k: z[k] for k in z.files}
    g["d"], g["r"] = int(g["d"]), int(g["r"])
    g["shape"] = str(g["shape"])
    g["offsets"] = [tuple(int(c) for c in row) for row in g["offsets"]]
    g["weights"] = [float(w) for w in g["weights"]]
    g["steps"] = [int(s) for s in g["steps"]]
    return g


def golden_spec(g):
    from paper_2103_08825_b200.core import StencilSpec
    return StencilSpec("golden", g["d"], g["r"], g["shape"],
                       dict(zip(g["offsets"], g["weights"])))


def seeded_box(dims, r, seed=12345, halo="full", dtype=np.float64):
    """Halo-inclusive box; ``halo='zero'`` matches harness.seed_grid (halo 0)."""
    rng = np.random.default_rng(seed)
    if halo == "zero":
        box = np.zeros(tuple(n + 2 * r for n in dims))
        box[tuple(slice(r, r + n) for n in dims)] = rng.random(dims)
    else:
        box = rng.random(tuple(n + 2 * r for n in dims))
    return box.astype(dtype)


def interior(box, r):
    return box[tuple(slice(r, s - r) for s in box.shape)]


def rel_err(got, want):
    from oracle.np_oracle import max_rel_error
    return max_rel_error(got, want)


@pytest.fixture(scope="session")
def have_gpu():
    import torch
    return torch.cuda.is_available()
