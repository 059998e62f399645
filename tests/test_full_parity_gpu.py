"""Parity after ALL steps at the full BASELINE sizes (north_star: fp64 max
relative error <= 1e-12 after all steps, fp32 <= 1e-5).

Every benched configuration -- C1 (2^20, T=64), C2 (2^26, T=1000, both halo
conventions), C3a / C3b (16384^2, T=500), C4 (512^3, T=200), C5 (768^3,
T=100) in fp64 and fp32 -- runs its bench kernel path (FMA, the bench's
fusion depth) and EXACT mode (bit-identical) on the device, against the C
oracle on the host cores (tools/full_parity.py; ~3 min on a 16-core box).
"""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import full_parity  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", list(full_parity.CASES))
def test_full_size_full_T(case):
    res = full_parity.run_case(case, full_parity.CASES[case], log=lambda s: None)
    for v in res["variants"]:
        assert v["ok"], (case, v)
        if v["arith"] == "exact":
            assert v["bit_identical"], (case, v)
