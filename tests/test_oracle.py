"""Pin the CPU oracles to the reference before trusting them.

The golden fixtures were produced by running the reference's own
``scalar_step`` (tests/golden/make_golden.py).  Both restatements must
reproduce every fixture bit-for-bit, for both halo conventions and every
recorded step count, and must also reproduce the reference's known-answer
tests (``tests/test_kernels.py:80-104`` of the reference).
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden, seeded_box
from oracle import c_oracle, np_oracle

NAMES = golden_names()


def test_golden_fixtures_present():
    assert len(NAMES) >= 15
    for must in ("c1_1d3p", "c2_1d5p", "c3a_2d9p_avg", "c3b_2d9p_rand",
                 "c4_3d7p", "c5_3d27p"):
        assert must in NAMES


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("halo", ["zero", "full"])
def test_np_oracle_matches_reference(name, halo):
    g = load_golden(name)
    for T in g["steps"]:
        got = np_oracle.sweep(g[f"in_{halo}"], g["r"], g["offsets"], g["weights"], T)
        assert np.array_equal(got, g[f"out_{halo}_T{T}"]), (name, halo, T)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("halo", ["zero", "full"])
@pytest.mark.parametrize("threads", [1, 3])
def test_c_oracle_matches_reference(name, halo, threads):
    g = load_golden(name)
    for T in g["steps"]:
        got = c_oracle.sweep(g[f"in_{halo}"], g["r"], g["offsets"], g["weights"], T,
                             threads=threads)
        want = g[f"out_{halo}_T{T}"]
        assert got.tobytes() == want.tobytes(), (name, halo, T)


def test_c_oracle_halo_untouched():
    g = load_golden("c4_3d7p")
    box = g["in_full"]
    out = c_oracle.sweep(box, 1, g["offsets"], g["weights"], 5)
    mask = np.ones(box.shape, bool)
    mask[1:-1, 1:-1, 1:-1] = False
    assert np.array_equal(out[mask], box[mask])


def test_known_answer_impulse():
    # reference tests/test_kernels.py:90-94
    box = np.zeros(7)
    box[3] = 1.0
    out = c_oracle.sweep(box, 1, [(-1,), (0,), (1,)], [0.25, 0.5, 0.25], 1)
    assert out[1:-1].tolist() == [0, 0.25, 0.5, 0.25, 0]


def test_known_answer_ramp_and_constant():
    # reference tests/test_kernels.py:80-104 (ramp fixed point, constant preserved)
    n = 32
    box = np.zeros(n + 2)
    box[1:-1] = np.arange(float(n))
    out = c_oracle.sweep(box, 1, [(-1,), (0,), (1,)], [0.25, 0.5, 0.25], 1)
    assert np.array_equal(out[2:-2], np.arange(1.0, n - 1))
    from paper_2103_08825_b200.core import make_stencil_spec, canonical
    spec = make_stencil_spec("2d9p")
    offs, ws = canonical(spec)
    box = np.full((14, 34), 2.5)
    out = c_oracle.sweep(box, 1, offs, ws, 3)
    assert np.all(out == 2.5)


def test_fp32_restatement_close_to_fp64():
    from paper_2103_08825_b200.core import config_spec, canonical
    spec = config_spec("c5")
    offs, ws = canonical(spec)
    box = seeded_box((10, 12, 40), 1)
    box32 = box.astype(np.float32)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs,
                          [float(np.float32(w)) for w in ws], 20)
    got = c_oracle.sweep(box32, 1, offs, ws, 20)
    assert np_oracle.max_rel_error(got, want) < 1e-5
