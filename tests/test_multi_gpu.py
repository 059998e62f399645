"""Single-process multi-GPU sweep (sb_multi_*, plan.MultiPlan, sweep(ngpu=...)).

The decomposition is emulated on one B200 by giving several slabs the same
device: the code path is the one a multi-GPU node runs (range launches for
the edge planes, peer copies of the ghost planes on copy streams, event
ordering, interiors overlapping the copies); only the copy engine's route
differs.  Results must be bit-identical to one device (EXACT and FMA alike:
the per-point arithmetic does not depend on the split) and EXACT bit-identical
to the oracle.
"""

import numpy as np
import pytest

from conftest import seeded_box
from oracle import c_oracle

from paper_2103_08825_b200.core import canonical, config_spec
from paper_2103_08825_b200.plan import MultiPlan, sweep

pytestmark = pytest.mark.gpu


def oracle(spec, box, T):
    offs, ws = canonical(spec)
    return c_oracle.sweep(box, spec.r, offs, ws, T)


CASES = [
    ("c2", (90001,), 37, "fma", 0, 3), ("c2", (40000,), 21, "exact", 8, 2), ("c1", (50000,), 70, "fma", 16, 4),
    ("c3a", (301, 530), 45, "fma", 0, 3), ("c3b", (257, 300), 13, "fma", 4, 2), ("c3b", (130, 200), 9, "exact", 8, 3),
    ("c4", (61, 40, 70), 11, "fma", 2, 3), ("c4", (40, 33, 50), 7, "exact", 4, 2),
    ("c5", (50, 40, 130), 9, "fma", 2, 3), ("c5", (37, 33, 70), 5, "exact", 2, 4),
]


@pytest.mark.parametrize("cfg,dims,T,arith,k,g", CASES)
def test_multi_equals_single_device(cfg, dims, T, arith, k, g):
    spec = config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=sum(dims) + T)
    one = sweep(spec, box, T, arith=arith, k=k)
    many = sweep(spec, box, T, arith=arith, k=k, devices=[0] * g)
    assert many.tobytes() == one.tobytes()
    if arith == "exact":
        assert many.tobytes() == oracle(spec, box, T).tobytes()


def test_multi_fp32_and_slab_geometry():
    spec = config_spec("c5")
    box = seeded_box((48, 40, 66), 1, seed=3).astype(np.float32)
    with MultiPlan(spec, (48, 40, 66), ngpu=3, devices=[0, 0, 0], dtype="f32", k=2) as mp:
        assert [(a, b) for a, b, _ in mp.slabs()] == [(0, 16), (16, 32), (32, 48)]
        mp.upload(box)
        t = mp.run(10)
        got = mp.download()
    assert t.point_updates == 48 * 40 * 66 * 10 and t.launches > 0
    assert got.tobytes() == sweep(spec, box, 10, k=2).tobytes()


def test_multi_repeated_runs_and_reupload():
    spec = config_spec("c4")
    dims = (40, 30, 64)
    box = seeded_box(dims, 1, seed=8)
    with MultiPlan(spec, dims, ngpu=2, devices=[0, 0], arith="exact", k=2) as mp:
        mp.upload(box)
        mp.run(3)
        mp.run(4)                                    # odd split across runs, tail at k=1
        got = mp.download()
        assert got.tobytes() == oracle(spec, box, 7).tobytes()
        mp.upload(box)
        mp.run(7)
        assert mp.download().tobytes() == got.tobytes()


def test_multi_rejects_thin_slabs():
    from paper_2103_08825_b200.core import GridError
    with pytest.raises(GridError, match="thinner"):
        MultiPlan(config_spec("c4"), (5, 20, 20), ngpu=4, devices=[0] * 4, k=2)
