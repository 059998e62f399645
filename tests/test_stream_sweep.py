"""sb_sweep_host: host box in, T steps, host box out, transfers overlapped with the
sweep on 3D plans (blocks of planes, every launch shifted down by the reach of the
launches before it).  The streamed result must be bit-identical to upload + run +
download of the same plan (same range-launch kernels), and match the oracle."""

import numpy as np
import pytest

from conftest import seeded_box
from oracle import c_oracle, np_oracle

from paper_2103_08825_b200.core import canonical, config_spec, make_stencil_spec
from paper_2103_08825_b200.grid import alloc_grid, compact_view
from paper_2103_08825_b200.kernels import b200_sweep
from paper_2103_08825_b200.plan import Plan, sweep

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def streamed(monkeypatch):
    # opt-in (read per call by sb_sweep_host): off by default, see sb200.cu
    monkeypatch.setenv("SB200_STREAM_SWEEP", "1")

BIG = (256, 200, 200)      # 84 MB fp64 box: above the streaming threshold (64 MB)


def plain(p, box, T):
    p.upload(box)
    p.run(T)
    return p.download()


@pytest.mark.parametrize("cfg,arith,T", [("c5", "fma", 7), ("c5", "exact", 6), ("c4", "fma", 11), ("c4", "exact", 9),
                                         ("c5", "fma", 1), ("c4", "fma", 2)])
def test_streamed_equals_plain_and_oracle(cfg, arith, T):
    spec = config_spec(cfg)
    box = seeded_box(BIG, 1, seed=T)
    with Plan(spec, BIG, arith=arith) as p:
        want = plain(p, box, T)
        got = p.sweep_host(box, T)
        again = p.sweep_host(box, T)              # plan state after a streamed sweep is reusable
        p.run(2)                                  # ... and consistent with a normal run
        cont = p.download()
    assert got.tobytes() == want.tobytes()
    assert again.tobytes() == want.tobytes()
    offs, ws = canonical(spec)
    ref = c_oracle.sweep(box, spec.r, offs, ws, T)
    if arith == "exact":
        assert got.tobytes() == ref.tobytes()
    else:
        assert np_oracle.max_rel_error(got, ref) <= 1e-12
    if arith == "exact" or T % 2 == 0:            # (FMA: an odd T changes where the composed k=2 launches fall)
        with Plan(spec, BIG, arith=arith) as p:
            want2 = plain(p, box, T + 2)
        assert cont.tobytes() == want2.tobytes()


def test_streamed_fp32_and_generic_kernel():
    spec = config_spec("c5")
    box32 = seeded_box(BIG, 1, seed=3).astype(np.float32)
    big32 = (320, 256, 256)                       # 86 MB in fp32
    box32 = seeded_box(big32, 1, seed=3).astype(np.float32)
    with Plan(spec, big32, dtype="f32") as p:
        want = plain(p, box32, 5)
        got = p.sweep_host(box32, 5)
    assert got.tobytes() == want.tobytes()
    spec2 = make_stencil_spec("3d7p")
    box = seeded_box(BIG, 1, seed=8, halo="zero")
    with Plan(spec2, BIG, arith="exact", kernel="generic") as p:
        want = plain(p, box, 3)
        got = p.sweep_host(box, 3)
    assert got.tobytes() == want.tobytes()


def test_sweep_call_and_gridbuffer_in_place_streamed():
    spec = config_spec("c5")
    box = seeded_box(BIG, 1, seed=21)
    offs, ws = canonical(spec)
    ref = c_oracle.sweep(box, spec.r, offs, ws, 4)
    assert sweep(spec, box, 4, arith="exact").tobytes() == ref.tobytes()
    g = alloc_grid(spec, BIG)                     # NATURAL GridBuffer: pitched rows, in place
    g.data[...] = np.random.default_rng(5).random(g.data.shape)
    snap = g.data.copy()
    before = np.array(compact_view(g), copy=True)
    b200_sweep(g, spec, 2, 4, arith="exact")
    want = c_oracle.sweep(before, spec.r, offs, ws, 4)
    assert np.array_equal(compact_view(g), want)
    outside = np.ones(g.data.shape, bool)
    hu = g.halo_unit
    outside[..., hu - 1:hu + g.unit_n + 1] = False
    assert np.array_equal(g.data[outside], snap[outside])


def test_long_sweep_falls_back_when_the_shift_exceeds_the_grid():
    # T so long that the launches' cumulative reach passes half the grid: plain sequence
    spec = config_spec("c4")
    box = seeded_box(BIG, 1, seed=2)
    with Plan(spec, BIG, arith="exact") as p:
        want = plain(p, box, 140)
        got = p.sweep_host(box, 140)
    assert got.tobytes() == want.tobytes()


def test_streamed_pinned_memory_direct(monkeypatch):
    # pinned host memory on both sides: the copy engines read / write the caller's rows
    # directly (no bounce buffers) and streaming is the default for few-launch sweeps
    torch = pytest.importorskip("torch")
    monkeypatch.delenv("SB200_STREAM_SWEEP", raising=False)
    spec = config_spec("c5")
    box = seeded_box(BIG, 1, seed=33)
    pin_in = torch.empty(box.shape, dtype=torch.float64, pin_memory=True)
    pin_in.numpy()[...] = box
    pin_out = torch.empty_like(pin_in, pin_memory=True)
    with Plan(spec, BIG, arith="exact") as p:
        want = plain(p, box, 6)
        p.sweep_host(pin_in.numpy(), 6, out=pin_out.numpy())
        assert pin_out.numpy().tobytes() == want.tobytes()
        # in place, and mixed pinned / pageable
        p.sweep_host(pin_in.numpy(), 6, out=pin_in.numpy())
        assert pin_in.numpy().tobytes() == want.tobytes()
        monkeypatch.setenv("SB200_STREAM_SWEEP", "1")
        pin_in.numpy()[...] = box
        got = p.sweep_host(pin_in.numpy(), 6)
        assert got.tobytes() == want.tobytes()
        got2 = p.sweep_host(box, 6, out=pin_out.numpy())
        assert got2.tobytes() == want.tobytes()
