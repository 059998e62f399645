"""The b200 harness (paper_2103_08825_b200/harness.py): the reference's
run_benchmark contract with a multi-step device dispatch.  Modelled on the
reference's own harness tests (test_harness.py:45: err == 0.0 for every
method; the CSV field order of harness.py:31-33)."""

import numpy as np
import pytest

from oracle import c_oracle

from paper_2103_08825_b200.core import canonical
from paper_2103_08825_b200.grid import compact_view
from paper_2103_08825_b200.harness import (B200_METHODS, CSV_HEADER, BenchConfig, BenchResult, Counters,
                                           UsageError, run_benchmark, seed_grid, validate_config)


def oracle_interior(cfg, spec):
    """harness.run_oracle restated on the C oracle: seed_grid, T exact steps."""
    g = seed_grid(BenchConfig(cfg.stencil, cfg.dims, cfg.steps, "b200", seed=cfg.seed, weights=cfg.weights), spec)
    offs, ws = canonical(spec)
    out = c_oracle.sweep(np.ascontiguousarray(compact_view(g)), spec.r, offs, ws, cfg.steps)
    r = spec.r
    return out[tuple(slice(r, s - r) for s in out.shape)]


@pytest.mark.parametrize("bad,match", [
    (dict(method="scalar"), "unknown"), (dict(dims=(10, 10)), "needs 1 extents"),
    (dict(steps=0), "steps"), (dict(vl=6), "vl"), (dict(jam_k=-1), "jam-k"), (dict(dims=(0,)), "positive"),
    (dict(block=(16,), tile_height=4), "device"), (dict(workers=0), "threads"),
])
def test_validate_config_rejects(bad, match):
    kw = dict(stencil="1d3p", dims=(64,), steps=3)
    kw.update(bad)
    with pytest.raises(UsageError, match=match):
        validate_config(BenchConfig(**kw))


def test_verify_needs_an_oracle():
    with pytest.raises(UsageError, match="oracle"):
        run_benchmark(BenchConfig("1d3p", (64,), 3, verify=True))


def test_seed_grid_matches_reference_convention():
    cfg = BenchConfig("2d9p", (7, 30), 1, "b200_transpose", seed=99)
    g = seed_grid(cfg, cfg.spec())
    assert g.unit_np == 32                                       # padded for BLOCK_TRANSPOSE, vl=4
    assert np.array_equal(g.natural_interior(), np.random.default_rng(99).random((7, 30)))
    mask = np.ones(g.data.shape, bool)
    mask[1:-1, 2:2 + 30] = False                                 # unit halo 2r = 2
    assert not g.data[mask].any()                                # halo and padding 0


def test_csv_row_field_order():
    res = BenchResult(BenchConfig("1d5p", (100,), 4), 0.5, 0.1, 2.0, Counters(point_updates=400))
    assert len(res.csv_row().split(",")) == len(CSV_HEADER.split(","))
    assert res.csv_row().startswith("1d5p,b200,4,0,100,4,,,1,")


def test_default_depth_is_valid_for_every_stencil_class():
    # jam_k defaults to 0 = the plan's own depth, so a default BenchConfig is
    # valid for 3D stencils too (a fixed default of 8 is rejected by the 3D kernels)
    for stencil, dims in (("1d3p", (64,)), ("2d9p", (8, 8)), ("3d7p", (4, 4, 4)), ("3d27p", (4, 4, 4))):
        cfg = BenchConfig(stencil, dims, 3)
        assert cfg.jam_k == 0
        validate_config(cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("method", list(B200_METHODS))
@pytest.mark.parametrize("stencil,dims,steps,k", [
    ("1d5p", (333,), 9, 4), ("2d9p", (21, 45), 6, 2), ("3d27p", (7, 9, 33), 5, 2), ("3d7p", (9, 10, 40), 7, 3),
])
def test_run_benchmark_bit_identical_to_oracle(method, stencil, dims, steps, k):
    cfg = BenchConfig(stencil, dims, steps, method, jam_k=k, verify=True)
    res = run_benchmark(cfg, oracle=oracle_interior)
    assert res.max_rel_err == 0.0
    assert res.counters.point_updates == int(np.prod(dims)) * steps
    assert res.gflops > 0 and (res.layout_seconds > 0) == (method != "b200")


@pytest.mark.gpu
@pytest.mark.parametrize("stencil,dims", [("3d7p", (9, 10, 40)), ("3d27p", (7, 9, 33)), ("2d9p", (21, 45))])
def test_run_benchmark_default_depth(stencil, dims):
    res = run_benchmark(BenchConfig(stencil, dims, 5, verify=True), oracle=oracle_interior)
    assert res.max_rel_err == 0.0


@pytest.mark.gpu
def test_run_benchmark_custom_weights_config():
    cfg = BenchConfig("c5", (8, 20, 66), 4, "b200", jam_k=2, verify=True, weights="c5")
    res = run_benchmark(cfg, oracle=oracle_interior)
    assert res.max_rel_err == 0.0
