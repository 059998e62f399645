"""Host-side logic (no GPU): the spec mirror restates the reference's rules,
the BASELINE config weights are what BASELINE.json says, and the grid
marshalling (compact halo box) round-trips."""

import itertools

import numpy as np
import pytest

from paper_2103_08825_b200 import core
from paper_2103_08825_b200.core import (SpecError, StencilSpec, config_spec, canonical,
                                        flops_per_point, make_stencil_spec)
from paper_2103_08825_b200.grid import alloc_grid, alloc_like, compact_view, interior_view
from paper_2103_08825_b200.plan import host_shape


def test_presets_match_reference_semantics():
    # reference tests/test_core.py: presets exist, weights sum exactly to 1
    for name in core.PRESET_NAMES:
        spec = make_stencil_spec(name)
        assert sum(spec.weights.values()) == 1.0
    assert make_stencil_spec("1d3p").weights[(0,)] == 0.5
    assert make_stencil_spec("3d27p").weights[(0, 0, 0)] == 0.125
    with pytest.raises(SpecError, match="unknown stencil preset"):
        make_stencil_spec("4d9p")


def test_spec_validation_rules():
    with pytest.raises(SpecError, match="dimension"):
        StencilSpec("x", 4, 1, "star", {(0, 0, 0, 0): 1.0})
    with pytest.raises(SpecError, match="order"):
        StencilSpec("x", 1, 0, "star", {(0,): 1.0})
    with pytest.raises(SpecError, match="zero offset"):
        StencilSpec("x", 1, 1, "star", {(-1,): 0.5, (1,): 0.5, (2,): 0.0})
    with pytest.raises(SpecError, match="outside radius"):
        StencilSpec("x", 1, 1, "star", {(-2,): 0.5, (0,): 0.5, (1,): 0.0})
    with pytest.raises(SpecError, match="non-axis-aligned"):
        StencilSpec("x", 2, 1, "star", {(0, 0): 1, (1, 1): 0, (0, 1): 0, (-1, 0): 0, (1, 0): 0})
    with pytest.raises(SpecError, match="needs 9 weights"):
        StencilSpec("x", 2, 1, "box", {(0, 0): 1.0})
    with pytest.raises(SpecError, match="shape"):
        StencilSpec("x", 1, 1, "ring", {(0,): 1.0})


def test_canonical_order_is_lexicographic():
    spec = make_stencil_spec("3d7p")
    offs, _ = canonical(spec)
    assert offs == sorted(offs)
    assert offs[0] == (-1, 0, 0) and offs[3] == (0, 0, 0) and offs[-1] == (1, 0, 0)


def test_flops_per_point():
    assert [flops_per_point(config_spec(k)) for k in ("c1", "c2", "c3a", "c4", "c5")] == \
        [5, 9, 17, 13, 53]


def test_config_weights_match_baseline():
    assert [w for _, w in sorted(config_spec("c1").weights.items())] == [0.25, 0.5, 0.25]
    assert [w for _, w in sorted(config_spec("c2").weights.items())] == \
        [0.0625, 0.25, 0.375, 0.25, 0.0625]
    assert set(config_spec("c3a").weights.values()) == {1.0 / 9.0}
    c4 = config_spec("c4").weights
    assert c4[(0, 0, 0)] == 0.4 and sorted(c4.values())[:6] == [0.1] * 6
    for key, n in (("c3b", 9), ("c5", 27)):
        w = np.array([v for _, v in sorted(config_spec(key).weights.items())])
        assert len(w) == n and np.all(w > 0) and abs(w.sum() - 1.0) < 1e-15
    seed = core.WEIGHT_SEEDS["3d27p_rand"]
    raw = np.random.default_rng(seed).random(27)
    offs = sorted(itertools.product((-1, 0, 1), repeat=3))
    assert config_spec("c5").weights[offs[5]] == (raw / raw.sum())[5]


def test_host_shape():
    assert host_shape(1, 2, (100,)) == (104,)
    assert host_shape(3, 1, (4, 5, 6)) == (6, 7, 8)
    assert host_shape(3, 1, (4, 5, 6), ghost=(8, 0)) == (4 + 8 + 1, 7, 8)


def test_grid_mirror_compact_round_trip():
    spec = make_stencil_spec("2d9p")
    g = alloc_grid(spec, (5, 7))
    assert g.data.shape == (7, 11)             # r outer, 2r unit halo (core.py:260-266)
    vals = np.arange(35.0).reshape(5, 7)
    g.set_interior(vals)
    box = compact_view(g)
    assert box.shape == (7, 9)
    assert np.array_equal(box[1:-1, 1:-1], vals)
    assert np.array_equal(interior_view(g), vals)
    h = alloc_like(g)
    assert h.data.shape == g.data.shape and not h.data.any()


def test_compact_view_of_reference_layout_if_available():
    ref = pytest.importorskip("stencilbench.core", reason="reference not importable here")
    spec = ref.make_stencil_spec("1d5p")
    g = ref.alloc_grid(spec, 37, ref.Layout.NATURAL, 4)
    g.set_interior(np.arange(37.0))
    box = compact_view(g)
    assert box.shape == (41,) and np.array_equal(box[2:-2], np.arange(37.0))
