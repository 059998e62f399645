"""The reference-facing drop-in: METHODS-compatible step and jam_sweep-
compatible sweep on GridBuffer objects (the package's NATURAL mirror of
stencilbench.core.GridBuffer), checked the way the reference checks its own
methods (tests/test_kernels.py:113-133, test_timejam.py:156-164)."""

import numpy as np
import pytest

from conftest import seeded_box
from oracle import c_oracle

from paper_2103_08825_b200.core import GridError, canonical, config_spec, make_stencil_spec
from paper_2103_08825_b200.grid import Layout, alloc_grid, alloc_like, compact_view
from paper_2103_08825_b200.kernels import b200_step, b200_sweep, register


class Counters:   # shape of stencilbench.kernels.Counters (kernels.py:43-69)
    def __init__(self):
        self.scalar_loads = self.scalar_stores = self.point_updates = 0


def test_register_into_methods_registry():
    methods = {"scalar": (Layout.NATURAL, None)}
    register(methods, Layout.NATURAL)
    assert methods["b200"] == (Layout.NATURAL, b200_step)


def test_step_rejects_aliasing_and_bad_ranges():
    spec = make_stencil_spec("1d3p")
    g = alloc_grid(spec, 16)
    with pytest.raises(GridError, match="out-of-place"):
        b200_step(g, g, spec)
    with pytest.raises(GridError, match="outside"):
        b200_step(g, alloc_like(g), spec, ranges=[(0, 17)])
    with pytest.raises(GridError, match="axes"):
        b200_step(g, alloc_like(g), spec, ranges=[(0, 4), (0, 4)])
    c = Counters()
    b200_step(g, alloc_like(g), spec, c, ranges=[(5, 5)])    # empty box: no work, no count
    assert c.point_updates == 0


@pytest.mark.parametrize("preset,dims,ranges", [
    ("1d5p", (1000,), [(17, 403)]),
    ("2d9p", (41, 66), [(40, 41), (65, 66)]),
    ("3d27p", (9, 20, 33), [(2, 7), (5, 6), (1, 32)]),
    ("3d7p", (6, 7, 9), [(0, 6), (0, 7), (0, 9)]),
])
def test_box_as_own_grid_is_the_whole_step_restricted(preset, dims, ranges):
    # the premise of b200_step's NATURAL ranges path, checked on the oracle:
    # stepping the box + r neighbourhood as a grid of its own (its halo = src
    # around the box) gives bit for bit the whole-grid step on the box
    spec = make_stencil_spec(preset)
    src = alloc_grid(spec, dims)
    src.set_interior(np.random.default_rng(11).random(dims))
    offs, ws = canonical(spec)
    r = spec.r
    box = compact_view(src)[tuple(slice(lo, hi + 2 * r) for lo, hi in ranges)]
    got = c_oracle.sweep(np.ascontiguousarray(box), r, offs, ws, 1)
    got = got[tuple(slice(r, s - r) for s in got.shape)]
    want = _oracle_step(spec, src)[tuple(slice(lo, hi) for lo, hi in ranges)]
    assert np.array_equal(got, want)


def _oracle_step(spec, src):
    offs, ws = canonical(spec)
    want = c_oracle.sweep(np.ascontiguousarray(compact_view(src)), spec.r, offs, ws, 1)
    r = spec.r
    return want[tuple(slice(r, s - r) for s in want.shape)]


@pytest.mark.gpu
@pytest.mark.parametrize("preset,dims,ranges", [
    ("1d5p", (1000,), [(17, 403)]),
    ("2d9p", (41, 66), [(3, 40), (0, 9)]),
    ("2d5p", (40, 70), [(0, 40), (33, 70)]),
    ("3d27p", (9, 20, 33), [(2, 7), (5, 6), (1, 32)]),
    ("3d7p", (8, 21, 30), [(0, 8), (0, 21), (0, 30)]),
    ("2d9p", (41, 66), [(40, 41), (65, 66)]),          # one corner point
    ("1d3p", (64,), [(0, 1)]),
    ("3d27p", (6, 7, 9), [(0, 1), (3, 7), (8, 9)]),
])
def test_step_ranges_writes_only_the_box(preset, dims, ranges):
    # scalar_step(..., ranges=...) semantics (kernels.py:88-134)
    spec = make_stencil_spec(preset)
    src = alloc_grid(spec, dims)
    src.set_interior(np.random.default_rng(7).random(dims))
    dst = alloc_like(src)
    dst.set_interior(np.full(dims, -7.0))
    c = Counters()
    b200_step(src, dst, spec, c, ranges=ranges)
    got = dst.natural_interior()
    want = _oracle_step(spec, src)
    sel = tuple(slice(lo, hi) for lo, hi in ranges)
    assert np.array_equal(got[sel], want[sel])
    outside = np.ones(dims, bool)
    outside[sel] = False
    assert np.all(got[outside] == -7.0)
    assert c.point_updates == int(np.prod([hi - lo for lo, hi in ranges]))


@pytest.mark.gpu
def test_tiled_steps_cover_exactly_once():
    # a tile runner in the reference's style (tiling.py:353-354): disjoint
    # ranges covering the interior, T ping-pong steps -> the untiled result
    spec = config_spec("c3b")
    dims = (37, 50)
    a = alloc_grid(spec, dims)
    a.set_interior(np.random.default_rng(3).random(dims))
    b = alloc_like(a)
    start = a.natural_interior().copy()
    tiles = [[(0, 12), (0, 20)], [(0, 12), (20, 50)], [(12, 37), (0, 7)], [(12, 37), (7, 50)]]
    c = Counters()
    for _ in range(3):
        for t in tiles:
            b200_step(a, b, spec, c, ranges=t)
        a, b = b, a
    assert c.point_updates == 3 * 37 * 50
    ref = alloc_grid(spec, dims)
    ref.set_interior(start)
    b200_sweep(ref, spec, 1, 3)
    assert np.array_equal(a.natural_interior(), ref.natural_interior())


@pytest.mark.gpu
@pytest.mark.parametrize("preset,dims", [("1d3p", (1000,)), ("1d5p", (999,)), ("2d5p", (40, 70)),
                                         ("2d9p", (41, 66)), ("3d7p", (9, 20, 33)), ("3d27p", (8, 21, 30))])
def test_step_equals_oracle_step(preset, dims):
    spec = make_stencil_spec(preset)
    src = alloc_grid(spec, dims)
    src.set_interior(np.random.default_rng(5).random(dims))
    dst = alloc_like(src)
    c = Counters()
    b200_step(src, dst, spec, c)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(np.ascontiguousarray(compact_view(src)), spec.r, offs, ws, 1)
    r = spec.r
    assert np.array_equal(dst.natural_interior(), want[tuple(slice(r, s - r) for s in want.shape)])
    assert c.point_updates == int(np.prod(dims))
    assert not dst.data[..., :r].any()          # halo untouched (still zero)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,dims,k,T", [("c2", (4096,), 2, 100), ("c2", (4096,), 16, 100),
                                          ("c4", (20, 30, 40), 4, 10), ("c3b", (100, 90), 8, 20)])
def test_sweep_in_place_like_jam_sweep(cfg, dims, k, T):
    spec = config_spec(cfg)
    g = alloc_grid(spec, dims)
    g.set_interior(np.random.default_rng(99).random(dims))
    before = np.array(compact_view(g), copy=True)   # 1D views are contiguous: copy
    buf = g.data
    c = Counters()
    b200_sweep(g, spec, k, T, c)
    assert g.data is buf                      # advanced in place (test_timejam.py:148-153)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(before, spec.r, offs, ws, T)
    r = spec.r
    assert np.array_equal(g.natural_interior(), want[tuple(slice(r, s - r) for s in want.shape)])
    assert c.point_updates == int(np.prod(dims)) * T


@pytest.mark.gpu
def test_reference_gridbuffer_if_importable():
    ref = pytest.importorskip("stencilbench.core", reason="reference not present on this host")
    from stencilbench.kernels import scalar_step
    spec = ref.make_stencil_spec("2d9p")
    a = ref.alloc_grid(spec, (33, 47), ref.Layout.NATURAL, 4)
    a.set_interior(np.random.default_rng(1).random((33, 47)))
    b, b2 = ref.alloc_like(a), ref.alloc_like(a)
    scalar_step(a, b, spec)
    b200_step(a, b2, spec)
    assert np.array_equal(b.natural_interior(), b2.natural_interior())


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,dims,k,T", [("c3b", (130, 300), 4, 9), ("c5", (20, 30, 70), 2, 5),
                                          ("c4", (17, 33, 129), 2, 6)])
def test_sweep_natural_grid_in_place_pitched(cfg, dims, k, T):
    # a NATURAL GridBuffer is uploaded / written back in place as pitched rows
    # (sb_upload_pitched / sb_download_pitched): every cell of the storage array is seeded,
    # the compact box (halo held at its values) must equal the oracle's bit for bit and the
    # cells outside it (the unit axis' extra halo, core.py:335-362) must not be touched
    spec = config_spec(cfg)
    g = alloc_grid(spec, dims)
    g.data[...] = np.random.default_rng(int(np.prod(dims))).random(g.data.shape)
    snap = g.data.copy()
    before = np.array(compact_view(g), copy=True)
    b200_sweep(g, spec, k, T, arith="exact")
    offs, ws = canonical(spec)
    want = c_oracle.sweep(before, spec.r, offs, ws, T)
    assert np.array_equal(compact_view(g), want)
    outside = np.ones(g.data.shape, bool)
    hu, r = g.halo_unit, spec.r
    outside[..., hu - r:hu + g.unit_n + r] = False
    assert np.array_equal(g.data[outside], snap[outside])
