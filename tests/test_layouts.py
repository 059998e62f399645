"""BLOCK_TRANSPOSE / DLT storage layouts.

Fixtures ``tests/golden/l_*.npz`` come from the reference itself
(``make_golden_layouts.py``: ``transpose.to_block_transpose`` / ``to_dlt``,
``transpose_layout_step``, ``dlt_step``, ``jam_sweep``).  CPU tests pin the
host-side index map and the oracle against them; GPU tests pin the device
conversions (``sb_layout_convert``), the plan's storage upload/download and
the layout-aware drop-ins, bit for bit, the way the reference pins its own
layouts (test_kernels.py:82, test_timejam.py:94, test_transpose.py).
"""

from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from oracle import c_oracle

from paper_2103_08825_b200.core import GridError, StencilSpec, canonical
from paper_2103_08825_b200.grid import GridBuffer, Layout, alloc_grid, unit_permutation

NAMES = sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "l_*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = {k: z[k] for k in z.files}
    for k in ("d", "r", "vl", "unit_np", "halo_unit"):
        g[k] = int(g[k])
    g["layout"] = str(g["layout"])
    g["shape"] = str(g["shape"])
    g["dims"] = tuple(int(n) for n in g["dims"])
    g["offsets"] = [tuple(int(c) for c in row) for row in g["offsets"]]
    g["weights"] = [float(w) for w in g["weights"]]
    g["spec"] = StencilSpec("golden", g["d"], g["r"], g["shape"], dict(zip(g["offsets"], g["weights"])))
    return g


def grid_of(g, key):
    lay = Layout.NATURAL if key == "nat" else Layout(g["layout"])
    return GridBuffer(g[key].copy(), g["dims"], g["r"], g["dims"][-1], g["unit_np"], lay, g["vl"])


def step_keys(g):
    return sorted((int(k[len("step_T"):]), k) for k in g if k.startswith("step_T"))


def test_fixtures_present():
    assert len(NAMES) == 8


# ------------------------------------------------------------------ CPU


@pytest.mark.parametrize("name", NAMES)
def test_host_permutation_matches_reference(name):
    # core.py:206-229 restated in grid.unit_permutation; the reference's own
    # to_block_transpose / to_dlt produced `lay` from `nat`
    g = load(name)
    hu, unp = g["halo_unit"], g["unit_np"]
    perm = unit_permutation(g["layout"], unp, g["vl"])
    want = g["nat"].copy()
    want[..., hu + perm] = g["nat"][..., hu:hu + unp]
    assert want.tobytes() == g["lay"].tobytes()


@pytest.mark.parametrize("name", NAMES)
def test_alloc_geometry_and_interior_accessors(name):
    g = load(name)
    a = alloc_grid(g["spec"], g["dims"], Layout(g["layout"]), g["vl"])
    assert a.data.shape == g["lay"].shape and a.unit_np == g["unit_np"]
    n = alloc_grid(g["spec"], g["dims"], Layout.NATURAL, g["vl"], pad_for=Layout(g["layout"]))
    assert n.data.shape == g["nat"].shape
    lay, nat = grid_of(g, "lay"), grid_of(g, "nat")
    assert lay.natural_interior().tobytes() == nat.natural_interior().tobytes()
    fresh = alloc_grid(g["spec"], g["dims"], Layout(g["layout"]), g["vl"])
    fresh.set_interior(nat.natural_interior())
    assert fresh.natural_interior().tobytes() == nat.natural_interior().tobytes()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_layout_methods(name):
    # transpose_layout_step / dlt_step / jam_sweep == scalar_step in natural
    # order: the C oracle on the natural box reproduces every stored result
    g = load(name)
    spec, r, hu = g["spec"], g["r"], g["halo_unit"]
    offs, ws = canonical(spec)
    box = np.ascontiguousarray(g["nat"][..., hu - r:hu + g["dims"][-1] + r])
    for T, key in step_keys(g) + [(int(k.rsplit("T", 1)[1]), k) for k in g if k.startswith("jam_k2_T")]:
        want = c_oracle.sweep(box, r, offs, ws, T)
        got = grid_of(g, key)
        inner = want[tuple(slice(r, s - r) for s in want.shape)]
        assert got.natural_interior().tobytes() == inner.tobytes(), key


def test_register_adds_layout_methods():
    from paper_2103_08825_b200.kernels import b200_step, register
    methods = {}
    register(methods, Layout.NATURAL)
    assert methods["b200"] == (Layout.NATURAL, b200_step)
    assert methods["b200_transpose"] == (Layout.BLOCK_TRANSPOSE, b200_step)
    assert methods["b200_dlt"] == (Layout.DLT, b200_step)


def test_conversion_argument_checks():
    from paper_2103_08825_b200 import transpose as tr
    spec = StencilSpec("s", 1, 1, "star", {(-1,): 0.25, (0,): 0.5, (1,): 0.25})
    g = alloc_grid(spec, 30, Layout.NATURAL, 4)           # unit_np 30: not a multiple of 16
    with pytest.raises(GridError, match="multiple of 16"):
        tr.to_block_transpose(g, 4)
    with pytest.raises(GridError, match="vl=4"):
        tr.to_dlt(g, 8)
    with pytest.raises(GridError, match="BLOCK_TRANSPOSE"):
        tr.from_block_transpose(g)
    with pytest.raises(GridError, match="vl must be"):
        alloc_grid(spec, 30, Layout.NATURAL, 6)


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_conversion_bit_exact(name):
    from paper_2103_08825_b200 import transpose as tr
    g = load(name)
    nat = grid_of(g, "nat")
    conv = tr.to_block_transpose if g["layout"] == "block_transpose" else tr.to_dlt
    back = tr.from_block_transpose if g["layout"] == "block_transpose" else tr.from_dlt
    conv(nat, g["vl"])
    assert nat.layout is Layout(g["layout"])
    assert nat.data.tobytes() == g["lay"].tobytes()
    back(nat)
    assert nat.layout is Layout.NATURAL
    assert nat.data.tobytes() == g["nat"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_plan_storage_sweep_matches_layout_method(name):
    # storage in the layout -> device (un-permuted) -> T exact steps ->
    # re-permuted storage: the whole array equals the reference method's result
    from paper_2103_08825_b200.plan import Plan
    g = load(name)
    lay = grid_of(g, "lay")
    for T, key in step_keys(g):
        with Plan(g["spec"], g["dims"], arith="exact", k=1) as p:
            p.upload_storage(lay)
            p.run(T)
            out = p.download_storage(lay)
        assert out.tobytes() == g[key].tobytes(), key


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in NAMES if "_bt" in n and n.startswith("l_1d")])
def test_sweep_is_a_jam_sweep_dropin(name):
    # b200_sweep on a BLOCK_TRANSPOSE grid == timejam.jam_sweep(grid, spec, 2, T)
    from paper_2103_08825_b200.kernels import b200_sweep
    g = load(name)
    for key in [k for k in g if k.startswith("jam_k2_T")]:
        T = int(key.rsplit("T", 1)[1])
        grid = grid_of(g, "lay")
        b200_sweep(grid, g["spec"], 2, T)
        assert grid.data.tobytes() == g[key].tobytes(), key


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_step_on_layout_grids(name):
    # METHODS-style step on layout grids: dst interior written, dst halo untouched
    from paper_2103_08825_b200.kernels import b200_step
    g = load(name)
    src = grid_of(g, "lay")
    dst = grid_of(g, "lay")
    dst.data[...] = -1.0
    b200_step(src, dst, g["spec"])
    want = grid_of(g, "step_T1")
    assert dst.natural_interior().tobytes() == want.natural_interior().tobytes()
    untouched = dst.data == -1.0
    hu, r = g["halo_unit"], g["r"]
    perm = unit_permutation(g["layout"], g["unit_np"], g["vl"])
    mask = np.ones(dst.data.shape, bool)
    outer = tuple(slice(r, r + n) for n in g["dims"][:-1])
    mask[outer + (hu + perm[:g["dims"][-1]],)] = False
    assert untouched[mask].all()


@pytest.mark.gpu
def test_step_ranges_on_layout_grid():
    from paper_2103_08825_b200.kernels import b200_step
    g = load("l_2d9p_bt4")
    src, dst = grid_of(g, "lay"), grid_of(g, "lay")
    before = dst.natural_interior()
    ranges = [(2, 7), (5, 30)]
    b200_step(src, dst, g["spec"], ranges=ranges)
    got = dst.natural_interior()
    want = grid_of(g, "step_T1").natural_interior()
    box = (slice(2, 7), slice(5, 30))
    assert got[box].tobytes() == want[box].tobytes()
    mask = np.ones(got.shape, bool)
    mask[box] = False
    assert (got[mask] == before[mask]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("layout,vl,shape", [("block_transpose", 8, (1030, 4096 + 8)),
                                             ("dlt", 4, (515, 8200)), ("dlt", 8, (3, 2**20 + 16))])
def test_device_conversion_large_round_trip(layout, vl, shape):
    # sizes far past one tile per row: device result == host index map, and
    # converting back restores the input bit for bit
    import torch
    from paper_2103_08825_b200 import transpose as tr
    hu = 4
    unp = shape[1] - 2 * hu
    like = GridBuffer(np.zeros((1, 1)), (shape[0] - 2, unp), 2, unp, unp, Layout(layout), vl)
    host = np.random.default_rng(5).random(shape)
    src = torch.from_numpy(host).cuda()
    dst = torch.empty_like(src)
    tr.convert_device(src, dst, like, True)
    back = torch.empty_like(src)
    tr.convert_device(dst, back, like, False)
    torch.cuda.synchronize()
    perm = unit_permutation(layout, unp, vl)
    want = host.copy()
    want[:, hu + perm] = host[:, hu:hu + unp]
    assert dst.cpu().numpy().tobytes() == want.tobytes()
    assert back.cpu().numpy().tobytes() == host.tobytes()
