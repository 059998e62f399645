"""The b200 methods driven by the REFERENCE's own code paths.

``register`` puts ``"b200"`` (NATURAL), ``"b200_transpose"`` (BLOCK_TRANSPOSE)
and ``"b200_dlt"`` (DLT) into the real ``stencilbench.kernels.METHODS``
(kernels.py:538-544); then, unchanged reference code dispatches to them:

* ``stencilbench.harness.run_benchmark`` -> ``_execute`` one step per time
  step (harness.py:187-201), verified against the reference's own
  ``run_oracle`` (harness.py:149-157, 233-235): ``err == 0.0`` like
  test_harness.py:45;
* ``stencilbench.tiling.run_tiled`` -> ``METHODS[m][1](..., ranges=slab)``
  from ThreadPoolExecutor workers (tiling.py:353-354, 372-417), bit-identical
  for workers in {1, 2, 4, 8} (test_tiling.py:175-185) and to the oracle;
* the reference CLI's validation accepts the registered methods.

The reference comes from baseline/_ref (the per-pod install, which travels to
the GPU box) or the build container's source tree; absent both, these skip.
"""

import numpy as np
import pytest

sb = pytest.importorskip("stencilbench", reason="reference package not installed (baseline/_ref)")

from stencilbench import harness as ref_harness  # noqa: E402
from stencilbench import kernels as ref_kernels  # noqa: E402
from stencilbench import tiling as ref_tiling  # noqa: E402
from stencilbench.core import Layout, alloc_grid, alloc_like, make_stencil_spec  # noqa: E402
from stencilbench.transpose import to_block_transpose  # noqa: E402

from paper_2103_08825_b200.kernels import b200_step, register  # noqa: E402

METHODS = ("b200", "b200_transpose", "b200_dlt")


@pytest.fixture(autouse=True)
def registered():
    register(ref_kernels.METHODS, Layout)
    yield
    for m in METHODS:
        ref_kernels.METHODS.pop(m, None)


def natural(spec, dims, values):
    g = alloc_grid(spec, dims, Layout.NATURAL, 4)
    g.set_interior(values)
    return g


def oracle_steps(spec, values, dims, T):
    a = natural(spec, dims, values)
    b = alloc_like(a)
    for _ in range(T):
        ref_kernels.scalar_step(a, b, spec)
        a, b = b, a
    return a.natural_interior()


# ---------------------------------------------------------------- CPU (no device)

def test_register_into_reference_registry():
    assert ref_kernels.METHODS["b200"] == (Layout.NATURAL, b200_step)
    assert ref_kernels.METHODS["b200_transpose"][0] is Layout.BLOCK_TRANSPOSE
    assert ref_kernels.METHODS["b200_dlt"][0] is Layout.DLT
    assert ref_kernels.method_layout("b200") is Layout.NATURAL
    # the reference's own validation now accepts the methods (harness.py:86-128)
    ref_harness.validate_config(ref_harness.BenchConfig("3d27p", (8, 8, 8), 4, "b200"))
    ref_harness.validate_config(ref_harness.BenchConfig("1d3p", (256,), 8, "b200", block=(64,), tile_height=4))


def test_reference_tile_runner_rejects_layout_mismatch():
    spec = make_stencil_spec("1d3p")
    g = natural(spec, 64, np.zeros(64))
    sched = ref_tiling.build_tessellation_1d(64, 16, 4, 1, total_steps=8)
    with pytest.raises(sb.core.GridError, match="layout"):
        ref_tiling.run_tiled(g, spec, sched, "b200_transpose")


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("stencil,dims,steps", [
    ("1d3p", (300,), 7), ("1d5p", (257,), 6), ("2d9p", (19, 37), 5), ("2d5p", (16, 40), 4),
    ("3d7p", (6, 9, 21), 4), ("3d27p", (5, 7, 18), 3),
])
def test_reference_run_benchmark_verify(method, stencil, dims, steps):
    cfg = ref_harness.BenchConfig(stencil, dims, steps, method, verify=True)
    res = ref_harness.run_benchmark(cfg)
    assert res.max_rel_err == 0.0                                  # test_harness.py:45
    assert res.counters.point_updates == int(np.prod(dims)) * steps
    assert res.gflops > 0


@pytest.mark.gpu
@pytest.mark.parametrize("stencil,n,B,T_b,T", [("1d3p", 1024, 256, 16, 32), ("1d5p", 512, 128, 16, 31)])
def test_reference_run_tiled_1d_worker_determinism(stencil, n, B, T_b, T):
    spec = make_stencil_spec(stencil)
    vals = np.random.default_rng(21).random(n)
    want = oracle_steps(spec, vals, (n,), T)
    outs = []
    for workers in (1, 2, 4, 8):
        g = natural(spec, n, vals)
        sched = ref_tiling.build_tessellation_1d(n, B, T_b, spec.r, total_steps=T)
        counters = ref_kernels.Counters()
        ref_tiling.run_tiled(g, spec, sched, "b200", workers=workers, counters=counters)
        assert counters.point_updates == n * T                    # each point once per level
        outs.append(g.natural_interior())
    for o in outs:
        assert np.array_equal(o, want)


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 2, 4, 8])
def test_reference_run_tiled_2d(workers):
    spec = make_stencil_spec("2d9p")
    dims, B, T_b, T = (32, 48), 16, 4, 12
    vals = np.random.default_rng(11).random(dims)
    g = natural(spec, dims, vals)
    sched = ref_tiling.build_tessellation_2d(dims, B, T_b, 1, total_steps=T)
    ref_tiling.run_tiled(g, spec, sched, "b200", workers=workers)
    assert np.array_equal(g.natural_interior(), oracle_steps(spec, vals, dims, T))


@pytest.mark.gpu
def test_reference_run_tiled_block_transpose_grid():
    spec = make_stencil_spec("1d3p")
    n, T = 512, 16
    vals = np.random.default_rng(3).random(n)
    g = alloc_grid(spec, n, Layout.NATURAL, 4, pad_for=Layout.BLOCK_TRANSPOSE)
    g.set_interior(vals)
    to_block_transpose(g, 4)
    sched = ref_tiling.build_tessellation_1d(n, 128, 8, 1, total_steps=T)
    ref_tiling.run_tiled(g, spec, sched, "b200_transpose", workers=4)
    assert np.array_equal(g.natural_interior(), oracle_steps(spec, vals, (n,), T))


@pytest.mark.gpu
def test_reference_harness_tiled_config():
    cfg = ref_harness.BenchConfig("1d5p", (512,), 24, "b200", block=(128,), tile_height=8, workers=4, verify=True)
    res = ref_harness.run_benchmark(cfg)
    assert res.max_rel_err == 0.0 and res.tile_height_used == 8


@pytest.mark.gpu
def test_grid_sized_for_larger_order():
    # a grid whose halo was sized for r=2 stepped with an r=1 stencil: the
    # reference's _region offsets by the grid's own halo (kernels.py:88-100)
    spec = make_stencil_spec("2d9p")
    r2 = sb.core.StencilSpec("r2", 2, 2, "box", {(i, j): 1.0 / 25 for i in range(-2, 3) for j in range(-2, 3)})
    big = alloc_grid(r2, (9, 14), Layout.NATURAL, 4)
    big.set_interior(np.random.default_rng(5).random((9, 14)))
    big.data[0, :] = 7.0                                          # halo beyond r=1: never read
    for ranges in (None, [(2, 7), (3, 11)]):
        dst, ref = alloc_like(big), alloc_like(big)
        b200_step(big, dst, spec, ranges=ranges)
        ref_kernels.scalar_step(big, ref, spec, ranges=ranges)
        assert np.array_equal(dst.data, ref.data)
