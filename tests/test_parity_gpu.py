"""Parity of the sm_100a path against the reference (GPU, ``-m gpu``).

* EXACT arithmetic is bit-identical to the reference's own outputs (golden
  fixtures made by ``stencilbench.kernels.scalar_step``), for every fixture,
  both halo conventions, the generic and the fused kernels, every fused depth.
* FMA arithmetic stays within the north_star fp64 bar (1e-12 relative).
* fp32 stays within 1e-5 of the fp64 oracle run on fp32-rounded inputs and
  weights (the reference is fp64-only).
* Full BASELINE sizes are checked through the C oracle and size-independent
  properties (constant preservation, halo preservation, linearity).
"""

import os

import numpy as np
import pytest

from conftest import golden_names, golden_spec, interior, load_golden, seeded_box
from oracle import c_oracle, np_oracle

from paper_2103_08825_b200.core import canonical, config_spec, make_stencil_spec
from paper_2103_08825_b200.plan import Plan, sweep

pytestmark = pytest.mark.gpu

NAMES = golden_names()
FP64_TOL = 1e-12
FP32_TOL = 1e-5


def oracle(spec, box, T):
    offs, ws = canonical(spec)
    return c_oracle.sweep(box, spec.r, offs, ws, T)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("halo", ["zero", "full"])
@pytest.mark.parametrize("kernel", ["generic", "auto"])
def test_exact_bit_identical_to_reference(name, halo, kernel):
    g = load_golden(name)
    spec = golden_spec(g)
    for T in g["steps"]:
        got = sweep(spec, g[f"in_{halo}"], T, arith="exact", kernel=kernel)
        want = g[f"out_{halo}_T{T}"]
        assert got.tobytes() == want.tobytes(), (name, halo, kernel, T)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("halo", ["zero", "full"])
def test_fma_within_fp64_bar(name, halo):
    g = load_golden(name)
    spec = golden_spec(g)
    T = g["steps"][-1]
    got = sweep(spec, g[f"in_{halo}"], T, arith="fma")
    want = g[f"out_{halo}_T{T}"]
    assert np_oracle.max_rel_error(interior(got, g["r"]), interior(want, g["r"])) <= FP64_TOL
    mask = np.ones(got.shape, bool)
    mask[tuple(slice(g["r"], s - g["r"]) for s in got.shape)] = False
    assert np.array_equal(got[mask], want[mask])          # halo untouched


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("k", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("n", [1, 5, 63, 1000, 70001])
def test_fused1d_every_depth_exact(cfg, k, n):
    spec = config_spec(cfg)
    box = seeded_box((n,), spec.r, seed=n + k)
    T = 37                                   # not a multiple of k: exercises the tail
    got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, T).tobytes()


@pytest.mark.parametrize("k", [1, 8, 16])
def test_fused1d_fp32(k):
    spec = config_spec("c2")
    box = seeded_box((100003,), 2, seed=3)
    box32 = box.astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 2, offs, [float(np.float32(w)) for w in ws], 50)
    got = sweep(spec, box32, 50, arith="fma", k=k)
    assert got.dtype == np.float32
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


@pytest.mark.parametrize("key,dims", [("c3b", (67, 300)), ("c5", (20, 24, 70)), ("c4", (17, 30, 40))])
def test_generic_fp32(key, dims):
    spec = config_spec(key)
    box32 = seeded_box(dims, 1, seed=9).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs, [float(np.float32(w)) for w in ws], 12)
    got = sweep(spec, box32, 12, arith="fma")
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


# --- reference known-answer tests (stencilbench tests/test_kernels.py:80-104)

def test_impulse_response():
    spec = make_stencil_spec("1d3p")
    box = np.zeros(7)
    box[3] = 1.0
    for kernel in ("generic", "fused"):
        out = sweep(spec, box, 1, arith="exact", kernel=kernel)
        assert out[1:-1].tolist() == [0, 0.25, 0.5, 0.25, 0]


def test_linear_ramp_fixed_point():
    spec = make_stencil_spec("1d3p")
    n = 32
    box = np.zeros(n + 2)
    box[1:-1] = np.arange(float(n))
    out = sweep(spec, box, 1, arith="exact")
    assert np.array_equal(out[2:-2], np.arange(1.0, n - 1))


@pytest.mark.parametrize("preset,dims", [("2d9p", (12, 32)), ("3d27p", (6, 7, 20)), ("1d5p", (64,))])
def test_constant_preserved(preset, dims):
    spec = make_stencil_spec(preset)
    box = np.full(tuple(n + 2 * spec.r for n in dims), 2.5)
    for arith in ("exact", "fma"):
        assert np.all(sweep(spec, box, 9, arith=arith) == 2.5)


def test_impulse_locality():
    spec = make_stencil_spec("1d5p")
    box = np.zeros(68)
    box[2 + 31] = 1.0
    out = sweep(spec, box, 1, arith="exact")
    support = np.flatnonzero(out[2:-2])
    assert support.min() >= 31 - 2 and support.max() <= 31 + 2


# --- full BASELINE sizes --------------------------------------------------------

def test_c1_full_size_exact():
    spec = config_spec("c1")
    box = seeded_box((1 << 20,), 1)
    got = sweep(spec, box, 64, arith="exact")
    assert got.tobytes() == oracle(spec, box, 64).tobytes()


def test_c2_full_size_fma_k8():
    spec = config_spec("c2")
    box = seeded_box((1 << 26,), 2)
    got = sweep(spec, box, 24, arith="fma", k=8)
    want = oracle(spec, box, 24)
    assert np_oracle.max_rel_error(got, want) <= FP64_TOL


def test_c2_full_size_exact_k16_halo_zero():
    spec = config_spec("c2")
    box = seeded_box((1 << 26,), 2, halo="zero")
    got = sweep(spec, box, 16, arith="exact", k=16)
    assert got.tobytes() == oracle(spec, box, 16).tobytes()


def test_linearity_full_c2():
    spec = config_spec("c2")
    a = seeded_box((1 << 26,), 2, seed=1)
    b = seeded_box((1 << 26,), 2, seed=2)
    sa = sweep(spec, a, 40, k=8)
    sb = sweep(spec, b, 40, k=8)
    sab = sweep(spec, 0.5 * a + 0.25 * b, 40, k=8)
    assert np_oracle.max_rel_error(sab, 0.5 * sa + 0.25 * sb) <= 1e-12


# --- composed 1D path (FMA, depth k as one (2rk+1)-tap stencil + exact boundary windows)

@pytest.mark.parametrize("cfg,k", [("c1", 16), ("c1", 32), ("c1", 64), ("c2", 16), ("c2", 32)])
@pytest.mark.parametrize("n", [12288, 12289, 100003])
@pytest.mark.parametrize("halo", ["full", "zero"])
def test_composed1d_within_fp64_bar(cfg, k, n, halo):
    spec = config_spec(cfg)
    box = seeded_box((n,), spec.r, seed=n + k, halo=halo)
    T = 2 * k + 7                            # full-depth launches plus a shallower tail
    with Plan(spec, (n,), k=k, arith="fma") as p:
        p.upload(box)
        t = p.run(T)
        got = p.download()
    assert t.kernel_name in ("compose1d_kernel", "fused1d_kernel")
    want = oracle(spec, box, T)
    assert np_oracle.max_rel_error(interior(got, spec.r), interior(want, spec.r)) <= FP64_TOL
    assert np.array_equal(got[:spec.r], box[:spec.r]) and np.array_equal(got[-spec.r:], box[-spec.r:])


def test_composed1d_boundary_values_exact_level_by_level():
    # outputs within r*k of the Dirichlet halo come from the exact window kernel:
    # with an impulse next to the boundary they match the level-by-level oracle
    spec = config_spec("c1")
    n = 20000
    box = np.zeros(n + 2)
    box[1:40] = np.linspace(1.0, 2.0, 39)
    box[0] = 3.0
    box[-1] = -1.0
    box[-40:-1] = 0.5
    got = sweep(spec, box, 64, arith="fma", k=64)
    want = oracle(spec, box, 64)
    assert np_oracle.max_rel_error(got, want) <= FP64_TOL


def test_composed1d_fp32_k32():
    spec = config_spec("c2")
    box32 = seeded_box((100003,), 2, seed=4).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 2, offs, [float(np.float32(w)) for w in ws], 64)
    got = sweep(spec, box32, 64, arith="fma", k=32)
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


def test_c1_full_size_one_launch_k64():
    spec = config_spec("c1")
    box = seeded_box((1 << 20,), 1)
    with Plan(spec, (1 << 20,), k=64, arith="fma") as p:
        p.upload(box)
        t = p.run(64)
        got = p.download()
    assert t.launches == 1 and t.kernel_name == "compose1d_kernel"   # composed + boundary windows, one launch
    assert np_oracle.max_rel_error(got, oracle(spec, box, 64)) <= FP64_TOL


def test_composed_depth_rejected_when_unavailable():
    spec = config_spec("c2")
    with pytest.raises(ValueError):
        Plan(spec, (100000,), k=64, arith="fma")       # r*k = 128 > 64
    with pytest.raises(ValueError):
        Plan(spec, (100000,), k=32, arith="exact")     # composed path is FMA-only


def test_plan_reuse_and_timing():
    spec = config_spec("c2")
    box = seeded_box((100000,), 2)
    with Plan(spec, (100000,), k=8) as p:
        p.upload(box)
        t = p.run(20)
        assert t.point_updates == 100000 * 20
        assert t.k_used == 8 and t.launches == 6          # (8 + 8 + 4) x (interior + boundary kernel)
        assert t.kernel_name == "fused1d_kernel"
        mid = p.download()
        p.run(20)
        end = p.download()
    want_mid = oracle(spec, box, 20)
    assert np_oracle.max_rel_error(mid, want_mid) <= FP64_TOL
    assert np_oracle.max_rel_error(end, oracle(spec, want_mid, 20)) <= FP64_TOL


# --- fused 3D kernel (TMA-fed 2.5D temporal blocking) ---------------------------

@pytest.mark.parametrize("cfg", ["c4", "c5"])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("dims", [(3, 5, 7), (9, 40, 70), (37, 33, 130)])
def test_fused3d_every_depth_exact(cfg, k, dims):
    spec = config_spec(cfg)
    box = seeded_box(dims, 1, seed=sum(dims) + k)
    T = 7                                    # not a multiple of k for k in {2,3,4}
    got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, T).tobytes()


@pytest.mark.parametrize("cfg,k", [("c4", 4), ("c5", 2)])
def test_fused3d_halo_zero_exact(cfg, k):
    spec = config_spec(cfg)
    box = seeded_box((20, 70, 66), 1, seed=5, halo="zero")
    got = sweep(spec, box, 9, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, 9).tobytes()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_fused3d_fp32(k):
    spec = config_spec("c5")
    box32 = seeded_box((30, 70, 130), 1, seed=11).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs, [float(np.float32(w)) for w in ws], 12)
    got = sweep(spec, box32, 12, arith="fma", kernel="fused", k=k)
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


def test_c5_full_size_fma():
    spec = config_spec("c5")
    box = seeded_box((768, 768, 768), 1)
    got = sweep(spec, box, 4, arith="fma", k=2)
    want = oracle(spec, box, 4)
    assert np_oracle.max_rel_error(got, want) <= FP64_TOL


# --- non-finite values: NaN / Inf spread through exactly the oracle's cone

@pytest.mark.parametrize("cfg,dims,k,arith", [
    ("c2", (20000,), 32, "fma"), ("c2", (5000,), 8, "exact"), ("c3a", (40, 130), 4, "fma"),
    ("c3b", (40, 130), 8, "exact"), ("c4", (12, 30, 70), 2, "fma"), ("c5", (10, 30, 66), 2, "fma"),
])
def test_nonfinite_propagation_matches_oracle(cfg, dims, k, arith):
    spec = config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=3)
    mid = tuple(n // 2 + spec.r for n in dims)
    box[mid] = np.nan
    edge = tuple(spec.r for _ in dims)                 # first interior point, next to the halo
    box[edge] = np.inf
    T = 2 * k + 1
    got = sweep(spec, box, T, arith=arith, k=k)
    want = oracle(spec, box, T)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isposinf(got), np.isposinf(want))
    fin = np.isfinite(want)
    assert np_oracle.max_rel_error(got[fin], want[fin]) <= FP64_TOL


# --- range launches (slab edge planes first, interior later: sb_launch_range)

@pytest.mark.parametrize("cfg,dims,k,arith", [
    ("c3b", (60, 130), 4, "exact"), ("c3a", (61, 140), 8, "fma"), ("c3a", (130, 150), 32, "fma"),
    ("c3a", (90, 150), 16, "fma"), ("c4", (30, 37, 70), 2, "fma"),
    ("c4", (30, 37, 70), 3, "exact"), ("c5", (25, 33, 66), 2, "fma"), ("p:2d5p", (33, 50), 1, "exact"),
])
def test_range_launches_compose_a_full_launch(cfg, dims, k, arith):
    spec = make_stencil_spec(cfg[2:]) if cfg.startswith("p:") else config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=sum(dims))
    n0 = dims[0]
    with Plan(spec, dims, k=k, arith=arith) as p:
        p.upload(box)
        p.launch(k)
        p.synchronize()
        want = p.download()
    cuts = [0, 3, n0 - 5, n0]
    with Plan(spec, dims, k=k, arith=arith) as p:
        p.upload(box)
        for i, (lo, hi) in enumerate(zip(cuts[:-1], cuts[1:])):
            p.launch_range(k, lo, hi, i == len(cuts) - 2)
        p.synchronize()
        got = p.download()
    assert got.tobytes() == want.tobytes()


# --- separable 2D box (FMA, rank-1 weights: horizontal pass + vertical push)

@pytest.mark.parametrize("k", [1, 2, 4, 8])
@pytest.mark.parametrize("dims", [(5, 7), (40, 130), (97, 301)])
def test_separable2d_within_fp64_bar(k, dims):
    from paper_2103_08825_b200.core import StencilSpec
    a, b = np.array([0.2, 0.5, 0.3]), np.array([0.15, 0.6, 0.25])
    w = {(dy, dx): float(a[dy + 1] * b[dx + 1]) for dy in (-1, 0, 1) for dx in (-1, 0, 1)}
    for spec in (config_spec("c3a"), StencilSpec("rank1", 2, 1, "box", w)):
        box = seeded_box(dims, 1, seed=sum(dims) + k)
        T = 2 * k + 3
        got = sweep(spec, box, T, arith="fma", kernel="fused", k=k)
        assert np_oracle.max_rel_error(got, oracle(spec, box, T)) <= FP64_TOL


# --- separable composed 2D (FMA, rank-1 weights, K = 16 / 32 as two 1D passes + exact bands)

@pytest.mark.parametrize("k", [16, 32])
@pytest.mark.parametrize("dims", [(2 * 32 + 1, 2 * 32 + 1), (77, 300), (400, 1037), (1000, 513)])
@pytest.mark.parametrize("halo", ["full", "zero"])
def test_sep2d_composed_within_fp64_bar(k, dims, halo):
    from paper_2103_08825_b200.core import StencilSpec
    if min(dims) <= 2 * k:
        pytest.skip("grid too small for the composed depth")
    a, b = np.array([0.2, 0.5, 0.3]), np.array([0.15, 0.6, 0.25])
    w = {(dy, dx): float(a[dy + 1] * b[dx + 1]) for dy in (-1, 0, 1) for dx in (-1, 0, 1)}
    for spec in (config_spec("c3a"), StencilSpec("rank1", 2, 1, "box", w)):
        box = seeded_box(dims, 1, seed=sum(dims) + k, halo=halo)
        if halo == "full":                       # halo values far from the interior's
            box[0], box[-1], box[:, 0], box[:, -1] = 3.0, -2.0, 5.0, 0.25
        T = 2 * k + 5                            # two composed launches + a level-by-level tail
        with Plan(spec, dims, k=k, arith="fma") as p:
            p.upload(box)
            t = p.run(T)
            got = p.download()
        assert t.kernel_name.startswith("sep2d") or t.kernel_name in ("fused2d_kernel", "split2d_kernel")
        want = oracle(spec, box, T)
        assert np_oracle.max_rel_error(interior(got, 1), interior(want, 1)) <= FP64_TOL
        mask = np.ones(box.shape, bool)
        mask[1:-1, 1:-1] = False
        assert np.array_equal(got[mask], box[mask])


def test_sep2d_is_the_default_for_rank1_fma_and_not_exact():
    spec = config_spec("c3a")
    with Plan(spec, (300, 400), arith="fma") as p:
        assert p.k in (16, 32)
    with Plan(spec, (300, 400), arith="exact") as p:
        assert p.k == 4
    with Plan(config_spec("c3b"), (300, 400), arith="fma") as p:
        assert p.k == 4


def test_sep2d_nonfinite_propagation():
    spec = config_spec("c3a")
    dims = (200, 300)
    box = seeded_box(dims, 1, seed=3)
    box[100, 150] = np.nan
    box[1, 1] = np.inf
    box[150, 3] = np.inf
    got = sweep(spec, box, 32, arith="fma", k=16)
    want = oracle(spec, box, 32)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isposinf(got), np.isposinf(want))
    fin = np.isfinite(want)
    assert np_oracle.max_rel_error(got[fin], want[fin]) <= FP64_TOL


def test_c3a_full_size_sep2d():
    spec = config_spec("c3a")
    box = seeded_box((16384, 16384), 1, seed=12)
    with Plan(spec, (16384, 16384), arith="fma") as p:
        p.upload(box)
        t = p.run(40)
        got = p.download()
    assert t.kernel_name.startswith("sep2d") or t.k_used >= 16
    assert np_oracle.max_rel_error(got, oracle(spec, box, 40)) <= FP64_TOL


# --- composed 3D star (FMA, k=2 as one 25-point pass + exact physical shell)

@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 9, 7), (9, 40, 70), (37, 33, 130), (20, 17, 131)])
@pytest.mark.parametrize("halo", ["full", "zero"])
def test_composed3d_within_fp64_bar(dims, halo):
    spec = config_spec("c4")
    box = seeded_box(dims, 1, seed=sum(dims), halo=halo)
    T = 9                                    # four composed launches plus a k=1 tail
    with Plan(spec, dims, k=2, arith="fma") as p:
        p.upload(box)
        t = p.run(T)
        got = p.download()
    assert t.kernel_name in ("compose3d_kernel", "fused3d_kernel")
    want = oracle(spec, box, T)
    assert np_oracle.max_rel_error(interior(got, 1), interior(want, 1)) <= FP64_TOL
    mask = np.ones(box.shape, bool)
    mask[1:-1, 1:-1, 1:-1] = False
    assert np.array_equal(got[mask], box[mask])          # halo untouched


def test_composed3d_shell_next_to_dirichlet_values():
    # the interior's outer layer is recomputed level by level: with halo values far
    # from the interior ones, a composition there would be visibly wrong
    spec = config_spec("c4")
    dims = (12, 21, 70)
    box = seeded_box(dims, 1, seed=8)
    box[0], box[-1] = 5.0, -3.0
    box[:, 0], box[:, -1] = 2.0, 7.0
    box[:, :, 0], box[:, :, -1] = -4.0, 9.0
    got = sweep(spec, box, 6, arith="fma", k=2)
    assert np_oracle.max_rel_error(got, oracle(spec, box, 6)) <= FP64_TOL


def test_composed3d_fp32():
    spec = config_spec("c4")
    box32 = seeded_box((30, 70, 130), 1, seed=12).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs, [float(np.float32(w)) for w in ws], 10)
    got = sweep(spec, box32, 10, arith="fma", k=2)
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


def test_c4_full_size_fma_composed():
    spec = config_spec("c4")
    box = seeded_box((512, 512, 512), 1, seed=4)
    with Plan(spec, (512, 512, 512), k=2, arith="fma") as p:
        p.upload(box)
        t = p.run(8)
        got = p.download()
    assert t.kernel_name == "compose3d_kernel" and t.launches == 8   # 4 x (main + shell)
    assert np_oracle.max_rel_error(got, oracle(spec, box, 8)) <= FP64_TOL


def test_c4_full_size_exact():
    spec = config_spec("c4")
    box = seeded_box((512, 512, 512), 1, halo="zero")
    got = sweep(spec, box, 8, arith="exact", k=4)
    assert got.tobytes() == oracle(spec, box, 8).tobytes()


def test_c5_full_size_fp32():
    spec = config_spec("c5")
    box32 = seeded_box((768, 768, 768), 1, seed=2).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs, [float(np.float32(w)) for w in ws], 4)
    got = sweep(spec, box32, 4, arith="fma", k=2)
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


# --- fused 2D kernel (warp-independent y-streaming) -------------------------------

@pytest.mark.parametrize("cfg", ["c3a", "c3b"])
@pytest.mark.parametrize("k", [1, 2, 4, 8])
@pytest.mark.parametrize("dims", [(3, 5), (40, 127), (301, 530)])
def test_fused2d_every_depth_exact(cfg, k, dims):
    spec = config_spec(cfg)
    box = seeded_box(dims, 1, seed=sum(dims) + k)
    T = 11
    got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, T).tobytes()


@pytest.mark.parametrize("k", [1, 4, 8])
def test_fused2d_star_and_halo_zero(k):
    spec = make_stencil_spec("2d5p")
    box = seeded_box((129, 260), 1, seed=k, halo="zero")
    got = sweep(spec, box, 13, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, 13).tobytes()


def test_fused2d_fp32():
    spec = config_spec("c3b")
    box32 = seeded_box((200, 1000), 1, seed=4).astype(np.float32)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(box32.astype(np.float64), 1, offs, [float(np.float32(w)) for w in ws], 24)
    got = sweep(spec, box32, 24, arith="fma", kernel="fused", k=8)
    assert np_oracle.max_rel_error(got, want) <= FP32_TOL


# split2d_kernel: the halo-free (strip, y-range) items of a k = 4 fp64 launch run the lean
# path (plain2d.cuh), the rest the general one, in one launch (launch2d.cu split_plain_2d);
# grids wide and tall enough to have plain strips, ragged last strips, and T not a multiple
# of k (tails on the k = 1 path)
@pytest.mark.parametrize("cfg", ["c3a", "c3b"])
@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("dims", [(64, 400), (700, 1500), (1025, 2049), (23, 260)])
def test_plain2d_split_exact(cfg, k, dims):
    spec = config_spec(cfg)
    box = seeded_box(dims, 1, seed=sum(dims) + k)
    T = 10
    got = sweep(spec, box, T, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, T).tobytes()


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("halo", ["zero", "full"])
def test_plain2d_split_star_and_fma(k, halo):
    box = seeded_box((900, 1300), 1, seed=k, halo=halo)
    spec = make_stencil_spec("2d5p")
    got = sweep(spec, box, 12, arith="exact", kernel="fused", k=k)
    assert got.tobytes() == oracle(spec, box, 12).tobytes()
    for cfg in ("c3a", "c3b"):     # c3a: the separable push (rank-1 weights), c3b: 9 terms
        spec = config_spec(cfg)
        got = sweep(spec, box, 12, arith="fma", kernel="fused", k=k)
        assert np_oracle.max_rel_error(got, oracle(spec, box, 12)) <= FP64_TOL
        r = 1
        mask = np.ones(got.shape, bool)
        mask[r:-r, r:-r] = False
        assert np.array_equal(got[mask], box[mask])          # halo untouched


@pytest.mark.parametrize("cfg", ["c3a", "c3b"])
def test_c3_full_size_fma(cfg):
    spec = config_spec(cfg)
    box = seeded_box((16384, 16384), 1)
    got = sweep(spec, box, 16, arith="fma", k=8)
    want = oracle(spec, box, 16)
    assert np_oracle.max_rel_error(got, want) <= FP64_TOL


@pytest.mark.parametrize("cfg", ["c3a", "c3b"])
def test_c3_full_size_exact(cfg):
    # EXACT mode at the full BASELINE size: bit-identical to the oracle
    spec = config_spec(cfg)
    box = seeded_box((16384, 16384), 1, seed=9, halo="zero")
    got = sweep(spec, box, 9, arith="exact", k=4)
    assert got.tobytes() == oracle(spec, box, 9).tobytes()


def test_c5_full_size_exact():
    spec = config_spec("c5")
    box = seeded_box((768, 768, 768), 1, seed=10)
    got = sweep(spec, box, 3, arith="exact", k=2)
    assert got.tobytes() == oracle(spec, box, 3).tobytes()


# --- seeded fuzz: random stencil class, extents, depth and T, EXACT = bit-identical

FUZZ_CASES = []
_frng = np.random.default_rng(20261020)
for _i in range(36):
    _d = int(_frng.integers(1, 4))
    _cfg = {1: ["c1", "c2", "p:1d3p", "p:1d5p"], 2: ["c3a", "c3b", "p:2d5p", "p:2d9p"],
            3: ["c4", "c5", "p:3d7p", "p:3d27p"]}[_d][int(_frng.integers(0, 4))]
    if _d == 1:
        _dims = (int(_frng.integers(16, 70000)),)
        _k = int(_frng.choice([1, 2, 4, 8, 16]))
    elif _d == 2:
        _dims = (int(_frng.integers(3, 90)), int(_frng.integers(3, 700)))
        _k = int(_frng.choice([1, 2, 4, 8]))
    else:
        _dims = (int(_frng.integers(3, 30)), int(_frng.integers(3, 50)), int(_frng.integers(3, 140)))
        _k = int(_frng.integers(1, 5))
    FUZZ_CASES.append((_cfg, _dims, _k, int(_frng.integers(1, 3 * _k + 3)), str(_frng.choice(["full", "zero"]))))


@pytest.mark.parametrize("cfg,dims,k,T,halo", FUZZ_CASES)
def test_fuzz_exact_bit_identical(cfg, dims, k, T, halo):
    spec = make_stencil_spec(cfg[2:]) if cfg.startswith("p:") else config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=sum(dims) + k + T, halo=halo)
    got = sweep(spec, box, T, arith="exact", k=k)
    assert got.tobytes() == oracle(spec, box, T).tobytes()


@pytest.mark.parametrize("cfg,dims,k,T,halo", FUZZ_CASES[::2])
def test_fuzz_fma_within_bar(cfg, dims, k, T, halo):
    spec = make_stencil_spec(cfg[2:]) if cfg.startswith("p:") else config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=sum(dims) + 2 * k + T, halo=halo)
    got = sweep(spec, box, T, arith="fma", k=k)
    assert np_oracle.max_rel_error(got, oracle(spec, box, T)) <= FP64_TOL


# --- beyond 2^31 elements: 64-bit addressing in every fused path (impulse response)

@pytest.mark.parametrize("cfg,dims,k,dtype", [
    ("c3b", (46000, 47000), 4, np.float32),    # 2.16e9 points: level-by-level 2D
    ("c3a", (46000, 47000), 32, np.float32),   # separable composed 2D
    ("c4", (1290, 1290, 1300), 2, np.float32), # 3D star, level-by-level (fp32)
    ("c4", (1290, 1290, 1300), 2, np.float64), # composed 3D star + shell (17 GB per buffer)
    ("c5", (1290, 1290, 1300), 2, np.float32), # 3D box
    ("c2", ((1 << 31) + 4096,), 32, np.float32),   # composed 1D
])
def test_beyond_2_31_elements_impulse(cfg, dims, k, dtype):
    spec = config_spec(cfg)
    assert int(np.prod(dims)) > (1 << 31)
    box = np.zeros(tuple(n + 2 * spec.r for n in dims), dtype=dtype)
    T = k
    at = tuple(n - spec.r * T - 5 for n in dims)   # past 2^31 linearly, cone clear of the halo
    box[tuple(a + spec.r for a in at)] = 1.0
    got = sweep(spec, box, T, arith="fma", k=k)
    # the impulse response is T-fold convolution of the weights, centred at `at`
    offs, ws = canonical(spec)
    w = 2 * spec.r * T + 1
    small = np.zeros((w + 2 * spec.r * T + 2,) * spec.d)
    c = tuple(sz // 2 for sz in small.shape)
    small[c] = 1.0
    for _ in range(T):
        nxt = np.zeros_like(small)
        for o, wt in zip(offs, ws):
            nxt += wt * np.roll(small, shift=tuple(-x for x in o), axis=tuple(range(spec.d)))
        small = nxt
    win = tuple(slice(a + spec.r - spec.r * T, a + spec.r + spec.r * T + 1) for a in at)
    want = small[tuple(slice(cc - spec.r * T, cc + spec.r * T + 1) for cc in c)]
    np.testing.assert_allclose(got[win], want, rtol=1e-5 if dtype == np.float32 else 1e-12,
                               atol=1e-7 if dtype == np.float32 else 1e-15)
    got[win] = 0.0
    assert not got.any()                    # nothing anywhere else


FRESH_PROCESS_CHECK = r"""
import sys, numpy as np
sys.path[:0] = [%r, %r]
from conftest import seeded_box
from oracle import c_oracle
from paper_2103_08825_b200.core import canonical, config_spec
from paper_2103_08825_b200.plan import sweep
for cfg, dims, k in (("c3a", (4096, 4096), 4), ("c2", (1 << 22,), 8), ("c5", (96, 130, 200), 2)):
    spec = config_spec(cfg)
    box = seeded_box(dims, spec.r, seed=1)
    offs, ws = canonical(spec)
    got = sweep(spec, box, 2 * k + 1, arith="exact", k=k)
    want = c_oracle.sweep(box, spec.r, offs, ws, 2 * k + 1)
    assert got.tobytes() == want.tobytes(), cfg
print("fresh ok")
"""


def test_first_sweep_of_a_fresh_process_exact():
    # regression: schedule tables were uploaded with a pageable cudaMemcpy on the
    # legacy stream while the kernels run on a non-blocking stream -- the first
    # sweep of a process could read a half-written schedule
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = FRESH_PROCESS_CHECK % (repo, os.path.join(repo, "tests"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fresh ok" in r.stdout, r.stderr[-2000:]


def test_async_transfers_pipelined_two_plans():
    # sb_upload_async / sb_launch / sb_download_async on two plans and two
    # streams (the bench's pipelined e2e): same bytes as the synchronous calls
    import torch
    spec = config_spec("c2")
    n = 200003
    boxes = [seeded_box((n,), 2, seed=s) for s in (1, 2, 3, 4)]
    want = [sweep(spec, b, 40, arith="fma") for b in boxes]
    plans = [Plan(spec, (n,), arith="fma") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    ins = [torch.from_numpy(b).pin_memory() for b in boxes]
    outs = [torch.empty_like(i).pin_memory() for i in ins]
    try:
        for p, s in zip(plans, streams):
            p.set_stream(s.cuda_stream)
        for i in range(4):
            p = plans[i % 2]
            p.upload_async(ins[i].numpy())
            p.launch(40)
            p.download_async(outs[i].numpy())
        for p in plans:
            p.synchronize()
        for o, w in zip(outs, want):
            assert o.numpy().tobytes() == w.tobytes()
    finally:
        for p in plans:
            p.close()
