"""The vector-set step on the device (vectorset.vs_step) against the
reference's own vs_step (kernels.py:478-511) and its tests
(test_kernels.py:204-243): constant and ramp fixed points, the oracle block,
missing-dependency errors, and bit-identity on random blocks for 1D/2D/3D,
star and box, r = 1 and 2, vl = 4 and 8 (cross-dependency bands for d > 1)."""

import itertools

import numpy as np
import pytest

sb = pytest.importorskip("stencilbench", reason="reference package not installed (baseline/_ref)")

from stencilbench.core import VectorSet, make_stencil_spec  # noqa: E402
from stencilbench.kernels import Band  # noqa: E402
from stencilbench.kernels import vs_step as ref_vs_step  # noqa: E402
from stencilbench.simd import VectorValue  # noqa: E402

from paper_2103_08825_b200.vectorset import vs_step  # noqa: E402

SPEC1 = make_stencil_spec("1d3p")


def test_missing_dependency_errors_before_the_device():
    # both packages' GridError are ValueError subclasses (core.py:42-43)
    const = VectorSet(tuple(VectorValue((0.0,) * 4) for _ in range(4)))
    with pytest.raises(ValueError, match="dependency"):
        vs_step(const, (), (), None, SPEC1)
    dep = (VectorValue((0.0,) * 4),)
    with pytest.raises(ValueError, match="outer offset"):
        vs_step(const, dep, dep, None, make_stencil_spec("2d5p"))


def _vec(rng, vl):
    return VectorValue(rng.random(vl).tolist())


def _case(spec, vl, seed):
    rng = np.random.default_rng(seed)
    r, d = spec.r, spec.d
    vs = VectorSet(tuple(_vec(rng, vl) for _ in range(vl)))
    left = tuple(_vec(rng, vl) for _ in range(r))
    right = tuple(_vec(rng, vl) for _ in range(r))
    cross = None
    if d > 1:
        cross = {}
        for key in itertools.product(range(-r, r + 1), repeat=d - 1):
            if key == (0,) * (d - 1):
                continue
            cross[key] = Band(tuple(_vec(rng, vl) for _ in range(vl)), tuple(_vec(rng, vl) for _ in range(r)),
                              tuple(_vec(rng, vl) for _ in range(r)))
    return vs, left, right, cross


@pytest.mark.gpu
def test_constant_and_ramp_fixed_points():
    vl = 4
    const = VectorSet(tuple(VectorValue((5.0,) * vl) for _ in range(vl)))
    dep = (VectorValue((5.0,) * vl),)
    assert vs_step(const, dep, dep, None, SPEC1).rows == const.rows
    nat = np.arange(16.0)
    rows = tuple(VectorValue(nat[l * vl + j] for l in range(vl)) for j in range(vl))
    left = (VectorValue([-1.0, 3.0, 7.0, 11.0]),)
    right = (VectorValue([4.0, 8.0, 12.0, 16.0]),)
    assert vs_step(VectorSet(rows), left, right, None, SPEC1).rows == rows


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["1d3p", "1d5p", "2d5p", "2d9p", "3d7p", "3d27p"])
@pytest.mark.parametrize("vl", [4, 8])
@pytest.mark.parametrize("seed", [0, 1])
def test_bit_identical_to_reference_vs_step(preset, vl, seed):
    spec = make_stencil_spec(preset)
    vs, left, right, cross = _case(spec, vl, seed + vl)
    want = ref_vs_step(vs, left, right, cross, spec)
    got = vs_step(vs, left, right, cross, spec)
    assert isinstance(got, VectorSet) and got.base == vs.base
    assert got.rows == want.rows
