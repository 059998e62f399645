"""Stencil specifications: the host-side mirror of ``stencilbench.core``.

The product accepts either a reference ``stencilbench.core.StencilSpec``
(duck-typed: ``.d .r .shape .weights``) or :class:`StencilSpec` defined here,
which restates the reference's validation rules
(``stencilbench/core.py:54-106``), its six presets (``core.py:109-148``) and
``flops_per_point`` (``core.py:161-163``) so callers that never import the
reference get identical semantics and error types.

It also defines the five BASELINE.json workloads (C1-C5) with their exact
weights, including the seeded random-weight variants whose seeds are recorded
here (``WEIGHT_SEEDS``) and in DESIGN.md.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from fractions import Fraction
from typing import Mapping

import numpy as np

Offset = tuple[int, ...]


class SpecError(ValueError):
    """Invalid stencil specification or preset name (``core.py:38-39``)."""


class GridError(ValueError):
    """Invalid grid geometry, layout, or buffer (``core.py:42-43``)."""


@dataclass(frozen=True, eq=False)
class StencilSpec:
    """Constant-coefficient stencil (mirror of ``core.py:54-106``).

    ``weights`` maps each length-``d`` integer offset to its fp64 weight;
    ``shape`` is ``"star"`` or ``"box"``.  Immutable, compares by identity.
    """

    name: str
    d: int
    r: int
    shape: str
    weights: Mapping[Offset, float]

    def __post_init__(self):
        validate(self)

    @property
    def offsets(self) -> tuple[Offset, ...]:
        """Canonical (lexicographic) order -- the accumulation order (core.py:96-103)."""
        return tuple(sorted(self.weights))

    def weight(self, off: Offset) -> float:
        return self.weights[off]


def validate(spec) -> None:
    """The reference's spec checks (``core.py:71-94``), on any duck-typed spec."""
    d, r, shape, weights = spec.d, spec.r, spec.shape, spec.weights
    if d not in (1, 2, 3):
        raise SpecError(f"dimension must be 1, 2 or 3, got {d}")
    if r < 1:
        raise SpecError(f"order must be positive, got {r}")
    offs = set(weights)
    if (0,) * d not in offs:
        raise SpecError("zero offset missing from weight table")
    for off in offs:
        if len(off) != d or max(abs(c) for c in off) > r:
            raise SpecError(f"offset {off} outside radius {r}")
    if shape == "star":
        expected = 2 * d * r + 1
        if any(sum(c != 0 for c in off) > 1 for off in offs):
            raise SpecError("star stencil has a non-axis-aligned offset")
    elif shape == "box":
        expected = (2 * r + 1) ** d
    else:
        raise SpecError(f"shape must be 'star' or 'box', got {shape!r}")
    if len(offs) != expected:
        raise SpecError(f"{shape} stencil of d={d} r={r} needs {expected} "
                        f"weights, got {len(offs)}")


def canonical(spec) -> tuple[list[Offset], list[float]]:
    """(offsets, weights) in canonical order for any duck-typed spec."""
    offs = sorted(spec.weights)
    return offs, [float(spec.weights[o]) for o in offs]


def flops_per_point(spec) -> int:
    """``|W|`` multiplies plus ``|W|-1`` adds (core.py:161-163)."""
    return 2 * len(spec.weights) - 1


# --- presets (core.py:109-148) ----------------------------------------------

def _star_weights(d: int, r: int, off_weight: Fraction) -> dict[Offset, float]:
    weights: dict[Offset, float] = {}
    count = 0
    for axis in range(d):
        for dist in range(1, r + 1):
            for sign in (-1, 1):
                off = [0] * d
                off[axis] = sign * dist
                weights[tuple(off)] = float(off_weight)
                count += 1
    weights[(0,) * d] = float(1 - count * off_weight)
    return weights


def _box_weights(d: int) -> dict[Offset, float]:
    kernel = {-1: Fraction(1, 4), 0: Fraction(1, 2), 1: Fraction(1, 4)}
    weights: dict[Offset, float] = {}
    for off in itertools.product((-1, 0, 1), repeat=d):
        w = Fraction(1)
        for c in off:
            w *= kernel[c]
        weights[off] = float(w)
    return weights


_PRESETS = {
    "1d3p": StencilSpec("1d3p", 1, 1, "star", _star_weights(1, 1, Fraction(1, 4))),
    "1d5p": StencilSpec("1d5p", 1, 2, "star", _star_weights(1, 2, Fraction(1, 8))),
    "2d5p": StencilSpec("2d5p", 2, 1, "star", _star_weights(2, 1, Fraction(1, 8))),
    "2d9p": StencilSpec("2d9p", 2, 1, "box", _box_weights(2)),
    "3d7p": StencilSpec("3d7p", 3, 1, "star", _star_weights(3, 1, Fraction(1, 8))),
    "3d27p": StencilSpec("3d27p", 3, 1, "box", _box_weights(3)),
}
PRESET_NAMES = tuple(_PRESETS)


def make_stencil_spec(name: str) -> StencilSpec:
    """One of the six reference presets by name (core.py:151-158)."""
    try:
        return _PRESETS[name.lower()]
    except KeyError:
        raise SpecError(f"unknown stencil preset {name!r}; choose from "
                        f"{', '.join(_PRESETS)}") from None


# --- BASELINE.json workloads ------------------------------------------------

#: Seeds of the "seeded random weights" variants (BASELINE.json leaves them
#: open): U[0,1) from default_rng(seed) assigned to canonical offsets in order,
#: then normalised as w / w.sum() in float64.
WEIGHT_SEEDS = {"2d9p_rand": 20210316, "3d27p_rand": 20210317}


def random_box_weights(d: int, r: int, seed: int) -> dict[Offset, float]:
    offs = sorted(itertools.product(range(-r, r + 1), repeat=d))
    w = np.random.default_rng(seed).random(len(offs))
    w = w / w.sum()
    return {o: float(v) for o, v in zip(offs, w)}


def weights_from_list(d: int, r: int, shape: str, values) -> dict[Offset, float]:
    """Assign ``values`` to the canonical offsets of a star/box pattern."""
    if shape == "box":
        offs = sorted(itertools.product(range(-r, r + 1), repeat=d))
    else:
        offs = sorted(set(_star_weights(d, r, Fraction(0))))
    if len(offs) != len(values):
        raise SpecError(f"{shape} d={d} r={r} needs {len(offs)} weights")
    return {o: float(v) for o, v in zip(offs, values)}


def _config_specs() -> dict[str, StencilSpec]:
    c3a = {o: 1.0 / 9.0 for o in itertools.product((-1, 0, 1), repeat=2)}
    c4 = {o: 0.1 for o in _star_weights(3, 1, Fraction(1, 10))}
    c4[(0, 0, 0)] = 0.4
    return {
        "c1": StencilSpec("c1_1d3p", 1, 1, "star",
                          weights_from_list(1, 1, "star", (0.25, 0.5, 0.25))),
        "c2": StencilSpec("c2_1d5p", 1, 2, "star",
                          weights_from_list(1, 2, "star",
                                            (0.0625, 0.25, 0.375, 0.25, 0.0625))),
        "c3a": StencilSpec("c3a_2d9p_avg", 2, 1, "box", c3a),
        "c3b": StencilSpec("c3b_2d9p_rand", 2, 1, "box",
                           random_box_weights(2, 1, WEIGHT_SEEDS["2d9p_rand"])),
        "c4": StencilSpec("c4_3d7p", 3, 1, "star", c4),
        "c5": StencilSpec("c5_3d27p", 3, 1, "box",
                          random_box_weights(3, 1, WEIGHT_SEEDS["3d27p_rand"])),
    }


CONFIG_SPECS = _config_specs()

#: BASELINE.json configs: spec key, interior dims (g=1), steps, dtypes.
CONFIGS = {
    "c1": dict(spec="c1", dims=(1 << 20,), steps=64, dtypes=("f64",)),
    "c2": dict(spec="c2", dims=(1 << 26,), steps=1000, dtypes=("f64",)),
    "c3a": dict(spec="c3a", dims=(16384, 16384), steps=500, dtypes=("f64",)),
    "c3b": dict(spec="c3b", dims=(16384, 16384), steps=500, dtypes=("f64",)),
    "c4": dict(spec="c4", dims=(512, 512, 512), steps=200, dtypes=("f64",)),
    "c5": dict(spec="c5", dims=(768, 768, 768), steps=100, dtypes=("f64", "f32")),
}


def config_spec(key: str) -> StencilSpec:
    try:
        return CONFIG_SPECS[key]
    except KeyError:
        raise SpecError(f"unknown config {key!r}; choose from {', '.join(CONFIG_SPECS)}") from None
