"""Benchmark harness for the b200 methods: the reference's ``run_benchmark``
contract (``stencilbench/harness.py:40-83`` BenchConfig / BenchResult,
``:221-240`` run_benchmark, ``:256-258`` verify_tolerance, ``:261-270``
emit_csv) with the multi-step dispatch branch SURVEY §8(f)1 asks for.

The reference's ``_execute`` (harness.py:176-211) steps a method one
``METHODS[...][1]`` call per time step (a registered ``"b200"`` works there
unchanged, one device round trip per step).  Here the ``"b200*"`` methods go
through :func:`kernels.b200_sweep`: the grid is seeded exactly like
``seed_grid`` (harness.py:139-146: PCG64 from the seed, uniform [0, 1)
interior, halo 0), converted to the method's layout on the device for the
permuted layouts (timed as ``layout_seconds``, like the reference), and
advanced T steps with k fused per HBM round trip.  GFlop/s comes from the
counters (point updates x flops per point, harness.py:228).

``BenchConfig`` also accepts ``weights`` (a StencilSpec or the name of a
BASELINE config), lifting the preset-only restriction of harness.py:56-57.
Verification needs the caller's oracle (``run_benchmark(cfg, oracle=...)``):
the product path never runs a CPU stencil.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .core import StencilSpec, config_spec, flops_per_point, make_stencil_spec
from .grid import Layout, alloc_grid
from .kernels import b200_sweep

CSV_HEADER = ("stencil,method,vl,jam_k,size,steps,block,tile_height,threads,"
              "seconds,layout_seconds,gflops,max_rel_err,loads,stores,reorg_ops")

#: b200 method -> storage layout of the grid it sweeps (kernels.register)
B200_METHODS = {"b200": Layout.NATURAL, "b200_transpose": Layout.BLOCK_TRANSPOSE, "b200_dlt": Layout.DLT}


class UsageError(ValueError):
    """Invalid or conflicting benchmark configuration (harness.py:37-38)."""


@dataclass
class Counters:
    """Shape of ``stencilbench.kernels.Counters`` (kernels.py:43-69)."""

    vec_loads: int = 0
    vec_stores: int = 0
    scalar_loads: int = 0
    scalar_stores: int = 0
    reorg_ops: int = 0
    point_updates: int = 0
    vs_loads: int = 0
    vs_stores: int = 0

    def element_loads(self, vl: int) -> int:
        return self.vec_loads * vl + self.scalar_loads

    def element_stores(self, vl: int) -> int:
        return self.vec_stores * vl + self.scalar_stores


@dataclass
class BenchConfig:
    stencil: str
    dims: tuple[int, ...]
    steps: int
    method: str = "b200"
    vl: int = 4
    jam_k: int = 0                 # fused steps per HBM round trip (the reference's jam
                                   # factor); 0 = the plan's default depth for the stencil class
    block: tuple | None = None     # host tiling (harness.py:47-48): the b200 methods tile on
    tile_height: int | None = None  # the device, so these must stay None (UsageError)
    workers: int = 1
    seed: int = 12345
    csv_path: str | None = None
    verify: bool = False
    weights: object = None         # StencilSpec | BASELINE config key | None (preset `stencil`)

    def spec(self) -> StencilSpec:
        if isinstance(self.weights, StencilSpec):
            return self.weights
        if isinstance(self.weights, str):
            return config_spec(self.weights)
        return make_stencil_spec(self.stencil)


@dataclass
class BenchResult:
    config: BenchConfig
    seconds: float
    layout_seconds: float
    gflops: float
    counters: Counters
    max_rel_err: float | None = None

    def csv_row(self) -> str:
        # field order of harness.py:62-83 (block/tile_height empty: the GPU tiles internally)
        cfg = self.config
        err = "" if self.max_rel_err is None else f"{self.max_rel_err:.17g}"
        return ",".join([
            cfg.stencil, cfg.method, str(cfg.vl), str(cfg.jam_k), "x".join(map(str, cfg.dims)),
            str(cfg.steps), "", "", str(cfg.workers), f"{self.seconds:.17g}", f"{self.layout_seconds:.17g}",
            f"{self.gflops:.17g}", err, str(self.counters.element_loads(cfg.vl)),
            str(self.counters.element_stores(cfg.vl)), str(self.counters.reorg_ops),
        ])


def validate_config(cfg: BenchConfig) -> None:
    """Reject invalid combinations with a message naming the conflict (harness.py:86-128)."""
    spec = cfg.spec()
    if cfg.method not in B200_METHODS:
        raise UsageError(f"--method {cfg.method}: unknown; choose from {', '.join(B200_METHODS)}")
    if len(cfg.dims) != spec.d:
        raise UsageError(f"--size: {cfg.stencil} needs {spec.d} extents, got {len(cfg.dims)}")
    if any(int(n) <= 0 for n in cfg.dims):
        raise UsageError(f"--size: extents must be positive, got {cfg.dims}")
    if cfg.steps < 1:
        raise UsageError(f"--steps {cfg.steps}: must be >= 1")
    if cfg.vl not in (4, 8):
        raise UsageError(f"--vl {cfg.vl}: supported vector lengths are 4 and 8")
    if cfg.jam_k < 0:
        raise UsageError(f"--jam-k {cfg.jam_k}: must be >= 0 (0 = the plan's default depth)")
    if cfg.block is not None or cfg.tile_height is not None:
        raise UsageError("--block/--tile-height: the b200 methods tile on the device; for host "
                         "tessellate tiling register them in the reference's METHODS and use run_tiled")
    if cfg.workers < 1:
        raise UsageError(f"--threads {cfg.workers}: must be >= 1")


def seed_grid(cfg: BenchConfig, spec: StencilSpec):
    """harness.py:139-146: PCG64 interior from the seed, halo 0, padded for the layout."""
    layout = B200_METHODS[cfg.method]
    grid = alloc_grid(spec, cfg.dims, Layout.NATURAL, cfg.vl,
                      pad_for=layout if layout is not Layout.NATURAL else None)
    grid.set_interior(np.random.default_rng(cfg.seed).random(tuple(cfg.dims)))
    return grid


def _execute(cfg: BenchConfig, spec: StencilSpec, counters: Counters, arith: str = "exact"):
    from . import transpose as tr
    layout = B200_METHODS[cfg.method]
    grid = seed_grid(cfg, spec)
    t_start = time.perf_counter()
    layout_s = 0.0
    if layout is not Layout.NATURAL:
        t0 = time.perf_counter()
        (tr.to_block_transpose if layout is Layout.BLOCK_TRANSPOSE else tr.to_dlt)(grid, cfg.vl)
        layout_s += time.perf_counter() - t0
    b200_sweep(grid, spec, cfg.jam_k, cfg.steps, counters, arith=arith)
    if layout is not Layout.NATURAL:
        t0 = time.perf_counter()
        (tr.from_block_transpose if layout is Layout.BLOCK_TRANSPOSE else tr.from_dlt)(grid)
        layout_s += time.perf_counter() - t0
    return grid.natural_interior(), time.perf_counter() - t_start, layout_s


def max_rel_error(got: np.ndarray, want: np.ndarray) -> float:
    denom = np.maximum(np.abs(want), np.finfo(np.float64).tiny)
    return float(np.max(np.abs(got - want) / denom))


def run_benchmark(cfg: BenchConfig, oracle=None, arith: str = "exact") -> BenchResult:
    """One configuration: timing, counters, and with ``cfg.verify`` the max
    relative error against ``oracle(cfg, spec) -> natural interior`` (the
    caller's reference, e.g. ``stencilbench.harness.run_oracle``).
    ``arith`` 'exact' (default, bit-identical) or 'fma'."""
    validate_config(cfg)
    spec = cfg.spec()
    if cfg.verify and oracle is None:
        raise UsageError("--verify needs the reference oracle (run_benchmark(cfg, oracle=...))")
    warm = BenchConfig(cfg.stencil, (1,) * (spec.d - 1) + (max(16, 8 * spec.r),), 1, cfg.method,
                       vl=cfg.vl, jam_k=1, seed=cfg.seed, weights=cfg.weights)
    _execute(warm, spec, Counters(), arith)               # harness.py:165-172
    counters = Counters()
    result, total_s, layout_s = _execute(cfg, spec, counters, arith)
    gflops = counters.point_updates * flops_per_point(spec) / max(total_s, 1e-12) / 1e9
    err = max_rel_error(result, oracle(cfg, spec)) if cfg.verify else None
    return BenchResult(cfg, total_s, layout_s, gflops, counters, err)


def verify_tolerance(steps: int) -> float:
    """harness.py:256-258: 1e-13 relative per time step."""
    return 1e-13 * max(steps, 1)


def emit_csv(results, path: str) -> None:
    try:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(CSV_HEADER + "\n")
            for res in results:
                fh.write(res.csv_row() + "\n")
    except OSError as exc:
        raise UsageError(f"cannot write CSV to {path!r}: {exc}") from exc


__all__ = ["BenchConfig", "BenchResult", "Counters", "UsageError", "run_benchmark", "validate_config",
           "seed_grid", "emit_csv", "verify_tolerance", "max_rel_error", "CSV_HEADER", "B200_METHODS"]
