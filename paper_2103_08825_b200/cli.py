"""Command-line front end of the b200 methods (mirrors stencilbench/cli.py).

    python -m paper_2103_08825_b200 run    --stencil 3d27p --size 256 --steps 100 --method b200
    python -m paper_2103_08825_b200 verify --stencil 2d9p --size 512 --steps 50 --method b200_transpose
    python -m paper_2103_08825_b200 plan   --stencil 3d7p --size 512 [--weights c4] [--k 2]

Same subcommands, flags, defaults and exit codes as the reference CLI
(cli.py:59-170): ``run`` times a configuration and prints the summary (and
the CSV row with ``--csv``); ``verify`` exits 1 when the max relative error
exceeds 1e-13 per step (cli.py:120-127); every configuration error exits 2
with ``error: <message>`` (cli.py:167-170).  Differences, all additive:

* ``--method`` choices are the b200 methods (``b200`` NATURAL,
  ``b200_transpose`` BLOCK_TRANSPOSE, ``b200_dlt`` DLT);
* ``--weights`` takes a BASELINE config key (c1 .. c5) or a comma list of
  weights in canonical offset order, lifting the preset-only restriction;
* ``--jam-k`` is the device fusion depth (default 0: the plan's own);
  ``--arith fma`` runs the FMA kernels (the default ``exact`` is bit-identical
  to the reference);
* ``--block`` / ``--tile-height`` are rejected: the device tiles internally
  (register the methods in the reference's METHODS to drive ``run_tiled``);
* ``verify`` compares against the reference's own ``run_oracle``
  (harness.py:149-157), so it needs the reference package importable;
* ``plan`` prints the device plan (kernel, fusion depth, roofline per depth)
  instead of the SIMD shuffle plan, which has no GPU counterpart.
"""

from __future__ import annotations

import argparse
import sys

from .core import GridError, SpecError, StencilSpec, config_spec, flops_per_point, make_stencil_spec, \
    weights_from_list, PRESET_NAMES
from .harness import B200_METHODS, BenchConfig, UsageError, emit_csv, run_benchmark, verify_tolerance


def _parse_extents(text: str, what: str) -> tuple[int, ...]:
    try:
        parts = tuple(int(p) for p in text.lower().replace(",", "x").split("x"))
    except ValueError:
        raise UsageError(f"{what} {text!r}: expected N or NxM[xK]") from None
    if not parts or any(p <= 0 for p in parts):
        raise UsageError(f"{what} {text!r}: extents must be positive")
    return parts


def _spec(stencil: str, weights: str | None):
    base = make_stencil_spec(stencil)
    if not weights:
        return base, None
    if weights.lower() in ("c1", "c2", "c3a", "c3b", "c4", "c5"):
        spec = config_spec(weights.lower())
        if (spec.d, spec.r, spec.shape) != (base.d, base.r, base.shape):
            raise UsageError(f"--weights {weights}: config is a d={spec.d} r={spec.r} {spec.shape} stencil, "
                             f"--stencil {stencil} is d={base.d} r={base.r} {base.shape}")
        return spec, spec
    try:
        values = [float(v) for v in weights.split(",")]
    except ValueError:
        raise UsageError(f"--weights {weights!r}: expected a config key or comma-separated numbers") from None
    spec = StencilSpec(f"{stencil}_custom", base.d, base.r, base.shape,
                       weights_from_list(base.d, base.r, base.shape, values))
    return spec, spec


def _add_common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--stencil", required=True, choices=PRESET_NAMES, help="stencil preset (shape)")
    p.add_argument("--size", required=True, help="interior extents: N (broadcast per dimension) or NxM[xK]")
    p.add_argument("--steps", type=int, default=16, help="time steps (default 16)")
    p.add_argument("--method", required=True, choices=list(B200_METHODS), help="b200 method (grid layout)")
    p.add_argument("--weights", help="BASELINE config key (c1..c5) or comma list of weights, canonical order")
    p.add_argument("--jam-k", type=int, default=0, dest="jam_k",
                   help="fused steps per HBM round trip (default 0: the plan's depth)")
    p.add_argument("--arith", default="exact", choices=["exact", "fma"],
                   help="exact (bit-identical to the reference, default) or fma")
    p.add_argument("--vl", type=int, default=4, help="vector lanes of the storage layout, 4 or 8 (default 4)")
    p.add_argument("--block", help="(rejected: the device tiles internally)")
    p.add_argument("--tile-height", type=int, dest="tile_height", help="(rejected)")
    p.add_argument("--threads", type=int, default=1, help="host workers (accepted for compatibility)")
    p.add_argument("--seed", type=int, default=12345, help="grid seed (default 12345)")
    p.add_argument("--csv", dest="csv", help="CSV output path")


def parse_cli(argv) -> argparse.Namespace:
    parser = argparse.ArgumentParser(prog="python -m paper_2103_08825_b200",
                                     description="B200 multistep stencil sweep: benchmark, verify, plan.")
    sub = parser.add_subparsers(dest="command", required=True)
    run_p = sub.add_parser("run", help="time a configuration")
    _add_common(run_p)
    run_p.add_argument("--verify", action="store_true", help="also compare against the reference oracle")
    ver_p = sub.add_parser("verify", help="compare against the reference oracle")
    _add_common(ver_p)
    plan_p = sub.add_parser("plan", help="print the device plan of a configuration")
    plan_p.add_argument("--stencil", required=True, choices=PRESET_NAMES)
    plan_p.add_argument("--size", required=True)
    plan_p.add_argument("--weights")
    plan_p.add_argument("--k", type=int, default=0, help="fusion depth (0: the plan's)")
    plan_p.add_argument("--arith", default="fma", choices=["exact", "fma"])
    plan_p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    args = parser.parse_args(argv)
    spec, custom = _spec(args.stencil, args.weights)
    dims = _parse_extents(args.size, "--size")
    if len(dims) == 1 and spec.d > 1:
        dims = dims * spec.d
    args.spec, args.dims = spec, dims
    if args.command in ("run", "verify"):
        if args.block is not None or args.tile_height is not None:
            raise UsageError("--block/--tile-height: the b200 methods tile on the device; register them in the "
                             "reference's METHODS (kernels.register) to drive its tessellate runner")
        args.cfg = BenchConfig(stencil=args.stencil, dims=dims, steps=args.steps, method=args.method, vl=args.vl,
                               jam_k=args.jam_k, workers=args.threads, seed=args.seed, csv_path=args.csv,
                               verify=(args.command == "verify" or getattr(args, "verify", False)),
                               weights=custom)
    return args


def _reference_oracle():
    """The reference's own run_oracle (harness.py:149-157) for this config."""
    try:
        from stencilbench import harness as ref_harness
        from stencilbench.core import StencilSpec as RefSpec
    except ImportError:
        raise UsageError("verify needs the reference package (stencilbench) importable: it is the oracle") from None

    def oracle(cfg, spec):
        ref_spec = RefSpec(spec.name, spec.d, spec.r, spec.shape, dict(spec.weights))
        rcfg = ref_harness.BenchConfig(cfg.stencil, tuple(cfg.dims), cfg.steps, "scalar", vl=cfg.vl, seed=cfg.seed)
        rcfg.spec = lambda: ref_spec   # custom weights: the reference's BenchConfig only builds presets
        return ref_harness.run_oracle(rcfg)
    return oracle


def _cmd_run(args) -> int:
    cfg = args.cfg
    res = run_benchmark(cfg, oracle=_reference_oracle() if cfg.verify else None, arith=args.arith)
    print(f"{cfg.stencil} {cfg.method} vl={cfg.vl} jam_k={cfg.jam_k} arith={args.arith} "
          f"size={'x'.join(map(str, cfg.dims))} steps={cfg.steps} threads={cfg.workers}")
    print(f"  wall {res.seconds:.6f} s (layout {res.layout_seconds:.6f} s)  {res.gflops:.3f} GFlop/s  "
          f"{res.counters.point_updates / max(res.seconds, 1e-12) / 1e9:.3f} GStencil/s")
    c = res.counters
    print(f"  element loads {c.element_loads(cfg.vl)}  stores {c.element_stores(cfg.vl)}  reorg ops {c.reorg_ops}")
    if res.max_rel_err is not None:
        print(f"  max rel err vs oracle: {res.max_rel_err:.3e}")
    if cfg.csv_path:
        emit_csv([res], cfg.csv_path)
        print(f"  csv -> {cfg.csv_path}")
    return 0


def _cmd_verify(args) -> int:
    cfg = args.cfg
    res = run_benchmark(cfg, oracle=_reference_oracle(), arith=args.arith)
    tol = verify_tolerance(cfg.steps)
    err = res.max_rel_err
    status = "PASS" if err <= tol else "FAIL"
    print(f"{status} {cfg.stencil} {cfg.method} jam_k={cfg.jam_k} arith={args.arith}: max rel err {err:.3e} "
          f"(tolerance {tol:.3e} over {cfg.steps} steps)")
    if cfg.csv_path:
        emit_csv([res], cfg.csv_path)
    return 0 if err <= tol else 1


def _cmd_plan(args) -> int:
    import json
    import os
    spec, dims = args.spec, args.dims
    if len(dims) != spec.d:
        raise UsageError(f"--size: {args.stencil} needs {spec.d} extents, got {len(dims)}")
    es = 8 if args.dtype == "f64" else 4
    peaks = {"hbm_gbs": 6543.7, "fp64_tflops": 37.1, "fp32_tflops": 74.1}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for path, keys in ((os.path.join(root, "MEASURED_PEAKS.json"), ("hbm_gbs",)),
                       (os.path.join(root, "profiles", "fp_peak.json"), ("fp64_tflops", "fp32_tflops"))):
        if os.path.exists(path):
            with open(path) as fh:
                m = json.load(fh)
            peaks.update({k: m[k] for k in keys if m.get(k)})
    F = flops_per_point(spec)
    P = peaks["fp64_tflops" if es == 8 else "fp32_tflops"] * 1e12
    print(f"{spec.name}: d={spec.d} r={spec.r} {spec.shape}, |W|={len(spec.weights)}, F={F} flops/update, "
          f"interior {'x'.join(map(str, dims))}, {args.dtype}, {args.arith}")
    for off in spec.offsets:
        print(f"  w{off} = {spec.weights[off]!r}")
    print("roofline R(k) = min(BW*k/(2s), P/F) GStencil/s per GPU:")
    for k in (1, 2, 3, 4, 8, 16, 32):
        hb = peaks["hbm_gbs"] * 1e9 * k / (2 * es) / 1e9
        print(f"  k={k:2d}: HBM {hb:8.0f}  FP {P / F / 1e9:8.0f}  -> {min(hb, P / F / 1e9):8.0f}")
    try:
        from . import _abi
        ndev = _abi.device_count()
    except Exception as exc:   # library missing: report, do not fail the plan dump
        print(f"device plan: unavailable ({exc})")
        return 0
    if ndev == 0:
        print("device plan: no CUDA device visible")
        return 0
    from .plan import Plan
    with Plan(spec, dims, dtype=args.dtype, arith=args.arith, k=args.k) as p:
        print(f"device plan: fused depth k={p.k}, host box {p.shape}")
    return 0


def main(argv=None) -> int:
    try:
        args = parse_cli(argv if argv is not None else sys.argv[1:])
        if args.command == "run":
            return _cmd_run(args)
        if args.command == "verify":
            return _cmd_verify(args)
        return _cmd_plan(args)
    except (UsageError, SpecError, GridError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
