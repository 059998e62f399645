"""Measure every BASELINE.json config (C1-C5) at full size and full T on one GPU.

Device-resident sweeps (CUDA events inside sb_run), one warm-up sweep, the
k sweep per config, roofline R(k) = min(BW*k/(2s), P/F) with BW and P the
measured peaks (MEASURED_PEAKS.json, profiles/fp_peak.json), and a bounded
CPU-oracle sample (oracle/oracle.c, all host threads) on the same grid.

    python tools/measure_configs.py [--out profiles/r01_configs.json] [--no-cpu]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2103_08825_b200.core import CONFIGS, config_spec  # noqa: E402
from paper_2103_08825_b200.plan import Plan  # noqa: E402

KS = {1: (1, 2, 4, 8, 16, 32, 64), 2: (1, 2, 4, 8, 16, 32), 3: (1, 2, 3, 4)}


def peaks():
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
        hbm = json.load(fh)["hbm_gbs"]
    with open(os.path.join(REPO, "profiles", "fp_peak.json")) as fh:
        fp = json.load(fh)
    return hbm, fp["fp64_tflops"], fp["fp32_tflops"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    hbm, p64, p32 = peaks()
    results = {}
    for key, cfg in CONFIGS.items():
        if args.only and key not in args.only.split(","):
            continue
        spec = config_spec(cfg["spec"])
        dims, T = cfg["dims"], cfg["steps"]
        n = int(np.prod(dims))
        F = 2 * len(spec.weights) - 1
        box = np.random.default_rng(12345).random(tuple(d + 2 * spec.r for d in dims))
        for dt in cfg["dtypes"]:
            s = 8 if dt == "f64" else 4
            P = (p64 if dt == "f64" else p32) * 1e12
            b = box if dt == "f64" else box.astype(np.float32)
            entry = {"dims": list(dims), "T": T, "stencil": spec.name, "flops_per_update": F, "k": {}}
            for k in KS[spec.d]:
                try:
                    plan = Plan(spec, dims, k=k, arith="fma", dtype=dt)
                except ValueError:          # depth not offered for this stencil
                    continue
                with plan as p:
                    for _ in range(2):      # eager (first-use setup), then graph capture
                        p.upload(b)
                        p.run(T)
                    p.upload(b)
                    t = p.run(T)            # CUDA-graph replay (sb200.cu run_graphed)
                g = n * T / (t.device_ms * 1e-3) / 1e9
                roof = min(hbm * 1e9 * k / (2 * s), P / F) / 1e9
                # executed FMAs per update of the kernel that ran (the composed paths do
                # less arithmetic than the step-by-step algorithm BASELINE's F counts)
                if spec.d == 1 and k >= 16:                          # compose1d (FMA)
                    fma_u = (2 * spec.r * k + 1) / k
                elif spec.d == 2 and k >= 16:                        # separable composed passes
                    fma_u = 2 * (2 * k + 1) / k
                elif spec.d == 3 and spec.shape == "star" and k == 2 and dt == "f64":   # compose3d
                    fma_u = 12.5
                else:
                    fma_u = len(spec.weights)
                roof_x = min(hbm * 1e9 * k / (2 * s), P / 2 / fma_u) / 1e9
                entry["k"][str(k)] = {"gstencil": round(g, 1), "ms": round(t.device_ms, 2),
                                      "roofline_gstencil": round(roof, 1), "frac": round(g / roof, 3),
                                      "fma_per_update_executed": round(fma_u, 3),
                                      "roofline_executed_gstencil": round(roof_x, 1),
                                      "frac_executed": round(g / roof_x, 3),
                                      "binding": "hbm" if hbm * 1e9 * k / (2 * s) < P / F else dt,
                                      "kernel": t.kernel_name, "launches": t.launches}
            best = max(entry["k"].items(), key=lambda kv: kv[1]["gstencil"])
            entry["best_k"] = int(best[0])
            entry["best_gstencil"] = best[1]["gstencil"]
            entry["best_frac"] = best[1]["frac"]
            if not args.no_cpu:
                # bench.py's cpu_baseline leg (the oracle port on all host threads, ~8 s sample)
                from bench import cpu_reference_rate
                rate, threads, sample = cpu_reference_rate(spec, dims, budget_s=8.0)
                entry["cpu_oracle"] = {"gstencil": round(rate, 4), "sample": sample,
                                       "threads": threads, "dtype": "f64",
                                       "source": "bench.cpu_reference_rate (the cpu_baseline leg)"}
                entry["speedup_vs_cpu_oracle"] = round(entry["best_gstencil"] / entry["cpu_oracle"]["gstencil"], 1)
            results[f"{key}_{dt}"] = entry
            print(key, dt, {k: (v["gstencil"], v["frac"]) for k, v in entry["k"].items()},
                  "cpu", entry.get("cpu_oracle", {}).get("gstencil"), flush=True)
    out = {"peaks": {"hbm_gbs": hbm, "fp64_tflops": p64, "fp32_tflops": p32},
           "arith": "fma", "timer": "CUDA events around sb_run (device-resident), third sweep of T steps (graph replay)",
           "configs": results}
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
