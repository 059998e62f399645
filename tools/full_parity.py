#!/usr/bin/env python
"""Parity after ALL steps, at full BASELINE size, for every benched config.

north_star: "fp64: max relative error <= 1e-12 after all steps; fp32 <= 1e-5".
Each case runs the device sweep (the bench's kernel path: FMA mode at the
bench's fusion depth, plus EXACT mode, which must be bit-identical) on the
full grid for the full T, and the C oracle (oracle/oracle.c, the bit-exact
restatement of stencilbench scalar_step, pinned to reference fixtures by
tests/test_oracle.py) on the host cores concurrently (ctypes releases the
GIL).  The relative error is the reference's max_rel_error
(harness.py:214-216) over the whole box (halo included: it must be unchanged).

TEST INFRASTRUCTURE: the oracle is the checker here, never the thing measured.

    python tools/full_parity.py [--cases c2,c4] [--out gpurun_out/full_parity.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

FP64_TOL = 1e-12
FP32_TOL = 1e-5

# name -> config key, interior, T, halo convention, input seed, dtype, device variants
#   variant = (arith, k): k = 0 is the plan default (the bench's kernel path)
CASES = {
    "c1": dict(spec="c1", dims=(1 << 20,), T=64, halo="full", seed=101, dtype="f64",
               variants=[("fma", 64), ("exact", 0)]),
    "c2": dict(spec="c2", dims=(1 << 26,), T=1000, halo="full", seed=102, dtype="f64",
               variants=[("fma", 32), ("exact", 0)]),
    "c2_halo0": dict(spec="c2", dims=(1 << 26,), T=1000, halo="zero", seed=103, dtype="f64",
                     variants=[("fma", 32)]),
    "c3a": dict(spec="c3a", dims=(16384, 16384), T=500, halo="full", seed=104, dtype="f64",
                variants=[("fma", 0), ("exact", 0)]),
    "c3b": dict(spec="c3b", dims=(16384, 16384), T=500, halo="full", seed=105, dtype="f64",
                variants=[("fma", 0), ("exact", 0)]),
    "c4": dict(spec="c4", dims=(512, 512, 512), T=200, halo="full", seed=106, dtype="f64",
               variants=[("fma", 0), ("exact", 0)]),
    "c5": dict(spec="c5", dims=(768, 768, 768), T=100, halo="full", seed=107, dtype="f64",
               variants=[("fma", 0), ("exact", 0)]),
    "c5f32": dict(spec="c5", dims=(768, 768, 768), T=100, halo="full", seed=108, dtype="f32",
                  variants=[("fma", 0)]),
}


def seeded(dims, r, seed, halo):
    rng = np.random.default_rng(seed)
    shape = tuple(n + 2 * r for n in dims)
    if halo == "zero":
        box = np.zeros(shape)
        box[tuple(slice(r, r + n) for n in dims)] = rng.random(dims)
        return box
    return rng.random(shape)


def max_rel_error(got, want):
    """harness.py:214-216 over the whole box, chunked (bounded temporaries)."""
    g = got.reshape(-1)
    w = want.reshape(-1)
    tiny = np.finfo(np.float64).tiny
    worst = 0.0
    step = 1 << 24
    for i in range(0, g.size, step):
        a = g[i:i + step].astype(np.float64)
        b = w[i:i + step]
        e = np.abs(a - b) / np.maximum(np.abs(b), tiny)
        if np.isnan(e).any():
            return float("nan")
        worst = max(worst, float(e.max()))
    return worst


def run_case(name, cfg, log=print):
    from oracle import c_oracle
    from paper_2103_08825_b200.core import canonical, config_spec
    from paper_2103_08825_b200.plan import Plan

    spec = config_spec(cfg["spec"])
    dims, T = tuple(cfg["dims"]), int(cfg["T"])
    box = seeded(dims, spec.r, cfg["seed"], cfg["halo"])
    offs, ws = canonical(spec)
    f32 = cfg["dtype"] == "f32"
    if f32:   # fp64 oracle on the fp32-rounded inputs and weights (the reference is fp64-only)
        dev_box = box.astype(np.float32)
        o_box = dev_box.astype(np.float64)
        o_ws = [float(np.float32(w)) for w in ws]
    else:
        dev_box = box
        o_box = box.copy()
        o_ws = ws
    res = {"case": name, "workload": cfg["spec"], "dims": list(dims), "T": T, "halo": cfg["halo"],
           "dtype": cfg["dtype"], "seed": cfg["seed"], "variants": []}
    oracle_out = {}

    def oracle_thread():
        t0 = time.perf_counter()
        oracle_out["box"] = c_oracle.sweep(o_box, spec.r, offs, o_ws, T, inplace=True)
        oracle_out["seconds"] = time.perf_counter() - t0

    th = threading.Thread(target=oracle_thread)
    th.start()
    outs = []
    for arith, k in cfg["variants"]:
        with Plan(spec, dims, k=k, arith=arith, dtype=cfg["dtype"]) as p:
            p.upload(dev_box)
            tim = p.run(T)
            outs.append((arith, p.k, tim, p.download()))
        log(f"  {name}: device {arith} k={p.k} {tim.kernel_name}: {tim.device_ms:.1f} ms "
            f"({np.prod(dims) * T / tim.device_ms / 1e6:.0f} GStencil/s)")
    th.join()
    want = oracle_out["box"]
    res["oracle_seconds"] = oracle_out["seconds"]
    res["oracle_threads"] = c_oracle.max_threads()
    for arith, k, tim, got in outs:
        err = max_rel_error(got, want)
        tol = FP32_TOL if f32 else (0.0 if arith == "exact" else FP64_TOL)
        v = {"arith": arith, "k": k, "kernel": tim.kernel_name, "launches": tim.launches,
             "device_ms": tim.device_ms, "max_rel_err": err, "tol": tol,
             "bit_identical": bool(got.tobytes() == want.tobytes()) if not f32 else None,
             "ok": bool(err <= tol)}
        res["variants"].append(v)
        log(f"  {name}: {arith} k={k} max_rel_err {err:.3e} (tol {tol:g}) "
            f"{'bit-identical' if v['bit_identical'] else ''} -> {'ok' if v['ok'] else 'FAIL'}")
    res["ok"] = all(v["ok"] for v in res["variants"])
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "full_parity.json"))
    a = ap.parse_args()
    results = []
    t0 = time.time()
    for name in a.cases.split(","):
        print(f"[{time.time() - t0:6.1f}s] {name}", flush=True)
        results.append(run_case(name, CASES[name], log=lambda s: print(s, flush=True)))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump({"tool": "tools/full_parity.py", "wall_seconds": time.time() - t0,
                   "cpu_count": os.cpu_count(), "results": results}, fh, indent=1)
    ok = all(r["ok"] for r in results)
    print(f"full-T parity: {'ALL OK' if ok else 'FAILURES'} in {time.time() - t0:.0f} s", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
