#!/usr/bin/env python
"""Benchmark of the multistep stencil sweep (BASELINE.json metric).

Workload (default): BASELINE configs[4] = C5, the 3D 27-point box stencil in
fp64 with seeded random weights, 768x768x(768*g) interior (+1 halo), T=100,
fused depth k=2 -- the configuration the north_star's 3D targets (>= 70% of
the fusion-depth roofline, >= 85% weak-scaling efficiency at 8 GPUs) name.
One bench "step" = one full sweep (T time steps over the whole grid).  At
N>1 GPUs every rank owns a 768^3 z-slab of the 768^2 x 768N grid ("weak"),
with an r*k-deep ghost exchange (NCCL send/recv) every k steps, overlapped
with the slab interior.  ``--scaling strong`` splits the single-GPU grid
instead (BASELINE's C3: 16384/g rows, C4: 512/g planes).
``--workload c1|c2|c3a|c3b|c4|c5|c5f32`` runs any BASELINE config the same way.

Prints ONE JSON line (rank 0).  ``value`` = whole-job GStencil/s with the
grid resident in HBM (CUDA events on the launching stream, max over ranks);
``e2e`` = the same metric through the C-ABI call with host buffers (pinned
H2D of the input grid + sweep + D2H of the output grid, every step); at N=1
the headline is independent grids pipelined over a ring of plans/streams
(grid i+1's H2D and grid i-1's D2H overlap grid i's sweep), ``serial_value``
the three phases back to back.  ``roofline`` times every main launch of the
timed region with its own CUDA events (``avg_launch_ms`` = the dominant
kernel's mean duration) and reports BASELINE's F-based fraction and the
executed-work fraction side by side.  ``--verify`` checks the final grid of
the timed run against the C oracle (test infrastructure, outside the timed
region).

``--impl reference`` times the reference's algorithm on the host CPU: the
oracle port (oracle/oracle.c, a bit-exact C+OpenMP restatement of
stencilbench's scalar oracle -- the reference is pure Python and cannot be
compiled into oracle/_ref) on all host threads, on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# BASELINE.json configs; at N > 1 every workload is weak-scaled along its
# slowest axis (each rank owns a slab of the single-GPU size) unless
# --scaling strong (the single-GPU grid split over the ranks).
WORKLOADS = {
    "c1": dict(spec="c1", dims=(1 << 20,), T=64, name="1D3P fp64 N=2^20 T=64"),
    "c2": dict(spec="c2", dims=(1 << 26,), T=1000, name="1D5P fp64 N=2^26 T=1000"),
    # slab_k: the fused depth of the slab plans at N > 1 (N = 1 takes the plan default)
    "c3a": dict(spec="c3a", dims=(16384, 16384), T=500, slab_k=32, name="2D9P fp64 16384^2 T=500 (weights 1/9)"),
    "c3b": dict(spec="c3b", dims=(16384, 16384), T=500, slab_k=4, name="2D9P fp64 16384^2 T=500 (seeded random weights)"),
    "c4": dict(spec="c4", dims=(512, 512, 512), T=200, slab_k=2, name="3D7P fp64 512^3 T=200"),
    "c5": dict(spec="c5", dims=(768, 768, 768), T=100, slab_k=2, name="3D27P fp64 768^3 T=100"),
    "c5f32": dict(spec="c5", dims=(768, 768, 768), T=100, slab_k=2, dtype="f32", name="3D27P fp32 768^3 T=100"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=list(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = a single-GPU-size slab per rank; strong = the single-GPU grid split")
    ap.add_argument("--verify", action="store_true", help="check the final grid against the C oracle")
    ap.add_argument("--k", type=int, default=0, help="fusion depth (0: the plan default -- 32 for C2 in FMA "
                                                 "mode, 4 for 2D, 2 for 3D)")
    ap.add_argument("--arith", default="fma", choices=["fma", "exact"])
    ap.add_argument("--sweep-k", action="store_true", help="also time k in {1,2,4,8,16}")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------- utilities

def measured_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "source": {}}
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            m = json.load(fh)
        peaks["hbm_gbs"] = m.get("hbm_gbs")
        peaks["source"]["hbm"] = "measured (MEASURED_PEAKS.json)"
    if peaks["hbm_gbs"] is None:
        peaks["hbm_gbs"] = 6650.0
        peaks["source"]["hbm"] = "fallback (B200_PROFILING.md)"
    fp = os.path.join(REPO, "profiles", "fp_peak.json")
    if os.path.exists(fp):
        with open(fp) as fh:
            f = json.load(fh)
        peaks["fp64_tflops"] = f["fp64_tflops"]
        peaks["fp32_tflops"] = f["fp32_tflops"]
        peaks["source"]["fp64"] = peaks["source"]["fp32"] = "measured (profiles/fp_peak.json, tools/fp_peak.cu)"
    else:
        peaks["fp64_tflops"], peaks["fp32_tflops"] = 37.0, 74.0
        peaks["source"]["fp64"] = peaks["source"]["fp32"] = "datasheet (not measured)"
    return peaks


class ClockSampler:
    """nvidia-smi clocks/throttle sampling around the timed region.

    Started before warm-up (nvidia-smi needs ~1 s to start); every sample is
    time-stamped on arrival and summary() keeps those inside the timed window
    [mark_start, mark_end] (the two nearest ones if the window is shorter
    than the sampling period)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")
    NAMES = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.samples = []          # (wall time, line)
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            deadline = time.time() + 5
            while not self.samples and time.time() < deadline:
                time.sleep(0.05)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        parsed = []
        for t, line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                parsed.append((t, float(parts[0]), float(parts[1]), parts[3:7], float(parts[2])))
            except ValueError:
                continue
        if not parsed:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        inside = [p for p in parsed if self.t0 is not None and self.t0 <= p[0] <= (self.t1 or p[0])]
        window = "timed region"
        if not inside:
            mid = ((self.t0 or 0) + (self.t1 or 0)) / 2
            inside = sorted(parsed, key=lambda p: abs(p[0] - mid))[:2]
            window = "nearest to a timed region shorter than the sampling period"
        reasons = sorted({nm for p in inside for nm, v in zip(self.NAMES, p[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(p[1] for p in inside), "sm_max_mhz": inside[-1][2],
                "reasons": reasons, "samples": len(inside), "window": window,
                "power_w_median": statistics.median(p[4] for p in inside)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------ CPU reference

def seeded_host_box(dims, r, seed=12345):
    return np.random.default_rng(seed).random(tuple(int(d) + 2 * r for d in dims))


def cpu_reference_rate(spec, dims, sample_steps=None, budget_s=10.0):
    """Oracle port (C+OpenMP, all host threads) on a bounded sample of the
    workload grid; returns (GStencil/s, threads, sample description)."""
    from oracle import c_oracle
    from paper_2103_08825_b200.core import canonical
    offs, ws = canonical(spec)
    threads = c_oracle.max_threads()
    n = int(np.prod(dims))
    box = seeded_host_box(dims, spec.r)
    t0 = time.perf_counter()
    c_oracle.sweep(box, spec.r, offs, ws, 1, threads=threads, inplace=True)
    t1 = time.perf_counter()
    c_oracle.sweep(box, spec.r, offs, ws, 3, threads=threads, inplace=True)
    t3 = time.perf_counter()
    one = max((t3 - t1) - (t1 - t0), 1e-6) / 2       # marginal step (a call also copies the grid)
    if sample_steps is None:
        sample_steps = int(max(2, min(1000, budget_s / one)))
    t0 = time.perf_counter()
    c_oracle.sweep(box, spec.r, offs, ws, sample_steps, threads=threads, inplace=True)
    dt = time.perf_counter() - t0
    rate = n * sample_steps / dt / 1e9
    return rate, threads, f"{sample_steps} steps of the full {'x'.join(map(str, dims))} grid (same spec)"


def reference_numpy_rate(spec, dims, budget_s=6.0):
    """The reference's own code: ``stencilbench.kernels.scalar_step`` (numpy,
    one core) from the installed reference (baseline/_ref), one step over a
    slab of the workload grid sized to ~budget_s.  None when not installed."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "stencilbench")) and ref not in sys.path:
        sys.path.append(ref)
    try:
        from stencilbench import core as sc
        from stencilbench import kernels as sk
    except ImportError:
        return None
    rspec = sc.StencilSpec(spec.name, spec.d, spec.r, spec.shape, dict(spec.weights))
    plane = int(np.prod(dims[1:])) if len(dims) > 1 else 1

    def one(n0):
        sub = (n0,) + tuple(dims[1:])
        a = sc.alloc_grid(rspec, sub, sc.Layout.NATURAL, 4)
        a.set_interior(np.random.default_rng(1).random(sub))
        b = sc.alloc_like(a)
        t0 = time.perf_counter()
        sk.scalar_step(a, b, rspec)
        return n0 * plane / (time.perf_counter() - t0), sub

    n0 = max(1, min(dims[0], (1 << 16) // plane if plane < (1 << 16) else 1))
    rate, sub = one(n0)
    n0 = int(max(1, min(dims[0], budget_s * rate / plane)))
    rate, sub = one(n0)
    return {"value": rate / 1e9, "unit": "GStencil/s", "cores": 1, "kind": "reference",
            "sample": f"one stencilbench.kernels.scalar_step (numpy) over {'x'.join(map(str, sub))} "
                      f"of the workload grid, from the installed reference (baseline/_ref)"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2103_08825_b200.core import config_spec
    wl = WORKLOADS[args.workload]
    spec = config_spec(wl["spec"])
    dims = wl["dims"]
    n = int(np.prod(dims))
    from oracle import c_oracle
    from paper_2103_08825_b200.core import canonical
    offs, ws = canonical(spec)
    threads = c_oracle.max_threads()
    box = seeded_host_box(dims, spec.r)
    # marginal cost of a step (a call also allocates and copies the partner grid)
    t0 = time.perf_counter()
    c_oracle.sweep(box, spec.r, offs, ws, 1, threads=threads, inplace=True)
    t1 = time.perf_counter()
    c_oracle.sweep(box, spec.r, offs, ws, 3, threads=threads, inplace=True)
    t3 = time.perf_counter()
    one = max((t3 - t1) - (t1 - t0), 1e-6) / 2
    per_step = int(max(2, min(wl["T"], 8.0 / one)))   # ~8 s per bench step
    for _ in range(args.warmup):
        c_oracle.sweep(box, spec.r, offs, ws, max(1, per_step // 4), threads=threads, inplace=True)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c_oracle.sweep(box, spec.r, offs, ws, per_step, threads=threads, inplace=True)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n * per_step * args.steps / total / 1e9
    sample = (f"{per_step} of T={wl['T']} steps of the full {'x'.join(map(str, dims))} grid per bench step"
              + (" (fp64 oracle; the reference is fp64-only)" if wl.get("dtype") == "f32" else ""))
    line = {
        "impl": "reference", "metric": "GStencil/s", "value": value, "unit": "GStencil/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": wl.get("dtype", "f64"), "data": "synthetic",
        "config": {"workload": wl["name"], "k": 1, "host": "cpu"},
        "cpu_baseline": {"value": value, "unit": "GStencil/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "GStencil/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    try:
        line["reference_numpy"] = reference_numpy_rate(spec, dims)
    except MemoryError:
        pass
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def kernel_label(spec, wl, k, arith):
    """Main kernel a sweep of this workload launches (see sb200.cu / launch*.cu)."""
    d = len(wl["dims"])
    if d == 1:
        return (f"compose1d_kernel<double, {spec.r * k}, {spec.r}>" if arith == "fma" and k >= 16
                else f"fused1d_kernel (K={k})")
    if d == 2:
        if k >= 16:
            return f"sep_vpass_kernel + sep_hpass_kernel (K={k}, separable composed)"
        if wl.get("dtype", "f64") == "f64" and k == 4:
            return f"split2d_kernel (K={k}: halo-free items on the lean path, plain2d.cuh)"
        return f"fused2d_kernel (K={k})"
    if spec.shape == "star" and arith == "fma" and k == 2 and wl.get("dtype", "f64") == "f64":
        return "compose3d_kernel (two steps as one 25-point pass)"
    if spec.shape == "box" and k == 2:
        return "box3d_kernel (64xTY output tiles, ring-only level-1 recompute)"
    return f"fused3d_kernel (K={k})"


def executed_ops(spec, wl, k, arith, kernel_name):
    """FP-pipe instructions per point update the main kernel's algorithm
    issues (FMA and MUL/ADD each one op; overlapped-tile recompute excluded),
    and a description -- the denominator of the executed-work roofline."""
    W = len(spec.weights)
    if arith == "exact":
        return 2 * W - 1, "EXACT: one rounded multiply + one rounded add per term"
    if kernel_name.startswith("compose1d"):
        return (2 * spec.r * k + 1) / k, f"K-fold composed ({2 * spec.r * k + 1}-tap) stencil per {k} steps"
    if kernel_name.startswith("sep_vpass"):
        return 2 * (2 * k + 1) / k, "two composed 1D passes of 2K+1 taps per K steps"
    if kernel_name.startswith("compose3d"):
        return 12.5, "25-point two-step composition per 2 steps"
    if len(wl["dims"]) == 2 and wl["spec"] == "c3a":
        return 6, "separable push: 3 horizontal + 3 vertical FMAs per level"
    return W, f"{W} FMA per update (one MUL + {W - 1} FMA)"


def run_gpu_arm(args):
    import torch
    rank, world, local = dist_env()
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")           # lets the driver count communicator ranks
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # stdout carries only the JSON line
        import torch.distributed as dist
        # SB200_SHARE_GPU=1 (TEST mode, tools/share_gpu_bench.sh): every rank on cuda:0 over
        # gloo, the slab exchange staged through the host -- checks this N>1 code path on a
        # one-GPU box; its numbers are not scaling measurements
        share_gpu = bool(os.environ.get("SB200_SHARE_GPU"))
        torch.cuda.set_device(0 if share_gpu else local)
        dist.init_process_group("gloo" if share_gpu else "nccl")
    else:
        torch.cuda.set_device(0)
    device = torch.cuda.current_device()

    from paper_2103_08825_b200.core import config_spec
    from paper_2103_08825_b200.plan import Plan
    wl = WORKLOADS[args.workload]
    spec = config_spec(wl["spec"])
    dims, T, k = tuple(wl["dims"]), wl["T"], args.k
    dtype = wl.get("dtype", "f64")
    torch_dtype = torch.float64 if dtype == "f64" else torch.float32
    es = 8 if dtype == "f64" else 4
    strong = args.scaling == "strong" and world > 1
    # a dedicated stream: torch's default (legacy) stream has handle 0, which
    # sb_set_stream treats as "use the plan's own stream"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rng = np.random.default_rng(12345 + rank)

    if world > 1:
        from paper_2103_08825_b200.slab import SlabSweep
        k = k or wl.get("slab_k") or (32 if args.arith == "fma" else 16)
        gdims = dims if strong else (dims[0] * world,) + dims[1:]
        runner = SlabSweep(spec, gdims, rank=rank, world=world, k=k, arith=args.arith, dtype=dtype,
                           device=device, stream_ptr=stream.cuda_stream)
        plan = runner.plan
        n_total = int(np.prod(gdims))
    else:
        plan = Plan(spec, dims, k=k, arith=args.arith, dtype=dtype, device=device)
        k = plan.k
        plan.set_stream(stream.cuda_stream)
        n_total = int(np.prod(dims))
    n_local = int(np.prod(plan.dims))
    host_in = torch.empty(plan.shape, dtype=torch_dtype, pin_memory=True)
    host_in.numpy()[...] = rng.random(plan.shape)
    host_out = torch.empty_like(host_in, pin_memory=True)
    # slab runs upload through the runner (it re-exchanges the uploaded ghost planes)
    upload = ((lambda: runner.upload(host_in.numpy())) if world > 1      # noqa: E731
              else (lambda: plan.upload(host_in.numpy())))
    download = lambda: plan.download(host_out.numpy())       # noqa: E731

    # one sweep = T steps; at N=1 a CUDA event on the plan stream precedes every
    # launch of the timed region (one more closes it): consecutive events
    # bracket each launch, so the per-launch durations are measured live
    n_full, tail = divmod(T, k)
    chunks = [k] * n_full + ([tail] if tail else [])

    def sweep_events(evs):
        for j, kk in enumerate(chunks):
            evs[j].record(stream)
            plan.launch(kk)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(device).start()
    upload()
    for _ in range(args.warmup):
        if world > 1:
            runner.run(T)
        else:
            plan.launch(T)
    barrier()

    launch_evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(chunks))]
                  for _ in range(args.steps)] if world == 1 else None
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernels_before = plan.kernel_count()
    barrier()
    clocks.mark_start()
    # a sweep that is ONE launch (C1: ~10 us) is enqueued natively, K back-to-back
    # sweeps with an event around each (sb_launch_repeat): a Python loop with
    # per-launch events would bound it by the interpreter, not the GPU
    native_repeat = world == 1 and len(chunks) == 1
    ev0.record(stream)
    if native_repeat:
        plan.launch_repeat(T, args.steps)
    else:
        for i in range(args.steps):
            if world > 1:
                runner.run(T)
            else:
                sweep_events(launch_evs[i])
    ev1.record(stream)
    barrier()
    clocks.mark_end()
    clocks.stop()
    ms = ev0.elapsed_time(ev1)
    kernels = plan.kernel_count() - kernels_before            # this rank's launches, timed region
    if dist is not None:
        t = torch.tensor([ms], device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n_total * T / (ms_per_step * 1e-3) / 1e9

    # Dominant kernel: the main launch of k fused steps.  N=1: mean of the
    # event-timed full-depth launches of the timed region; N>1: the step time
    # spread over the launches (edge/interior/exchange overlap inside).
    if native_repeat:
        # the timed region is nothing but the dominant kernel, back to back (programmatic
        # dependent launch between sweeps): its mean duration is the region / launches
        # (events between launches would add ~2.5 us of device time to each ~10 us sweep)
        total = plan.repeat_times()[0]
        launch_ms = total / args.steps
        launch_src = (f"CUDA events around the {args.steps} back-to-back launches of the timed region (one k={k} "
                      f"launch per sweep, nothing else on the stream; sb_launch_repeat)")
        share = total / ms
    elif world == 1:
        flat = [e for evs in launch_evs for e in evs] + [ev1]
        full = [flat[i * len(chunks) + j].elapsed_time(flat[i * len(chunks) + j + 1])
                for i in range(args.steps) for j in range(n_full)]
        launch_ms = statistics.mean(full)
        launch_src = (f"CUDA events around each of the {len(full)} full-depth (k={k}) launches of the timed "
                      f"region, on the plan stream")
        share = launch_ms * n_full / ms_per_step
    else:
        launch_ms = ms_per_step / len(chunks)
        launch_src = "step time / launches per sweep (slab mode: edge + interior + exchange per launch)"
        share = None
    peaks = measured_peaks()
    fp_key = "fp64" if dtype == "f64" else "fp32"
    fp_peak = peaks[f"{fp_key}_tflops"]
    per_gpu = value / world
    F = 2 * len(spec.weights) - 1                             # BASELINE's F = 2|W| - 1
    alg_bytes_per_point = 2 * es                              # read + write once per fused launch
    fp_bound = fp_peak * 1e12 / F / 1e9
    hbm_bound = peaks["hbm_gbs"] * 1e9 * k / alg_bytes_per_point / 1e9
    binding = "hbm" if hbm_bound < fp_bound else fp_key
    kernel_name = kernel_label(spec, wl, k, args.arith)
    # algorithmic work per launch of k steps: 2s B per point
    # (read + write once), F flops per point update
    alg_bytes = alg_bytes_per_point * n_local
    alg_flops = F * n_local * k
    achieved_gbs = alg_bytes / (launch_ms * 1e-3) / 1e9
    achieved_tflops = alg_flops / (launch_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    tpath = os.path.join(REPO, "profiles", "kernel_traffic.json")
    if os.path.exists(tpath) and world == 1:
        with open(tpath) as fh:
            tj = json.load(fh)
        ent = tj.get(f"{args.workload}:{args.arith}:k{k}")
        if ent and ent.get("dims") == list(dims):
            traffic = ent["traffic_bytes"]
            traffic_src = ent["source"]
    hbm_view = {"achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved_gbs / peaks["hbm_gbs"], "alg_bytes_per_launch": alg_bytes,
                "peak_source": peaks["source"]["hbm"]}
    fp_view = {"achieved": achieved_tflops, "peak": fp_peak, "unit": "TFLOP/s",
               "frac": achieved_tflops / fp_peak, "alg_flops_per_launch": alg_flops,
               "peak_source": peaks["source"][fp_key]}
    main = hbm_view if binding == "hbm" else fp_view
    ops, ops_desc = executed_ops(spec, wl, k, args.arith, kernel_name)
    exec_fp_bound = fp_peak * 1e12 / 2 / ops / 1e9           # pipe ops/s (an FMA = 2 flops of the peak)
    exec_bound = min(hbm_bound, exec_fp_bound)
    kern_rate = n_local * k / (launch_ms * 1e-3) / 1e9       # dominant kernel alone, GStencil/s
    roofline = {
        "bound": binding, "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"],
        "frac": main["frac"], "traffic": traffic, "traffic_source": traffic_src,
        "kernel": kernel_name, "avg_launch_ms": launch_ms, "avg_launch_source": launch_src,
        "kernel_share_of_step": share,
        "executed_frac": kern_rate / exec_bound,
        "executed": {"fp_ops_per_update": ops, "what": ops_desc,
                     "roofline_gstencil": exec_bound, "kernel_gstencil": kern_rate,
                     "fp_pipe_frac": kern_rate * 1e9 * ops * 2 / (fp_peak * 1e12),
                     "note": "executed_frac = the dominant kernel's rate / min(HBM bound, FP peak over the "
                             "FP-pipe ops its algorithm issues); 'frac' uses BASELINE's F = 2|W|-1 flops"},
        "note": f"bound = the lower of the HBM roofline ({alg_bytes_per_point} B/point/launch) and the "
                f"{fp_key.upper()} roofline (F flops/update); '{fp_key}' is the CUDA-core {fp_key.upper()} "
                "pipe (a stencil is not a tensor-core contraction)",
        "hbm": hbm_view, fp_key: fp_view,
    }
    stencil_roofline = {
        "k": k, "hbm_bound_gstencil": hbm_bound, f"{fp_key}_bound_gstencil": fp_bound,
        "binding": binding, "achieved_gstencil_per_gpu": per_gpu,
        "frac": per_gpu / min(hbm_bound, fp_bound),
        "executed_frac": per_gpu / exec_bound,
        "note": "frac uses BASELINE's algorithmic F = 2|W|-1 flops per update; executed_frac the "
                "FP-pipe ops the kernel's algorithm issues (roofline.executed)",
    }

    # End to end through the C-ABI with host buffers: every step uploads its
    # input grid from pinned host memory (H2D), sweeps T steps and downloads
    # the result grid (D2H).  "serial": one plan, the three phases back to
    # back.  Headline (N=1): independent grids pipelined over a ring of plans on
    # their own streams (sb_upload_async / sb_launch / sb_download_async), so
    # grid i+1's H2D and grid i-1's D2H run on the copy engines during grid i's sweep.
    e2e = None
    run_once = (lambda: runner.run(T)) if world > 1 else (lambda: plan.launch(T))   # noqa: E731
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if world == 1:
                # the one-call form of upload + T steps + download (sb_sweep_host; pinned buffers:
                # on 3D plans the transfers stream block by block beside the sweep)
                plan.sweep_host(host_in.numpy(), T, out=host_out.numpy())
            else:
                upload()
                run_once()
                download()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device="cpu" if dist is not None and dist.get_backend() == "gloo" else "cuda")
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        serial = n_total * T * args.steps / dt / 1e9
        e2e = {"value": serial, "unit": "GStencil/s",
               "h2d_bytes_per_step": int(host_in.numel() * es * world),
               "d2h_bytes_per_step": int(host_out.numel() * es * world),
               "mode": "serial", "timer": "host wall clock around upload+sweep+download (N=1: one sb_sweep_host "
                                          "call per step), max over ranks"}
        grid_bytes = host_in.numel() * es
        if world == 1:
            want = host_out.numpy().copy()                       # serial result of the last step
            NP = 3 if grid_bytes <= (8 << 30) else 2             # plans in the ring (device memory)
            plans = [plan] + [Plan(spec, dims, k=k, arith=args.arith, dtype=dtype, device=device)
                              for _ in range(NP - 1)]
            streams = [stream] + [torch.cuda.Stream() for _ in range(NP - 1)]
            for p, st in zip(plans[1:], streams[1:]):
                p.set_stream(st.cuda_stream)
            outs = [host_out] + [torch.empty_like(host_out, pin_memory=True) for _ in range(NP - 1)]

            def pipelined(i):
                p = plans[i % NP]
                p.upload_async(host_in.numpy())
                p.launch(T)
                p.download_async(outs[i % NP].numpy())

            for i in range(2 * NP):                              # warm-up: eager + graph capture per plan
                pipelined(i)
            for p in plans:
                p.synchronize()
            t0 = time.perf_counter()
            for i in range(args.steps):
                pipelined(i)
            for p in plans:
                p.synchronize()
            dt = time.perf_counter() - t0
            same = all(np.array_equal(o.numpy(), want) for o in outs)
            for p in plans[1:]:
                p.close()
            # the plain drop-in call: sweep(spec, numpy box, T) on PAGEABLE arrays, as a caller of
            # the reference hands them over (plan from the per-thread cache, pageable transfers
            # through the pinned bounce buffers of hostxfer.cu, a fresh output array per call)
            from paper_2103_08825_b200.plan import sweep as sweep_call, clear_plan_cache
            page_in = np.array(host_in.numpy(), copy=True)       # pageable copy of the workload grid
            sweep_call(spec, page_in, T, arith=args.arith, k=k, dtype=dtype, device=device)   # warm: plan, bounce buffers
            tc = []
            for _ in range(2):
                t0 = time.perf_counter()
                got = sweep_call(spec, page_in, T, arith=args.arith, k=k, dtype=dtype, device=device)
                tc.append(time.perf_counter() - t0)
            call_same = bool(np.array_equal(got, want))
            clear_plan_cache()
            del page_in, got
            e2e["pageable_call"] = {"value": n_total * T / min(tc) / 1e9, "unit": "GStencil/s", "ms": min(tc) * 1e3,
                                    "what": "sweep(spec, box, T) with pageable numpy arrays in and out (best of 2 "
                                            "after one warm call)", "result_matches_serial": call_same}
            e2e.update({"value": n_total * T * args.steps / dt / 1e9, "mode": "pipelined",
                        "serial_value": serial, "result_matches_serial": bool(same),
                        "timer": f"host wall clock from the first enqueue to every plan's sync; "
                                 f"{args.steps} independent grids over a ring of {NP} plans/streams "
                                 f"(includes the unoverlapped first H2D and last D2H)"})

    verify = None
    if args.verify and world == 1:
        # the bench path's output for one sweep of host_in vs the C oracle (test
        # infrastructure; outside every timed region)
        from oracle import c_oracle
        from paper_2103_08825_b200.core import canonical
        offs, ws = canonical(spec)
        upload()
        plan.launch(T)
        download()
        torch.cuda.synchronize()
        o_in = host_in.numpy().astype(np.float64)
        o_ws = [float(np.float32(w)) for w in ws] if dtype == "f32" else ws
        t0 = time.perf_counter()
        want = c_oracle.sweep(o_in, spec.r, offs, o_ws, T, inplace=True)
        g = host_out.numpy().astype(np.float64)
        err = float(np.max(np.abs(g - want) / np.maximum(np.abs(want), np.finfo(np.float64).tiny)))
        tol = 1e-5 if dtype == "f32" else (0.0 if args.arith == "exact" else 1e-12)
        verify = {"max_rel_err": err, "tol": tol, "ok": bool(err <= tol), "T": T,
                  "oracle": f"oracle/oracle.c on {c_oracle.max_threads()} threads, "
                            f"{time.perf_counter() - t0:.1f} s"}

    sweep = None
    if args.sweep_k and world == 1:
        sweep = {}
        ks = {1: (1, 2, 4, 8, 16, 32), 2: (1, 2, 4, 8), 3: (1, 2, 3, 4)}[len(dims)]
        for kk in ks:
            with Plan(spec, dims, k=kk, arith=args.arith, dtype=dtype, device=device) as p:
                p.upload(host_in.numpy())
                p.run(T // 4)
                tim = p.run(T)
                g = n_local * T / (tim.device_ms * 1e-3) / 1e9
                hb = peaks["hbm_gbs"] * kk / alg_bytes_per_point
                sweep[str(kk)] = {"gstencil": g, "ms": tim.device_ms, "launches": tim.launches,
                                  "kernel": tim.kernel_name, "roofline_gstencil": min(hb, fp_bound),
                                  "binding": "hbm" if hb < fp_bound else fp_key,
                                  "frac": g / min(hb, fp_bound)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, threads, sample = cpu_reference_rate(spec, dims)
        cpu = {"value": rate, "unit": "GStencil/s", "cores": threads, "kind": "port",
               "sample": sample + "; oracle/oracle.c (bit-exact restatement of "
                                  "stencilbench scalar_step), OpenMP"
                                  + (", fp64 (the reference is fp64-only)" if dtype == "f32" else "")}
        try:
            cpu["reference_numpy"] = reference_numpy_rate(spec, dims)
        except MemoryError:
            pass

    if rank == 0:
        grid_bytes = int(np.prod([d + 2 * spec.r for d in plan.dims])) * es
        if world > 1:
            scale = (f", strong-scaled over {world} GPUs (1/{world} slab per GPU)" if strong
                     else f", weak-scaled x{world} (a single-GPU-size slab per GPU)")
        else:
            scale = ""
        line = {
            "metric": "GStencil/s", "value": value, "unit": "GStencil/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic",
            "config": {"workload": wl["name"] + scale, "dims_per_gpu": list(plan.dims),
                       "k": k, "arith": args.arith, "grid_bytes_per_gpu": grid_bytes,
                       "l2": (f"inputs larger than L2 ({grid_bytes / 1e6:.0f} MB grid vs 126 MB L2)"
                              if grid_bytes > (126 << 20) else "grid fits in L2"),
                       "parallelism": (f"slab{world}" if world > 1 else "single"),
                       **({"test_mode": "SB200_SHARE_GPU: all ranks on one GPU over gloo, host-staged exchange -- "
                                        "a code-path check, not a scaling measurement"}
                          if world > 1 and os.environ.get("SB200_SHARE_GPU") else {})},
            "roofline": roofline, "stencil_roofline": stencil_roofline,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": kernels * world,
            "gpu_launches_note": "all ranks; per sweep and rank: ceil(T/k) main launches (1D composed: "
                                 "boundary windows inside the same launch) + the level-by-level tail's "
                                 "boundary kernel / the 3D shell kernel on a side stream",
            "clocks": clocks.summary(),
        }
        if verify is not None:
            line["verify"] = verify
        if sweep is not None:
            line["k_sweep"] = sweep
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
