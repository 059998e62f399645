"""Summarise an ncu report: key throughput metrics, stall breakdown, top SASS by stall."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]}")
st = [(h, v) for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
tot = sum(float(v.replace(",", "") or 0) for _, v in st) or 1
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {float(v.replace(',', '') or 0) / tot * 100:.1f}%"
                           for h, v in sorted(st, key=lambda x: -float(x[1].replace(",", "") or 0))[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
h = srows[1]
isrc, iall, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
by, ex, tot = collections.Counter(), collections.Counter(), 0.0
for r in srows[2:]:
    try:
        a, e = float(r[iall] or 0), float(r[iex] or 0)
    except (ValueError, IndexError):
        continue
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    by[op] += a
    ex[op] += e
    tot += a
print("samples by opcode:", ", ".join(f"{op} {c / tot * 100:.1f}% (x{ex[op]:.3g})" for op, c in by.most_common(12)))
