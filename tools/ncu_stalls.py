"""Per-opcode and per-stall-reason breakdown of an ncu report's source page
(development tool): python tools/ncu_stalls.py report.ncu-rep [topN]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
isrc = h.index("Source")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
by_op = collections.defaultdict(collections.Counter)
lines = []
tot = collections.Counter()
for i, r in enumerate(rows[2:]):
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[0] if not toks[0].startswith("@") else toks[1]
    op = op.split(".")[0]
    c = collections.Counter()
    for k, j in idx.items():
        try:
            v = float(r[j] or 0)
        except ValueError:
            v = 0
        c[k] += v
    by_op[op].update(c)
    tot.update(c)
    lines.append((sum(c.values()), i, r[isrc].strip(), c))
T = sum(tot.values()) or 1
print("total samples", T)
print("by reason:", ", ".join(f"{k[6:]} {v / T * 100:.1f}%" for k, v in tot.most_common(10)))
print("by opcode (share, top reasons):")
for op, c in sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:14]:
    s = sum(c.values())
    print(f"  {op:10s} {s / T * 100:5.1f}%  " + ", ".join(f"{k[6:]} {v / T * 100:.1f}" for k, v in c.most_common(4)))
print("hottest lines:")
for s, i, txt, c in sorted(lines, reverse=True)[:top]:
    print(f"  {i:5d} {s / T * 100:5.2f}% {txt[:70]:70s} " + ", ".join(f"{k[6:]} {v / T * 100:.1f}" for k, v in c.most_common(2)))
