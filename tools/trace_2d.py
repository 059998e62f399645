"""Run one C3 launch with the per-item trace on and summarise the tail."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SB200_TRACE", "/tmp/sb200_trace2d.bin")
from paper_2103_08825_b200.core import config_spec  # noqa: E402
from paper_2103_08825_b200.plan import Plan  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec = config_spec("c3a")
dims = (16384, 16384)
box = np.random.default_rng(1).random(tuple(n + 2 for n in dims))
with Plan(spec, dims, k=k) as p:
    p.upload(box)
    p.run(k * 2)
    t = p.run(k)
tr = np.fromfile(os.environ["SB200_TRACE"], dtype=np.uint64).reshape(-1, 4)
sm = (tr[:, 0] >> 32).astype(int)
warp = (tr[:, 0] & 0xffffffff).astype(int)
t0 = tr[:, 1].astype(np.int64)
t1 = tr[:, 2].astype(np.int64)
strip = (tr[:, 3] >> 40).astype(int)
rows = (tr[:, 3] & 0xffffffffff).astype(int)
base = t0.min()
t0 -= base
t1 -= base
dur = (t1 - t0) / 1e3
print(f"k={k} launch {t.device_ms*1e3:.0f} us, items {len(tr)}, span {t1.max()/1e3:.0f} us")
end_sm = collections.defaultdict(int)
for s_, b in zip(sm, t1):
    end_sm[s_] = max(end_sm[s_], b)
ends = np.array(sorted(end_sm.values())) / 1e3
print("SM finish us: min %.0f p10 %.0f median %.0f p90 %.0f max %.0f" % (
    ends.min(), np.percentile(ends, 10), np.median(ends), np.percentile(ends, 90), ends.max()))
us_per_row = dur / (rows + 2 * k)
print("us per row: p10 %.2f median %.2f p90 %.2f max %.2f" % tuple(np.percentile(us_per_row, [10, 50, 90, 100])))
order = np.argsort(-t1)[:12]
print("last-finishing items: idx strip rows start_us end_us dur_us us/row sm warp")
for i in order:
    print(f"  {i:6d} {strip[i]:4d} {rows[i]:5d} {t0[i]/1e3:8.0f} {t1[i]/1e3:8.0f} {dur[i]:7.0f} {us_per_row[i]:6.2f} {sm[i]:4d} {warp[i]:5d}")
# first-round items: duration by warp slot within the SM (warp priority)
slot = warp % 16
first = np.argsort(t0)[: len(set(warp))]
by_slot = collections.defaultdict(list)
for i in first:
    by_slot[slot[i]].append(us_per_row[i])
print("first-item us/row by warp slot:", {k_: round(float(np.median(v)), 2) for k_, v in sorted(by_slot.items())})
