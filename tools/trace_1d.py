"""Run one C2 sweep with the per-chunk trace on and summarise it."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SB200_TRACE", "/tmp/sb200_trace.bin")
from paper_2103_08825_b200.core import config_spec  # noqa: E402
from paper_2103_08825_b200.plan import Plan  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec = config_spec("c2")
n = 1 << 26
box = np.random.default_rng(1).random(n + 4)
with Plan(spec, (n,), k=k) as p:
    p.upload(box)
    p.run(k * 4)
    t = p.run(k)
tr = np.fromfile(os.environ["SB200_TRACE"], dtype=np.uint64).reshape(-1, 4)
sm = (tr[:, 0] >> 32).astype(int)
warp = (tr[:, 0] & 0xffffffff).astype(int)
t0 = tr[:, 1].astype(np.int64)
t1 = tr[:, 2].astype(np.int64)
base = t0.min()
t0 -= base
t1 -= base
dur = t1 - t0
print(f"k={k} launch {t.device_ms*1e3:.0f} us, chunks {len(tr)}, span {t1.max()/1e3:.0f} us")
import collections
end_by_sm = collections.defaultdict(int)
busy_by_sm = collections.defaultdict(int)
for s, a, b in zip(sm, t0, t1):
    end_by_sm[s] = max(end_by_sm[s], b)
    busy_by_sm[s] += b - a
ends = np.array(sorted(end_by_sm.values())) / 1e3
print("SM finish time us: min %.0f p10 %.0f median %.0f p90 %.0f max %.0f" % (
    ends.min(), np.percentile(ends, 10), np.median(ends), np.percentile(ends, 90), ends.max()))
wend = collections.defaultdict(int)
for w, b in zip(warp, t1):
    wend[w] = max(wend[w], b)
we = np.array(list(wend.values())) / 1e3
print("warp finish us: min %.0f median %.0f max %.0f" % (we.min(), np.median(we), we.max()))
first = np.argsort(t0)[:8]
print("first chunks (sm, warp, t0, dur us):", [(int(sm[i]), int(warp[i]), int(t0[i] / 1e3), int(dur[i] / 1e3)) for i in first])
# rate per chunk: duration vs position in schedule
q = np.array_split(np.arange(len(tr)), 10)
print("mean chunk duration by schedule decile (us):", [int(dur[i].mean() / 1e3) for i in q])
sms = np.array(sorted(busy_by_sm))
print("per-SM chunks: min %d max %d" % (min(collections.Counter(sm).values()), max(collections.Counter(sm).values())))

S = (tr[:, 3] >> 40).astype(np.int64)
start = (tr[:, 3] & ((1 << 39) - 1)).astype(np.int64)
edge = (tr[:, 3] >> 39) & 1
rate = dur / (32 * S)      # ns per point
slow = np.argsort(-rate)[:6]
print("slowest chunks (id, sm, warp, start, S, edge, dur us, ns/pt, median ns/pt %.3f):" % np.median(rate))
for i in slow:
    print("   ", int(i), int(sm[i]), int(warp[i]), int(start[i]), int(S[i]), int(edge[i]), int(dur[i] / 1e3), round(float(rate[i]), 3))
