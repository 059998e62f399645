"""C1 per-sweep device time under three enqueue styles (development tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
spec = config_spec("c1")
n, T, R = 1 << 20, 64, 300
box = np.random.default_rng(1).random(n + 2)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
p = Plan(spec, (n,), k=64); p.set_stream(st.cuda_stream); p.upload(box)
for _ in range(20): p.launch(T)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(R): p.launch(T)
e1.record(st); torch.cuda.synchronize()
print("python loop of launch(T):", e0.elapsed_time(e1) / R * 1e3, "us/sweep")
e0.record(st); p.launch_repeat(T, R); e1.record(st); torch.cuda.synchronize()
print("launch_repeat (events):", e0.elapsed_time(e1) / R * 1e3, "us/sweep; mean event", np.mean(p.repeat_times()) * 1e3)
t = p.run(T * R)
print("one run(T*R):", t.device_ms / R * 1e3, "us/sweep", t.launches)
t = p.run(T * R)
print("one run(T*R) again:", t.device_ms / R * 1e3, "us/sweep", t.launches)
