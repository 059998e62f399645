"""H2D / D2H throughput of a C5 plan upload/download vs plain 1D copies (development tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
spec = config_spec("c5")
dims = (768, 768, 768)
p = Plan(spec, dims, k=2)
host = torch.empty(p.shape, dtype=torch.float64, pin_memory=True)
host.numpy()[...] = 1.0
out = torch.empty_like(host, pin_memory=True)
nb = host.numel() * 8
for name, fn in (("plan.upload (2D pitched)", lambda: p.upload(host.numpy())),
                 ("plan.download (2D pitched)", lambda: p.download(out.numpy()))):
    fn()
    t0 = time.perf_counter(); fn(); dt = time.perf_counter() - t0
    print(f"{name}: {nb / dt / 1e9:.1f} GB/s")
dev = torch.empty(host.numel(), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for name, fn in (("torch 1D H2D", lambda: dev.copy_(host.view(-1), non_blocking=True)),
                 ("torch 1D D2H", lambda: out.view(-1).copy_(dev, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {nb / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    dev.copy_(host.view(-1), non_blocking=True)
with torch.cuda.stream(s2):
    out.view(-1).copy_(dev, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"concurrent H2D+D2H: {2 * nb / dt / 1e9:.1f} GB/s total")
