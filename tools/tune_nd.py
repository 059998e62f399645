"""Time a config (c3a/c3b/c4/c5) sweep for several k; one process per env setting."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2103_08825_b200.core import config_spec, CONFIGS
from paper_2103_08825_b200.plan import Plan
cfg = %r; dtype = %r
c = CONFIGS[cfg]; spec = config_spec(c["spec"]); dims = c["dims"]
npts = int(np.prod(dims))
box = np.random.default_rng(1).random(tuple(n + 2 for n in dims))
if dtype == "f32": box = box.astype(np.float32)
out = {}
for k in %s:
    with Plan(spec, dims, k=k, arith="fma", dtype=dtype) as p:
        p.upload(box); p.run(2 * k); t = p.run(%d)
        out[k] = round(npts * %d / (t.device_ms * 1e-3) / 1e9, 1)
print(json.dumps(out))
'''
cfg = sys.argv[1]
dtype = sys.argv[2]
ks = sys.argv[3]
settings = json.loads(sys.argv[4]) if len(sys.argv) > 4 else [{}]
T = int(sys.argv[5]) if len(sys.argv) > 5 else 24
for env in settings:
    e = dict(os.environ, **{k: str(v) for k, v in env.items()})
    r = subprocess.run([sys.executable, "-c", CHILD % (REPO, cfg, dtype, ks, T, T)], env=e, capture_output=True, text=True)
    print(cfg, dtype, json.dumps(env), r.stdout.strip() or r.stderr[-600:], flush=True)
