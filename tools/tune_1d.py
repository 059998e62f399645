"""Time the C2 sweep under several env knobs (one subprocess per setting)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2103_08825_b200.core import config_spec
from paper_2103_08825_b200.plan import Plan
spec = config_spec("c2"); n = 1 << 26
box = np.random.default_rng(1).random(n + 4)
out = {}
for k in %s:
    with Plan(spec, (n,), k=k, arith="fma") as p:
        p.upload(box); p.run(64); t = p.run(%d)
        out[k] = round(n * %d / (t.device_ms * 1e-3) / 1e9, 1)
print(json.dumps(out))
'''
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
ks = sys.argv[2] if len(sys.argv) > 2 else "[8, 16]"
T = 400
for env in settings:
    e = dict(os.environ, **{k: str(v) for k, v in env.items()})
    r = subprocess.run([sys.executable, "-c", CHILD % (REPO, ks, T, T)], env=e, capture_output=True, text=True)
    print(json.dumps(env), r.stdout.strip() or r.stderr[-400:], flush=True)
