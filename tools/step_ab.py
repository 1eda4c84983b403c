"""A/B of environment knobs the library reads once per process: one fresh
process per setting (joined with +), per-stage and whole-step medians, L2
flushed between runs, and the sum of D as a cheap identity check.
usage: python tools/step_ab.py cfg5 TFG_ZERO_EARLY=1 TFG_ZERO_EARLY=0 ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2407_00243_b200 as P
from paper_2407_00243_b200 import workloads as W
w = W.make(%r)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
plan = P.Plan(prob, P.build_schedule(prob.a, w.scheduler_config()))
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
fl = torch.empty(64 << 20, device="cuda")
res, ts = {}, []
for k in range(14):
    fl.fill_(k); r = plan.profile(out)
    if k >= 2:
        for name, ms, by in r: res.setdefault(name, []).append(ms)
for k in range(24):
    fl.fill_(k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.execute(out); e1.record(); torch.cuda.synchronize()
    if k >= 4: ts.append(e0.elapsed_time(e1))
print(json.dumps({"stages_ms": {k: round(float(np.median(v)), 4) for k, v in res.items()},
                  "step_ms": round(float(np.median(ts)), 4), "step_min_ms": round(min(ts), 4),
                  "sum": float(out.double().sum().item())}))
'''
cfg = sys.argv[1]
for spec in sys.argv[2:]:
    env = dict(os.environ)
    for kv in spec.split("+"):
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True, env=env)
    print(cfg, spec, r.stdout.strip() or r.stderr[-400:], flush=True)
