"""Sweep environment knobs on a BASELINE config and print per-stage device
times; each setting runs in a fresh process.
usage: python tools/spmm_sweep.py cfg5 @TFG_TC_RING=4,@TFG_TC_RING=5+@TFG_W1_SORT=0"""
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
res = {}
for k in range(12):
    fl.fill_(k); r = plan.profile(out)
    if k >= 2:
        for name, ms, by in r: res.setdefault(name, []).append((ms, by))
print(json.dumps({k: [float(np.median([m for m, _ in v])), v[0][1] / float(np.median([m for m, _ in v])) / 1e6] for k, v in res.items()}))
'''


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["@TFG_DEBUG=0"]
    for spec in variants:
        env = dict(os.environ)
        # "@A=1+@B=2" sets several knobs for one run
        parts = spec.split("+")
        for extra in [q for q in parts if q.startswith("@")]:  # "@VAR=value": any env knob
            k_, v_ = extra[1:].split("=", 1)
            env[k_] = v_
        r = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True, env=env)
        print(cfg, "variant", spec, r.stdout.strip() or r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
