"""Tile / ring / occupancy sweep of the grid-stencil kernel on a BASELINE
config (knobs read at plan creation): python tools/stencil_sweep.py cfg4"""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = W.make(name)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
s = P.build_schedule(prob.a, w.scheduler_config())
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = []
for nw, ctas, ns, zc in itertools.product(["4", "8"], ["1", "2", "3", "4"], ["0", "3", "5"], ["0", "6", "12", "32"]):
    for k, v in (("TFG_STENCIL_NW", nw), ("TFG_STENCIL_CTAS", ctas), ("TFG_STENCIL_NS", ns),
                 ("TFG_STENCIL_ZC", zc)):
        os.environ[k] = v
    try:
        plan = P.Plan(prob, s)
    except Exception as e:  # noqa: BLE001
        continue
    ts = []
    for _ in range(6):
        flush.fill_(1.0)
        st = plan.profile(out)
        ts.append(st[0][1])  # first-op pass (the same kernel as wave 1)
    ts.sort()
    res.append({"nw": nw, "ctas": ctas, "ns": ns, "zc": zc, "pass_ms": ts[len(ts) // 2]})
    print(res[-1], flush=True)
    del plan
res.sort(key=lambda r: r["pass_ms"])
print(json.dumps({"config": name, "best": res[:5], "all": res}))
