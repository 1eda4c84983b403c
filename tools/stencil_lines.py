"""Time the grid-stencil kernel variants (TFG_STENCIL_LINES / NW / CTAS / NS /
ZC, read at plan creation) on cfg4 (or cfg2) in one process; D compared with
the first variant.  usage: python tools/stencil_lines.py cfg4 "LINES=1;LINES=2;LINES=2,NW=2,CTAS=4" [out.json]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
variants = (sys.argv[2] if len(sys.argv) > 2 else "LINES=1;LINES=2").split(";")
w = W.make(name)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
sched = P.build_schedule(prob.a, w.scheduler_config())
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
fl = torch.empty(64 << 20, device="cuda")
ref, res = None, {}
for spec in variants:
    for k in list(os.environ):
        if k.startswith("TFG_STENCIL_"):
            del os.environ[k]
    for kv in spec.split(","):
        k, v = kv.split("=")
        os.environ["TFG_STENCIL_" + k] = v
    plan = P.Plan(prob, sched)
    out.fill_(float("nan"))
    plan.execute(out)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    err = float((out - ref).abs().max() / ref.abs().max())
    st = {}
    for k in range(10):
        fl.fill_(k)
        r = plan.profile(out)
        if k >= 2:
            for nm, ms, by in r:
                st.setdefault(nm, []).append(ms)
    res[spec] = {"stages_ms": {k: float(np.median(v)) for k, v in st.items()}, "max_rel_diff_vs_first": err,
                 "bitwise": bool(torch.equal(out, ref))}
    print(spec, json.dumps(res[spec]), flush=True)
    del plan
if len(sys.argv) > 3:
    json.dump({"config": name, "runs": res}, open(sys.argv[3], "w"), indent=1)
