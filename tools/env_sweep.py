"""Time plan-creation knobs (TFG_* environment variables read when a plan is
built: TFG_STENCIL_NW / CTAS / NS / ZC, TFG_WINDOW / WINDOW_RPC / WINDOW_HALO,
TFG_W1_SORT ...) on one BASELINE config in one process: per-stage device
times, D compared with the first variant.
usage: python tools/env_sweep.py cfg1 "WINDOW=0;WINDOW=1;WINDOW=1,WINDOW_RPC=32" [out.json]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
variants = (sys.argv[2] if len(sys.argv) > 2 else "DEBUG=0").split(";")
w = W.make(name)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
sched = P.build_schedule(prob.a, w.scheduler_config())
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
fl = torch.empty(64 << 20, device="cuda")
ref, res, set_keys = None, {}, []
for spec in variants:
    for k in set_keys:
        os.environ.pop(k, None)
    set_keys = []
    for kv in spec.split(","):
        k, v = kv.split("=")
        os.environ["TFG_" + k] = v
        set_keys.append("TFG_" + k)
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
    res[spec] = {"stages_ms": {k: float(np.median(v)) for k, v in st.items()}, "kernels": plan.kernels(),
                 "max_rel_diff_vs_first": err,
                 "bitwise": bool(torch.equal(out, ref))}
    print(spec, json.dumps(res[spec]), flush=True)
    del plan
if len(sys.argv) > 3:
    json.dump({"config": name, "runs": res}, open(sys.argv[3], "w"), indent=1)
