"""Build one BASELINE workload's plan and execute it a few times (a target for
ncu captures).  usage: python tools/run_plan.py cfg5 [reps] [scale]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
w = W.make(name, scale=scale)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
plan = P.Plan(prob, P.build_schedule(prob.a, w.scheduler_config()))
out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device="cuda")
for _ in range(reps):
    plan.execute(out)
torch.cuda.synchronize()
print("ok", name)
