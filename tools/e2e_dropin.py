"""Time the drop-in by-value call (tfg_run_host) on one BASELINE config, with
TFG_DEBUG=1 printing the call's internal timeline.
usage: [TFG_DEBUG=1] python tools/e2e_dropin.py cfg5 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.make(name)
prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
sched = P.build_schedule(prob.a, w.scheduler_config())
del prob
r = bench.e2e_dropin(w, sched, steps, 1)
print(name, "drop-in e2e ms/step", round(r["ms_per_step"], 2))
