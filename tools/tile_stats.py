import sys, os
sys.path.insert(0, os.getcwd())
import paper_2407_00243_b200 as P
from paper_2407_00243_b200 import workloads as W
for name in sys.argv[1:]:
    w = W.make(name)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    plan = P.Plan(prob, P.build_schedule(prob.a, w.scheduler_config()))
    print(name, w.n, flush=True)
