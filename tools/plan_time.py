import sys, time
sys.path.insert(0, '/root/repo')
import paper_2407_00243_b200 as P
from paper_2407_00243_b200 import workloads as W
import torch
for name in sys.argv[1:]:
    w = W.make(name)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    s = P.build_schedule(prob.a, w.scheduler_config())
    torch.cuda.synchronize()
    t = time.perf_counter(); plan = P.Plan(prob, s); torch.cuda.synchronize()
    print(name, 'plan create s', round(time.perf_counter() - t, 3), plan.kernels(), flush=True)
