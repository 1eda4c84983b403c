"""Time the GPU inspector on a BASELINE config (run under ncu for the
per-kernel launch list).  usage: python tools/inspect_time.py cfg3 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.make(name)
d = P.DeviceCsr(w.a)
cfg = w.scheduler_config()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = P.build_schedule(d, cfg)
    print(name, "inspector", round(time.perf_counter() - t0, 4), "s", s.num_tiles_per_wave, flush=True)
