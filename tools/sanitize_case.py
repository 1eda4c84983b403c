"""Small end-to-end case for compute-sanitizer (one tool per gpurun call):
inspector, band SpMM (TMA + mbarrier), strip/segment SpMM, pipelined GEMM,
fused dense-B tiles, checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00243_b200 as P  # noqa: E402
from oracle.oracle import Oracle, SchedulerConfig  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

orc = Oracle()
fails = 0
for name, scale in [("cfg2", 1 / 256), ("cfg3", 1 / 512), ("cfg1", 1 / 64)]:
    w = W.make(name, scale=scale)
    cfg = w.scheduler_config(num_workers=16)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    got = P.Plan(prob, P.build_schedule(prob.a, cfg)).execute().cpu().numpy()
    torch.cuda.synchronize()
    osched = orc.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, SchedulerConfig(**cfg.__dict__))
    ob = w.b if not isinstance(w.b, P.Csr) else (w.b.row_ptr, w.b.col_idx, w.b.values, w.b.n_cols)
    want = orc.run(w.n, (w.a.row_ptr, w.a.col_idx, w.a.values), ob, w.c, osched, w.dtype)
    err = np.abs(got - want).max() / np.abs(want).max()
    tol = 1e-12 if w.dtype == np.float64 else 1e-5
    print(name, w.n, "max_rel_err", err, "ok" if err <= tol else "FAIL")
    fails += err > tol
sys.exit(1 if fails else 0)
