"""Multi-GPU partition model on one GPU: for BASELINE configs at P = 2/4/8,
the cost-balanced cuts (tfg_partition_bounds), each rank's halo (D1 rows it
needs from other blocks), the NVLink exchange time vs the time to recompute
the halo from the resident B rows (the model tfg_halo_create uses to pick),
and the per-rank share of nonzeros.  usage: python tools/halo_model.py [cfg..]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00243_b200 as P  # noqa: E402
from paper_2407_00243_b200 import distributed as PD  # noqa: E402
from paper_2407_00243_b200 import workloads as W  # noqa: E402

names = sys.argv[1:] or ["cfg5", "cfg4", "cfg3", "cfg2", "cfg1"]
out = {}
for name in names:
    w = W.make(name)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    sched = P.build_schedule(prob.a, w.scheduler_config())
    rb = w.c_cols * np.dtype(w.dtype).itemsize
    out[name] = {}
    for world in (2, 4, 8):
        bounds = PD.partition_bounds(sched, w.a, w.b_cols, w.c_cols, w.dtype, w.op == "gemm-spmm", world)
        ranks = []
        for r in range(world):
            dp = PD.NativeDistributedPlan(prob, sched, bounds, r, PD.HALO_AUTO)
            lo, hi = bounds[r]
            ranks.append({"rows": [lo, hi], "nnz": int(w.a.row_ptr[hi] - w.a.row_ptr[lo]),
                          "halo_rows": dp.halo_rows, "halo_mb": dp.halo_rows * rb / 1e6,
                          "t_exchange_us": dp.t_exchange_us,
                          "t_recompute_us": dp.t_recompute_us if dp.t_recompute_us < 1e200 else None,
                          "mode": dp.mode_name})
            dp.close()
        nnz = [x["nnz"] for x in ranks]
        out[name][f"P{world}"] = {"max_halo_rows": max(x["halo_rows"] for x in ranks),
                                  "max_halo_mb": max(x["halo_mb"] for x in ranks),
                                  "nnz_imbalance": max(nnz) / (sum(nnz) / world),
                                  "modes": sorted({x["mode"] for x in ranks}), "ranks": ranks}
        print(name, world, out[name][f"P{world}"]["max_halo_mb"], out[name][f"P{world}"]["modes"],
              round(out[name][f"P{world}"]["nnz_imbalance"], 3), flush=True)
    del prob, sched
print(json.dumps(out))
