"""Benchmark report rows in the reference's format.

Mirrors `bench::Row` and its CSV / JSON emitters (bench.hpp:37-55,
bench.cpp:460-513) and `run_rows` (bench.cpp:221-316): median of `runs`
after `warmup` (bench.cpp:161-175), GFLOP/s from `theoretical_flops`
(bench.cpp:152-159), and `runs_to_amortize` = scheduler seconds / per-run
saving of fused over unfused (bench.cpp:309-314) -- here for the GPU
inspector and the GPU executors (device time per run, CUDA events).
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

HEADER = ("matrix,n,nnz,op,variant,precision,bcol,ccol,workers,runs,median_seconds,gflops,"
          "fused_ratio,scheduler_seconds,runs_to_amortize,replicated_rows,binding")


@dataclass
class Row:
    matrix: str
    n: int
    nnz: int
    op: str
    variant: str
    precision: str
    bcol: int
    ccol: int
    workers: int
    runs: int
    median_seconds: float
    gflops: float
    fused_ratio: float = -1.0
    scheduler_seconds: float = -1.0
    runs_to_amortize: float = -1.0
    replicated_rows: int = -1
    binding: str = "gpu"


def _fmt(x: float) -> str:
    if x < 0:
        return ""
    if math.isinf(x):
        return "inf"
    return f"{x:.6g}"


def rows_to_csv(rows) -> str:
    out = [HEADER]
    for r in rows:
        out.append(",".join([r.matrix, str(r.n), str(r.nnz), r.op, r.variant, r.precision,
                             str(r.bcol), str(r.ccol), str(r.workers), str(r.runs),
                             _fmt(r.median_seconds), _fmt(r.gflops), _fmt(r.fused_ratio),
                             _fmt(r.scheduler_seconds), _fmt(r.runs_to_amortize),
                             "" if r.replicated_rows < 0 else str(r.replicated_rows), r.binding]))
    return "\n".join(out) + "\n"


def rows_to_json(rows) -> str:
    arr = []
    for r in rows:
        d = asdict(r)
        for k in ("fused_ratio", "scheduler_seconds", "replicated_rows"):
            if d[k] < 0:
                d[k] = None
        if r.runs_to_amortize < 0:
            d["runs_to_amortize"] = None
        elif math.isinf(r.runs_to_amortize):
            d["runs_to_amortize"] = "inf"
        arr.append(d)
    return json.dumps(arr, indent=2) + "\n"


def median_seconds(fn, runs=7, warmup=1):
    """bench.cpp:161-175 with device time (CUDA events around each run)."""
    import torch

    for _ in range(warmup):
        fn()
    times = []
    for _ in range(runs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    times.sort()
    m = len(times) // 2
    return times[m] if len(times) % 2 else 0.5 * (times[m - 1] + times[m])


def run_rows(workload, cfg, runs=7, warmup=1, name=None):
    """GPU fused and unfused rows for one workload (run_rows, bench.cpp:221-316)."""
    import time

    import torch

    from . import tilefuse as P

    prob = P.DeviceProblem(workload.a, workload.b, workload.c, workload.dtype)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sched = P.build_schedule(prob.a, cfg)
    sched_s = time.perf_counter() - t0
    fused = P.Plan(prob, sched)
    unfused = P.Plan(prob, None)
    out = torch.empty((workload.n, workload.c_cols), dtype=getattr(torch, workload.dtype.name),
                      device="cuda")
    flops = workload.flops()
    prec = "dp" if workload.dtype == np.float64 else "sp"
    rows = []
    for variant, plan in (("fused", fused), ("unfused", unfused)):
        med = median_seconds(lambda: plan.execute(out), runs, warmup)
        r = Row(name or workload.name, workload.n, workload.a.nnz, workload.op, variant, prec,
                workload.b_cols, workload.c_cols, cfg.num_workers, runs, med, flops / med / 1e9)
        if variant == "fused":
            r.fused_ratio = sched.fused_ratio()
            r.scheduler_seconds = sched_s
        rows.append(r)
    saved = rows[1].median_seconds - rows[0].median_seconds
    rows[0].runs_to_amortize = sched_s / saved if saved > 0 else math.inf
    return rows
