#!/usr/bin/env python
"""Benchmark of the fused D = A(BC) hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
  python bench.py --impl reference ...     (the reference CPU executor)

A "step" is one execution of the tile-fusion plan (wavefront 0 + wavefront
1) over one synthetic problem resident in HBM.  Default workload = BASELINE
configs[1] (cfg2: SpMM-SpMM fp64, 9-point stencil on 1024^2, cCol = 64).
Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA
events on the launching stream, the L2 flushed (256 MiB write) between steps
outside the events; barrier + synchronize around the timed region; the max
over ranks is reported.  One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective GFLOP/s of fused D=A(BC) and % of HBM/tensor roofline at 1/2/4/8 B200"
UNIT = "GFLOP/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink the workload (testing only)")
    ap.add_argument("--ct-size", type=int, default=2048)
    ap.add_argument("--cache-kb", type=float, default=1280.0)
    ap.add_argument("--workers", type=int, default=148, help="p of the pinned SchedulerConfig")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--flush-mib", type=int, default=256)
    ap.add_argument("--quick", action="store_true",
                    help="timed loop only (no clock tail / profile / e2e / cpu legs): for ncu")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the run."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def problem_bytes(w):
    s = np.dtype(w.dtype).itemsize
    a = 4 * (w.n + 1) + w.a.nnz * (4 + s)
    from paper_2407_00243_b200 import Csr

    b = (4 * (w.n + 1) + w.b.nnz * (4 + s)) if isinstance(w.b, Csr) else w.b.size * s
    return a + b + w.c.size * s, w.n * w.c_cols * s


# ---------------------------------------------------------------------------
def cpu_reference_time(w, args, workers, steps, warmup, budget_s=25.0):
    """Time the reference CPU executor (oracle/_ref, the unmodified reference
    compiled from its own sources) -- or the C port when _ref is absent --
    on the host cores.  Returns (seconds list, kind, sample text, sched secs)."""
    from oracle.oracle import (Oracle, RefProblem, Reference, SchedulerConfig as OCfg, have_reference,
                               ref_schedule_handle)
    from paper_2407_00243_b200 import Csr

    cfg = w.scheduler_config(num_workers=workers, ct_size=args.ct_size, cache_kb=args.cache_kb)
    ocfg = OCfg(**cfg.__dict__)
    a = (w.a.row_ptr, w.a.col_idx, w.a.values)
    b = (w.b.row_ptr, w.b.col_idx, w.b.values, w.b.n_cols) if isinstance(w.b, Csr) else w.b
    os.environ.setdefault("OMP_PROC_BIND", "close")  # main.cpp:56-57
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    times = []
    if have_reference():
        ref = Reference()
        t0 = time.perf_counter()
        sched = ref.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
        sched_s = time.perf_counter() - t0
        prob = RefProblem(ref, w.n, a, b, w.c, w.dtype)
        h = ref_schedule_handle(ref, sched)
        start = time.perf_counter()
        for k in range(warmup + steps):
            _, _, secs = prob.run(h, True, workers, out=False)
            if k >= warmup:
                times.append(secs)
            if time.perf_counter() - start > budget_s and len(times) >= 1:
                break
        kind = "reference"
        what = (f"reference fused_{'gemm' if w.op == 'gemm-spmm' else 'spmm'}_spmm on the full "
                f"{w.name} problem, workers={workers}, OMP_PROC_BIND=close; per-run steady_clock "
                f"time includes the executor's own zeroed D1/D allocation (kernels.hpp:97-98)")
    else:
        orc = Oracle()
        t0 = time.perf_counter()
        sched = orc.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
        sched_s = time.perf_counter() - t0
        start = time.perf_counter()
        for k in range(warmup + steps):
            t1 = time.perf_counter()
            orc.run(w.n, a, b, w.c, sched, w.dtype, workers=workers)
            if k >= warmup:
                times.append(time.perf_counter() - t1)
            if time.perf_counter() - start > budget_s and len(times) >= 1:
                break
        kind = "port"
        what = f"C port (oracle/tf_oracle.c) fused executor on the full {w.name} problem, workers={workers}"
    return times, kind, what, sched_s


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2407_00243_b200 import workloads as W

    w = W.make(args.config, scale=args.scale, device="cpu")
    cores = os.cpu_count() or 1
    times, kind, what, sched_s = cpu_reference_time(w, args, cores, args.steps, args.warmup,
                                                    budget_s=240.0)
    per = float(np.mean(times))
    value = w.flops() / per / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if w.dtype == np.float64 else "f32",
            "data": "synthetic (seeded generator with the BASELINE config's shape and distributions)",
            "impl": "reference",
            "config": {"workload": f"{args.config}: {w.description}", "n": w.n, "nnz_a": w.a.nnz,
                       "flops_per_step": w.flops(), "scheduler_seconds_cpu": sched_s},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": what + f"; {len(times)} timed runs after {args.warmup} warm-up"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, dist):
    import torch

    import paper_2407_00243_b200 as P
    from paper_2407_00243_b200 import workloads as W

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    sampler = ClockSampler(dev.index if dev.index is not None else 0)

    w = W.make(args.config, scale=args.scale)
    cfg = w.scheduler_config(num_workers=args.workers, ct_size=args.ct_size, cache_kb=args.cache_kb)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    torch.cuda.synchronize()
    sched = P.build_schedule(prob.a, cfg)  # GPU inspector, outside the timed region
    inspect_cold = sched.inspect_seconds  # includes first-call module loading
    sched = P.build_schedule(prob.a, cfg)
    out = torch.empty((w.n, w.c_cols), dtype=getattr(torch, w.dtype.name), device=dev)
    flush = torch.empty(args.flush_mib * (1 << 20) // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    plan = P.Plan(prob, sched) if rank == 0 else None
    dplan, bounds, halo = None, None, None
    if world > 1:
        # row-block partition of the same global problem (strong scaling)
        from paper_2407_00243_b200 import distributed as PD

        flat = sched.export()
        bounds = PD.tile_boundaries(flat, w.n, world)
        halo = PD.halo_plan(w.a.row_ptr, w.a.col_idx, flat, bounds, rank)
        eng = PD.GpuEngine(prob, sched, *bounds[rank])
        dplan = PD.DistributedPlan(eng, halo, dist, w.c_cols)
        launches = eng.launches + 3  # + gather, scatter, NCCL all-to-all

        def step():
            dplan.execute(out)
    else:
        launches = plan.launches

        def step():
            plan.execute(out, stream)

    def timed_loop(body, flush_between=True):
        for _ in range(args.warmup):
            if flush_between:
                flush.fill_(1.0)
            body()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for k in range(args.steps):
            if flush_between:
                flush.fill_(float(k))
            evs[k][0].record(stream)
            body()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        tot = float(sum(a.elapsed_time(b) for a, b in evs))
        if dist:
            t = torch.tensor([tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        return tot

    total_ms = timed_loop(step)
    mean_ms = total_ms / args.steps
    value = w.flops() * args.steps / (total_ms * 1e-3) / 1e9  # the global problem, all ranks

    if args.quick:
        sampler.stop()
        if rank == 0:
            print(json.dumps({"quick": True, "config": args.config, "n_gpus": world,
                              "ms_per_step": mean_ms, "value": value}))
        return

    # end to end: pinned host A,B,C -> HBM, execute, D -> pinned host, every step.
    # Steps are pipelined over two device input/output buffer sets and three
    # streams (H2D | compute | D2H), so step k+1's upload overlaps step k's
    # download (PCIe is full duplex); every step still moves all its inputs
    # and its result across PCIe inside the timed region.
    e2e = None
    if not args.no_e2e:
        e2e = _e2e_pipelined(args, w, prob, sched, bounds, rank, world, dist, dev, out, plan, dplan)

    if rank != 0:
        sampler.stop()
        return

    # a short same-kernel load tail (rank 0, local plan) so the sampler sees steady clocks
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        for _ in range(20):
            plan.execute(out, stream)
        torch.cuda.synchronize()
    clocks = sampler.stop()

    # roofline of the dominant stage of the single-GPU plan (CUDA events per stage)
    prof = []
    for _ in range(5):
        flush.fill_(2.0)
        prof.append(plan.profile(out, stream))
    stages = {}
    for rec in prof:
        for name, ms, by in rec:
            stages.setdefault(name, []).append((ms, by))
    stage_avg = {k: (float(np.mean([m for m, _ in v])), int(v[0][1])) for k, v in stages.items()}
    dom = max(stage_avg, key=lambda k: stage_avg[k][0])
    dom_ms, dom_bytes = stage_avg[dom]
    peak, peak_src = peaks()
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):  # committed ncu --set full capture of the same kernel
        rec = json.load(open(tp)).get(args.config, {}).get(dom)
        if rec:
            traffic = rec["dram_bytes"]
    step_bytes = sum(b for _, b in stage_avg.values())
    single_ms = sum(v[0] for v in stage_avg.values())

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        times, kind, what, sched_s = cpu_reference_time(w, args, cores, 7, 1)
        med = float(np.median(times))
        cpu = {"value": w.flops() / med / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": what + f"; median of {len(times)} runs after 1 warm-up",
               "ms_per_run": med * 1e3, "scheduler_seconds": sched_s}

    parallelism = "single GPU"
    if world > 1:
        parallelism = (f"row-block partition x{world} at tile boundaries; D1 halo via one NCCL "
                       f"all_to_all per step (rank-0 halo rows {dplan.halo_rows})")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if w.dtype == np.float64 else "f32",
        "data": "synthetic (seeded generator with the BASELINE config's shape and distributions; "
                "SuiteSparse corpus not available)",
        "config": {
            "workload": f"{args.config}: {w.description}", "n": w.n, "nnz_a": w.a.nnz,
            "b_cols": w.b_cols, "c_cols": w.c_cols, "flops_per_step": w.flops(),
            "schedule": {**cfg.__dict__, "tile_size": sched.tile_size,
                         "tiles": list(sched.num_tiles_per_wave),
                         "fused_ratio": sched.fused_ratio(),
                         "inspector_seconds_gpu": sched.inspect_seconds,
                         "inspector_seconds_gpu_cold": inspect_cold},
            "spill_rows": plan.spill_rows, "bytes_min": w.bytes_min(),
            "bytes_alg": w.bytes_alg(plan.spill_rows), "bytes_alg_stages": step_bytes,
            "step_hbm_frac_of_peak": (step_bytes / (single_ms * 1e-3) / 1e9) / peak,
            "stages_ms": {k: v[0] for k, v in stage_avg.items()},
            "kernels": plan.kernels(),
            "l2": f"flushed between timed steps ({args.flush_mib} MiB write, outside the events)",
            "parallelism": parallelism},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                     "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def _e2e_pipelined(args, w, prob, sched, bounds, rank, world, dist, dev, out, plan, dplan):
    import torch

    import paper_2407_00243_b200 as P

    sets = [prob, prob.clone()]
    host_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in prob.device_inputs()]
    if world > 1:
        from paper_2407_00243_b200 import distributed as PD

        own = torch.as_tensor(PD.owned_output_rows(sched.export(), bounds, rank), device=dev)
        flat = sched.export()
        engines = [dplan.engine, PD.GpuEngine(sets[1], sched, *bounds[rank])]
        dplans = [dplan, PD.DistributedPlan(engines[1], dplan.halo, dist, w.c_cols)]
        execs = [lambda o, i=i: dplans[i].execute(o) for i in range(2)]
        del flat
    else:
        own = None
        plans = [plan, P.Plan(sets[1], sched)]
        execs = [lambda o, i=i: plans[i].execute(o, torch.cuda.current_stream()) for i in range(2)]
    outs = [out, torch.empty_like(out)]
    nout = w.n if own is None else int(own.numel())
    host_out = [torch.empty((nout, w.c_cols), dtype=out.dtype, pin_memory=True) for _ in range(2)]
    h2d = int(sum(h.numel() * h.element_size() for h in host_in))
    d2h = int(host_out[0].numel() * host_out[0].element_size())
    s_h, s_c, s_d = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_h = [torch.cuda.Event() for _ in range(2)]
    ev_c = [torch.cuda.Event() for _ in range(2)]
    ev_d = [torch.cuda.Event() for _ in range(2)]

    def run(nsteps):
        for k in range(nsteps):
            b = k & 1
            with torch.cuda.stream(s_h):
                if k >= 2:
                    s_h.wait_event(ev_c[b])  # inputs of step k-2 consumed
                for hsrc, ddst in zip(host_in, sets[b].device_inputs()):
                    ddst.copy_(hsrc, non_blocking=True)
                ev_h[b].record(s_h)
            with torch.cuda.stream(s_c):
                s_c.wait_event(ev_h[b])
                if k >= 2:
                    s_c.wait_event(ev_d[b])  # output buffer of step k-2 drained
                execs[b](outs[b])
                ev_c[b].record(s_c)
            with torch.cuda.stream(s_d):
                s_d.wait_event(ev_c[b])
                src = outs[b] if own is None else outs[b].index_select(0, own)
                host_out[b].copy_(src, non_blocking=True)
                ev_d[b].record(s_d)

    run(max(2, args.warmup))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s_h)
    run(args.steps)
    s_h.wait_stream(s_d)
    t1.record(s_h)
    torch.cuda.synchronize()
    e_ms = t0.elapsed_time(t1)
    if dist:
        t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    return {"value": w.flops() * args.steps / (e_ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / args.steps,
            "path": ("pinned host A, B (aliased when B is A), C -> HBM, plan execute, D -> pinned host, "
                     "every step; steps pipelined over two buffer sets and H2D/compute/D2H streams; "
                     "max over ranks")}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    run_ours(args, rank, world, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
