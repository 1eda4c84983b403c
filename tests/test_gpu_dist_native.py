"""The native multi-GPU path (include/tfg.h multi-GPU section) on one B200.

Every rank of a partition runs in this process one after another
(tfg_plan_execute_dist_emulated: the NCCL transfer replaced by device copies
between the ranks' halo buffers, no kernel waits on another), so the cuts,
the device-built halo lists, the exchange / recompute choice and the split
of wavefront 1 into local-only and halo rows are all checked against the
oracle.  The NCCL binding itself is exercised with a one-rank communicator.
"""
import numpy as np
import pytest
import torch

import paper_2407_00243_b200 as P
from helpers import TOL, max_rel_err
from oracle.oracle import SchedulerConfig
from paper_2407_00243_b200 import distributed as PD

pytestmark = pytest.mark.gpu


def oracle_d(oracle, w, cfg):
    osched = oracle.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, SchedulerConfig(**cfg.__dict__))
    ob = w.b if not isinstance(w.b, P.Csr) else (w.b.row_ptr, w.b.col_idx, w.b.values, w.b.n_cols)
    return oracle.run(w.n, (w.a.row_ptr, w.a.col_idx, w.a.values), ob, w.c, osched, w.dtype, workers=8)


def run_emulated(w, cfg, world, mode, bits=False):
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    sched = P.build_schedule(prob.a, cfg)
    bounds = PD.partition_bounds(sched, w.a, w.b_cols, w.c_cols, w.dtype, w.op == "gemm-spmm", world)
    assert bounds[0][0] == 0 and bounds[-1][1] == w.n
    dps = [PD.NativeDistributedPlan(prob, sched, bounds, r, mode, reference_bits=bits)
           for r in range(world)]
    outs = [torch.full((w.n, w.c_cols), float("nan"), dtype=getattr(torch, w.dtype.name), device="cuda")
            for _ in range(world)]
    PD.execute_emulated(dps, outs)
    torch.cuda.synchronize()
    flat = sched.export()
    got = np.full((w.n, w.c_cols), np.nan)
    for r in range(world):
        rows = PD.owned_output_rows(flat, bounds, r)
        got[rows] = outs[r].cpu().numpy()[rows]
    return got, dps, bounds


@pytest.mark.parametrize("name,world,mode", [
    ("cfg1", 3, PD.HALO_EXCHANGE), ("cfg1", 4, PD.HALO_RECOMPUTE),
    ("cfg3", 4, PD.HALO_EXCHANGE), ("cfg3", 4, PD.HALO_AUTO),
    ("cfg5", 8, PD.HALO_AUTO), ("cfg5", 2, PD.HALO_EXCHANGE),
    ("cfg2", 4, PD.HALO_EXCHANGE), ("cfg4", 8, PD.HALO_AUTO)])
def test_native_partition_matches_oracle(cuda, oracle, name, world, mode):
    from paper_2407_00243_b200 import workloads as W

    scale = {"cfg1": 1 / 4, "cfg2": 1 / 16, "cfg3": 1 / 32, "cfg4": 1 / 64, "cfg5": 1 / 64}[name]
    w = W.make(name, scale=scale)
    cfg = w.scheduler_config(num_workers=8)
    got, dps, _ = run_emulated(w, cfg, world, mode)
    assert not np.isnan(got).any()
    want = oracle_d(oracle, w, cfg)
    assert max_rel_err(got, want) <= TOL[np.dtype(w.dtype).itemsize]
    if mode == PD.HALO_AUTO:
        expect = PD.HALO_RECOMPUTE if w.op == "gemm-spmm" else PD.HALO_EXCHANGE
        assert all(d.mode == expect for d in dps), [d.mode_name for d in dps]
    else:
        assert all(d.mode == mode for d in dps)
    assert sum(d.halo_rows for d in dps) > 0
    assert sum(d.halo_rows for d in dps) == sum(d.send_rows for d in dps)


def test_native_partition_reference_bits(cuda, oracle):
    """SpMM-SpMM with reference bits: the partitioned result is bit-exact."""
    from paper_2407_00243_b200 import workloads as W

    w = W.make("cfg2", scale=1 / 16)
    cfg = w.scheduler_config(num_workers=8)
    got, _, _ = run_emulated(w, cfg, 4, PD.HALO_EXCHANGE, bits=True)
    assert np.array_equal(got, oracle_d(oracle, w, cfg))


def test_cuts_balance_work_not_rows(cuda):
    """R-MAT rows differ a lot in length: the cost-balanced cuts give ranks
    similar nonzero counts (row-count cuts would not)."""
    from paper_2407_00243_b200 import workloads as W

    w = W.make("cfg5", scale=1 / 16)
    sched = P.build_schedule(w.a, w.scheduler_config())
    bounds = PD.partition_bounds(sched, w.a, w.b_cols, w.c_cols, w.dtype, True, 4)
    nnz = [int(w.a.row_ptr[hi] - w.a.row_ptr[lo]) for lo, hi in bounds]
    assert max(nnz) < 1.35 * (sum(nnz) / 4), nnz


def test_nccl_one_rank_communicator(cuda):
    """The NCCL binding (resolved in-process) builds a communicator and the
    native step runs through tfg_plan_execute_dist with it (world 1: no
    peers, the plan's own result)."""
    from paper_2407_00243_b200 import workloads as W

    w = W.make("cfg1", scale=1 / 8)
    cfg = w.scheduler_config(num_workers=8)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    sched = P.build_schedule(prob.a, cfg)
    comm = PD.nccl_comm(None, 1, 0)
    try:
        dp = PD.NativeDistributedPlan(prob, sched, [(0, w.n)], 0, PD.HALO_EXCHANGE, comm=comm)
        out = torch.empty((w.n, w.c_cols), dtype=torch.float64, device="cuda")
        got = dp.execute(out).cpu().numpy()
        want = P.Plan(prob, sched).execute().cpu().numpy()
        assert np.array_equal(got, want)
        dp.close()
    finally:
        PD.nccl_comm_destroy(comm)
