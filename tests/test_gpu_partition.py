"""GPU partition plans (tfg_plan_create_partition) and the halo pack/unpack
kernels, with P ranks emulated sequentially in one process on one GPU (the
NCCL all-to-all is replaced by direct device copies between the emulated
ranks' D1 buffers; the NCCL path itself is covered by the gloo tests)."""
import numpy as np
import pytest
import torch

import paper_2407_00243_b200 as P
from helpers import TOL, max_rel_err
from oracle.oracle import SchedulerConfig
from paper_2407_00243_b200 import distributed as PD

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 4), ("cfg4", 8), ("cfg3", 4), ("cfg1", 3)])
def test_emulated_ranks_match_oracle(cuda, oracle, name, world):
    from paper_2407_00243_b200 import workloads as W

    scale = {"cfg1": 1 / 4, "cfg2": 1 / 16, "cfg3": 1 / 64, "cfg4": 1 / 64}[name]
    w = W.make(name, scale=scale)
    cfg = w.scheduler_config(num_workers=8)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    sched = P.build_schedule(prob.a, cfg)
    flat = sched.export()
    bounds = PD.tile_boundaries(flat, w.n, world)
    engines = [PD.GpuEngine(prob, sched, *bounds[r], reference_bits=True) for r in range(world)]
    halos = [PD.halo_plan(w.a.row_ptr, w.a.col_idx, flat, bounds, r) for r in range(world)]
    outs = [torch.full((w.n, w.c_cols), float("nan"), dtype=engines[0].torch_dtype, device="cuda")
            for _ in range(world)]
    for r in range(world):
        engines[r].stage0(outs[r])
    moved = 0
    for r in range(world):
        for s in range(world):
            rows = torch.as_tensor(halos[r].recv[s], dtype=torch.int32, device="cuda")
            if rows.numel():
                engines[r].scatter_d1(rows, engines[s].gather_d1(rows))
                moved += rows.numel()
    for r in range(world):
        engines[r].stage1(outs[r])
    torch.cuda.synchronize()
    got = np.full((w.n, w.c_cols), np.nan)
    for r in range(world):
        rows = PD.owned_output_rows(flat, bounds, r)
        got[rows] = outs[r].cpu().numpy()[rows]
    assert not np.isnan(got).any()
    ocfg = SchedulerConfig(**cfg.__dict__)
    osched = oracle.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
    ob = w.b if not isinstance(w.b, P.Csr) else (w.b.row_ptr, w.b.col_idx, w.b.values, w.b.n_cols)
    want = oracle.run(w.n, (w.a.row_ptr, w.a.col_idx, w.a.values), ob, w.c, osched, w.dtype, workers=8)
    assert max_rel_err(got, want) <= TOL[np.dtype(w.dtype).itemsize]
    if w.op == "spmm-spmm":
        assert np.array_equal(got, want)
    assert moved > 0
