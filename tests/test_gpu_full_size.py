"""Full-size parity for the two BASELINE configurations that exercise fusion
(cfg3: GCN R-MAT 2^20, cfg5: R-MAT 2^23): the GPU inspector's schedule is
bit-identical to the oracle's (schedules_equal, support.hpp:150-165) at the
pinned configs the bench uses (p = 148 and p = 8, 1280 KB), and the GPU's D
(tensor-core 3xTF32 first op, fused tiles staged in shared memory, skewed
wavefront-1 gathers with segmented rows of up to 258k nonzeros) is within the
north-star max-norm tolerance (1e-5, fp32) of the oracle's D computed with the
reference's order on the host cores.  The measured errors are printed (run
with -s) and recorded in DESIGN.md."""
import os

import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import TOL, max_rel_err, schedules_equal
from oracle.oracle import SchedulerConfig

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_full_size_schedule_and_d(cuda, oracle, name):
    from paper_2407_00243_b200 import workloads as W

    w = W.make(name)  # full BASELINE size
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    keep = None
    for p in (148, 8):
        cfg = w.scheduler_config(num_workers=p)
        ocfg = SchedulerConfig(**cfg.__dict__)
        want_s = oracle.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
        got_s = P.build_schedule(prob.a, cfg)
        assert schedules_equal(got_s.export(), want_s), (name, p)
        if p == 148:
            keep = (got_s, want_s)
    got_s, want_s = keep
    got = P.Plan(prob, got_s).execute().cpu().numpy()
    unfused = P.Plan(prob, None).execute().cpu().numpy()
    want = oracle.run(w.n, (w.a.row_ptr, w.a.col_idx, w.a.values), w.b, w.c, want_s, w.dtype,
                      workers=os.cpu_count() or 1)
    err = max_rel_err(got, want)
    err_u = max_rel_err(unfused, want)
    print(f"\n[parity] {name} full size: max|D_gpu - D_ref| / max|D_ref| = {err:.3e} (fused), "
          f"{err_u:.3e} (unfused); max|D_ref| = {np.abs(want).max():.4g}; "
          f"fused_ratio = {got_s.fused_ratio():.4f}")
    assert err <= TOL[4] and err_u <= TOL[4]
    assert np.isfinite(got).all()
