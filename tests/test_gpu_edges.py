"""Edge cases the reference's tests exercise (empty rows, n = 1, dense rows,
width-1 tiles, schedules imported from the reference inspector) on the GPU."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import TOL, golden_cfg, golden_sched, load, max_rel_err, to_product_cfg
from oracle.oracle import SchedulerConfig

pytestmark = pytest.mark.gpu


def test_reference_schedules_execute_bit_exact(cuda, oracle):
    """Golden schedules built by the reference inspector, imported into
    libtfg and executed: SpMM-SpMM bit-identical to the oracle."""
    z = load("schedules.npz")
    rng = np.random.default_rng(3)
    for key in list(z["keys"])[:40]:
        rp, ci = z[f"{key}/row_ptr"], z[f"{key}/col_idx"]
        n = rp.size - 1
        v = rng.uniform(-1, 1, ci.size)
        c = rng.uniform(-1, 1, (n, 8))
        flat = golden_sched(z, key)
        s = P.import_schedule(flat)
        a = P.Csr(n, n, rp, ci, v)
        got = P.run(a, a, c, s)
        want = oracle.run(n, (rp, ci, v), (rp, ci, v, n), c, flat)
        assert np.array_equal(got, want), key


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_degenerate_shapes(cuda, oracle, dt):
    size = np.dtype(dt).itemsize
    # n = 1
    a = P.Csr(1, 1, [0, 1], [0], [2.0])
    d = P.fused_gemm_spmm(a, np.array([[3.0]]), np.array([[4.0, 5.0]]), dtype=dt)
    assert d.tolist() == [[24.0, 30.0]]
    # all rows empty
    a = P.Csr(50, 50, np.zeros(51, np.int32), np.zeros(0, np.int32), np.zeros(0))
    b = np.ones((50, 3))
    c = np.ones((3, 4))
    assert not P.fused_gemm_spmm(a, b, c, dtype=dt).any()
    s = P.build_schedule(a, P.SchedulerConfig(ct_size=8, num_workers=3))
    assert s.fused_ratio() == 0.5  # every empty row fuses into its own tile
    # half the rows empty, SpMM-SpMM, odd column count (generic kernels)
    rng = np.random.default_rng(1)
    n = 301
    rows = [np.sort(rng.choice(n, rng.integers(1, 9), replace=False)) if i % 2 else np.zeros(0, int)
            for i in range(n)]
    rp = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int32)
    ci = np.concatenate(rows).astype(np.int32)
    v = rng.uniform(-1, 1, ci.size)
    a = P.Csr(n, n, rp, ci, v)
    c = rng.uniform(-1, 1, (n, 7))
    cfg = SchedulerConfig(ct_size=16, num_workers=5, cache_size_words=300, b_is_dense=False)
    osched = oracle.build_schedule(n, n, rp, ci, cfg)
    want = oracle.run(n, (rp, ci, v), (rp, ci, v, n), c, osched, dt)
    got = P.run(a.astype(dt), a.astype(dt), c.astype(dt), P.build_schedule(a, to_product_cfg(cfg)), dt)
    assert np.array_equal(got, want)
    assert max_rel_err(got, want) <= TOL[size]


def test_dense_and_long_rows_spmm_spmm(cuda, oracle):
    """A dense 6000-wide row (segmented path) next to banded rows, B = A."""
    n = 6000
    rng = np.random.default_rng(2)
    rows = [np.arange(n)] + [np.arange(max(0, i - 2), min(n, i + 3)) for i in range(1, n)]
    rp = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int32)
    ci = np.concatenate(rows).astype(np.int32)
    v = rng.uniform(-1, 1, ci.size)
    a = P.Csr(n, n, rp, ci, v)
    c = rng.uniform(-1, 1, (n, 64))
    for ct, budget in [(2048, 163840), (512, 10 ** 12)]:
        cfg = SchedulerConfig(ct_size=ct, num_workers=16, cache_size_words=budget, b_is_dense=False,
                              c_cols=64, b_cols=n)
        osched = oracle.build_schedule(n, n, rp, ci, cfg)
        want = oracle.run(n, (rp, ci, v), (rp, ci, v, n), c, osched)
        got = P.run(a, a, c, P.build_schedule(a, to_product_cfg(cfg)))
        assert max_rel_err(got, want) <= 1e-12
        # rows that neither are the segmented row nor read its D1 row
        # (columns 0..2 of the band touch row 0) are bit-exact
        assert np.array_equal(got[3:], want[3:])


def test_width_one_tiles_and_tiny_budget(cuda, oracle):
    rp, ci, v = oracle.gen_random_sparse(400, 0.05, 17)
    cfg = SchedulerConfig(ct_size=64, num_workers=8, cache_size_words=1, b_cols=4, c_cols=4)
    osched = oracle.build_schedule(400, 400, rp, ci, cfg)
    a = P.Csr(400, 400, rp, ci, v)
    s = P.build_schedule(a, to_product_cfg(cfg))
    from helpers import schedules_equal

    assert schedules_equal(s.export(), osched)
    rng = np.random.default_rng(0)
    b, c = rng.uniform(-1, 1, (400, 4)), rng.uniform(-1, 1, (4, 4))
    want = oracle.run(400, (rp, ci, v), b, c, osched)
    assert max_rel_err(P.run(a, b, c, s), want) <= 1e-12


def test_plan_reuse_with_new_values(cuda, oracle):
    """A plan reads the live CSR values: updating A's values in place (same
    pattern) and re-executing gives the new product."""
    import torch

    rp, ci, v = oracle.gen_banded(3000, 4)
    a = P.Csr(3000, 3000, rp, ci, v)
    rng = np.random.default_rng(5)
    c = rng.uniform(-1, 1, (3000, 64))
    prob = P.DeviceProblem(a, a, c)
    plan = P.Plan(prob, P.build_schedule(a, P.SchedulerConfig(b_is_dense=False, c_cols=64)))
    d0 = plan.execute().cpu().numpy()
    v2 = rng.uniform(-1, 1, v.size)
    prob.a.values.copy_(torch.from_numpy(v2))
    prob.b.values.copy_(torch.from_numpy(v2))
    d1 = plan.execute().cpu().numpy()
    want = oracle.run(3000, (rp, ci, v2), (rp, ci, v2, 3000), c, None)
    assert np.array_equal(d1, want) and not np.array_equal(d0, d1)


@pytest.mark.parametrize("cc", [64, 128])
def test_skewed_rows_spmm_spmm_bit_exact(cuda, oracle, cc):
    """Power-law (R-MAT) rows take the ring-gather kernel; SpMM-SpMM stays
    bit-identical to the reference order."""
    from paper_2407_00243_b200 import workloads as W

    w = W.make("cfg5", scale=1 / 256)
    a = w.a.astype(np.float64)
    rng = np.random.default_rng(4)
    c = rng.uniform(-1, 1, (a.n_rows, cc))
    cfg = SchedulerConfig(ct_size=2048, num_workers=148, cache_size_words=163840, b_is_dense=False,
                          c_cols=cc, b_cols=a.n_rows)
    osched = oracle.build_schedule(a.n_rows, a.n_rows, a.row_ptr, a.col_idx, cfg)
    want = oracle.run(a.n_rows, (a.row_ptr, a.col_idx, a.values), (a.row_ptr, a.col_idx, a.values,
                                                                      a.n_rows), c, osched, workers=8)
    got = P.run(a, a, c, P.build_schedule(a, to_product_cfg(cfg)))
    long_rows = np.diff(a.row_ptr) > 4096
    assert max_rel_err(got, want) <= 1e-12
    if not long_rows.any():
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name,scale", [("cfg1", 1 / 16), ("cfg2", 1 / 16), ("cfg3", 1 / 64),
                                        ("cfg4", 1 / 8), ("cfg5", 1 / 512)])
def test_poisoned_scratch_and_output(cuda, name, scale):
    """Stand-in for a memory checker: the plan's D1 scratch and D are filled
    with NaN bytes before executing, so any read of a D1 row the step did not
    write first, or any D row the step forgets, shows up as NaN or as a
    difference from an unpoisoned run."""
    import ctypes as C

    import torch
    from cuda.bindings import runtime as rt

    from paper_2407_00243_b200 import workloads as W
    from paper_2407_00243_b200._lib import check, lib

    w = W.make(name, scale=scale)
    s = P.build_schedule(w.a, w.scheduler_config())
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    want = P.Plan(prob, s).execute().cpu().numpy()
    plan = P.Plan(prob, s)
    d1 = C.c_void_p()
    check(lib().tfg_plan_d1(plan._h, C.byref(d1)))
    tdt = getattr(torch, w.dtype.name)
    if d1.value:
        (err,) = rt.cudaMemset(d1.value, 0xFF, w.n * w.c_cols * np.dtype(w.dtype).itemsize)
        assert err == rt.cudaError_t.cudaSuccess
    out = torch.full((w.n, w.c_cols), float("nan"), dtype=tdt, device="cuda")
    got = plan.execute(out).cpu().numpy()
    assert not np.isnan(got).any()
    assert np.array_equal(got, want)
