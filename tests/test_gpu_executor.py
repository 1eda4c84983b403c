"""Executor parity: the sm_100a fused / unfused executors against the CPU
oracle and the reference's golden D.  Tolerance (north star, max-norm
relative): 1e-12 fp64, 1e-5 fp32.  SpMM-SpMM with short rows is checked
bit-exact: the SpMM kernels keep the reference's per-element order
(kernels.hpp:71-80) with separately rounded mul and add."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import TOL, golden_cfg, golden_sched, load, max_rel_err, to_product_cfg
from oracle.oracle import SchedulerConfig

pytestmark = pytest.mark.gpu


def as_csr(t, n_cols=None):
    rp, ci, v = t[:3]
    n = len(rp) - 1
    return P.Csr(n, n if n_cols is None else n_cols, rp, ci, v, validate=False)


def test_golden_executors(cuda):
    z = load("executors.npz")
    for key in z["keys"]:
        n = int(z[f"{key}/n"])
        size = int(z[f"{key}/dtype"])
        dt = np.float64 if size == 8 else np.float32
        a = P.Csr(n, n, z[f"{key}/a_rp"], z[f"{key}/a_ci"], z[f"{key}/a_v"])
        dense = f"{key}/b" in z
        b = z[f"{key}/b"] if dense else P.Csr(n, int(z[f"{key}/b_cols"]), z[f"{key}/b_rp"],
                                               z[f"{key}/b_ci"], z[f"{key}/b_v"])
        c = z[f"{key}/c"]
        cfg = golden_cfg(z, key)
        s = P.build_schedule(a, to_product_cfg(cfg))
        d_f = P.run(a.astype(dt), b if dense else b.astype(dt), c.astype(dt), s, dt)
        d_u = P.run(a.astype(dt), b if dense else b.astype(dt), c.astype(dt), None, dt)
        want_f, want_u = z[f"{key}/d_fused"], z[f"{key}/d_unfused"]
        assert max_rel_err(d_f, want_f) <= TOL[size], key
        assert max_rel_err(d_u, want_u) <= TOL[size], key
        assert np.array_equal(d_f, d_u), key  # fused == unfused bitwise on the GPU too
        if not dense:
            assert np.array_equal(d_f, want_f), key  # SpMM-SpMM: bit-exact vs reference


def test_known_answers(cuda):  # test_kernels.cpp:26-64
    i2 = P.Csr(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    d = P.unfused_gemm_spmm(i2, np.array([[1., 2.], [3., 4.]]), np.array([[5., 6.], [7., 8.]]))
    assert d.ravel().tolist() == [19, 22, 43, 50]
    a = P.Csr(2, 2, [0, 1, 2], [1, 0], [2.0, 3.0])
    d = P.unfused_spmm_spmm(a, i2, np.array([[1., 2.], [3., 4.]]))
    assert d.ravel().tolist() == [6, 8, 3, 6]


def test_row_range_helpers(cuda, oracle):  # test_kernels.cpp:26-64, kernels.hpp:159-180
    b = np.array([[1., 2.], [3., 4.]])
    c = np.array([[5., 6.], [7., 8.]])
    d1 = np.zeros((2, 2))
    assert P.gemm(b, c, 0, 2, d1).ravel().tolist() == [19, 22, 43, 50]
    part = np.zeros((2, 2))
    assert P.gemm(b, c, 1, 2, part).ravel().tolist() == [0, 0, 43, 50]
    with pytest.raises(ValueError):
        P.gemm(b, c, 0, 2, np.zeros((3, 2)))
    a = P.Csr(2, 2, [0, 1, 2], [1, 0], [2.0, 3.0])
    x = np.array([[1., 2.], [3., 4.]])
    assert P.spmm(a, x, [0, 1], np.zeros((2, 2))).ravel().tolist() == [6, 8, 3, 6]
    assert P.spmm(a, x, [1], np.zeros((2, 2))).ravel().tolist() == [0, 0, 3, 6]
    with pytest.raises(ValueError):
        P.spmm(a, np.zeros((3, 2)), [0], np.zeros((2, 2)))
    # a larger random row subset is bit-exact against the reference order
    rp, ci, v = oracle.gen_random_sparse(500, 0.02, 8)
    a = P.Csr(500, 500, rp, ci, v)
    xx = np.random.default_rng(0).uniform(-1, 1, (500, 64))
    rows = np.sort(np.random.default_rng(1).choice(500, 200, replace=False))
    got = P.spmm(a, xx, rows, np.zeros((500, 64)))
    want = oracle.run(500, (rp, ci, v), np.eye(500), xx, None)  # D = A (I X)
    assert np.array_equal(got[rows], want[rows]) and not got[np.setdiff1d(np.arange(500), rows)].any()


def test_matches_numpy_like_reference_smoke(cuda):  # tests/python/test_smoke.py:60-90
    rng = np.random.default_rng(3)
    a = P.gen_random_sparse(80, 0.08, seed=3)
    b = rng.uniform(-1.0, 1.0, size=(80, 8))
    c = rng.uniform(-1.0, 1.0, size=(8, 5))
    want = a.to_dense() @ (b @ c)
    got = P.fused_gemm_spmm(a, b, c, workers=2)
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)
    assert np.array_equal(got, P.unfused_gemm_spmm(a, b, c, workers=2))
    rng = np.random.default_rng(4)
    a = P.gen_random_sparse(60, 0.1, seed=4)
    bs = P.gen_random_sparse(60, 0.15, seed=5)
    c = rng.uniform(-1.0, 1.0, size=(60, 4))
    got = P.fused_spmm_spmm(a, bs, c, workers=2)
    np.testing.assert_allclose(got, a.to_dense() @ (bs.to_dense() @ c), rtol=1e-10, atol=1e-12)
    assert np.array_equal(got, P.unfused_spmm_spmm(a, bs, c, workers=2))
    a = P.gen_random_sparse(100, 0.05, seed=9)
    b = rng.uniform(-1.0, 1.0, size=(100, 16))
    c = rng.uniform(-1.0, 1.0, size=(16, 16))
    assert np.array_equal(P.fused_gemm_spmm(a, b, c, workers=1), P.fused_gemm_spmm(a, b, c, workers=8))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("dense", [True, False])
def test_random_vs_oracle(cuda, oracle, dt, dense):
    rng = np.random.default_rng(5 + dense)
    size = np.dtype(dt).itemsize
    for trial in range(24):
        n = int(rng.integers(2, 700))
        rp, ci, v = oracle.gen_random_sparse(n, float(rng.choice([0.004, 0.02, 0.08])),
                                             int(rng.integers(1, 2**62)))
        bc = int(rng.choice([1, 3, 4, 8, 16, 32, 64, 128, 256]))
        cc = int(rng.choice([1, 2, 4, 5, 8, 13, 16, 32, 64, 96, 128, 256]))
        if dense:
            b = rng.uniform(-1, 1, (n, bc))
            ob = b
        else:
            brp, bci, bv = oracle.gen_rect_random(n, bc, 0.2, int(rng.integers(1, 2**62)))
            b = P.Csr(n, bc, brp, bci, bv)
            ob = (brp, bci, bv, bc)
        c = rng.uniform(-1, 1, (bc, cc))
        cfg = SchedulerConfig(ct_size=int(rng.choice([8, 64, 512, 4096])), num_workers=int(rng.integers(1, 9)),
                              cache_size_words=int(rng.choice([256, 4096, 163840, 10 ** 9])),
                              b_cols=bc, c_cols=cc, b_is_dense=dense,
                              index_to_scalar_ratio=0.5 if size == 8 else 1.0)
        osched = oracle.build_schedule(n, n, rp, ci, cfg)
        want = oracle.run(n, (rp, ci, v), ob, c, osched, dt)
        a = P.Csr(n, n, rp, ci, v)
        s = P.build_schedule(a, to_product_cfg(cfg))
        prob = P.DeviceProblem(a, b, c, dt)
        plan = P.Plan(prob, s)
        got = plan.execute().cpu().numpy()
        assert max_rel_err(got, want) <= TOL[size], (trial, n, bc, cc, cfg)
        st = plan.stats()
        assert st["first_op_rows"] == n and st["second_op_rows"] == n
        un = P.Plan(prob, None).execute().cpu().numpy()
        assert np.array_equal(got, un), (trial, n, bc, cc)
        if not dense:
            assert np.array_equal(got, want), (trial, "spmm-spmm must be bit-exact")


def test_global_staging_and_long_rows(cuda, oracle):
    """Tiles wider than shared memory (staged through HBM/L2 inside the CTA)
    and rows longer than the segmentation threshold."""
    n = 12000
    rp, ci, v = oracle.gen_banded(n, 3)
    rng = np.random.default_rng(1)
    c = rng.uniform(-1, 1, (n, 128))
    cfg = SchedulerConfig(ct_size=8192, num_workers=1, cache_size_words=10 ** 12, b_is_dense=False,
                          c_cols=128, b_cols=n)
    osched = oracle.build_schedule(n, n, rp, ci, cfg)
    assert osched.j_off[0][-1] > 0
    want = oracle.run(n, (rp, ci, v), (rp, ci, v, n), c, osched)
    a = P.Csr(n, n, rp, ci, v)
    got = P.run(a, a, c, P.build_schedule(a, to_product_cfg(cfg)))
    assert np.array_equal(got, want)
    # arrow: first row dense (long, segmented), others short
    rows_ci = [np.arange(n)] + [np.array([0, i]) for i in range(1, n)]
    ci2 = np.concatenate(rows_ci).astype(np.int32)
    rp2 = np.concatenate([[0], np.cumsum([r.size for r in rows_ci])]).astype(np.int32)
    v2 = rng.uniform(-1, 1, ci2.size)
    b = rng.uniform(-1, 1, (n, 16))
    c2 = rng.uniform(-1, 1, (16, 64))
    a2 = P.Csr(n, n, rp2, ci2, v2)
    for dt in (np.float64, np.float32):
        want = oracle.run(n, (rp2, ci2, v2), b, c2, None, dt)
        got = P.unfused_gemm_spmm(a2, b, c2, dtype=dt)
        assert max_rel_err(got, want) <= TOL[np.dtype(dt).itemsize]


def test_executor_errors(cuda):  # test_kernels.cpp:194-229
    a = P.gen_banded(16, 1)
    cfg = P.SchedulerConfig(b_cols=4, c_cols=4)
    other = P.build_schedule(P.gen_banded(8, 1), cfg)
    b = np.ones((16, 4))
    c = np.ones((4, 4))
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, b, c, sched=other)
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, b, c, workers=0)
    with pytest.raises(ValueError):
        P.unfused_gemm_spmm(a, b, c, workers=-1)
    with pytest.raises(ValueError):
        P.fused_spmm_spmm(a, b, c)
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, P.gen_banded(16, 0), c)
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, b, np.ones((5, 4)))
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, np.ones((15, 4)), c)
    prob = P.DeviceProblem(a, b, c)
    with pytest.raises(ValueError):
        P.Plan(prob, other)


def test_determinism_repeated_runs(cuda, oracle):  # acceptance.cpp:323-366
    rp, ci, v = oracle.gen_random_sparse(2000, 0.01, 4242)
    a = P.Csr(2000, 2000, rp, ci, v)
    rng = np.random.default_rng(0)
    b, c = rng.uniform(-1, 1, (2000, 16)), rng.uniform(-1, 1, (16, 16))
    s = P.build_schedule(a, P.SchedulerConfig(ct_size=64, num_workers=8, cache_size_words=4096,
                                              b_cols=16, c_cols=16))
    plan = P.Plan(P.DeviceProblem(a, b, c), s)
    d0 = plan.execute().cpu().numpy()
    for _ in range(5):
        assert np.array_equal(plan.execute().cpu().numpy(), d0)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_baseline_configs(cuda, oracle, name):
    """BASELINE configs (cfg1, cfg2, cfg4 at full size; R-MAT configs reduced
    so the CPU oracle finishes in seconds) against the multithreaded oracle."""
    import os

    from paper_2407_00243_b200 import workloads as W

    scale = {"cfg1": 1.0, "cfg2": 1.0, "cfg3": 1 / 8, "cfg4": 1.0, "cfg5": 1 / 64}[name]
    w = W.make(name, scale=scale)
    cfg = w.scheduler_config()
    s = P.build_schedule(w.a, cfg)
    prob = P.DeviceProblem(w.a, w.b, w.c, w.dtype)
    got = P.Plan(prob, s).execute().cpu().numpy()  # default: FMA stencil terms
    exact = P.Plan(prob, s, reference_bits=True).execute().cpu().numpy()
    ocfg = SchedulerConfig(**cfg.__dict__)
    osched = oracle.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
    ob = w.b if not isinstance(w.b, P.Csr) else (w.b.row_ptr, w.b.col_idx, w.b.values, w.b.n_cols)
    want = oracle.run(w.n, (w.a.row_ptr, w.a.col_idx, w.a.values), ob, w.c, osched, w.dtype,
                      workers=os.cpu_count() or 1)
    size = np.dtype(w.dtype).itemsize
    assert max_rel_err(got, want) <= TOL[size]
    assert max_rel_err(exact, want) <= TOL[size]
    if w.op == "spmm-spmm":
        assert np.array_equal(exact, want)
