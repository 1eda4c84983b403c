"""The fp32 first op on tcgen05 tensor cores (csrc/tfg_tc.cu, 3xTF32).

Dense-B fp32 problems with bCol % 32 == 0 and cCol % 64 == 0 run their first
op on the tensor cores (TFG_TC=1, the default).  The rounding differs from the
FFMA path, so D is checked against the reference within the north-star fp32
tolerance (max-norm 1e-5), fused == unfused bitwise (every first-op path of a
plan uses the same kernel), and against the FFMA path (TFG_TC=0)."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import TOL, max_rel_err, to_product_cfg
from oracle.oracle import SchedulerConfig

pytestmark = pytest.mark.gpu

SHAPES = [  # n (ragged last 128-row block), bCol, cCol
    (1000, 32, 64),
    (777, 64, 128),
    (2048, 128, 128),
    (1500, 256, 64),
    (300, 96, 256),
    (5000, 128, 64),
    (129, 512, 64),
]


def _problem(oracle, n, bc, cc, seed, density=0.01):
    rng = np.random.default_rng(seed)
    rp, ci, v = oracle.gen_random_sparse(n, density, seed + 11)
    b = rng.standard_normal((n, bc)).astype(np.float32)
    c = (rng.standard_normal((bc, cc)) / np.sqrt(bc)).astype(np.float32)
    return rp, ci, v, b, c


@pytest.mark.parametrize("n,bc,cc", SHAPES)
def test_tc_within_tolerance_and_fused_equals_unfused(cuda, oracle, monkeypatch, n, bc, cc):
    monkeypatch.setenv("TFG_TC", "1")
    rp, ci, v, b, c = _problem(oracle, n, bc, cc, n + bc + cc)
    cfg = SchedulerConfig(ct_size=256, num_workers=7, cache_size_words=40960, b_cols=bc,
                          c_cols=cc, index_to_scalar_ratio=1.0)
    osched = oracle.build_schedule(n, n, rp, ci, cfg)
    want = oracle.run(n, (rp, ci, v), b, c, osched, np.float32)
    a = P.Csr(n, n, rp, ci, v)
    s = P.build_schedule(a, to_product_cfg(cfg))
    prob = P.DeviceProblem(a, b, c, np.float32)
    fused = P.Plan(prob, s).execute().cpu().numpy()
    unfused = P.Plan(prob, None).execute().cpu().numpy()
    assert max_rel_err(fused, want) <= TOL[4]
    assert np.array_equal(fused, unfused)
    monkeypatch.setenv("TFG_TC", "0")
    ffma = P.Plan(P.DeviceProblem(a, b, c, np.float32), s).execute().cpu().numpy()
    assert max_rel_err(fused, ffma) <= TOL[4]


def test_tc_staged_and_wide_tiles(cuda, oracle, monkeypatch):
    """A banded matrix with large tiles: some tiles stage their D1 rows in
    shared memory, tiles beyond the stage capacity spill and read D1 via L2."""
    monkeypatch.setenv("TFG_TC", "1")
    n, bc, cc = 20000, 64, 64
    rp, ci, v = oracle.gen_banded(n, 2)
    rng = np.random.default_rng(4)
    b = rng.standard_normal((n, bc)).astype(np.float32)
    c = (rng.standard_normal((bc, cc)) / 8).astype(np.float32)
    for ct in (512, 4096):
        cfg = SchedulerConfig(ct_size=ct, num_workers=3, cache_size_words=10 ** 9, b_cols=bc,
                              c_cols=cc, index_to_scalar_ratio=1.0)
        osched = oracle.build_schedule(n, n, rp, ci, cfg)
        want = oracle.run(n, (rp, ci, v), b, c, osched, np.float32)
        a = P.Csr(n, n, rp, ci, v)
        got = P.Plan(P.DeviceProblem(a, b, c, np.float32),
                     P.build_schedule(a, to_product_cfg(cfg))).execute().cpu().numpy()
        assert max_rel_err(got, want) <= TOL[4], ct


def test_tc_dense_rows_exact_inputs(cuda, monkeypatch):
    """Inputs exactly representable in tf32 (small integers): the 3xTF32
    product is exact, so D equals the integer result bit for bit."""
    monkeypatch.setenv("TFG_TC", "1")
    rng = np.random.default_rng(9)
    n, bc, cc = 640, 64, 128
    b = rng.integers(-4, 5, (n, bc)).astype(np.float32)
    c = rng.integers(-4, 5, (bc, cc)).astype(np.float32)
    rows = [np.unique(np.concatenate([[i], rng.integers(0, n, 5)])) for i in range(n)]
    rp = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int32)
    ci = np.concatenate(rows).astype(np.int32)
    v = rng.integers(-2, 3, ci.size).astype(np.float64)
    a = P.Csr(n, n, rp, ci, v)
    dense_a = np.zeros((n, n))
    for i in range(n):
        dense_a[i, rows[i]] = v[rp[i]:rp[i + 1]]
    want = dense_a @ (b.astype(np.float64) @ c.astype(np.float64))
    got = P.fused_gemm_spmm(a, b, c, dtype=np.float32, ct_size=128)
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("ring", ["2", "3"])
def test_tc_shallow_ring_many_blocks(cuda, oracle, monkeypatch, ring):
    """Many 128-row blocks per CTA through a 2-3 slot TMA ring: every slot is
    refilled many times, so a missing ordering between the converters'
    reads and the next TMA write shows up as wrong rows."""
    monkeypatch.setenv("TFG_TC", "1")
    monkeypatch.setenv("TFG_TC_RING", ring)
    n, bc, cc = 150000, 128, 64
    rng = np.random.default_rng(17)
    rp, ci, v = oracle.gen_banded(n, 1)
    b = rng.standard_normal((n, bc)).astype(np.float32)
    c = (rng.standard_normal((bc, cc)) / 11).astype(np.float32)
    a = P.Csr(n, n, rp, ci, v)
    prob = P.DeviceProblem(a, b, c, np.float32)
    got = P.Plan(prob, None).execute().cpu().numpy()
    want = oracle.run(n, (rp, ci, v), b, c, None, np.float32, workers=8)
    assert max_rel_err(got, want) <= TOL[4]
