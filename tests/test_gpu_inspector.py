"""GPU inspector parity: the sm_100a build_schedule must be bit-identical to
the reference inspector (schedules_equal, tests/support.hpp:150-165) --
tile order, i ranges, j lists and the exact double costs."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import golden_cfg, golden_sched, load, schedules_equal, to_product_cfg
from oracle.oracle import SchedulerConfig

pytestmark = pytest.mark.gpu


def gpu_sched(rp, ci, cfg, n_cols=None):
    n = len(rp) - 1
    a = P.Csr(n, n if n_cols is None else n_cols, rp, ci, np.ones(len(ci)), validate=False)
    return P.build_schedule(a, to_product_cfg(cfg))


def test_golden_schedules_bit_exact(cuda):
    z = load("schedules.npz")
    for key in z["keys"]:
        rp, ci = z[f"{key}/row_ptr"], z[f"{key}/col_idx"]
        s = gpu_sched(rp, ci, golden_cfg(z, key))
        assert schedules_equal(s.export(), golden_sched(z, key)), key
        assert s.fused_ratio() == float(z[f"{key}/fused_ratio"]), key


def test_random_battery_vs_oracle(cuda, oracle):
    rng = np.random.default_rng(31)
    for trial in range(150):
        n = 1 + int(rng.integers(0, 600))
        dens = 0.002 + 0.4 * int(rng.integers(0, 100)) / 100
        rp, ci, _ = oracle.gen_random_sparse(n, dens, int(rng.integers(1, 2**62)))
        cfg = SchedulerConfig(num_workers=int(1 + rng.integers(0, 8)),
                              ct_size=int(1 << (1 + rng.integers(0, 10))),
                              cache_size_words=int(rng.choice([16, 512, 4096, 163840])),
                              b_is_dense=trial % 2 == 0, whole_b_cost=trial % 5 == 0,
                              b_cols=int(rng.integers(1, 65)), c_cols=int(rng.integers(1, 129)),
                              index_to_scalar_ratio=float(rng.choice([0.5, 1.0, 0.3, 0.7])))
        want = oracle.build_schedule(n, n, rp, ci, cfg)
        got = gpu_sched(rp, ci, cfg)
        assert schedules_equal(got.export(), want), (trial, n, cfg)


def test_structured_patterns_vs_oracle(cuda, oracle):
    cases = []
    for n, hb in [(16, 1), (97, 0), (500, 7), (4096, 33), (20000, 3)]:
        rp, ci, _ = oracle.gen_banded(n, hb)
        cases.append((rp, ci))
    # arrow (dense first row/col), identity, dense, empty rows
    n = 300
    rows = {0: list(range(n))}
    rows.update({i: [0, i] for i in range(1, n)})
    rp = [0]
    ci = []
    for r in range(n):
        ci += rows[r]
        rp.append(len(ci))
    cases.append((np.array(rp, np.int32), np.array(ci, np.int32)))
    cases.append((np.arange(65, dtype=np.int32), np.arange(64, dtype=np.int32)))
    rpe = np.zeros(51, np.int32)
    rpe[20:] = 1
    cases.append((rpe, np.array([5], np.int32)))  # one nonzero, 49 empty rows
    for rp, ci in cases:
        n = len(rp) - 1
        for ct, p, budget in [(4, 3, 64), (64, 8, 4096), (2048, 148, 163840), (16, 1, 10 ** 12)]:
            for dense in (True, False):
                cfg = SchedulerConfig(ct_size=ct, num_workers=p, cache_size_words=budget,
                                      b_is_dense=dense)
                assert schedules_equal(gpu_sched(rp, ci, cfg).export(),
                                       oracle.build_schedule(n, n, rp, ci, cfg)), (n, ct, p, budget)


def test_known_answers(cuda):  # test_scheduler.cpp:302-374, test_smoke.py:93-109
    a = P.gen_banded(16, 1)
    s = P.build_schedule(a, P.SchedulerConfig(ct_size=4, num_workers=2))
    assert s.fused_ratio() == 0.3125
    fl = s.export()
    assert (fl.i_lo[0][0], fl.i_hi[0][0]) == (0, 4)
    assert fl.j_rows[0][fl.j_off[0][0]:fl.j_off[0][1]].tolist() == [0, 1, 2]
    assert sorted(fl.j_rows[1].tolist()) == [3, 4, 7, 8, 11, 12]
    assert P.validate_schedule(a, s, P.SchedulerConfig(ct_size=4, num_workers=2))[0]
    assert P.fused_ratio(P.gen_banded(8, 0), tile_size=4) == 0.5
    assert P.fused_ratio(P.gen_banded(8, 7), tile_size=4) == 0.0
    assert P.fused_ratio(P.gen_banded(16, 1), tile_size=4) == 0.3125
    import json

    doc = json.loads(P.schedule_json(P.gen_banded(16, 1), workers=2, ct_size=4))
    assert doc["n"] == 16 and doc["tile_size_t"] == 4 and doc["fused_ratio"] == 0.3125
    assert len(doc["wavefronts"]) == 2
    t0 = doc["wavefronts"][0][0]
    assert [t0["i_lo"], t0["i_hi"]] == [0, 4] and t0["j_list"] == [0, 1, 2]


def test_errors(cuda):
    rect = P.Csr(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        P.build_schedule(rect, P.SchedulerConfig())
    with pytest.raises(ValueError):
        P.build_schedule(P.gen_banded(8, 1), P.SchedulerConfig(num_workers=0))
    with pytest.raises(ValueError):
        P.build_schedule(P.gen_banded(8, 1), P.SchedulerConfig(ct_size=0))


def test_json_round_trip(cuda):  # test_schedule_io.cpp:11-71 (row f1)
    a = P.gen_random_sparse(200, 0.03, 5)
    cfg = P.SchedulerConfig(ct_size=16, num_workers=4, cache_size_words=2048)
    s = P.build_schedule(a, cfg)
    back = P.schedule_from_json(P.schedule_to_json(s))
    assert schedules_equal(back.export(), s.export())
    with pytest.raises(RuntimeError):
        P.schedule_from_json("{not json")


def test_determinism(cuda):  # test_scheduler.cpp:500-509
    a = P.gen_random_sparse(3000, 0.004, 5)
    cfg = P.SchedulerConfig(num_workers=4, ct_size=64, cache_size_words=2048)
    assert schedules_equal(P.build_schedule(a, cfg).export(), P.build_schedule(a, cfg).export())


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_baseline_configs_full_size(cuda, oracle, name):
    """Full BASELINE sizes with the pinned configs the bench uses."""
    from paper_2407_00243_b200 import workloads as W

    w = W.make(name, scale=1.0 if name != "cfg5" else 1 / 8)
    for p, kb in [(148, 1280.0), (8, 1280.0)]:
        cfg = w.scheduler_config(num_workers=p, cache_kb=kb)
        ocfg = SchedulerConfig(**cfg.__dict__)
        want = oracle.build_schedule(w.n, w.n, w.a.row_ptr, w.a.col_idx, ocfg)
        got = P.build_schedule(w.a, cfg)
        assert schedules_equal(got.export(), want), (name, p, kb)
