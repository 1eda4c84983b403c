"""Shared test helpers: golden fixture access and schedule comparison."""
from __future__ import annotations

import os

import numpy as np

from oracle.oracle import OSchedule, SchedulerConfig, schedules_equal  # noqa: F401

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_cfg(z, key) -> SchedulerConfig:
    f = z[f"{key}/cfg"]
    return SchedulerConfig(ct_size=int(f[0]), num_workers=int(f[1]), cache_size_words=int(f[2]),
                           b_cols=int(f[3]), c_cols=int(f[4]), b_is_dense=bool(f[5]),
                           whole_b_cost=bool(f[6]), index_to_scalar_ratio=float(z[f"{key}/ratio"]))


def golden_sched(z, key) -> OSchedule:
    s = OSchedule(int(z[f"{key}/n"]), int(z[f"{key}/t"]))
    for w in range(2):
        s.i_lo.append(z[f"{key}/w{w}/i_lo"])
        s.i_hi.append(z[f"{key}/w{w}/i_hi"])
        s.cost.append(z[f"{key}/w{w}/cost"])
        s.j_off.append(z[f"{key}/w{w}/j_off"])
        s.j_rows.append(z[f"{key}/w{w}/j_rows"])
    return s


def to_product_cfg(cfg):
    import paper_2407_00243_b200 as P

    return P.SchedulerConfig(**cfg.__dict__)


def max_rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = max(float(np.abs(want).max()) if want.size else 0.0, 1e-300)
    return float(np.abs(got - want).max()) / scale if want.size else 0.0


TOL = {8: 1e-12, 4: 1e-5}  # north star: max-norm relative, fp64 / fp32
