"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref/libtfref.so,
compiled from /root/reference/proj by `make -C oracle ref`).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Outputs (committed, small):
  tests/golden/schedules.npz  -- reference build_schedule on a seeded battery
                                 (patterns from the reference's own
                                 gen_random_sparse / gen_banded + BASELINE-shaped
                                 scaled configs), with every SchedulerConfig field
  tests/golden/executors.npz  -- reference fused_/unfused_ D for seeded problems
                                 (dense and CSR B, fp64 and fp32)
The reference is not available on the GPU box; tests read only these files.
"""
from __future__ import annotations

import os
import sys

import ctypes as C

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, RefProblem, SchedulerConfig, ref_schedule_handle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cfg_fields(c: SchedulerConfig):
    return np.array([c.ct_size, c.num_workers, c.cache_size_words, c.b_cols, c.c_cols,
                     int(c.b_is_dense), int(c.whole_b_cost)], np.int64), np.float64(
        c.index_to_scalar_ratio)


def pack_sched(d, key, s):
    d[f"{key}/n"] = np.int64(s.n)
    d[f"{key}/t"] = np.int64(s.tile_size)
    for w in range(2):
        d[f"{key}/w{w}/i_lo"] = s.i_lo[w]
        d[f"{key}/w{w}/i_hi"] = s.i_hi[w]
        d[f"{key}/w{w}/cost"] = s.cost[w]
        d[f"{key}/w{w}/j_off"] = s.j_off[w]
        d[f"{key}/w{w}/j_rows"] = s.j_rows[w]


def main():
    ref = Reference()
    rng = np.random.default_rng(20241020)
    sched = {}
    cases = []
    # 1. random battery, reference generators, randomised configs
    for k in range(60):
        n = int(rng.integers(1, 400))
        dens = float(rng.choice([0.005, 0.02, 0.05, 0.15, 0.4]))
        seed = int(rng.integers(1, 2**62))
        rp, ci, _ = ref.gen_random_sparse(n, dens, seed)
        cfg = SchedulerConfig(ct_size=int(2 ** rng.integers(1, 10)), num_workers=int(rng.integers(1, 9)),
                              cache_size_words=int(rng.choice([64, 512, 4096, 163840])),
                              b_cols=int(rng.integers(1, 64)), c_cols=int(rng.integers(1, 64)),
                              index_to_scalar_ratio=float(rng.choice([0.5, 1.0, 0.3])),
                              b_is_dense=bool(rng.integers(0, 2)), whole_b_cost=bool(rng.integers(0, 2)))
        cases.append((f"rand{k}", rp, ci, cfg))
    # 2. banded / structured
    for (n, hb, ct, p, budget) in [(16, 1, 4, 2, 163840), (200, 3, 16, 3, 64), (1000, 8, 64, 8, 4096),
                                   (5000, 30, 2048, 4, 163840), (4096, 2, 256, 148, 2048)]:
        rp, ci, _ = ref.gen_banded(n, hb)
        cases.append((f"band{n}_{hb}_{ct}_{p}_{budget}", rp, ci,
                      SchedulerConfig(ct_size=ct, num_workers=p, cache_size_words=budget)))
    # 3. BASELINE-shaped patterns at reduced scale (pinned configs as bench uses them)
    from paper_2407_00243_b200 import workloads as W
    for name, scale in [("cfg1", 1 / 16), ("cfg2", 1 / 64), ("cfg3", 1 / 256), ("cfg4", 1 / 64),
                        ("cfg5", 1 / 1024)]:
        w = W.make(name, scale=scale, device="cpu")
        for p, kb in [(148, 1280.0), (8, 64.0)]:
            cfg = w.scheduler_config(num_workers=p, cache_kb=kb)
            cases.append((f"{name}_p{p}_kb{int(kb)}", w.a.row_ptr, w.a.col_idx, cfg))
    for key, rp, ci, cfg in cases:
        n = len(rp) - 1
        s = ref.build_schedule(n, n, rp, ci, cfg)
        sched[f"{key}/row_ptr"] = np.asarray(rp, np.int32)
        sched[f"{key}/col_idx"] = np.asarray(ci, np.int32)
        ci_, cr = cfg_fields(cfg)
        sched[f"{key}/cfg"] = ci_
        sched[f"{key}/ratio"] = cr
        cs, keep = s.to_c()
        sched[f"{key}/fused_ratio"] = np.float64(ref.lib.tfr_fused_ratio(C.byref(cs)))
        del keep
        pack_sched(sched, key, s)
    sched["keys"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(OUT, "schedules.npz"), **sched)

    # executors
    ex = {}
    keys = []
    for k in range(16):
        n = int(rng.integers(2, 240))
        seed = int(rng.integers(1, 2**62))
        rp, ci, v = ref.gen_random_sparse(n, float(rng.choice([0.02, 0.06, 0.2])), seed)
        bc, cc = int(rng.choice([1, 4, 8, 32, 64])), int(rng.choice([1, 4, 8, 32, 64, 128]))
        dense_b = k % 2 == 0
        dt = np.float64 if k % 4 < 2 else np.float32
        if dense_b:
            b = ref.random_dense(n, bc, seed + 1)
            bb = b
        else:
            brp, bci, bv = ref.gen_rect_random(n, bc, 0.25, seed + 1)
            bb = (brp, bci, bv, bc)
        c = ref.random_dense(bc, cc, seed + 2)
        cfg = SchedulerConfig(ct_size=int(rng.choice([8, 16, 64])), num_workers=4,
                              cache_size_words=int(rng.choice([256, 4096, 163840])), b_cols=bc,
                              c_cols=cc, index_to_scalar_ratio=0.5 if dt == np.float64 else 1.0,
                              b_is_dense=dense_b)
        s = ref.build_schedule(n, n, rp, ci, cfg)
        prob = RefProblem(ref, n, (rp, ci, v), bb, c, dt)
        h = ref_schedule_handle(ref, s)
        d_f, st, _ = prob.run(h, True, 4)
        d_u, _, _ = prob.run(None, False, 4)
        key = f"ex{k}"
        keys.append(key)
        ex[f"{key}/n"] = np.int64(n)
        ex[f"{key}/dtype"] = np.int64(8 if dt == np.float64 else 4)
        ex[f"{key}/a_rp"], ex[f"{key}/a_ci"], ex[f"{key}/a_v"] = rp, ci, v
        if dense_b:
            ex[f"{key}/b"] = b
        else:
            ex[f"{key}/b_rp"], ex[f"{key}/b_ci"], ex[f"{key}/b_v"] = brp, bci, bv
            ex[f"{key}/b_cols"] = np.int64(bc)
        ex[f"{key}/c"] = c
        ci_, cr = cfg_fields(cfg)
        ex[f"{key}/cfg"] = ci_
        ex[f"{key}/ratio"] = cr
        ex[f"{key}/d_fused"] = d_f
        ex[f"{key}/d_unfused"] = d_u
        ex[f"{key}/stats"] = st
        pack_sched(ex, key, s)
    ex["keys"] = np.array(keys)
    np.savez_compressed(os.path.join(OUT, "executors.npz"), **ex)
    print("wrote", len(cases), "schedules and", len(keys), "executor cases")


if __name__ == "__main__":
    main()
