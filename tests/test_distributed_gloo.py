"""Multi-GPU row-block partition, exercised on CPU with gloo (world size 2
and 3).  The partition, halo lists and the all-to-all exchange are the
product code (paper_2407_00243_b200/distributed.py); a NumPy engine stands
in for the GPU kernels.  Each rank's D1 starts NaN-poisoned, so a missing or
misplaced halo row shows up as NaN in D; the union of the ranks' D rows must
equal the oracle's D."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Oracle, SchedulerConfig
from paper_2407_00243_b200 import distributed as PD


class NumpyEngine:
    """Stage semantics of a libtfg partition plan, in NumPy (test only)."""

    def __init__(self, a, b, c, flat, lo, hi):
        self.a, self.b, self.c, self.flat = a, b, c, flat
        self.lo, self.hi = lo, hi
        n, cc = a[0].size - 1, c.shape[1]
        self.d1 = np.full((n, cc), np.nan)
        self.device = torch.device("cpu")
        self.torch_dtype = torch.float64

    def _row(self, rp, ci, v, x, r):
        return v[rp[r]:rp[r + 1]] @ x[ci[rp[r]:rp[r + 1]]] if rp[r + 1] > rp[r] else np.zeros(x.shape[1])

    def _first(self, i):
        if isinstance(self.b, tuple):
            return self._row(*self.b[:3], self.c, i)
        return self.b[i] @ self.c

    def stage0(self, out):
        f = self.flat
        d = out.numpy()
        for v in range(len(f.i_lo[0])):
            lo_t, hi_t = int(f.i_lo[0][v]), int(f.i_hi[0][v])
            if not (self.lo <= lo_t < self.hi):
                continue
            for i in range(lo_t, hi_t):
                self.d1[i] = self._first(i)
            for j in f.j_rows[0][f.j_off[0][v]:f.j_off[0][v + 1]]:
                d[j] = self._row(*self.a, self.d1, j)

    def stage1(self, out):
        d = out.numpy()
        for j in PD.wave1_rows(self.flat):
            if self.lo <= j < self.hi:
                d[j] = self._row(*self.a, self.d1, j)

    def gather_d1(self, rows):
        return torch.from_numpy(self.d1[rows.numpy()].copy())

    def scatter_d1(self, rows, data):
        self.d1[rows.numpy()] = data.numpy().reshape(rows.numel(), -1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b, c, flat = case
        n = a[0].size - 1
        bounds = PD.tile_boundaries(flat, n, world)
        halo = PD.halo_plan(a[0], a[1], flat, bounds, rank)
        eng = NumpyEngine(a, b, c, flat, *bounds[rank])
        plan = PD.DistributedPlan(eng, halo, dist, c.shape[1])
        out = torch.full((n, c.shape[1]), np.nan, dtype=torch.float64)
        plan.execute(out)
        rows = PD.owned_output_rows(flat, bounds, rank)
        q.put((rank, rows, out.numpy()[rows], plan.halo_rows))
    finally:
        dist.destroy_process_group()


def _cases():
    orc = Oracle()
    out = []
    # banded (stencil-like), SpMM-SpMM
    rp, ci, v = orc.gen_banded(600, 5)
    cfg = SchedulerConfig(ct_size=64, num_workers=4, cache_size_words=4096, b_is_dense=False, c_cols=4)
    flat = orc.build_schedule(600, 600, rp, ci, cfg)
    c = np.random.default_rng(0).uniform(-1, 1, (600, 4))
    out.append(((rp, ci, v), (rp, ci, v, 600), c, flat))
    # random sparse, GeMM-SpMM (halo from many peers)
    rp, ci, v = orc.gen_random_sparse(500, 0.01, 9)
    cfg = SchedulerConfig(ct_size=32, num_workers=3, cache_size_words=2048, b_cols=6, c_cols=5)
    flat = orc.build_schedule(500, 500, rp, ci, cfg)
    rng = np.random.default_rng(1)
    out.append(((rp, ci, v), rng.uniform(-1, 1, (500, 6)), rng.uniform(-1, 1, (6, 5)), flat))
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("which", [0, 1])
def test_partitioned_product_matches_oracle(world, which):
    case = _cases()[which]
    a, b, c, flat = case
    n = a[0].size - 1
    want = Oracle().run(n, a, b, c, flat)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.full((n, c.shape[1]), np.nan)
    covered = np.zeros(n, int)
    for rank, rows, vals, halo_rows in res:
        got[rows] = vals
        covered[rows] += 1
    assert (covered == 1).all(), "every D row computed by exactly one rank"
    assert not np.isnan(got).any(), "a halo row was missing"
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    assert sum(r[3] for r in res) > 0  # the exchange actually moved rows


def test_tile_boundaries_cut_at_tiles():
    orc = Oracle()
    rp, ci, v = orc.gen_banded(1000, 3)
    flat = orc.build_schedule(1000, 1000, rp, ci, SchedulerConfig(ct_size=64, num_workers=8))
    for world in (1, 2, 4, 8):
        b = PD.tile_boundaries(flat, 1000, world)
        assert b[0][0] == 0 and b[-1][1] == 1000 and len(b) == world
        starts = set(int(x) for x in flat.i_lo[0]) | {1000}
        for lo, hi in b:
            assert lo in starts and hi in starts and lo <= hi
