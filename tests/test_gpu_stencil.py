"""Grid-stencil SpMM (csrc/tfg_stencil.cu) against the CPU oracle.

The plan switches a row-list SpMM over every row of a grid-stencil CSR to the
plane-streaming kernel.  Its per-row order is the reference's (kernels.hpp:
71-80: ascending nonzeros from 0).  With reference bits (separately rounded
mul and add) SpMM-SpMM results must be bit-identical to the oracle -- for
interior rows (register path, no col_idx reads) and grid-face rows (per-row
path) alike; the default (one FMA per term) must be within the north-star
max-norm tolerance and equal between fused and unfused plans.  Values are
random so a wrong neighbour or a wrong order shows up."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from helpers import max_rel_err
from oracle.oracle import SchedulerConfig as OCfg

pytestmark = pytest.mark.gpu

BOX2 = [(dz, 0, dx) for dz in (-1, 0, 1) for dx in (-1, 0, 1)]          # 9-point
BOX3 = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
FIVE = [(-1, 0, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (1, 0, 0)]        # 5-point
SEVEN = [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)]


def grid_stencil(nx, ny, nz, offs, seed, dtype=np.float64):
    """CSR of stencil `offs` ((dz, dy, dx) triples) on an nx * ny * nz grid
    (row r = (z * ny + y) * nx + x), out-of-grid neighbours dropped, values
    U(-1, 1)."""
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    z, rem = np.divmod(idx, nx * ny)
    y, x = np.divmod(rem, nx)
    rows, cols = [], []
    for dz, dy, dx in offs:
        ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny) & (z + dz >= 0)
              & (z + dz < nz))
        r = idx[ok]
        rows.append(r)
        cols.append(r + (dz * ny + dy) * nx + dx)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    v = np.random.default_rng(seed).uniform(-1, 1, c.size).astype(dtype)
    return P.Csr(n, n, rp.astype(np.int32), c.astype(np.int32), v)


def run_plan(a, b, c, dt, sched=None, bits=True):
    prob = P.DeviceProblem(a, b, c, dt)
    plan = P.Plan(prob, sched, reference_bits=bits)
    d = plan.execute().cpu().numpy()
    return d, plan.kernels()


def oracle_d(oracle, a, b, c, dt, osched=None):
    return oracle.run(a.n_rows, (a.row_ptr, a.col_idx, a.values),
                      (b.row_ptr, b.col_idx, b.values, b.n_cols), c, osched, dt)


CASES = [
    # (nx, ny, nz, offsets, c_cols, dtype, expected kernel)
    (64, 1, 40, BOX2, 64, np.float64, "stencil2d"),    # whole tiles
    (70, 1, 33, BOX2, 128, np.float64, "stencil2d"),   # partial tile, 2 column slices
    (37, 1, 29, FIVE, 64, np.float64, "stencil2d"),    # partial lines
    (64, 1, 21, BOX2, 128, np.float32, "stencil2d"),   # fp32: 128-float slices
    (16, 16, 12, BOX3, 64, np.float64, "stencil3d"),
    (12, 10, 9, BOX3, 128, np.float64, "stencil3d"),     # partial tiles in x and y
    (9, 11, 7, SEVEN, 64, np.float64, "stencil3d"),
    (16, 8, 10, BOX3, 256, np.float32, "stencil3d"),
]


@pytest.mark.parametrize("nx,ny,nz,offs,cc,dt,kind", CASES)
def test_stencil_unfused_bit_exact(cuda, oracle, nx, ny, nz, offs, cc, dt, kind):
    a = grid_stencil(nx, ny, nz, offs, 1, dt)
    b = grid_stencil(nx, ny, nz, offs, 2, dt)  # same pattern, other values
    c = np.random.default_rng(3).uniform(-1, 1, (a.n_rows, cc)).astype(dt)
    d, ks = run_plan(a, b, c, dt)
    assert ks["first_op"] == kind and ks["wave1"] == kind, ks
    want = oracle_d(oracle, a, b, c, dt)
    assert np.array_equal(d, want), max_rel_err(d, want)


def test_stencil_different_patterns(cuda, oracle):
    """A and B different stencils on the same grid (B = 5-point, A = 9-point)."""
    a = grid_stencil(64, 1, 30, BOX2, 4)
    b = grid_stencil(64, 1, 30, FIVE, 5)
    c = np.random.default_rng(6).uniform(-1, 1, (a.n_rows, 64))
    d, ks = run_plan(a, b, c, np.float64)
    assert ks["first_op"] == "stencil2d" and ks["wave1"] == "stencil2d", ks
    assert np.array_equal(d, oracle_d(oracle, a, b, c, np.float64))


def test_wrapped_neighbour_is_not_a_stencil(cuda, oracle):
    """A row at x = 0 that references row r - 1 (the previous grid line's
    last point) is not an in-grid neighbour: the plan must keep the
    row-list SpMM and still be bit-exact."""
    a = grid_stencil(64, 1, 16, BOX2, 7)
    rp, ci, v = a.row_ptr.copy(), list(a.col_idx), list(a.values)
    r = 64 * 5  # x = 0, z = 5: add column r - 1
    k = int(rp[r])
    ci.insert(k, r - 1 - 64)  # keep columns ascending: (z-1, x=-1) wraps to (z-2, x=63)
    v.insert(k, 0.5)
    rp[r + 1:] += 1
    bad = P.Csr(a.n_rows, a.n_cols, rp, np.array(ci, np.int32), np.array(v))
    c = np.random.default_rng(8).uniform(-1, 1, (a.n_rows, 64))
    d, ks = run_plan(bad, bad, c, np.float64)
    assert "stencil" not in ks["first_op"] and "stencil" not in ks["wave1"], ks
    assert np.array_equal(d, oracle_d(oracle, bad, bad, c, np.float64))


def test_stencil_with_schedule(cuda, oracle):
    """Through the reference schedule: whatever rows it fuses, D is bit-exact
    and fused == unfused."""
    a = grid_stencil(64, 1, 48, BOX2, 9)
    c = np.random.default_rng(10).uniform(-1, 1, (a.n_rows, 64))
    cfg = P.SchedulerConfig(ct_size=256, num_workers=8, cache_size_words=16384, b_cols=a.n_cols,
                            c_cols=64, b_is_dense=False)
    s = P.build_schedule(a, cfg)
    osched = oracle.build_schedule(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, OCfg(**cfg.__dict__))
    d_f, _ = run_plan(a, a, c, np.float64, s)
    d_u, ks = run_plan(a, a, c, np.float64)
    assert ks["wave1"] == "stencil2d"
    want = oracle_d(oracle, a, a, c, np.float64, osched)
    assert np.array_equal(d_f, want) and np.array_equal(d_u, want)


def test_stencil_nan_poison(cuda, oracle):
    """Every output row is written: a NaN-filled D comes back finite and exact."""
    import torch

    a = grid_stencil(12, 10, 9, BOX3, 11)
    c = np.random.default_rng(12).uniform(-1, 1, (a.n_rows, 128))
    prob = P.DeviceProblem(a, a, c, np.float64)
    plan = P.Plan(prob, None, reference_bits=True)
    out = torch.full((a.n_rows, 128), float("nan"), dtype=torch.float64, device="cuda")
    d = plan.execute(out).cpu().numpy()
    assert np.isfinite(d).all()
    assert np.array_equal(d, oracle_d(oracle, a, a, c, np.float64))


@pytest.mark.parametrize("knobs", [{"TFG_STENCIL_NW": "8"}, {"TFG_STENCIL_CTAS": "2"},
                                   {"TFG_STENCIL_CTAS": "4"}, {"TFG_STENCIL_NS": "3"},
                                   {"TFG_STENCIL_ZC": "5"}])
def test_stencil_tile_configs(cuda, oracle, monkeypatch, knobs):
    """Every tile / ring / occupancy configuration the plan can pick gives the
    same bits (partial tiles in x, y and z included)."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    for nx, ny, nz, offs, cc in ((12, 10, 9, BOX3, 128), (70, 1, 33, BOX2, 64)):
        a = grid_stencil(nx, ny, nz, offs, 13)
        c = np.random.default_rng(14).uniform(-1, 1, (a.n_rows, cc))
        d, ks = run_plan(a, a, c, np.float64)
        assert "stencil" in ks["wave1"], ks
        assert np.array_equal(d, oracle_d(oracle, a, a, c, np.float64))


@pytest.mark.parametrize("nx,ny,nz,offs,cc,dt,kind", CASES)
def test_stencil_fma_default_within_tolerance(cuda, oracle, nx, ny, nz, offs, cc, dt, kind):
    """The default plan (one FMA per term) stays within the north-star
    max-norm tolerance of the reference and is identical fused vs unfused."""
    from helpers import TOL

    a = grid_stencil(nx, ny, nz, offs, 1, dt)
    b = grid_stencil(nx, ny, nz, offs, 2, dt)
    c = np.random.default_rng(3).uniform(-1, 1, (a.n_rows, cc)).astype(dt)
    d, ks = run_plan(a, b, c, dt, bits=False)
    assert ks["wave1"] == kind, ks
    want = oracle_d(oracle, a, b, c, dt)
    assert max_rel_err(d, want) <= TOL[np.dtype(dt).itemsize]
    cfg = P.SchedulerConfig(ct_size=256, num_workers=8, cache_size_words=16384, b_cols=a.n_cols,
                            c_cols=cc, b_is_dense=False)
    d_f, _ = run_plan(a, b, c, dt, P.build_schedule(b, cfg), bits=False)
    assert np.array_equal(d_f, d)


def test_unsorted_columns_are_not_a_stencil(cuda, oracle):
    """a stencil CSR whose row has its columns out of order (or a
    duplicate) must not take the rank-indexed stencil kernel."""
    a = grid_stencil(40, 1, 12, BOX2, 23)
    ci = a.col_idx.copy()
    r = 40 * 6 + 7  # an interior row: swap two of its columns (and values)
    k = int(a.row_ptr[r])
    ci[k], ci[k + 1] = ci[k + 1], ci[k]
    v = a.values.copy()
    v[k], v[k + 1] = v[k + 1], v[k]
    bad = P.Csr(a.n_rows, a.n_cols, a.row_ptr, ci, v, validate=False)
    c = np.random.default_rng(24).uniform(-1, 1, (a.n_rows, 64))
    d, ks = run_plan(bad, bad, c, np.float64)
    assert "stencil" not in ks["first_op"] and "stencil" not in ks["wave1"], ks
    assert np.array_equal(d, oracle_d(oracle, bad, bad, c, np.float64))


@pytest.mark.parametrize("nx,ny,nz,offs,world", [(64, 1, 48, BOX2, 2), (64, 1, 48, BOX2, 4),
                                                 (8, 8, 16, BOX3, 4)])
def test_stencil_partitions(cuda, oracle, nx, ny, nz, offs, world):
    """Row-block partitions at plane boundaries (the multi-GPU path, ranks
    emulated in one process): each rank's stencil kernel computes its slab of
    z, D1 halo planes arrive by the pack/unpack exchange; D bit-exact."""
    import torch

    from paper_2407_00243_b200 import distributed as PD

    a = grid_stencil(nx, ny, nz, offs, 18)
    n = a.n_rows
    c = np.random.default_rng(19).uniform(-1, 1, (n, 64))
    cfg = P.SchedulerConfig(ct_size=nx * ny, num_workers=8, cache_size_words=4096, b_cols=n,
                            c_cols=64, b_is_dense=False)
    prob = P.DeviceProblem(a, a, c, np.float64)
    sched = P.build_schedule(prob.a, cfg)
    flat = sched.export()
    bounds = PD.tile_boundaries(flat, n, world)
    assert all(lo % (nx * ny) == 0 for lo, _ in bounds)
    engines = [PD.GpuEngine(prob, sched, *bounds[r], reference_bits=True) for r in range(world)]
    for e in engines:
        ks = e.kernels()
        assert "stencil" in ks["first_op"] and "stencil" in ks["wave1"], ks
    halos = [PD.halo_plan(a.row_ptr, a.col_idx, flat, bounds, r) for r in range(world)]
    outs = [torch.full((n, 64), float("nan"), dtype=torch.float64, device="cuda")
            for _ in range(world)]
    for r in range(world):
        engines[r].stage0(outs[r])
    for r in range(world):
        for s_ in range(world):
            rows = torch.as_tensor(halos[r].recv[s_], dtype=torch.int32, device="cuda")
            if rows.numel():
                engines[r].scatter_d1(rows, engines[s_].gather_d1(rows))
    for r in range(world):
        engines[r].stage1(outs[r])
    torch.cuda.synchronize()
    got = np.full((n, 64), np.nan)
    for r in range(world):
        rows = PD.owned_output_rows(flat, bounds, r)
        got[rows] = outs[r].cpu().numpy()[rows]
    osched = oracle.build_schedule(n, n, a.row_ptr, a.col_idx, OCfg(**cfg.__dict__))
    assert np.array_equal(got, oracle_d(oracle, a, a, c, np.float64, osched))


def test_stencil_random_battery(cuda, oracle):
    """Seeded random grids, stencil subsets, dropped entries, column counts and
    dtypes: whatever kernel the plan picks, SpMM-SpMM stays bit-exact."""
    rng = np.random.default_rng(2024)
    kinds = set()
    for case in range(24):
        d3 = bool(rng.integers(0, 2))
        if d3:
            nx, ny, nz = (int(v) for v in rng.integers(3, 14, size=3))
            box = BOX3
        else:
            nx, ny, nz = int(rng.integers(3, 90)), 1, int(rng.integers(2, 40))
            box = BOX2
        keep = [o for o in box if o == (0, 0, 0) or rng.random() < 0.8]
        dt = np.float32 if rng.random() < 0.3 else np.float64
        cc = int(rng.choice([64, 128, 256] if dt == np.float32 else [64, 128]))
        a = grid_stencil(nx, ny, nz, keep, 100 + case, dt)
        b = grid_stencil(nx, ny, nz, keep, 200 + case, dt)
        if rng.random() < 0.3:  # drop a few nonzeros of A: some rows lose neighbours
            rp, ci, v = a.row_ptr, a.col_idx, a.values
            drop = np.zeros(ci.size, bool)
            drop[rng.choice(ci.size, size=max(1, ci.size // 50), replace=False)] = True
            rows = np.repeat(np.arange(a.n_rows), np.diff(rp))
            keep_m = ~drop
            rp2 = np.zeros(a.n_rows + 1, np.int64)
            np.cumsum(np.bincount(rows[keep_m], minlength=a.n_rows), out=rp2[1:])
            a = P.Csr(a.n_rows, a.n_cols, rp2.astype(np.int32), ci[keep_m], v[keep_m])
        c = rng.uniform(-1, 1, (a.n_rows, cc)).astype(dt)
        d, ks = run_plan(a, b, c, dt)
        kinds.add(ks["wave1"])
        want = oracle_d(oracle, a, b, c, dt)
        assert np.array_equal(d, want), (case, nx, ny, nz, len(keep), cc, dt, ks,
                                         max_rel_err(d, want))
    assert any("stencil" in k for k in kinds), kinds
