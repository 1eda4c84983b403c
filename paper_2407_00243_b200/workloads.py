"""Seeded synthetic stand-ins for the BASELINE.json configurations.

The paper measures on the SuiteSparse corpus, which is not
available here; these generators reproduce the shapes, sparsity structure and
value distributions BASELINE.json names.  Seeds follow the
reference bench: base 42, B = seed+1, C = seed+2 (bench.hpp:28,
bench.cpp:118-133).  Everything is deterministic for (config, scale, seed).

cfg1  GeMM-SpMM fp64: band +-8 plus 8 distinct random off-band columns per row,
      A,B,C ~ U(-1,1); n = 65536, bCol = cCol = 64.
cfg2  SpMM-SpMM fp64: 2-D 9-point stencil on 1024^2 (diag 8, off -1); B = A;
      C ~ U(-1,1) n x 64.
cfg3  GCN GeMM-SpMM fp32: R-MAT(.57,.19,.19,.05) n = 2^20, n*16/2 edge draws,
      symmetrised, deduplicated, self loops dropped, + I, values
      d_i^-1/2 d_j^-1/2; B ~ N(0,1) n x 128; C Glorot-U(+-sqrt(6/256)) 128x128.
cfg4  SpMM-SpMM fp64: 3-D 27-point stencil on 128^3 (diag 26, off -1); B = A;
      C ~ U(-1,1) n x 128.
cfg5  GeMM-SpMM fp32: R-MAT n = 2^23, n*32/2 draws, symmetrised, deduplicated,
      self loops dropped, values 1/row_nnz (empty rows stay empty);
      B ~ N(0,1) n x 256; C ~ N(0,1/256) 256 x 64.

`scale` shrinks a config for parity tests (grid side / R-MAT scale / n).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tilefuse import Csr, SchedulerConfig

BASE_SEED = 42


@dataclass
class Workload:
    name: str
    op: str               # "gemm-spmm" | "spmm-spmm"
    dtype: np.dtype
    a: Csr
    b: object             # np.ndarray (dense) or Csr
    c: np.ndarray
    description: str

    @property
    def n(self):
        return self.a.n_rows

    @property
    def b_cols(self):
        return self.b.n_cols if isinstance(self.b, Csr) else self.b.shape[1]

    @property
    def c_cols(self):
        return self.c.shape[1]

    def flops(self) -> float:
        """theoretical_flops (bench.cpp:152-159): the unfused count."""
        second = 2.0 * self.a.nnz * self.c_cols
        if self.op == "gemm-spmm":
            return 2.0 * self.n * self.b_cols * self.c_cols + second
        return 2.0 * self.b.nnz * self.c_cols + second

    def scheduler_config(self, num_workers: int = 148, ct_size: int = 2048,
                         cache_kb: float = 1280.0) -> SchedulerConfig:
        """Pinned SchedulerConfig, as bench.cpp:135-150 builds it with an
        explicit cache budget: words = cache_kb*1024/sizeof(T); ratio 0.5
        (dp) or 1.0 (sp); b_cols = the actual columns of B."""
        s = np.dtype(self.dtype).itemsize
        words = max(1, int(cache_kb * 1024.0 / s))
        return SchedulerConfig(ct_size=ct_size, num_workers=num_workers, cache_size_words=words,
                               b_cols=self.b_cols, c_cols=self.c_cols,
                               index_to_scalar_ratio=0.5 if s == 8 else 1.0,
                               b_is_dense=self.op == "gemm-spmm")

    def bytes_min(self) -> int:
        """|A| + |B| + |C| + |D| (fused ideal)."""
        s = np.dtype(self.dtype).itemsize
        a = 4 * (self.n + 1) + self.a.nnz * (4 + s)
        if isinstance(self.b, Csr):
            b = 4 * (self.n + 1) + self.b.nnz * (4 + s)
        else:
            b = self.b.size * s
        return a + b + self.c.size * s + self.n * self.c_cols * s

    def bytes_alg(self, spill_rows: int) -> int:
        """bytes_min + 2 |S| cCol s: the compulsory D1 spill and reload."""
        s = np.dtype(self.dtype).itemsize
        return self.bytes_min() + 2 * spill_rows * self.c_cols * s


# ---------------------------------------------------------------------------
def _csr_from_sorted(n, rows, cols, vals, dtype) -> Csr:
    counts = np.bincount(rows, minlength=n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    return Csr(n, n, rp.astype(np.int32), cols.astype(np.int32), vals.astype(dtype), validate=False)


def stencil_2d(side: int, dtype=np.float64) -> Csr:
    """9-point Laplacian-style stencil on side x side, natural ordering."""
    n = side * side
    y, x = np.divmod(np.arange(n, dtype=np.int64), side)
    rows, cols, vals = [], [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            ok = (y + dy >= 0) & (y + dy < side) & (x + dx >= 0) & (x + dx < side)
            r = np.nonzero(ok)[0]
            rows.append(r)
            cols.append(r + dy * side + dx)
            vals.append(np.full(r.size, 8.0 if (dx == 0 and dy == 0) else -1.0))
    return _finish(n, rows, cols, vals, dtype)


def stencil_3d(side: int, dtype=np.float64) -> Csr:
    """27-point stencil on side^3, natural ordering."""
    n = side ** 3
    idx = np.arange(n, dtype=np.int64)
    z, rem = np.divmod(idx, side * side)
    y, x = np.divmod(rem, side)
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((z + dz >= 0) & (z + dz < side) & (y + dy >= 0) & (y + dy < side)
                      & (x + dx >= 0) & (x + dx < side))
                r = np.nonzero(ok)[0]
                rows.append(r)
                cols.append(r + (dz * side + dy) * side + dx)
                center = dx == 0 and dy == 0 and dz == 0
                vals.append(np.full(r.size, 26.0 if center else -1.0))
    return _finish(n, rows, cols, vals, dtype)


def _finish(n, rows, cols, vals, dtype) -> Csr:
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    order = np.lexsort((c, r))
    return _csr_from_sorted(n, r[order], c[order], v[order], dtype)


def band_plus_random(n: int, half: int, extra: int, rng: np.random.Generator,
                     dtype=np.float64) -> Csr:
    """Band |i-j| <= half plus `extra` distinct uniformly random off-band
    columns per row; values U(-1,1)."""
    chosen = np.full((n, extra), -1, np.int64)
    need = np.arange(n)
    filled = np.zeros(n, np.int64)
    while need.size:
        cand = rng.integers(0, n, size=(need.size, 3 * extra))
        r = need[:, None]
        ok = np.abs(cand - r) > half
        for q in range(cand.shape[1]):
            rows_q = need[ok[:, q]]
            cq = cand[ok[:, q], q]
            f = filled[rows_q]
            room = f < extra
            rows_q, cq, f = rows_q[room], cq[room], f[room]
            # reject duplicates of already chosen columns
            dup = (chosen[rows_q] == cq[:, None]).any(axis=1)
            rows_q, cq, f = rows_q[~dup], cq[~dup], f[~dup]
            # several candidates of one row in the same column q cannot clash
            chosen[rows_q, f] = cq
            filled[rows_q] = f + 1
        need = np.nonzero(filled < extra)[0]
    rows, cols = [], []
    base = np.arange(n, dtype=np.int64)
    for d in range(-half, half + 1):
        ok = (base + d >= 0) & (base + d < n)
        rows.append(base[ok])
        cols.append(base[ok] + d)
    rows.append(np.repeat(base, extra))
    cols.append(chosen.reshape(-1))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    v = rng.uniform(-1.0, 1.0, size=r.size)
    return _csr_from_sorted(n, r, c, v, dtype)


_M64 = (1 << 64) - 1


def _i64(c: int) -> int:
    """A uint64 constant as the int64 with the same bits."""
    c &= _M64
    return c - (1 << 64) if c >= 1 << 63 else c


def _srl(x, k: int):
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix64(x):
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    x = x ^ _srl(x, 30)
    x = x * _i64(0xBF58476D1CE4E5B9)
    x = x ^ _srl(x, 27)
    x = x * _i64(0x94D049BB133111EB)
    return x ^ _srl(x, 31)


def _uniform(seed: int, idx, level: int):
    """U[0,1) for draw `idx` at recursion level `level`: a counter-based hash,
    so CPU and GPU produce identical bits (both arms of bench.py, and the
    tests, see the same matrix whatever device generated it)."""
    import torch

    base = _i64(seed * 0xD1B54A32D192ED03 + level * 0x8CB92BA72F3D8DD7 + 0x9E3779B97F4A7C15)
    x = _mix64(idx * _i64(0x9E3779B97F4A7C15) + base)
    return _srl(x, 11).to(torch.float64) * (1.0 / (1 << 53))


def rmat_pattern(scale: int, draws: int, seed: int, abc=(0.57, 0.19, 0.19), device=None):
    """Symmetrised, deduplicated R-MAT edge set without self loops, as sorted
    (rows, cols) int64 numpy arrays.  Each draw descends `scale` levels; at
    level l it picks quadrant a / b / c / d from a counter-based uniform
    (`_uniform`), so the result is identical on CPU and CUDA.  torch (on
    `device`, default CUDA when available) only supplies the speed."""
    import torch

    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    a, b, c = abc
    n = 1 << scale
    chunk = 1 << 24
    keys = []
    for d0 in range(0, draws, chunk):
        idx = torch.arange(d0, min(draws, d0 + chunk), dtype=torch.int64, device=device)
        r = torch.zeros_like(idx)
        col = torch.zeros_like(idx)
        for lev in range(scale):
            u = _uniform(seed, idx, lev)
            rb = (u >= a + b).to(torch.int64)
            cb = (((u >= a) & (u < a + b)) | (u >= a + b + c)).to(torch.int64)
            r = r * 2 + rb
            col = col * 2 + cb
        keep = r != col
        r, col = r[keep], col[keep]
        keys.append(torch.cat([r * n + col, col * n + r]))
        del idx, r, col
    key = torch.unique(torch.cat(keys))
    rows = (key // n).cpu().numpy()
    cols = (key % n).cpu().numpy()
    return n, rows, cols


def make(name: str, scale: float = 1.0, seed: int = BASE_SEED, device=None) -> Workload:
    """Build BASELINE config `name` ('cfg1'..'cfg5').  scale < 1 shrinks it
    (used by the parity tests); scale = 1 is the BASELINE size."""
    rng_a = np.random.default_rng(seed)
    rng_b = np.random.default_rng(seed + 1)
    rng_c = np.random.default_rng(seed + 2)
    if name == "cfg1":
        n = max(64, int(65536 * scale))
        a = band_plus_random(n, 8, 8, rng_a)
        b = rng_b.uniform(-1, 1, size=(n, 64))
        c = rng_c.uniform(-1, 1, size=(64, 64))
        return Workload(name, "gemm-spmm", np.dtype(np.float64), a, b, c,
                        f"GeMM-SpMM fp64 band+-8+8rand n={n} bCol=cCol=64")
    if name == "cfg2":
        side = max(8, int(round(1024 * np.sqrt(scale))))
        a = stencil_2d(side)
        c = rng_c.uniform(-1, 1, size=(a.n_rows, 64))
        return Workload(name, "spmm-spmm", np.dtype(np.float64), a, a, c,
                        f"SpMM-SpMM fp64 9-pt {side}^2 n={a.n_rows} cCol=64")
    if name == "cfg4":
        side = max(4, int(round(128 * scale ** (1.0 / 3.0))))
        a = stencil_3d(side)
        c = rng_c.uniform(-1, 1, size=(a.n_rows, 128))
        return Workload(name, "spmm-spmm", np.dtype(np.float64), a, a, c,
                        f"SpMM-SpMM fp64 27-pt {side}^3 n={a.n_rows} cCol=128")
    if name in ("cfg3", "cfg5"):
        full_scale, deg = (20, 16) if name == "cfg3" else (23, 32)
        sc = max(6, int(round(full_scale + np.log2(scale)))) if scale < 1 else full_scale
        n = 1 << sc
        _, rows, cols = rmat_pattern(sc, n * deg // 2, seed, device=device)
        if name == "cfg3":
            diag = np.arange(n, dtype=np.int64)
            r = np.concatenate([rows, diag])
            c_ = np.concatenate([cols, diag])
            order = np.lexsort((c_, r))
            r, c_ = r[order], c_[order]
            deg_i = np.bincount(r, minlength=n).astype(np.float64)
            dinv = deg_i ** -0.5
            vals = dinv[r] * dinv[c_]
            a = _csr_from_sorted(n, r, c_, vals, np.float32)
            b = rng_b.standard_normal(size=(n, 128), dtype=np.float32)
            lim = np.sqrt(6.0 / 256.0)
            c = rng_c.uniform(-lim, lim, size=(128, 128)).astype(np.float32)
            return Workload(name, "gemm-spmm", np.dtype(np.float32), a, b, c,
                            f"GCN GeMM-SpMM fp32 R-MAT 2^{sc} deg16 bCol=cCol=128")
        deg_i = np.bincount(rows, minlength=n).astype(np.float64)
        vals = 1.0 / deg_i[rows]
        a = _csr_from_sorted(n, rows, cols, vals, np.float32)
        b = rng_b.standard_normal(size=(n, 256), dtype=np.float32)
        c = (rng_c.standard_normal(size=(256, 64)) / 16.0).astype(np.float32)
        return Workload(name, "gemm-spmm", np.dtype(np.float32), a, b, c,
                        f"GeMM-SpMM fp32 R-MAT 2^{sc} deg32 bCol=256 cCol=64")
    raise ValueError(f"unknown workload {name}")
