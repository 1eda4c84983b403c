"""The reference's synthetic generators (generate.hpp:15-94; exposed by the
reference's Python module, bindings.cpp:111-114) as host-side Python.

Inputs, not the hot path: the random stream must match the reference's
std::mt19937_64 (53-bit draws, geometric column skips), so a 64-bit
Mersenne Twister is restated here (the standard MT19937-64 recurrence:
312-word state, tempering (29, 17, 37, 43)).  Checked bit-for-bit against
the reference's own generator in tests/test_generate.py.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (seed via the standard 6364136223846793005 init)."""

    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self.N
        mt[0] = seed & _M64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.idx = mt, self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        x = self.mt[self.idx]
        self.idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


def gen_random_sparse(n: int, density: float, seed: int = 42):
    """generate.hpp:15-63: each entry present with probability `density`
    (geometric skips), values U[0.1, 1], an empty row gets its diagonal."""
    from .tilefuse import Csr

    n = int(n)
    if n < 1:
        raise ValueError("gen_random_sparse: n must be >= 1")
    if not (density > 0.0) or density > 1.0:
        raise ValueError("gen_random_sparse: density must be in (0,1]")
    rng = MT19937_64(int(seed))
    two53 = 2.0 ** -53

    def value():
        return 0.1 + 0.9 * float(rng() >> 11) * two53

    full = density >= 1.0
    log_skip = 0.0 if full else math.log1p(-density)
    rp, ci, v = [0], [], []
    for r in range(n):
        start = len(ci)
        if full:
            for c in range(n):
                ci.append(c)
                v.append(value())
        else:
            c = -1
            while True:
                c += 1 + int(math.floor(math.log((float(rng() >> 11) + 0.5) * two53) / log_skip))
                if c >= n:
                    break
                ci.append(c)
                v.append(value())
        if len(ci) == start:
            ci.append(r)
            v.append(value())
        rp.append(len(ci))
    return Csr(n, n, np.array(rp, np.int32), np.array(ci, np.int32), np.array(v, np.float64))


def gen_banded(n: int, half_bandwidth: int):
    """generate.hpp:66-94: |i - j| <= half_bandwidth, every value 1."""
    from .tilefuse import Csr

    n, hb = int(n), int(half_bandwidth)
    if n < 1:
        raise ValueError("gen_banded: n must be >= 1")
    if hb < 0 or hb >= n:
        raise ValueError("gen_banded: need 0 <= half_bandwidth < n")
    r = np.arange(n)
    lo, hi = np.maximum(0, r - hb), np.minimum(n - 1, r + hb)
    counts = hi - lo + 1
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.concatenate([np.arange(a, b + 1) for a, b in zip(lo, hi)]) if n else np.zeros(0)
    return Csr(n, n, rp.astype(np.int32), ci.astype(np.int32), np.ones(ci.size))
