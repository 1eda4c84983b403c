"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tfg.h declares, host-only entry points work, and compute
entry points fail loudly (no CPU fallback) when no device is present."""
import os
import re

import numpy as np
import pytest

import paper_2407_00243_b200 as P
from paper_2407_00243_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tfg.h")).read()
    return sorted(set(re.findall(r"\b(tfg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(decl) == bound, set(decl) ^ bound


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_config_defaults_match_reference():
    c = _lib.TfgConfig()
    P.lib().tfg_config_default(c)
    d = P.SchedulerConfig()
    assert (c.ct_size, c.num_workers, c.cache_size_words, c.b_cols, c.c_cols) == (
        d.ct_size, d.num_workers, d.cache_size_words, d.b_cols, d.c_cols) == (2048, 1, 163840, 32, 32)
    assert c.index_to_scalar_ratio == 0.5 and c.b_is_dense == 1 and c.whole_b_cost == 0


def test_choose_tile_size_host(oracle):
    for args in [(10000, 3, 2048), (4096, 8, 2048), (8, 3, 4), (1, 1, 1), (65536, 148, 2048)]:
        assert P.choose_tile_size(*args) == oracle.choose_tile_size(*args)
    with pytest.raises(ValueError):
        P.choose_tile_size(0, 1, 1)


def test_generators_match_reference(oracle):
    for n, d, s in [(50, 0.1, 7), (300, 0.02, 123), (10, 1.0, 5), (1, 0.5, 3)]:
        a = P.gen_random_sparse(n, d, s)
        rp, ci, v = oracle.gen_random_sparse(n, d, s)
        assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
        assert np.array_equal(a.values, v)
        a.validate()
    b = P.gen_banded(6, 2)
    i, j = np.indices((6, 6))
    assert np.array_equal(b.to_dense(), np.where(np.abs(i - j) <= 2, 1.0, 0.0))
    with pytest.raises(ValueError):
        P.gen_banded(4, 4)
    with pytest.raises(ValueError):
        P.gen_random_sparse(4, 0.0)


def test_csr_validation_errors():  # csr.hpp:36-61, test_smoke.py:28-34
    a = P.Csr(2, 3, [0, 2, 3], [0, 2, 1], [1.0, 2.0, 3.0])
    assert a.nnz == 3 and np.array_equal(a.to_dense(), [[1, 0, 2], [0, 3, 0]]) and "Csr(2x3" in repr(a)
    with pytest.raises(ValueError):
        P.Csr(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError):
        P.Csr(1, 2, [0, 1], [5], [1.0])
    with pytest.raises(ValueError):
        P.Csr(1, 3, [0, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        P.Csr(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])


def test_shape_errors_raise_before_device():  # kernels.hpp:35-42, test_smoke.py:112-124
    a = P.gen_banded(8, 1)
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, np.ones((8, 4)), np.ones((5, 3)))
    with pytest.raises(ValueError):
        P.fused_gemm_spmm(a, np.ones((8, 4)), np.ones((4, 3)), workers=0)
    with pytest.raises(ValueError):
        P.unfused_spmm_spmm(a, np.ones((8, 4)), np.ones((4, 3)))
    with pytest.raises(ValueError):
        P.fused_spmm_spmm(a, np.ones((8, 4)), np.ones((4, 3)))
    rect = P.Csr(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        P.schedule_json(rect)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    a = P.gen_banded(16, 1)
    with pytest.raises(Exception) as e:
        P.build_schedule(a, P.SchedulerConfig())
    assert "CUDA" in str(e.value)


def test_workload_sizes_match_survey():
    from paper_2407_00243_b200 import workloads as W

    w = W.make("cfg1")
    assert w.n == 65536 and w.a.nnz == 1638328 and w.flops() == 746576896
    w = W.make("cfg2", scale=1 / 16)
    assert w.a.n_rows == 256 * 256
    w.a.validate()
    w = W.make("cfg4", scale=1 / 512)
    w.a.validate()
    assert w.a.n_rows == 16 ** 3
