"""Matrix Market I/O (row f3) -- the reference's parse rules and errors
(matrix_market.cpp:21-89, test_smoke.py:48-57), and report rows (row f2)."""
import numpy as np
import pytest

from paper_2407_00243_b200 import matrix_market as MM
from paper_2407_00243_b200 import report as R


def test_reference_smoke_file(tmp_path):  # tests/python/test_smoke.py:48-57
    p = tmp_path / "tiny.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 4.0\n2 1 -1.5\n")
    a = MM.load_matrix_market(str(p))
    assert np.array_equal(a.to_dense(), [[4.0, 0.0], [-1.5, 0.0]])


def test_symmetric_pattern_duplicates_comments(tmp_path):
    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n% c\n\n3 3 3\n1 1\n3 1\n% mid\n3 1\n")
    a = MM.load_matrix_market(str(p))
    assert np.array_equal(a.to_dense(), [[1, 0, 2], [0, 0, 0], [2, 0, 0]])
    a.validate()


@pytest.mark.parametrize("text", [
    "", "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n"])
def test_malformed_inputs_raise(tmp_path, text):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(RuntimeError):
        MM.load_matrix_market(str(p))


def test_round_trip_exact(tmp_path, oracle):
    rp, ci, v = oracle.gen_random_sparse(40, 0.1, 3)
    from paper_2407_00243_b200 import Csr

    a = Csr(40, 40, rp, ci, v / 3.0)
    p = tmp_path / "rt.mtx"
    MM.write_matrix_market(a, str(p))
    b = MM.load_matrix_market(str(p))
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
    with pytest.raises(RuntimeError):
        MM.load_matrix_market(str(tmp_path / "missing.mtx"))


def test_report_csv_and_json():
    rows = [R.Row("m", 4, 7, "gemm-spmm", "fused", "dp", 2, 3, 1, 7, 0.5, 1.0, 0.25, 0.1, float("inf")),
            R.Row("m", 4, 7, "gemm-spmm", "unfused", "dp", 2, 3, 1, 7, 0.4, 1.25)]
    csv = R.rows_to_csv(rows).splitlines()
    assert csv[0] == R.HEADER and csv[1].endswith(",inf,,gpu") and csv[2].split(",")[12] == ""
    js = R.rows_to_json(rows)
    assert '"runs_to_amortize": "inf"' in js and '"fused_ratio": null' in js


@pytest.mark.gpu
@pytest.mark.parametrize("symmetric", [False, True])
def test_loaded_mtx_through_gpu_path(tmp_path, cuda, oracle, symmetric):
    """Row f3 end to end: a .mtx file written with the reference's rules
    (matrix_market.cpp:21-89; symmetric files mirror the off-diagonal entries,
    duplicates add) is loaded, scheduled by the GPU inspector and executed on
    the B200; schedule and D are checked against the oracle on the same CSR."""
    import paper_2407_00243_b200 as P
    from helpers import max_rel_err, schedules_equal
    from oracle.oracle import SchedulerConfig as OCfg

    n = 600
    rp, ci, v = oracle.gen_random_sparse(n, 0.015, 11)
    p = tmp_path / ("sym.mtx" if symmetric else "gen.mtx")
    if symmetric:
        rows = np.repeat(np.arange(n), np.diff(rp))
        keep = rows >= ci  # lower triangle; the loader mirrors it
        lines = [f"{r + 1} {c + 1} {x:.17g}" for r, c, x in zip(rows[keep], ci[keep], v[keep])]
        lines.append(lines[0])  # a duplicate entry: values add (matrix_market.cpp:70-85)
        p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% from test\n"
                     f"{n} {n} {len(lines)}\n" + "\n".join(lines) + "\n")
    else:
        MM.write_matrix_market(P.Csr(n, n, rp, ci, v), str(p))
    a = MM.load_matrix_market(str(p))
    a.validate()
    rng = np.random.default_rng(2)
    b = rng.uniform(-1, 1, (n, 32))
    c = rng.uniform(-1, 1, (32, 16))
    cfg = P.SchedulerConfig(ct_size=64, num_workers=8, cache_size_words=4096, b_cols=32, c_cols=16)
    sched = P.build_schedule(a, cfg)
    want_s = oracle.build_schedule(n, n, a.row_ptr, a.col_idx, OCfg(**cfg.__dict__))
    assert schedules_equal(sched.export(), want_s)
    triple = (a.row_ptr, a.col_idx, a.values)
    got = P.run(a, b, c, sched, np.float64)
    assert max_rel_err(got, oracle.run(n, triple, b, c, want_s, np.float64)) <= 1e-12
    # SpMM-SpMM with the loaded matrix on both sides: bit-exact with reference bits
    cs = rng.uniform(-1, 1, (n, 8))
    cfg2 = P.SchedulerConfig(ct_size=64, num_workers=8, cache_size_words=4096, b_cols=n, c_cols=8,
                             b_is_dense=False)
    s2 = P.build_schedule(a, cfg2)
    w2 = oracle.build_schedule(n, n, a.row_ptr, a.col_idx, OCfg(**cfg2.__dict__))
    assert schedules_equal(s2.export(), w2)
    got2 = P.run(a, a, cs, s2, np.float64)
    assert max_rel_err(got2, oracle.run(n, triple, triple + (n,), cs, w2, np.float64)) <= 1e-12
