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
