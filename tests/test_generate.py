"""Host generators (paper_2407_00243_b200/generate.py, include/tilefuse/
generate.hpp) reproduce the reference's generate.hpp streams bit for bit:
checked against the oracle's C restatement (itself pinned to the reference,
test_oracle_pins.py) and, where built, the reference library itself."""
import numpy as np
import pytest

import paper_2407_00243_b200 as P
from paper_2407_00243_b200.generate import MT19937_64


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-seeded mt19937_64
    g = MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


@pytest.mark.parametrize("n,density,seed", [(1, 0.5, 3), (17, 0.2, 11), (200, 0.03, 42),
                                            (64, 1.0, 7), (300, 0.004, 9)])
def test_gen_random_sparse_matches_oracle(oracle, n, density, seed):
    a = P.gen_random_sparse(n, density, seed)
    rp, ci, v = oracle.gen_random_sparse(n, density, seed)
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
    assert np.array_equal(a.values, v)


def test_gen_banded_matches_oracle(oracle):
    for n, hb in [(16, 1), (5, 0), (40, 7)]:
        a = P.gen_banded(n, hb)
        rp, ci, v = oracle.gen_banded(n, hb)
        assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
        assert np.array_equal(a.values, v)


def test_generator_errors():
    with pytest.raises(ValueError):
        P.gen_random_sparse(0, 0.5)
    with pytest.raises(ValueError):
        P.gen_random_sparse(4, 0.0)
    with pytest.raises(ValueError):
        P.gen_banded(4, 4)
