"""CPU tests of the library's host-side polynomial set-up (no GPU): polya_homogenize and
polya_simplex_map (include/polya.h) against the oracle's explicit polynomial multiplication
(oracle.polya.homogenize / simplex_map, pinned in tests/test_oracle_examples.py).  The library
computes homogenisation by the closed form multinomial(d_a - d_t; gamma - e_t) and the map by
dense coefficient products; both are exact up to FP64 rounding of sums of integer-weighted terms."""
import numpy as np
import pytest

from oracle import polya
from oracle.monomials import enumerate_W


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    return pb


@pytest.mark.parametrize("l,n,seed", [(3, 2, 0), (4, 3, 1), (2, 1, 2), (5, 2, 3)])
def test_homogenize_matches_oracle(pb, l, n, seed):
    rng = np.random.default_rng(seed)
    terms = {}
    for _ in range(6):
        e = tuple(int(v) for v in rng.integers(0, 3, size=l))
        terms[e] = rng.normal(size=(n, n))
    da, B = pb.homogenize(terms, l)
    da_o, B_o = polya.homogenize(terms, l)
    assert da == da_o and B.shape == B_o.shape
    assert np.abs(B - B_o).max() <= 1e-13 * max(1.0, np.abs(B_o).max())


@pytest.mark.parametrize("l,d,n,seed", [(3, 3, 3, 0), (8, 1, 2, 1), (4, 2, 2, 2), (2, 5, 1, 3)])
def test_simplex_map_matches_oracle(pb, l, d, n, seed):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(len(enumerate_W(l, d)), n, n))
    scale, shift = rng.uniform(0.2, 2.0, size=l), rng.uniform(-1.0, 1.0, size=l)
    got = pb.simplex_map(A, l, d, scale, shift)
    want = polya.simplex_map(A, l, d, scale, shift)
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_homogenize_rejects_bad_input(pb):
    with pytest.raises(pb.PolyaError):
        pb.homogenize({(1, -1): np.eye(2)}, 2)
