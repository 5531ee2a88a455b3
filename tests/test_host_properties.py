"""Property tests (hypothesis) of the library's host-side logic on random small shapes, no GPU:
polya_plan's shares partition the Schur work items (output tiles) and the Polya blocks (block
sharding) for any rank count, and the FLOP accounting always sums to W_G = n^4 (sum nu^2 +
4 sum mu^2) with nu, mu counted from the oracle's beta and H; polya_homogenize agrees with the
oracle's polynomial multiplication on random term sets."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import polya


def _wg(n, l, dp, d1, d2):
    beta = polya.beta_table(l, dp, d1)
    A = np.random.default_rng(0).normal(size=(l, 2, 2))
    H = polya.H_table(A, l, dp, d2)
    nu = (beta != 0).sum(axis=0)
    mu = np.array([sum(np.any(H[h, m] != 0) for h in range(H.shape[0])) for m in range(H.shape[1])])
    return float(n) ** 4 * (float((nu ** 2).sum()) + 4.0 * float((mu ** 2).sum()))


shapes = st.tuples(st.integers(1, 24), st.integers(1, 4), st.integers(0, 3), st.integers(0, 3), st.integers(0, 3))


@settings(max_examples=40, deadline=None)
@given(shape=shapes, world=st.integers(1, 9))
def test_plan_partitions(shape, world):
    import paper_1411_3769_b200 as pb
    n, l, dp, d1, d2 = shape
    wg = _wg(*shape)
    total = pb.plan(*shape)["item1"]
    nb = pb.plan(*shape)["b1"]
    t = [pb.plan(*shape, rank=r, nranks=world) for r in range(world)]
    b = [pb.plan(*shape, rank=r, nranks=world, shard=pb.SHARD_BLOCKS) for r in range(world)]
    assert t[0]["item0"] == 0 and t[-1]["item1"] == total
    assert all(t[r]["item1"] == t[r + 1]["item0"] for r in range(world - 1))
    assert b[0]["b0"] == 0 and b[-1]["b1"] == nb
    assert all(b[r]["b1"] == b[r + 1]["b0"] for r in range(world - 1))
    for d in (t, b):
        assert abs(sum(x["useful_flops_schur"] for x in d) - wg) <= 1e-9 * max(wg, 1.0)


@settings(max_examples=30, deadline=None)
@given(l=st.integers(1, 4), n=st.integers(1, 3), seed=st.integers(0, 10 ** 6))
def test_homogenize_property(l, n, seed):
    import paper_1411_3769_b200 as pb
    rng = np.random.default_rng(seed)
    terms = {}
    for _ in range(int(rng.integers(1, 5))):
        terms[tuple(int(v) for v in rng.integers(0, 3, size=l))] = rng.normal(size=(n, n))
    da, B = pb.homogenize(terms, l)
    da_o, B_o = polya.homogenize(terms, l)
    assert da == da_o
    assert np.abs(B - B_o).max() <= 1e-13 * max(1.0, np.abs(B_o).max())
