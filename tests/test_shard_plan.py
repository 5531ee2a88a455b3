"""Host-only checks of the block partition of SHARD_BLOCKS (polya_plan, no GPU): for every
BASELINE config shape and 1..8 ranks, the ranges [b0, b1) tile the Polya blocks contiguously,
each rank's algorithmic FLOPs equal n^4 (sum over its blocks of nu_j^2 + 4 mu_m^2) with nu, mu
counted from the ORACLE's beta and H, and the split is balanced to within one block's cost
(the paper's count balancing leaves up to 50 % idle)."""
import numpy as np
import pytest

SHAPES = [(4, 2, 1, 1, 1), (10, 3, 2, 2, 2), (30, 4, 2, 3, 3), (100, 4, 2, 4, 4), (120, 6, 2, 4, 4)]


def _block_costs(n, l, dp, d1, d2):
    from oracle import polya
    beta = polya.beta_table(l, dp, d1)
    A = np.random.default_rng(0).normal(size=(l, 2, 2))
    H = polya.H_table(A, l, dp, d2)
    nu = (beta != 0).sum(axis=0)
    mu = np.array([sum(np.any(H[h, m] != 0) for h in range(H.shape[0])) for m in range(H.shape[1])])
    return float(n) ** 4 * np.concatenate([nu.astype(float) ** 2, 4.0 * mu.astype(float) ** 2])


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "n%d_l%d" % (s[0], s[1]))
def test_block_partition(shape):
    import paper_1411_3769_b200 as pb
    cost = _block_costs(*shape)
    nb = len(cost)
    for world in range(1, 9):
        ds = [pb.plan(*shape, rank=r, nranks=world, shard=pb.SHARD_BLOCKS) for r in range(world)]
        assert ds[0]["b0"] == 0 and ds[-1]["b1"] == nb
        for r in range(world - 1):
            assert ds[r]["b1"] == ds[r + 1]["b0"]
        for d in ds:
            own = cost[d["b0"]:d["b1"]].sum()
            assert abs(d["useful_flops_schur"] - own) <= 1e-9 * max(own, 1.0)
            assert d["item0"] == 0 and d["item1"] == ds[0]["item1"]
            npairs, Ntil, t = d["npairs"], d["Ntil"], d["combine_tiles"]
            groups = -(-npairs // (world * t))
            assert t >= 1 and d["reduce_count"] == groups * t * Ntil * Ntil
            assert (groups - 1) * world * t < npairs <= groups * world * t     # no empty group
            assert t == 1 or world * t * Ntil * Ntil * 8 <= 2 << 30 or t == -(-npairs // world)
        mx = max(d["useful_flops_schur"] for d in ds)
        assert mx <= cost.sum() / world + cost.max() + 1e-6
        # tiles mode: all blocks on every rank
        dt = pb.plan(*shape, rank=0, nranks=world)
        assert dt["b0"] == 0 and dt["b1"] == nb and dt["reduce_count"] == 0


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "n%d_l%d" % (s[0], s[1]))
def test_cyclic_partition(shape):
    """SHARD_CYCLIC (the distributed factorisation's layout): rank r holds the pair rows h = r mod N
    completely -- local pairs of all ranks partition the pairs, their FLOPs add up to the total, and
    the item numbering is per rank from 0."""
    import paper_1411_3769_b200 as pb
    total = pb.plan(*shape)["useful_flops_schur"]
    for world in (1, 2, 3, 8):
        ds = [pb.plan(*shape, rank=r, nranks=world, shard=pb.SHARD_CYCLIC) for r in range(world)]
        L0 = ds[0]["L0"]
        assert sum(d["npairs_local"] for d in ds) == ds[0]["npairs"]
        for r, d in enumerate(ds):
            rows = [h for h in range(L0) if h % world == r]
            assert d["npairs_local"] == sum(L0 - h for h in rows)
            assert d["item0"] == 0
            assert d["tiles_bytes"] == d["npairs_local"] * d["Ntil"] ** 2 * 8
        assert abs(sum(d["useful_flops_schur"] for d in ds) - total) <= 1e-9 * total
