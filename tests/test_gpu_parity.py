"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): exponent tables, beta and the pair /
item bookkeeping bit-exact; H, C, B^T(y) blocks and G within 1e-10 relative
Frobenius error; B(X) within 1e-10 relative 2-norm; configs 4-5 G on sampled
entries |dG_ij| <= 1e-10 sqrt(G_ii G_jj) and probes ||G v - (G v)_ref|| / ||(G v)_ref|| <= 1e-10.
"""
import numpy as np
import pytest

import synth
from oracle import polya as opolya
from oracle import sdp as osdp
from oracle.monomials import enumerate_W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    assert torch.cuda.is_available()
    return pb


def _setup(pb, cfg, seed=0, rank=0, nranks=1, A=None, nblocks=None):
    rng = np.random.default_rng(seed)
    if A is None:
        A = synth.vertex_matrices(cfg, rng)
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=nranks)
    X, W = synth.spd_blocks(cfg.n, ctx.nblocks, rng)
    return ctx, A, X, W


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


SMALL = [synth.CONFIGS[1], synth.CONFIGS["1u"], synth.CONFIGS[2],
         synth.small_config(12, 3, 2, 1, 2),      # np = 16: two chunks, ragged tail of 4
         synth.small_config(9, 2, 1, 2, 1),       # ragged tail of 1
         synth.small_config(20, 2, 2, 1, 1),      # three chunks, ragged tail of 4
         synth.small_config(1, 3, 1, 1, 1),       # n = 1 (single padded chunk)
         synth.small_config(5, 1, 0, 2, 3),       # l = 1, dp = 0 (K = Ntil)
         synth.small_config(6, 3, 2, 0, 0)]       # d1 = d2 = 0: pairs with no common block


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
def test_setup_parity(pb, cfg):
    ctx, A, X, W = _setup(pb, cfg)
    l, dp = cfg.l, cfg.dp
    for which, d in ((0, dp), (1, dp + cfg.d1), (2, dp + 1 + cfg.d2), (3, 1)):
        assert np.array_equal(ctx.exponents(which), np.array(enumerate_W(l, d), dtype=np.int32).reshape(-1, l))
    assert np.array_equal(ctx.beta(), opolya.beta_table(l, dp, cfg.d1))
    Href = opolya.H_table(A, l, dp, cfg.d2)
    assert _rel(ctx.H(), Href) <= TOL
    cref = opolya.C_scalars(opolya.beta_table(l, dp, cfg.d1), l, dp, 1e-3)
    assert np.array_equal(ctx.C(), cref) or _rel(ctx.C(), cref) <= 1e-15
    ctx.close()


@pytest.mark.parametrize("cfg", SMALL + [synth.CONFIGS[3]], ids=lambda c: c.name)
def test_apply_adjoint_parity(pb, cfg):
    ctx, A, X, W = _setup(pb, cfg)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    rng = np.random.default_rng(42)
    y = rng.normal(size=P.K)
    got = ctx.apply(_dev(y)).cpu().numpy()
    assert _rel(got, osdp.apply_vmap(P, y)) <= TOL
    R = rng.normal(size=X.shape)            # non-symmetric argument: only sym part matters
    gy = ctx.adjoint(_dev(R)).cpu().numpy()
    assert _rel(gy, osdp.adjoint_trace(P, R)) <= TOL
    ctx.close()


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
def test_schur_full_parity(pb, cfg):
    ctx, A, X, W = _setup(pb, cfg)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    G = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    Gref = osdp.schur_literal(P, X, W)
    assert _rel(G, Gref) <= TOL
    assert np.array_equal(G, G.T)           # FULL layout mirrors bit-exactly
    ctx.close()


def test_schur_pair_tiles_matches_full(pb):
    cfg = synth.small_config(12, 3, 2, 1, 2)
    ctx, A, X, W = _setup(pb, cfg)
    Gf = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    T = ctx.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES).cpu().numpy()
    N = ctx.Ntil
    p = 0
    for h in range(ctx.L0):
        for h2 in range(h, ctx.L0):
            assert np.array_equal(T[p], Gf[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N])
            p += 1
    ctx.close()


def test_schur_rank_sharding_bitwise(pb):
    """Output-tile sharding: the union of the ranks' work items equals the single-rank G bit for bit."""
    cfg = synth.CONFIGS[2]
    ctx, A, X, W = _setup(pb, cfg)
    Xd, Wd = _dev(X), _dev(W)
    G1 = ctx.schur(Xd, Wd)
    ctx.close()
    for nranks in (2, 3, 5):
        G = torch.full_like(G1, float("nan"))
        items = []
        for r in range(nranks):
            c = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=nranks)
            items.append((c.dims["item0"], c.dims["item1"]))
            c.schur(Xd, Wd, G=G)
            c.close()
        assert items[0][0] == 0 and all(items[i][1] == items[i + 1][0] for i in range(nranks - 1))
        assert torch.equal(G, G1)


def test_schur_config3(pb):
    cfg = synth.CONFIGS[3]
    ctx, A, X, W = _setup(pb, cfg)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    G = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    rng = np.random.default_rng(3)
    rows = sorted(set([h * P.Ntil + k for h in range(P.L0) for k in (0, 1, cfg.n, P.Ntil - 1)]) |
                  set(rng.integers(0, P.K, size=64).tolist()))
    Gref = osdp.schur_literal(P, X, W, rows=rows)
    assert _rel(G[rows], Gref) <= TOL
    assert np.array_equal(G, G.T)
    ctx.close()


def _tiles_matvec(T, v, L0, N):
    out = torch.zeros_like(v)
    p = 0
    for h in range(L0):
        for h2 in range(h, L0):
            out[h * N:(h + 1) * N] += T[p] @ v[h2 * N:(h2 + 1) * N]
            if h2 != h:
                out[h2 * N:(h2 + 1) * N] += T[p].T @ v[h * N:(h + 1) * N]
            p += 1
    return out


def _tiles_entry(T, i, j, L0, N):
    hi, si = divmod(i, N)
    hj, sj = divmod(j, N)
    if hi > hj:
        hi, hj, si, sj = hj, hi, sj, si
    p = hi * L0 - hi * (hi - 1) // 2 + (hj - hi)
    return float(T[p, si, sj])


def _sample_pairs(P, rng, count):
    """Stratified (i, j): P/Lyapunov-heavy rows x diagonal/off-diagonal basis x h = h' / h != h'."""
    out = []
    n = P.n
    for c in range(count):
        h = int(rng.integers(P.L0))
        h2 = h if c % 2 == 0 else int(rng.integers(P.L0))
        k1 = int(rng.integers(n)) if c % 4 < 2 else int(rng.integers(n, P.Ntil))
        k2 = int(rng.integers(n)) if (c // 4) % 2 == 0 else int(rng.integers(n, P.Ntil))
        out.append((h * P.Ntil + k1, h2 * P.Ntil + k2))
    return out


@pytest.mark.parametrize("cfg_id,layout,nsamp", [(4, 0, 24), (5, 1, 8)])
def test_schur_large_sampled_and_probe(pb, cfg_id, layout, nsamp):
    cfg = synth.CONFIGS[cfg_id]
    ctx, A, X, W = _setup(pb, cfg)
    G = ctx.schur(_dev(X), _dev(W), layout=layout)
    torch.cuda.synchronize()
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    rng = np.random.default_rng(11)
    pairs = _sample_pairs(P, rng, nsamp)
    diag_idx = sorted({i for pr in pairs for i in pr})
    dref = dict(zip(diag_idx, osdp.schur_entries(P, X, W, [(i, i) for i in diag_idx])))
    ref = osdp.schur_entries(P, X, W, pairs)
    for (i, j), r in zip(pairs, ref):
        got = float(G[i, j]) if layout == 0 else _tiles_entry(G, i, j, P.L0, P.Ntil)
        assert abs(got - r) <= TOL * np.sqrt(dref[i] * dref[j]), (i, j, got, r)
    v = rng.normal(size=P.K)
    gv_ref = osdp.schur_probe(P, X, W, v)
    vd = _dev(v)
    gv = (G @ vd if layout == 0 else _tiles_matvec(G, vd, P.L0, P.Ntil)).cpu().numpy()
    assert _rel(gv, gv_ref) <= TOL
    del G
    ctx.close()
    torch.cuda.empty_cache()


def test_schur_more_ranks_than_items(pb):
    """Config 1 has 3 work items; with 8 ranks most shares are empty (allowed): those ranks
    write nothing, polya_schur returns OK, and the union is still G bit for bit."""
    cfg = synth.CONFIGS[1]
    ctx, A, X, W = _setup(pb, cfg)
    Xd, Wd = _dev(X), _dev(W)
    G1 = ctx.schur(Xd, Wd)
    ctx.close()
    G = torch.full_like(G1, float("nan"))
    empty = 0
    for r in range(8):
        c = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=8)
        empty += c.dims["item1"] == c.dims["item0"]
        if c.dims["item1"] == c.dims["item0"]:
            assert c.dims["useful_flops_schur"] == 0.0
        c.schur(Xd, Wd, G=G)
        c.close()
    assert empty >= 5
    assert torch.equal(G, G1)
