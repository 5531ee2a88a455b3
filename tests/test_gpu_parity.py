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
         synth.small_config(14, 2, 2, 1, 1),      # ragged tail of 6 (rows x, z = 6, 7 never formed)
         synth.small_config(13, 3, 1, 1, 1),      # ragged tail of 5
         synth.small_config(1, 3, 1, 1, 1),       # n = 1 (single padded chunk)
         synth.small_config(5, 1, 0, 2, 3),       # l = 1, dp = 0 (K = Ntil)
         synth.small_config(6, 3, 2, 0, 0)]       # d1 = d2 = 0: pairs with no common block


FULL5 = [synth.CONFIGS[c] for c in (1, "1u", 2, 3, 4, 5)]   # BASELINE.json's five configs (+ cfg 1's unstable copy)


@pytest.mark.parametrize("cfg", SMALL[3:] + FULL5, ids=lambda c: c.name)
def test_setup_parity(pb, cfg):
    """Polya set-up (Eq. Cj): exponent tables and beta bit-exact, C exact
    to rounding, H within 1e-10 -- on every config (config 5's H, 21 x 792 blocks of 120 x 120, row by
    row through oracle.polya.H_row)."""
    ctx, A, X, W = _setup(pb, cfg)
    l, dp = cfg.l, cfg.dp
    for which, d in ((0, dp), (1, dp + cfg.d1), (2, dp + 1 + cfg.d2), (3, 1)):
        assert np.array_equal(ctx.exponents(which), np.array(enumerate_W(l, d), dtype=np.int32).reshape(-1, l))
    beta = opolya.beta_table(l, dp, cfg.d1)
    assert np.array_equal(ctx.beta(), beta)
    Hg = ctx.H()
    if ctx.L0 * ctx.M * cfg.n ** 2 <= 2e7:
        assert _rel(Hg, opolya.H_table(A, l, dp, cfg.d2)) <= TOL
    else:
        for h in range(ctx.L0):
            assert _rel(Hg[h], opolya.H_row(A, l, dp, cfg.d2, h)) <= TOL, h
    del Hg
    cref = opolya.C_scalars(beta, l, dp, 1e-3)
    assert np.array_equal(ctx.C(), cref) or _rel(ctx.C(), cref) <= 1e-15
    ctx.close()


@pytest.mark.parametrize("cfg", SMALL + [synth.CONFIGS[c] for c in (3, 4, 5)], ids=lambda c: c.name)
def test_apply_adjoint_parity(pb, cfg):
    """B^T(y) (Eq. AT) and B(X) on every config."""
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
    """Config 3: every entry of G (K = 4,650) against the literal Eq. T2 (dense F, traces)."""
    cfg = synth.CONFIGS[3]
    ctx, A, X, W = _setup(pb, cfg)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    G = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    Gref = osdp.schur_literal(P, X, W)
    assert _rel(G, Gref) <= TOL
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


def _tiles_row(T, i, L0, N):
    """Row i of G from the PAIR_TILES layout (tile p(h, h') holds G[h-rows, h'-columns], h <= h')."""
    h, s = divmod(i, N)
    parts = []
    for h2 in range(L0):
        a, b = (h, h2) if h <= h2 else (h2, h)
        p = a * L0 - a * (a - 1) // 2 + (b - a)
        parts.append(T[p, s, :] if h <= h2 else T[p, :, s])
    return torch.cat(parts)


def _strat_indices(P, rng, count):
    """Stratified dual indices i = (h, k): every h, diagonal / off-diagonal basis elements, the first and
    last elements of each kind and off-diagonal elements touching the ragged last index n-1."""
    n, N = P.n, P.Ntil
    pos = {ab: k for k, ab in enumerate(osdp.basis(n))}
    out = []
    for c in range(count):
        h = c % P.L0
        kind = (c // P.L0) % 4
        if kind == 0 or n == 1:
            k = int(rng.integers(n))                           # diagonal (a, a)
        elif kind == 1:
            k = int(rng.integers(n, N))                        # off-diagonal (a, a+o)
        elif kind == 2:
            k = (0, n - 1, n, N - 1)[(c // (4 * P.L0)) % 4]    # edges of the basis order
        else:
            o = int(rng.integers(1, n))                        # (n-1-o, n-1): the ragged last index
            k = pos[(n - 1 - o, n - 1)]
        out.append(h * N + k)
    return out


def _sample_pairs(P, rng, count, pool):
    """Stratified (i, j) from the index pool: diagonal / off-diagonal k on each side x h = h' / h != h'
    (SURVEY 8(c) O6'(i))."""
    n, N = P.n, P.Ntil
    diag = lambda i: (i % N) < n   # noqa: E731
    side = {True: [i for i in pool if diag(i)], False: [i for i in pool if not diag(i)]}
    out = []
    for c in range(count):
        want_i, same_h, want_j = (c // 2) % 2 == 0, c % 2 == 0, (c // 4) % 2 == 0
        ci = side[want_i] or pool
        i = ci[int(rng.integers(len(ci)))]
        cj = [j for j in side[want_j] if (j // N == i // N) == same_h] or pool
        out.append((i, cj[int(rng.integers(len(cj)))]))
    return out


@pytest.mark.parametrize("cfg_id,layout,nrows,npool,nent", [(4, 0, 64, 256, 2048), (5, 1, 8, 64, 256)])
def test_schur_large_rows_entries_probes(pb, cfg_id, layout, nrows, npool, nent):
    """Configs 4 and 5 (G of 20 GB / 186 GB): against the literal Eq. T2 of the oracle --
    whole stratified rows (oracle.sdp.schur_rows: row k = B(X F_k Z^-1) with dense F_k), stratified
    entries (oracle.sdp.schur_entries: one trace of the four-matrix product per entry) with the bar
    |dG_ij| <= 1e-10 sqrt(G_ii G_jj), and 8 matrix-free probes G v = B(Z^-1 B^T(v) X)
    (SURVEY 8(c) O6'(i)-(ii)).  None of these routes goes through the rank-structured four-term
    expansion the kernel uses."""
    cfg = synth.CONFIGS[cfg_id]
    ctx, A, X, W = _setup(pb, cfg)
    G = ctx.schur(_dev(X), _dev(W), layout=layout)
    torch.cuda.synchronize()
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    rng = np.random.default_rng(11)
    # whole rows
    rows = _strat_indices(P, rng, nrows)
    ref = osdp.schur_rows(P, X, W, rows)
    for r, i in enumerate(rows):
        got = (G[i] if layout == 0 else _tiles_row(G, i, P.L0, P.Ntil)).cpu().numpy()
        assert _rel(got, ref[r]) <= TOL, i
    # stratified entries
    pool = sorted(set(_strat_indices(P, rng, npool)))
    pairs = _sample_pairs(P, rng, nent, pool)
    dref = dict(zip(pool, osdp.schur_entries(P, X, W, [(i, i) for i in pool])))
    ent = osdp.schur_entries(P, X, W, pairs)
    for (i, j), r in zip(pairs, ent):
        got = float(G[i, j]) if layout == 0 else _tiles_entry(G, i, j, P.L0, P.Ntil)
        assert abs(got - r) <= TOL * np.sqrt(dref[i] * dref[j]), (i, j, got, r)
    # 8 probes
    V = rng.normal(size=(8, P.K))
    gv_ref = osdp.schur_probe(P, X, W, V)
    for p in range(8):
        vd = _dev(V[p])
        gv = (G @ vd if layout == 0 else _tiles_matvec(G, vd, P.L0, P.Ntil)).cpu().numpy()
        assert _rel(gv, gv_ref[p]) <= TOL, p
    del G
    ctx.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [125, 128, 130, 168])
def test_schur_precompute_size_boundary(pb, n):
    """The SCM precompute switches kernels at np = 128 (K3b row-gathered GEMMs up to it, K3 batched GEMMs
    beyond): n = 125 (np = 128, ragged tail of 5), 128 (np = 128, no tail), 130 (np = 136), and the
    largest block order 168 (21 chunks) -- whole stratified rows, stratified entries and 2 probes of G
    against the literal Eq. T2."""
    cfg = synth.small_config(n, 2, 1, 1, 1)
    ctx, A, X, W = _setup(pb, cfg)
    G = ctx.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES)
    torch.cuda.synchronize()
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    rng = np.random.default_rng(5)
    rows = _strat_indices(P, rng, 8)
    ref = osdp.schur_rows(P, X, W, rows)
    for r, i in enumerate(rows):
        assert _rel(_tiles_row(G, i, P.L0, P.Ntil).cpu().numpy(), ref[r]) <= TOL, i
    pool = sorted(set(_strat_indices(P, rng, 32)))
    pairs = _sample_pairs(P, rng, 128, pool)
    dref = dict(zip(pool, osdp.schur_entries(P, X, W, [(i, i) for i in pool])))
    for (i, j), r in zip(pairs, osdp.schur_entries(P, X, W, pairs)):
        got = _tiles_entry(G, i, j, P.L0, P.Ntil)
        assert abs(got - r) <= TOL * np.sqrt(dref[i] * dref[j]), (i, j, got, r)
    V = rng.normal(size=(2, P.K))
    gv_ref = osdp.schur_probe(P, X, W, V)
    for p in range(2):
        gv = _tiles_matvec(G, _dev(V[p]), P.L0, P.Ntil).cpu().numpy()
        assert _rel(gv, gv_ref[p]) <= TOL, p
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
