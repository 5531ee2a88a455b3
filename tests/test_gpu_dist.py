"""The distributed factorisation (SHARD_CYCLIC) on one GPU:

* each rank's CYCLIC assembly is exactly the single-rank pair tiles of its pair rows h = r mod N;
* polya_factor_solve_loopback -- all ranks' contexts in one process, one host thread per rank running
  the same dist_potrf (with look-ahead) / dist_potrs as the NCCL path, the collectives through an
  in-process group (barrier + device copies) -- solves G x = b like a dense solve (1e-10) and bit for
  bit like the one-rank factorisation, for N = 1..4 ranks; a failure on one rank (an indefinite
  diagonal tile met by its owner at a later step) reaches every rank through the per-step agreement;
* polya_ipm_step with SHARD_CYCLIC (one rank, with and without a one-rank NCCL communicator)
  equals the single-GPU tiled step; the solve converges the same way.
"""
import numpy as np
import pytest

import synth
from oracle import sdp as osdp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    assert torch.cuda.is_available()
    return pb


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


CASES = [synth.CONFIGS[2], synth.small_config(9, 3, 3, 1, 1), synth.small_config(6, 4, 2, 1, 1)]


def _tiles(pb, cfg, A, X, W, rank=0, nranks=1, shard=0):
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=nranks, shard=shard)
    return ctx, ctx.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES)


def _pairs(L0):
    return [(h, h2) for h in range(L0) for h2 in range(h, L0)]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_cyclic_assembly_is_the_owned_tiles(pb, cfg):
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    ctx0 = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    X, W = synth.spd_blocks(cfg.n, ctx0.nblocks, rng)
    full = ctx0.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES).cpu().numpy()
    pairs = _pairs(ctx0.L0)
    for world in (2, 3):
        for r in range(world):
            ctx, G = _tiles(pb, cfg, A, X, W, rank=r, nranks=world, shard=pb.SHARD_CYCLIC)
            mine = [p for p, (h, _) in enumerate(pairs) if h % world == r]
            assert G.shape[0] == len(mine) == ctx.dims["npairs_local"]
            assert np.array_equal(G.cpu().numpy(), full[mine])
            ctx.close()
    ctx0.close()


def _dense(full, L0, N):
    G = np.zeros((L0 * N, L0 * N))
    for p, (h, h2) in enumerate(_pairs(L0)):
        G[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N] = full[p]
        G[h2 * N:(h2 + 1) * N, h * N:(h + 1) * N] = full[p].T
    return G


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_loopback_factor_solve(pb, cfg):
    rng = np.random.default_rng(1)
    A = synth.vertex_matrices(cfg, rng)
    ctx0 = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    X, W = synth.spd_blocks(cfg.n, ctx0.nblocks, rng)
    full = ctx0.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES).cpu().numpy()
    L0, N, K = ctx0.L0, ctx0.Ntil, ctx0.K
    ctx0.close()
    b = rng.normal(size=K)
    ref = np.linalg.solve(_dense(full, L0, N), b)
    pairs = _pairs(L0)
    xs = {}
    for world in (1, 2, 3, 4):
        ctxs = [pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world, shard=pb.SHARD_CYCLIC)
                for r in range(world)]
        Gs = [_dev(full[[p for p, (h, _) in enumerate(pairs) if h % world == r]]) for r in range(world)]
        x = _dev(b)
        pb.factor_solve_loopback(ctxs, Gs, x)
        xs[world] = x.cpu().numpy()
        assert np.linalg.norm(xs[world] - ref) <= 1e-10 * np.linalg.norm(ref), world
        for c in ctxs:
            c.close()
    for world in (2, 3, 4):   # same cuBLAS calls per tile in the same order: bit for bit
        assert np.array_equal(xs[world], xs[1]), world


def test_loopback_more_ranks_than_tile_rows(pb):
    """N > L0: some ranks own no block column (no tiles, no work) and only relay broadcasts."""
    cfg = synth.CONFIGS[1]          # L0 = 2
    rng = np.random.default_rng(4)
    A = synth.vertex_matrices(cfg, rng)
    ctx0 = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    X, W = synth.spd_blocks(cfg.n, ctx0.nblocks, rng)
    full = ctx0.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES).cpu().numpy()
    L0, N, K = ctx0.L0, ctx0.Ntil, ctx0.K
    ctx0.close()
    b = rng.normal(size=K)
    ref = np.linalg.solve(_dense(full, L0, N), b)
    world = 5
    ctxs = [pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world, shard=pb.SHARD_CYCLIC)
            for r in range(world)]
    assert [c.dims["npairs_local"] for c in ctxs] == [2, 1, 0, 0, 0]
    pairs = _pairs(L0)
    Gs = [_dev(full[[p for p, (h, _) in enumerate(pairs) if h % world == r]]) if ctxs[r].dims["npairs_local"]
          else torch.zeros(1, dtype=torch.float64, device="cuda") for r in range(world)]
    x = _dev(b)
    pb.factor_solve_loopback(ctxs, Gs, x)
    assert np.linalg.norm(x.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    for c in ctxs:
        c.close()


def test_loopback_reports_indefinite_G(pb):
    cfg = synth.CONFIGS[2]
    rng = np.random.default_rng(2)
    A = synth.vertex_matrices(cfg, rng)
    ctxs = [pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=2, shard=pb.SHARD_CYCLIC) for r in range(2)]
    X, W = synth.spd_blocks(cfg.n, ctxs[0].nblocks, rng)
    Gs = [-c.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES) for c in ctxs]
    with pytest.raises(pb.PolyaError, match="not positive definite"):
        pb.factor_solve_loopback(ctxs, Gs, _dev(rng.normal(size=ctxs[0].K)))
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_indefinite_tile_at_a_later_step(pb, world):
    """The diagonal tile (1, 1) -- owned by rank 1 -- made indefinite: rank 0 factors step 0 and its
    look-ahead update runs, rank 1's potrf fails at step 1, and the per-step all-reduce of {error, info}
    brings every rank out of dist_potrf with the same verdict (no rank left waiting in a broadcast)."""
    cfg = synth.CONFIGS[2]
    rng = np.random.default_rng(5)
    A = synth.vertex_matrices(cfg, rng)
    ctxs = [pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world, shard=pb.SHARD_CYCLIC)
            for r in range(world)]
    X, W = synth.spd_blocks(cfg.n, ctxs[0].nblocks, rng)
    Gs = [c.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES) for c in ctxs]
    N = ctxs[0].Ntil
    Gs[1][0] -= 1e9 * torch.eye(N, dtype=torch.float64, device="cuda")   # rank 1's first tile is (1, 1)
    with pytest.raises(pb.PolyaError, match="not positive definite"):
        pb.factor_solve_loopback(ctxs, Gs, _dev(rng.normal(size=ctxs[0].K)))
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("nccl", [False, True])
def test_cyclic_ipm_step_equals_tiled(pb, nccl):
    cfg = synth.CONFIGS[2]
    A = synth.vertex_matrices(cfg, np.random.default_rng(0))
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    ref = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    ref.set_factorization(2)     # the single-GPU tiled factorisation
    cyc = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, shard=pb.SHARD_CYCLIC)
    if nccl:
        cyc.nccl_init(pb.nccl_unique_id())   # one-rank communicator: the NCCL broadcasts run
    from oracle import ipm as oipm
    X, Z, y, mu = oipm.initial_state(P)
    st = [[_dev(v.copy()) for v in (X, Z, y)] for _ in range(2)]
    m = [mu, mu]
    for it in range(4):
        for i, ctx in enumerate((ref, cyc)):
            s = ctx.ipm_step(*st[i], m[i], it)
            m[i] = s["mu"]
        for a, b in zip(st[0], st[1]):
            assert np.array_equal(a.cpu().numpy(), b.cpu().numpy()), it
    r = cyc.ipm_solve()
    assert r["converged"]
    ref.close()
    cyc.close()


def test_loopback_generalised_form(pb):
    """The distributed factorisation on a generalised-form problem (discrete time, N = n): same x as
    a dense solve of the one-rank G."""
    A = synth.discrete_vertex_matrices(5, 3, 0.8, np.random.default_rng(3))
    terms = synth.discrete_time_terms(A)
    ref_ctx = pb.Polya.general(terms, 5, 3, 2, 1, 1)
    rng = np.random.default_rng(4)
    X, W = synth.spd_blocks(5, ref_ctx.nblocks, rng)
    full = ref_ctx.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES).cpu().numpy()
    L0, N, K = ref_ctx.L0, ref_ctx.Ntil, ref_ctx.K
    ref_ctx.close()
    b = rng.normal(size=K)
    ref = np.linalg.solve(_dense(full, L0, N), b)
    world = 3
    ctxs = [pb.Polya.general(terms, 5, 3, 2, 1, 1, rank=r, nranks=world, shard=pb.SHARD_CYCLIC) for r in range(world)]
    Gs = [c.schur(_dev(X), _dev(W), layout=pb.G_PAIR_TILES) for c in ctxs]
    pairs = _pairs(L0)
    for r in range(world):
        assert np.array_equal(Gs[r].cpu().numpy(), full[[p for p, (h, _) in enumerate(pairs) if h % world == r]])
    x = _dev(b)
    pb.factor_solve_loopback(ctxs, Gs, x)
    assert np.linalg.norm(x.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    for c in ctxs:
        c.close()


def test_multi_rank_ipm_needs_cyclic_and_nccl(pb):
    """polya_ipm_step on several ranks: EINVAL without SHARD_CYCLIC, ENCCL (not a hang) with
    SHARD_CYCLIC but no communicator -- the distributed factorisation's first broadcast fails
    cleanly."""
    cfg = synth.CONFIGS[1]
    A = synth.vertex_matrices(cfg, np.random.default_rng(0))
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    from oracle import ipm as oipm
    X, Z, y, mu = oipm.initial_state(P)
    for shard, msg in ((pb.SHARD_TILES, "invalid argument"), (pb.SHARD_CYCLIC, "NCCL")):
        ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=0, nranks=2, shard=shard)
        st = [_dev(v.copy()) for v in (X, Z, y)]
        with pytest.raises(pb.PolyaError, match=msg):
            ctx.ipm_step(*st, mu, 0)
        ctx.close()
