"""GPU tests of the block-sharded Schur complement (SHARD_BLOCKS: the paper's decentralised
scheme) and its NCCL combine (polya_reduce_G).

On one GPU the N ranks are N contexts (rank r of N) on the same device; each assembles its
partial G^(r) over its Polya blocks [b0, b1), and sum_r G^(r) must equal the single-rank G
(to 1e-12 relative: multi-GPU vs 1) and the oracle's literal G (1e-10).  The NCCL
collective itself is exercised with a one-rank communicator (ReduceScatter / AllReduce of one
rank is the identity), since only one GPU is available; the N > 1 host logic is covered by
tests/test_multirank_cpu.py over gloo."""
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


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _inputs(cfg, seed=0):
    rng = np.random.default_rng(seed)
    A = synth.vertex_matrices(cfg, rng)
    from math import comb
    nb = comb(cfg.l + cfg.dp + cfg.d1 - 1, cfg.l - 1) + comb(cfg.l + cfg.dp + cfg.d2, cfg.l - 1)
    X, W = synth.spd_blocks(cfg.n, nb, rng)
    return A, X, W


CASES = [(synth.CONFIGS[2], 3), (synth.small_config(12, 3, 2, 1, 2), 2), (synth.small_config(20, 2, 2, 1, 1), 5),
         (synth.CONFIGS[3], 4)]


@pytest.mark.parametrize("cfg,world", CASES, ids=lambda v: getattr(v, "name", str(v)))
def test_block_partials_sum_to_G(pb, cfg, world):
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    ref = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    G_tiles = ref.schur(Xd, Wd, layout=pb.G_PAIR_TILES).cpu().numpy().ravel()
    G_full = ref.schur(Xd, Wd, layout=pb.G_FULL).cpu().numpy()
    ref.close()
    acc_t = np.zeros_like(G_tiles)
    acc_f = np.zeros_like(G_full)
    flops = 0.0
    for r in range(world):
        ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world, shard=pb.SHARD_BLOCKS)
        part = ctx.schur(Xd, Wd, layout=pb.G_PAIR_TILES).cpu().numpy()
        assert part.size == world * ctx.dims["reduce_count"]
        assert not np.any(part[G_tiles.size:])          # padding stays zero
        acc_t += part[:G_tiles.size]
        acc_f += ctx.schur(Xd, Wd, layout=pb.G_FULL).cpu().numpy()
        flops += ctx.dims["useful_flops_schur"]
        ctx.close()
    assert _rel(acc_t, G_tiles) <= 1e-12
    assert _rel(acc_f, G_full) <= 1e-12
    if cfg.n <= 12:
        P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
        assert _rel(acc_f, osdp.schur_literal(P, X, W)) <= 1e-10


def test_nccl_one_rank_combine(pb):
    cfg = synth.CONFIGS[2]
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=0, nranks=1, shard=pb.SHARD_BLOCKS)
    ctx.nccl_init(pb.nccl_unique_id())
    part = ctx.schur(Xd, Wd, layout=pb.G_PAIR_TILES)
    out = ctx.reduce_G(part, layout=pb.G_PAIR_TILES)
    torch.cuda.synchronize()
    assert torch.equal(out, part[:out.numel()])
    Gf = ctx.schur(Xd, Wd, layout=pb.G_FULL)
    before = Gf.clone()
    ctx.reduce_G(Gf, layout=pb.G_FULL)           # in-place AllReduce over one rank
    torch.cuda.synchronize()
    assert torch.equal(Gf, before)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    assert _rel(Gf.cpu().numpy(), osdp.schur_literal(P, X, W)) <= 1e-10
    ctx.close()


def test_reduce_without_nccl_or_tiles_mode_fails_loudly(pb):
    cfg = synth.CONFIGS[1]
    A, X, W = _inputs(cfg)
    G = torch.zeros(16, dtype=torch.float64, device="cuda")
    t = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    with pytest.raises(pb.PolyaError):
        t.reduce_G(G, out=G)                         # SHARD_TILES: no combine step
    b = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, shard=pb.SHARD_BLOCKS)
    with pytest.raises(pb.PolyaError):
        b.reduce_G(G, out=G)                         # no communicator yet
    t.close()
    b.close()


@pytest.mark.parametrize("cfg", [synth.CONFIGS[2], synth.small_config(12, 3, 2, 1, 2)], ids=lambda c: c.name)
@pytest.mark.parametrize("world", [1, 3])
def test_chunked_assembly_is_bitwise_the_full_call(pb, cfg, world):
    """polya_schur_prepare + polya_schur_assemble over pair chunks (the streaming form bench.py's e2e
    uses) writes exactly the entries polya_schur writes, bit for bit, for every rank's share."""
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    for r in range(world):
        ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world)
        npl = ctx.dims["pair1"] - ctx.dims["pair0"]
        for layout in (pb.G_PAIR_TILES, pb.G_FULL):
            ref = ctx.schur(Xd, Wd, layout=layout)
            G = torch.zeros_like(ref)
            ctx.schur_prepare(Xd, Wd)
            cuts = sorted({0, npl // 3, (2 * npl) // 3, npl})
            for a, b in zip(cuts[:-1], cuts[1:]):
                ctx.schur_assemble(G, a, b, layout=layout)
            torch.cuda.synchronize()
            assert torch.equal(G, ref)
        with pytest.raises(pb.PolyaError):
            ctx.schur_assemble(G, 0, npl + 1, layout=pb.G_FULL)
        ctx.close()


@pytest.mark.parametrize("cfg", [synth.CONFIGS[2], synth.small_config(12, 3, 2, 1, 2), synth.CONFIGS[3]],
                         ids=lambda c: c.name)
@pytest.mark.parametrize("tiles", [1, 2, 4, 0])
@pytest.mark.parametrize("with_nccl", [False, True])
def test_pipelined_combine_is_bitwise_schur_plus_reduce(pb, cfg, tiles, with_nccl):
    """polya_schur_reduce (the partial G assembled tile group by tile group into two ping-pong slots,
    each group's reduce-scatter on the comm stream overlapping the next group's assembly) gives
    exactly polya_schur + polya_reduce_G: one rank, with a one-rank NCCL communicator or the
    communicator-less identity; t = 1, 2, 4 tiles per group (several groups, a zero-padded last
    group) and the automatic t."""
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, shard=pb.SHARD_BLOCKS)
    if with_nccl:
        ctx.nccl_init(pb.nccl_unique_id())
    ctx.set_combine_tiles(tiles)
    t = ctx.dims["combine_tiles"]
    assert t == (tiles if tiles else t) and t >= 1
    ref = ctx.schur(Xd, Wd, layout=pb.G_PAIR_TILES)          # whole partial (+ zero tiles)
    assert ref.numel() == ctx.dims["reduce_count"]            # one rank: receives everything
    ctx.set_timing(True)
    for _ in range(2):                                        # the second call reuses the slots
        out = torch.full((ctx.dims["reduce_count"],), float("nan"), dtype=torch.float64, device="cuda")
        ctx.schur_reduce(Xd, Wd, out=out)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    assert ctx.combine_timing() >= 0.0
    N = ctx.Ntil
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    if P.K <= 1000:
        Gl = osdp.schur_literal(P, X, W)
        tiles_ref = np.concatenate([Gl[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N].ravel()
                                    for h in range(P.L0) for h2 in range(h, P.L0)])
        assert _rel(out.cpu().numpy()[:tiles_ref.size], tiles_ref) <= 1e-10
    ctx.close()


def test_pipelined_combine_needs_communicator_for_several_ranks(pb):
    cfg = synth.CONFIGS[2]
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    c = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=0, nranks=2, shard=pb.SHARD_BLOCKS)
    with pytest.raises(pb.PolyaError):
        c.schur_reduce(Xd, Wd)
    c.close()
    t = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    with pytest.raises(pb.PolyaError):
        t.schur_reduce(Xd, Wd)                      # SHARD_TILES: nothing to combine
    t.close()


@pytest.mark.parametrize("cfg,world,tiles", [(synth.CONFIGS[2], 2, 0), (synth.CONFIGS[2], 3, 1),
                                             (synth.small_config(12, 3, 2, 1, 2), 5, 1), (synth.CONFIGS[3], 4, 2)],
                         ids=lambda v: getattr(v, "name", str(v)))
def test_fused_p2p_combine_loopback(pb, cfg, world, tiles):
    """The fused P2P combine (polya_schur_reduce_p2p): K4 of every rank stores its partial tiles straight
    into the owners' receive slots, each owner sums its slots in rank order.  On one GPU the ranks are
    contexts wired by polya_p2p_loopback, phase 1 (assembly + signal) for all of them before phase 2
    (wait + sum).  Every rank's result is bit for bit the rank-order sum of the ranks' partial G tiles
    (polya_schur per rank), in the tile-group layout of polya_reduce_G; a second call (next epoch) too."""
    A, X, W = _inputs(cfg)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    ctxs = [pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=world, shard=pb.SHARD_BLOCKS)
            for r in range(world)]
    for c in ctxs:
        c.set_combine_tiles(tiles)
    parts = [c.schur(Xd, Wd, layout=pb.G_PAIR_TILES).cpu().numpy() for c in ctxs]
    total = parts[0].copy()
    for q in parts[1:]:
        total += q                      # rank order, as the owners sum their slots
    pb.p2p_loopback(ctxs)
    N = ctxs[0].Ntil
    NN = N * N
    t = ctxs[0].dims["combine_tiles"]
    npairs = ctxs[0].dims["npairs"]
    for _ in range(2):
        for c in ctxs:
            c.schur_reduce_p2p(Xd, Wd, phases=1)
        outs = [c.schur_reduce_p2p(Xd, Wd, phases=2).cpu().numpy() for c in ctxs]
        for r, out in enumerate(outs):
            assert out.size == ctxs[r].dims["reduce_count"]
            for slot in range(out.size // NN):
                g, j = divmod(slot, t)
                p = g * world * t + r * t + j
                if p < npairs:
                    assert np.array_equal(out[slot * NN:(slot + 1) * NN], total[p * NN:(p + 1) * NN]), (r, slot)
    for c in ctxs:
        c.close()
