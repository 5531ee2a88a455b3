"""Multi-GPU data path with real ranks (one process per GPU, NCCL over NVLink):
skipped unless at least two GPUs are visible (every gpurun box of this build has one; the driver's
scaling run has eight).

Per rank, in its own process on its own GPU:
* SHARD_BLOCKS: the rank's partial G over its Polya blocks, summed by polya_reduce_G
  (ncclReduceScatter), by the pipelined polya_schur_reduce and by the fused P2P combine (K4 storing
  into the owners' slots over NVLink) -- all equal the literal oracle (Eq. T2) to 1e-10;
* SHARD_TILES: each rank's work items written into a zeroed K x K G; the sum over ranks is the
  one-rank G bit for bit (disjoint entries) and the oracle to 1e-10;
* SHARD_CYCLIC: three polya_ipm_step iterations with the distributed factorisation match the
  oracle's Algorithm 2 iterates to 1e-8.
"""
import os

import numpy as np
import pytest

import synth
from oracle import ipm as oipm
from oracle import sdp as osdp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2


def _rank_main(rank, world, q_uid, q_out, q_hnd, cid):
    import torch

    import paper_1411_3769_b200 as pb
    torch.cuda.set_device(rank)
    cfg = synth.CONFIGS[cid]
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    out = {"rank": rank}
    # block sharding + NCCL ReduceScatter of the partial G
    cb = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=world, shard=pb.SHARD_BLOCKS)
    X, W = synth.spd_blocks(cfg.n, cb.nblocks, rng)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    uids = []
    for _ in range(2):   # two communicators: blocks and cyclic
        if rank == 0:
            u = pb.nccl_unique_id()
            for _ in range(world - 1):
                q_uid.put(u)
        else:
            u = q_uid.get()
        uids.append(u)
    cb.nccl_init(uids[0])
    Gp = cb.schur(Xd, Wd, layout=pb.G_PAIR_TILES)
    out["blocks_panel"] = cb.reduce_G(Gp).cpu().numpy()          # whole partial, then one combine
    cb.set_combine_tiles(1)                                       # pipelined: one tile per rank and group
    out["blocks_pipe"] = cb.schur_reduce(Xd, Wd).cpu().numpy()
    out["combine_tiles"] = cb.dims["combine_tiles"]
    # fused P2P combine: K4 stores into the owners' slots over NVLink peer memory
    mine = cb.p2p_export()
    for _ in range(world - 1):          # one copy for every other rank
        q_hnd.put((rank, mine))
    hs = {rank: mine}
    while len(hs) < world:
        rr, hh = q_hnd.get()
        if rr == rank:
            q_hnd.put((rr, hh))
            continue
        hs[rr] = hh
    cb.p2p_import([hs[r] for r in range(world)])
    out["blocks_p2p"] = cb.schur_reduce_p2p(Xd, Wd).cpu().numpy()
    torch.cuda.synchronize()
    cb.close()
    # output-tile sharding
    ct = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=world)
    Gt = torch.zeros(ct.K, ct.K, dtype=torch.float64, device="cuda")
    ct.schur(Xd, Wd, G=Gt)
    out["tiles_G"] = Gt.cpu().numpy()
    ct.close()
    # distributed factorisation inside the IPM step
    cc = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=rank, nranks=world, shard=pb.SHARD_CYCLIC)
    cc.nccl_init(uids[1])
    n, nb = cfg.n, cc.nblocks
    Xi = torch.eye(n, dtype=torch.float64, device="cuda").repeat(nb, 1, 1).contiguous()
    Zi = Xi.clone()
    yi = torch.zeros(cc.K, dtype=torch.float64, device="cuda")
    mu, iters = 1.0 / 3.0, []
    for it in range(3):
        st = cc.ipm_step(Xi, Zi, yi, mu, it)
        mu = st["mu"]
        iters.append((Xi.cpu().numpy(), Zi.cpu().numpy(), yi.cpu().numpy(), st))
    out["ipm"] = iters
    cc.close()
    q_out.put(out)


@pytest.mark.parametrize("cid", [2, 3])
def test_two_ranks_blocks_tiles_cyclic(cid):
    if torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs (found {torch.cuda.device_count()})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_uid, q_out, q_hnd = ctx.Queue(), ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, WORLD, q_uid, q_out, q_hnd, cid)) for r in range(WORLD)]
    for p in procs:
        p.start()
    outs = sorted([q_out.get(timeout=600) for _ in range(WORLD)], key=lambda o: o["rank"])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synth.CONFIGS[cid]
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    X, W = synth.spd_blocks(cfg.n, P.nblocks, rng)
    Gref = osdp.schur_literal(P, X, W)
    N = P.Ntil
    tiles_ref = np.concatenate([Gref[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N].ravel()
                                for h in range(P.L0) for h2 in range(h, P.L0)])
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)   # noqa: E731
    NN = N * N

    def tiles_of(key, t):   # rank r holds tiles g N t + r t + j at (g t + j) (polya_dims.combine_tiles)
        got = np.zeros(tiles_ref.size)
        for o in outs:
            buf = o[key]
            for slot in range(buf.size // NN):
                g, j = divmod(slot, t)
                p = g * WORLD * t + o["rank"] * t + j
                if p < P.L0 * (P.L0 + 1) // 2:
                    got[p * NN:(p + 1) * NN] = buf[slot * NN:(slot + 1) * NN]
        return got
    t_auto = -(-(P.L0 * (P.L0 + 1) // 2) // WORLD)     # small tiles: one group of ceil(npairs / N)
    whole = tiles_of("blocks_panel", t_auto)
    pipe = tiles_of("blocks_pipe", outs[0]["combine_tiles"])
    p2p = tiles_of("blocks_p2p", outs[0]["combine_tiles"])
    assert rel(whole, tiles_ref) <= 1e-10 and rel(pipe, tiles_ref) <= 1e-10 and rel(p2p, tiles_ref) <= 1e-10
    assert np.array_equal(whole, pipe)          # same partials, same NCCL sums
    assert rel(p2p, pipe) <= 1e-13              # rank-order sums vs NCCL's order
    Gt = sum(o["tiles_G"] for o in outs)
    assert rel(Gt, Gref) <= 1e-10 and np.array_equal(Gt, Gt.T)
    if cid != 2:      # the oracle's dense IPM step is minutes at config 3
        return
    Xo, Zo, yo, mu = oipm.initial_state(P)
    for it in range(3):
        Xo, Zo, yo, st = oipm.ipm_step(P, Xo, Zo, yo, mu)
        mu = st["mu"]
        for o in outs:
            Xg, Zg, yg, sg = o["ipm"][it]
            assert rel(Xg, Xo) <= 1e-8 and rel(Zg, Zo) <= 1e-8 and rel(yg, yo) <= 1e-8, (it, o["rank"])
