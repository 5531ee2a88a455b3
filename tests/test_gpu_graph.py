"""The public calls are capturable as one CUDA graph (stream-ordered, no host synchronisation inside):
apply + adjoint + schur (precompute + assembly, the work counter's reset included) captured once and
replayed give exactly the direct calls' results, and a replay after the inputs change in place
computes the new G (the graph holds the buffers, not their values).  Small configurations are
launch-bound (config 1: ~12 launches per step), which replaying a graph removes (bench.py --graph)."""
import numpy as np
import pytest

import synth
from oracle import sdp as osdp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid", [1, 2])
def test_step_as_cuda_graph(cid):
    import paper_1411_3769_b200 as pb
    cfg = synth.CONFIGS[cid]
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    X, W = synth.spd_blocks(cfg.n, ctx.nblocks, rng)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    y = torch.from_numpy(rng.normal(size=ctx.K)).cuda()
    Bt = torch.empty((ctx.nblocks, ctx.bn, ctx.bn), dtype=torch.float64, device="cuda")
    yv = torch.empty(ctx.K, dtype=torch.float64, device="cuda")
    G = torch.zeros((ctx.dims["npairs_local"], ctx.Ntil, ctx.Ntil), dtype=torch.float64, device="cuda")

    def step():
        ctx.apply(y, out=Bt)
        ctx.adjoint(Xd, out=yv)
        ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)

    step()                                   # warm-up outside the capture (attributes, workspaces)
    torch.cuda.synchronize()
    ref = (Bt.clone(), yv.clone(), G.clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for t in (Bt, yv, G):
        t.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Bt, ref[0]) and torch.equal(yv, ref[1]) and torch.equal(G, ref[2])
    # new inputs in place: the replay computes the new G, equal to the oracle's
    X2, W2 = synth.spd_blocks(cfg.n, ctx.nblocks, np.random.default_rng(5))
    Xd.copy_(torch.from_numpy(X2))
    Wd.copy_(torch.from_numpy(W2))
    g.replay()
    torch.cuda.synchronize()
    P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
    Gl = osdp.schur_literal(P, X2, W2)
    N = ctx.Ntil
    tiles = np.array([Gl[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N] for h in range(P.L0) for h2 in range(h, P.L0)])
    got = G.cpu().numpy()
    assert np.linalg.norm(got - tiles) <= 1e-10 * np.linalg.norm(tiles)
    ctx.close()
