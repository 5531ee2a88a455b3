"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):
configs 1 and 2 and a ragged n = 12 case through setup, apply, adjoint, schur (FULL and pair
tiles, 2-rank shares), one IPM step (dense and tiled factorisation) and the verdict kernel."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402
from paper_1411_3769_b200 import robust  # noqa: E402

for cfg in (synth.CONFIGS[1], synth.CONFIGS[2], synth.small_config(12, 3, 2, 1, 2)):
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(cfg, rng)
    ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
    X, W = synth.spd_blocks(cfg.n, ctx.nblocks, rng)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    y = torch.from_numpy(rng.normal(size=ctx.K)).cuda()
    ctx.apply(y)
    ctx.adjoint(Xd)
    ctx.schur(Xd, Wd, layout=pb.G_FULL)
    ctx.schur(Xd, Wd, layout=pb.G_PAIR_TILES)
    for r in range(2):
        c2 = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=2)
        c2.schur(Xd, Wd, layout=pb.G_PAIR_TILES)
        c2.close()
    for mode in (1, 2):
        ctx.set_factorization(mode)
        Xi = torch.eye(cfg.n, dtype=torch.float64, device="cuda").repeat(ctx.nblocks, 1, 1).contiguous()
        Zi = Xi.clone()
        yi = torch.zeros(ctx.K, dtype=torch.float64, device="cuda")
        ctx.ipm_step(Xi, Zi, yi, 1.0 / 3.0, 0)
    ctx.verdict(y, robust.simplex_points(cfg.l, 20, 0))
    ctx.sync()
    ctx.close()
torch.cuda.synchronize()
print("sanitize case done")
