"""Experiment (SCHUR_EXP bit 64 build): where do consumer warps wait for operand stages?  Histogram
of warp 0's wait cycles on the `full` barrier by stage index within an orientation (0, 1, 2, 3,
4..last-1, last), written by the kernel past the end of the pair tiles.  Timing only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402
from bench import counts  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
L0, L, M = counts(cfg)
A, X, W = synth.make_case(cfg, L + M, seed=0)
ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
npl = ctx.dims["pair1"] - ctx.dims["pair0"]
G = torch.zeros(npl * ctx.Ntil * ctx.Ntil + 16, dtype=torch.float64, device="cuda")
ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)   # warm-up
G[-16:] = 0
ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
torch.cuda.synchronize()
h = G[-16:].cpu().numpy()
cyc, cnt = h[:6], h[8:14]
names = ["stage 0", "stage 1", "stage 2", "stage 3", "stages 4..", "last stage"]
tot = cyc.sum()
for nm, c_, n_ in zip(names, cyc, cnt):
    print(f"{nm:12s} waits {int(n_):10d}  mean {c_ / max(n_, 1):9.1f} cyc  share {100 * c_ / tot:5.1f} %")
print("total wait cycles (warp 0 of every CTA):", tot)
