#!/usr/bin/env python
"""Projected multi-GPU strong scaling from ONE GPU (no multi-GPU hardware in round 1): for N in
{1, 2, 4, 8}, every rank's share of polya_schur (output-tile sharding, and the paper's block
sharding) is run and timed on the same B200, one rank after another; the projected N-GPU time
is the max over ranks (the shards share no data-path traffic in tile mode; in block mode the
NCCL ReduceScatter of (N-1)/N of G_half per GPU is added at an assumed 700 GB/s bus bandwidth,
SURVEY 8(e): serially as in round 1's single combine call (`projected_ms`), and as the pipelined
combine of polya_schur_reduce overlaps it -- max(assembly, reduce-scatter) + one group's
reduce-scatter (`projected_ms_pipelined`)).  A projection for load balance and per-share
efficiency, not a bench value.  Usage: python scripts/shard_projection.py [config] [tiles|blocks|both]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402
from bench import counts  # noqa: E402


def time_share(ctx, Xd, Wd, G, reps=3):
    ctx.set_timing(True)
    ts = []
    for _ in range(reps + 1):
        ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
        pre, asm = ctx.timing()
        ts.append(pre + asm)
    return float(np.median(ts[1:]))


def main(cid="4", which="both"):
    cfg = synth.CONFIGS[int(cid)]
    L0, L, M = counts(cfg)
    A, X, W = synth.make_case(cfg, L + M, seed=0)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    out = {"config": cid, "note": __doc__.split("\n")[0], "tiles": {}, "blocks": {}}
    t1 = None
    for N in (1, 2, 4, 8):
        for mode, key in ((pb.SHARD_TILES, "tiles"), (pb.SHARD_BLOCKS, "blocks")):
            if which != "both" and key != which and not (key == "tiles" and N == 1):
                continue
            times, flops = [], []
            for r in range(N):
                ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A, rank=r, nranks=N, shard=mode)
                if mode == pb.SHARD_TILES:
                    npl = max(ctx.dims["pair1"] - ctx.dims["pair0"], 1)
                    G = torch.empty((npl, ctx.Ntil, ctx.Ntil), dtype=torch.float64, device="cuda")
                else:
                    G = torch.zeros(N * ctx.dims["reduce_count"], dtype=torch.float64, device="cuda")
                times.append(time_share(ctx, Xd, Wd, G))
                flops.append(ctx.dims["useful_flops_schur"])
                ghalf = ctx.dims["npairs"] * ctx.Ntil * ctx.Ntil * 8
                groups = -(-ctx.dims["npairs"] // (N * max(ctx.dims["combine_tiles"], 1))) if mode == pb.SHARD_BLOCKS else 1
                ctx.close()
                del G
                torch.cuda.empty_cache()
            tmax = max(times)
            comm = 0.0 if mode == pb.SHARD_TILES or N == 1 else (N - 1) / N * ghalf / 700e9 * 1e3
            if mode == pb.SHARD_TILES and N == 1:
                t1 = tmax
            pipe = max(tmax, comm) + comm / groups
            rec = {"rank_ms": times, "max_ms": tmax, "mean_ms": float(np.mean(times)), "comm_ms_est": comm,
                   "projected_ms": tmax + comm, "tflops_projected": sum(flops) / ((tmax + comm) * 1e-3) / 1e12,
                   "efficiency_vs_1gpu_tiles": t1 / (N * (tmax + comm)),
                   "projected_ms_pipelined": pipe, "efficiency_pipelined": t1 / (N * pipe)}
            out[key][str(N)] = rec
            print(key, N, json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in rec.items()
                                      if k != "rank_ms"}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "4", sys.argv[2] if len(sys.argv) > 2 else "both")
