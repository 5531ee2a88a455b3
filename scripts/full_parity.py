#!/usr/bin/env python
"""Every entry of G at a BASELINE config, GPU (polya_schur, PAIR_TILES) against the oracle's
structured assembly (oracle.sdp.schur_structured_tile, pinned to the literal Eq. T2 on configs 1-3
and ragged shapes in tests/test_oracle_sdp.py), pair tile by pair tile.  Reports per pair the
relative Frobenius error and the worst |dG_ij| / sqrt(G_ii G_jj).  Test infrastructure: the oracle
runs on the host's cores (minutes at config 4).
Usage: python scripts/full_parity.py [CONFIG]   (JSON on stdout)"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402
from oracle import sdp as osdp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[cid]
A = synth.vertex_matrices(cfg, np.random.default_rng(0))
ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
X, W = synth.spd_blocks(cfg.n, ctx.nblocks, np.random.default_rng(1))
Gt = ctx.schur(torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), layout=pb.G_PAIR_TILES)
torch.cuda.synchronize()
P = osdp.build_problem(A, cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2)
N, L0 = P.Ntil, P.L0
pairs = [(h, h2) for h in range(L0) for h2 in range(h, L0)]
# diagonal of G for the scale-free entry bound
diag = np.concatenate([np.diag(Gt[p].cpu().numpy()) for p, (h, h2) in enumerate(pairs) if h == h2])
t0 = time.time()
worst_rel, worst_ent, per = 0.0, 0.0, []
for p, (h, h2) in enumerate(pairs):
    got = Gt[p].cpu().numpy()
    ref = osdp.schur_structured_tile(P, X, W, h, h2)
    rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))
    scale = np.sqrt(np.outer(np.abs(diag[h * N:(h + 1) * N]), np.abs(diag[h2 * N:(h2 + 1) * N])))
    ent = float(np.max(np.abs(got - ref) / np.maximum(scale, 1e-300)))
    worst_rel, worst_ent = max(worst_rel, rel), max(worst_ent, ent)
    per.append({"h": h, "h2": h2, "rel_fro": rel, "max_entry_rel": ent})
out = {"config": cid, "K": P.K, "entries_checked": int(len(pairs) * N * N), "pairs": len(pairs),
       "worst_rel_fro": worst_rel, "worst_entry_rel": worst_ent, "bar": 1e-10,
       "pass": bool(worst_rel <= 1e-10 and worst_ent <= 1e-10), "oracle_s": time.time() - t0, "per_pair": per}
print(json.dumps(out))
