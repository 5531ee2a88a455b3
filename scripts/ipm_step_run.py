#!/usr/bin/env python
"""Two polya_ipm_step iterations on config ${1:-4} from X = Z = I (the IPM leg of bench.py), for a launch
list of the step's kernels under ncu:  ncu --metrics gpu__time_duration.sum --csv python scripts/ipm_step_run.py 4"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1411_3769_b200 as pb  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[cid]
A = synth.vertex_matrices(cfg, np.random.default_rng(0))
ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
if os.environ.get("FACT"):   # polya_set_factorization mode (1 dense look-ahead, 3 dense one-call cuSOLVER, 2 tiled)
    ctx.set_factorization(int(os.environ["FACT"]))
X = torch.eye(cfg.n, dtype=torch.float64, device="cuda").repeat(ctx.nblocks, 1, 1).contiguous()
Z = X.clone()
y = torch.zeros(ctx.K, dtype=torch.float64, device="cuda")
mu = 1.0 / 3.0
for it in range(int(os.environ.get("ITERS", "2"))):
    st = ctx.ipm_step(X, Z, y, mu, it)
    mu = st["mu"]
    print({k: st[k] for k in ("ms_schur", "ms_factor", "ms_other", "tp", "td", "gap")}, flush=True)
