#!/usr/bin/env python
"""The generalised LMI form on the GPU path at a moderate size: discrete-time robust stability
A(alpha)^T P A(alpha) - P < 0 (synth.discrete_time_terms) through polya_setup_general -- Schur
assembly throughput (same K4 kernel, 4 Q_h Q_h' terms per block) and the whole certification.
Usage: python scripts/general_measure.py [n] [l] [dp] [d1] [d2]  (JSON on stdout)."""
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
from paper_1411_3769_b200 import robust  # noqa: E402

n, l, dp, d1, d2 = (int(v) for v in (sys.argv[1:6] + ["20", "3", "2", "2", "2"][len(sys.argv[1:6]):]))
A = synth.discrete_vertex_matrices(n, l, 0.9, np.random.default_rng(0))
terms = synth.discrete_time_terms(A)
t0 = time.time()
ctx = pb.Polya.general(terms, n, l, dp, d1, d2)
setup_s = time.time() - t0
X, W = synth.spd_blocks(n, ctx.nblocks, np.random.default_rng(1))
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
G = torch.zeros((ctx.dims["pair1"] - ctx.dims["pair0"], ctx.Ntil, ctx.Ntil), dtype=torch.float64, device="cuda")
ctx.set_timing(True)
for _ in range(3):
    ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
pre, asm = [], []
for _ in range(10):
    ctx.schur(Xd, Wd, G=G, layout=pb.G_PAIR_TILES)
    a, b = ctx.timing()
    pre.append(a)
    asm.append(b)
flops = ctx.dims["useful_flops_schur"]
ms_asm = float(np.median(asm))
del G
t1 = time.time()
r = robust.certify(None, n, l, dp, d1, d2, terms=terms, samples=1000)
cert_s = time.time() - t1
out = {"form": "discrete time A^T P A - P < 0 (generalised LMI, polya_setup_general)", "n": n, "l": l, "dp": dp,
       "d1": d1, "d2": d2, "K": ctx.K, "nblocks": ctx.nblocks, "terms_per_block_total": ctx.dims["nnz_H"],
       "setup_s": setup_s, "schur_precompute_ms": float(np.median(pre)), "schur_assembly_ms": ms_asm,
       "useful_flops_schur": flops, "assembly_tflops": flops / ms_asm * 1e-9,
       "certified": r["certified"], "iterations": r["iterations"], "gap": r["gap"], "certify_s": cert_s}
print(json.dumps(out))
ctx.close()
