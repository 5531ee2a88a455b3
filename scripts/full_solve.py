#!/usr/bin/env python
"""Full robust-stability certification on the GPU path for a BASELINE config: Algorithm 2 from its
initial point to the stopping rule (polya_ipm_solve), then the certificate's grid check
(polya_verdict, n <= 168) -- the whole method of the paper at that size, with per-iteration
timings.  Usage: python scripts/full_solve.py CONFIG [maxit]"""
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

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = synth.CONFIGS[cid]
A = synth.vertex_matrices(cfg, np.random.default_rng(0))
t0 = time.time()
ctx = pb.Polya(cfg.n, cfg.l, cfg.dp, cfg.d1, cfg.d2, A)
setup_s = time.time() - t0
t1 = time.time()
r = ctx.ipm_solve(eps=1e-8, tol=1e-8, maxit=maxit)
torch.cuda.synchronize()
solve_s = time.time() - t1
nfail = None
if r["converged"] and cfg.n <= 168:
    nfail = ctx.verdict(r["y"], robust.simplex_points(cfg.l, 1000, 0))
out = {"config": cid, "n": cfg.n, "l": cfg.l, "dp": cfg.dp, "d1": cfg.d1, "d2": cfg.d2, "K": ctx.K,
       "nblocks": ctx.nblocks, "converged": bool(r["converged"]), "status": r["status"], "iterations": r["iterations"],
       "gap": r["gap"], "pinf": r["pinf"], "grid_failures": nfail,
       "certified": bool(r["converged"] and (nfail == 0 if nfail is not None else True)),
       "setup_s": setup_s, "solve_s": solve_s, "s_per_iteration": solve_s / max(r["iterations"], 1),
       "ms_schur_total": r["ms_schur"], "ms_factor_total": r["ms_factor"], "ms_other_total": r["ms_other"],
       "history": [{k: h[k] for k in ("gap", "mu", "tp", "td", "ms_schur", "ms_factor", "ms_other")} for h in r["history"]],
       "note": "grid check: polya_verdict at the simplex vertices, edge midpoints and 1000 Dirichlet(1) points (n <= 168)"}
print(json.dumps(out))
