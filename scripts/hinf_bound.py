#!/usr/bin/env python
"""Robust H-infinity bound of a polytopic system on the GPU path: the bounded-real lemma in the
generalised form (polya_setup_general with N = n + m, reading R19), bisection on gamma
(robust.bisect), against the brute-force worst case over the simplex (frequency sweep at the
vertices, edge midpoints and random points -- a lower bound on the true robust norm).
Usage: python scripts/hinf_bound.py CONFIG [dp] [d1] [steps]   (JSON on stdout)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1411_3769_b200 as pb  # noqa: E402
import synth  # noqa: E402
from paper_1411_3769_b200 import robust  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d1 = int(sys.argv[3]) if len(sys.argv) > 3 else 1
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
cfg = synth.CONFIGS[cid]
rng = np.random.default_rng(0)
A = synth.vertex_matrices(cfg, rng)
n, l = cfg.n, cfg.l
Bu = np.zeros((n, 1))
Bu[0, 0] = 1.0          # input at the first state, output at the last
Cy = np.zeros((1, n))
Cy[0, -1] = 1.0
w = np.concatenate([[0.0], np.logspace(-3, 4, 600)])


def hinf(M):
    return max(np.linalg.svd(Cy @ np.linalg.solve(1j * x * np.eye(n) - M, Bu), compute_uv=False)[0] for x in w)


pts = robust.simplex_points(l, 40, 1)
lower = max(hinf(np.tensordot(p, A, 1)) for p in pts)


def cert(gamma):
    terms, R0 = synth.bounded_real_terms(A, Bu, Cy, gamma)
    _, R = pb.homogenize({tuple([dp + 1] + [0] * (l - 1)): 0.0 * R0, tuple([0] * l): R0}, l)
    return robust.certify(None, n, l, dp, d1, d1, terms=terms, R=R, samples=300)["certified"]


t0 = time.time()
hi = 2.0 * lower
while not cert(hi):
    hi *= 2.0
upper, lo, trace = robust.bisect(cert, lower, hi, steps=steps)
out = {"config": cid, "n": n, "l": l, "dp": dp, "d1": d1, "d2": d1, "N": n + 1,
       "worst_case_lower_bound": lower, "certified_upper_bound": upper, "ratio": upper / lower,
       "bisection_steps": steps, "seconds": time.time() - t0, "trace": trace}
print(json.dumps(out))
