#!/usr/bin/env python
"""Example 2 of the paper: upper bounds on L_opt = -0.111 by bisection on L
with the GPU path (robust.certify = polya_setup + polya_ipm_solve + polya_verdict), for growing
(d_p, d1 = d2) -- the experiment behind the paper's Figs. (conserve1/2), whose plotted values are
not in the text.  Prints one JSON line per degree and a summary; the brute-force stability boundary
of A(g(alpha)) is -0.1115 (tests/test_oracle_examples.py)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1411_3769_b200 as pb  # noqa: E402
from paper_1411_3769_b200 import robust  # noqa: E402
from test_oracle_examples import example2_terms  # noqa: E402  (the paper's printed A1..A6)

da, A = pb.homogenize(example2_terms(), 3)


def A_at(L):
    return pb.simplex_map(A, 3, da, [1 - L] * 3, [L] * 3)


degs = [(1, 1, 1), (1, 2, 2), (2, 2, 2), (2, 4, 4), (3, 4, 4), (3, 6, 6), (4, 6, 6), (4, 8, 8), (5, 10, 10)]
if len(sys.argv) > 1:
    degs = [tuple(int(x) for x in d.split(",")) for d in sys.argv[1:]]
out = []
for deg in degs:
    t0 = time.time()
    info = {}

    def cert(L):
        r = robust.certify(A_at(L), 3, 3, *deg, da=3, samples=1000, maxit=80)
        info.update(K=r["K"], nblocks=r["nblocks"])
        return r["certified"]

    hi, lo, trace = robust.bisect(cert, -0.2, 0.6, steps=14)
    rec = {"dp": deg[0], "d1": deg[1], "d2": deg[2], "L_upper_bound": hi, "bracket": [lo, hi], "K": info.get("K"),
           "nblocks": info.get("nblocks"), "seconds": round(time.time() - t0, 2), "bisection_steps": len(trace)}
    out.append(rec)
    print(json.dumps(rec), flush=True)
print(json.dumps({"summary": [(r["dp"], r["d1"], r["L_upper_bound"]) for r in out], "L_opt_printed": -0.111,
                  "brute_force_boundary": -0.1115}))
