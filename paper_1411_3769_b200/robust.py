"""Robust-stability driver: Algorithm 2 to convergence, the certificate's grid check, and bisection
on a margin parameter -- the outer loop of the paper's Examples 1-2.

Outer driver only: every step of the method runs in libpolya.so -- set-up
(polya_setup, with polya_homogenize / polya_simplex_map for non-homogeneous systems on parameter
boxes), the iteration (polya_ipm_solve: apply / adjoint / Schur kernels + the K x K factorisation)
and the verdict (polya_verdict: grid check on the device).  The seeded sample points of the grid
check are drawn here and passed in (they are inputs, not part of the method's arithmetic).
"""
from __future__ import annotations

import numpy as np

from . import Polya

__all__ = ["simplex_points", "certify", "bisect"]


def simplex_points(l, samples=1000, seed=0):
    """Vertices, edge midpoints and `samples` Dirichlet(1) points of Delta_l."""
    eye = np.eye(l)
    pts = [eye[i] for i in range(l)]
    pts += [0.5 * (eye[i] + eye[j]) for i in range(l) for j in range(i + 1, l)]
    pts += list(np.random.default_rng(seed).dirichlet(np.ones(l), size=samples))
    return np.array(pts)


def certify(A, n, l, dp, d1, d2, da=1, delta=1e-3, eps=1e-8, tol=1e-8, maxit=60, samples=1000, seed=0, terms=None, R=None):
    """Is x' = A(alpha) x certified robustly stable on Delta_l by the Polya LMIs of degree
    (dp, d1, d2)?  A: coefficients double[f(l,da)][n][n] of the homogeneous A(alpha) in W_da order.
    Certified = Algorithm 2 met its stopping rule with Z positive definite (polya_ipm_solve) and the
    reconstructed P(alpha) passes the grid check at every sample point (polya_verdict).
    With ``terms`` (A ignored) the LMI is the generalised form sum_i (At_i P Bt_i + transpose) < 0
    (polya_setup_general), e.g. discrete-time stability A^T P A - P < 0."""
    ctx = Polya(n, l, dp, d1, d2, A, da=da, delta=delta, terms=terms, R=R)
    try:
        r = ctx.ipm_solve(eps=eps, tol=tol, maxit=maxit)
        nfail = -1
        if r["converged"]:
            nfail = ctx.verdict(r["y"], simplex_points(l, samples, seed))
        return {"certified": bool(r["converged"] and nfail == 0), "converged": bool(r["converged"]),
                "status": r["status"], "iterations": r["iterations"], "gap": r["gap"], "pinf": r["pinf"],
                "nfail": nfail, "K": ctx.K, "nblocks": ctx.nblocks,
                "ms": r["ms_schur"] + r["ms_factor"] + r["ms_other"]}
    finally:
        ctx.close()


def bisect(certify_at, lo, hi, steps=12):
    """Smallest certified value of a scalar margin by bisection: certify_at(v)
    -> bool, with certify_at(hi) True and certify_at(lo) False assumed monotone in between.
    Returns (upper bound hi, lower bracket lo, trace)."""
    trace = []
    for _ in range(steps):
        mid = 0.5 * (lo + hi)
        ok = bool(certify_at(mid))
        trace.append((mid, ok))
        if ok:
            hi = mid
        else:
            lo = mid
    return hi, lo, trace
