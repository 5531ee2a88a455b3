"""One iteration of the primal-dual predictor-corrector method, Algorithm 2.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md Sec. IV.A (Eqs. 33-46) and Algorithm 2 step by
step, on block stacks (every iterate lies in S_{L,M,n}, Theorem 3):

  Rd  = -B^T(y) + Z + C                                    (Eq. G; reading R13)
  O1  = B(Z^-1 Rd X) - a,  a = 1                           (Processors/Root step 1)
  G   = [tr(B_k Z^-1 B_l X)]                               (Eq. T2)
  dy^ = G^-1 O1                                            (Eq. SAE1)
  dZ^ = B^T(y) - Z - C + B^T(dy^) = -Rd + B^T(dy^)         (Eq. delZ_hat)
  dX^ = -X + Z^-1 (Rd - B^T(dy^)) X, symmetrised           (reading R3)
  O2  = mu B(Z^-1) - B(Z^-1 dZ^ dX^)                       (Processors/Root step 2)
  dy- = G^-1 O2                                            (Eq. SAE2)
  dZ- = B^T(dy-)                                           (Eq. delz_bar)
  dX- = mu Z^-1 - Z^-1 dZ^ dX^ - Z^-1 dZ- X, symmetrised   (Eq. delx_bar)
  t_p, t_d: reading R5 (fraction 0.98 of the distance to the PSD boundary, capped at 1)
  X += t_p dX,  Z += t_d dZ,  y += t_d dy                  (Eqs. 33-35; reading R6)
  mu = (1/3) sum tr(Z X) / N, N = (L+M) n the order of X (reading R4: the literal (1/3) tr(ZX)
       of P:591/729/871 makes the target grow ~10x per step and the method diverge on config 1;
       read as the centring factor 1/3 times the average complementarity),
  phi = tr(C X),  psi = a^T y,  gap = |phi - psi|

Library primitives used as steps: matrix products, inverse, a dense linear solve and a
symmetric eigenvalue routine.  Parity with the CUDA path is "iterates to ~1e-8 over a
few steps" (reading R15: the IPM's certificate is not unique).
"""
from __future__ import annotations

import math

import numpy as np

from . import sdp
from .monomials import enumerate_W

__all__ = ["initial_state", "barrier", "step_length", "ipm_step", "C_blocks", "grid_check", "solve", "verdict", "DIVERGENCE_BOUND"]


def C_blocks(P):
    """C = diag(c_1 I, ..., c_L I, 0, ..., 0) (Eq. C, Eq. Cj); the generalised form's constant term
    R puts (sum alpha)^{d2} R(alpha)'s coefficients on the Lyapunov blocks (reading R18)."""
    C = np.zeros((P.nblocks, P.bn, P.bn))
    for j in range(P.L):
        C[j] = -np.eye(P.bn)          # the padding of a P-block (non-square form, R19): slack Z = I there
        C[j][:P.n, :P.n] = P.c[j] * np.eye(P.n)
    if P.CL is not None:
        C[P.L:] = P.CL
    return C


def initial_state(P):
    """Algorithm 2 initialisation: X = Z = I, y = 0, mu = barrier(Z, X)."""
    X = np.broadcast_to(np.eye(P.bn), (P.nblocks, P.bn, P.bn)).copy()
    Z = X.copy()
    y = np.zeros(P.K)
    return X, Z, y, barrier(P, Z, X)


def barrier(P, Z, X):
    """Reading R4: mu = (1/3) sum_b tr(Z_b X_b) / ((L+M) n)."""
    return sum(np.trace(Z[b] @ X[b]) for b in range(P.nblocks)) / (3.0 * P.nblocks * P.bn)


def _sym(M):
    return 0.5 * (M + np.swapaxes(M, -1, -2))


def step_length(S, dS, frac=0.98):
    """Reading R5: t = min(1, frac * t_max), t_max = sup{t : S_b + t dS_b >= 0 for all b}
    = 1 / max(0, -min_b lambda_min(L_b^-1 dS_b L_b^-T)), S_b = L_b L_b^T."""
    lam = np.inf
    for b in range(S.shape[0]):
        Lc = np.linalg.cholesky(S[b])
        Li = np.linalg.inv(Lc)
        ev = np.linalg.eigvalsh(_sym(Li @ dS[b] @ Li.T))
        lam = min(lam, ev.min())
    if lam >= 0:
        return 1.0
    return min(1.0, frac * (1.0 / -lam))


def ipm_step(P, X, Z, y, mu):
    """One iteration; returns (X, Z, y, stats)."""
    C = C_blocks(P)
    W = np.linalg.inv(Z)
    W = _sym(W)
    BTy = sdp.apply_vmap(P, y)
    Rd = -BTy + Z + C
    O1 = sdp.adjoint_trace(P, W @ Rd @ X) - 1.0
    G = sdp.schur_literal(P, X, W)
    dy1 = np.linalg.solve(G, O1)
    BTd1 = sdp.apply_vmap(P, dy1)
    dZ1 = -Rd + BTd1
    dX1 = _sym(-X + W @ (Rd - BTd1) @ X)
    delta = sdp.adjoint_trace(P, W)
    tau = sdp.adjoint_trace(P, W @ dZ1 @ dX1)
    O2 = mu * delta - tau
    dy2 = np.linalg.solve(G, O2)
    dZ2 = sdp.apply_vmap(P, dy2)
    dX2 = _sym(mu * W - W @ dZ1 @ dX1 - W @ dZ2 @ X)
    dX, dZ, dy = dX1 + dX2, dZ1 + dZ2, dy1 + dy2
    tp = step_length(X, dX)
    td = step_length(Z, dZ)
    X = X + tp * dX
    Z = Z + td * dZ
    y = y + td * dy
    mu_new = barrier(P, Z, X)
    phi = float(sum(np.trace(C[b] @ X[b]) for b in range(P.nblocks)))
    psi = float(y.sum())
    stats = dict(gap=abs(phi - psi), mu=mu_new, tp=tp, td=td, phi=phi, psi=psi,
                 dy1=dy1, dy2=dy2, dX1=dX1, dZ1=dZ1, dX2=dX2, dZ2=dZ2, G=G, O1=O1, O2=O2, Rd=Rd, W=W)
    return X, Z, y, stats


def grid_check(P, y, samples=1000, seed=0):
    """O8 verdict check: P(alpha) = sum_h V_h(y) alpha^h (R7) at vertices, edge midpoints and
    Dirichlet(1) samples: lambda_min P > 0 and lambda_max(A^T P + P A) < 0 (Theorem 1)."""
    Wp = enumerate_W(P.l, P.dp)
    Ph = [sdp.vmap(P, y, h) for h in range(P.L0)]
    rng = np.random.default_rng(seed)
    pts = [np.eye(P.l)[i] for i in range(P.l)]
    pts += [0.5 * (np.eye(P.l)[i] + np.eye(P.l)[j]) for i in range(P.l) for j in range(i + 1, P.l)]
    pts += list(rng.dirichlet(np.ones(P.l), size=samples))
    from . import polya as _polya
    for al in pts:
        Pa = sum(math.prod(a ** e for a, e in zip(al, h)) * Ph[i] for i, h in enumerate(Wp))
        if P.gen is not None:   # generalised form: sum_i At_i(alpha) P Bt_i(alpha) + transpose < 0
            Lm = sum(_polya.evaluate(At, P.l, a, al) @ Pa @ _polya.evaluate(Bt, P.l, b, al) for At, a, Bt, b in P.pairs)
            Lm = Lm + Lm.T
            if P.R is not None:
                Lm = Lm + _polya.evaluate(P.R, P.l, P.dp + P.da, al)
        else:
            Aa = _polya.evaluate(P.A, P.l, P.da, al)
            Lm = Aa.T @ Pa + Pa @ Aa
        if np.linalg.eigvalsh(Pa).min() <= 0 or np.linalg.eigvalsh(Lm).max() >= 0:
            return False
    return True


DIVERGENCE_BOUND = 1e12   # reading R20; the same bound as POLYA_DIVERGENCE_BOUND


def solve(P, eps=1e-8, tol=1e-8, maxit=60, info=None):
    """Algorithm 2 iterated from its initial point until the duality gap is below eps
    (stopping rule) and the primal residual ||B(X) - a|| below tol.  Returns
    (converged, X, Z, y, iterations); converged requires every Z block PD (reading R10).
    Divergence exit (reading R20): when tr(CX), a^T y or mu leaves DIVERGENCE_BOUND in magnitude (an
    unbounded primal iterate: the LMI is infeasible) the iteration stops, before any product can
    overflow.  info (optional dict) receives "status": converged / notpd / diverged / maxit."""
    info = {} if info is None else info
    X, Z, y, mu = initial_state(P)
    for it in range(1, maxit + 1):
        try:
            X, Z, y, st = ipm_step(P, X, Z, y, mu)
        except np.linalg.LinAlgError:
            info["status"] = "notpd"
            return False, X, Z, y, it
        mu = st["mu"]
        vals = (st["phi"], st["psi"], mu)
        if not all(np.isfinite(v) for v in vals) or max(abs(v) for v in vals) > DIVERGENCE_BOUND \
                or not np.all(np.isfinite(y)):
            info["status"] = "diverged"
            return False, X, Z, y, it
        pinf = np.linalg.norm(sdp.adjoint_trace(P, X) - 1.0)
        if st["gap"] <= eps and pinf <= tol:
            ok = all(np.linalg.eigvalsh(z).min() > 0 for z in Z)
            info["status"] = "converged" if ok else "notpd"
            return ok, X, Z, y, it
    info["status"] = "maxit"
    return False, X, Z, y, maxit


def verdict(P, eps=1e-8, tol=1e-8, maxit=60, samples=1000, seed=0):
    """Robust-stability certificate (Theorem 1 via Polya): converged SDP and the
    reconstructed P(alpha) (reading R7) passing the grid check (O8)."""
    ok, _, _, y, _ = solve(P, eps, tol, maxit)
    return bool(ok and grid_check(P, y, samples, seed))
