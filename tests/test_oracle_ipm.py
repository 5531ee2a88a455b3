"""Pins for oracle.ipm (Algorithm 2; readings R3-R6).

An iteration has no unique "right answer" beyond the Newton equations it solves, so the
pins are (a) the Newton identities the directions must satisfy -- B(dX^) = a - B(X)
(primal feasibility of the predictor, which ties the Schur complement G to the operators:
it only holds if G dy = B(W B^T(dy) X) for the G that was factorised) and B(dX-) = 0;
(b) Theorem 3's structure invariance on a dense block-diagonal shadow; (c) the verdicts of
Theorem 1 on constructed systems: config 1 (stable by construction) is
certified, its unstable copy and SPEC's unstable scalar system are not.
"""
import numpy as np
import pytest

import synth
from oracle import ipm, sdp


def _problem(key):
    c = synth.CONFIGS[key]
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    return sdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)


@pytest.mark.parametrize("key", [1, "1u"])
def test_newton_identities(key):
    P = _problem(key)
    X, Z, y, mu = ipm.initial_state(P)
    for _ in range(3):
        BX = sdp.adjoint_trace(P, X)
        Xn, Zn, yn, st = ipm.ipm_step(P, X, Z, y, mu)
        r1 = sdp.adjoint_trace(P, st["dX1"]) - (1.0 - BX)
        assert np.linalg.norm(r1) <= 1e-9 * max(1.0, np.linalg.norm(BX))
        r2 = sdp.adjoint_trace(P, st["dX2"])
        assert np.linalg.norm(r2) <= 1e-9 * max(1.0, np.linalg.norm(BX))
        G = st["G"]
        assert np.abs(G - G.T).max() <= 1e-12 * np.abs(G).max()
        X, Z, y, mu = Xn, Zn, yn, st["mu"]


def _dense(blocks):
    nb, n, _ = blocks.shape
    D = np.zeros((nb * n, nb * n))
    for b in range(nb):
        D[b * n:(b + 1) * n, b * n:(b + 1) * n] = blocks[b]
    return D


def test_theorem3_dense_shadow():
    """One iteration on the full (L+M)n x (L+M)n matrices with dense B_i (Eqs. 28, 31):
    the iterate stays block diagonal (Theorem 3) and equals the block computation."""
    P = _problem(1)
    X, Z, y, mu = ipm.initial_state(P)
    X1, Z1, y1, st = ipm.ipm_step(P, X, Z, y, mu)
    Bi = [_dense(np.array([sdp.F_block(P, i, b) for b in range(P.nblocks)])) for i in range(P.K)]
    Xd, Zd, Cd = _dense(X), _dense(Z), _dense(ipm.C_blocks(P))
    W = np.linalg.inv(Zd)
    BT = lambda v: sum(v[i] * Bi[i] for i in range(P.K))          # noqa: E731
    Bop = lambda M: np.array([np.trace(Bi[i] @ M) for i in range(P.K)])  # noqa: E731
    Rd = -BT(y) + Zd + Cd
    G = np.array([[np.trace(Bi[k] @ W @ Bi[l] @ Xd) for l in range(P.K)] for k in range(P.K)])
    dy1 = np.linalg.solve(G, Bop(W @ Rd @ Xd) - 1.0)
    dZ1 = -Rd + BT(dy1)
    dX1 = -Xd + W @ (Rd - BT(dy1)) @ Xd
    dX1 = 0.5 * (dX1 + dX1.T)
    dy2 = np.linalg.solve(G, mu * Bop(W) - Bop(W @ dZ1 @ dX1))
    dZ2 = BT(dy2)
    dX2 = mu * W - W @ dZ1 @ dX1 - W @ dZ2 @ Xd
    dX2 = 0.5 * (dX2 + dX2.T)
    Xn = Xd + st["tp"] * (dX1 + dX2)
    Zn = Zd + st["td"] * (dZ1 + dZ2)
    mask = _dense(np.ones_like(X)) == 0
    assert np.abs(Xn[mask]).max() <= 1e-14 and np.abs(Zn[mask]).max() <= 1e-14
    assert np.allclose(Xn, _dense(X1), atol=1e-12) and np.allclose(Zn, _dense(Z1), atol=1e-12)
    assert np.allclose(y + st["td"] * (dy1 + dy2), y1, atol=1e-12)


def _solve(P, iters=60, eps=1e-8):
    ok, X, Z, y, it = ipm.solve(P, eps=eps, maxit=iters)
    return ok, y


def test_verdict_config1_stable_certified():
    P = _problem(1)
    ok, y = _solve(P)
    assert ok and ipm.grid_check(P, y)


def test_verdict_config1_unstable_not_certified():
    P = _problem("1u")
    ok, y = _solve(P)
    assert not (ok and ipm.grid_check(P, y))


@pytest.mark.parametrize("a1,stable", [(-1.0, True), (1.0, False)])
def test_verdict_scalar_spec_cases(a1, stable):
    # n = 1, l = 2, A1 = a1, A2 = -1
    A = np.array([[[a1]], [[-1.0]]])
    P = sdp.build_problem(A, 1, 2, 1, 1, 1)
    ok, y = _solve(P)
    assert (ok and ipm.grid_check(P, y)) == stable


def test_step_length_closed_form():
    """Reading R5 ("standard line-search between 0 and 1"): for diagonal blocks the
    distance to the PSD boundary is min_i S_ii / (-dS_ii) over the entries with dS_ii < 0, so
    t = min(1, 0.98 * that); with no decreasing direction t = 1."""
    rng = np.random.default_rng(4)
    for _ in range(20):
        nb, n = int(rng.integers(1, 4)), int(rng.integers(1, 6))
        s = rng.uniform(0.1, 3.0, size=(nb, n))
        ds = rng.normal(scale=rng.choice([0.05, 1.0, 20.0]), size=(nb, n))
        S = np.array([np.diag(v) for v in s])
        dS = np.array([np.diag(v) for v in ds])
        neg = ds < 0
        tmax = (s[neg] / -ds[neg]).min() if neg.any() else np.inf
        want = min(1.0, 0.98 * tmax)
        assert abs(ipm.step_length(S, dS) - want) <= 1e-13 * want
        assert abs(ipm.step_length(S, dS, frac=0.5) - min(1.0, 0.5 * tmax)) <= 1e-13
    # no decreasing direction: the full step
    S = np.array([np.eye(3)])
    assert ipm.step_length(S, np.array([np.diag([0.0, 1.0, 2.0])])) == 1.0
    # a congruence leaves t unchanged (t depends on L^-1 dS L^-T only): S = Q D Q^T, dS = Q dD Q^T
    Q, _ = np.linalg.qr(rng.normal(size=(4, 4)))
    D, dD = np.diag([1.0, 2.0, 0.5, 4.0]), np.diag([-3.0, 1.0, -0.1, -1.0])
    assert abs(ipm.step_length(np.array([Q @ D @ Q.T]), np.array([Q @ dD @ Q.T])) - 0.98 / 3.0) <= 1e-12


@pytest.mark.parametrize("case", ["scalar", "1u", "discrete"])
def test_infeasible_cases_exit_by_divergence(case):
    """Reading R20: an infeasible LMI makes the primal iterate unbounded; the solve stops with
    status "diverged" once tr(CX), a^T y or mu passes DIVERGENCE_BOUND -- with no floating-point
    overflow on the way (warnings are errors here)."""
    import warnings
    if case == "scalar":
        P = sdp.build_problem(np.array([[[1.0]], [[-1.0]]]), 1, 2, 1, 1, 1)
    elif case == "1u":
        P = _problem("1u")
    else:
        A = synth.discrete_vertex_matrices(4, 3, 0.8, np.random.default_rng(3), unstable=True)
        P = sdp.build_problem_general(synth.discrete_time_terms(A), 4, 3, 1, 1, 1)
    info = {}
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        ok, X, Z, y, it = ipm.solve(P, info=info)
    assert not ok and info["status"] == "diverged", info
