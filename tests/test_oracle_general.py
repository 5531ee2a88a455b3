"""Pins for the oracle's generalised LMI form (reading R18 in DESIGN.md):
    sum_i (At_i(alpha) P(alpha) Bt_i(alpha) + Bt_i(alpha)^T P(alpha) At_i(alpha)^T) < 0,  square case, R_i = 0.

* the continuous-time LMI is the case [(A^T, 1, I, 0)]: every operator and the Schur complement
  equal those of build_problem (itself pinned in test_oracle_sdp.py);
* Polya's coefficient blocks are a polynomial identity: at random alpha,
  sum_gamma alpha^gamma B^T(y)_{L+gamma} = -(sum alpha)^{d2} sum_i (At_i P Bt_i + transpose)(alpha)
  with P(alpha) = sum_h alpha^h V_h(y), evaluated by plain substitution (not by build's products);
* the adjoint identity <B^T(y), X> = y^T B(X) and G y = B(X B^T(y) W) (two routes to G);
* discrete-time robust stability (A^T P A - P < 0): a contraction polytope is certified, a polytope
  with a vertex of spectral radius 1.05 is not (Theorem 1's certificate is sufficient, and no P
  exists when a vertex is unstable).
"""
import math

import numpy as np
import pytest

import synth
from oracle import ipm, polya, sdp
from oracle.monomials import enumerate_W


def _f(l):
    return lambda d: len(enumerate_W(l, d))


def test_continuous_time_is_the_special_case():
    c = synth.small_config(4, 3, 2, 1, 2)
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(c, rng)
    P = sdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    Pg = sdp.build_problem_general([(np.array([a.T for a in A]), 1, np.eye(c.n)[None], 0)], c.n, c.l, c.dp, c.d1, c.d2)
    assert (P.M, P.K, P.L) == (Pg.M, Pg.K, Pg.L)
    assert all(P.active(h, b) == Pg.active(h, b) for h in range(P.L0) for b in range(P.nblocks))
    X, W = synth.spd_blocks(c.n, P.nblocks, rng)
    y = rng.normal(size=P.K)
    G = sdp.schur_literal(P, X, W)
    assert np.abs(sdp.schur_literal(Pg, X, W) - G).max() <= 1e-13 * np.abs(G).max()
    T = sdp.apply_vmap(P, y)
    assert np.abs(sdp.apply_vmap(Pg, y) - T).max() <= 1e-13 * np.abs(T).max()
    b = sdp.adjoint_trace(P, X)
    assert np.abs(sdp.adjoint_trace(Pg, X) - b).max() <= 1e-13 * np.abs(b).max()


@pytest.mark.parametrize("degs,shape", [([(1, 1), (2, 0)], (3, 2, 1, 1, 2)), ([(0, 2), (1, 1), (2, 0)], (2, 3, 1, 2, 1)),
                                        ([(1, 0)], (3, 2, 2, 1, 0))])
def test_polya_blocks_are_a_polynomial_identity(degs, shape):
    n, l, dp, d1, d2 = shape
    rng = np.random.default_rng(1)
    terms = synth.random_terms(n, l, degs, rng, _f(l))
    P = sdp.build_problem_general(terms, n, l, dp, d1, d2)
    y = rng.normal(size=P.K)
    out = sdp.apply_vmap(P, y)
    Wp, Wm = enumerate_W(l, dp), enumerate_W(l, P.da + dp + d2)
    V = [sdp.vmap(P, y, h) for h in range(P.L0)]
    for _ in range(4):
        al = rng.dirichlet(np.ones(l)) * rng.uniform(0.5, 2.0)     # identity holds off the simplex too
        mono = lambda e: math.prod(a ** k for a, k in zip(al, e))
        Pa = sum(mono(h) * V[i] for i, h in enumerate(Wp))
        lhs = sum(mono(g) * out[P.L + m] for m, g in enumerate(Wm))
        S = sum(polya.evaluate(At, l, a, al) @ Pa @ polya.evaluate(Bt, l, b, al) for At, a, Bt, b in terms)
        rhs = -(sum(al) ** d2) * (S + S.T)
        assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    # the P-blocks are untouched by the generalisation: sum_h beta_hj V_h
    for j in range(P.L):
        assert np.allclose(out[j], sum(P.beta[h, j] * V[h] for h in range(P.L0)), rtol=0, atol=1e-13 * np.abs(out[j]).max() + 1e-300)


def test_adjoint_and_two_routes_to_G():
    n, l, dp, d1, d2 = 3, 2, 1, 1, 1
    rng = np.random.default_rng(2)
    terms = synth.random_terms(n, l, [(1, 1), (2, 0)], rng, _f(l))
    P = sdp.build_problem_general(terms, n, l, dp, d1, d2)
    X, W = synth.spd_blocks(n, P.nblocks, rng)
    y = rng.normal(size=P.K)
    T = sdp.apply_vmap(P, y)
    lhs = sum(np.sum(T[b] * X[b]) for b in range(P.nblocks))
    assert abs(lhs - y @ sdp.adjoint_trace(P, X)) <= 1e-12 * abs(lhs)
    G = sdp.schur_literal(P, X, W)
    Gs = sdp.schur_structured(P, X, W)      # the rank-structured route (used at larger sizes)
    assert np.abs(Gs - G).max() <= 1e-12 * np.abs(G).max()
    assert np.allclose(G, G.T, rtol=0, atol=1e-12 * np.abs(G).max())
    rows = [0, 3, P.K - 1]
    assert np.abs(sdp.schur_rows(P, X, W, rows) - G[rows]).max() <= 1e-12 * np.abs(G).max()
    pairs = [(int(i), int(j)) for i, j in rng.integers(0, P.K, size=(9, 2))]
    assert np.abs(sdp.schur_entries(P, X, W, pairs) - [G[i, j] for i, j in pairs]).max() <= 1e-12 * np.abs(G).max()
    Y = np.array([X[b] @ T[b] @ W[b] for b in range(P.nblocks)])
    Y = 0.5 * (Y + Y.transpose(0, 2, 1))
    Gy = sdp.adjoint_trace(P, Y)
    assert np.abs(G @ y - Gy).max() <= 1e-11 * np.abs(Gy).max()
    assert np.linalg.eigvalsh(G).min() > -1e-10 * np.abs(G).max()


@pytest.mark.parametrize("unstable", [False, True])
def test_discrete_time_verdicts(unstable):
    n, l = 3, 2
    A = synth.discrete_vertex_matrices(n, l, 0.8, np.random.default_rng(3), unstable=unstable)
    P = sdp.build_problem_general(synth.discrete_time_terms(A), n, l, 1, 1, 1)
    assert ipm.verdict(P, samples=200) == (not unstable)
    if unstable:   # the vertex itself violates A^T P A - P < 0 for every P > 0
        assert max(abs(np.linalg.eigvals(A[0]))) > 1.0


def _scalar_vertex_problem(avals, r, d2=0):
    """n = 1, dp = 0: A(alpha) = sum a_i alpha_i, R(alpha) = r sum alpha_i; min y = p s.t. p >= delta c
    and -(2 a_i p + r) >= 0 at every vertex, so p* = max(delta, max_i r / (2 |a_i|))."""
    l = len(avals)
    A = np.array(avals, dtype=float).reshape(l, 1, 1)
    R = np.full((l, 1, 1), float(r))
    return sdp.build_problem_general([(A, 1, np.ones((1, 1, 1)), 0)], 1, l, 0, 0, d2, R=R)


@pytest.mark.parametrize("avals,r", [([-1.0], 3.0), ([-1.0, -0.5], 3.0), ([-2.0, -1.0, -4.0], 1.0)])
def test_constant_term_scalar_closed_form(avals, r):
    """R enters as C on the Lyapunov blocks with the sign of the paper's LMI (sum ... + R < 0): the
    IPM's optimum is the closed form p* = max_i r / (2 |a_i|) (a sign error gives p* = delta c)."""
    P = _scalar_vertex_problem(avals, r)
    ok, X, Z, y, it = ipm.solve(P)
    assert ok
    assert abs(y[0] - max(r / (2 * abs(a)) for a in avals)) <= 1e-6


def test_constant_term_polynomial_identity():
    n, l, dp, d1, d2 = 3, 2, 1, 1, 2
    rng = np.random.default_rng(4)
    terms = synth.random_terms(n, l, [(1, 1)], rng, _f(l))
    Wr = enumerate_W(l, dp + 2)
    R = rng.normal(size=(len(Wr), n, n))
    R = R + R.transpose(0, 2, 1)
    P = sdp.build_problem_general(terms, n, l, dp, d1, d2, R=R)
    C = ipm.C_blocks(P)
    Wm = enumerate_W(l, dp + 2 + d2)
    for _ in range(3):
        al = rng.uniform(0.2, 1.5, size=l)
        lhs = sum(math.prod(a ** k for a, k in zip(al, g)) * C[P.L + m] for m, g in enumerate(Wm))
        rhs = sum(al) ** d2 * polya.evaluate(R, l, dp + 2, al)
        assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    # and the P-blocks keep c_j I
    assert np.array_equal(C[0], P.c[0] * np.eye(n))


# ---- non-square form (reading R19): the bounded-real lemma, N = n + m --------------------------------

def _brl_problem(A, Bu, Cy, gamma, dp, d1, d2):
    terms, R0 = synth.bounded_real_terms(A, Bu, Cy, gamma)
    l, n = A.shape[0], A.shape[1]
    _, R = polya.homogenize({tuple([dp + 1] + [0] * (l - 1)): 0.0 * R0, tuple([0] * l): R0}, l)
    return sdp.build_problem_general(terms, n, l, dp, d1, d2, R=R)


def _hinf(A, Bu, Cy, w=np.concatenate([[0.0], np.logspace(-3, 3, 2001)])):
    """max over a frequency grid of sigma_max(Cy (jw I - A)^-1 Bu) (brute force)."""
    n = A.shape[0]
    return max(np.linalg.svd(Cy @ np.linalg.solve(1j * x * np.eye(n) - A, Bu), compute_uv=False)[0] for x in w)


@pytest.mark.parametrize("a,b,c", [(1.0, 1.0, 1.0), (2.0, 3.0, 0.5), (0.5, 1.0, 2.0)])
def test_bounded_real_scalar_closed_form(a, b, c):
    """x' = -a x + b u, y = c x: ||G||_inf = |c b| / a.  Certified at 1.05 of it, not at 0.95: the
    non-square blocks (N = 2 > n = 1), the padded P-blocks and R together."""
    A, Bu, Cy = np.array([[[-a]]]), np.array([[b]]), np.array([[c]])
    g = abs(c * b) / a
    assert abs(_hinf(A[0], Bu, Cy) - g) <= 1e-6 * g
    assert ipm.verdict(_brl_problem(A, Bu, Cy, 1.05 * g, 0, 0, 0), samples=10)
    assert not ipm.verdict(_brl_problem(A, Bu, Cy, 0.95 * g, 0, 0, 0), samples=10)


def test_bounded_real_polytope_bounds_the_worst_vertex():
    """A certificate at gamma implies ||G_alpha||_inf < gamma for every alpha: never certified below
    the brute-force worst case over the simplex; certified comfortably above it."""
    rng = np.random.default_rng(6)
    c = synth.small_config(2, 2, 1, 1, 1)
    A = synth.vertex_matrices(c, rng)
    Bu, Cy = rng.normal(size=(2, 1)), rng.normal(size=(1, 2))
    worst = max(_hinf(t * A[0] + (1 - t) * A[1], Bu, Cy) for t in np.linspace(0, 1, 11))
    assert not ipm.verdict(_brl_problem(A, Bu, Cy, 0.97 * worst, 1, 1, 1), samples=50)
    assert ipm.verdict(_brl_problem(A, Bu, Cy, 1.5 * worst, 1, 1, 1), samples=50)


def test_non_square_polynomial_identity_and_adjoint():
    n, N, l, dp, d1, d2 = 2, 3, 2, 1, 1, 1
    rng = np.random.default_rng(8)
    f = _f(l)
    terms = [(rng.normal(size=(f(1), N, n)), 1, rng.normal(size=(f(1), n, N)), 1),
             (rng.normal(size=(f(2), N, n)), 2, rng.normal(size=(f(0), n, N)), 0)]
    P = sdp.build_problem_general(terms, n, l, dp, d1, d2)
    assert P.bn == N
    y = rng.normal(size=P.K)
    out = sdp.apply_vmap(P, y)
    assert out.shape == (P.nblocks, N, N)
    assert not np.any(out[:P.L, n:, :]) and not np.any(out[:P.L, :, n:])   # P-blocks: top-left only
    Wp, Wm = enumerate_W(l, dp), enumerate_W(l, dp + 2 + d2)
    V = [sdp.vmap(P, y, h) for h in range(P.L0)]
    al = rng.uniform(0.2, 1.5, size=l)
    mono = lambda e: math.prod(a ** k for a, k in zip(al, e))
    Pa = sum(mono(h) * V[i] for i, h in enumerate(Wp))
    lhs = sum(mono(g) * out[P.L + m] for m, g in enumerate(Wm))
    S = sum(polya.evaluate(At, l, a, al) @ Pa @ polya.evaluate(Bt, l, b, al) for At, a, Bt, b in terms)
    assert np.abs(lhs + sum(al) ** d2 * (S + S.T)).max() <= 1e-12 * np.abs(lhs).max()
    X, W = synth.spd_blocks(N, P.nblocks, rng)
    lhs = sum(np.sum(out[b] * X[b]) for b in range(P.nblocks))
    assert abs(lhs - y @ sdp.adjoint_trace(P, X)) <= 1e-12 * abs(lhs)
    G = sdp.schur_literal(P, X, W)
    assert np.abs(sdp.schur_structured(P, X, W) - G).max() <= 1e-12 * np.abs(G).max()
    rows = [1, P.K // 2, P.K - 1]
    assert np.abs(sdp.schur_rows(P, X, W, rows) - G[rows]).max() <= 1e-12 * np.abs(G).max()
