"""Pins for the oracle's homogenisation, simplex map and full-solve verdicts (SURVEY 8(f) NEXT-1 /
NEXT-3), against what the paper prints:

* homogenisation: the worked example of PAPER.md:120-131 (A = C a1^2 + D a2 + E a3 + F gives
  B1..B6 = C+F, D+2F, E+2F, D+F, D+E+2F, E+F) and B = A on the simplex;
* simplex map: A'(alpha) = A(g(alpha)) at simplex points, and homogeneity of degree d;
* Example 2 (matrices in tests/golden/example2_A.txt): the printed optimum
  L_opt = -0.111 is the 3-decimal value of the stability boundary found by brute force
  (eigenvalues of A(g(alpha)) on a grid of Delta_3: stable at -0.111, unstable at -0.112), which
  also pins reading R17 (g_i = (1-L) alpha_i + L);
* verdicts of the whole method (Theorem 1 via Polya): certified well inside the stable range,
  never certified where brute force finds an unstable point (necessity), and the certified
  range grows with d_p, d1, d2.
"""
import os

import numpy as np
import pytest

from oracle import ipm, polya, sdp
from oracle.monomials import enumerate_W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def example2_terms():
    lines = [ln for ln in open(os.path.join(GOLD, "example2_A.txt")) if not ln.startswith("#")]
    terms = {}
    for k in range(6):
        e = tuple(int(x) for x in lines[4 * k].split()[1:4])
        terms[e] = np.array([[float(x) for x in lines[4 * k + j].split()] for j in range(1, 4)])
    return terms


def example2_A(L):
    da, A = polya.homogenize(example2_terms(), 3)
    assert da == 3
    return polya.simplex_map(A, 3, 3, [1 - L] * 3, [L] * 3)


def test_homogenize_paper_example():
    rng = np.random.default_rng(0)
    C, D, E, F = (rng.normal(size=(2, 2)) for _ in range(4))
    terms = {(2, 0, 0): C, (0, 1, 0): D, (0, 0, 1): E, (0, 0, 0): F}
    da, B = polya.homogenize(terms, 3)
    assert da == 2
    # W_2 order (R1): a1^2, a1a2, a1a3, a2^2, a2a3, a3^2 (tests/golden/homogenize_W2_l3.txt)
    want = [C + F, D + 2 * F, E + 2 * F, D + F, D + E + 2 * F, E + F]
    for got, w in zip(B, want):
        assert np.allclose(got, w, rtol=0, atol=1e-15)
    for al in rng.dirichlet(np.ones(3), size=20):
        a = C * al[0] ** 2 + D * al[1] + E * al[2] + F
        assert np.allclose(polya.evaluate(B, 3, 2, al), a, rtol=1e-13, atol=1e-14)


def test_simplex_map_agrees_with_substitution():
    rng = np.random.default_rng(1)
    l, d = 3, 3
    A = rng.normal(size=(len(enumerate_W(l, d)), 2, 2))
    scale, shift = rng.uniform(0.5, 2.0, size=l), rng.uniform(-1.0, 1.0, size=l)
    Ap = polya.simplex_map(A, l, d, scale, shift)
    for al in rng.dirichlet(np.ones(l), size=20):
        g = scale * al + shift           # on the simplex sum(alpha) = 1
        assert np.allclose(polya.evaluate(Ap, l, d, al), polya.evaluate(A, l, d, g), rtol=1e-12, atol=1e-12)
        t = 1.7                           # homogeneous of degree d off the simplex
        assert np.allclose(polya.evaluate(Ap, l, d, t * al), t ** d * polya.evaluate(Ap, l, d, al), rtol=1e-12)
    # Example 1's map: g_i = 2|rho|(alpha_i - 0.5) sends Delta_l onto S_rho
    rho, l8 = 0.3, 8
    for al in rng.dirichlet(np.ones(l8), size=5):
        g = 2 * rho * al - rho
        assert abs(g.sum() - (2 * rho - l8 * rho)) <= 1e-12 and np.all(np.abs(g) <= rho + 1e-12)


def _max_real_eig(L, N=60):
    A = example2_A(L)
    m = -np.inf
    for i in range(N + 1):
        for j in range(N + 1 - i):
            al = np.array([i, j, N - i - j]) / N
            m = max(m, np.linalg.eigvals(polya.evaluate(A, 3, 3, al)).real.max())
    return m


def test_example2_printed_optimum_is_the_stability_boundary():
    assert _max_real_eig(-0.111) < 0 < _max_real_eig(-0.112)


def _P(L, dp, d1, d2):
    return sdp.build_problem(example2_A(L), 3, 3, dp, d1, d2, da=3)


@pytest.mark.parametrize("L,deg,certified", [(0.4, (1, 1, 1), True), (0.1, (1, 2, 2), True),
                                               (0.0, (1, 1, 1), False), (-0.2, (2, 2, 2), False)])
def test_example2_verdicts(L, deg, certified):
    # -0.2 is unstable (brute force): no Polya certificate may exist at any degree (Theorem 1)
    assert ipm.verdict(_P(L, *deg), samples=300) == certified


def test_example2_unstable_point_exists_below_optimum():
    assert _max_real_eig(-0.2, N=20) > 0
