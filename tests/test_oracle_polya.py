"""Pins for oracle.polya: beta, H, C.

Pins used: the paper's worked beta/H tables
(golden files), the multinomial closed forms (beta_{h,g} = multinomial(d1; g-h),
H_{h,g} = sum_i multinomial(d2; g-h-e_i) A_i, c_g = delta multinomial(dp+d1; g)),
row sums, the literal recursions, and agreement of the polynomial with its
expansion at random (non-normalised) points and at the simplex vertices.
"""
import math
import os

import numpy as np
import pytest

from oracle import polya
from oracle.monomials import enumerate_W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SHAPES = [(2, 1, 1, 1), (3, 2, 2, 2), (4, 2, 3, 3), (3, 1, 2, 3), (4, 2, 4, 4), (2, 3, 0, 2), (3, 0, 2, 1)]


def mnom(d, parts):
    if any(p < 0 for p in parts) or sum(parts) != d:
        return 0
    return math.factorial(d) // math.prod(math.factorial(p) for p in parts)


def _golden(name):
    return [[int(x) for x in ln.split()] for ln in open(os.path.join(GOLD, name))
            if ln.strip() and not ln.startswith("#")]


def test_beta_paper_table():
    want = np.array(_golden("beta_l2_dp1_d1.txt"))
    assert np.array_equal(polya.beta_table(2, 1, 1), want)
    assert np.array_equal(polya.beta_recursion(2, 1, 1), want)


def test_H_paper_table():
    rng = np.random.default_rng(7)
    A = rng.normal(size=(2, 3, 3))
    H = polya.H_table(A, 2, 1, 1)
    Hr = polya.H_recursion(A, 2, 1, 1)
    assert H.shape == (2, 4, 3, 3)
    for h, g, c1, c2 in _golden("H_l2_dp1_da1_d2_1.txt"):
        want = c1 * A[0] + c2 * A[1]
        assert np.array_equal(H[h - 1, g - 1], want)
        assert np.array_equal(Hr[h - 1, g - 1], want)


@pytest.mark.parametrize("l,dp,d1,d2", SHAPES)
def test_beta_closed_form_recursion_rowsums(l, dp, d1, d2):
    B = polya.beta_table(l, dp, d1)
    Wp, WL = enumerate_W(l, dp), enumerate_W(l, dp + d1)
    closed = np.array([[mnom(d1, [a - b for a, b in zip(g, h)]) for g in WL] for h in Wp])
    assert np.array_equal(B, closed)
    assert np.array_equal(B, polya.beta_recursion(l, dp, d1))
    assert np.all(B.sum(axis=1) == l ** d1)


@pytest.mark.parametrize("l,dp,d1,d2", SHAPES)
def test_H_closed_form_recursion_rowsums(l, dp, d1, d2):
    rng = np.random.default_rng(l * 100 + dp * 10 + d2)
    n = 3
    A = rng.normal(size=(l, n, n))
    H = polya.H_table(A, l, dp, d2)
    Wp, WM = enumerate_W(l, dp), enumerate_W(l, dp + 1 + d2)
    for hi, h in enumerate(Wp):
        Hrow = polya.H_row(A, l, dp, d2, hi)     # one row h alone (used at config 5's size)
        assert Hrow.shape == (len(WM), n, n)
        for gi, g in enumerate(WM):
            want = np.zeros((n, n))
            for i in range(l):
                parts = [g[j] - h[j] - (1 if j == i else 0) for j in range(l)]
                want += mnom(d2, parts) * A[i]
            assert np.allclose(H[hi, gi], want, rtol=0, atol=1e-12 * max(1.0, np.abs(want).max()))
            assert np.allclose(Hrow[gi], want, rtol=0, atol=1e-12 * max(1.0, np.abs(want).max()))
    assert np.allclose(H, polya.H_recursion(A, l, dp, d2), rtol=0, atol=1e-12)
    rs = H.sum(axis=1)
    for hi in range(len(Wp)):
        assert np.allclose(rs[hi], l ** d2 * A.sum(axis=0), rtol=1e-12, atol=1e-12)


def test_H_degree_two_A():
    # d_a = 2 (general closed form H = sum_lambda multinomial(d2; g-h-lambda) A_lambda)
    l, dp, d2, da, n = 3, 1, 2, 2, 2
    rng = np.random.default_rng(3)
    Wa = enumerate_W(l, da)
    A = rng.normal(size=(len(Wa), n, n))
    H = polya.H_table(A, l, dp, d2, da)
    assert np.allclose(H, polya.H_recursion(A, l, dp, d2, da), atol=1e-12)
    for hi, h in enumerate(enumerate_W(l, dp)):
        for gi, g in enumerate(enumerate_W(l, dp + da + d2)):
            want = sum(mnom(d2, [g[j] - h[j] - lam[j] for j in range(l)]) * A[li] for li, lam in enumerate(Wa))
            assert np.allclose(H[hi, gi], want, atol=1e-12)
            assert np.allclose(polya.H_row(A, l, dp, d2, hi, da)[gi], want, atol=1e-12)


def test_C_spec_example_and_closed_form():
    # l=2, dp=d1=1, delta=1 -> c = (1, 2, 1)
    c = polya.C_scalars(polya.beta_table(2, 1, 1), 2, 1, 1.0)
    assert np.array_equal(c, [1.0, 2.0, 1.0])
    for l, dp, d1, _ in SHAPES:
        c = polya.C_scalars(polya.beta_table(l, dp, d1), l, dp, 1e-3)
        want = [1e-3 * mnom(dp + d1, g) for g in enumerate_W(l, dp + d1)]
        assert np.allclose(c, want, rtol=1e-15, atol=0)


def _mono(alpha, g):
    return math.prod(a ** e for a, e in zip(alpha, g))


@pytest.mark.parametrize("l,dp,d1,d2", SHAPES)
def test_polynomial_agreement(l, dp, d1, d2):
    """Expansion vs direct evaluation at 20 random POSITIVE points (not normalised, so a dropped
    (sum alpha)^d factor fails) and at all l vertices."""
    rng = np.random.default_rng(11 + l + dp + d1 + d2)
    n = 3
    A = rng.normal(size=(l, n, n))
    Wp, WL, WM = enumerate_W(l, dp), enumerate_W(l, dp + d1), enumerate_W(l, dp + 1 + d2)
    Ph = [(lambda m: m + m.T)(rng.normal(size=(n, n))) for _ in Wp]
    B = polya.beta_table(l, dp, d1)
    H = polya.H_table(A, l, dp, d2)
    pts = [rng.uniform(0.1, 2.0, size=l) for _ in range(20)] + [np.eye(l)[i] for i in range(l)]
    for al in pts:
        s = al.sum()
        P = sum(_mono(al, h) * Ph[i] for i, h in enumerate(Wp))
        Aa = sum(al[i] * A[i] for i in range(l))
        lhs1 = sum(_mono(al, g) * sum(B[h, gi] * Ph[h] for h in range(len(Wp))) for gi, g in enumerate(WL))
        rhs1 = s ** d1 * P
        lhs2 = sum(_mono(al, g) * sum(H[h, gi].T @ Ph[h] + Ph[h] @ H[h, gi] for h in range(len(Wp)))
                   for gi, g in enumerate(WM))
        rhs2 = s ** d2 * (Aa.T @ P + P @ Aa)
        assert np.linalg.norm(lhs1 - rhs1) <= 1e-12 * max(1.0, np.linalg.norm(rhs1))
        assert np.linalg.norm(lhs2 - rhs2) <= 1e-12 * max(1.0, np.linalg.norm(rhs2))
