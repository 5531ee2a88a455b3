"""Pins for oracle.monomials and the counting formulas."""
import math
import os

import pytest

from oracle import polya
from oracle.monomials import enumerate_W, eq1_printed, f, index_map

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_cardinality_examples():
    # SPEC.md:43-46 examples; Eq. (2) "0 for l = 0"
    assert f(0, 5) == 0
    assert f(3, 0) == 1
    assert f(3, 2) == 6
    assert f(10, 6) == 5005


@pytest.mark.parametrize("l", range(1, 7))
def test_enumeration_count_matches_binomial(l):
    # |W_d| by brute force against Eq. (2)'s binomial, 1 <= l <= 6, 0 <= d <= 8
    for d in range(0, 9):
        assert len(enumerate_W(l, d)) == math.comb(l + d - 1, l - 1)


def test_enumeration_examples():
    assert enumerate_W(2, 1) == [(1, 0), (0, 1)]
    assert enumerate_W(1, 4) == [(4,)]
    rows = [tuple(int(x) for x in ln.split()) for ln in open(os.path.join(GOLD, "homogenize_W2_l3.txt"))
            if ln.strip() and not ln.startswith("#")]
    assert enumerate_W(3, 2) == rows      # PAPER.md:128-131 order of B1..B6
    idx = index_map(3, 2)
    assert idx[(2, 0, 0)] + 1 == 1 and idx[(0, 0, 2)] + 1 == 6 and idx[(0, 1, 1)] + 1 == 5


@pytest.mark.parametrize("l,d", [(2, 3), (3, 2), (3, 4), (4, 3), (5, 2), (6, 4)])
def test_order_property_and_R1_complement(l, d):
    W = enumerate_W(l, d)
    # prose order: leftmost non-zero entry of gamma - eta is positive
    for g, e in zip(W, W[1:]):
        diff = [a - b for a, b in zip(g, e)]
        first = next(x for x in diff if x != 0)
        assert first > 0
    # reading R1: printed Eq. (1) ranks the reverse order; <gamma> = f(l,d) + 1 - Eq1(gamma)
    for pos, g in enumerate(W):
        assert pos + 1 == f(l, d) + 1 - eq1_printed(g)


def test_printed_sizes():
    for ln in open(os.path.join(GOLD, "sizes.txt")):
        if not ln.strip() or ln.startswith("#"):
            continue
        n, l, dp, da, d1, d2, K, dim, LM = (int(x) for x in ln.split()[:9])
        L0, L, M = polya.counts(l, dp, da, d1, d2)
        assert L0 * n * (n + 1) // 2 == K
        assert (L + M) * n == dim
        assert L + M == LM


def test_baseline_config_counts():
    # SURVEY.md 8.0 table (derived there; re-derived here by enumeration)
    table = {(4, 2, 1, 1, 1): (2, 3, 4), (10, 3, 2, 2, 2): (6, 15, 21), (30, 4, 2, 3, 3): (10, 56, 84),
             (100, 4, 2, 4, 4): (10, 84, 120), (120, 6, 2, 4, 4): (21, 462, 792)}
    for (n, l, dp, d1, d2), want in table.items():
        assert polya.counts(l, dp, 1, d1, d2) == want


def test_enumeration_brute_force_small():
    import itertools
    for l in range(1, 5):
        for d in range(0, 5):
            brute = sorted((g for g in itertools.product(range(d + 1), repeat=l) if sum(g) == d), reverse=True)
            assert enumerate_W(l, d) == brute
