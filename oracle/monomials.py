"""Exponent sets W_d and their index map (Notation).  TEST INFRASTRUCTURE ONLY.

Reading R1: the prose at PAPER.md:58 orders W_d lexicographically
with gamma preceding eta "if the left most non-zero entry of gamma-eta is
positive", i.e. (d,0,...,0) first -- *descending* lexicographic order.  Every
worked example uses that order (B1..B6 at PAPER.md:128-131, the beta/H tables
at PAPER.md:197-215).  Eq. (1) as printed gives the reverse
rank; ``eq1_printed`` evaluates it literally so a test can pin the complement
identity  <gamma> = f(l,d) + 1 - Eq1(gamma).
"""
from __future__ import annotations

import math

__all__ = ["f", "enumerate_W", "index_map", "eq1_printed", "multinomial"]


def f(l: int, d: int) -> int:
    """Eq. (2): |W_d| = 0 for l = 0, else C(l+d-1, l-1)."""
    if l == 0:
        return 0
    return math.comb(l + d - 1, l - 1)


def _compositions(l: int, d: int):
    """Every tuple of l non-negative integers with sum d (first entry, then the rest)."""
    if l == 1:
        yield (d,)
        return
    for first in range(d + 1):
        for rest in _compositions(l - 1, d - first):
            yield (first,) + rest


def enumerate_W(l: int, d: int):
    """W_d: every exponent in N^l with sum d, sorted by the prose order:
    gamma precedes eta iff the leftmost non-zero entry of gamma-eta is positive, i.e.
    descending lexicographic order.  Returns a list of tuples."""
    if l == 0:
        return []
    cands = list(_compositions(l, d))
    assert all(sum(g) == d and min(g) >= 0 for g in cands)
    cands.sort(reverse=True)
    return cands


def index_map(l: int, d: int):
    """{gamma: 0-based position in W_d}.  The paper's <gamma> is position + 1."""
    return {g: i for i, g in enumerate(enumerate_W(l, d))}


def eq1_printed(gamma) -> int:
    """Eq. (1) exactly as printed, 1-based:
    <gamma> = sum_{j=1}^{l-1} sum_{i=1}^{gamma_j} f(l-j, d+1-sum_{k<j} gamma_k - i) + 1.
    (the printed inner sum is over i = 1..gamma_i with gamma_i read as gamma_j)."""
    l = len(gamma)
    d = sum(gamma)
    total = 0
    for j in range(1, l):
        prefix = sum(gamma[: j - 1])
        for i in range(1, gamma[j - 1] + 1):
            total += f(l - j, d + 1 - prefix - i)
    return total + 1


def multinomial(d: int, parts) -> int:
    """d! / prod(parts_i!) with sum(parts) = d; 0 if any part is negative."""
    if any(p < 0 for p in parts) or sum(parts) != d:
        return 0
    out = math.factorial(d)
    for p in parts:
        out //= math.factorial(p)
    return out
