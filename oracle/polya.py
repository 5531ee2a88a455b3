"""Polya coefficients beta, H and the SDP element C.  TEST INFRASTRUCTURE ONLY.

Definitions followed (Sec. III.A "Polya's Algorithm"):
* beta_{<h>,<gamma>} "is the scalar coefficient which multiplies P_<h> in the
  <gamma>-th monomial of (sum_i alpha_i)^{d1} P(alpha)";
* H_{<h>,<gamma>} "is the term which left or right multiplies P_<h> in the
  <gamma>-th monomial of (sum_i alpha_i)^{d2} (A^T P + P A)",
  i.e. the coefficient of alpha^gamma in (sum alpha)^{d2} alpha^h A(alpha);
* C_i = delta I_n sum_h beta_{<h>,i} d_p!/(h_1!...h_l!) for i <= L, 0 otherwise
  (Eq. Cj).

``beta_table`` / ``H_table`` compute these by *explicit polynomial
multiplication* (dict exponent -> coefficient), ``beta_recursion`` /
``H_recursion`` run Eqs. (19)-(22) literally, for d_p + i
and d_pa + i at step i (reading R8: exactly d1 and d2 steps).
Index convention: positions in W_d under reading R1 (0-based).
"""
from __future__ import annotations

import math

import numpy as np

from .monomials import enumerate_W, index_map

__all__ = ["poly_mul", "simplex_power", "beta_table", "H_table", "beta_recursion",
           "H_recursion", "C_scalars", "counts", "H_row", "homogenize", "simplex_map", "evaluate"]


def poly_mul(p: dict, q: dict) -> dict:
    """Product of two polynomials in alpha given as {exponent tuple: coefficient}.
    Coefficients may be ints, floats or numpy arrays (p's coefficient is the left factor)."""
    out = {}
    for e1, c1 in p.items():
        for e2, c2 in q.items():
            e = tuple(a + b for a, b in zip(e1, e2))
            term = c1 * c2 if not isinstance(c1, np.ndarray) or not isinstance(c2, np.ndarray) else c1 @ c2
            if e in out:
                out[e] = out[e] + term
            else:
                out[e] = term
    return out


def simplex_power(l: int, d: int) -> dict:
    """(sum_i alpha_i)^d by d repeated multiplications of S = sum_i alpha_i."""
    S = {tuple(1 if j == i else 0 for j in range(l)): 1 for i in range(l)}
    out = {tuple([0] * l): 1}
    for _ in range(d):
        out = poly_mul(out, S)
    return out


def counts(l, dp, da, d1, d2):
    """(L0, L, M) of Eqs. (23)-(25) via len(W_d)."""
    return (len(enumerate_W(l, dp)), len(enumerate_W(l, dp + d1)), len(enumerate_W(l, dp + da + d2)))


def beta_table(l: int, dp: int, d1: int) -> np.ndarray:
    """beta[h, g] (L0 x L, int64): coefficient of alpha^gamma_g in (sum alpha)^{d1} alpha^{h}."""
    Wp = enumerate_W(l, dp)
    idx = index_map(l, dp + d1)
    S = simplex_power(l, d1)
    out = np.zeros((len(Wp), len(idx)), dtype=np.int64)
    for hi, h in enumerate(Wp):
        prod = poly_mul(S, {h: 1})
        for e, c in prod.items():
            out[hi, idx[e]] += c
    return out


def H_table(A: np.ndarray, l: int, dp: int, d2: int, da: int = 1) -> np.ndarray:
    """H[h, g] (L0 x M x n x n): coefficient of alpha^gamma_g in (sum alpha)^{d2} alpha^h A(alpha),
    with A(alpha) = sum_{lambda in W_da} A[<lambda>] alpha^lambda (Eq. A_alpha)."""
    Wp = enumerate_W(l, dp)
    Wa = enumerate_W(l, da)
    idx = index_map(l, dp + da + d2)
    n = A.shape[-1]
    Apoly = {lam: A[i] for i, lam in enumerate(Wa)}
    S = simplex_power(l, d2)
    out = np.zeros((len(Wp), len(idx), n, n))
    for hi, h in enumerate(Wp):
        prod = poly_mul(S, poly_mul({h: 1}, Apoly))
        for e, c in prod.items():
            out[hi, idx[e]] += c
    return out


def beta_recursion(l: int, dp: int, d1: int) -> np.ndarray:
    """Eqs. (19)-(20) literally: beta^(0) = Kronecker delta on W_dp; for i = 1..d1,
    beta^(i)_{h,gamma} = sum_{lambda in W_1} beta^(i-1)_{h,gamma-lambda}, gamma in W_{dp+i}
    (terms with a negative entry of gamma-lambda are absent)."""
    Wp = enumerate_W(l, dp)
    prev_idx = index_map(l, dp)
    prev = np.eye(len(Wp), dtype=np.int64)
    W1 = enumerate_W(l, 1)
    for i in range(1, d1 + 1):
        Wi = enumerate_W(l, dp + i)
        cur = np.zeros((len(Wp), len(Wi)), dtype=np.int64)
        for gi, g in enumerate(Wi):
            for lam in W1:
                e = tuple(a - b for a, b in zip(g, lam))
                if min(e) < 0:
                    continue
                cur[:, gi] += prev[:, prev_idx[e]]
        prev, prev_idx = cur, index_map(l, dp + i)
    return prev


def H_recursion(A: np.ndarray, l: int, dp: int, d2: int, da: int = 1) -> np.ndarray:
    """Eqs. (21)-(22) literally: H^(0)_{h,gamma} = sum_{lambda in W_da: lambda+h=gamma} A_lambda
    for gamma in W_{dp+da}; then d2 steps of the W_1 shift-and-sum recursion."""
    Wp = enumerate_W(l, dp)
    Wa = enumerate_W(l, da)
    W0 = enumerate_W(l, dp + da)
    n = A.shape[-1]
    prev = np.zeros((len(Wp), len(W0), n, n))
    prev_idx = index_map(l, dp + da)
    for hi, h in enumerate(Wp):
        for gi, g in enumerate(W0):
            for li, lam in enumerate(Wa):
                if tuple(a + b for a, b in zip(lam, h)) == g:
                    prev[hi, gi] += A[li]
    W1 = enumerate_W(l, 1)
    for i in range(1, d2 + 1):
        Wi = enumerate_W(l, dp + da + i)
        cur = np.zeros((len(Wp), len(Wi), n, n))
        for gi, g in enumerate(Wi):
            for lam in W1:
                e = tuple(a - b for a, b in zip(g, lam))
                if min(e) < 0:
                    continue
                cur[:, gi] += prev[:, prev_idx[e]]
        prev, prev_idx = cur, index_map(l, dp + da + i)
    return prev


def C_scalars(beta: np.ndarray, l: int, dp: int, delta: float) -> np.ndarray:
    """c_i with C_i = c_i I_n, i < L (Eq. Cj):
    c_i = delta * sum_h beta_{h,i} * dp! / (h_1! ... h_l!)."""
    Wp = enumerate_W(l, dp)
    w = np.array([math.factorial(dp) // math.prod(math.factorial(x) for x in h) for h in Wp], dtype=np.int64)
    return delta * (w @ beta).astype(np.float64)


def H_row(A: np.ndarray, l: int, dp: int, d2: int, h_index: int, da: int = 1) -> np.ndarray:
    """One row h of ``H_table`` (M x n x n), same polynomial multiplication, for large configs."""
    Wp = enumerate_W(l, dp)
    Wa = enumerate_W(l, da)
    idx = index_map(l, dp + da + d2)
    n = A.shape[-1]
    Apoly = {lam: A[i] for i, lam in enumerate(Wa)}
    prod = poly_mul(simplex_power(l, d2), poly_mul({Wp[h_index]: 1}, Apoly))
    out = np.zeros((len(idx), n, n))
    for e, c in prod.items():
        out[idx[e]] += c
    return out


def homogenize(terms: dict, l: int):
    """The homogenisation procedure of PAPER.md:113-132: with d_a the degree of A(alpha), the
    i-th monomial of A is multiplied by (sum_j alpha_j)^{d_a - d_{a_i}} (so B = A on Delta_l).
    terms: {exponent tuple: coefficient (scalar or n x n array)}.  Returns (d_a, coefficient array
    of B in W_{d_a} order), expanded by explicit polynomial multiplication."""
    da = max(sum(e) for e in terms)
    idx = index_map(l, da)
    c0 = np.asarray(next(iter(terms.values())), dtype=float)
    out = np.zeros((len(idx),) + c0.shape)
    for e, c in terms.items():
        for e2, k in poly_mul(simplex_power(l, da - sum(e)), {tuple(e): 1}).items():
            out[idx[e2]] += k * np.asarray(c, dtype=float)
    return da, out


def simplex_map(A: np.ndarray, l: int, d: int, scale, shift) -> np.ndarray:
    """Coefficients (W_d order) of A'(alpha) = A(g(alpha)) for a homogeneous A of degree d given in
    W_d order and the affine simplex map g_i(alpha) = scale_i alpha_i + shift_i, homogenised on
    Delta_l as g_i = scale_i alpha_i + shift_i (sum_j alpha_j).  Example 1's map is
    scale = 2|rho|, shift = -|rho|; Example 2 "defines g as in Example 1" for
    S_L, read as scale = 1 - L, shift = L (reading R17)."""
    Wd = enumerate_W(l, d)
    idx = index_map(l, d)
    unit = lambda i: tuple(1 if j == i else 0 for j in range(l))  # noqa: E731
    g = []
    for i in range(l):
        gi = {unit(j): float(shift[i]) for j in range(l)}
        gi[unit(i)] = gi[unit(i)] + float(scale[i])
        g.append(gi)
    out = np.zeros_like(np.asarray(A, dtype=float))
    for k, lam in enumerate(Wd):
        prod = {tuple([0] * l): 1.0}
        for i in range(l):
            for _ in range(lam[i]):
                prod = poly_mul(prod, g[i])
        for e, c in prod.items():
            out[idx[e]] += c * A[k]
    return out


def evaluate(A: np.ndarray, l: int, d: int, alpha) -> np.ndarray:
    """sum_{lambda in W_d} A[<lambda>] alpha^lambda (Eq. A_alpha)."""
    return sum(math.prod(a ** e for a, e in zip(alpha, lam)) * A[i] for i, lam in enumerate(enumerate_W(l, d)))
