"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the Polya/SDP method (no enumeration, no
beta/H, no operators, no Schur complement).  It only draws the random data the
paper's experiments use ("random linear systems", Sec. V
Ex. 3) in the shapes BASELINE.json's five configs name, following the recipe in
SURVEY.md Sec. 8(d) / DESIGN.md "Input recipe".  Both sides receive the same
bytes; neither side imports the other.

Draw order (all from one ``numpy.random.default_rng(seed)``, PCG64):
  1. the vertex matrices A_1..A_l (config-specific recipe below);
  2. for b = 0 .. nblocks-1: R (n x (n+5)) then R' (n x (n+5)), iid N(0,1);
     X_b = R R^T/(n+5), Z_b = R' R'^T/(n+5) (Wishart, n+5 dof, E = I).
``nblocks`` (= L + M, the number of Polya blocks) is supplied by the caller.
Z_b^{-1} is formed here in FP64 (an *input* of the Schur assembly, BASELINE.json
config 4: "Z_h^-1 precomputed") and X_b, Z_b^{-1} are symmetrised exactly.
"""
from __future__ import annotations

import dataclasses

import numpy as np

__all__ = ["CONFIGS", "Config", "vertex_matrices", "spd_blocks", "make_case", "small_config",
           "discrete_vertex_matrices", "discrete_time_terms", "random_terms", "bounded_real_terms"]


@dataclasses.dataclass(frozen=True)
class Config:
    """Problem shape: n states, l uncertain parameters, degrees dp (of P), da (of A), d1, d2."""
    name: str
    n: int
    l: int
    dp: int
    d1: int
    d2: int
    da: int = 1
    recipe: str = "random"      # "cfg1" | "random" | "sparse" | "heat"
    unstable: bool = False      # config 1's unstable copy (A_2 += 3I)


# BASELINE.json "configs" (indices 1..5 here; configs[0] of BASELINE.json is cfg 1).
CONFIGS = {
    1: Config("cfg1", n=4, l=2, dp=1, d1=1, d2=1, recipe="cfg1"),
    "1u": Config("cfg1_unstable", n=4, l=2, dp=1, d1=1, d2=1, recipe="cfg1", unstable=True),
    2: Config("cfg2", n=10, l=3, dp=2, d1=2, d2=2, recipe="random"),
    3: Config("cfg3", n=30, l=4, dp=2, d1=3, d2=3, recipe="sparse"),
    4: Config("cfg4", n=100, l=4, dp=2, d1=4, d2=4, recipe="heat"),
    5: Config("cfg5", n=120, l=6, dp=2, d1=4, d2=4, recipe="random"),
}


def small_config(n, l, dp, d1, d2, name=None):
    """Extra parity shapes (ragged tails, several tiles) drawn with the config-2 recipe."""
    return Config(name or f"n{n}l{l}dp{dp}d{d1}{d2}", n=n, l=l, dp=dp, d1=d1, d2=d2, recipe="random")


def _sym_upper(rng, n, std):
    u = np.triu(rng.normal(0.0, std, size=(n, n)))
    return u + np.triu(u, 1).T


def _skew(rng, n):
    u = np.triu(rng.normal(0.0, 1.0, size=(n, n)), 1)
    return u - u.T


def vertex_matrices(cfg: Config, rng) -> np.ndarray:
    """A_1..A_l, shape (l, n, n), float64, for A(alpha) = sum_i alpha_i A_i (d_a = 1)."""
    n, l = cfg.n, cfg.l
    if cfg.recipe == "cfg1":
        A = []
        for _ in range(l):
            S = _sym_upper(rng, n, 0.1)
            K = _skew(rng, n)
            A.append(-2.0 * np.eye(n) + S + K)
        A = np.array(A)
        if cfg.unstable:
            A[1] += 3.0 * np.eye(n)
        return A
    if cfg.recipe in ("random", "sparse"):
        G = np.array([rng.normal(0.0, 1.0, size=(n, n)) for _ in range(l)])
        if cfg.recipe == "sparse":
            nz = int(round(0.2 * n * n))
            for i in range(l):
                idx = rng.choice(n * n, nz, replace=False)
                G[i].reshape(-1)[idx] = 0.0
        lam = max(np.linalg.eigvalsh((g + g.T) / (2.0 * np.sqrt(n))).max() for g in G)
        c = 0.5 + lam + 0.01
        return np.array([-c * np.eye(n) + g / np.sqrt(n) for g in G])
    if cfg.recipe == "heat":
        D = -2.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
        kappa = rng.uniform(0.5, 1.5, size=l)
        A = []
        for i in range(l):
            E = rng.normal(0.0, 0.1, size=(n, n))        # N(0, 0.01): 0.01 read as the variance
            A.append(kappa[i] * (n + 1) ** 2 * D + E)
        A = np.array(A)
        for a in A:
            assert np.linalg.eigvalsh(a + a.T).max() < 0.0
        return A
    raise ValueError(cfg.recipe)


def spd_blocks(n: int, nblocks: int, rng):
    """X_b, Z_b^{-1} stacks (nblocks, n, n): Wishart(n+5)/(n+5), exactly symmetric."""
    X = np.empty((nblocks, n, n))
    W = np.empty((nblocks, n, n))
    for b in range(nblocks):
        R = rng.normal(0.0, 1.0, size=(n, n + 5))
        R2 = rng.normal(0.0, 1.0, size=(n, n + 5))
        x = R @ R.T / (n + 5)
        z = R2 @ R2.T / (n + 5)
        w = np.linalg.inv(z)
        X[b] = 0.5 * (x + x.T)
        W[b] = 0.5 * (w + w.T)
    return X, W


def make_case(cfg: Config, nblocks: int, seed: int = 0):
    """Return (A, X, W) for one config: A (l,n,n); X, W = Z^{-1} (nblocks,n,n)."""
    rng = np.random.default_rng(seed)
    A = vertex_matrices(cfg, rng)
    X, W = spd_blocks(cfg.n, nblocks, rng)
    return A, X, W


# ---- generalised LMI form (reading R18) --------------------------------
# A term list is [(At, a, Bt, b), ...]: At has shape (f(l, a), n, n), Bt (f(l, b), n, n), the
# coefficients of At_i(alpha), Bt_i(alpha) in the library's W_d order; for degree 1 that order is
# e_1, ..., e_l (vertex order), the only one used below.

def discrete_vertex_matrices(n: int, l: int, rho: float, rng, unstable: bool = False) -> np.ndarray:
    """Vertices of a discrete-time polytope x+ = A(alpha) x: iid N(0,1) matrices scaled to spectral
    norm rho (< 1: every A(alpha) on the simplex is a contraction, so P = I certifies it).  With
    ``unstable`` vertex 1 becomes 1.05 Q (Q orthogonal): spectral radius 1.05, not Schur stable."""
    A = []
    for _ in range(l):
        g = rng.normal(0.0, 1.0, size=(n, n))
        A.append(rho * g / np.linalg.norm(g, 2))
    A = np.array(A)
    if unstable:
        q, _ = np.linalg.qr(rng.normal(0.0, 1.0, size=(n, n)))
        A[0] = 1.05 * q
    return A


def discrete_time_terms(A: np.ndarray):
    """A(alpha)^T P A(alpha) - (sum alpha)^2 P < 0 (discrete-time robust stability, both sides
    homogeneous of degree 2) as generalised terms:
        (1/2 A^T(alpha)) P A(alpha) + transpose   and   (-1/2 sum alpha I) P (sum alpha I) + transpose."""
    l, n, _ = A.shape
    half = np.array([0.5 * a.T for a in A])
    neg = np.array([-0.5 * np.eye(n)] * l)
    eye = np.array([np.eye(n)] * l)
    return [(half, 1, A.copy(), 1), (neg, 1, eye, 1)]


def random_terms(n: int, l: int, degs, rng, counts):
    """Random term list with degree pairs ``degs`` [(a, b), ...]; ``counts(d)`` = f(l, d) is passed
    in by the caller (this module enumerates nothing)."""
    return [(rng.normal(0.0, 1.0, size=(counts(a), n, n)), a, rng.normal(0.0, 1.0, size=(counts(b), n, n)), b)
            for a, b in degs]


def bounded_real_terms(A: np.ndarray, Bu: np.ndarray, Cy: np.ndarray, gamma: float):
    """The bounded-real lemma for x' = A(alpha) x + Bu u, y = Cy x (A polytopic with vertices
    A (l, n, n); Bu (n, m), Cy (p, n) constant):
        [[A^T P + P A + Cy^T Cy, P Bu], [Bu^T P, -gamma^2 I]] < 0,  P > 0   <=>  ||G_alpha||_inf < gamma
    as one generalised term (At, 0, Bt, 1) with At = [I; 0] (N x n, N = n + m) and
    Bt(alpha) = [A(alpha), Bu] (n x N, vertex coefficients [A_i, Bu]), plus the constant
    R0 = [[Cy^T Cy, 0], [0, -gamma^2 I]] -- returned as is: the caller homogenises it to the
    degree dp + 1 of the term (each side with its own homogenisation)."""
    l, n, _ = A.shape
    m = Bu.shape[1]
    N = n + m
    At = np.zeros((1, N, n))
    At[0, :n, :n] = np.eye(n)
    Bt = np.array([np.hstack([a, Bu]) for a in A])
    R0 = np.zeros((N, N))
    R0[:n, :n] = Cy.T @ Cy
    R0[n:, n:] = -gamma ** 2 * np.eye(m)
    return [(At, 0, Bt, 1)], R0
