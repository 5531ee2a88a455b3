"""Pins for oracle.sdp: basis, V-map, operators and the Schur complement.

Pins: the printed F_k basis elements, SPEC's V-map
examples, two independent routes for B^T and B, the adjoint identity, the P = I
certificate closed form, the K = 1 scalar closed form, the A = 0 Kronecker closed
form, the certificate quadratic form v*^T G v* = sum_b tr(C_b W_b C_b X_b) with
closed-form C_b, symmetry, PSD-ness, and the probe / sampled-entry routes.
"""
import math

import numpy as np
import pytest

import synth
from oracle import sdp
from oracle.monomials import enumerate_W


def mnom(d, parts):
    if any(p < 0 for p in parts) or sum(parts) != d:
        return 0
    return math.factorial(d) // math.prod(math.factorial(p) for p in parts)


def _case(n, l, dp, d1, d2, seed=0, A=None):
    cfg = synth.small_config(n, l, dp, d1, d2)
    rng = np.random.default_rng(seed)
    if A is None:
        A = synth.vertex_matrices(cfg, rng)
    P = sdp.build_problem(A, n, l, dp, d1, d2)
    X, W = synth.spd_blocks(n, P.nblocks, rng)
    return P, X, W


def test_basis_matches_printed_elements():
    for n in (1, 2, 5, 7):
        B = sdp.basis(n)
        assert len(B) == n * (n + 1) // 2
        # Eq. (5): for k > n (1-based) [F_k]_{ij} = 1 iff i = j - 1 = k - n: first super-diagonal
        for k1 in range(n + 1, 2 * n):
            assert B[k1 - 1] == (k1 - n - 1, k1 - n)
        # spanning set of S^n: the E_k are linearly independent
        M = np.array([sdp.E_matrix(n, ab).ravel() for ab in B])
        assert np.linalg.matrix_rank(M) == len(B)


def test_vmap_spec_examples():
    P, _, _ = _case(2, 2, 1, 1, 1)
    e1 = np.zeros(P.K); e1[0] = 1
    assert np.array_equal(sdp.vmap(P, e1, 0), np.diag([1.0, 0.0]))
    e = np.zeros(P.K); e[P.Ntil] = 1
    assert np.array_equal(sdp.vmap(P, e, 1), np.diag([1.0, 0.0]))
    x = np.arange(1.0, P.K + 1)
    V = sdp.vmap(P, x, 0)
    assert np.array_equal(V, [[1.0, 3.0], [3.0, 2.0]])                   # S:273 (reading R2)


@pytest.mark.parametrize("shape", [(3, 2, 1, 1, 1), (4, 3, 2, 1, 2), (2, 3, 2, 2, 2)])
def test_operator_routes_and_adjoint_identity(shape):
    P, X, W = _case(*shape)
    rng = np.random.default_rng(5)
    y = rng.normal(size=P.K)
    T1 = sdp.apply_literal(P, y)
    T2 = sdp.apply_vmap(P, y)
    assert np.linalg.norm(T1 - T2) <= 1e-13 * np.linalg.norm(T1)
    assert np.allclose(T1, T1.transpose(0, 2, 1), atol=1e-14 * np.abs(T1).max())
    y1 = sdp.adjoint_literal(P, X)
    y2 = sdp.adjoint_trace(P, X)
    assert np.linalg.norm(y1 - y2) <= 1e-13 * np.linalg.norm(y1)
    # <B^T(y), X> = y^T B(X)
    lhs = sum(np.sum(T1[b] * X[b]) for b in range(P.nblocks))
    assert abs(lhs - y @ y1) <= 1e-12 * abs(lhs)


def certificate(P):
    """y* with P_h = multinomial(dp; h) I, i.e. P(alpha) = (sum alpha)^dp I, and the closed-form
    blocks of B^T(y*): multinomial(dp+d1; g) I on P-blocks and
    -sum_i multinomial(dp+d2; g - e_i)(A_i + A_i^T) on Lyapunov blocks."""
    Wp = enumerate_W(P.l, P.dp)
    y = np.zeros(P.K)
    for h, hexp in enumerate(Wp):
        for k in range(P.n):            # diagonal basis elements come first (R2)
            y[k + P.Ntil * h] = mnom(P.dp, hexp)
    blocks = np.zeros((P.nblocks, P.n, P.n))
    for j, g in enumerate(enumerate_W(P.l, P.dp + P.d1)):
        blocks[j] = mnom(P.dp + P.d1, g) * np.eye(P.n)
    for m, g in enumerate(enumerate_W(P.l, P.dp + 1 + P.d2)):
        for i in range(P.l):
            parts = [g[t] - (1 if t == i else 0) for t in range(P.l)]
            blocks[P.L + m] -= mnom(P.dp + P.d2, parts) * (P.A[i] + P.A[i].T)
    return y, blocks


@pytest.mark.parametrize("cfg", [1, 2])
def test_certificate_closed_form(cfg):
    c = synth.CONFIGS[cfg]
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    P = sdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    y, want = certificate(P)
    got = sdp.apply_vmap(P, y)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    # stable configs: B^T(y*) - C is blockwise PD (SURVEY 8(c) verdict pins)
    Z = got.copy()
    for j in range(P.L):
        Z[j] -= P.c[j] * np.eye(P.n)
    assert min(np.linalg.eigvalsh(z).min() for z in Z) > 0


def test_scalar_closed_form():
    # n = 1, l = 1, dp = 0: K = 1, one P-block (beta = 1) and one Lyapunov block (H = A):
    # G = X_0 W_0 + 4 A^2 X_1 W_1   ("K=1 ... Lambda = B1^2 X/Z")
    A = np.array([[[-0.7]]])
    P = sdp.build_problem(A, 1, 1, 0, 2, 3)
    assert (P.K, P.L, P.M) == (1, 1, 1)
    X = np.array([[[1.3]], [[0.4]]])
    W = np.array([[[0.8]], [[2.5]]])
    G = sdp.schur_literal(P, X, W)
    assert abs(G[0, 0] - (1.3 * 0.8 + 4 * 0.49 * 0.4 * 2.5)) < 1e-15


def test_A_zero_kronecker_closed_form():
    # A = 0 -> H = 0 -> only P-blocks; with X_j = W_j = I: tr(E_s E_t) = [s=t] (1 diag, 2 off-diag),
    # so G = (sum_j beta_j beta_j^T) (x) diag(d_k)
    n, l, dp, d1, d2 = 3, 3, 2, 1, 1
    P = sdp.build_problem(np.zeros((l, n, n)), n, l, dp, d1, d2)
    I = np.broadcast_to(np.eye(n), (P.nblocks, n, n)).copy()
    G = sdp.schur_literal(P, I, I)
    dk = np.array([1.0 if a == b else 2.0 for a, b in P.E])
    want = np.kron(P.beta @ P.beta.T, np.diag(dk))
    assert np.array_equal(G, want)


@pytest.mark.parametrize("shape", [(3, 2, 1, 1, 1), (4, 3, 2, 1, 2), (5, 2, 2, 2, 1)])
def test_schur_invariants(shape):
    P, X, W = _case(*shape, seed=3)
    G = sdp.schur_literal(P, X, W)
    # symmetry and PSD
    assert np.abs(G - G.T).max() <= 1e-13 * np.abs(G).max()
    ev = np.linalg.eigvalsh(0.5 * (G + G.T))
    assert ev.min() >= -1e-12 * ev.max()
    # certificate quadratic form with closed-form F_{v*} blocks
    v, C = certificate(P)
    want = sum(np.trace(C[b] @ W[b] @ C[b] @ X[b]) for b in range(P.nblocks))
    assert abs(v @ G @ v - want) <= 1e-12 * abs(want)
    # probe route  G v = B(W B^T(v) X)
    rng = np.random.default_rng(9)
    for _ in range(3):
        u = rng.normal(size=P.K)
        assert np.linalg.norm(G @ u - sdp.schur_probe(P, X, W, u)) <= 1e-12 * np.linalg.norm(G @ u)
    U = rng.normal(size=(3, P.K))      # a batch of probes
    assert np.abs(sdp.schur_probe(P, X, W, U) - U @ G.T).max() <= 1e-12 * np.abs(U @ G.T).max()
    # sampled-entry route and row restriction
    pairs = [(int(i), int(j)) for i, j in rng.integers(0, P.K, size=(20, 2))]
    ent = sdp.schur_entries(P, X, W, pairs)
    assert np.allclose(ent, [G[i, j] for i, j in pairs], rtol=1e-12, atol=1e-13 * np.abs(G).max())
    rows = [0, P.K // 2, P.K - 1]
    assert np.array_equal(sdp.schur_literal(P, X, W, rows=rows), G[rows])
    # whole-row route (row k = B(X F_k W), PAPER.md:318-324 applied to Eq. T2 by cyclicity)
    rows2 = [int(i) for i in rng.integers(0, P.K, size=7)] + [P.K - 1]
    Gr = sdp.schur_rows(P, X, W, rows2, chunk=3)
    assert np.abs(Gr - G[rows2]).max() <= 1e-12 * np.abs(G).max()
    # batched dense F equals the one-at-a-time Eq. (31)
    for b in (0, P.L - 1, P.L, P.nblocks - 1):
        want = np.array([sdp.F_block(P, i, b) for i in rows2])
        assert np.array_equal(sdp.F_stack(P, b, rows2), want) or np.abs(sdp.F_stack(P, b, rows2) - want).max() <= 1e-15


def test_config1_unstable_copy_no_certificate():
    # Theorem 1 necessity: A_2 + 3I has an eigenvalue with positive real part,
    # so the P = I certificate must fail: some Lyapunov block of B^T(y*) is not negative semidefinite.
    c = synth.CONFIGS["1u"]
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    assert np.linalg.eigvals(A[1]).real.max() > 0
    P = sdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    y, _ = certificate(P)
    T = sdp.apply_vmap(P, y)
    assert max(np.linalg.eigvalsh(-T[P.L + m]).max() for m in range(P.M)) > 0 or \
        min(np.linalg.eigvalsh(T[P.L + m]).min() for m in range(P.M)) < 0


@pytest.mark.parametrize("key", [1, "1u", 2, "n5_l1", "n9", "n12", "ex2"])
def test_schur_structured_equals_literal(key):
    """oracle.sdp.schur_structured (the rank-structured route of SURVEY O6'(iii), derived from the
    trace) reproduces the literal Eq. T2 (schur_literal) -- a different computation of the same
    definition -- including ragged n, l = 1 / d_p = 0, and d_a = 3 (Example 2's A)."""
    import synth
    from oracle import polya
    rng = np.random.default_rng(3)
    if key == "ex2":
        from test_oracle_examples import example2_A
        P = sdp.build_problem(example2_A(0.1), 3, 3, 1, 1, 1, da=3)
    else:
        c = {"n5_l1": synth.small_config(5, 1, 0, 2, 3), "n9": synth.small_config(9, 2, 1, 2, 1),
             "n12": synth.small_config(12, 3, 2, 1, 2)}.get(key) or synth.CONFIGS[key]
        A = synth.vertex_matrices(c, rng)
        P = sdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    X, W = synth.spd_blocks(P.n, P.nblocks, rng)
    G1 = sdp.schur_literal(P, X, W)
    G2 = sdp.schur_structured(P, X, W)
    assert np.abs(G1 - G2).max() <= 1e-12 * np.abs(G1).max()
    # a subset of pairs fills exactly those tiles
    G3 = sdp.schur_structured(P, X, W, pairs=[(0, P.L0 - 1)])
    N = P.Ntil
    assert np.array_equal(G3[:N, (P.L0 - 1) * N:], G2[:N, (P.L0 - 1) * N:])
