"""GPU parity of the generalised LMI form (polya_setup_general, reading R18)
against the oracle's build_problem_general (pinned in tests/test_oracle_general.py).

Bars as tests/test_gpu_parity.py: B^T(y), B(X) and G within 1e-10 relative error; plus the
continuous-time special case against the standard context, the block / tile shardings, and
discrete-time certificates end to end (polya_ipm_solve + polya_verdict on the device).
"""
import numpy as np
import pytest

import synth
from oracle import ipm as oipm
from oracle import sdp as osdp
from oracle.monomials import enumerate_W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    assert torch.cuda.is_available()
    return pb


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# (n, l, dp, d1, d2, degree pairs): ragged n, several chunks, mixed degrees, d2 = 0, dp = 0
CASES = [(3, 2, 1, 1, 1, [(1, 1), (2, 0)]),
         (9, 2, 1, 1, 1, [(1, 1), (0, 2)]),
         (13, 3, 1, 1, 1, [(1, 0), (0, 1)]),
         (6, 2, 2, 1, 0, [(1, 1)]),
         (5, 1, 0, 2, 2, [(2, 0), (1, 1), (0, 2)]),
         (20, 2, 1, 1, 1, [(1, 1)])]


def _case(n, l, dp, d1, d2, degs, seed=0):
    rng = np.random.default_rng(seed)
    terms = synth.random_terms(n, l, degs, rng, lambda d: len(enumerate_W(l, d)))
    P = osdp.build_problem_general(terms, n, l, dp, d1, d2)
    X, W = synth.spd_blocks(n, P.nblocks, rng)
    return terms, P, X, W


@pytest.mark.parametrize("case", CASES, ids=lambda c: "n{}l{}dp{}d{}{}_{}".format(*c[:5], len(c[5])))
def test_operators_and_schur_parity(pb, case):
    terms, P, X, W = _case(*case)
    n, l, dp, d1, d2, _ = case
    ctx = pb.Polya.general(terms, n, l, dp, d1, d2)
    assert (ctx.K, ctx.M, ctx.nblocks) == (P.K, P.M, P.nblocks)
    rng = np.random.default_rng(7)
    y = rng.normal(size=P.K)
    assert _rel(ctx.apply(_dev(y)).cpu().numpy(), osdp.apply_vmap(P, y)) <= TOL
    R = rng.normal(size=X.shape)
    assert _rel(ctx.adjoint(_dev(R)).cpu().numpy(), osdp.adjoint_trace(P, R)) <= TOL
    Gref = osdp.schur_literal(P, X, W)     # Eq. T2 literally (dense F, traces)
    G = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    assert _rel(G, Gref) <= TOL
    assert np.array_equal(G, G.T)
    ctx.close()


def test_continuous_time_case_equals_standard_context(pb):
    c = synth.small_config(12, 3, 2, 1, 2)
    rng = np.random.default_rng(0)
    A = synth.vertex_matrices(c, rng)
    std = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    gen = pb.Polya.general([(np.array([a.T for a in A]), 1, np.eye(c.n)[None], 0)], c.n, c.l, c.dp, c.d1, c.d2)
    X, W = synth.spd_blocks(c.n, std.nblocks, rng)
    Gs = std.schur(_dev(X), _dev(W)).cpu().numpy()
    Gg = gen.schur(_dev(X), _dev(W)).cpu().numpy()
    assert _rel(Gg, Gs) <= 1e-13
    y = rng.normal(size=std.K)
    assert _rel(gen.apply(_dev(y)).cpu().numpy(), std.apply(_dev(y)).cpu().numpy()) <= 1e-14
    assert std.dims["useful_flops_schur"] == gen.dims["useful_flops_schur"]
    assert std.dims["nnz_H"] == gen.dims["nnz_H"]       # one term per (h, gamma): (H^T, I)
    with pytest.raises(pb.PolyaError):
        gen.H()
    std.close()
    gen.close()


@pytest.mark.parametrize("world", [2, 3])
def test_shardings_partition_G(pb, world):
    terms, P, X, W = _case(13, 3, 1, 1, 1, [(1, 1), (2, 0)], seed=3)
    Xd, Wd = _dev(X), _dev(W)
    ref = pb.Polya.general(terms, 13, 3, 1, 1, 1)
    G = ref.schur(Xd, Wd).cpu().numpy()
    ref.close()
    acc_b = np.zeros_like(G)
    acc_t = np.zeros_like(G)
    for r in range(world):
        cb = pb.Polya.general(terms, 13, 3, 1, 1, 1, rank=r, nranks=world, shard=pb.SHARD_BLOCKS)
        acc_b += cb.schur(Xd, Wd).cpu().numpy()
        cb.close()
        ct = pb.Polya.general(terms, 13, 3, 1, 1, 1, rank=r, nranks=world)
        Gr = ct.schur(Xd, Wd, G=torch.zeros(P.K, P.K, dtype=torch.float64, device="cuda")).cpu().numpy()
        acc_t += Gr
        ct.close()
    assert _rel(acc_b, G) <= 1e-12
    assert _rel(acc_t, G) == 0.0     # tile sharding writes disjoint entries


@pytest.mark.parametrize("unstable", [False, True])
def test_discrete_time_certificates(pb, unstable):
    from paper_1411_3769_b200 import robust
    n, l = 4, 3
    A = synth.discrete_vertex_matrices(n, l, 0.8, np.random.default_rng(3), unstable=unstable)
    terms = synth.discrete_time_terms(A)
    r = robust.certify(None, n, l, 1, 1, 1, terms=terms, samples=300)
    assert r["certified"] == (not unstable), r
    P = osdp.build_problem_general(terms, n, l, 1, 1, 1)
    assert oipm.verdict(P, samples=100) == (not unstable)


def test_verdict_kernel_matches_oracle_grid_check(pb):
    from paper_1411_3769_b200 import robust
    n, l = 3, 2
    A = synth.discrete_vertex_matrices(n, l, 0.7, np.random.default_rng(5))
    terms = synth.discrete_time_terms(A)
    P = osdp.build_problem_general(terms, n, l, 1, 1, 1)
    ok, X, Z, y, it = oipm.solve(P)
    assert ok
    ctx = pb.Polya.general(terms, n, l, 1, 1, 1)
    pts = robust.simplex_points(l, 200, 0)
    assert ctx.verdict(_dev(y), pts) == 0 and oipm.grid_check(P, y, 200, 0)
    bad = y.copy()
    bad[:P.Ntil] *= -1.0
    assert ctx.verdict(_dev(bad), pts) > 0 and not oipm.grid_check(P, bad, 200, 0)
    ctx.close()


@pytest.mark.parametrize("avals,r", [([-1.0], 3.0), ([-1.0, -0.5], 3.0), ([-2.0, -1.0, -4.0], 1.0)])
def test_constant_term_scalar_closed_form(pb, avals, r):
    """R on the device (C on the Lyapunov blocks): polya_ipm_solve reaches the closed-form optimum
    p* = max_i r / (2 |a_i|) of tests/test_oracle_general.py."""
    l = len(avals)
    A = np.array(avals).reshape(l, 1, 1)
    ctx = pb.Polya.general([(A, 1, np.ones((1, 1, 1)), 0)], 1, l, 0, 0, 0, R=np.full((l, 1, 1), r))
    res = ctx.ipm_solve()
    assert res["converged"]
    assert abs(res["y"].cpu().numpy()[0] - max(r / (2 * abs(a)) for a in avals)) <= 1e-6
    ctx.close()


def test_constant_term_ipm_step_parity_and_verdict(pb):
    from paper_1411_3769_b200 import robust
    n, l, dp, d1, d2 = 4, 2, 1, 1, 1
    rng = np.random.default_rng(11)
    A = synth.discrete_vertex_matrices(n, l, 0.6, rng)
    terms = synth.discrete_time_terms(A)
    Wr = enumerate_W(l, dp + 2)
    Q = rng.normal(size=(n, n))
    R = np.array([0.1 * (Q @ Q.T) * (1.0 if sum(w) == w[0] or sum(w) == w[-1] else 2.0) for w in Wr])
    P = osdp.build_problem_general(terms, n, l, dp, d1, d2, R=R)
    ctx = pb.Polya.general(terms, n, l, dp, d1, d2, R=R)
    X, Z, y, mu = oipm.initial_state(P)
    Xd, Zd, yd = (torch.from_numpy(v.copy()).cuda() for v in (X, Z, y))
    mud = mu
    for it in range(3):
        X, Z, y, st = oipm.ipm_step(P, X, Z, y, mu)
        mu = st["mu"]
        s = ctx.ipm_step(Xd, Zd, yd, mud, it)
        mud = s["mu"]
        assert _rel(Xd.cpu().numpy(), X) <= 1e-8, it
        assert _rel(Zd.cpu().numpy(), Z) <= 1e-8, it
        assert _rel(yd.cpu().numpy(), y) <= 1e-8, it
        for k in ("tp", "td", "mu", "phi", "psi"):
            assert abs(s[k] - st[k]) <= 1e-8 * max(1.0, abs(st[k])), (it, k)
    ctx.close()
    ok = oipm.verdict(P, samples=100)
    r = robust.certify(None, n, l, dp, d1, d2, terms=terms, R=R, samples=100)
    assert r["certified"] == ok


def test_discrete_time_terms_merge_to_l_plus_one(pb):
    """The exact merges of polya_setup_general: the identity term (-1/2 sum alpha I, sum alpha I)
    collapses to one term per (h, gamma), so (h, gamma) holds at most l + 1 terms instead of 2 l,
    and the operators still match the (unmerged) oracle."""
    import math
    n, l, dp, d1, d2 = 5, 3, 1, 1, 2
    A = synth.discrete_vertex_matrices(n, l, 0.8, np.random.default_rng(2))
    terms = synth.discrete_time_terms(A)
    ctx = pb.Polya.general(terms, n, l, dp, d1, d2)
    Wp, Wm, W1 = enumerate_W(l, dp), enumerate_W(l, dp + 2 + d2), enumerate_W(l, 1)

    def mnom(d, parts):
        if any(p < 0 for p in parts) or sum(parts) != d:
            return 0
        return math.factorial(d) // math.prod(math.factorial(p) for p in parts)

    want = 0
    for h in Wp:
        for g in Wm:
            w = [[mnom(d2, [gi - hi - li - mi for gi, hi, li, mi in zip(g, h, lam, mu)]) for mu in W1] for lam in W1]
            want += sum(1 for row in w if any(row))     # term 0: one per lambda with a non-zero weight
            want += 1 if sum(map(sum, w)) else 0        # term 1: a single merged term
    assert ctx.dims["nnz_H"] == want
    P = osdp.build_problem_general(terms, n, l, dp, d1, d2)
    rng = np.random.default_rng(3)
    X, W = synth.spd_blocks(n, P.nblocks, rng)
    y = rng.normal(size=P.K)
    assert _rel(ctx.apply(_dev(y)).cpu().numpy(), osdp.apply_vmap(P, y)) <= TOL
    assert _rel(ctx.schur(_dev(X), _dev(W)).cpu().numpy(), osdp.schur_literal(P, X, W)) <= TOL
    ctx.close()


# ---- non-square form (reading R19): N x N blocks, the bounded-real lemma ------------------------------

def _brl(pb, A, Bu, Cy, gamma, dp):
    """Terms and R for the GPU side: R0 homogenised to degree dp + 1 by the library's own
    polya_homogenize (the oracle side uses oracle.polya.homogenize)."""
    terms, R0 = synth.bounded_real_terms(A, Bu, Cy, gamma)
    l = A.shape[0]
    _, R = pb.homogenize({tuple([dp + 1] + [0] * (l - 1)): 0.0 * R0, tuple([0] * l): R0}, l)
    return terms, R


def _brl_oracle(A, Bu, Cy, gamma, dp, d1, d2):
    from oracle import polya as opolya
    terms, R0 = synth.bounded_real_terms(A, Bu, Cy, gamma)
    l, n = A.shape[0], A.shape[1]
    _, R = opolya.homogenize({tuple([dp + 1] + [0] * (l - 1)): 0.0 * R0, tuple([0] * l): R0}, l)
    return osdp.build_problem_general(terms, n, l, dp, d1, d2, R=R)


@pytest.mark.parametrize("n,N,l,dp,d1,d2", [(3, 5, 2, 1, 1, 1), (9, 12, 2, 1, 1, 1), (4, 7, 3, 1, 1, 0)])
def test_non_square_parity(pb, n, N, l, dp, d1, d2):
    rng = np.random.default_rng(21)
    f = lambda d: len(enumerate_W(l, d))
    terms = [(rng.normal(size=(f(1), N, n)), 1, rng.normal(size=(f(1), n, N)), 1),
             (rng.normal(size=(f(2), N, n)), 2, rng.normal(size=(f(0), n, N)), 0)]
    Rr = rng.normal(size=(f(dp + 2), N, N))
    Rr = Rr + Rr.transpose(0, 2, 1)
    P = osdp.build_problem_general(terms, n, l, dp, d1, d2, R=Rr)
    ctx = pb.Polya.general(terms, n, l, dp, d1, d2, R=Rr)
    assert ctx.bn == N and (ctx.K, ctx.nblocks) == (P.K, P.nblocks)
    y = rng.normal(size=P.K)
    assert _rel(ctx.apply(_dev(y)).cpu().numpy(), osdp.apply_vmap(P, y)) <= TOL
    X, W = synth.spd_blocks(N, P.nblocks, rng)
    R = rng.normal(size=X.shape)
    assert _rel(ctx.adjoint(_dev(R)).cpu().numpy(), osdp.adjoint_trace(P, R)) <= TOL
    G = ctx.schur(_dev(X), _dev(W)).cpu().numpy()
    assert _rel(G, osdp.schur_literal(P, X, W)) <= TOL
    ctx.close()


@pytest.mark.parametrize("a,b,c", [(1.0, 1.0, 1.0), (0.5, 1.0, 2.0)])
def test_bounded_real_scalar_closed_form(pb, a, b, c):
    from paper_1411_3769_b200 import robust
    A, Bu, Cy = np.array([[[-a]]]), np.array([[b]]), np.array([[c]])
    g = abs(c * b) / a
    for fac, want in ((1.05, True), (0.95, False)):
        terms, R = _brl(pb, A, Bu, Cy, fac * g, 0)
        r = robust.certify(None, 1, 1, 0, 0, 0, terms=terms, R=R, samples=10)
        assert r["certified"] == want, (fac, r)


def test_bounded_real_polytope_and_ipm_parity(pb):
    from paper_1411_3769_b200 import robust
    from oracle import ipm as oipm
    rng = np.random.default_rng(6)
    c = synth.small_config(2, 2, 1, 1, 1)
    A = synth.vertex_matrices(c, rng)
    Bu, Cy = rng.normal(size=(2, 1)), rng.normal(size=(1, 2))
    w = np.concatenate([[0.0], np.logspace(-3, 3, 2001)])
    hinf = lambda M: max(np.linalg.svd(Cy @ np.linalg.solve(1j * x * np.eye(2) - M, Bu), compute_uv=False)[0] for x in w)
    worst = max(hinf(t * A[0] + (1 - t) * A[1]) for t in np.linspace(0, 1, 11))
    for fac, want in ((1.5, True), (0.97, False)):
        terms, R = _brl(pb, A, Bu, Cy, fac * worst, 1)
        r = robust.certify(None, 2, 2, 1, 1, 1, terms=terms, R=R, samples=50)
        assert r["certified"] == want, (fac, r)
    # three predictor-corrector steps against the oracle's
    terms, R = _brl(pb, A, Bu, Cy, 1.5 * worst, 1)
    P = _brl_oracle(A, Bu, Cy, 1.5 * worst, 1, 1, 1)
    ctx = pb.Polya.general(terms, 2, 2, 1, 1, 1, R=R)
    X, Z, y, mu = oipm.initial_state(P)
    Xd, Zd, yd = (torch.from_numpy(v.copy()).cuda() for v in (X, Z, y))
    mud = mu
    for it in range(3):
        X, Z, y, st = oipm.ipm_step(P, X, Z, y, mu)
        mu = st["mu"]
        s = ctx.ipm_step(Xd, Zd, yd, mud, it)
        mud = s["mu"]
        assert _rel(Xd.cpu().numpy(), X) <= 1e-8 and _rel(Zd.cpu().numpy(), Z) <= 1e-8
        assert _rel(yd.cpu().numpy(), y) <= 1e-8, it
        for k in ("tp", "td", "mu", "phi", "psi"):
            assert abs(s[k] - st[k]) <= 1e-8 * max(1.0, abs(st[k])), (it, k)
    ctx.close()
