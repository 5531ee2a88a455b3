"""GPU tests of the full method beyond one iteration: Algorithm 2
to its stopping rule (polya_ipm_solve), the certificate's grid check on the device
(polya_verdict), and bisection on the paper's Example 2.

Bars: the verdicts (certified or not) equal the oracle's on the same problems (reading R15: the
certificate itself is not unique, the verdict is); a bisection whose every verdict agrees returns
the oracle's bound exactly; every certified bound lies above the brute-force stability boundary
(-0.1115, see tests/test_oracle_examples.py: Theorem 1 makes a certificate impossible below it)
and tightens as (d_p, d1, d2) grow."""
import numpy as np
import pytest

import synth
from oracle import ipm as oipm
from oracle import polya as opolya
from oracle import sdp as osdp

from test_oracle_examples import example2_A

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BOUNDARY = -0.1115   # brute-force stability boundary of Example 2 (stable at -0.1115, unstable at -0.112)


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    assert torch.cuda.is_available()
    return pb


@pytest.mark.parametrize("key,stable", [(1, True), ("1u", False), (2, True)])
def test_solve_and_verdict_on_constructed_systems(pb, key, stable):
    from paper_1411_3769_b200 import robust
    c = synth.CONFIGS[key]
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    r = robust.certify(A, c.n, c.l, c.dp, c.d1, c.d2, samples=300)
    assert r["certified"] == stable, r
    if stable:
        assert r["gap"] <= 1e-8 and r["pinf"] <= 1e-8 and r["nfail"] == 0


@pytest.mark.parametrize("case", ["scalar", "1u", "discrete"])
def test_infeasible_exit_status_matches_oracle(pb, case):
    """Reading R20: polya_ipm_solve stops an infeasible LMI with status EDIVERGED at the same
    iteration as the oracle's divergence exit (the GPU steps match the oracle's to rounding)."""
    if case == "scalar":
        A = np.array([[[1.0]], [[-1.0]]])
        P = osdp.build_problem(A, 1, 2, 1, 1, 1)
        ctx = pb.Polya(1, 2, 1, 1, 1, A)
    elif case == "1u":
        c = synth.CONFIGS["1u"]
        A = synth.vertex_matrices(c, np.random.default_rng(0))
        P = osdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
        ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    else:
        A = synth.discrete_vertex_matrices(4, 3, 0.8, np.random.default_rng(3), unstable=True)
        terms = synth.discrete_time_terms(A)
        P = osdp.build_problem_general(terms, 4, 3, 1, 1, 1)
        ctx = pb.Polya.general(terms, 4, 3, 1, 1, 1)
    info = {}
    ok, _, _, _, it = oipm.solve(P, info=info)
    assert not ok and info["status"] == "diverged"
    r = ctx.ipm_solve()
    assert not r["converged"] and r["status"] == pb.EDIVERGED, r
    assert r["iterations"] == it
    ctx.close()


def test_solve_matches_oracle_solution_config1(pb):
    """Same stopping iteration and the same certificate y to 1e-6 on config 1 (the GPU steps match
    the oracle's to ~1e-15 each, tests/test_gpu_ipm.py)."""
    c = synth.CONFIGS[1]
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    P = osdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    ok, X, Z, y, it = oipm.solve(P)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    r = ctx.ipm_solve()
    assert bool(r["converged"]) == ok and r["iterations"] == it
    hist = r["history"]                       # per-iteration log
    assert len(hist) == it and hist[-1]["gap"] == r["gap"] and hist[-1]["gap"] <= 1e-8 < hist[0]["gap"]
    yg = r["y"].cpu().numpy()
    assert np.linalg.norm(yg - y) <= 1e-6 * np.linalg.norm(y)
    ctx.close()


def test_verdict_kernel_matches_oracle_grid_check(pb):
    """polya_verdict on a converged certificate and on a perturbed (invalid) one, vs oracle.grid_check."""
    from paper_1411_3769_b200 import robust
    P = osdp.build_problem(example2_A(0.4), 3, 3, 1, 1, 1, da=3)
    ok, X, Z, y, it = oipm.solve(P)
    assert ok
    ctx = pb.Polya(3, 3, 1, 1, 1, example2_A(0.4), da=3)
    pts = robust.simplex_points(3, 300, 0)
    yd = torch.from_numpy(y).cuda()
    assert ctx.verdict(yd, pts) == 0 and oipm.grid_check(P, y, 300, 0)
    bad = y.copy()
    bad[:6] *= -1.0                         # P_0 -> -P_0: not positive at the first vertex
    assert ctx.verdict(torch.from_numpy(bad).cuda(), pts) > 0 and not oipm.grid_check(P, bad, 300, 0)
    ctx.close()


@pytest.mark.parametrize("L,deg,certified", [(0.4, (1, 1, 1), True), (0.1, (1, 2, 2), True),
                                               (0.0, (1, 1, 1), False), (-0.2, (2, 2, 2), False)])
def test_example2_verdicts_match_oracle(pb, L, deg, certified):
    from paper_1411_3769_b200 import robust
    r = robust.certify(example2_A(L), 3, 3, *deg, da=3, samples=300)
    assert r["certified"] == certified == oipm.verdict(osdp.build_problem(example2_A(L), 3, 3, *deg, da=3), samples=300)


def test_example2_bisection_equals_oracle(pb):
    from paper_1411_3769_b200 import robust
    deg = (1, 2, 2)

    def gpu(L):
        Ap = robust_A(pb, L)
        return robust.certify(Ap, 3, 3, *deg, da=3, samples=300)["certified"]

    def cpu(L):
        return oipm.verdict(osdp.build_problem(example2_A(L), 3, 3, *deg, da=3), samples=300)

    hg, lg, tg = robust.bisect(gpu, -0.2, 0.4, steps=8)
    hc, lc, tc = robust.bisect(cpu, -0.2, 0.4, steps=8)
    assert tg == tc and hg == hc
    assert BOUNDARY < hg < 0.4


def robust_A(pb, L):
    """Example 2's A(g(alpha)) through the library's own set-up (polya_homogenize + polya_simplex_map)."""
    from test_oracle_examples import example2_terms
    da, A = pb.homogenize(example2_terms(), 3)
    return pb.simplex_map(A, 3, da, [1 - L] * 3, [L] * 3)


def test_example2_bounds_tighten_with_degree(pb):
    """Upper bounds on L_opt = -0.111 from bisection at growing (d_p, d1 = d2): never below
    the stability boundary (Theorem 1) and non-increasing in the degrees."""
    from paper_1411_3769_b200 import robust
    bounds = []
    for deg in [(1, 1, 1), (2, 2, 2), (2, 4, 4), (3, 6, 6)]:
        hi, lo, _ = robust.bisect(lambda L: robust.certify(robust_A(pb, L), 3, 3, *deg, da=3, samples=300)["certified"],
                                  -0.2, 0.6, steps=9)
        bounds.append(hi)
    assert all(b > BOUNDARY for b in bounds)
    assert all(bounds[i + 1] <= bounds[i] + 1e-12 for i in range(len(bounds) - 1)), bounds
    assert bounds[-1] < bounds[0]


def test_verdict_beyond_118_states(pb):
    """polya_verdict at n = 130 (> the former 118 shared-memory limit; config 5 has n = 120): the
    P = I certificate y* (P_h = multinomial(dp; h) I) of a system with A_i + A_i^T < 0 passes at every
    point, -y* fails at every point; the oracle's grid check agrees."""
    import math
    from paper_1411_3769_b200 import robust
    c = synth.small_config(130, 2, 1, 1, 1)
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    P = osdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
    ystar = np.zeros(P.K)
    from oracle.monomials import enumerate_W
    for h, e in enumerate(enumerate_W(c.l, c.dp)):
        ystar[h * P.Ntil:h * P.Ntil + c.n] = math.factorial(c.dp) / math.prod(math.factorial(k) for k in e)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    pts = robust.simplex_points(c.l, 12, 0)
    assert ctx.verdict(torch.from_numpy(ystar).cuda(), pts) == 0
    assert oipm.grid_check(P, ystar, 12, 0)
    assert ctx.verdict(torch.from_numpy(-ystar).cuda(), pts) == len(pts)
    assert not oipm.grid_check(P, -ystar, 12, 0)
    ctx.close()


@pytest.mark.parametrize("stable", [True, False], ids=["stable", "unstable"])
def test_solve_at_max_block_order(pb, stable):
    """Block order n = 168, the IPM's shared-memory limit (k_block_inv / k_block_lmin at their largest
    layouts, K4 with 21 index chunks, K = 28,392): a stable polytope (config-2 recipe) is certified and
    the oracle's grid check accepts the GPU's certificate; with a vertex shifted by +3I (unstable) it is
    not certified (Theorem 1 rules a certificate out)."""
    from paper_1411_3769_b200 import robust
    c = synth.small_config(168, 2, 1, 1, 1)
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    if not stable:
        A[1] = A[1] + 3.0 * np.eye(c.n)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    r = ctx.ipm_solve()
    if stable:
        assert r["converged"] and r["gap"] <= 1e-8 and r["pinf"] <= 1e-8, {k: r[k] for k in ("status", "gap", "pinf")}
        assert ctx.verdict(r["y"], robust.simplex_points(c.l, 50, 0)) == 0
        P = osdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)
        assert oipm.grid_check(P, r["y"].cpu().numpy(), 50, 0)
    else:
        assert not r["converged"]
    ctx.close()
    torch.cuda.empty_cache()
