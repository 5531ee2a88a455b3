"""GPU parity of polya_ipm_step (row a10: Algorithm 2, readings R3-R6) against
oracle.ipm on the same seeded inputs, plus verdicts of the full iteration driven from Python.

Tolerance: iterates X, Z, y within 1e-8 relative Frobenius error after each of the first
iterations (the IPM's certificate is not unique, so only a few steps are
compared; the step lengths come from eigenvalues in the oracle and from bisection on the
Cholesky test on the GPU, equal to ~1e-15 relative).
"""
import numpy as np
import pytest

import synth
from oracle import ipm as oipm
from oracle import sdp as osdp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    return pb


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _case(key):
    c = synth.CONFIGS[key] if not isinstance(key, synth.Config) else key
    A = synth.vertex_matrices(c, np.random.default_rng(0))
    return c, A, osdp.build_problem(A, c.n, c.l, c.dp, c.d1, c.d2)


@pytest.mark.parametrize("key", [1, "1u", 2, synth.small_config(9, 2, 1, 2, 1)],
                         ids=lambda k: str(k) if not isinstance(k, synth.Config) else k.name)
def test_ipm_step_parity(pb, key):
    c, A, P = _case(key)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
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
            assert abs(s[k] - st[k]) <= 1e-8 * max(1.0, abs(st[k])), (it, k, s[k], st[k])
        assert s["ms_schur"] >= 0 and s["ms_factor"] >= 0
    ctx.close()


def _drive(ctx, P, iters=60, eps=1e-8):
    X, Z, y, mu = oipm.initial_state(P)
    Xd, Zd, yd = (torch.from_numpy(v.copy()).cuda() for v in (X, Z, y))
    for it in range(iters):
        try:
            s = ctx.ipm_step(Xd, Zd, yd, mu, it)
        except Exception:
            return False, yd.cpu().numpy()
        mu = s["mu"]
        pinf = np.linalg.norm(ctx.adjoint(Xd).cpu().numpy() - 1.0)
        if s["gap"] <= eps and pinf <= 1e-8:
            ok = all(np.linalg.eigvalsh(z).min() > 0 for z in Zd.cpu().numpy())
            return ok, yd.cpu().numpy()
    return False, yd.cpu().numpy()


@pytest.mark.parametrize("key,stable", [(1, True), ("1u", False)])
def test_ipm_verdicts(pb, key, stable):
    c, A, P = _case(key)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    ok, y = _drive(ctx, P)
    assert (ok and oipm.grid_check(P, y)) == stable
    ctx.close()


def test_ipm_step_config3_runs(pb):
    """One step at config 3 (K = 4,650, 140 blocks of 30x30): status ok, finite, G factorised."""
    c, A, P = _case(3)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    X, Z, y, mu = oipm.initial_state(P)
    Xd, Zd, yd = (torch.from_numpy(v.copy()).cuda() for v in (X, Z, y))
    s = ctx.ipm_step(Xd, Zd, yd, mu, 0)
    assert np.isfinite([s["gap"], s["mu"], s["tp"], s["td"]]).all()
    assert 0 < s["tp"] <= 1 and 0 < s["td"] <= 1
    # primal feasibility of the predictor is inherited after a full step: B(X) -> 1 when tp = 1
    if s["tp"] == 1.0:
        assert np.linalg.norm(ctx.adjoint(Xd).cpu().numpy() - 1.0) <= 1e-6 * np.sqrt(P.K)
    ctx.close()


@pytest.mark.parametrize("key", [2, 3, synth.small_config(9, 2, 1, 2, 1)],
                         ids=lambda k: str(k) if not isinstance(k, synth.Config) else k.name)
def test_tiled_factorisation_matches_dense(pb, key):
    """polya_set_factorization(2): G as pair tiles + blocked Cholesky / solves (the path config 5
    needs) gives the same iterates as the dense K x K dpotrf path, to 1e-10."""
    c, A, P = _case(key)
    X, Z, y, mu = oipm.initial_state(P)
    runs = []
    for mode in (1, 2):
        ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
        ctx.set_factorization(mode)
        Xd, Zd, yd = (torch.from_numpy(v.copy()).cuda() for v in (X, Z, y))
        m = mu
        for it in range(3):
            m = ctx.ipm_step(Xd, Zd, yd, m, it)["mu"]
        runs.append((Xd.cpu().numpy(), Zd.cpu().numpy(), yd.cpu().numpy()))
        ctx.close()
    for a, b in zip(runs[0], runs[1]):
        assert _rel(b, a) <= 1e-10


@pytest.mark.parametrize("mode", [1, 2])
def test_factorisation_regularised_retry(pb, mode):
    """A singular Schur complement (X = 0 except on P-block 0, so only the dual rows of h with
    beta_{h,0} != 0 are excited) fails the first Cholesky; the step re-assembles G, retries once on
    G + 1e-12 tr(G)/K I and completes (reg_retries = 1).  A regular state needs no retry.
    With X = 0 everywhere tr(G) = 0 and the retry cannot help: ENOTPD naming the retry."""
    c, A, P = _case(2)
    ctx = pb.Polya(c.n, c.l, c.dp, c.d1, c.d2, A)
    ctx.set_factorization(mode)
    Z = torch.eye(c.n, dtype=torch.float64, device="cuda").repeat(P.nblocks, 1, 1).contiguous()
    y = torch.zeros(P.K, dtype=torch.float64, device="cuda")
    assert ctx.ipm_step(Z.clone(), Z.clone(), y.clone(), 1.0 / 3.0, 0)["reg_retries"] == 0
    X = torch.zeros_like(Z)
    X[0] = torch.eye(c.n, dtype=torch.float64)
    assert ctx.ipm_step(X, Z.clone(), y.clone(), 1.0 / 3.0, 0)["reg_retries"] == 1
    with pytest.raises(pb.PolyaError) as e2:
        ctx.ipm_step(torch.zeros_like(Z), Z.clone(), y.clone(), 1.0 / 3.0, 0)
    assert "regularised retry" in str(e2.value), str(e2.value)
    ctx.close()
