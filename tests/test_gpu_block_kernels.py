"""GPU parity of the IPM's blockwise kernels (row a10) through the test hook
polya_block_kernels_test, at block orders from 1 to the limit n = 168 (odd, even, multiples of 32
and their neighbours, the shared-memory limit):

* W = S^{-1} (k_block_inv; Algorithm 2's Z^{-1}) against the oracle's inverse
  (oracle.ipm.ipm_step: W = sym(inv(Z))), within 64 eps kappa(S) relative Frobenius error;
* the step length of reading R5 (k_block_inv's L^{-1} mode, two block GEMMs, k_block_lmin: Householder
  tridiagonalisation + Sturm multisection) against oracle.ipm.step_length block by block (eigenvalues
  by LAPACK), within 1e-10 relative, plus its closed form for diagonal blocks;
* the degenerate cases: dS >= 0 (no bound: t = 1/0.98 before the cap), S not positive definite (the
  fail flag, t = -1 for that block only), n = 1 and 2 (no Householder step).
"""
import numpy as np
import pytest

import synth
from oracle import ipm as oipm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TCAP = 1.0 / 0.98


@pytest.fixture(scope="module")
def pb():
    import paper_1411_3769_b200 as pb
    pb.lib()
    return pb


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _sym_indefinite(n, nb, rng):
    D = rng.normal(size=(nb, n, n))
    return 0.5 * (D + np.transpose(D, (0, 2, 1)))


def _run(pb, S, dS):
    Sd = torch.from_numpy(np.ascontiguousarray(S)).cuda()
    dSd = torch.from_numpy(np.ascontiguousarray(dS)).cuda()
    W, Li, M, t, fail = pb.block_kernels_test(Sd, dSd)
    return W.cpu().numpy(), Li.cpu().numpy(), M.cpu().numpy(), t.cpu().numpy(), fail


@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 32, 33, 64, 100, 127, 128, 167, 168])
def test_inverse_and_step_length_vs_oracle(pb, n):
    rng = np.random.default_rng(1000 + n)
    nb = 3
    S, _ = synth.spd_blocks(n, nb, rng)
    dS = _sym_indefinite(n, nb, rng)
    W, Li, M, t, fail = _run(pb, S, dS)
    assert fail == 0
    for b in range(nb):
        kappa = np.linalg.cond(S[b])
        Wo = np.linalg.inv(S[b])
        Wo = 0.5 * (Wo + Wo.T)                       # the oracle's W (oracle.ipm.ipm_step)
        assert _rel(W[b], Wo) <= max(64 * np.finfo(float).eps * kappa, 1e-14), (n, b, kappa)
        assert np.array_equal(W[b], W[b].T)          # exactly symmetric
        Lo = np.linalg.inv(np.linalg.cholesky(S[b]))
        assert _rel(Li[b], Lo) <= max(64 * np.finfo(float).eps * np.sqrt(kappa) * n, 1e-14)
        assert np.all(np.triu(Li[b], 1) == 0.0)
        to = oipm.step_length(S[b:b + 1], dS[b:b + 1])
        tg = min(1.0, 0.98 * t[b])
        assert abs(tg - to) <= 1e-10 * to, (n, b, tg, to)


@pytest.mark.parametrize("n", [1, 2, 7, 100, 168])
def test_step_length_closed_form_diagonal(pb, n):
    """S = I, dS = diag(d): t = min(1, 0.98 min_i 1 / (-d_i)) over the negative d_i (reading R5's closed
    form, the same one that pins oracle.ipm.step_length); dS >= 0 gives the uncapped 1/0.98."""
    rng = np.random.default_rng(7 + n)
    S = np.stack([np.eye(n)] * 2)
    d_neg = rng.uniform(-3.0, 1.0, size=n)
    d_neg[rng.integers(n)] = -2.5                   # at least one negative entry
    d_pos = rng.uniform(0.0, 1.0, size=n)
    dS = np.stack([np.diag(d_neg), np.diag(d_pos)])
    _, _, _, t, fail = _run(pb, S, dS)
    assert fail == 0
    expect = min(1.0, 0.98 / -d_neg.min())
    assert abs(min(1.0, 0.98 * t[0]) - expect) <= 1e-13 * expect
    assert t[1] == TCAP


@pytest.mark.parametrize("n", [3, 100, 168])
def test_not_positive_definite_block(pb, n):
    """A block with an indefinite S: the fail flag is raised, its t is -1 (step_len's bisection
    fallback), the other blocks are unaffected."""
    rng = np.random.default_rng(55 + n)
    S, _ = synth.spd_blocks(n, 3, rng)
    S[1] = S[1] - 2.0 * np.linalg.eigvalsh(S[1]).max() * np.eye(n)   # negative definite
    dS = _sym_indefinite(n, 3, rng)
    W, _, _, t, fail = _run(pb, S, dS)
    assert fail == 1
    assert t[1] == -1.0
    for b in (0, 2):
        to = oipm.step_length(S[b:b + 1], dS[b:b + 1])
        assert abs(min(1.0, 0.98 * t[b]) - to) <= 1e-10 * to


def test_hook_rejects_out_of_range(pb):
    S = torch.zeros((1, 169, 169), dtype=torch.float64, device="cuda")
    with pytest.raises(pb.PolyaError):
        pb.block_kernels_test(S, S)
