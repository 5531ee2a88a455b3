"""SDP elements, operators and the Schur complement, literally.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md Sec. III.B "SDP Problem Elements" and Algorithm 2:
* basis E_k of S^n (Eqs. 4-5) under reading R2:
  k < n -> (k,k); then offsets o = 1..n-1, rows i = 0..n-1-o -> (i, i+o);
  E = e_a e_b^T + e_b e_a^T (unnormalised) off the diagonal.  The printed formula
  defines exactly the first n-1 of these off-diagonal elements (the first
  super-diagonal) and the paper notes "any other basis could be used";
* V_<h>(x) = sum_j E_j x_{j + Ntil(<h>-1)} (Eq. 30);
* blocks B_{i,j} (Eq. 31): P-blocks j < L: sum_h beta_{h,j} V_h(e_i);
  Lyapunov blocks L+m: -sum_h (H_{h,m}^T V_h(e_i) + V_h(e_i) H_{h,m});
* B(X) = [tr(B_1 X) ... tr(B_K X)]^T,
  B^T(y) = sum_i y_i B_i (Eq. AT);
* lambda_{k,l} = sum_blocks tr(B_k Z^{-1} B_l X) (Eq. T2).
* the generalised form sum_i (At_i P Bt_i + Bt_i^T P At_i^T) < 0 (reading R18):
  build_problem_general; Lyapunov block m of the element (h, k) is -sum_q (A_q E_k B_q + B_q^T E_k A_q^T).

Block order: P-blocks 0..L-1 in W_{dp+d1} order, then Lyapunov blocks in
W_{dp+da+d2} order.  Dual index i = k + Ntil*h (0-based).
"""
from __future__ import annotations

import dataclasses
import functools

import numpy as np

from . import polya
from .monomials import enumerate_W

__all__ = ["basis", "trE", "Problem", "build_problem", "vmap", "F_block", "F_stack",
           "apply_literal", "apply_vmap", "adjoint_literal", "adjoint_trace",
           "schur_literal", "schur_rows", "schur_entries", "schur_probe", "schur_structured", "schur_structured_tile",
           "build_problem_general"]


def basis(n: int):
    """[(a, b)] for k = 0..Ntil-1 (reading R2, diagonal-major)."""
    out = [(k, k) for k in range(n)]
    for o in range(1, n):
        for i in range(n - o):
            out.append((i, i + o))
    return out


def E_matrix(n: int, ab):
    a, b = ab
    E = np.zeros((n, n))
    E[a, b] = 1.0
    E[b, a] = 1.0
    return E


def trE(ab, M):
    """tr(E_k M): M[a,a] on the diagonal, M[a,b] + M[b,a] off it."""
    a, b = ab
    return M[a, a] if a == b else M[a, b] + M[b, a]


@dataclasses.dataclass
class Problem:
    n: int
    l: int
    dp: int
    da: int
    d1: int
    d2: int
    delta: float
    L0: int
    L: int
    M: int
    Ntil: int
    K: int
    beta: np.ndarray          # (L0, L) int64
    H: np.ndarray             # (L0, M, n, n)
    c: np.ndarray             # (L,)
    A: np.ndarray
    E: list
    gen: list = None          # generalised form: gen[h][m] = [(A_q, B_q), ...] (build_problem_general)
    pairs: list = None        # its (Atil_i, deg_a, Btil_i, deg_b) terms
    R: np.ndarray = None      # its constant term R(alpha), coefficients in W_{dp+e} order (or None)
    CL: np.ndarray = None     # C on the Lyapunov blocks: coefficients of (sum alpha)^{d2} R(alpha)
    N: int = None             # block order (generalised form with N x n At_i: N > n, reading R19); None: n

    @property
    def bn(self):
        """Order of every block of X, Z, C and B^T(y): n, or N for the non-square generalised form."""
        return self.n if self.N is None else self.N

    def embed(self, M):
        """An n x n P-block quantity as the top-left corner of a bn x bn block (reading R19)."""
        if self.bn == self.n:
            return M
        out = np.zeros((self.bn, self.bn))
        out[:self.n, :self.n] = M
        return out

    @property
    def nblocks(self):
        return self.L + self.M

    def active(self, h: int, b: int) -> bool:
        """Whether F^b_{(h,.)} is structurally non-zero."""
        if b < self.L:
            return self.beta[h, b] != 0
        if self.gen is not None:
            return len(self.gen[h][b - self.L]) > 0
        return bool(np.any(self.H[h, b - self.L] != 0))


def build_problem(A, n, l, dp, d1, d2, da=1, delta=1e-3) -> Problem:
    """Algorithm 1's outputs in dense form: beta, H, C (and K)."""
    beta = polya.beta_table(l, dp, d1)
    H = polya.H_table(A, l, dp, d2, da)
    L0, L = beta.shape
    M = H.shape[1]
    Ntil = n * (n + 1) // 2
    c = polya.C_scalars(beta, l, dp, delta)
    return Problem(n, l, dp, da, d1, d2, delta, L0, L, M, Ntil, L0 * Ntil, beta, H, c, A, basis(n))


def build_problem_general(pairs, n, l, dp, d1, d2, delta=1e-3, R=None) -> Problem:
    """(Non-square: At_i coefficients N x n, Bt_i n x N, R N x N with N > n -- the bounded-real-lemma
    shape -- make every block N x N, the P-blocks' n x n LMI sitting in the top-left corner with C
    = -I on the rest, so that their slack Z is I there; reading R19.)"""
    """The generalised LMI form of PAPER.md:454-459, square case:
        P(alpha) > 0,   sum_i (At_i(alpha) P(alpha) Bt_i(alpha) + Bt_i(alpha)^T P(alpha) At_i(alpha)^T) + R(alpha) < 0,
    with pairs = [(At_i coefficients [f(l,a_i)][n][n] in W_{a_i} order, a_i, Bt_i coefficients, b_i)],
    all with the same total degree e = a_i + b_i.  Polya's multiplier (sum alpha)^{d2} turns the
    second condition into M = |W_{dp+e+d2}| coefficient blocks (as Eqs. LMI_2/LMI_4 do for A^T P + P A),
    found here by explicit polynomial multiplication: the coefficient of alpha^gamma in
    (sum alpha)^{d2} alpha^h At_i(alpha) (.) Bt_i(alpha) is the list of pairs
    (multinomial(d2; gamma - h - lambda - mu) At_{i,lambda}, Bt_{i,mu}), and block m of the dual
    basis element (h, k) is F = -sum_pairs (A E_k B + B^T E_k A^T).  A^T P + P A is the case
    [(A^T, 1, I, 0)] (tests/test_oracle_general.py).  R (optional; the sum of the paper's R_i) is
    homogeneous of degree dp + e, coefficients [f(l, dp+e)][n][n] symmetric in W_{dp+e} order; the
    dual constraint B^T(y) - C >= 0 then carries C_{L+m} = coefficient of alpha^{gamma_m} in
    (sum alpha)^{d2} R(alpha) on the Lyapunov blocks (reading R18)."""
    es = {a + b for _, a, _, b in pairs}
    assert len(es) == 1, "all terms must have the same total degree"
    e = es.pop()
    beta = polya.beta_table(l, dp, d1)
    L0, L = beta.shape
    Wp = enumerate_W(l, dp)
    idx = polya.index_map(l, dp + e + d2)
    M = len(idx)
    S = polya.simplex_power(l, d2)
    gen = [[[] for _ in range(M)] for _ in range(L0)]
    for hi, h in enumerate(Wp):
        for At, a, Bt, b in pairs:
            Wa, Wb = enumerate_W(l, a), enumerate_W(l, b)
            for li, lam in enumerate(Wa):
                for mi, mu in enumerate(Wb):
                    mono = tuple(x + y + z for x, y, z in zip(h, lam, mu))
                    for e2, w in polya.poly_mul(S, {mono: 1}).items():
                        gen[hi][idx[e2]].append((float(w) * np.asarray(At[li], dtype=float),
                                                 np.asarray(Bt[mi], dtype=float)))
    Ntil = n * (n + 1) // 2
    c = polya.C_scalars(beta, l, dp, delta)
    CL = None
    if R is not None:
        CL = np.zeros((M,) + np.asarray(R).shape[1:])
        for ri, rho in enumerate(enumerate_W(l, dp + e)):
            for e2, w in polya.poly_mul(S, {tuple(rho): 1}).items():
                CL[idx[e2]] += float(w) * np.asarray(R[ri], dtype=float)
    Nb = int(np.asarray(pairs[0][0]).shape[1])
    return Problem(n, l, dp, e, d1, d2, delta, L0, L, M, Ntil, L0 * Ntil, beta, np.zeros((L0, M, 0, 0)), c, None,
                   basis(n), gen=gen, pairs=pairs, R=R, CL=CL, N=None if Nb == n else Nb)


def vmap(P: Problem, x, h: int):
    """V_<h>(x) = sum_j E_j x_{j+Ntil h} (Eq. 30) as a dense symmetric n x n matrix (x may carry
    leading batch dimensions: (..., K) -> (..., n, n))."""
    ia, ib = _ab(P.n)
    x = np.asarray(x, dtype=np.float64)
    seg = x[..., P.Ntil * h:P.Ntil * (h + 1)]
    out = np.zeros(x.shape[:-1] + (P.n, P.n))
    out[..., ia, ib] += seg
    off = ia != ib
    out[..., ib[off], ia[off]] += seg[..., off]
    return out


@functools.lru_cache(maxsize=None)
def _ab(n):
    """Index arrays (a_k, b_k) of the basis (cached, read-only)."""
    ab = np.array(basis(n), dtype=np.int64).reshape(-1, 2)
    ia, ib = ab[:, 0].copy(), ab[:, 1].copy()
    ia.flags.writeable = False
    ib.flags.writeable = False
    return ia, ib


def trE_all(n, M):
    """[tr(E_k M)]_k for every basis element at once (same rule as ``trE``); M may carry leading
    batch dimensions."""
    ia, ib = _ab(n)
    return np.where(ia == ib, M[..., ia, ia], M[..., ia, ib] + M[..., ib, ia])


def F_block(P: Problem, i: int, b: int):
    """B_{i,b} of Eq. (31), dense n x n."""
    h, k = divmod(i, P.Ntil)
    E = E_matrix(P.n, P.E[k])
    if b < P.L:
        return P.embed(float(P.beta[h, b]) * E)
    if P.gen is not None:
        F = np.zeros((P.bn, P.bn))
        for Aq, Bq in P.gen[h][b - P.L]:
            F -= Aq @ E @ Bq + Bq.T @ E @ Aq.T
        return F
    Hm = P.H[h, b - P.L]
    return -(Hm.T @ E + E @ Hm)


def F_stack(P: Problem, b: int, rows=None):
    """(len(rows), bn, bn) stack of B_{i,b} for i in rows (default all K): Eq. (31) for every row at
    once -- the same dense products as ``F_block`` (E_k built densely, then H^T E + E H or the
    generalised terms), batched over the rows that share h."""
    rows = np.arange(P.K) if rows is None else np.asarray(list(rows), dtype=np.int64)
    out = np.zeros((len(rows), P.bn, P.bn))
    if len(rows) == 0:
        return out
    ia, ib = _ab(P.n)
    hs, ks = np.divmod(rows, P.Ntil)
    for h in np.unique(hs):
        sel = np.nonzero(hs == h)[0]
        E = np.zeros((len(sel), P.n, P.n))
        r = np.arange(len(sel))
        E[r, ia[ks[sel]], ib[ks[sel]]] = 1.0
        E[r, ib[ks[sel]], ia[ks[sel]]] = 1.0
        if b < P.L:
            out[sel, :P.n, :P.n] = float(P.beta[h, b]) * E
        elif P.gen is not None:
            F = np.zeros((len(sel), P.bn, P.bn))
            for Aq, Bq in P.gen[h][b - P.L]:
                F -= Aq @ E @ Bq + Bq.T @ E @ Aq.T
            out[sel] = F
        else:
            Hm = P.H[h, b - P.L]
            out[sel] = -(Hm.T @ E + E @ Hm)
    return out


def apply_literal(P: Problem, y):
    """B^T(y) = sum_i y_i B_i (Eq. AT), blockwise, dense F."""
    out = np.zeros((P.nblocks, P.bn, P.bn))
    for b in range(P.nblocks):
        for i in range(P.K):
            if y[i] != 0.0:
                out[b] += y[i] * F_block(P, i, b)
    return out


def apply_vmap(P: Problem, y):
    """B^T(y) via Eq. (31) with e_i replaced by y (V is linear, Eq. 30):
    P-block j: sum_h beta_{h,j} V_h(y); Lyapunov block m: -sum_h (H^T V_h(y) + V_h(y) H)
    (terms with a structurally zero beta_{h,j} / H_{h,m} add nothing and are skipped).
    y may carry leading batch dimensions: (..., K) -> (..., nblocks, bn, bn)."""
    y = np.asarray(y, dtype=np.float64)
    out = np.zeros(y.shape[:-1] + (P.nblocks, P.bn, P.bn))
    V = [vmap(P, y, h) for h in range(P.L0)]
    for j in range(P.L):
        for h in range(P.L0):
            if P.beta[h, j] == 0:
                continue
            out[..., j, :P.n, :P.n] += float(P.beta[h, j]) * V[h]
    for m in range(P.M):
        for h in range(P.L0):
            if P.gen is not None:
                for Aq, Bq in P.gen[h][m]:
                    out[..., P.L + m, :, :] -= Aq @ V[h] @ Bq + Bq.T @ V[h] @ Aq.T
                continue
            Hm = P.H[h, m]
            if not np.any(Hm):
                continue
            out[..., P.L + m, :, :] -= Hm.T @ V[h] + V[h] @ Hm
    return out


def adjoint_literal(P: Problem, Xb):
    """B(X)_i = sum_b tr(B_{i,b} X_b), dense F."""
    y = np.zeros(P.K)
    for i in range(P.K):
        for b in range(P.nblocks):
            y[i] += np.trace(F_block(P, i, b) @ Xb[b])
    return y


def adjoint_trace(P: Problem, Xb):
    """B(X)_i with tr(B_{i,b} X_b) expanded by cyclicity of the trace:
    P-block: beta tr(E_k X); Lyapunov: -tr(H^T E X) - tr(E H X) = -tr(E_k (X H^T + H X)).
    Xb: (nblocks, bn, bn), or a batch (..., nblocks, bn, bn) giving y of shape (..., K)."""
    Xb = np.asarray(Xb)
    y = np.zeros(Xb.shape[:-3] + (P.K,))
    for h in range(P.L0):
        for b in range(P.nblocks):
            Xk = Xb[..., b, :, :]
            if b < P.L:
                if P.beta[h, b] == 0:
                    continue
                M = float(P.beta[h, b]) * Xk[..., :P.n, :P.n]
            elif P.gen is not None:
                terms = P.gen[h][b - P.L]
                if not terms:
                    continue
                # tr(F X) with F = -sum (A E B + B^T E A^T) = tr(E_k M), M = -sum (B X A + A^T X B^T)
                M = -sum(Bq @ Xk @ Aq + Aq.T @ Xk @ Bq.T for Aq, Bq in terms)
            else:
                Hm = P.H[h, b - P.L]
                if not np.any(Hm):
                    continue
                M = -(Xk @ Hm.T + Hm @ Xk)
            y[..., P.Ntil * h:P.Ntil * (h + 1)] += trE_all(P.n, M)
    return y


def schur_literal(P: Problem, Xb, Wb, rows=None):
    """lambda_{k,l} = sum_b tr(B_{k,b} Z_b^{-1} B_{l,b} X_b) (Eq. T2) for k in rows, all l.
    Per block: Y_l = W_b F_l X_b (two library matmuls), then
    tr(F_k Y_l) = sum_pq F_k[p,q] Y_l[q,p] (one library matmul over the flattened blocks)."""
    rows = list(range(P.K)) if rows is None else list(rows)
    G = np.zeros((len(rows), P.K))
    n2 = P.bn * P.bn
    for b in range(P.nblocks):
        Fb = F_stack(P, b)
        Y = np.matmul(np.matmul(Wb[b], Fb), Xb[b])
        Yt = Y.transpose(0, 2, 1).reshape(P.K, n2)
        G += Fb[rows].reshape(len(rows), n2) @ Yt.T
    return G


def schur_rows(P: Problem, Xb, Wb, rows, chunk=16):
    """Whole rows lambda_{k,.} of Eq. T2 for k in rows.  By cyclicity,
    lambda_{k,l} = sum_b tr(B_{k,b} Z_b^{-1} B_{l,b} X_b) = sum_b tr(B_{l,b} (X_b B_{k,b} Z_b^{-1})),
    i.e. row k is B(.) applied to the blocks M_b = X_b B_{k,b} Z_b^{-1}, with B_{k,b}
    the dense F of Eq. (31) (``F_stack``) and B(.) by ``adjoint_trace``.  Independent of the
    rank-structured four-term route (``schur_structured``) the CUDA path follows."""
    rows = list(rows)
    G = np.zeros((len(rows), P.K))
    for c0 in range(0, len(rows), chunk):
        rr = rows[c0:c0 + chunk]
        Mb = np.zeros((len(rr), P.nblocks, P.bn, P.bn))
        for b in range(P.nblocks):
            Mb[:, b] = Xb[b] @ F_stack(P, b, rr) @ Wb[b]
        G[c0:c0 + len(rr)] = adjoint_trace(P, Mb)
    return G


def schur_entries(P: Problem, Xb, Wb, pairs):
    """lambda_{k,l} = sum_b tr(B_{k,b} Z_b^{-1} B_{l,b} X_b) (Eq. T2) for an explicit list of (k, l)
    pairs: dense F (Eq. 31) and one trace of the four-matrix product per pair and block, blocks where
    B_{k,b} or B_{l,b} is structurally zero skipped; batched over the pairs of a block."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    out = np.zeros(len(pairs))
    hk, hl = pairs[:, 0] // P.Ntil, pairs[:, 1] // P.Ntil
    for b in range(P.nblocks):
        act = np.array([P.active(h, b) for h in range(P.L0)], dtype=bool)
        sel = np.nonzero(act[hk] & act[hl])[0]
        for c0 in range(0, len(sel), 256):
            s = sel[c0:c0 + 256]
            FkW = F_stack(P, b, pairs[s, 0]) @ Wb[b]
            FlX = F_stack(P, b, pairs[s, 1]) @ Xb[b]
            out[s] += np.einsum("epq,eqp->e", FkW, FlX)
    return out


def schur_probe(P: Problem, Xb, Wb, v):
    """(G v)_k = sum_l lambda_{k,l} v_l = sum_b tr(B_{k,b} W_b (sum_l v_l B_{l,b}) X_b)
    = B(W B^T(v) X)_k by linearity of Eq. (T2) in B_l.  v: (K,) or a batch (p, K) of probes."""
    Fv = apply_vmap(P, v)
    Y = np.matmul(np.matmul(Wb, Fv), Xb)
    return adjoint_trace(P, Y)


def schur_structured(P: Problem, Xb, Wb, pairs=None):
    """The SCM of Eq. T2 by the rank structure of the blocks (SURVEY 8(c) O6'(iii)/O7), derived here
    directly from the trace: with F_(h,s)^m = -(H^T E_s + E_s H), H = H_{h,m}, H' = H_{h',m},
    E_s = sum_{(a1,b1) in or(s)} e_a1 e_b1^T and tr(A e_a1 e_b1^T B e_c1 e_d1^T C) = B[b1,c1] (C A)[d1,a1],
      tr(F_(h,s) W F_(h',t) X) = sum_{or(s), or(t)} sum_k L_k[b1,c1] R_k[d1,a1]
    over the four terms (L, R) = (W H'^T, X H^T), (W, H' X H^T), (H W H'^T, X), (H W, H' X) of each
    Lyapunov block and (beta_hj beta_h'j W_j, X_j) of each P-block.  Per pair (h <= h') the sum over
    k is one library matmul Raw = [vec L_k]^T [vec R_k] (n^2 x n^2), folded by the four orientation
    gathers.  pairs: optional list of (h, h') to compute (the rest of G stays zero)."""
    G = np.zeros((P.K, P.K))
    N = P.Ntil
    todo = pairs if pairs is not None else [(h, h2) for h in range(P.L0) for h2 in range(h, P.L0)]
    for h, h2 in todo:
        blk = schur_structured_tile(P, Xb, Wb, h, h2)
        G[h * N:(h + 1) * N, h2 * N:(h2 + 1) * N] = blk
        if h2 != h:
            G[h2 * N:(h2 + 1) * N, h * N:(h + 1) * N] = blk.T
    return G


def schur_structured_tile(P: Problem, Xb, Wb, h, h2):
    """The (h, h') block G[h-rows, h'-columns] of ``schur_structured`` alone (Ntil x Ntil; the same
    arithmetic, so large configurations can be checked pair by pair)."""
    n, N, L = P.n, P.Ntil, P.L
    ia, ib = _ab(n)
    a, b = ia[:, None], ib[:, None]
    c, d = ia[None, :], ib[None, :]
    Ls, Rs = [], []
    for j in range(L):
        if P.beta[h, j] and P.beta[h2, j]:
            Ls.append(float(P.beta[h, j] * P.beta[h2, j]) * Wb[j][:n, :n])
            Rs.append(Xb[j][:n, :n])
    for m in range(P.M):
        W, X = Wb[L + m], Xb[L + m]
        if P.gen is not None:
            # F = -sum_q (A_q E B_q + B_q^T E A_q^T): the same four terms per (q, q'), here
            # (B W A', B' X A), (B W B'^T, A'^T X A), (A^T W A', B' X B^T), (A^T W B'^T, A'^T X B^T)
            # (H^T, I) for (A, B) gives back the continuous-time terms below (reading R18)
            for A1, B1 in P.gen[h][m]:
                for A2, B2 in P.gen[h2][m]:
                    Ls += [B1 @ W @ A2, B1 @ W @ B2.T, A1.T @ W @ A2, A1.T @ W @ B2.T]
                    Rs += [B2 @ X @ A1, A2.T @ X @ A1, B2 @ X @ B1.T, A2.T @ X @ B1.T]
            continue
        H, H2 = P.H[h, m], P.H[h2, m]
        if not (np.any(H) and np.any(H2)):
            continue
        Ls += [W @ H2.T, W, H @ W @ H2.T, H @ W]
        Rs += [X @ H.T, H2 @ X @ H.T, X, H2 @ X]
    if not Ls:
        return np.zeros((N, N))
    k = len(Ls)
    R4 = (np.stack(Ls).reshape(k, n * n).T @ np.stack(Rs).reshape(k, n * n)).reshape(n, n, n, n)
    sw, tw = a != b, c != d
    blk = R4[b, c, d, a] + np.where(sw, R4[a, c, d, b], 0.0) + np.where(tw, R4[b, d, c, a], 0.0) \
        + np.where(sw & tw, R4[a, d, c, b], 0.0)
    return blk
