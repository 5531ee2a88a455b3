"""Python binding of libpolya.so (include/polya.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; PyTorch only
provides device memory and the stream.  There is no CPU fallback: if the
shared library is missing or CUDA is unavailable, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["lib", "Polya", "PolyaError", "G_FULL", "G_PAIR_TILES", "SHARD_TILES", "SHARD_BLOCKS", "SHARD_CYCLIC",
           "EXPORTS", "LIB_PATH", "plan", "nccl_unique_id", "homogenize", "simplex_map", "factor_solve_loopback",
           "p2p_loopback"]

# POLYA_LIB overrides the library path (timing-experiment variants built by tools/schur_exp.py)
LIB_PATH = os.environ.get("POLYA_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpolya.so")
G_FULL, G_PAIR_TILES = 0, 1
EDIVERGED, EMAXIT, ENOTPD, ESTEP = 9, 8, 6, 7
SHARD_TILES, SHARD_BLOCKS, SHARD_CYCLIC = 0, 1, 2
EXPORTS = ["polya_setup", "polya_dims_get", "polya_plan", "polya_get_exponents", "polya_get_beta", "polya_get_H",
           "polya_get_C", "polya_apply", "polya_adjoint", "polya_schur", "polya_ipm_step", "polya_sync",
           "polya_strerror", "polya_last_error", "polya_launch_count", "polya_destroy", "polya_set_timing",
           "polya_get_timing", "polya_nccl_unique_id", "polya_nccl_init", "polya_reduce_G", "polya_homogenize",
           "polya_simplex_map", "polya_ipm_solve", "polya_verdict", "polya_set_factorization", "polya_schur_prepare",
           "polya_schur_assemble", "polya_setup_general", "polya_factor_solve_loopback", "polya_schur_reduce",
           "polya_get_combine_timing", "polya_set_combine_tiles", "polya_p2p_export", "polya_p2p_import",
           "polya_p2p_loopback", "polya_schur_reduce_p2p", "polya_block_kernels_test"]


class PolyaError(RuntimeError):
    pass


class _Config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("l", ctypes.c_int32), ("dp", ctypes.c_int32), ("da", ctypes.c_int32),
                ("d1", ctypes.c_int32), ("d2", ctypes.c_int32), ("delta", ctypes.c_double),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("shard", ctypes.c_int32)]


class _Dims(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("L0", "L", "M", "nblocks", "Ntil", "K", "nnz_beta", "nnz_H",
                                              "npairs", "pair0", "pair1", "item0", "item1")] + \
               [("useful_flops_schur", ctypes.c_double), ("tiles_bytes", ctypes.c_int64), ("b0", ctypes.c_int64),
                ("b1", ctypes.c_int64), ("reduce_count", ctypes.c_int64), ("npairs_local", ctypes.c_int64),
                ("block_n", ctypes.c_int64), ("combine_tiles", ctypes.c_int64)]


class _IpmState(ctypes.Structure):
    _fields_ = [("X", ctypes.c_void_p), ("Z", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("mu", ctypes.c_double), ("iter", ctypes.c_int32)]


class _SolveResult(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int32), ("iterations", ctypes.c_int32), ("status", ctypes.c_int32),
                ("gap", ctypes.c_double), ("pinf", ctypes.c_double), ("mu", ctypes.c_double),
                ("ms_schur", ctypes.c_float), ("ms_factor", ctypes.c_float), ("ms_other", ctypes.c_float)]


class _IpmStats(ctypes.Structure):
    _fields_ = [("gap", ctypes.c_double), ("mu", ctypes.c_double), ("tp", ctypes.c_double), ("td", ctypes.c_double),
                ("phi", ctypes.c_double), ("psi", ctypes.c_double), ("ms_schur", ctypes.c_float),
                ("ms_factor", ctypes.c_float), ("ms_other", ctypes.c_float), ("reg_retries", ctypes.c_int32)]


class _SolveOpts(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("tol", ctypes.c_double), ("maxit", ctypes.c_int32), ("init", ctypes.c_int32),
                ("history", ctypes.POINTER(_IpmStats))]


_lib = None


def lib():
    """Load libpolya.so (loud failure if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1411_3769_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.polya_setup.argtypes = [ctypes.POINTER(_Config), vp, ctypes.POINTER(vp)]
    L.polya_setup_general.argtypes = [ctypes.POINTER(_Config), i32, i32, vp, vp, vp, vp, vp, ctypes.POINTER(vp)]
    L.polya_factor_solve_loopback.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(vp), vp, vp]
    L.polya_block_kernels_test.argtypes = [i32, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
    L.polya_dims_get.argtypes = [vp, ctypes.POINTER(_Dims)]
    L.polya_plan.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_Dims)]
    L.polya_get_exponents.argtypes = [vp, ctypes.c_int, vp]
    L.polya_get_beta.argtypes = [vp, vp]
    L.polya_get_H.argtypes = [vp, vp]
    L.polya_get_C.argtypes = [vp, vp]
    L.polya_apply.argtypes = [vp, vp, vp, vp]
    L.polya_adjoint.argtypes = [vp, vp, vp, vp]
    L.polya_schur.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp]
    L.polya_schur_prepare.argtypes = [vp, vp, vp, vp]
    L.polya_schur_assemble.argtypes = [vp, vp, ctypes.c_int, i64, i64, vp]
    L.polya_ipm_step.argtypes = [vp, ctypes.POINTER(_IpmState), ctypes.POINTER(_IpmStats), vp]
    L.polya_sync.argtypes = [vp]
    L.polya_set_timing.argtypes = [vp, ctypes.c_int]
    L.polya_get_timing.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
    L.polya_nccl_unique_id.argtypes = [vp]
    L.polya_nccl_init.argtypes = [vp, vp]
    L.polya_reduce_G.argtypes = [vp, vp, vp, ctypes.c_int, vp]
    L.polya_schur_reduce.argtypes = [vp, vp, vp, vp, vp]
    L.polya_get_combine_timing.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
    L.polya_set_combine_tiles.argtypes = [vp, i64]
    L.polya_p2p_export.argtypes = [vp, vp]
    L.polya_p2p_import.argtypes = [vp, vp]
    L.polya_p2p_loopback.argtypes = [ctypes.POINTER(vp), i32]
    L.polya_schur_reduce_p2p.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp]
    L.polya_homogenize.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.polya_simplex_map.argtypes = [i32, i32, i32, vp, vp, vp, vp]
    L.polya_ipm_solve.argtypes = [vp, ctypes.POINTER(_IpmState), ctypes.POINTER(_SolveOpts), ctypes.POINTER(_SolveResult),
                                  vp]
    L.polya_verdict.argtypes = [vp, vp, i32, vp, vp, vp]
    L.polya_set_factorization.argtypes = [vp, ctypes.c_int]
    L.polya_strerror.argtypes = [ctypes.c_int]
    L.polya_strerror.restype = ctypes.c_char_p
    L.polya_last_error.argtypes = [vp]
    L.polya_last_error.restype = ctypes.c_char_p
    L.polya_launch_count.argtypes = [vp]
    L.polya_launch_count.restype = i64
    L.polya_destroy.argtypes = [vp]
    L.polya_destroy.restype = None
    for name in EXPORTS:
        if name not in ("polya_strerror", "polya_last_error", "polya_launch_count", "polya_destroy"):
            getattr(L, name).restype = ctypes.c_int
    del i32, dbl
    _lib = L
    return L


def plan(n, l, dp, d1, d2, da=1, delta=1e-3, rank=0, nranks=1, shard=SHARD_TILES):
    """polya_plan: host-only dims and this rank's share of the Schur work (no GPU)."""
    cfg = _Config(n, l, dp, da, d1, d2, delta, rank, nranks, shard)
    d = _Dims()
    st = lib().polya_plan(ctypes.byref(cfg), ctypes.byref(d))
    if st != 0:
        raise PolyaError(f"polya_plan: {lib().polya_strerror(st).decode()}")
    return {k: getattr(d, k) for k, _ in _Dims._fields_}


def nccl_unique_id():
    """polya_nccl_unique_id (rank 0): 128 opaque bytes the caller distributes to every rank."""
    buf = ctypes.create_string_buffer(128)
    st = lib().polya_nccl_unique_id(buf)
    if st != 0:
        raise PolyaError(f"polya_nccl_unique_id: {lib().polya_strerror(st).decode()}")
    return bytes(buf.raw)


def factor_solve_loopback(ctxs, G_local, x, stream=None):
    """polya_factor_solve_loopback: the SHARD_CYCLIC distributed Cholesky + solve with all ranks'
    contexts in this process (test hook; device copies in place of the NCCL broadcasts).
    G_local[r]: rank r's pair tiles (overwritten by its factor tiles); x (K doubles) <- G^{-1} x."""
    n = len(ctxs)
    hs = (ctypes.c_void_p * n)(*[c._h.value for c in ctxs])
    gs = (ctypes.c_void_p * n)(*[_dev_ptr(g, None, "G_local").value for g in G_local])
    st = lib().polya_factor_solve_loopback(hs, n, gs, _dev_ptr(x, ctxs[0].K, "x"), _stream_ptr(stream))
    if st != 0:
        raise PolyaError(f"polya_factor_solve_loopback: {lib().polya_strerror(st).decode()} "
                         f"({lib().polya_last_error(ctxs[0]._h).decode()})")
    return x


def block_kernels_test(S, dS, stream=None):
    """polya_block_kernels_test (test hook): the IPM's blockwise kernels on (nb, n, n) device stacks.
    Returns (W = S^-1, L^-1, M = L^-1 dS L^-T, t, fail) with t_b = min(1/0.98, 1/max(0, -lambda_min(M_b)))
    (-1 for a block whose S_b is not positive definite) and fail = 1 if some S_b is not."""
    import torch
    nb, n = int(S.shape[0]), int(S.shape[1])
    W, Li, M = (torch.empty_like(S) for _ in range(3))
    t = torch.empty(nb, dtype=torch.float64, device=S.device)
    fail = torch.zeros(1, dtype=torch.int32, device=S.device)
    st = lib().polya_block_kernels_test(n, nb, _dev_ptr(S, nb * n * n, "S"), _dev_ptr(dS, nb * n * n, "dS"),
                                        _dev_ptr(W, None, "W"), _dev_ptr(Li, None, "Linv"), _dev_ptr(M, None, "M"),
                                        _dev_ptr(t, nb, "t"), ctypes.c_void_p(fail.data_ptr()), _stream_ptr(stream))
    if st != 0:
        raise PolyaError(f"polya_block_kernels_test: {lib().polya_strerror(st).decode()}")
    return W, Li, M, t, int(fail.item())


def p2p_loopback(ctxs):
    """polya_p2p_loopback: wire the P2P combine of the contexts of one process (test hook)."""
    n = len(ctxs)
    hs = (ctypes.c_void_p * n)(*[c._h.value for c in ctxs])
    st = lib().polya_p2p_loopback(hs, n)
    if st != 0:
        raise PolyaError(f"polya_p2p_loopback: {lib().polya_strerror(st).decode()} "
                         f"({lib().polya_last_error(ctxs[0]._h).decode()})")


def homogenize(terms, l):
    """polya_homogenize: terms = {exponent tuple: n x n array}; returns
    (d_a, coefficients double[f(l,d_a)][n][n] in W_{d_a} order)."""
    exps = np.ascontiguousarray(np.array([list(e) for e in terms], dtype=np.int32))
    coeffs = np.ascontiguousarray(np.array([np.asarray(c, dtype=np.float64) for c in terms.values()]))
    n = coeffs.shape[-1]
    da = ctypes.c_int32()
    vp = ctypes.c_void_p
    st = lib().polya_homogenize(l, n, len(exps), exps.ctypes.data_as(vp), coeffs.ctypes.data_as(vp), ctypes.byref(da),
                                None)
    if st != 0:
        raise PolyaError(f"polya_homogenize: {lib().polya_strerror(st).decode()}")
    from math import comb
    out = np.zeros((comb(l + da.value - 1, l - 1), n, n))
    st = lib().polya_homogenize(l, n, len(exps), exps.ctypes.data_as(vp), coeffs.ctypes.data_as(vp), ctypes.byref(da),
                                out.ctypes.data_as(vp))
    if st != 0:
        raise PolyaError(f"polya_homogenize: {lib().polya_strerror(st).decode()}")
    return da.value, out


def simplex_map(A, l, d, scale, shift):
    """polya_simplex_map: coefficients of A(g(alpha)), g_i = scale_i alpha_i + shift_i sum_j alpha_j."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    sc = np.ascontiguousarray(np.asarray(scale, dtype=np.float64))
    sh = np.ascontiguousarray(np.asarray(shift, dtype=np.float64))
    out = np.zeros_like(A)
    vp = ctypes.c_void_p
    st = lib().polya_simplex_map(l, d, A.shape[-1], sc.ctypes.data_as(vp), sh.ctypes.data_as(vp), A.ctypes.data_as(vp),
                                 out.ctypes.data_as(vp))
    if st != 0:
        raise PolyaError(f"polya_simplex_map: {lib().polya_strerror(st).decode()}")
    return out


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev_ptr(t, numel=None, name="tensor"):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise PolyaError(f"{name} must be a CUDA torch tensor")
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise PolyaError(f"{name} must be contiguous float64")
    if numel is not None and t.numel() != numel:
        raise PolyaError(f"{name} has {t.numel()} elements, expected {numel}")
    return ctypes.c_void_p(t.data_ptr())


class Polya:
    """One context = one rank / GPU (``polya_setup``).  ``A`` is the host array
    double[f(l,da)][n][n] of A(alpha)'s coefficients in W_da order.  With ``terms`` =
    [(At_i, deg_a_i, Bt_i, deg_b_i), ...] (A ignored, da = deg_a + deg_b) the context is the
    generalised form sum_i (At_i P Bt_i + transpose) < 0 (``polya_setup_general``)."""

    @classmethod
    def general(cls, terms, n, l, dp, d1, d2, delta=1e-3, rank=0, nranks=1, shard=SHARD_TILES, R=None):
        """R: optional constant term, coefficients double[f(l, dp+e)][n][n] in W_{dp+e} order."""
        return cls(n, l, dp, d1, d2, None, delta=delta, rank=rank, nranks=nranks, shard=shard, terms=terms, R=R)

    def __init__(self, n, l, dp, d1, d2, A, da=1, delta=1e-3, rank=0, nranks=1, shard=SHARD_TILES, terms=None, R=None):
        L = lib()
        h = ctypes.c_void_p()
        if terms is None:
            A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
            cfg = _Config(n, l, dp, da, d1, d2, delta, rank, nranks, shard)
            st = L.polya_setup(ctypes.byref(cfg), A.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h))
            what = "polya_setup"
        else:   # generalised form (polya_setup_general): terms = [(At, deg_a, Bt, deg_b), ...]
            da = int(terms[0][1]) + int(terms[0][3])
            cfg = _Config(n, l, dp, da, d1, d2, delta, rank, nranks, shard)
            dega = np.array([t[1] for t in terms], dtype=np.int32)
            degb = np.array([t[3] for t in terms], dtype=np.int32)
            At = np.ascontiguousarray(np.concatenate([np.asarray(t[0], dtype=np.float64).reshape(-1) for t in terms]))
            Bt = np.ascontiguousarray(np.concatenate([np.asarray(t[2], dtype=np.float64).reshape(-1) for t in terms]))
            cp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
            Rh = None if R is None else np.ascontiguousarray(np.asarray(R, dtype=np.float64))
            nlmi = int(np.asarray(terms[0][0]).shape[1])   # At_0 is N x n
            st = L.polya_setup_general(ctypes.byref(cfg), nlmi, len(terms), cp(dega), cp(degb), cp(At), cp(Bt),
                                       None if Rh is None else cp(Rh), ctypes.byref(h))
            what = "polya_setup_general"
        if st != 0:
            raise PolyaError(f"{what}: {L.polya_strerror(st).decode()}")
        self._h = h
        self.n, self.l, self.dp, self.da, self.d1, self.d2 = n, l, dp, da, d1, d2
        self.delta, self.rank, self.nranks, self.shard = delta, rank, nranks, shard
        d = _Dims()
        self._check(L.polya_dims_get(self._h, ctypes.byref(d)), "polya_dims_get")
        self.dims = {k: getattr(d, k) for k, _ in _Dims._fields_}
        for k in ("L0", "L", "M", "nblocks", "Ntil", "K"):
            setattr(self, k, int(self.dims[k]))
        self.bn = int(self.dims["block_n"])   # order of every block (n, or the generalised form's N)

    def _check(self, st, what):
        if st != 0:
            L = lib()
            raise PolyaError(f"{what}: {L.polya_strerror(st).decode()} ({L.polya_last_error(self._h).decode()})")

    # -- set-up queries ----------------------------------------------------------------------------
    def exponents(self, which):
        counts = {0: self.L0, 1: self.L, 2: self.M}
        if which == 3:
            from math import comb
            cnt = comb(self.l + self.da - 1, self.l - 1)
        else:
            cnt = counts[which]
        out = np.zeros((cnt, self.l), dtype=np.int32)
        self._check(lib().polya_get_exponents(self._h, which, out.ctypes.data_as(ctypes.c_void_p)), "get_exponents")
        return out

    def beta(self):
        out = np.zeros((self.L0, self.L), dtype=np.int64)
        self._check(lib().polya_get_beta(self._h, out.ctypes.data_as(ctypes.c_void_p)), "get_beta")
        return out

    def H(self):
        out = np.zeros((self.L0, self.M, self.n, self.n), dtype=np.float64)
        self._check(lib().polya_get_H(self._h, out.ctypes.data_as(ctypes.c_void_p)), "get_H")
        return out

    def C(self):
        out = np.zeros(self.L, dtype=np.float64)
        self._check(lib().polya_get_C(self._h, out.ctypes.data_as(ctypes.c_void_p)), "get_C")
        return out

    # -- operators ----------------------------------------------------------------------------------
    def apply(self, y, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.nblocks, self.bn, self.bn), dtype=torch.float64, device=y.device)
        self._check(lib().polya_apply(self._h, _dev_ptr(y, self.K, "y"), _dev_ptr(out, self.nblocks * self.bn ** 2, "out"),
                                      _stream_ptr(stream)), "polya_apply")
        return out

    def adjoint(self, X, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.K, dtype=torch.float64, device=X.device)
        self._check(lib().polya_adjoint(self._h, _dev_ptr(X, self.nblocks * self.bn ** 2, "X"), _dev_ptr(out, self.K, "y"),
                                        _stream_ptr(stream)), "polya_adjoint")
        return out

    def schur(self, X, Zinv, G=None, layout=G_FULL, stream=None):
        import torch
        if G is None:
            if layout == G_FULL:
                G = torch.zeros((self.K, self.K), dtype=torch.float64, device=X.device)
            elif self.shard == SHARD_BLOCKS:   # flat partial-G buffer: all pair tiles + zero padding
                G = torch.zeros(self.nranks * self.dims["reduce_count"], dtype=torch.float64, device=X.device)
            else:
                npl = self.dims["npairs_local"]
                G = torch.zeros((npl, self.Ntil, self.Ntil), dtype=torch.float64, device=X.device)
        nbn = self.nblocks * self.bn ** 2
        self._check(lib().polya_schur(self._h, _dev_ptr(X, nbn, "X"), _dev_ptr(Zinv, nbn, "Zinv"), _dev_ptr(G, None, "G"),
                                      layout, _stream_ptr(stream)), "polya_schur")
        return G

    def schur_prepare(self, X, Zinv, stream=None):
        nbn = self.nblocks * self.bn ** 2
        self._check(lib().polya_schur_prepare(self._h, _dev_ptr(X, nbn, "X"), _dev_ptr(Zinv, nbn, "Zinv"),
                                              _stream_ptr(stream)), "polya_schur_prepare")

    def schur_assemble(self, G, pair_begin, pair_end, layout=G_PAIR_TILES, stream=None):
        self._check(lib().polya_schur_assemble(self._h, _dev_ptr(G, None, "G"), layout, int(pair_begin), int(pair_end),
                                               _stream_ptr(stream)), "polya_schur_assemble")
        return G

    def ipm_step(self, X, Z, y, mu, it=0, stream=None):
        st = _IpmState(_dev_ptr(X, None, "X").value, _dev_ptr(Z, None, "Z").value, _dev_ptr(y, self.K, "y").value,
                       float(mu), int(it))
        stats = _IpmStats()
        self._check(lib().polya_ipm_step(self._h, ctypes.byref(st), ctypes.byref(stats), _stream_ptr(stream)),
                    "polya_ipm_step")
        return {k: getattr(stats, k) for k, _ in _IpmStats._fields_}

    def nccl_init(self, uid):
        """polya_nccl_init: collective over the nranks contexts (SHARD_BLOCKS combine, SHARD_CYCLIC
        distributed factorisation)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        self._check(lib().polya_nccl_init(self._h, buf), "polya_nccl_init")

    def reduce_G(self, Gpart, out=None, layout=G_PAIR_TILES, stream=None):
        """polya_reduce_G: sum of the ranks' partial G (ReduceScatter of the pair tiles, or AllReduce
        of the FULL matrix)."""
        import torch
        if out is None:
            out = (torch.empty(self.dims["reduce_count"], dtype=torch.float64, device=Gpart.device)
                   if layout == G_PAIR_TILES else Gpart)
        self._check(lib().polya_reduce_G(self._h, _dev_ptr(Gpart, None, "Gpart"), _dev_ptr(out, None, "Grecv"), layout,
                                         _stream_ptr(stream)), "polya_reduce_G")
        return out

    def schur_reduce(self, X, Zinv, out=None, stream=None):
        """polya_schur_reduce: the block-sharded partial G assembled tile group by tile group, each
        group's NCCL reduce-scatter overlapping the next group's assembly; returns this rank's summed
        tiles (reduce_count doubles, layout of polya_dims.combine_tiles)."""
        import torch
        if out is None:
            out = torch.empty(self.dims["reduce_count"], dtype=torch.float64, device=X.device)
        nbn = self.nblocks * self.bn ** 2
        self._check(lib().polya_schur_reduce(self._h, _dev_ptr(X, nbn, "X"), _dev_ptr(Zinv, nbn, "Zinv"),
                                             _dev_ptr(out, self.dims["reduce_count"], "Grecv"), _stream_ptr(stream)),
                    "polya_schur_reduce")
        return out

    def set_combine_tiles(self, t):
        """polya_set_combine_tiles: tiles per rank and group of the combine (0 = automatic)."""
        self._check(lib().polya_set_combine_tiles(self._h, int(t)), "polya_set_combine_tiles")
        d = _Dims()
        self._check(lib().polya_dims_get(self._h, ctypes.byref(d)), "polya_dims_get")
        self.dims = {k: getattr(d, k) for k, _ in _Dims._fields_}

    def p2p_export(self):
        """polya_p2p_export: this rank's 64-byte IPC handle of its receive slots (fused P2P combine)."""
        buf = ctypes.create_string_buffer(64)
        self._check(lib().polya_p2p_export(self._h, buf), "polya_p2p_export")
        return bytes(buf.raw)

    def p2p_import(self, handles):
        """polya_p2p_import: every rank's handle, in rank order."""
        blob = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * len(handles))
        self._check(lib().polya_p2p_import(self._h, blob), "polya_p2p_import")

    def schur_reduce_p2p(self, X, Zinv, out=None, phases=3, stream=None):
        """polya_schur_reduce_p2p: the assembly writing each partial tile into its owner's slot over peer
        memory (phases bit 1) and the owner's ordered sum of the slots (bit 2)."""
        import torch
        if out is None and phases & 2:
            out = torch.empty(self.dims["reduce_count"], dtype=torch.float64, device=X.device)
        nbn = self.nblocks * self.bn ** 2
        self._check(lib().polya_schur_reduce_p2p(self._h, _dev_ptr(X, nbn, "X") if phases & 1 else None,
                                                 _dev_ptr(Zinv, nbn, "Zinv") if phases & 1 else None,
                                                 _dev_ptr(out, self.dims["reduce_count"], "Grecv") if phases & 2 else None,
                                                 int(phases), _stream_ptr(stream)), "polya_schur_reduce_p2p")
        return out

    def combine_timing(self):
        a = ctypes.c_float()
        self._check(lib().polya_get_combine_timing(self._h, ctypes.byref(a)), "polya_get_combine_timing")
        return float(a.value)

    def ipm_solve(self, X=None, Z=None, y=None, eps=1e-8, tol=1e-8, maxit=60, init=True, mu=None, it=0,
                  stream=None):
        """polya_ipm_solve: Algorithm 2 to its stopping rule (state on the device, updated in place).
        init=True starts from X = Z = I, y = 0 (the library sets mu = 1/3); init=False resumes from the
        given X, Z, y with the caller's barrier parameter mu (e.g. the last step's stats["mu"])."""
        import torch
        if not init and (X is None or Z is None or y is None or mu is None):
            raise PolyaError("ipm_solve(init=False) resumes a state: pass X, Z, y and mu")
        nbn = (self.nblocks, self.bn, self.bn)
        X = torch.empty(nbn, dtype=torch.float64, device="cuda") if X is None else X
        Z = torch.empty(nbn, dtype=torch.float64, device="cuda") if Z is None else Z
        y = torch.empty(self.K, dtype=torch.float64, device="cuda") if y is None else y
        st = _IpmState(_dev_ptr(X, None, "X").value, _dev_ptr(Z, None, "Z").value, _dev_ptr(y, self.K, "y").value,
                       1.0 / 3.0 if init else float(mu), 0 if init else int(it))
        hist = (_IpmStats * max(int(maxit), 1))()
        opt = _SolveOpts(float(eps), float(tol), int(maxit), int(bool(init)), hist)
        res = _SolveResult()
        self._check(lib().polya_ipm_solve(self._h, ctypes.byref(st), ctypes.byref(opt), ctypes.byref(res),
                                          _stream_ptr(stream)), "polya_ipm_solve")
        out = {k: getattr(res, k) for k, _ in _SolveResult._fields_}
        out["history"] = [{k: getattr(hist[i], k) for k, _ in _IpmStats._fields_} for i in range(res.iterations)]
        out.update(X=X, Z=Z, y=y)
        return out

    def verdict(self, y, pts, stream=None):
        """polya_verdict: number of points of the simplex where the certificate fails the grid check."""
        pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, self.l))
        nf = ctypes.c_int32()
        self._check(lib().polya_verdict(self._h, _dev_ptr(y, self.K, "y"), len(pts), pts.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.byref(nf), _stream_ptr(stream)), "polya_verdict")
        return int(nf.value)

    def set_factorization(self, mode):
        """polya_set_factorization: 0 auto, 1 dense K x K, 2 tiled (pair tiles)."""
        self._check(lib().polya_set_factorization(self._h, int(mode)), "polya_set_factorization")

    def set_timing(self, on=True):
        self._check(lib().polya_set_timing(self._h, int(bool(on))), "polya_set_timing")

    def timing(self):
        a, b = ctypes.c_float(), ctypes.c_float()
        self._check(lib().polya_get_timing(self._h, ctypes.byref(a), ctypes.byref(b)), "polya_get_timing")
        return float(a.value), float(b.value)

    def sync(self):
        self._check(lib().polya_sync(self._h), "polya_sync")

    def launch_count(self):
        return int(lib().polya_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib().polya_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
