/*
 * polya.h -- C ABI of the B200-native hot path of Kamyar, Peet & Peet,
 * "Solving Large-Scale Robust Stability Problems by Exploiting the Parallel
 * Structure of Polya's Theorem" (IEEE TAC 2013, arxiv 1411.3769).
 *
 * Citations "PAPER.md:n" are lines of the paper's LaTeX source; "R1".."R16"
 * are the readings of ambiguous passages listed in DESIGN.md.
 *
 * Problem: robust stability of x' = A(alpha) x,
 * alpha in the unit simplex, A(alpha) = sum_{lambda in W_da} A_lambda alpha^lambda.
 * Polya's multipliers turn P(alpha) > 0 and A^T P + P A < 0 into L + M
 * coefficient LMIs ("blocks"), posed as one block-diagonal SDP (Eqs. 26-32,
 * PAPER.md:341-379):
 *   blocks b = 0 .. L-1      P-blocks,        gamma_b in W_{dp+d1}  (Eq. LMI_3)
 *   blocks b = L .. L+M-1    Lyapunov blocks, gamma_b in W_{dp+da+d2} (Eq. LMI_4)
 *   dual index i = k + Ntil*h (0-based), h in W_dp, k in the basis of S^n (R2),
 *   Ntil = n(n+1)/2, K = |W_dp| * Ntil (Eq. K).
 *   F_i^b = beta_{h,b} E_k                      (P-block, Eq. 31 case I)
 *   F_i^b = -(H_{h,m}^T E_k + E_k H_{h,m})       (Lyapunov block m=b-L, case II)
 *
 * Conventions (binding for every entry point):
 *  - 0-based indices.  The paper's <gamma> = position + 1 in W_d, W_d ordered by
 *    PAPER.md:58's prose (descending lexicographic; reading R1).
 *  - Basis of S^n (reading R2, diagonal-major): k < n -> (k,k); then for offset
 *    o = 1..n-1 and row a = 0..n-1-o: (a, a+o).  E = e_a e_b^T + e_b e_a^T off the
 *    diagonal (unnormalised), so y holds actual matrix entries.
 *  - Matrices are row-major, contiguous, FP64.  A "block stack" is
 *    double[nblocks][n][n] in block order above.
 *  - Pointers named *_host are host memory; *_dev are device memory on the
 *    context's device (caller-owned, 16-byte aligned; torch tensors qualify).
 *  - apply / adjoint / schur are stream-ordered and asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).  Asynchronous
 *    kernel faults surface at polya_sync() or the next call.
 *  - Every entry point returns a polya_status; nothing aborts or throws across
 *    the boundary.  polya_last_error(ctx) gives a human-readable detail.
 *  - One context per rank / GPU; a context is not thread-safe; no global state.
 */
#ifndef POLYA_H_
#define POLYA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct polya_ctx polya_ctx;

typedef enum {
  POLYA_OK = 0,
  POLYA_EINVAL = 1,     /* bad dimension, null pointer, unsupported option        */
  POLYA_EOVERFLOW = 2,  /* checked int64 failure on f(l,d), K, K*K or a byte size */
  POLYA_ENOMEM = 3,     /* device or host allocation failed                       */
  POLYA_ECUDA = 4,      /* CUDA runtime / kernel error                            */
  POLYA_ENCCL = 5,      /* NCCL error, or a collective called without polya_nccl_init */
  POLYA_ENOTPD = 6,     /* a Z block or the Schur complement is not positive definite */
  POLYA_ESTEP = 7,      /* line search found no admissible step                   */
  POLYA_EMAXIT = 8,     /* iteration limit of a driver (polya_ipm_solve outcome)  */
  POLYA_EDIVERGED = 9   /* iterates left every bound (polya_ipm_solve outcome): max(|phi|, |psi|, mu)
                           > POLYA_DIVERGENCE_BOUND or non-finite -- an unbounded primal, i.e. an
                           infeasible LMI (reading R20) */
} polya_status;

/* Divergence exit of polya_ipm_solve (reading R20): the iteration stops with status
 * EDIVERGED as soon as tr(CX), a^T y or mu exceeds this bound in magnitude.  The problems are scaled
 * so that a = 1 and X = Z = I at the start (mu = 1/3); a converging run stays many orders below. */
#define POLYA_DIVERGENCE_BOUND 1e12

/* How the Schur complement is split across ranks:
 *  POLYA_SHARD_TILES   output-tile sharding: every rank holds all blocks' X, Z^{-1} and
 *                      computes a cost-balanced range of G's work items completely; no
 *                      inter-GPU traffic (the default).
 *  POLYA_SHARD_BLOCKS  the paper's decentralised scheme: rank r owns a
 *                      cost-balanced contiguous range [b0, b1) of the Polya blocks and computes
 *                      the partial G^(r) = sum_{b in [b0,b1)} G^(b) over ALL entries; the partials
 *                      are summed by polya_reduce_G (NCCL ReduceScatter / AllReduce).
 *  POLYA_SHARD_CYCLIC  the distributed factorisation's layout:
 *                      rank r assembles the pair tiles (h, h') with h = r mod nranks -- the block
 *                      columns r, r + nranks, ... of the lower Cholesky factor -- completely, in
 *                      the PAIR_TILES layout in pair order; polya_ipm_step / polya_ipm_solve then
 *                      factor G across the ranks (NCCL broadcasts of each factored panel).  */
typedef enum { POLYA_SHARD_TILES = 0, POLYA_SHARD_BLOCKS = 1, POLYA_SHARD_CYCLIC = 2 } polya_shard;

/* Problem shape.  delta > 0 is the P-positivity margin of Eq. Cj ("a small
 * positive parameter"; R9 default 1e-3).  rank / nranks select
 * this context's share of the Schur complement (per `shard`, see polya_schur);
 * nranks = 1 for a single GPU. */
typedef struct {
  int32_t n, l, dp, da, d1, d2;
  double delta;
  int32_t rank, nranks;
  int32_t shard;     /* polya_shard */
} polya_config;

typedef struct {
  int64_t L0;        /* |W_dp|                        Eq. L0 */
  int64_t L;         /* |W_{dp+d1}|  P-blocks          Eq. L */
  int64_t M;         /* |W_{dp+da+d2}| Lyapunov blocks Eq. M */
  int64_t nblocks;   /* L + M                                                    */
  int64_t Ntil;      /* n(n+1)/2                                                 */
  int64_t K;         /* L0 * Ntil, dual dimension      Eq. K */
  int64_t nnz_beta;  /* #(h, P-block) with beta != 0 (h <= gamma)                */
  int64_t nnz_H;     /* #(h, Lyapunov block) with h + lambda <= gamma for some lambda */
  int64_t npairs;    /* #(h <= h') dual-row pairs = L0(L0+1)/2                   */
  int64_t pair0, pair1;   /* this rank's pairs [pair0, pair1) of the pair order   */
  int64_t item0, item1;   /* this rank's Schur work items [item0, item1)          */
  double useful_flops_schur;  /* W_G: algorithmic FP64 FLOPs of one polya_schur on
                                 this rank (upper triangle) */
  int64_t tiles_bytes;  /* bytes of G in POLYA_G_PAIR_TILES layout on this rank   */
  int64_t b0, b1;       /* this rank's Polya blocks [b0, b1) (all blocks with SHARD_TILES) */
  int64_t reduce_count; /* SHARD_BLOCKS: doubles each rank receives from polya_reduce_G /
                           polya_schur_reduce in the PAIR_TILES layout = groups * combine_tiles *
                           Ntil^2 (see combine_tiles); a whole partial-G buffer for polya_reduce_G
                           holds nranks*reduce_count doubles (zero tiles past npairs) */
  int64_t npairs_local; /* pair tiles held by this rank (PAIR_TILES layout: npairs_local tiles);
                           = pair1 - pair0 except with SHARD_CYCLIC (pairs not contiguous) */
  int64_t block_n;      /* order of every block of X, Z, C, B^T(y): cfg->n, or the generalised
                           form's N (polya_setup_general with nlmi > n) */
  int64_t combine_tiles; /* SHARD_BLOCKS: t = pair tiles per rank and tile group of the combine.
                           Group g = pair tiles [g*nranks*t, (g+1)*nranks*t) (pair order; zero tiles
                           past npairs); rank r receives the summed tiles g*nranks*t + r*t + j
                           (j < t) at Grecv + (g*t + j)*Ntil^2.  t is chosen so that a group is
                           about 2 GiB (at least one tile).  0 for the other shardings. */
} polya_dims;

/* Output layouts of the Schur complement G (symmetric K x K):
 *  POLYA_G_FULL       double[K][K] row-major.  Entries of this rank's work items
 *                     are written together with their mirror images (bitwise
 *                     symmetric); other entries are left untouched.
 *  POLYA_G_PAIR_TILES this rank's pair tiles p = pair0 .. pair1-1, each
 *                     double[Ntil][Ntil] row-major = G[h*Ntil.., h'*Ntil..] for the
 *                     p-th pair (h <= h') of the order (h ascending, h' ascending);
 *                     diagonal tiles (h = h') are stored full and symmetric.       */
typedef enum { POLYA_G_FULL = 0, POLYA_G_PAIR_TILES = 1 } polya_G_layout;

/* Algorithm 1 without materialising B_i: enumerates W_dp,
 * W_{dp+d1}, W_{dp+da+d2}; beta (Eq. beta, closed form multinomial(d1; gamma-h));
 * H (Eq. H, closed form sum_lambda multinomial(d2; gamma-h-lambda) A_lambda,
 * computed on the device); C (Eq. Cj); block descriptors; this rank's share.
 * A_host: double[f(l,da)][n][n], coefficient of alpha^lambda in W_da order; copied.
 * Synchronous.  Selects the current CUDA device at call time as the ctx's device.
 * Errors: EINVAL (n<1, l<1, dp<0, da<0, d1<0, d2<0, delta<=0, rank outside
 * [0,nranks), null pointers), EOVERFLOW, ENOMEM, ECUDA.  *out = NULL on error. */
polya_status polya_setup(const polya_config* cfg, const double* A_host, polya_ctx** out);

/* The generalised form (reading R18):
 *     P(alpha) > 0,   sum_i (At_i(alpha) P(alpha) Bt_i(alpha) + Bt_i(alpha)^T P(alpha) At_i(alpha)^T) < 0,
 * nlmi = N: the order of the LMI (0 or cfg->n: the square case, At_i, Bt_i n x n; N > n: At_i is
 * N x n, Bt_i n x N, R N x N -- e.g. the bounded-real lemma, N = n + m -- and every block of the SDP
 * is N x N, a P-block's n x n LMI in its top-left corner with C = -I on the rest; reading R19:
 * X, Z and B^T(y) stacks are then double[nblocks][N][N], see polya_dims.block_n).
 * Term i has At_i of degree deg_a[i] and Bt_i of degree
 * deg_b[i] with deg_a[i] + deg_b[i] = cfg->da for every i (homogenise first; EINVAL otherwise).
 * At: the concatenation over i of double[f(l,deg_a[i])][N][n] (coefficients in W_{deg_a[i]} order),
 * Bt of double[f(l,deg_b[i])][n][N]; both copied.  The continuous-time polya_setup is the case nterms = 1,
 * (A^T, 1, I, 0); discrete time A^T P A - P < 0 is [(A^T/2, 1, A, 1), (-I/2 per vertex, 1, I per
 * vertex, 1)].  R_host (nullable = 0): the constant term sum_i R_i(alpha), homogeneous of degree
 * dp + da, double[f(l,dp+da)][N][N] symmetric, W_{dp+da} order; it becomes C on the Lyapunov blocks,
 * C_{L+m} = sum_rho multinomial(d2; gamma_m - rho) R_rho (the dual constraint B^T(y) - C >= 0 is then
 * the LMI with "+ R < 0").  Lyapunov block gamma of the dual element (h, k) is
 *     -sum_{i,lambda,mu} multinomial(d2; gamma - h - lambda - mu) (At_{i,lambda} E_k Bt_{i,mu} + transpose);
 * every other entry point (apply, adjoint, Schur, IPM, solve, verdict, sharding) works unchanged
 * on the resulting context, except polya_get_H (EINVAL: no H table).  Errors as polya_setup. */
polya_status polya_setup_general(const polya_config* cfg, int32_t nlmi, int32_t nterms, const int32_t* deg_a,
                                 const int32_t* deg_b, const double* At_host, const double* Bt_host, const double* R_host,
                                 polya_ctx** out);

polya_status polya_dims_get(const polya_ctx* ctx, polya_dims* out);

/* Host-only planning (no CUDA call, no A needed: the sparsity of beta and H depends
 * only on the exponents): the dims this rank's polya_setup would report, including
 * its share [item0, item1) of the Schur work items (cost-balanced prefix split of
 * K_pair-weighted items across nranks).  Errors as polya_setup. */
polya_status polya_plan(const polya_config* cfg, polya_dims* out);

/* Exponent table `which` (0: W_dp, 1: W_{dp+d1}, 2: W_{dp+da+d2}, 3: W_da) as
 * int32[f(l,d)][l], in the R1 order.  Synchronous. */
polya_status polya_get_exponents(const polya_ctx* ctx, int which, int32_t* out_host);

/* beta as int64[L0][L] (zeros where h is not <= gamma).  Synchronous. */
polya_status polya_get_beta(const polya_ctx* ctx, int64_t* out_host);

/* H as double[L0][M][n][n] (zeros where structurally zero), copied back from the
 * device.  Synchronous. */
polya_status polya_get_H(const polya_ctx* ctx, double* out_host);

/* c_j with C_j = c_j I_n for the L P-blocks (Eq. Cj); C is 0 on
 * Lyapunov blocks.  Synchronous. */
polya_status polya_get_C(const polya_ctx* ctx, double* out_host);

/* Forward map B^T(y) = sum_i y_i B_i (Eq. AT), blockwise:
 * P-block j: sum_h beta_{h,j} V_h(y); Lyapunov block m: -(S + S^T), S = sum_h V_h(y) H_{h,m}.
 * y_dev: double[K]; blocks_dev: double[nblocks][n][n] (all blocks, written fully). */
polya_status polya_apply(polya_ctx* ctx, const double* y_dev, double* blocks_dev, void* stream);

/* Adjoint B(X)_i = sum_b tr(F_i^b X_b).  X_dev: double[nblocks][n][n]
 * (need not be symmetric; only its symmetric part matters); y_dev: double[K], overwritten. */
polya_status polya_adjoint(polya_ctx* ctx, const double* X_dev, double* y_dev, void* stream);

/* Schur complement matrix (Eq. T2; Case 1):
 *   G_{ij} = sum_b tr(F_i^b Z_b^{-1} F_j^b X_b)
 * X_dev, Zinv_dev: double[nblocks][n][n]; both triangles are read and the
 * expansion assumes exact symmetry (callers symmetrise).  G_dev per layout.
 * SHARD_TILES: this rank computes its work items [item0, item1) completely (inputs
 * replicated on every rank, no inter-GPU traffic).  SHARD_BLOCKS: this rank computes
 * every entry of the partial sum over its blocks [b0, b1) (to be summed by
 * polya_reduce_G); X_dev / Zinv_dev still hold all blocks, only [b0, b1) are read by
 * the assembly.  Uses the rank-structured expansion of DESIGN.md ("4-term raw GEMM +
 * fold"), never the dense B_i.                                                   */
polya_status polya_schur(polya_ctx* ctx, const double* X_dev, const double* Zinv_dev,
                         double* G_dev, int layout, void* stream);

/* The two halves of polya_schur, for callers that stream G out while it is assembled:
 * polya_schur_prepare pads X, Z^{-1} and runs the SCM precompute of this rank (U, V, Q, R; kernels K3 / K3b:
 *   U^T, V^T are stored as transposes, which relies on the symmetry of X and Z^{-1});
 * polya_schur_assemble then assembles this rank's local pairs [pair_begin, pair_end), 0-based among
 * its npairs_local local pairs (polya_dims; = pair0 .. pair1-1 except with SHARD_CYCLIC, whose local
 * pairs are the pair rows h = rank mod nranks); G_dev is the same buffer / layout as for polya_schur
 * and only those pairs' entries are written.  polya_schur = prepare + assemble(0, npairs_local).
 * Inputs must not change between the prepare and the assembles.  Stream-ordered; the assembles of
 * one context share its work counter, so they must be serialised on one stream (no two in flight
 * on different streams).  Errors: EINVAL (bad range / layout), ECUDA.                           */
polya_status polya_schur_prepare(polya_ctx* ctx, const double* X_dev, const double* Zinv_dev, void* stream);
polya_status polya_schur_assemble(polya_ctx* ctx, double* G_dev, int layout, int64_t pair_begin, int64_t pair_end,
                                  void* stream);

/* One predictor-corrector iteration of Algorithm 2 with the
 * readings R3-R6.  nranks must be 1, or the context SHARD_CYCLIC: then every rank calls it
 * (collective) with identical replicated X, Z, y, assembles its pair tiles and the K x K
 * factorisation and solves run distributed (NCCL, polya_nccl_init first); the
 * ranks' X, Z, y stay bitwise identical.  State lives on the device:
 * X, Z: double[nblocks][block_n][block_n] (symmetric PD), y: double[K]; updated in place.
 * mu is the barrier parameter of the previous step (Eq. mu).
 * The K x K factorisation uses cuSOLVER dpotrf/dpotrs (timed separately in stats); if G is not
 * numerically positive definite it is re-assembled and factorised once more as G + eps I,
 * eps = 1e-12 tr(G) / K, before ENOTPD is returned.
 * Synchronous (returns after the step).  Errors: EINVAL (several ranks without SHARD_CYCLIC,
 * block_n > 168), ENOTPD, ESTEP, ENCCL, ECUDA, ENOMEM.   */
typedef struct { double* X; double* Z; double* y; double mu; int32_t iter; } polya_ipm_state;
typedef struct {
  double gap;      /* |a^T y - tr(C X)| after the step (stopping rule) */
  double mu;       /* new barrier parameter (1/3) sum tr(Z X)  (R4)                  */
  double tp, td;   /* primal / dual step sizes (R5)                                  */
  double phi, psi; /* primal cost tr(C X), dual cost a^T y                            */
  float ms_schur, ms_factor, ms_other;
  int32_t reg_retries;   /* 1 if G needed the regularised retry G + 1e-12 tr(G)/K I */
} polya_ipm_stats;
polya_status polya_ipm_step(polya_ctx* ctx, polya_ipm_state* st, polya_ipm_stats* stats, void* stream);

/* Factorisation of the K x K Schur complement inside polya_ipm_step (the root's Cholesky, Case 2,
 * PAPER.md:913-916): mode 0 = automatic (dense when K^2 doubles fit in 45 % of device memory,
 * else tiled), 1 = dense (G in POLYA_G_FULL layout, cuSOLVER dpotrf/dpotrs), 2 = tiled (G in
 * POLYA_G_PAIR_TILES layout -- half the memory -- right-looking block Cholesky: cuSOLVER dpotrf on
 * the diagonal tiles, cuBLAS dtrsm/dsyrk/dgemm on the others, blocked triangular solves).
 * Applies from the next polya_ipm_step.  Errors: EINVAL.                                     */
polya_status polya_set_factorization(polya_ctx* ctx, int mode);

/* Phase timing of polya_schur with CUDA events recorded on the call's stream:
 * enable != 0 turns the events on for subsequent calls; polya_get_timing waits for the
 * last call's events and returns the milliseconds of the SCM precompute (padding, U, V,
 * Q, R; kernel K3) and of the assembly kernel K4. */
polya_status polya_set_timing(polya_ctx* ctx, int enable);
polya_status polya_get_timing(polya_ctx* ctx, float* ms_pre, float* ms_assemble);

/* Multi-GPU combine of the block-sharded Schur complement (SHARD_BLOCKS; PAPER.md:749,
 * 755-778: the root's gather of the workers' partial sums, here one NCCL collective over
 * NVLink).  polya_nccl_unique_id (rank 0) fills a 128-byte id that the caller distributes;
 * polya_nccl_init (every rank, collectively) creates the context's communicator with
 * cfg.rank / cfg.nranks on the context's device.
 * polya_reduce_G sums the ranks' partial G^(r) on `stream`:
 *   layout PAIR_TILES: one ncclReduceScatter per tile group (polya_dims.combine_tiles) of the
 *     tile buffer Gpart_dev (nranks*reduce_count doubles, as written by polya_schur + zero tiles
 *     past npairs) into Grecv_dev (reduce_count doubles): this rank's whole summed tiles, in the
 *     group order of polya_dims.combine_tiles;
 *   layout FULL: ncclAllReduce of the K x K matrix (Grecv_dev may equal Gpart_dev).
 * Errors: EINVAL (not SHARD_BLOCKS, null pointers), ENCCL (no communicator, NCCL failure).
 *
 * polya_schur_reduce = polya_schur + polya_reduce_G(PAIR_TILES) pipelined: the
 * precompute, then per tile group the K4 assembly of the group into one of two library-owned
 * partial slots (2 x nranks*t tiles -- not the whole partial G) on `stream`, and the group's
 * ncclReduceScatter on the context's own comm stream, ordered by events: the reduction of group g
 * overlaps the assembly of group g+1.  Grecv_dev: reduce_count doubles, the same layout and values
 * (bit for bit) as polya_schur + polya_reduce_G.  On return `stream` is ordered after every
 * reduce-scatter.  One rank without a communicator: the reduce-scatter is a device copy.
 * Assemblies on one context must be serialised on one stream (they share the work counter).
 * Errors: EINVAL, ENCCL (several ranks without polya_nccl_init, NCCL failure), ENOMEM, ECUDA.
 * polya_get_combine_timing: with polya_set_timing on, the milliseconds between the end of the last
 * K4 launch and the end of the last reduce-scatter (the combine time NOT hidden under the assembly). */
polya_status polya_nccl_unique_id(char out_id[128]);
polya_status polya_nccl_init(polya_ctx* ctx, const char id[128]);
polya_status polya_reduce_G(polya_ctx* ctx, const double* Gpart_dev, double* Grecv_dev, int layout, void* stream);
polya_status polya_schur_reduce(polya_ctx* ctx, const double* X_dev, const double* Zinv_dev, double* Grecv_dev,
                                void* stream);
polya_status polya_get_combine_timing(polya_ctx* ctx, float* ms_exposed);
/* Fused P2P combine (SHARD_BLOCKS; the compute step and the collective in one kernel): the assembly
 * kernel K4 stores every tile of this rank's partial G straight into the tile's owner's receive slot
 * over NVLink peer memory (the owner / position of a tile as in polya_dims.combine_tiles), then each
 * owner sums its nranks slots in rank order into Grecv (same layout as polya_reduce_G) -- no separate
 * reduce-scatter, the transfer runs inside the assembly tile by tile.
 * polya_p2p_export: allocates this rank's receive slots (nranks x own tiles + flags, library-owned)
 *   and writes its 64-byte CUDA IPC handle; the caller exchanges the handles (e.g. all_gather).
 * polya_p2p_import: handles = nranks x 64 bytes in rank order (this rank's entry ignored); opens the
 *   peers' slots (peer access) and builds the destination tables.
 * polya_p2p_loopback: test hook -- the nranks contexts of one process on one device wired directly.
 * polya_schur_reduce_p2p: phases bit 1 = precompute + assembly into the owners' slots + a system-scope
 *   release of this rank's flag in every owner; bit 2 = wait for every source's flag, the sum, then an
 *   acknowledgement to every source.  From its second call on, bit 1 first waits for every owner's
 *   acknowledgement of the previous call, so a fast rank never overwrites a slot its owner is still
 *   summing.  A rank calls it with phases = 3; the loopback test runs bit 1 for every context, then
 *   bit 2 (no kernel waits on one launched after it on the same device).  Grecv: reduce_count doubles.
 *   A wait that is not satisfied within 60 s traps (the call's stream then reports a CUDA error)
 *   instead of hanging on a peer that died.
 * Errors: EINVAL (not SHARD_BLOCKS, more than 32 ranks, not imported, null pointers), ENOMEM, ECUDA. */
polya_status polya_p2p_export(polya_ctx* ctx, char handle_out[64]);
polya_status polya_p2p_import(polya_ctx* ctx, const char* handles);
polya_status polya_p2p_loopback(polya_ctx** ctxs, int32_t nranks);
polya_status polya_schur_reduce_p2p(polya_ctx* ctx, const double* X_dev, const double* Zinv_dev, double* Grecv_dev,
                                    int phases, void* stream);
/* polya_set_combine_tiles: override t (polya_dims.combine_tiles; 0 = automatic ~2 GiB groups), e.g.
 * for a finer overlap; all ranks must use the same t.  Frees the combine's slots (a P2P combine must
 * be exported / imported again).  SHARD_BLOCKS only.  Errors: EINVAL. */
polya_status polya_set_combine_tiles(polya_ctx* ctx, int64_t tiles);

/* ---- beyond one iteration: non-homogeneous systems, parameter boxes, solve, verdict ------------
 * (used by the bisection drivers of the paper's Examples 1-2.)
 *
 * polya_homogenize: the procedure of PAPER.md:113-132.  A(alpha) = sum_t coeffs_t alpha^{exps_t}
 * (exps: int32[nterms][l], coeffs: double[nterms][n][n], host) of degree d_a = max_t |exps_t| is
 * replaced by B(alpha) = sum_t coeffs_t (sum_j alpha_j)^{d_a - |exps_t|} alpha^{exps_t}, equal to A on
 * the simplex and homogeneous; out = B's coefficients double[f(l,d_a)][n][n] in W_{d_a} order (R1).
 * With out == NULL only *da_out is written (size query).  Host-only, synchronous.
 *
 * polya_simplex_map: A'(alpha) = A(g(alpha)) for the affine simplex maps of Examples 1-2
 * (reading R17): g_i(alpha) = scale_i alpha_i + shift_i (sum_j alpha_j), which
 * maps Delta_l affinely onto a box-constrained simplex (Example 1: scale = 2|rho|, shift = -|rho|; Example 2: scale = 1 - L, shift = L).  A_in, A_out: double[f(l,d)][n][n] in W_d
 * order (homogeneous of degree d).  Host-only, synchronous.  Errors: EINVAL, EOVERFLOW.      */
polya_status polya_homogenize(int32_t l, int32_t n, int32_t nterms, const int32_t* exps, const double* coeffs,
                              int32_t* da_out, double* out);
polya_status polya_simplex_map(int32_t l, int32_t d, int32_t n, const double* scale, const double* shift,
                               const double* A_in, double* A_out);

/* polya_ipm_solve: Algorithm 2 iterated (polya_ipm_step) until the stopping rule gap <= eps
 * with primal residual ||B(X) - a||_2 <= tol, or maxit iterations.  init != 0
 * starts from Algorithm 2's initial point X = Z = I, y = 0.  The outcome is a
 * result, not an error: res->converged = 1 iff the rule was met with every Z block positive
 * definite (reading R10); otherwise res->status says why (ENOTPD: a block or G lost definiteness,
 * ESTEP: no admissible step, EDIVERGED: the iterates left POLYA_DIVERGENCE_BOUND, EMAXIT).  The
 * return value reports misuse and failures: EINVAL, ENOMEM, ECUDA and ENCCL from any iteration are
 * returned as such (never folded into res->status).
 * Ranks as polya_ipm_step (collective with SHARD_CYCLIC).  Synchronous.                     */
typedef struct {
  double eps, tol;
  int32_t maxit, init;
  polya_ipm_stats* history;   /* optional host array of maxit entries: the stats of every iteration
                                 (the iteration log of S:448); NULL = none */
} polya_solve_opts;
typedef struct {
  int32_t converged, iterations, status;
  double gap, pinf, mu;
  float ms_schur, ms_factor, ms_other;   /* summed over the iterations */
} polya_solve_result;
polya_status polya_ipm_solve(polya_ctx* ctx, polya_ipm_state* st, const polya_solve_opts* opt,
                             polya_solve_result* res, void* stream);

/* polya_verdict: the grid check of the certificate (Theorem 1):
 * with P(alpha) = sum_h alpha^h V_h(y) (reading R7; y_dev: double[K] on the device) and A(alpha) the
 * set-up's A, counts the points alpha = pts_host[p] (double[npts][l], host, points of the simplex)
 * where P(alpha) > 0 or -(A^T P + P A)(alpha) > 0 fails a Cholesky test, into *nfail_out
 * (generalised form: -sum_i (At_i P Bt_i + transpose)(alpha) > 0 instead).
 * One CTA per point on the device (P(alpha), A(alpha) in a global scratch, each Cholesky test on
 * a shared-memory copy); block order <= 168 (the IPM's limit).  Synchronous.                    */
polya_status polya_verdict(polya_ctx* ctx, const double* y_dev, int32_t npts, const double* pts_host,
                           int32_t* nfail_out, void* stream);

/* Test hook of the distributed factorisation (SHARD_CYCLIC): ctxs[r] (r < nranks) are
 * the nranks contexts of one problem, all in this process on one device, ctxs[r] with rank r and
 * shard POLYA_SHARD_CYCLIC; G_local[r] is rank r's POLYA_G_PAIR_TILES output of polya_schur,
 * overwritten by its tiles of the Cholesky factor.  x (double[K], device) is overwritten by
 * G^{-1} x.  Runs the same per-step functions as the NCCL path of polya_ipm_step, the ranks one
 * after another, with device copies in place of the broadcasts.  Synchronous.
 * Errors: EINVAL (inconsistent contexts), ENOTPD (G not positive definite), ECUDA. */
polya_status polya_factor_solve_loopback(polya_ctx** ctxs, int32_t nranks, double* const* G_local, double* x_dev,
                                         void* stream);

/* Test hook of the IPM's blockwise kernels (reading R5): for nb blocks of order n
 * (1 <= n <= 168; device stacks of nb row-major n x n doubles, caller-owned) computes W_b = S_b^{-1}
 * (k_block_inv), Linv_b = L_b^{-1} with S_b = L_b L_b^T (lower, zeros above), M_b = L_b^{-1} dS_b
 * L_b^{-T} and t_b = min(1/0.98, 1 / max(0, -lambda_min(sym M_b))) (k_block_lmin; -1 when S_b is not
 * positive definite), and *fail (int32, device) = 1 if some S_b is not positive definite.
 * Synchronous.  Errors: EINVAL (n out of range, null pointers), ECUDA. */
polya_status polya_block_kernels_test(int32_t n, int64_t nb, const double* S_dev, const double* dS_dev, double* W_dev,
                                      double* Linv_dev, double* M_dev, double* t_dev, int32_t* fail_dev, void* stream);

/* Surfaces asynchronous errors (device synchronise + last-error check). */
polya_status polya_sync(polya_ctx* ctx);
const char* polya_strerror(polya_status s);
const char* polya_last_error(const polya_ctx* ctx);
/* Number of kernel launches this context has issued so far (for bench.py's
 * gpu_launches count). */
int64_t polya_launch_count(const polya_ctx* ctx);
void polya_destroy(polya_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* POLYA_H_ */
