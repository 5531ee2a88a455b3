// polya_internal.h -- context layout and kernel launchers shared by polya_host.cpp and the .cu files.
// Not part of the ABI (include/polya.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/polya.h"

namespace polya {

constexpr int kChunk = 8;  // index chunk q of the Schur "class blocks" (kernel K4)
constexpr int kKStage = 8;  // k terms per K4 pipeline stage; pair k-lists are zero-padded to it

// One term of a batched GEMM item: C += alpha * A[a_id] * op(B[b_id]), all np x np arena matrices.
struct GemmTerm {
  int32_t a_id, b_id;
  int32_t transB;
  int32_t pad_;
  double alpha;
};
// One output matrix of a batched GEMM: C[c_id] = sum_{t in [tbeg,tend)} terms[t]; if ct_id >= 0 its
// transpose is also stored to C[ct_id].
struct GemmItem {
  int32_t c_id, tbeg, tend, ct_id;
};

// Row-gathered GEMM (kernel K3b, the SCM precompute of the standard form with np <= 128): a group shares
// one right operand op(B[b_id]) and stacks the rows of its entries' A matrices; each entry's rows of
// A op(B) go to C[c_id] (and, if ct_id >= 0, transposed to C[ct_id]).  A tile = 64 stacked rows of a group.
struct RgGroup {
  int32_t b_id, transB, ebeg, eend;
};
struct RgEnt {
  int32_t a_id, c_id, ct_id, pad_;
};
struct RgTile {
  int32_t group, r0;
};

// dst = sum_terms w * coef[src] (or its transpose): the generalised form's A_t, A_t^T, B_t (set-up).
struct WsumItem {
  int32_t dst, beg, end, trans;
};
struct WsumTerm {
  int32_t src, pad_;
  double w;
};

// Device-side tables of the Schur assembly (kernel K4).
struct SchurTables {
  int32_t* pair_h = nullptr;      // [npairs_local]      h  (row block of the pair)
  int32_t* pair_h2 = nullptr;     // [npairs_local]      h' (column block), h <= h'
  int64_t* pair_kbeg = nullptr;   // [npairs_local + 1]  k-entry range of each pair
  int64_t* pair_item = nullptr;   // [npairs_local + 1]  global work-item prefix (offset item_base)
  int2* kdesc = nullptr;          // [nk] arena matrix ids (L_k, R_k) of the pair k-lists for K4
  int32_t* cls_a = nullptr;       // [ncls] chunk index i of class (i <= j)
  int32_t* cls_b = nullptr;       // [ncls] chunk index j
  unsigned long long* counter = nullptr;  // dynamic work counter
  int32_t* sched_pl = nullptr;    // [nsched] schedule of the rank's whole share: pairs by decreasing k-list
  int64_t* sched_lo = nullptr;    // [nsched] first item of the pair in [item0, item1)
  int64_t* sched_prefix = nullptr;  // [nsched + 1] pulled-index prefix
  int64_t nsched = 0;
};

struct Ctx {
  polya_config cfg{};
  int device = 0;
  int64_t n = 0, l = 0, L0 = 0, L = 0, M = 0, nb = 0, Ntil = 0, K = 0, nA = 0;
  int64_t nbas = 0;      // order of P (the basis E_k); n is the order of every block (= nbas, or the
                         // generalised form's N > nbas, reading R19)
  int64_t np = 0;        // padded matrix dimension (multiple of kChunk)
  int64_t r = 0;         // number of index chunks = np / kChunk
  int64_t ncls = 0;      // r (r+1) / 2 unordered chunk classes
  std::vector<int32_t> Wp, WL, WM, Wa;  // exponent tables, row-major [count][l]
  std::vector<int64_t> beta;           // [L0][L]
  std::vector<double> c;               // [L]
  std::vector<int32_t> Hh, Hm;         // nonzero H entries t -> (h, m), m-major
  std::vector<int32_t> Hidx;           // [L0][M] -> first t or -1
  std::vector<int32_t> Hcnt;           // [L0][M] -> number of terms t of (h, m): 0/1, or any (generalised)
  // generalised form (polya_setup_general, reading R18): term t = (A_t, B_t), F = -sum_t (A_t E B_t + B_t^T E A_t^T)
  bool gen = false;
  int64_t ncoef = 0;                   // coefficient matrices of all At_i, Bt_i (n x n each)
  std::vector<int32_t> gp_da, gp_db, gp_aoff, gp_boff;  // per input term i: degrees, coefficient offsets
  std::vector<int32_t> coef_exp;       // [ncoef][l] exponent of each coefficient matrix
  double* d_coef = nullptr;            // [ncoef][n][n] (the constant term R's coefficients last)
  int64_t r_off = 0, r_cnt = 0;        // R's coefficients in d_coef (r_cnt = 0: no constant term)
  double* d_CL = nullptr;              // [M][n][n] C on the Lyapunov blocks (from R), or null
  WsumItem* d_ws_items = nullptr; WsumTerm* d_ws_terms = nullptr; int64_t n_ws = 0;
  std::vector<double> Hw;              // [nnzH][nA] integer weights multinomial(d2; gamma-h-lambda)
  // pairs and work items
  int64_t npairs = 0, pair0 = 0, pair1 = 0;
  int64_t items_total = 0, item0 = 0, item1 = 0;
  int64_t b0 = 0, b1 = 0;  // this rank's Polya blocks (SHARD_BLOCKS; all blocks otherwise)
  void* nccl = nullptr;    // ncclComm_t of polya_nccl_init (SHARD_BLOCKS combine, SHARD_CYCLIC factorisation)
  void* loop = nullptr;    // LoopGroup of polya_factor_solve_loopback (in place of NCCL, tests)
  std::vector<int64_t> pair_item_global;  // [npairs + 1]
  std::vector<int64_t> local_pairs;       // this rank's pairs (global indices, ascending)
  std::vector<int64_t> local_item;        // [npairs_local + 1] item prefix of the local pairs (kernel numbering)
  std::vector<int32_t> pair_local;        // [npairs] local index of a pair, or -1
  double useful_flops_total = 0, useful_flops_rank = 0;
  // arena (np x np matrices)
  int64_t mstride = 0, nmats = 0;
  int64_t id_Ut = 0, id_Vt = 0, id_Zero = 0, id_Xb = 0, id_Wb = 0;
  int32_t* d_sc_dst = nullptr; int32_t* d_sc_src = nullptr; double* d_sc_w = nullptr; int64_t n_sc = 0;
  int64_t id_B = 0, id_Abar = 0, id_XA = 0, id_VB = 0;   // generalised form only
  int64_t id_X = 0, id_W = 0, id_H = 0, id_U = 0, id_V = 0, id_Q = 0, id_R = 0, id_Xt = 0, id_T = 0,
          id_Vy = 0, id_S = 0;
  int64_t nQR = 0;
  double* arena = nullptr;
  double* dA = nullptr;
  double* dHw = nullptr;
  // batched gemm descriptors
  GemmItem* d_items_UV = nullptr; GemmTerm* d_terms_UV = nullptr; int64_t n_items_UV = 0;
  GemmItem* d_items_QR = nullptr; GemmTerm* d_terms_QR = nullptr; int64_t n_items_QR = 0;
  // K3b row-gathered launches (standard form, np <= 128): [0] U, V (+ U^T, V^T), [1] Q, R (op(B) = H^T),
  // [2] the adjoint's T_t = H_t sym(X_m)
  static constexpr int kRgPhases = 3;
  RgGroup* d_rg_grp[kRgPhases] = {}; RgEnt* d_rg_ent[kRgPhases] = {};
  RgTile* d_rg_tile[kRgPhases] = {}; int64_t n_rg_tile[kRgPhases] = {};
  bool rg = false;
  GemmItem* d_items_T = nullptr; GemmTerm* d_terms_T = nullptr; int64_t n_items_T = 0;
  GemmItem* d_items_S = nullptr; GemmTerm* d_terms_S = nullptr; int64_t n_items_S = 0;
  GemmItem* d_items_T0 = nullptr; GemmTerm* d_terms_T0 = nullptr; int64_t n_items_T0 = 0;  // generalised: XA_t
  GemmItem* d_items_S0 = nullptr; GemmTerm* d_terms_S0 = nullptr; int64_t n_items_S0 = 0;  // generalised: VB_t
  // apply / adjoint tables
  int32_t* d_bP_beg = nullptr;   // [L+1]  P-block active-h ranges
  int32_t* d_bP_h = nullptr;     // [nnz_beta]
  double* d_bP_w = nullptr;      // [nnz_beta] beta
  int32_t* d_hP_beg = nullptr;   // [L0+1]  per h: P-blocks with beta != 0
  int32_t* d_hP_j = nullptr;
  double* d_hP_w = nullptr;
  int32_t* d_hL_beg = nullptr;   // [L0+1]  per h: nonzero H entries t (m ascending)
  int32_t* d_hL_t = nullptr;
  int32_t* d_hL_m = nullptr;
  int64_t nnz_beta = 0;
  SchurTables st;
  int64_t nk_local = 0, npairs_local = 0;
  // IPM workspace (allocated lazily)
  void* ipm = nullptr;
  bool timing = false;
  int fact_mode = 0;     // polya_set_factorization: 0 auto, 1 dense K x K, 2 tiled (pair tiles)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // schur: start, after precompute, after K4, after combine
  // pipelined block-sharded combine (polya_schur_reduce, combine.cpp): two partial-tile slots,
  // a dedicated comm stream, slot events (allocated on first use)
  double* comb_slot[2] = {nullptr, nullptr};
  int64_t comb_t = 0;                  // polya_set_combine_tiles (0: automatic, ~2 GiB groups)
  // fused P2P combine (polya_p2p_*): this rank's receive slots [nranks][own tiles] + a flag block
  // (ready[r] at int 0.., ack[o] at int kP2pAck..), the per-pair destination table (a slot in the
  // owner's buffer), the owners' ready-flag addresses for this rank, the sources' ack-flag addresses
  double* p2p_buf = nullptr;
  int64_t p2p_own = 0;                 // tiles each rank owns (groups x combine_tiles, padding included)
  double** d_tile_ptr = nullptr;
  int** d_flag_ptr = nullptr;
  int** d_ack_ptr = nullptr;
  std::vector<void*> p2p_opened;       // peers' buffers opened by IPC (closed at destroy)
  int p2p_epoch = 0;
  bool p2p_ready = false;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comb_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // assembled[2], reduced[2]
  std::string last_error;
  int64_t launches = 0;
  int64_t k4_ctas = 0;   // resident K4 CTAs on the device (computed at the first assembly)
};

// Tile groups of the block-sharded combine (SHARD_BLOCKS): group g holds pair tiles
// [g N t, (g+1) N t) (N = nranks, zero tiles past npairs); its reduce-scatter hands rank r the t tiles
// g N t + r t .. + t - 1, stored at Grecv + g t Ntil^2.  t = tiles per rank and group, sized so that
// a group is ~2 GiB (at least one tile): the granularity of the overlap and of the partial buffers.
inline void combine_shape(const Ctx& c, int64_t* t_out, int64_t* groups_out) {
  const int64_t N = c.cfg.nranks, tile_bytes = c.Ntil * c.Ntil * (int64_t)sizeof(double);
  int64_t t = c.comb_t > 0 ? c.comb_t : std::max<int64_t>(1, ((int64_t)2 << 30) / std::max<int64_t>(1, N * tile_bytes));
  t = std::min<int64_t>(t, std::max<int64_t>(1, (c.npairs + N - 1) / N));
  *t_out = t;
  *groups_out = (c.npairs + N * t - 1) / (N * t);
}
void combine_free(Ctx& c);

// ---- kernel launchers (kernels.cu / schur.cu) -------------------------------------------------
cudaError_t launch_setup_H(Ctx& c, cudaStream_t s);
cudaError_t launch_wsum(Ctx& c, cudaStream_t s);
cudaError_t launch_pad_copy(Ctx& c, const double* src, int64_t id0, int64_t count, int symmetrize,
                            cudaStream_t s);
cudaError_t launch_scale_copy(Ctx& c, cudaStream_t s);
cudaError_t launch_gemm(Ctx& c, const GemmItem* items, const GemmTerm* terms, int64_t nitems,
                        cudaStream_t s);
cudaError_t launch_rgemm(Ctx& c, int phase, cudaStream_t s);
cudaError_t launch_vmap(Ctx& c, const double* y, cudaStream_t s);
cudaError_t launch_apply_out(Ctx& c, const double* y, double* out, cudaStream_t s);
cudaError_t launch_adjoint_reduce(Ctx& c, double* y, cudaStream_t s);
cudaError_t launch_schur(Ctx& c, double* G, int layout, int64_t item0, int64_t item1, cudaStream_t s,
                         double* const* tile_ptr = nullptr);
// the P2P combine (kernels.cu): signal the owners, wait for every source, sum the slots in rank order
constexpr int kP2pAck = 32;           // ints: the flag block holds ready[<= 32] then ack[<= 32]
cudaError_t launch_p2p_signal(int* const* flag_ptrs, int n, int epoch, cudaStream_t s);
cudaError_t launch_p2p_wait(const int* flags, int n, int epoch, cudaStream_t s);
cudaError_t launch_p2p_sum(const double* slots, int n, int64_t count, double* out, cudaStream_t s);
// collectives of the distributed factorisation (combine.cpp; NCCL, or the loopback group of
// polya_factor_solve_loopback; no-ops with one rank)
struct LoopGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  int64_t gen = 0;
  bool abort = false;
  std::vector<const void*> ptr;            // each rank's buffer of the current collective
  std::vector<std::vector<double>> host;   // all-reduce staging
};
bool loop_barrier(LoopGroup* g);
void loop_abort(LoopGroup* g);
cudaError_t comm_bcast(Ctx& c, void* buf, size_t count, bool is_int, int root, cudaStream_t s);
cudaError_t comm_allreduce_sum(Ctx& c, double* buf, size_t count, cudaStream_t s);
cudaError_t comm_allreduce_max(Ctx& c, double* buf, size_t count, cudaStream_t s);
cudaError_t comm_bcast_tiles(Ctx& c, double* buf, size_t count, int64_t ntiles, cudaStream_t s);

}  // namespace polya

struct polya_ctx {
  polya::Ctx c;
};
