// combine.cpp -- multi-GPU combine of the block-sharded Schur complement (row a9 of SURVEY 8(a)).
//
// With POLYA_SHARD_BLOCKS every rank owns a contiguous, cost-balanced range of the Polya blocks and
// assembles the partial sum G^(r) = sum_{b in [b0,b1)} G^(b) over all entries -- the paper's
// decentralised structure -- and the partials are summed over NVLink with
// one NCCL collective instead of the paper's root gather.
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "polya_internal.h"

using namespace polya;

namespace {
polya_status nccl_fail(polya_ctx* ctx, const char* what, ncclResult_t r) {
  if (ctx) ctx->c.last_error = std::string(what) + ": " + ncclGetErrorString(r);
  return POLYA_ENCCL;
}
}  // namespace

extern "C" polya_status polya_nccl_unique_id(char out_id[128]) {
  if (!out_id) return POLYA_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return POLYA_ENCCL;
  std::memcpy(out_id, &id, sizeof(id));
  return POLYA_OK;
}

extern "C" polya_status polya_nccl_init(polya_ctx* ctx, const char id[128]) {
  if (!ctx || !id) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.nccl) return POLYA_OK;
  if (cudaSetDevice(c.device) != cudaSuccess) {
    c.last_error = "cudaSetDevice failed";
    return POLYA_ECUDA;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, c.cfg.nranks, uid, c.cfg.rank);
  if (r != ncclSuccess) return nccl_fail(ctx, "ncclCommInitRank", r);
  c.nccl = comm;
  return POLYA_OK;
}

extern "C" polya_status polya_reduce_G(polya_ctx* ctx, const double* Gpart, double* Grecv, int layout, void* stream) {
  if (!ctx || !Gpart || !Grecv) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.cfg.shard != POLYA_SHARD_BLOCKS) {
    c.last_error = "polya_reduce_G needs SHARD_BLOCKS";
    return POLYA_EINVAL;
  }
  if (!c.nccl) {
    c.last_error = "polya_reduce_G before polya_nccl_init";
    return POLYA_ENCCL;
  }
  ncclComm_t comm = (ncclComm_t)c.nccl;
  cudaStream_t s = (cudaStream_t)stream;
  ncclResult_t r;
  if (layout == POLYA_G_PAIR_TILES) {   // one reduce-scatter per tile group (combine_shape), fused
    int64_t t = 0, groups = 0;
    combine_shape(c, &t, &groups);
    const int64_t NN = c.Ntil * c.Ntil, N = c.cfg.nranks;
    r = ncclGroupStart();
    for (int64_t g = 0; g < groups && r == ncclSuccess; ++g)
      r = ncclReduceScatter(Gpart + g * N * t * NN, Grecv + g * t * NN, (size_t)(t * NN), ncclFloat64, ncclSum, comm, s);
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
  } else if (layout == POLYA_G_FULL) {
    r = ncclAllReduce(Gpart, Grecv, (size_t)(c.K * c.K), ncclFloat64, ncclSum, comm, s);
  } else {
    return POLYA_EINVAL;
  }
  if (r != ncclSuccess) return nccl_fail(ctx, "NCCL collective", r);
  return POLYA_OK;
}

// The pipelined block-sharded Schur complement: the rank's partial G is assembled one
// tile group at a time into one of two ping-pong slots on `stream`, and each group's reduce-scatter
// runs on the context's comm stream as soon as its K4 launch has finished (event), overlapping the
// assembly of the next group; a slot is reused only after its previous reduce-scatter has read it.
// With one rank and no communicator the "reduce-scatter" is the identity (a device copy).
extern "C" polya_status polya_schur_reduce(polya_ctx* ctx, const double* X, const double* Zinv, double* Grecv,
                                           void* stream) {
  if (!ctx || !X || !Zinv || !Grecv) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.cfg.shard != POLYA_SHARD_BLOCKS) {
    c.last_error = "polya_schur_reduce needs SHARD_BLOCKS";
    return POLYA_EINVAL;
  }
  if (!c.nccl && c.cfg.nranks > 1) {
    c.last_error = "polya_schur_reduce before polya_nccl_init";
    return POLYA_ENCCL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t t = 0, groups = 0;
  combine_shape(c, &t, &groups);
  const int64_t NN = c.Ntil * c.Ntil, N = c.cfg.nranks, gt = N * t;   // tiles per group
  auto cuda = [&](cudaError_t e) {
    if (e != cudaSuccess) {
      c.last_error = std::string("polya_schur_reduce: ") + cudaGetErrorString(e);
      return false;
    }
    return true;
  };
  if (!c.comm_stream) {
    if (!cuda(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking))) return POLYA_ECUDA;
    for (auto& e : c.comb_ev)
      if (!cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming))) return POLYA_ECUDA;
  }
  for (int q = 0; q < 2; ++q)
    if (!c.comb_slot[q]) {
      cudaError_t e = cudaMalloc(&c.comb_slot[q], (size_t)(gt * NN) * sizeof(double));
      if (e == cudaErrorMemoryAllocation) {
        c.last_error = "polya_schur_reduce: partial-tile slots";
        return POLYA_ENOMEM;
      }
      if (!cuda(e)) return POLYA_ECUDA;
    }
  polya_status st = polya_schur_prepare(ctx, X, Zinv, stream);
  if (st != POLYA_OK) return st;
  for (int64_t g = 0; g < groups; ++g) {
    const int q = (int)(g & 1);
    double* slot = c.comb_slot[q];
    const int64_t p0 = g * gt, p1 = std::min(c.npairs, p0 + gt);
    if (g >= 2 && !cuda(cudaStreamWaitEvent(s, c.comb_ev[2 + q], 0))) return POLYA_ECUDA;   // slot read
    if (p1 - p0 < gt && !cuda(cudaMemsetAsync(slot + (p1 - p0) * NN, 0, (size_t)((gt - (p1 - p0)) * NN) * sizeof(double), s)))
      return POLYA_ECUDA;   // zero tiles past npairs in the last group
    // K4 writes pair p's tile at G + p Ntil^2: shift the base so that pair p0 lands at the slot start
    const int64_t i0 = std::max(c.item0, c.local_item[p0]), i1 = std::min(c.item1, c.local_item[p1]);
    if (!cuda(launch_schur(c, slot - p0 * NN, POLYA_G_PAIR_TILES, i0, i1, s))) return POLYA_ECUDA;
    if (!cuda(cudaEventRecord(c.comb_ev[q], s))) return POLYA_ECUDA;
    if (!cuda(cudaStreamWaitEvent(c.comm_stream, c.comb_ev[q], 0))) return POLYA_ECUDA;
    if (c.nccl) {
      ncclResult_t r = ncclReduceScatter(slot, Grecv + g * t * NN, (size_t)(t * NN), ncclFloat64, ncclSum,
                                         (ncclComm_t)c.nccl, c.comm_stream);
      if (r != ncclSuccess) return nccl_fail(ctx, "ncclReduceScatter (pipelined combine)", r);
    } else if (!cuda(cudaMemcpyAsync(Grecv + g * t * NN, slot, (size_t)(t * NN) * sizeof(double), cudaMemcpyDeviceToDevice,
                                     c.comm_stream))) {
      return POLYA_ECUDA;
    }
    if (!cuda(cudaEventRecord(c.comb_ev[2 + q], c.comm_stream))) return POLYA_ECUDA;
  }
  if (c.timing && !cuda(cudaEventRecord(c.ev[2], s))) return POLYA_ECUDA;   // end of the assembly
  for (int q = 0; q < 2 && q < groups; ++q)   // the caller's stream sees every group reduced
    if (!cuda(cudaStreamWaitEvent(s, c.comb_ev[2 + q], 0))) return POLYA_ECUDA;
  if (c.timing && !cuda(cudaEventRecord(c.ev[3], s))) return POLYA_ECUDA;
  return POLYA_OK;
}

extern "C" polya_status polya_set_combine_tiles(polya_ctx* ctx, int64_t tiles) {
  if (!ctx || tiles < 0) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.cfg.shard != POLYA_SHARD_BLOCKS) return POLYA_EINVAL;
  polya::combine_free(c);   // the slots are sized by t
  c.comb_t = tiles;
  return POLYA_OK;
}

// ---- fused P2P combine (SHARD_BLOCKS): K4 writes each of this rank's partial tiles straight into
// its owner's receive slot over NVLink peer memory (the epilogue's stores go to the peer; no
// separate collective), then every owner sums its nranks slots in rank order.  Owner and position of
// a pair tile follow the tile groups of combine_shape, so Grecv has the layout of polya_reduce_G.
namespace {
inline void p2p_place(const Ctx& c, int64_t p, int64_t t, int* owner, int64_t* q) {
  const int64_t N = c.cfg.nranks, g = p / (N * t), w = p % (N * t);
  *owner = (int)(w / t);
  *q = g * t + w % t;
}
polya_status p2p_tables(Ctx& c, const std::vector<double*>& base) {
  int64_t t = 0, groups = 0;
  combine_shape(c, &t, &groups);
  const int64_t NN = c.Ntil * c.Ntil, N = c.cfg.nranks, own = groups * t;
  std::vector<double*> tp(c.npairs_local);
  for (int64_t pl = 0; pl < c.npairs_local; ++pl) {
    int o;
    int64_t q;
    p2p_place(c, c.local_pairs[pl], t, &o, &q);
    tp[pl] = base[o] + (c.cfg.rank * own + q) * NN;
  }
  // ready: owner o's flag for this rank (the slot is written); ack: source o's flag for this rank (this
  // rank, as owner, has summed o's slot, which o may then overwrite)
  std::vector<int*> fp(N), ap(N);
  for (int64_t o = 0; o < N; ++o) {
    fp[o] = reinterpret_cast<int*>(base[o] + N * own * NN) + c.cfg.rank;
    ap[o] = reinterpret_cast<int*>(base[o] + N * own * NN) + kP2pAck + c.cfg.rank;
  }
  if (tp.empty()) tp.push_back(nullptr);
  if (cudaMalloc(&c.d_tile_ptr, tp.size() * sizeof(double*)) != cudaSuccess ||
      cudaMalloc(&c.d_flag_ptr, fp.size() * sizeof(int*)) != cudaSuccess ||
      cudaMalloc(&c.d_ack_ptr, ap.size() * sizeof(int*)) != cudaSuccess ||
      cudaMemcpy(c.d_tile_ptr, tp.data(), tp.size() * sizeof(double*), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.d_flag_ptr, fp.data(), fp.size() * sizeof(int*), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(c.d_ack_ptr, ap.data(), ap.size() * sizeof(int*), cudaMemcpyHostToDevice) != cudaSuccess) {
    c.last_error = "polya_p2p: destination tables";
    return POLYA_ENOMEM;
  }
  c.p2p_ready = true;
  return POLYA_OK;
}
}  // namespace

extern "C" polya_status polya_p2p_export(polya_ctx* ctx, char handle_out[64]) {
  if (!ctx) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.cfg.shard != POLYA_SHARD_BLOCKS || c.cfg.nranks > kP2pAck) {
    c.last_error = "polya_p2p_export needs SHARD_BLOCKS and at most 32 ranks";
    return POLYA_EINVAL;
  }
  if (!c.p2p_buf) {
    int64_t t = 0, groups = 0;
    combine_shape(c, &t, &groups);
    c.p2p_own = groups * t;
    const size_t bytes = (size_t)(c.cfg.nranks * c.p2p_own * c.Ntil * c.Ntil) * sizeof(double) + 256;
    if (cudaMalloc(&c.p2p_buf, bytes) != cudaSuccess) {
      c.last_error = "polya_p2p_export: receive slots";
      return POLYA_ENOMEM;
    }
    cudaMemset(reinterpret_cast<char*>(c.p2p_buf) + bytes - 256, 0, 256);   // the flags
  }
  if (handle_out) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t hnd;
    if (cudaIpcGetMemHandle(&hnd, c.p2p_buf) != cudaSuccess) {
      c.last_error = "cudaIpcGetMemHandle failed";
      return POLYA_ECUDA;
    }
    std::memcpy(handle_out, &hnd, 64);
  }
  return POLYA_OK;
}

extern "C" polya_status polya_p2p_import(polya_ctx* ctx, const char* handles) {
  if (!ctx || !handles) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (!c.p2p_buf) {
    c.last_error = "polya_p2p_import before polya_p2p_export";
    return POLYA_EINVAL;
  }
  std::vector<double*> base(c.cfg.nranks);
  for (int r = 0; r < c.cfg.nranks; ++r) {
    if (r == c.cfg.rank) {
      base[r] = c.p2p_buf;
      continue;
    }
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, handles + 64 * r, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hnd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      c.last_error = "cudaIpcOpenMemHandle failed (peer access over NVLink needed)";
      return POLYA_ECUDA;
    }
    c.p2p_opened.push_back(p);
    base[r] = (double*)p;
  }
  return p2p_tables(c, base);
}

extern "C" polya_status polya_p2p_loopback(polya_ctx** ctxs, int32_t nranks) {
  if (!ctxs || nranks < 1) return POLYA_EINVAL;
  std::vector<double*> base(nranks);
  for (int32_t r = 0; r < nranks; ++r) {
    if (!ctxs[r] || ctxs[r]->c.cfg.rank != r || ctxs[r]->c.cfg.nranks != nranks) return POLYA_EINVAL;
    polya_status st = polya_p2p_export(ctxs[r], nullptr);
    if (st != POLYA_OK) return st;
    base[r] = ctxs[r]->c.p2p_buf;
  }
  for (int32_t r = 0; r < nranks; ++r) {
    polya_status st = p2p_tables(ctxs[r]->c, base);
    if (st != POLYA_OK) return st;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_schur_reduce_p2p(polya_ctx* ctx, const double* X, const double* Zinv, double* Grecv,
                                               int phases, void* stream) {
  if (!ctx || (phases & 1 && (!X || !Zinv)) || (phases & 2 && !Grecv) || !(phases & 3)) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (!c.p2p_ready) {
    c.last_error = "polya_schur_reduce_p2p before polya_p2p_import / polya_p2p_loopback";
    return POLYA_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t NN = c.Ntil * c.Ntil, N = c.cfg.nranks;
  const int* flags = reinterpret_cast<const int*>(c.p2p_buf + N * c.p2p_own * NN);
  if (phases & 1) {   // assemble into the owners' slots, then signal every owner
    polya_status st = polya_schur_prepare(ctx, X, Zinv, stream);
    if (st != POLYA_OK) return st;
    const int prev = c.p2p_epoch++;
    cudaError_t e = cudaSuccess;
    // the owners have summed the previous epoch's slots (their acks): only then overwrite them
    if (prev > 0) {
      e = launch_p2p_wait(flags + kP2pAck, (int)N, prev, s);
      ++c.launches;
    }
    if (e == cudaSuccess) e = launch_schur(c, nullptr, POLYA_G_PAIR_TILES, c.item0, c.item1, s, c.d_tile_ptr);
    if (e == cudaSuccess && c.timing) e = cudaEventRecord(c.ev[2], s);
    if (e == cudaSuccess) {
      e = launch_p2p_signal(c.d_flag_ptr, (int)N, c.p2p_epoch, s);
      ++c.launches;
    }
    if (e != cudaSuccess) {
      c.last_error = std::string("polya_schur_reduce_p2p: ") + cudaGetErrorString(e);
      return POLYA_ECUDA;
    }
  }
  if (phases & 2) {   // wait for every source's signal, sum the slots in rank order, acknowledge
    cudaError_t e = launch_p2p_wait(flags, (int)N, c.p2p_epoch, s);
    if (e == cudaSuccess) e = launch_p2p_sum(c.p2p_buf, (int)N, c.p2p_own * NN, Grecv, s);
    if (e == cudaSuccess) e = launch_p2p_signal(c.d_ack_ptr, (int)N, c.p2p_epoch, s);
    c.launches += 3;
    if (e == cudaSuccess && c.timing) e = cudaEventRecord(c.ev[3], s);
    if (e != cudaSuccess) {
      c.last_error = std::string("polya_schur_reduce_p2p: ") + cudaGetErrorString(e);
      return POLYA_ECUDA;
    }
  }
  return POLYA_OK;
}

namespace polya {
void combine_free(Ctx& c) {
  if (c.d_tile_ptr) cudaFree(c.d_tile_ptr);
  if (c.d_flag_ptr) cudaFree(c.d_flag_ptr);
  if (c.d_ack_ptr) cudaFree(c.d_ack_ptr);
  c.d_tile_ptr = nullptr;
  c.d_flag_ptr = nullptr;
  c.d_ack_ptr = nullptr;
  c.p2p_epoch = 0;
  for (void* p : c.p2p_opened) cudaIpcCloseMemHandle(p);
  c.p2p_opened.clear();
  if (c.p2p_buf) cudaFree(c.p2p_buf);
  c.p2p_buf = nullptr;
  c.p2p_ready = false;
  for (auto& p : c.comb_slot) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  for (auto& e : c.comb_ev) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  if (c.comm_stream) cudaStreamDestroy(c.comm_stream);
  c.comm_stream = nullptr;
}

// ---- in-process loopback group (polya_factor_solve_loopback): the ranks are host threads of one
// process on one device; a collective is stream sync -> publish the buffer -> barrier -> device
// copies from the root's buffer -> sync -> barrier.  Same call sequence as the NCCL path; a rank that
// fails aborts the group so the others leave their barriers with an error instead of hanging.
bool loop_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  if (g->abort) return false;
  const int64_t my = g->gen;
  if (++g->count == g->n) {
    g->count = 0;
    ++g->gen;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->gen != my || g->abort; });
  }
  return !g->abort;
}
void loop_abort(LoopGroup* g) {
  std::lock_guard<std::mutex> lk(g->m);
  g->abort = true;
  g->cv.notify_all();
}

namespace {
cudaError_t loop_fail(Ctx& c, const char* what) {
  c.last_error = std::string(what) + ": loopback group aborted (another rank failed)";
  return cudaErrorUnknown;
}
cudaError_t loop_bcast(Ctx& c, void* buf, size_t bytes, int root, cudaStream_t s) {
  LoopGroup* g = (LoopGroup*)c.loop;
  const int r = c.cfg.rank;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  g->ptr[r] = buf;
  if (!loop_barrier(g)) return loop_fail(c, "broadcast");
  if (r != root && bytes) {
    e = cudaMemcpyAsync(buf, g->ptr[root], bytes, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
  }
  if (!loop_barrier(g)) return loop_fail(c, "broadcast");
  return cudaSuccess;
}
cudaError_t loop_bcast_tiles(Ctx& c, double* buf, size_t count, int64_t ntiles, cudaStream_t s) {
  LoopGroup* g = (LoopGroup*)c.loop;
  const int r = c.cfg.rank, n = c.cfg.nranks;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  g->ptr[r] = buf;
  if (!loop_barrier(g)) return loop_fail(c, "tile broadcast");
  for (int64_t q = 0; q < ntiles && e == cudaSuccess; ++q)
    if (q % n != r)
      e = cudaMemcpyAsync(buf + q * count, (const double*)g->ptr[q % n] + q * count, count * sizeof(double),
                          cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  if (!loop_barrier(g)) return loop_fail(c, "tile broadcast");
  return cudaSuccess;
}
cudaError_t loop_allreduce(Ctx& c, double* buf, size_t count, bool max, cudaStream_t s) {
  LoopGroup* g = (LoopGroup*)c.loop;
  const int r = c.cfg.rank;
  g->host[r].resize(count);
  cudaError_t e = cudaMemcpyAsync(g->host[r].data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  if (!loop_barrier(g)) return loop_fail(c, "all-reduce");
  std::vector<double> acc(g->host[0]);
  for (int q = 1; q < g->n; ++q)   // rank order: every rank forms the same value
    for (size_t i = 0; i < count; ++i) acc[i] = max ? std::max(acc[i], g->host[q][i]) : acc[i] + g->host[q][i];
  if (!loop_barrier(g)) return loop_fail(c, "all-reduce");   // everyone has read every host[q]
  e = cudaMemcpyAsync(buf, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}
}  // namespace

// Collectives of the distributed factorisation (SHARD_CYCLIC): NCCL with polya_nccl_init, the loopback
// group inside polya_factor_solve_loopback; no-ops with one rank.
cudaError_t comm_bcast(Ctx& c, void* buf, size_t count, bool is_int, int root, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (c.loop) return loop_bcast(c, buf, count * (is_int ? sizeof(int32_t) : sizeof(double)), root, s);
  if (!c.nccl) return c.cfg.nranks == 1 ? cudaSuccess : cudaErrorNotReady;   // one rank: nothing to send
  ncclResult_t r = ncclBroadcast(buf, buf, count, is_int ? ncclInt32 : ncclFloat64, root, (ncclComm_t)c.nccl, s);
  if (r != ncclSuccess) {
    c.last_error = std::string("ncclBroadcast: ") + ncclGetErrorString(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}
// tile q of buf (count doubles each, q < ntiles) broadcast from rank q mod nranks, as one NCCL group
cudaError_t comm_bcast_tiles(Ctx& c, double* buf, size_t count, int64_t ntiles, cudaStream_t s) {
  if (count == 0 || ntiles == 0) return cudaSuccess;
  if (c.loop) return loop_bcast_tiles(c, buf, count, ntiles, s);
  if (!c.nccl) return c.cfg.nranks == 1 ? cudaSuccess : cudaErrorNotReady;
  ncclResult_t r = ncclGroupStart();
  for (int64_t q = 0; q < ntiles && r == ncclSuccess; ++q)
    r = ncclBroadcast(buf + q * count, buf + q * count, count, ncclFloat64, (int)(q % c.cfg.nranks), (ncclComm_t)c.nccl, s);
  ncclResult_t r2 = ncclGroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    c.last_error = std::string("ncclBroadcast (tiles): ") + ncclGetErrorString(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}
static cudaError_t comm_allreduce(Ctx& c, double* buf, size_t count, bool max, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (c.loop) return loop_allreduce(c, buf, count, max, s);
  if (!c.nccl) return c.cfg.nranks == 1 ? cudaSuccess : cudaErrorNotReady;
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat64, max ? ncclMax : ncclSum, (ncclComm_t)c.nccl, s);
  if (r != ncclSuccess) {
    c.last_error = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}
cudaError_t comm_allreduce_sum(Ctx& c, double* buf, size_t count, cudaStream_t s) {
  return comm_allreduce(c, buf, count, false, s);
}
cudaError_t comm_allreduce_max(Ctx& c, double* buf, size_t count, cudaStream_t s) {
  return comm_allreduce(c, buf, count, true, s);
}

void nccl_free(Ctx& c) {
  if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
  c.nccl = nullptr;
}
}  // namespace polya
