// combine.cpp -- multi-GPU combine of the block-sharded Schur complement (row a9 of SURVEY 8(a)).
//
// With POLYA_SHARD_BLOCKS every rank owns a contiguous, cost-balanced range of the Polya blocks and
// assembles the partial sum G^(r) = sum_{b in [b0,b1)} G^(b) over all entries -- the paper's
// decentralised structure -- and the partials are summed over NVLink with
// one NCCL collective instead of the paper's root gather.
#include <nccl.h>

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
  if (layout == POLYA_G_PAIR_TILES) {
    const int64_t tot = c.npairs * c.Ntil * c.Ntil;
    const size_t rc = (size_t)((tot + c.cfg.nranks - 1) / c.cfg.nranks);
    r = ncclReduceScatter(Gpart, Grecv, rc, ncclFloat64, ncclSum, comm, s);
  } else if (layout == POLYA_G_FULL) {
    r = ncclAllReduce(Gpart, Grecv, (size_t)(c.K * c.K), ncclFloat64, ncclSum, comm, s);
  } else {
    return POLYA_EINVAL;
  }
  if (r != ncclSuccess) return nccl_fail(ctx, "NCCL collective", r);
  return POLYA_OK;
}

namespace polya {
// Collectives of the distributed factorisation (SHARD_CYCLIC).  With one rank they are no-ops (the
// root's buffer is every rank's buffer); with more they need polya_nccl_init.
cudaError_t comm_bcast(Ctx& c, void* buf, size_t count, bool is_int, int root, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
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
cudaError_t comm_allreduce_sum(Ctx& c, double* buf, size_t count, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (!c.nccl) return c.cfg.nranks == 1 ? cudaSuccess : cudaErrorNotReady;
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c.nccl, s);
  if (r != ncclSuccess) {
    c.last_error = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

void nccl_free(Ctx& c) {
  if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
  c.nccl = nullptr;
}
}  // namespace polya
