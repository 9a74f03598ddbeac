// Data-parallel replicas over NCCL (one process per GPU, NVLink/NVSwitch).
//
// Replicated tables. Every global minibatch (the reference's batch at
// batch_size = global batch, training.cpp:120-161) is split into `world`
// contiguous shards of pairs; each rank runs the fused forward on its shard
// with the global 1/m upstream (training.cpp:84), accumulates its shard's
// transposed-SpMM gradient into a dense sink, the sinks are summed with
// ncclAllReduce over NVLink, and every rank applies the identical SGD step.
// Two extra floats ride along in the reduced buffer and carry the ranks'
// error flags, so a non-finite loss or gradient on any shard stops the update
// on every rank without an extra collective. The epoch sequence (shuffle,
// plan, per-batch kernels and NCCL calls) is captured in one CUDA graph.
#include <nccl.h>

#include <cstring>

#include "common.cuh"
#include "engine.cuh"
#include "ht.cuh"

namespace skg {

#define SKG_NCCL(call)                                                                        \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) throw CudaError(std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

struct DpState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

void dp_destroy(skg_ctx* ctx) {
  if (!ctx->dp) return;
  // captured graphs hold NCCL calls on this communicator: never replay them
  drop_graphs(ctx);
  if (ctx->dp->comm) ncclCommDestroy(ctx->dp->comm);
  delete ctx->dp;
  ctx->dp = nullptr;
}

int dp_rank(const skg_ctx* ctx) { return ctx->dp ? ctx->dp->rank : ctx->shard ? shard_rank(ctx) : 0; }
int dp_world(const skg_ctx* ctx) { return ctx->dp ? ctx->dp->world : ctx->shard ? shard_world(ctx) : 1; }
const void* dp_comm_tag(const skg_ctx* ctx) { return ctx->dp ? static_cast<const void*>(ctx->dp->comm) : nullptr; }

void dp_allreduce_sum(skg_ctx* ctx, float* buf, int64_t n, cudaStream_t s) {
  SKG_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(n), ncclFloat32, ncclSum, ctx->dp->comm, s));
}

}  // namespace skg

extern "C" {

skg_status skg_nccl_unique_id(char out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SKG_ERR_CUDA;
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  std::memcpy(out, &id, sizeof(id));
  return SKG_OK;
}

skg_status skg_dp_init(skg_ctx* ctx, const char unique_id[128], int rank, int world) {
  try {
    SKG_CUDA(cudaSetDevice(ctx->device));
    if (world < 1 || rank < 0 || rank >= world) throw skg::ConfigError("dp_init: bad rank/world");
    skg::dp_destroy(ctx);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    auto* st = new skg::DpState();
    st->rank = rank;
    st->world = world;
    if (ncclCommInitRank(&st->comm, world, id, rank) != ncclSuccess) {
      delete st;
      throw skg::CudaError("ncclCommInitRank failed");
    }
    ctx->dp = st;
    skg::drop_graphs(ctx);
    return SKG_OK;
  } catch (const skg::ConfigError& e) {
    ctx->err = e.what();
    return SKG_ERR_CONFIG;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return SKG_ERR_CUDA;
  }
}

}  // extern "C"
