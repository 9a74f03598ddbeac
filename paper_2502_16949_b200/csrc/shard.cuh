// Row-sharded data parallel state (shard.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "primitives.cuh"

struct skg_ctx;

namespace skg {

// Every rank's sharded buffers (peer pointers; index = rank).
struct ShardPtrs {
  float* ent[8];                 // entity shard: rows e / G of the entities e % G == rank
  float* rel[8];                 // relation replica (R x d)
  float* res[8];                 // residual rows of the rank's forward pairs (2 S x d)
  float* scal[8];                // their row scales (2 S)
  float* loss[8];                // per-batch shard losses
  unsigned long long* flags[8];  // barrier flags (G slots) + generation counter
};

struct ShardPlanBufs {
  int4* pair_ht = nullptr;  // this rank's forward pairs
  int32_t* pair_r = nullptr;
  uint32_t *cnt = nullptr, *off = nullptr;  // owned entries per global row, their offsets
  uint32_t *key = nullptr, *val = nullptr, *key_alt = nullptr, *val_alt = nullptr;
  uint32_t *seg_start = nullptr, *seg_col = nullptr, *seg_base = nullptr, *nseg = nullptr;
  const uint32_t* sorted_val = nullptr;
  int64_t cap_pairs = 0, cap_rows = 0, cap_entries = 0, cap_batches = 0;
  int64_t nb = 0, E = 0;
  SortPlan sort;
  ScanPlan scan;
  void reserve(int64_t pairs, int64_t rows2, int64_t entries, int64_t batches);
  void release();
  ~ShardPlanBufs() { release(); }
};

struct ShardState {
  int rank = 0, world = 1, glog = 0;
  int64_t B = 0, S = 0, d = 0;  // global batch, shard size of full batches, floats per row
  int64_t NEo = 0, NRo = 0;     // entities / relations owned by this rank
  int64_t nb_cap = 0;
  // one cudaMalloc arena (one IPC handle): entity shard | relation replica |
  // residual rows | row scales | shard losses | barrier flags + generation
  void* arena = nullptr;
  size_t arena_bytes = 0, off_ent = 0, off_rel = 0, off_res = 0, off_scal = 0, off_loss = 0, off_flags = 0;
  float** ptr_dev = nullptr;  // device copy of peers.loss (loss gather)
  ShardPtrs peers{};
  void* opened[8] = {};  // IPC-opened peer arenas (closed on destroy)
  bool linked = false;
  ShardPlanBufs plan[2];
  int64_t E = 0;                  // owned incidence entries per epoch (data-dependent only)
  uint64_t count_version = ~0ull;
  ~ShardState();
};

void shard_alloc(skg_ctx* ctx, int rank, int world, int64_t batch_size);
void shard_link(skg_ctx* ctx, void* const* bases);
void shard_scatter_store(skg_ctx* ctx);
void shard_gather_store(skg_ctx* ctx);
int64_t shard_entry_count(skg_ctx* ctx);
void shard_build_plan(skg_ctx* ctx, const int32_t* order, const int32_t* order_g, int64_t Mg, int slot,
                      cudaStream_t s);
void shard_barrier(skg_ctx* ctx, cudaStream_t s);
void shard_backward(skg_ctx* ctx, int kind, int slot, int64_t batch, cudaStream_t s);
void shard_finish_losses(skg_ctx* ctx, int64_t nb, cudaStream_t s);
void shard_fill_fwd(skg_ctx* ctx, FwdArgs& fa);
void shard_destroy(skg_ctx* ctx);

}  // namespace skg
