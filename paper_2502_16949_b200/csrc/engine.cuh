// Engine context: device-resident store, triples, epoch plan and workspaces
// behind the C ABI (include/skge_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/skge_b200.h"
#include "kernels.cuh"
#include "plan.cuh"
#include "sampling.cuh"

namespace skg {

// Host-side mirrors of the reference exception types (common.hpp:37-59).
struct ShapeError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct TrainingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegenerateTripleError : std::invalid_argument { using std::invalid_argument::invalid_argument; };

template <class T>
struct DevBuf {
  T* p = nullptr;
  int64_t n = 0;
  void ensure(int64_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (cudaMalloc(&p, sizeof(T) * (count > 0 ? count : 1)) != cudaSuccess)
      throw CudaError("cudaMalloc failed (" + std::to_string(sizeof(T) * count) + " bytes)");
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

struct DpState;     // NCCL replicas (dp.cu)
struct ShardState;  // row-sharded tables (shard.cu)

// One epoch's permutation and transposed-incidence plan. Two slots let the
// next epoch's plan be built on a side stream while the current one trains.
struct HostNarrow;  // engine.cu

struct PlanSlot {
  DevBuf<int32_t> order, order_g;
  EpochPlan plan;
  // TransH relation tiles of every batch (transh_tile_plan), built with the plan
  DevBuf<int4> th_meta, th_rows;
  DevBuf<int32_t> th_pos;
  DevBuf<uint32_t> th_info;
  bool th_on = false;
  // TransR relation tiles of every batch (transr_tile_plan)
  DevBuf<uint32_t> tr_seg, tr_p0, tr_total, tr_segtiles;
  bool tr_on = false;
  std::string key;  // which (epoch, seed, data version, shape) the slot holds
};

}  // namespace skg

struct skg_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  // ---- store (embedding.hpp:15-31)
  bool has_store = false;
  skg_model_config cfg{};
  int64_t N = 0, R = 0, de = 0, dr = 0;  // de / dr: floats per row (2 x dim for complex stores)
  skg::DevBuf<float> tables;  // [entity N x de ; relation R x dr]
  skg::DevBuf<float> proj, normals;

  // ---- triples
  int64_t M = 0, tN = 0, tR = 0;
  skg::DevBuf<int32_t> H, Rl, T, NH, NT;
  skg::DevBuf<int4> quad;            // {H, T, NH, NT} per triple, packed for the plan's gathers
  uint64_t quad_version = ~0ull;     // data_version quad was packed at
  bool has_neg = false;

  // ---- epoch machinery
  skg::DevBuf<int32_t> order;
  skg::EpochPlan plan;
  skg::ShuffleWork shuffle;
  skg::NegWork negw;
  skg::DevBuf<float> res, res_u, scal, block_partial, batch_loss, scores, grad_sink;
  skg::DevBuf<float> ht_work;  // ht models: per-row relation-side rows
  skg::DevBuf<uint32_t> err_words;  // [0] code [1] batch [2] aux [3] pending
  skg::DevBuf<unsigned> counter;
  skg::DevBuf<uint64_t> seed_eff;
  skg::DevBuf<float> lr_dev;
  skg::DevBuf<int32_t> tmp_i32;     // per-call id uploads
  skg::DevBuf<float> tmp_f32;
  skg::DevBuf<uint8_t> flush_buf;
  skg::DevBuf<int64_t> stage_i64;   // caller id arrays staged in HBM
  skg::DevBuf<float> dp_grad;       // data parallel: dense gradient sink + 2 flag slots
  skg::DevBuf<int32_t> order_g;     // data parallel: this rank's shards of the epoch order
  skg::DevBuf<uint32_t> bad_idx;
  uint64_t* h_seed = nullptr;   // pinned
  float* h_lr = nullptr;        // pinned
  uint32_t* h_err = nullptr;    // pinned
  float* h_loss = nullptr;      // pinned, per batch
  int64_t h_loss_cap = 0;

  // ---- training-loop plan slots and captured epoch graphs (one per slot)
  skg::PlanSlot slots[2];
  int cur = 0;        // slot holding (or to hold) the plan of the next epoch to train
  int last_slot = 0;  // slot the last trained epoch used (plan_stats)
  uint64_t data_version = 0;
  bool triples_valid = false;              // H/Rl/T hold the last successful set_triples
  uint64_t neg_valid_version = ~0ull;      // data_version at which NH/NT were last set (or sampled)
  uint64_t loops_version = ~0ull;          // data_version the self-loop scan below refers to
  bool has_loops = false;                  // some positive or negative triple has head == tail
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaStream_t aux = nullptr;  // per-batch side branch (TransH relation step beside the entity pass)
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  // Epoch permutations two epochs ahead: the graph of epoch e builds e + 1's
  // plan from perm[nxt] (made during epoch e - 1) while a second side branch
  // shuffles e + 2's order into perm[cur]; perm_key says which epoch each holds.
  skg::DevBuf<int32_t> perm[2];
  std::string perm_key[2];
  cudaStream_t side2 = nullptr;
  cudaEvent_t join2_ev = nullptr;
  cudaEvent_t snap_ev = nullptr;     // speculative epoch: parameter snapshot done (waited by batch 0's first write)
  cudaEvent_t snap_cap_ev = nullptr; // the same inside a speculative graph (an event used in a capture stays there)
  cudaEvent_t fork_up_ev = nullptr;
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};
  std::string graph_keys[2];
  // The epoch graph's first node writes this epoch's lr and the seed of the
  // permutation it shuffles (epoch + 2) to the device; its kernel arguments
  // are updated in the instantiated graph before each launch (no H2D copies
  // ahead of the graph). graph_src keeps the captured graph the node belongs to.
  cudaGraph_t graph_src[2] = {nullptr, nullptr};
  cudaGraphNode_t param_node[2] = {nullptr, nullptr};
  // finish_epoch: one kernel writes the batch losses, the error words and (in
  // a speculative epoch) the upload check's flags straight into the pinned
  // host buffers (mapped under UVA) instead of three D2H copies.
  const uint32_t* pub_spec = nullptr;
  // A speculative epoch's graph snapshots the parameters itself (a branch at
  // the graph's start, batch 0's first parameter write waits for it).
  bool spec_graph = false;
  int64_t graph_launches_k[2] = {0, 0};
  int64_t last_launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // PhaseTimer buckets (training.cpp:15-20): every batch's forward kernels
  // stamp their start and end (globaltimer) into `stamps`, read back with the
  // batch losses. No extra graph nodes.
  bool phase_timers = true;
  skg::DevBuf<unsigned long long> stamps;  // [2 * nb]: forward start, forward end
  unsigned long long* h_stamps = nullptr;  // pinned
  int64_t h_stamps_cap = 0;
  double last_epoch_ms = 0;  // device time of the last graph epoch (ev0 -> ev1)

  // ---- deferred id uploads (speculative epoch). A re-upload of pinned arrays
  // with the shape of the current triples is recorded, not copied; the next
  // train_epoch copies it on `up` (DMA) while the epoch runs on the current
  // device ids, then compares. Equal: done. Different or invalid: the
  // parameters are rolled back from `backup` and the call falls back to the
  // synchronous path (adopt + rerun, or the reference's ShapeError).
  bool pend_tri = false, pend_neg = false;
  const int64_t* pend_ptr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // h, r, t, nh, nt
  bool speculate = true;
  cudaStream_t up = nullptr;
  cudaEvent_t up_ev = nullptr;
  skg::DevBuf<float> backup;        // parameters before a speculative epoch
  skg::DevBuf<uint32_t> spec_flags; // first bad entity / relation / negative index, changed
  int64_t spec_hits = 0, spec_misses = 0;
  int64_t upload_bytes = 0;             // bytes DMA'd by deferred uploads (skg_upload_bytes)
  double last_shuffle_ms = 0.0;         // shuffle part of the last skg_profile_epoch
  skg::HostNarrow* narrow = nullptr;    // host threads narrowing deferred int64 uploads to int32
  int32_t* h_stage32 = nullptr;         // pinned: narrowed ids, wave-major
  int64_t h_stage32_cap = 0;
  skg::DevBuf<int32_t> stage_i32;       // device copy of h_stage32
  uint32_t* h_spec = nullptr;           // pinned: the check's flags

  // ---- data parallel
  skg::DpState* dp = nullptr;        // replicated tables, NCCL all-reduce
  skg::ShardState* shard = nullptr;  // row-sharded tables, peer memory
};
