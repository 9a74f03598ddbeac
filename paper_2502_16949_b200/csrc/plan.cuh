// Epoch plan: the transposed incidence of every minibatch of an epoch, built
// on device in one pass so the per-batch backward is a pure segmented reduce.
//
// For minibatch b (rows order[b*B .. b*B+Bb)), pass p (0 = positive,
// 1 = negative) and row i, the incidence row (build_hrt, incidence.hpp:62-85;
// canonical after coo_to_csr) has entries {h:+1, t:-1, N+r:+1}, with the
// entity pair dropped when h == t. Entries are emitted in (b, p, i) order,
// keyed by (b, column') with relation columns first, and stably radix-sorted;
// inside each (b, column) segment they therefore appear in exactly the order
// transpose() + spmm_transpose_add() visit them (sparse.hpp:164-183,
// 268-306), positives before negatives (training.cpp:146-147).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "primitives.cuh"

namespace skg {

// seg_col of the per-batch dummy segment (entries that do not exist); skipped.
constexpr uint32_t kDummyCol = 0xFFFFFFFFu;

struct EpochPlan {
  int64_t cap_entries = 0, cap_batches = 0;
  int64_t E = 0, nb = 0;
  int kb = 0, cb = 0;
  uint32_t* key = nullptr;
  uint32_t* val = nullptr;
  uint32_t* key_alt = nullptr;
  uint32_t* val_alt = nullptr;
  uint32_t* seg_start = nullptr;  // [E + 1]
  uint32_t* seg_col = nullptr;    // [E]
  uint32_t* seg_base = nullptr;   // [nb + 1]
  uint32_t* nseg = nullptr;       // [1]
  const uint32_t* sorted_val = nullptr;
  // per epoch position k: {h, t, neg h, neg t} and r of triple order[k], so the
  // forward reads one record per pair instead of chasing order -> ids
  int4* pair_ht = nullptr;
  int32_t* pair_r = nullptr;
  int64_t cap_pairs = 0;
  SortPlan sort;
  ScanPlan scan;
  void reserve(int64_t entries, int64_t batches);
  void release();
  ~EpochPlan() { release(); }
};

// Training epoch: pos/neg rows through `order`, batch size B. quad[id] =
// {H, T, NH, NT}[id] (pack_triple_quads, once per data version).
void build_epoch_plan(const int32_t* order, const int4* quad, const int32_t* R, int64_t M, int64_t B, int64_t N,
                      int64_t Rn, EpochPlan& p, cudaStream_t s);
void pack_triple_quads(const int32_t* H, const int32_t* T, const int32_t* NH, const int32_t* NT, int64_t M,
                       int4* quad, cudaStream_t s);
// One explicit batch (score_backward parity path): rows i with (H,R,T)[i].
// layout 0 = ht (no relation entries), 1 = hrt.
void build_batch_plan(const int32_t* H, const int32_t* R, const int32_t* T, int64_t m, int64_t N,
                      int64_t Rn, int layout, EpochPlan& p, cudaStream_t s);

}  // namespace skg
