// Launch interfaces of the hot-path kernels.
//
//   hrt_forward   TransE / TorusE forward: hrt gather (h - t) + r, distance,
//                 margin hinge, loss, per-row gradient scale (models.cpp:11-30,
//                 71-92; norms.hpp; training.cpp:73-94)
//   ht_forward    TransH hyperplane / TransR projection forward on the ht
//                 layout (models.cpp:110-134, 158-181)
//   mult_forward  DistMult / ComplEx / RotatE forward on the multiplicative
//                 layout: times-times (or mulsub) row, exact-order score sum,
//                 hinge, loss and the three per-entry gradient rows
//                 (models.cpp:201-263, sparse.hpp:91-106, 315-391)
//   segment_backward  transposed-SpMM scatter A^T D as a sorted-segment,
//                 warp-per-column reduction fused with the SGD update
//                 (sparse.hpp:273-306, embedding.cpp:165-190)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace skg {

// Score kinds: model x norm, fixed at kernel instantiation.
enum Kind : int {
  kTransE_L2 = 0,
  kTransE_L1 = 1,
  kTorusE_L2 = 2,
  kTorusE_L1 = 3,
  kTransH_L2 = 4,
  kTransH_L1 = 5,
  kTransR_L2 = 6,
  kTransR_L1 = 7,
  kPlainRows = 8,  // backward rows already hold a*D (ht models' du rows)
  kDistMult = 9,   // multiplicative family (norm ignored, as in the reference)
  kComplEx = 10,
  kRotatE = 11,
  kMultRows = 12,  // backward rows: per-entry gradient planes [head | tail | relation]
  kTileSlotRows = 13,  // TransR tcgen05 training: dU rows in tile-blocked order, scal = slot + 1 (0: inactive)
};
// kTileSlotRows layout of a d = 128 dU row (tile slot s = 128 * tile + lane):
// kDuGroup-float groups g of the row at s / 128 * 128 * 128 + g * 128 * kDuGroup
// + (s % 128) * kDuGroup: the producing warp (thread = row) stores whole groups
// with 32-byte stores into one contiguous run per group, a reader fetches whole
// kDuGroup * 4-byte pieces.
#ifndef SKG_TR_DU_GROUP
#define SKG_TR_DU_GROUP 16
#endif
constexpr int kDuGroup = SKG_TR_DU_GROUP;
__host__ __device__ inline int64_t tile_rows_floats(int64_t rows, int64_t R) { return (rows + 128 * (R + 1)) * 128; }
inline bool is_mult_kind(int k) { return k >= kDistMult && k <= kRotatE; }
inline bool is_ht_kind(int k) { return k >= kTransH_L2 && k <= kTransR_L1; }

struct FwdArgs {
  // parameters
  const float* X;        // stacked [entity (N x de); relation (R x dr)]
  const float* proj;     // TransR: R x (dr*de)
  const float* normals;  // TransH: R x de
  int64_t N;
  int de, dr;
  // rows. TRAIN: pairs p in [0, B) via order[p] -> (H,R,T) / (NH,R,NT);
  //       SCORE: rows i in [0, B) straight from (H,R,T).
  const int32_t* order;
  const int4* pair_ht;     // TRAIN: per pair {h, t, neg h, neg t} (epoch plan), may be null
  const int32_t* pair_r;
  const int32_t *H, *Rl, *T, *NH, *NT;
  int B;
  float margin, unit;
  float loss_div;  // divisor of the batch loss (0: B); data parallel shards use the global batch size
  const float* upstream;  // SCORE: optional per-row upstream -> scal
  // outputs
  float* res;     // residual rows (v or delta), 2B x d (TRAIN) / B x d (SCORE)
  float* res_u;   // ht models: u = h - t rows (de wide)
  float* scal;    // per-row gradient scale (0 = inactive)
  float* scores;  // SCORE mode
  int64_t plane_rows;  // multiplicative: rows per gradient plane (res holds 3 planes)
  float sign;          // multiplicative: energy_sign (models.hpp:35-38)
  // loss reduction
  float* block_partial;
  unsigned* counter;
  float* batch_loss;  // slot for this batch
  int batch;
  uint32_t* err;
  // PhaseTimer stamps (globaltimer ns, training.cpp:15-20): the batch's first
  // forward kernel writes stamp_start from its first block, the last block of
  // the loss reduction writes stamp_end. Null: no stamps.
  unsigned long long* stamp_start;
  unsigned long long* stamp_end;
  // Row-sharded tables (shard.cu): entity e lives on rank e % G at
  // local row e / G of ent_peer[e % G] (peer memory, G = 1 << glog); relation
  // rows come from the local replica rel_rows. ent_peer[0] == null: the
  // stacked table X as usual.
  const float* ent_peer[8];
  int glog;
  const float* rel_rows;
};

struct BwdArgs {
  float* X;            // tables updated in place (SGD) or gradient sink (accumulate)
  float* Xrel;         // ht models: relation table / sink (R x dr)
  const float* res;
  const float* scal;
  int64_t N;
  int d;
  const uint32_t* ent_val;    // sorted entries: row2 | sign << 31
  const uint32_t* seg_start;  // per segment: first entry; seg_start[nseg] = end
  const uint32_t* seg_col;    // per segment: stacked column
  const uint32_t* seg_base;   // per batch: first segment; [nb] = nseg
  int batch;
  const float* lr;  // device scalar (lets one captured graph serve every epoch)
  uint32_t* err;
  int entity_only;  // skip relation-column segments (ht models reduce them separately)
  int64_t plane_rows;  // kMultRows: rows per plane; slot = relation column ? 2 : tail entry ? 1 : 0
};

void configure_hrt_kernels();
int64_t bwd_trace(int enable, unsigned long long* out, uint32_t* info, int64_t cap);  // debug
void configure_ht_kernels();
void launch_hrt_forward(int kind, bool train, const FwdArgs& a, int num_sms, cudaStream_t s);
void launch_segment_backward(int kind, bool sgd, const BwdArgs& a, int num_sms, cudaStream_t s);
void configure_mult_kernels();
void launch_mult_forward(int kind, bool train, const FwdArgs& a, int num_sms, cudaStream_t s);

// Generic plus-times sparse operators (sparse_ops.cu; sparse.hpp:110-306), device buffers.
void sparse_coo_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_rows, const int64_t* d_cols,
                       const float* d_vals, int64_t* d_row_ptr, int64_t* d_col, float* d_val, int64_t* nnz_out,
                       cudaStream_t s);
void sparse_transpose(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_row_ptr, const int64_t* d_col,
                      const float* d_val, int64_t* d_trow_ptr, int64_t* d_tcol, float* d_tval, cudaStream_t s);
void sparse_spmm(int64_t rows, const int64_t* d_row_ptr, const int64_t* d_col, const float* d_val, int d,
                 const float* d_x, float* d_out, int num_sms, cudaStream_t s);
void sparse_spmm_transpose_add(int64_t rows, int64_t cols, int64_t nnz, const int64_t* d_row_ptr,
                               const int64_t* d_col, const float* d_val, int d, const float* d_g, float* d_sink,
                               int num_sms, cudaStream_t s);

}  // namespace skg
