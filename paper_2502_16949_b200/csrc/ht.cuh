// ht-layout models (TransH hyperplane, TransR projection) and data-parallel
// replicas: launch interfaces used by engine.cu.
#pragma once

#include <functional>

#include "../../include/skge_b200.h"
#include "kernels.cuh"

struct skg_ctx;

namespace skg {

// Data-parallel training of the ht models: the step writes this rank's
// gradients into zeroed sinks instead of applying SGD (the engine sums them
// over NVLink and applies one dense step); the entity sink is BwdArgs::X.
struct HtSinks {
  float* rel;      // R x d_r
  float* proj;     // TransR: R x (d_r d_e)
  float* normals;  // TransH: R x d_e
};

// A second stream and a fork / join event pair: work that may run beside the
// main stream's next launch (captured as a parallel graph branch).
struct Branch {
  cudaStream_t aux;
  cudaEvent_t fork, join;
};

// TransH relation tiles of every minibatch, precomputed on the plan branch
// (transh_tile_plan): per batch mt = transh_tile_plan_tiles(B, R) tile records.
struct ThTilePlan {
  int4* meta = nullptr;    // [nb][mt] {run, relation, pairs, 0}
  int4* rows = nullptr;    // [nb][mt][32] {h, t, neg h, neg t}
  int32_t* pos = nullptr;  // [nb][mt][32]
  uint32_t* info = nullptr;  // [nb][4 + 3R]
  int64_t B = 0;           // batch size the records were built for
};
int64_t transh_tile_plan_tiles(int64_t B, int64_t R);
// TransR relation tiles of every minibatch (transr_tile_plan): per batch b,
// tile_seg / tile_p0 at b * relation_max_tiles(2B, R), tile_total at 2b,
// seg_tiles at b (R + 2).
struct TrTilePlan {
  uint32_t *tile_seg = nullptr, *tile_p0 = nullptr, *tile_total = nullptr, *seg_tiles = nullptr;
  int64_t B = 0;
};
void transr_tile_plan(const BwdArgs& ba, int64_t B, int64_t nb, int64_t R, const TrTilePlan& tp, cudaStream_t s);
void transh_tile_plan(const FwdArgs& fa, const BwdArgs& ba, int64_t B, int64_t nb, int64_t M, int64_t R,
                      const ThTilePlan& tp, cudaStream_t s);

// embedding.cpp:181-189 on the TransH normals (after a data-parallel dense step)
void launch_normals_renorm(float* normals, int64_t R, int d, uint32_t* err, cudaStream_t s);
// Floats of per-batch scratch the ht kernels need for `rows` rows.
int64_t ht_work_floats(int kind, int64_t rows, int64_t de, int64_t dr, int64_t R);

// One minibatch of TransH / TransR training: forward + hinge, entity scatter
// through the sorted ht segments, relation-side reductions, SGD (+ normals
// renormalization). `mark` (nullable) is called after the forward and after
// the backward for per-phase profiling.
void ht_train_batch(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                    const std::function<void()>* mark, int64_t R, const HtSinks* sinks = nullptr,
                    const Branch* br = nullptr, const ThTilePlan* tp = nullptr, const TrTilePlan* trp = nullptr);
// score_batch for ht models (res = v, res_u = u, scores). `ba` carries the
// batch's plan (TransR groups rows by relation through it).
void ht_score(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s, int64_t R);
// score_backward for ht models, accumulating into the sink tables.
void ht_score_backward(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, float* g_proj, float* g_normals,
                       int num_sms, cudaStream_t s, int64_t R);

// Relation-grouped tiles of 64 (pos, neg) pairs (paired) or 128 rows over a
// batch's relation segments (transr.cu); shared by TransR and TransH.
int64_t relation_max_tiles(int64_t rows, int64_t R);
void launch_relation_tiles(const BwdArgs& ba, int paired, uint32_t* tile_seg, uint32_t* tile_p0, uint32_t* tile_total,
                           uint32_t* seg_tiles, cudaStream_t s, uint32_t* zero = nullptr, int nzero = 0);
// TransH training on relation tiles (transh_train.cu), d_e = d_r = 128
bool transh_tiles_supported(int de, int dr, int64_t R);
void configure_transh_tiles_kernels();
int64_t transh_tiles_work_floats(int64_t rows, int64_t R);
int64_t transh_trace(int enable, unsigned long long* out, int64_t cap);  // debug: phase timestamps
void transh_tiles_train_batch(bool l2, const FwdArgs& fa, const BwdArgs& ba, float* work, int64_t R, int num_sms,
                              cudaStream_t s, const std::function<void()>* mark, const HtSinks* sinks = nullptr,
                              const Branch* br = nullptr, const ThTilePlan* tp = nullptr);

// TransR (transr.cu)
int64_t transr_work_floats(int64_t rows, int64_t de, int64_t dr, int64_t R);
void configure_transr_kernels();
void transr_train_batch(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                        const std::function<void()>* mark, int64_t R, const HtSinks* sinks = nullptr,
                        const Branch* br = nullptr, const TrTilePlan* tp = nullptr);
void transr_score(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                  int64_t R);
void transr_score_backward(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, float* g_proj, int num_sms,
                           cudaStream_t s, int64_t R);

// TransR on tcgen05 (transr_tc.cu), d_e = d_r = 128
bool transr_tc_supported(int de, int dr);
void configure_transr_tc_kernels();
int64_t transr_tc_slots(int num_sms, int64_t R);
void launch_transr_tc(bool l2, int mode, const FwdArgs& fa, const uint32_t* ent_val, const uint32_t* seg_start,
                      const uint32_t* seg_col, const uint32_t* tile_seg, const uint32_t* tile_p0,
                      const uint32_t* tile_total, const uint32_t* seg_tiles, float* dm_part, float* dr_part,
                      float* mr_chunks, int64_t R, int num_sms, cudaStream_t s);
int64_t transr_tc_mr_floats(int64_t R);
void launch_transr_tc_apply(const uint32_t* tile_total, const uint32_t* seg_tiles, const uint32_t* tile_seg,
                            const uint32_t* seg_col, int64_t N, int G, const float* dm_part, const float* dr_part,
                            float* proj, float* rel, const float* lr, bool sgd, const uint32_t* err, int64_t R,
                            cudaStream_t s);
void transr_tc_selftest(int mode, const float* A, const float* B, float* D, cudaStream_t s);
// Warp-specialized training step (transr_train_tc.cu)
void configure_transr_train_tc_kernels();
int64_t transr_train_tc_mr_floats(int64_t R);
int64_t transr_trace(int enable, unsigned long long* out, int64_t cap);  // debug: phase timestamps
// sink != 0: write the summed gradient to proj / rel (zeroed sinks) and leave mr alone
void launch_transr_train_apply(const uint32_t* tile_total, const uint32_t* seg_tiles, const uint32_t* tile_seg,
                               const uint32_t* seg_col, int64_t N, int G, const float* dm_part, const float* dr_part,
                               float* proj, float* rel, const float* lr, const uint32_t* err, float* mr, int64_t R,
                               cudaStream_t s, int sink, int dr, int de);
// d_e, d_r multiples of 16 up to 128 (the training kernel zero-pads its tiles)
bool transr_train_tc_supported(int de, int dr);
// always_prep: re-split M_r into the tf32 ring chunks before this batch (data parallel:
// the dense step outside the kernel moved proj), otherwise only at batch 0
void launch_transr_train_tc(bool l2, const FwdArgs& fa, const uint32_t* ent_val, const uint32_t* seg_start,
                            const uint32_t* seg_col, const uint32_t* tile_seg, const uint32_t* tile_p0,
                            const uint32_t* tile_total, const uint32_t* seg_tiles, float* dm_part, float* dr_part,
                            float* mr, int64_t R, int num_sms, cudaStream_t s, bool always_prep = false);

// link-prediction ranking (eval.cu)
bool eval_supported(int kind);
bool eval_exact(int kind);
void eval_project(int kind, const float* E, const float* proj, const float* normals, int64_t r, int64_t N, int de,
                  int dr, float* out, cudaStream_t s);
void configure_eval_kernels();
uint64_t eval_filter_capacity(int64_t nf);
void eval_build_filter(const int32_t* h, const int32_t* r, const int32_t* t, int64_t nf, int64_t N, int64_t R,
                       uint64_t* table, uint64_t cap, cudaStream_t s);
void eval_rank(int kind, const float* X, const float* Rt, int64_t N, int64_t R, int d, const int32_t* qh,
               const int32_t* qr, const int32_t* qt, int64_t q, const uint64_t* table, uint64_t cap, uint32_t* better,
               float* te, int num_sms, cudaStream_t s);

// data parallel (dp.cu)
void dp_destroy(skg_ctx* ctx);
int dp_rank(const skg_ctx* ctx);
int dp_world(const skg_ctx* ctx);
const void* dp_comm_tag(const skg_ctx* ctx);
int shard_rank(const skg_ctx* ctx);
uint64_t shard_tag(const skg_ctx* ctx);
int shard_world(const skg_ctx* ctx);  // identity of the communicator (graph keys)
void drop_graphs(skg_ctx* ctx);               // destroys captured epoch graphs and plan-slot keys
void dp_allreduce_sum(skg_ctx* ctx, float* buf, int64_t n, cudaStream_t s);

}  // namespace skg
