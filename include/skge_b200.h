/* skge_b200.h — C ABI of the B200-native SparseTransX training engine.
 *
 * This is the drop-in boundary for the reference hot path (libsparsekge,
 * /root/reference/proj). The reference has no FFI layer: it is a C++ static
 * library whose callers (tools/kge.cpp, the doctest suites) call templated
 * C++ functions. Each entry point below names the reference function it
 * replaces (file:line under proj/). The C++ shim include/skge_b200.hpp
 * re-exposes the reference signatures (skge::score_batch, skge::fit, ...)
 * over these symbols and rethrows the reference exception types.
 *
 * Conventions
 *  - Plain pointers and sizes only; host arrays are borrowed for the call.
 *  - Ids are int64 on the boundary (reference Index = Eigen::Index) and are
 *    narrowed to int32 in HBM.
 *  - Tables are fp32 row-major, exactly the reference SPARSEKGE_REAL32 layout
 *    (embedding.hpp:15-31); TransR proj is R x (d_r*d_e), row r viewed as a
 *    d_r x d_e row-major matrix (models.cpp:127).
 *  - Every call returns skg_status; skg_last_error(ctx) holds the message the
 *    reference would have thrown. No exceptions cross the ABI.
 *  - One host thread per context; a context owns one device, two streams and
 *    all device buffers. No CPU fallback: every compute entry point runs CUDA
 *    kernels on the context's device or fails with SKG_ERR_CUDA.
 */
#ifndef SKGE_B200_H
#define SKGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum skg_status {
  SKG_OK = 0,
  SKG_ERR_SHAPE = 1,      /* ShapeError            common.hpp:37 */
  SKG_ERR_CONFIG = 2,     /* ConfigError           common.hpp:42 */
  SKG_ERR_DEGENERATE = 3, /* DegenerateTripleError common.hpp:47 */
  SKG_ERR_TRAINING = 4,   /* TrainingError         common.hpp:52 */
  SKG_ERR_PARSE = 5,      /* ParseError            common.hpp:57 */
  SKG_ERR_CUDA = 6        /* device/runtime failure (no reference analogue) */
} skg_status;

/* ModelKind tags (common.hpp:62-70). ComplEx and RotatE use complex stores:
 * every table row holds dim interleaved (re, im) float pairs, the reference's
 * std::complex<float> row-major layout (embedding.hpp:15-31), so a complex
 * table of dim d is passed as 2*d floats per row. Norm is ignored by the
 * multiplicative family, as in the reference. */
enum { SKG_TRANSE = 0, SKG_TRANSR = 1, SKG_TRANSH = 2, SKG_TORUSE = 3,
       SKG_DISTMULT = 4, SKG_COMPLEX = 5, SKG_ROTATE = 6 };
/* NormKind (common.hpp:72) */
enum { SKG_L1 = 0, SKG_L2 = 1 };
/* Incidence layouts: build_ht (incidence.hpp:38), build_hrt (:62),
 * build_multiplicative (:93) without / with the conjugate tail marker */
enum { SKG_LAYOUT_HT = 0, SKG_LAYOUT_HRT = 1, SKG_LAYOUT_MULT = 2, SKG_LAYOUT_MULT_CONJ = 3 };

typedef struct skg_model_config { /* ModelConfig, models.hpp:17-30 */
  uint32_t model;
  uint32_t norm;
  int64_t dim_entity;
  int64_t dim_relation;
} skg_model_config;

typedef struct skg_train_config { /* TrainConfig, training.hpp:29-50 */
  float lr;
  float margin;
  int64_t epochs;
  int64_t batch_size;
  uint64_t seed;
  int32_t has_scheduler; /* std::optional<StepDecay> */
  int64_t decay_every;
  float decay_factor;
  int32_t shuffle;
  int32_t resample_negatives;
  int32_t renorm_entities;
} skg_train_config;

typedef struct skg_epoch_report { /* EpochReport, training.hpp:74-80 */
  int64_t epoch;
  double loss;
  /* PhaseTimer buckets (training.cpp:15-20, 126, 141, 158), device time from
   * event-record nodes inside the epoch graph (skg_set_phase_timers). */
  double t_forward_s;  /* forward kernels: gather, score, hinge, loss      */
  double t_backward_s; /* transposed-SpMM backward with the fused SGD step  */
  double t_step_s;     /* standalone step kernels (0: the step is fused)   */
} skg_epoch_report;

typedef struct skg_ctx skg_ctx;

/* ---- context ------------------------------------------------------------ */
skg_status skg_create(int device, skg_ctx** out);
void skg_destroy(skg_ctx* ctx);
const char* skg_last_error(const skg_ctx* ctx); /* ctx may be NULL (create errors) */
const char* skg_version(void);
int skg_num_sms(const skg_ctx* ctx);

/* ---- parameter store (EmbeddingStoreT, embedding.hpp:15-31) -------------- */
/* Uploads fp32 tables into HBM. proj (TransR) / normals (TransH) may be NULL
 * when the model does not use them. Validates like check_config. */
skg_status skg_store_upload(skg_ctx* ctx, const skg_model_config* cfg, int64_t num_entities,
                            int64_t num_relations, const float* entity, const float* relation,
                            const float* proj, const float* normals);
skg_status skg_store_download(skg_ctx* ctx, float* entity, float* relation, float* proj,
                              float* normals);
/* sgd_step, embedding.cpp:165-190: store -= lr * grads, normals renormalized.
 * Grads are host tables shaped like the store; non-finite -> SKG_ERR_TRAINING. */
skg_status skg_sgd_step(skg_ctx* ctx, const float* g_entity, const float* g_relation,
                        const float* g_proj, const float* g_normals, float lr);
/* ---- checkpoints (embedding.cpp:35-125, 200-251: SKGECKPT v1) ------------
 * Host-side file I/O on host tables (download / upload the device store
 * around them). f64 on disk, fp32 in memory, exactly like the reference's
 * 32-bit build. Real-valued model tags only (0 TransE .. 3 TorusE); errors:
 * SKG_ERR_PARSE / SKG_ERR_CONFIG with skg_checkpoint_last_error(). */
typedef struct skg_checkpoint_header { /* CheckpointHeader, embedding.hpp:134-140 */
  uint32_t model;
  int64_t num_entities, num_relations, dim_entity, dim_relation;
} skg_checkpoint_header;
skg_status skg_peek_checkpoint(const char* path, skg_checkpoint_header* out);
skg_status skg_save_checkpoint(const char* path, uint32_t model, int64_t num_entities, int64_t num_relations,
                               int64_t dim_entity, int64_t dim_relation, const float* entity, const float* relation,
                               const float* proj, const float* normals);
skg_status skg_load_checkpoint(const char* path, uint32_t expected_model, float* entity, float* relation,
                               float* proj, float* normals);
const char* skg_checkpoint_last_error(void);

/* renormalize_entities, embedding.cpp:192-198 */
skg_status skg_renormalize_entities(skg_ctx* ctx);

/* ---- triples and negatives ------------------------------------------------ */
/* Training triples (TripleBatch, incidence.hpp:14-33) with their id space;
 * validated like TripleBatch::validate (ShapeError on a bad id).
 * By default the arrays are copied and validated inside the call (the
 * reference's by-value TripleBatch semantics).
 * Deferred re-upload (opt-in, skg_set_deferred_uploads): when the context
 * already holds triples + negatives of the same shape and the new arrays are
 * page-locked (cudaHostAlloc / torch pin_memory), skg_set_triples +
 * skg_set_negatives only record the pointers; the next skg_train_epoch copies
 * and validates them while it trains (an invalid id then fails that call with
 * the same ShapeError, the parameters untouched). Deferred arrays must stay
 * valid and unmodified until that skg_train_epoch RETURNS (any other engine
 * call applies the pending upload synchronously first). Pageable arrays are
 * never deferred. */
skg_status skg_set_deferred_uploads(skg_ctx* ctx, int32_t enable); /* default 0 (off) */
/* Deferred re-uploads so far: kept (identical data) / rolled back + retrained. */
skg_status skg_upload_stats(skg_ctx* ctx, int64_t* hits, int64_t* misses);
/* Bytes copied host -> device by deferred re-uploads so far: the five id arrays
 * narrowed by host threads (range-checked on the way) to uint16 when every
 * table has at most 65536 rows, else to int32; int64 with SKG_SPEC_I64=1. */
skg_status skg_upload_bytes(skg_ctx* ctx, int64_t* bytes);
skg_status skg_set_triples(skg_ctx* ctx, int64_t m, const int64_t* heads, const int64_t* relations,
                           const int64_t* tails, int64_t num_entities, int64_t num_relations);
/* Corrupted tails/heads aligned with the training triples (NegativeSet,
 * training.hpp:53-55), e.g. produced by the caller's own sampler. */
skg_status skg_set_negatives(skg_ctx* ctx, int64_t m, const int64_t* neg_heads,
                             const int64_t* neg_tails);
/* negative_sample, training.cpp:51-71: bit-exact libstdc++ mt19937_64 +
 * Lemire stream, generated on device for the context's triples. Results stay
 * resident as the context's negatives; out_* (may be NULL) receive a copy. */
skg_status skg_negative_sample(skg_ctx* ctx, uint64_t seed, int32_t avoid_self_loops,
                               int64_t* out_heads, int64_t* out_tails);
/* The epoch permutation of train_epoch, training.cpp:106-112 (std::shuffle
 * with mt19937_64(seed ^ 0x9E3779B97F4A7C15*(epoch+1))), built on device. */
skg_status skg_epoch_order(skg_ctx* ctx, int64_t m, uint64_t seed, int32_t shuffle, int64_t epoch,
                           int64_t* out_order);

/* ---- incidence and SpMM (parity surface) --------------------------------- */
/* build_ht / build_hrt + coo_to_csr (incidence.hpp:38-85, sparse.hpp:110-161)
 * on device. row_ptr has m+1 slots; col/val hold up to 3m; *nnz receives nnz. */
skg_status skg_build_incidence(skg_ctx* ctx, int32_t layout, int64_t m, const int64_t* heads,
                               const int64_t* relations, const int64_t* tails,
                               int64_t num_entities, int64_t num_relations, int64_t* row_ptr,
                               int64_t* col_idx, float* vals, int64_t* nnz);
/* The reference's generic plus-times sparse layer (sparse.hpp:110-306) on
 * device, host arrays in and out (int64 indices, fp32 values):
 *  coo_to_csr (sparse.hpp:110-161): canonical CSR, columns ascending per row,
 *    duplicates summed left to right in input order (std::sort's order for
 *    rows of <= 16 entries), exact zeros dropped. row_ptr: num_rows + 1;
 *    col_idx / out_vals: room for nnz; *out_nnz receives the canonical nnz.
 *  csr_transpose (sparse.hpp:164-183): stable counting sort over columns.
 *    t_row_ptr: num_cols + 1; t_col_idx / t_vals: row_ptr[num_rows].
 *  spmm (sparse.hpp:211-266): out (num_rows x d) = A X, X is x_rows x d.
 *  spmm_transpose_add (sparse.hpp:273-306): sink (num_cols x d) += A^T G,
 *    G is g_rows x d; each sink row accumulates over ascending source rows. */
skg_status skg_coo_to_csr(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, int64_t nnz, const int64_t* rows,
                          const int64_t* cols, const float* vals, int64_t* row_ptr, int64_t* col_idx,
                          float* out_vals, int64_t* out_nnz);
skg_status skg_csr_transpose(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                             const int64_t* col_idx, const float* vals, int64_t* t_row_ptr, int64_t* t_col_idx,
                             float* t_vals);
skg_status skg_spmm(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                    const int64_t* col_idx, const float* vals, int64_t x_rows, int64_t d, const float* x,
                    float* out);
skg_status skg_spmm_transpose_add(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                                  const int64_t* col_idx, const float* vals, int64_t g_rows, int64_t d,
                                  const float* g, float* sink);
/* score_batch, models.cpp:267-289, against the uploaded store. residual
 * (nullable) receives v (TransE/TransH/TransR, m x d_r) or delta (TorusE). */
skg_status skg_score_batch(skg_ctx* ctx, const skg_model_config* cfg, int64_t m,
                           const int64_t* heads, const int64_t* relations, const int64_t* tails,
                           float* scores, float* residual);
/* score_backward, models.cpp:291-325: ACCUMULATES d(sum up_i score_i) into
 * the host gradient tables (shaped like the store; NULL for absent tables). */
skg_status skg_score_backward(skg_ctx* ctx, const skg_model_config* cfg, int64_t m,
                              const int64_t* heads, const int64_t* relations,
                              const int64_t* tails, const float* upstream, float* g_entity,
                              float* g_relation, float* g_proj, float* g_normals);
/* rank_entity (eval.cpp:16-63) of q queries on device, tail side then head side
 * (the order evaluate() visits them, eval.cpp:80-86): ranks[2i] = tail rank,
 * ranks[2i + 1] = head rank, rank = 1 + #{c != truth : energy(c) < energy(truth)}.
 * protocol 1 (filtered) skips candidates whose triple is one of the nf filter
 * triples (TripleFilter / build_filter, eval.hpp:25-48); 0 = raw. TransE and
 * TorusE energies are bit-exact; TransH / TransR rank against per-relation
 * projected entity tables (P_r a - P_r b + r, equal to the reference's
 * P_r (a - b) + r up to rounding: these models are tolerance-only). */
skg_status skg_rank_entities(skg_ctx* ctx, const skg_model_config* cfg, int64_t q, const int64_t* heads,
                             const int64_t* relations, const int64_t* tails, int32_t protocol, int64_t nf,
                             const int64_t* filter_heads, const int64_t* filter_relations,
                             const int64_t* filter_tails, int64_t* ranks);
/* margin_ranking_loss, training.cpp:73-94 */
skg_status skg_margin_ranking_loss(skg_ctx* ctx, int64_t m, const float* pos_energy,
                                   const float* neg_energy, float margin, float* loss,
                                   float* d_pos, float* d_neg);

/* ---- training loop ------------------------------------------------------- */
/* train_epoch, training.cpp:96-164, over the context's triples and negatives:
 * per-epoch permutation, then per minibatch the fused forward (gather, score,
 * hinge, loss) and the fused transposed-SpMM backward + SGD step, all on
 * device and captured once in a CUDA graph. One device->host read per epoch. */
skg_status skg_train_epoch(skg_ctx* ctx, const skg_model_config* cfg, const skg_train_config* tc,
                           int64_t epoch, float lr, skg_epoch_report* report);
/* fit, training.cpp:166-195: negatives once (or per epoch), lr schedule,
 * optional entity renorm. reports has room for tc->epochs entries. */
skg_status skg_fit(skg_ctx* ctx, const skg_model_config* cfg, const skg_train_config* tc,
                   skg_epoch_report* reports);
/* Per-phase device timing of one epoch, phases in sequence (no overlap): the
 * epoch is captured into a graph whose event record nodes bracket the shuffle,
 * the incidence plan and every forward / backward (measurement hook for
 * bench.py). plan_ms excludes the shuffle; skg_profile_shuffle_ms reports it. */
skg_status skg_profile_epoch(skg_ctx* ctx, const skg_model_config* cfg,
                             const skg_train_config* tc, int64_t epoch, float lr,
                             skg_epoch_report* report, double* fwd_ms_per_batch,
                             double* bwd_ms_per_batch, double* plan_ms);
skg_status skg_profile_shuffle_ms(skg_ctx* ctx, double* shuffle_ms);
/* Phase buckets of the epoch report, default on. Off: t_forward_s = 0 and
 * t_backward_s = the whole epoch's device time (no event nodes in the graph). */
skg_status skg_set_phase_timers(skg_ctx* ctx, int32_t enable);
/* Number of CUDA kernels the last skg_train_epoch launched (graph nodes). */
int64_t skg_last_launch_count(const skg_ctx* ctx);
/* Synchronizes the context's streams. */
skg_status skg_synchronize(skg_ctx* ctx);

/* ---- host setup utilities (once per job, not on the hot path) ------------ */
/* generate_synthetic, data_io.cpp:128-211: triples in generation order; the
 * split is [0, n/20) test, next n/20 valid, rest train. */
skg_status skg_generate_synthetic(int64_t n_entities, int64_t n_relations, int64_t n_triples,
                                  uint64_t seed, int64_t* heads, int64_t* relations, int64_t* tails);
/* init_store, embedding.cpp:129-163 (fp32 tables; proj/normals may be NULL). */
skg_status skg_init_store(uint32_t model, int64_t num_entities, int64_t num_relations,
                          int64_t dim_entity, int64_t dim_relation, uint64_t seed, float* entity,
                          float* relation, float* proj, float* normals);
const char* skg_host_last_error(void);

/* ---- measurement hooks ----------------------------------------------------- */
/* Random-row gather bandwidth (GB/s) over a table of table_bytes with rows of
 * row_floats floats (128-bit loads, full occupancy): the roofline denominator
 * for the gather kernels when the table is L2-resident (C1-C4). */
skg_status skg_measure_gather(skg_ctx* ctx, int64_t table_bytes, int32_t row_floats, double* gbs);
/* Overwrites a 256 MiB scratch buffer on the context stream (evicts L2). */
skg_status skg_flush_l2(skg_ctx* ctx);
/* Plan statistics of minibatch `batch` of the last epoch: touched columns
 * (segments) and incidence entries (valid nnz of the transposed matrix). */
skg_status skg_plan_stats(skg_ctx* ctx, int64_t batch, int64_t* segments, int64_t* entries,
                          int64_t* relation_segments);

/* Tensor-core self test: D = A(m,k) . B(n,k) over 128^3 through the operand
 * views the TransR kernel uses (0: A,B K-major; 1: B MN-major; 2: both MN). */
skg_status skg_debug_tc_gemm(skg_ctx* ctx, int32_t mode, const float* A, const float* B, float* D);
/* Host-only check of the MT19937-64 jump-ahead (sampling streams): the state
 * J words ahead of std::mt19937_64(seed), from the jump polynomial, continues
 * the reference stream exactly. Returns 1 on success. */
int32_t skg_debug_mt_jump_selftest(uint64_t seed, int64_t jump);

/* ---- data-parallel replicas (one process per GPU) ------------------------ */
/* Joins an NCCL communicator (unique id produced by skg_nccl_unique_id on
 * rank 0 and broadcast by the caller). After this, skg_train_epoch treats the
 * context as rank `rank` of `world`: each global minibatch is split into
 * world contiguous shards, gradients are summed over NVLink, and every rank
 * applies the identical update (replicated tables). */
skg_status skg_nccl_unique_id(char out[128]);
skg_status skg_dp_init(skg_ctx* ctx, const char unique_id[128], int rank, int world);
/* Host-only: the shard rank `rank` of `world` trains in every global minibatch
 * (training.cpp:120-121 batches of batch_size): out = {pairs per full
 * minibatch, first pair of the last minibatch's shard, its size, pairs over
 * the epoch, minibatches}. */
skg_status skg_dp_shard(int64_t m, int64_t batch_size, int32_t world, int32_t rank, int64_t* out);

/* ---- run artifacts of `kge train` (tools/kge.cpp:181-247) -----------------
 * Host-side writers: train_log.jsonl (one compact JSON record per epoch,
 * flushed per line), loss.log ("<epoch> <loss %.17g>") and summary.json, in
 * the reference's formats (nlohmann::json output: sorted keys, shortest
 * round-trip doubles). Open appends to the files under out_dir (created if
 * needed); errors: SKG_ERR_PARSE with skg_run_log_last_error(). */
typedef struct skg_run_log skg_run_log;
typedef struct skg_run_summary { /* the parts of summary.json the engine cannot know */
  const char* engine;          /* "sparse" | "dense" (the CLI's --engine) */
  const char* dataset_source;  /* "synthetic" or the dataset directory */
  int64_t entities, relations, train, valid, test, dropped_valid, dropped_test;
  int32_t threads;
  int64_t epochs_run;          /* TrainingRun::epochs.size() */
  double final_loss;           /* TrainingRun::final_loss() */
  double t_forward_s, t_backward_s, t_step_s; /* TrainingRun totals */
  const char* checkpoint_path; /* NULL: <out_dir>/checkpoint.bin */
} skg_run_summary;
skg_status skg_run_log_open(const char* out_dir, skg_run_log** out);
skg_status skg_run_log_epoch(skg_run_log* log, const skg_epoch_report* report);
skg_status skg_run_log_summary(skg_run_log* log, const skg_model_config* cfg, const skg_train_config* tc,
                               const skg_run_summary* info);
void skg_run_log_close(skg_run_log* log);
const char* skg_run_log_last_error(void);

/* ---- row-sharded data parallel (wikikg2-scale tables) ---------
 * TransE / TorusE. The entity table is split by owner (entity e on rank e % G,
 * G in {1, 2, 4, 8}) and the relation table replicated; each global minibatch
 * (training.cpp:120-161 at batch_size = global batch) is split into G pair
 * shards. Per batch every rank runs the forward of its shard, gathering entity
 * rows from their owners over NVLink; after a barrier every rank reduces the
 * columns it owns over the WHOLE global batch in the reference's order
 * (pulling residual rows from the ranks that computed them) and applies SGD;
 * relation owners write the new row into every replica; a second barrier.
 * Results equal the single-device run at batch_size = global batch bit for
 * bit (tables; the loss within 1e-5: shard losses are summed per rank).
 * Set up after store upload, triples and negatives; batch_size is the GLOBAL
 * batch and must be a multiple of G. skg_store_download gathers the full
 * tables from all ranks; skg_store_upload re-scatters.
 *
 * One process driving all ranks (contexts on distinct GPUs, or on one GPU):
 *   skg_shard_group_init + skg_shard_group_train_epoch (ctxs[k] = rank k).
 * One process per GPU: skg_shard_export (this rank's IPC handle) on every
 * rank, an all-gather of the handles by the caller, skg_shard_import (all G
 * handles, rank order); then skg_train_epoch / skg_fit run sharded. */
#define SKG_SHARD_HANDLE_BYTES 128
skg_status skg_shard_group_init(skg_ctx* const* ctxs, int world, int64_t batch_size);
skg_status skg_shard_group_train_epoch(skg_ctx* const* ctxs, int world, const skg_model_config* cfg,
                                       const skg_train_config* tc, int64_t epoch, float lr,
                                       skg_epoch_report* reports);
skg_status skg_shard_export(skg_ctx* ctx, int rank, int world, int64_t batch_size, void* handle);
skg_status skg_shard_import(skg_ctx* ctx, const void* handles);
skg_status skg_shard_release(skg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SKGE_B200_H */
