// C ABI implementation: context, store, triples, per-op parity surface and the
// device training loop (train_epoch / fit) captured in one CUDA graph per
// epoch shape.
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <cstring>
#include <sstream>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "ht.cuh"
#include "primitives.cuh"
#include "shard.cuh"

using namespace skg;

namespace {
int grid_for(int64_t n);
void resolve_pending(skg_ctx* ctx);

thread_local std::string g_create_err;

const char* model_name(uint32_t m) {  // common.hpp:82-93
  switch (m) {
    case SKG_TRANSE: return "transe";
    case SKG_TRANSR: return "transr";
    case SKG_TRANSH: return "transh";
    case SKG_TORUSE: return "toruse";
    case SKG_DISTMULT: return "distmult";
    case SKG_COMPLEX: return "complex";
    case SKG_ROTATE: return "rotate";
  }
  return "unknown";
}

template <class F>
skg_status guard(skg_ctx* ctx, F&& f) {
  try {
    if (ctx) SKG_CUDA(cudaSetDevice(ctx->device));
    f();
    return SKG_OK;
  } catch (const ShapeError& e) {
    if (ctx) ctx->err = e.what();
    return SKG_ERR_SHAPE;
  } catch (const ConfigError& e) {
    if (ctx) ctx->err = e.what();
    return SKG_ERR_CONFIG;
  } catch (const TrainingError& e) {
    if (ctx) ctx->err = e.what();
    return SKG_ERR_TRAINING;
  } catch (const DegenerateTripleError& e) {
    if (ctx) ctx->err = e.what();
    return SKG_ERR_DEGENERATE;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return SKG_ERR_CUDA;
  }
}

int kind_of(const skg_model_config& c) {
  const bool l2 = c.norm == SKG_L2;
  switch (c.model) {
    case SKG_TRANSE: return l2 ? kTransE_L2 : kTransE_L1;
    case SKG_TORUSE: return l2 ? kTorusE_L2 : kTorusE_L1;
    case SKG_TRANSH: return l2 ? kTransH_L2 : kTransH_L1;
    case SKG_TRANSR: return l2 ? kTransR_L2 : kTransR_L1;
    case SKG_DISTMULT: return kDistMult;
    case SKG_COMPLEX: return kComplEx;
    case SKG_ROTATE: return kRotatE;
  }
  throw ConfigError("unknown model tag " + std::to_string(c.model));
}

bool is_ht(const skg_model_config& c) { return c.model == SKG_TRANSH || c.model == SKG_TRANSR; }
bool is_mult(const skg_model_config& c) { return c.model >= SKG_DISTMULT && c.model <= SKG_ROTATE; }  // common.hpp:80-82
bool is_complex(uint32_t m) { return m == SKG_COMPLEX || m == SKG_ROTATE; }                        // common.hpp:74-76
int64_t width(uint32_t m, int64_t dim) { return is_complex(m) ? 2 * dim : dim; }  // floats per table row

void validate_model(const skg_model_config& c) {  // models.hpp:23-29
  if (c.model > SKG_ROTATE) throw ConfigError("unknown model tag " + std::to_string(c.model));
  if (c.norm > SKG_L2) throw ConfigError("unknown norm tag " + std::to_string(c.norm));
  if (c.dim_entity < 1 || c.dim_relation < 1) throw ConfigError("embedding dimensions must be at least 1");
  if (c.model != SKG_TRANSR && c.dim_relation != c.dim_entity)
    throw ConfigError(std::string(model_name(c.model)) + " requires dim_relation == dim_entity");
}

void check_config(skg_ctx* ctx, const skg_model_config& c, int64_t n_ent, int64_t n_rel) {  // models.hpp:65-76
  validate_model(c);
  if (!ctx->has_store) throw ConfigError("no parameter store uploaded");
  // score_batch<Real> / <Complex> dispatch (models.cpp:267-289): the store's scalar type must match
  if (is_complex(c.model) && !is_complex(ctx->cfg.model))
    throw ConfigError(std::string(model_name(c.model)) + " needs a complex-valued store");
  if (!is_complex(c.model) && is_complex(ctx->cfg.model))
    throw ConfigError(std::string(model_name(c.model)) + " uses a real-valued store");
  if (ctx->de != width(c.model, c.dim_entity) || ctx->dr != width(c.model, c.dim_relation))
    throw ConfigError("store dimensions do not match the model config");
  if (ctx->N != n_ent || ctx->R != n_rel)
    throw ConfigError("store table sizes do not match the batch id space");
  if (c.model == SKG_TRANSR && ctx->proj.n == 0) throw ConfigError("transr store is missing the projection table");
  if (c.model == SKG_TRANSH && ctx->normals.n == 0)
    throw ConfigError("transh store is missing the hyperplane normals");
}

void validate_train(const skg_train_config& t) {  // training.hpp:42-49
  if (t.batch_size < 1) throw ConfigError("batch_size must be at least 1");
  if (!(t.margin >= 0.f)) throw ConfigError("margin must be nonnegative");
  if (!(t.lr >= 0.f) || !std::isfinite(t.lr)) throw ConfigError("lr must be finite and >= 0");
  if (t.epochs < 0) throw ConfigError("epochs must be nonnegative");
  if (t.has_scheduler && (t.decay_every < 1 || !(t.decay_factor > 0.f)))
    throw ConfigError("scheduler needs every_epochs >= 1 and a positive factor");
}

// TripleBatch::validate (incidence.hpp:23-32) + narrowing to int32 for HBM.
void validate_ids(int64_t m, const int64_t* h, const int64_t* r, const int64_t* t, int64_t n_ent,
                  int64_t n_rel, std::vector<int32_t>& out) {
  if (m > 0 && (!h || !r || !t)) throw ShapeError("triple batch: heads/relations/tails length mismatch");
  if (n_ent > INT32_MAX || n_rel > INT32_MAX) throw ShapeError("id space exceeds 32-bit device ids");
  out.resize(3 * static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) {
    if (h[i] < 0 || h[i] >= n_ent || t[i] < 0 || t[i] >= n_ent)
      throw ShapeError("triple " + std::to_string(i) + ": entity id out of range");
    if (r[i] < 0 || r[i] >= n_rel) throw ShapeError("triple " + std::to_string(i) + ": relation id out of range");
    out[i] = static_cast<int32_t>(h[i]);
    out[m + i] = static_cast<int32_t>(r[i]);
    out[2 * m + i] = static_cast<int32_t>(t[i]);
  }
}

// Uploads ids into ctx->tmp_i32: [h | r | t].
void upload_ids(skg_ctx* ctx, int64_t m, const int64_t* h, const int64_t* r, const int64_t* t,
                int64_t n_ent, int64_t n_rel) {
  std::vector<int32_t> host;
  validate_ids(m, h, r, t, n_ent, n_rel, host);
  ctx->tmp_i32.ensure(3 * m + 1);
  if (m > 0)
    SKG_CUDA(cudaMemcpyAsync(ctx->tmp_i32.p, host.data(), sizeof(int32_t) * 3 * m,
                             cudaMemcpyHostToDevice, ctx->stream));
}

// build_multiplicative (incidence.hpp:104-108): the first head == tail triple.
void reject_self_loops(int64_t m, const int64_t* h, const int64_t* t) {
  for (int64_t i = 0; i < m; ++i)
    if (h[i] == t[i])
      throw DegenerateTripleError("triple " + std::to_string(i) +
                                  ": head == tail is not representable in the "
                                  "multiplicative incidence layout");
}

void ensure_workspace(skg_ctx* ctx, int64_t rows, int kind) {
  const int64_t d = std::max(ctx->de, ctx->dr);
  ctx->res.ensure(rows * d * (is_mult_kind(kind) ? 3 : 1));  // multiplicative: 3 gradient planes
  // TransR tcgen05 training writes dU in tile-blocked slots (kTileSlotRows): up to R + 1 partial tiles more
  const bool tile_rows = (kind == kTransR_L2 || kind == kTransR_L1) &&
                         transr_train_tc_supported(static_cast<int>(ctx->de), static_cast<int>(ctx->dr));
  ctx->res_u.ensure(tile_rows ? std::max(rows * ctx->de, tile_rows_floats(rows, ctx->R)) : rows * ctx->de);
  ctx->scal.ensure(rows);
  ctx->scores.ensure(rows);
  ctx->block_partial.ensure(static_cast<int64_t>(ctx->num_sms) * 16 + 64);
}

FwdArgs base_fwd(skg_ctx* ctx) {
  FwdArgs a{};
  a.X = ctx->tables.p;
  a.proj = ctx->proj.p;
  a.normals = ctx->normals.p;
  a.N = ctx->N;
  a.de = static_cast<int>(ctx->de);
  a.dr = static_cast<int>(ctx->dr);
  a.res = ctx->res.p;
  a.res_u = ctx->res_u.p;
  a.scal = ctx->scal.p;
  a.scores = ctx->scores.p;
  a.block_partial = ctx->block_partial.p;
  a.counter = ctx->counter.p;
  a.batch_loss = ctx->batch_loss.p;
  a.err = ctx->err_words.p;
  a.sign = 1.f;
  return a;
}

void set_stamps(skg_ctx* ctx, FwdArgs& fa, int64_t b) {
  if (!ctx->phase_timers || ctx->stamps.n < 2 * (b + 1)) return;
  fa.stamp_start = ctx->stamps.p + 2 * b;
  fa.stamp_end = ctx->stamps.p + 2 * b + 1;
}

void reset_err(skg_ctx* ctx, cudaStream_t s) {
  SKG_CUDA(cudaMemsetAsync(ctx->err_words.p, 0, sizeof(uint32_t) * 4, s));
  SKG_CUDA(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned), s));
}
void reset_err(skg_ctx* ctx) { reset_err(ctx, ctx->stream); }

// Error word -> reference exception (training.cpp:135-137, embedding.cpp:173-186).
void raise_device_error(const uint32_t* w, int64_t epoch) {
  switch (w[0]) {
    case kErrNone: return;
    case kErrLossNonFinite:
      throw TrainingError("non-finite loss at epoch " + std::to_string(epoch) + ", batch " + std::to_string(w[1]));
    case kErrGradEntity: throw TrainingError("non-finite gradient in entity embeddings");
    case kErrGradRelation: throw TrainingError("non-finite gradient in relation embeddings");
    case kErrGradProj: throw TrainingError("non-finite gradient in relation projections");
    case kErrGradNormals: throw TrainingError("non-finite gradient in hyperplane normals");
    case kErrNormalCollapsed:
      throw TrainingError("hyperplane normal " + std::to_string(w[2]) + " collapsed to zero");
    case 8u: throw CudaError("sharded data parallel: a peer rank did not reach the barrier within 20 s");
    default: throw CudaError("device error word " + std::to_string(w[0]));
  }
}

uint64_t epoch_seed(uint64_t seed, int64_t epoch) {  // training.cpp:109-110
  return seed ^ (0x9E3779B97F4A7C15ULL * static_cast<uint64_t>(epoch + 1));
}

// ----------------------------------------------------------------- epoch body

// Data-parallel shard of rank `rank` in every global minibatch of B pairs
// (last minibatch Bl = M - (nb-1) B): full minibatches give each rank B/world
// contiguous pairs, the last one ceil(Bl/world) (the tail ranks may get fewer
// or none). out = {S, i0_last, s_last, Mg, nb}.
void dp_shard(int64_t M, int64_t B, int world, int rank, int64_t* out) {
  const int64_t nb = (M + B - 1) / B;
  const int64_t S = B / world;
  const int64_t Bl = M - (nb - 1) * B;
  const int64_t Sl = (Bl + world - 1) / world;
  const int64_t i0 = std::min<int64_t>(rank * Sl, Bl);
  const int64_t sl = std::min<int64_t>(i0 + Sl, Bl) - i0;
  out[0] = S;
  out[1] = i0;
  out[2] = sl;
  out[3] = (nb - 1) * S + sl;
  out[4] = nb;
}

struct EpochShape {
  int64_t B, nb;
  bool shuffle;
  int kind;
  // data parallel: this rank's shard of every global minibatch
  int world = 1, rank = 0;
  int64_t S = 0;        // shard size of full minibatches (B / world)
  int64_t i0_last = 0;  // shard start inside the last minibatch
  int64_t s_last = 0;   // shard size of the last minibatch (may be 0)
  int64_t Mg = 0;       // rows of this rank's shards over the epoch
  int64_t nb_run = -1;  // run only the first nb_run minibatches (-1: all)
};

// Multiplicative models: positions (in epoch order) of the first positive and
// first negative self-loop triple, which build_multiplicative rejects.
__global__ void first_loop_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ H,
                                  const int32_t* __restrict__ T, const int32_t* __restrict__ NH,
                                  const int32_t* __restrict__ NT, int64_t M, uint32_t* __restrict__ first) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < M;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = order ? order[k] : static_cast<int32_t>(k);
    if (H[id] == T[id]) atomicMin(first, static_cast<uint32_t>(k));
    if (NH[id] == NT[id]) atomicMin(first + 1, static_cast<uint32_t>(k));
  }
}

__global__ void shard_order_kernel(const int32_t* __restrict__ order, int64_t B, int64_t S, int rank,
                                   int64_t nb, int64_t i0_last, int64_t Mg, int32_t* __restrict__ order_g) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < Mg;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = j / S;
    order_g[j] = b < nb - 1 ? order[b * B + rank * S + (j - b * S)]
                            : order[(nb - 1) * B + i0_last + (j - (nb - 1) * S)];
  }
}

__global__ void dp_flags_kernel(const uint32_t* __restrict__ err, float* __restrict__ flags) {
  flags[0] = err[0] == kErrLossNonFinite ? 1.f : 0.f;
  flags[1] = (err[0] >= kErrGradEntity && err[0] <= kErrGradNormals) ? 1.f : 0.f;
}

// Dense step p -= lr * g after the all-reduce; any rank's flag stops every rank.
__global__ void dp_sgd_kernel(float* __restrict__ X, const float* __restrict__ G, int64_t n,
                              const float* __restrict__ lr, const float* __restrict__ flags,
                              uint32_t* __restrict__ err, int batch) {
  if (flags[0] > 0.f || flags[1] > 0.f) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const uint32_t code = flags[0] > 0.f ? kErrLossNonFinite : kErrGradEntity;
      if (atomicCAS(&err[0], 0u, code) == 0u) err[1] = static_cast<uint32_t>(batch);
    }
    return;
  }
  if (err[0] != 0) return;
  const float step = *lr;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    X[i] = __fsub_rn(X[i], __fmul_rn(step, G[i]));
}

// Enqueues one whole epoch on ctx->stream: permutation, plan, then per batch
// the fused forward and the fused backward + SGD. When `ev` is non-null the
// phases are bracketed with events (profiling; not used under capture).
void enqueue_plan(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s);
void enqueue_batches(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s,
                     const std::function<void()>* markp);
void enqueue_shard_batches(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s,
                           const std::function<void()>* markp);

// Row-sharded epoch (shard.cu): per global batch, the forward of this rank's
// pair shard (entity rows gathered from their owners over NVLink), a barrier,
// the owner-side reduce + SGD of the columns this rank owns (residual rows
// pulled from the ranks that computed them), a barrier.
void enqueue_shard_batches(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s,
                           const std::function<void()>* markp) {
  auto mark = [&]() {
    if (markp) (*markp)();
  };
  ShardState* st = ctx->shard;
  const ShardPlanBufs& sp = st->plan[slot];
  reset_err(ctx, s);
  SKG_CUDA(cudaMemsetAsync(st->peers.loss[st->rank], 0, sizeof(float) * es.nb, s));
  const int64_t nb_run = es.nb_run >= 0 ? es.nb_run : es.nb;
  for (int64_t b = 0; b < nb_run; ++b) {
    const int64_t lo = b * es.B;
    const int64_t Bb = std::min(es.B, ctx->M - lo);
    const int64_t Sb = b < es.nb - 1 ? es.S : es.s_last;
    if (Sb > 0) {
      FwdArgs fa = base_fwd(ctx);
      shard_fill_fwd(ctx, fa);
      fa.pair_ht = sp.pair_ht + b * es.S;
      fa.pair_r = sp.pair_r + b * es.S;
      fa.B = static_cast<int>(Sb);
      fa.unit = 1.0f / static_cast<float>(Bb);  // training.cpp:84 with the global batch
      fa.loss_div = static_cast<float>(Bb);
      fa.margin = ctx->h_lr[1];
      fa.batch = static_cast<int>(b);
      set_stamps(ctx, fa, b);
      launch_hrt_forward(es.kind, true, fa, ctx->num_sms, s);
    }
    mark();
    shard_barrier(ctx, s);
    shard_backward(ctx, es.kind, slot, b, s);
    shard_barrier(ctx, s);
    mark();
  }
  shard_finish_losses(ctx, es.nb, s);
  shard_barrier(ctx, s);  // every rank has read the shard losses before any rank clears them
}

void gen_perm(skg_ctx* ctx, const EpochShape& es, const uint64_t* seed, int32_t* dst, cudaStream_t s);
void build_plan_from_order(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s);

void enqueue_epoch(skg_ctx* ctx, const EpochShape& es, std::vector<cudaEvent_t>* ev) {
  cudaStream_t s = ctx->stream;
  std::function<void()> mark = [&]() {
    if (!ev) return;
    cudaEvent_t e;
    SKG_CUDA(cudaEventCreate(&e));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SKG_CUDA(cudaStreamIsCapturing(s, &cs));
    // under capture: an event record node of the graph
    SKG_CUDA(cudaEventRecordWithFlags(e, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
    ev->push_back(e);
  };
  mark();
  gen_perm(ctx, es, ctx->seed_eff.p + ctx->cur, ctx->slots[ctx->cur].order.p, s);  // the shuffle ...
  mark();
  build_plan_from_order(ctx, es, ctx->cur, s);  // ... and the incidence plan, timed apart
  mark();
  enqueue_batches(ctx, es, ctx->cur, s, ev ? &mark : nullptr);
}

// Permutation + (data-parallel shard) + transposed-incidence plan of one epoch
// into plan slot `slot`. Depends only on the seed, the triples and the
// negatives, so the next epoch's plan can be built while this one trains.
void copy_floats(const float* src, float* dst, int64_t n, int num_sms, cudaStream_t s);
void snapshot_params(skg_ctx* ctx, bool restore, cudaStream_t s);

void destroy_host_narrow(skg::HostNarrow* h);

void gen_perm(skg_ctx* ctx, const EpochShape& es, const uint64_t* seed, int32_t* dst, cudaStream_t s) {
  if (es.shuffle)
    device_shuffle(seed, ctx->M, dst, ctx->shuffle, s);
  else
    device_iota(dst, ctx->M, s);
}

void build_plan_from_order(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s);

ThTilePlan th_plan_of(const skg_ctx* ctx, const EpochShape& es, PlanSlot& ps) {
  ThTilePlan tp;
  if (!ps.th_on) return tp;
  tp.meta = ps.th_meta.p;
  tp.rows = ps.th_rows.p;
  tp.pos = ps.th_pos.p;
  tp.info = ps.th_info.p;
  tp.B = es.B;
  (void)ctx;
  return tp;
}

TrTilePlan tr_plan_of(const EpochShape& es, PlanSlot& ps) {
  TrTilePlan tp;
  if (!ps.tr_on) return tp;
  tp.tile_seg = ps.tr_seg.p;
  tp.tile_p0 = ps.tr_p0.p;
  tp.tile_total = ps.tr_total.p;
  tp.seg_tiles = ps.tr_segtiles.p;
  tp.B = es.B;
  return tp;
}

void transh_tile_plan_for(skg_ctx* ctx, const EpochShape& es, PlanSlot& ps, cudaStream_t s) {
  FwdArgs fa{};
  fa.pair_ht = ps.plan.pair_ht;
  fa.N = ctx->N;
  BwdArgs ba{};
  ba.ent_val = ps.plan.sorted_val;
  ba.seg_start = ps.plan.seg_start;
  ba.seg_col = ps.plan.seg_col;
  ba.seg_base = ps.plan.seg_base;
  ba.N = ctx->N;
  transh_tile_plan(fa, ba, es.B, es.nb, ctx->M, ctx->R, th_plan_of(ctx, es, ps), s);
}

void enqueue_plan(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s) {
  gen_perm(ctx, es, ctx->seed_eff.p + slot, ctx->slots[slot].order.p, s);
  build_plan_from_order(ctx, es, slot, s);
}

// The transposed-incidence plan of slot `slot` from the permutation in its order buffer.
void build_plan_from_order(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s) {
  PlanSlot& ps = ctx->slots[slot];
  if (ctx->shard) {  // this rank's forward pairs + the owned-column plan of the global batches
    shard_order_kernel<<<grid_for(es.Mg), 256, 0, s>>>(ps.order.p, es.B, es.S, es.rank, es.nb, es.i0_last, es.Mg,
                                                        ps.order_g.p);
    count_launch();
    SKG_LAUNCH_CHECK();
    shard_build_plan(ctx, ps.order.p, ps.order_g.p, es.Mg, slot, s);
    return;
  }
  if (es.world > 1 || ctx->dp != nullptr) {
    shard_order_kernel<<<grid_for(es.Mg), 256, 0, s>>>(ps.order.p, es.B, es.S, es.rank, es.nb, es.i0_last, es.Mg,
                                                        ps.order_g.p);
    count_launch();
    SKG_LAUNCH_CHECK();
    build_epoch_plan(ps.order_g.p, ctx->quad.p, ctx->Rl.p, es.Mg, es.S, ctx->N, ctx->R, ps.plan, s);
  } else {
    build_epoch_plan(ps.order.p, ctx->quad.p, ctx->Rl.p, ctx->M, es.B, ctx->N, ctx->R, ps.plan, s);
    if (ps.th_on) transh_tile_plan_for(ctx, es, ps, s);
    if (ps.tr_on) {
      BwdArgs ba{};
      ba.seg_start = ps.plan.seg_start;
      ba.seg_col = ps.plan.seg_col;
      ba.seg_base = ps.plan.seg_base;
      ba.N = ctx->N;
      transr_tile_plan(ba, es.B, es.nb, ctx->R, tr_plan_of(es, ps), s);
    }
  }
}

// Every minibatch of one epoch on plan slot `slot`.
void enqueue_batches(skg_ctx* ctx, const EpochShape& es, int slot, cudaStream_t s,
                     const std::function<void()>* markp) {
  auto mark = [&]() {
    if (markp) (*markp)();
  };
  if (ctx->shard) {
    enqueue_shard_batches(ctx, es, slot, s, markp);
    return;
  }
  PlanSlot& ps = ctx->slots[slot];
  const bool dp = es.world > 1 || ctx->dp != nullptr;
  reset_err(ctx, s);
  if (dp) SKG_CUDA(cudaMemsetAsync(ctx->batch_loss.p, 0, sizeof(float) * es.nb, s));
  const bool ht = is_ht_kind(es.kind);
  const bool mult = is_mult_kind(es.kind);
  // data-parallel gradient sink: [entity | relation | proj | normals] + 2 flag slots
  const int64_t n_params = ctx->N * ctx->de + ctx->R * ctx->dr;
  const int64_t n_proj = ctx->proj.n, n_norm = ctx->normals.n;
  const int64_t n_sink = n_params + (ht ? n_proj + n_norm : 0);
  const int64_t nb_run = es.nb_run >= 0 ? es.nb_run : es.nb;
  // A speculative epoch (deferred re-upload) snapshots the parameters on the
  // upload stream while batch 0's forward already runs: batch 0's first
  // parameter write waits for that copy (an external event node in the
  // graph; a no-op when no snapshot was recorded).
  bool snap_waited = false;
  const std::function<void()> wait_snapshot = [&]() {
    if (snap_waited) return;
    snap_waited = true;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SKG_CUDA(cudaStreamIsCapturing(s, &cs));
    // in a speculative graph the snapshot branch is part of this capture (an edge), otherwise an
    // external wait on the last record (a snapshot enqueued before the launch, or none)
    if (cs == cudaStreamCaptureStatusActive && ctx->spec_graph)
      SKG_CUDA(cudaStreamWaitEvent(s, ctx->snap_cap_ev, 0));
    else
      SKG_CUDA(cudaStreamWaitEvent(s, ctx->snap_ev, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
  };
  for (int64_t b = 0; b < nb_run; ++b) {
    const int64_t lo = b * es.B;
    const int Bb = static_cast<int>(std::min(es.B, ctx->M - lo));
    if (dp) {
      // shard of global minibatch b: forward with the global 1/m, gradient
      // into the dense sink, NCCL sum over NVLink, identical step on all ranks
      const int64_t Sb = b < es.nb - 1 ? es.S : es.s_last;
      float* G = ctx->dp_grad.p;
      SKG_CUDA(cudaMemsetAsync(G, 0, sizeof(float) * (n_sink + 2), s));
      if (Sb > 0) {
        FwdArgs fa = base_fwd(ctx);
        fa.order = ps.order_g.p + b * es.S;
        fa.pair_ht = ps.plan.pair_ht + b * es.S;
        fa.pair_r = ps.plan.pair_r + b * es.S;
        fa.H = ctx->H.p;
        fa.Rl = ctx->Rl.p;
        fa.T = ctx->T.p;
        fa.NH = ctx->NH.p;
        fa.NT = ctx->NT.p;
        fa.B = static_cast<int>(Sb);
        fa.unit = 1.0f / static_cast<float>(Bb);
        fa.loss_div = static_cast<float>(Bb);
        fa.margin = ctx->h_lr[1];
        fa.batch = static_cast<int>(b);
        set_stamps(ctx, fa, b);
        if (ht) {  // TransH / TransR: this rank's gradients into the sink, no in-place step
          BwdArgs hb{};
          hb.X = G;
          hb.Xrel = G + ctx->N * ctx->de;
          hb.res = ctx->res_u.p;
          hb.scal = ctx->scal.p;
          hb.N = ctx->N;
          hb.d = static_cast<int>(ctx->de);
          hb.ent_val = ps.plan.sorted_val;
          hb.seg_start = ps.plan.seg_start;
          hb.seg_col = ps.plan.seg_col;
          hb.seg_base = ps.plan.seg_base;
          hb.batch = static_cast<int>(b);
          hb.lr = ctx->lr_dev.p;
          hb.err = ctx->err_words.p;
          HtSinks sk{G + ctx->N * ctx->de, n_proj ? G + n_params : nullptr,
                     n_norm ? G + n_params + n_proj : nullptr};
          const Branch br{ctx->aux, ctx->aux_fork, ctx->aux_join};
          ht_train_batch(es.kind, fa, hb, ctx->ht_work.p, ctx->num_sms, s, nullptr, ctx->R, &sk, &br);
        } else if (mult) {
          fa.de = static_cast<int>(ctx->cfg.dim_entity);
          fa.plane_rows = 2 * es.S;
          fa.sign = (es.kind == kRotatE) ? 1.f : -1.f;
          fa.res_u = nullptr;
          launch_mult_forward(es.kind, true, fa, ctx->num_sms, s);
        } else {
          launch_hrt_forward(es.kind, true, fa, ctx->num_sms, s);
        }
        mark();
        BwdArgs ba{};
        ba.X = G;
        ba.plane_rows = 2 * es.S;
        ba.res = ctx->res.p;
        ba.scal = ctx->scal.p;
        ba.N = ctx->N;
        ba.d = static_cast<int>(ctx->de);
        ba.ent_val = ps.plan.sorted_val;
        ba.seg_start = ps.plan.seg_start;
        ba.seg_col = ps.plan.seg_col;
        ba.seg_base = ps.plan.seg_base;
        ba.batch = static_cast<int>(b);
        ba.lr = ctx->lr_dev.p;
        ba.err = ctx->err_words.p;
        if (!ht) launch_segment_backward(mult ? static_cast<int>(kMultRows) : es.kind, false, ba, ctx->num_sms, s);
      } else {
        mark();
      }
      float* flags = G + n_sink;
      dp_flags_kernel<<<1, 1, 0, s>>>(ctx->err_words.p, flags);
      dp_allreduce_sum(ctx, G, n_sink + 2, s);
      dp_sgd_kernel<<<grid_for(n_params), 256, 0, s>>>(ctx->tables.p, G, n_params, ctx->lr_dev.p, flags,
                                                        ctx->err_words.p, static_cast<int>(b));
      count_launch(2);
      if (ht && n_proj) {
        dp_sgd_kernel<<<grid_for(n_proj), 256, 0, s>>>(ctx->proj.p, G + n_params, n_proj, ctx->lr_dev.p, flags,
                                                        ctx->err_words.p, static_cast<int>(b));
        count_launch();
      }
      if (ht && n_norm) {
        dp_sgd_kernel<<<grid_for(n_norm), 256, 0, s>>>(ctx->normals.p, G + n_params + n_proj, n_norm, ctx->lr_dev.p,
                                                        flags, ctx->err_words.p, static_cast<int>(b));
        count_launch();
        launch_normals_renorm(ctx->normals.p, ctx->R, static_cast<int>(ctx->de), ctx->err_words.p, s);
      }
      SKG_LAUNCH_CHECK();
      mark();
      continue;
    }
    FwdArgs fa = base_fwd(ctx);
    fa.order = ps.order.p + lo;
    fa.pair_ht = ps.plan.pair_ht + lo;
    fa.pair_r = ps.plan.pair_r + lo;
    fa.H = ctx->H.p;
    fa.Rl = ctx->Rl.p;
    fa.T = ctx->T.p;
    fa.NH = ctx->NH.p;
    fa.NT = ctx->NT.p;
    fa.B = Bb;
    fa.unit = 1.0f / static_cast<float>(Bb);  // training.cpp:84
    fa.margin = ctx->h_lr[1];
    fa.batch = static_cast<int>(b);
    set_stamps(ctx, fa, b);
    BwdArgs ba{};
    ba.X = ctx->tables.p;
    ba.Xrel = ctx->tables.p + ctx->N * ctx->de;
    ba.res = ht ? ctx->res_u.p : ctx->res.p;
    ba.scal = ctx->scal.p;
    ba.N = ctx->N;
    ba.d = static_cast<int>(ctx->de);
    ba.ent_val = ps.plan.sorted_val;
    ba.seg_start = ps.plan.seg_start;
    ba.seg_col = ps.plan.seg_col;
    ba.seg_base = ps.plan.seg_base;
    ba.batch = static_cast<int>(b);
    ba.lr = ctx->lr_dev.p;
    ba.err = ctx->err_words.p;
    if (mult) {
      fa.de = static_cast<int>(ctx->cfg.dim_entity);
      fa.plane_rows = 2 * es.B;
      fa.sign = (es.kind == kRotatE) ? 1.f : -1.f;  // energy_sign (models.hpp:32-38)
      fa.res_u = nullptr;
      ba.res = ctx->res.p;
      ba.plane_rows = 2 * es.B;
      launch_mult_forward(es.kind, true, fa, ctx->num_sms, s);
      mark();
      if (b == 0) wait_snapshot();
      launch_segment_backward(kMultRows, true, ba, ctx->num_sms, s);
      mark();
    } else if (!ht) {
      launch_hrt_forward(es.kind, true, fa, ctx->num_sms, s);
      mark();
      if (b == 0) wait_snapshot();
      launch_segment_backward(es.kind, true, ba, ctx->num_sms, s);
      mark();
    } else {
      const Branch br{ctx->aux, ctx->aux_fork, ctx->aux_join};
      // the ht step calls its mark after the forward kernels (which write no parameters)
      const std::function<void()> mark0 = [&]() {
        if (markp) (*markp)();
        wait_snapshot();
      };
      const ThTilePlan tp = th_plan_of(ctx, es, ps);
      const TrTilePlan trp = tr_plan_of(es, ps);
      ht_train_batch(es.kind, fa, ba, ctx->ht_work.p, ctx->num_sms, s, b == 0 ? &mark0 : markp, ctx->R, nullptr, &br,
                     tp.meta ? &tp : nullptr, trp.tile_seg ? &trp : nullptr);
      if (b == 0) wait_snapshot();  // (if the step had no mark call)
    }
  }
  if (dp) dp_allreduce_sum(ctx, ctx->batch_loss.p, es.nb, s);  // shard losses -> global batch losses
}

void prepare_epoch(skg_ctx* ctx, const skg_model_config& cfg, const skg_train_config& tc,
                   EpochShape& es) {
  validate_train(tc);
  check_config(ctx, cfg, ctx->tN, ctx->tR);
  if (ctx->M < 1) throw ConfigError("training requires at least one triple");
  if (!ctx->has_neg) throw ShapeError("negative set is not aligned with the positive triples");
  es.nb = (ctx->M + tc.batch_size - 1) / tc.batch_size;
  // data parallel keeps the configured global batch (a single short batch is
  // the ragged last one of the shard geometry)
  es.B = (ctx->dp || ctx->shard) ? tc.batch_size : std::min<int64_t>(tc.batch_size, ctx->M);
  if (es.B > (1 << 30)) throw ConfigError("batch_size too large for 32-bit row ids");
  es.shuffle = tc.shuffle != 0;
  es.kind = kind_of(cfg);
  ctx->order.ensure(ctx->M);
  es.world = dp_world(ctx);
  es.rank = dp_rank(ctx);
  if (ctx->shard) {
    if (es.kind != kTransE_L2 && es.kind != kTransE_L1 && es.kind != kTorusE_L2 && es.kind != kTorusE_L1)
      throw ConfigError("sharded data parallel covers the hrt models (transe, toruse)");
    if (tc.batch_size != ctx->shard->B)
      throw ConfigError("sharded context was initialised for batch_size " + std::to_string(ctx->shard->B));
    if (es.nb > ctx->shard->nb_cap) throw ConfigError("sharded context: triples changed size since init");
    if (!ctx->shard->linked) throw ConfigError("sharded context: peers not linked");
  }
  if (ctx->dp || ctx->shard) {
    if (es.B % es.world != 0) throw ConfigError("data parallel: global batch_size must be a multiple of the world size");
    int64_t sh[5];
    dp_shard(ctx->M, es.B, es.world, es.rank, sh);
    es.S = sh[0];
    es.i0_last = sh[1];
    es.s_last = sh[2];
    es.Mg = sh[3];
    for (auto& sl : ctx->slots) sl.order_g.ensure(es.Mg + 1);
    if (ctx->dp) ctx->dp_grad.ensure(ctx->N * ctx->de + ctx->R * ctx->dr + ctx->proj.n + ctx->normals.n + 2);
  }
  for (auto& p : ctx->perm) p.ensure(ctx->M + 1);
  static const bool th_no_plan = std::getenv("SKG_TH_NO_PLAN") != nullptr;
  static const bool tr_no_plan = std::getenv("SKG_TR_NO_PLAN") != nullptr;
  // TransH relation tiles precomputed with the plan (single device, tile kernel, bounded size)
  const int64_t th_mt = transh_tile_plan_tiles(es.B, ctx->R);
  const bool th_on = (es.kind == kTransH_L2 || es.kind == kTransH_L1) && !ctx->dp && !ctx->shard &&
                     transh_tiles_supported(static_cast<int>(ctx->de), static_cast<int>(ctx->dr), ctx->R) &&
                     es.nb * th_mt * 656 <= (512ll << 20) && !th_no_plan;
  // TransR relation tiles precomputed with the plan (single device, tcgen05 step)
  const bool tr_on = (es.kind == kTransR_L2 || es.kind == kTransR_L1) && !ctx->dp && !ctx->shard &&
                     transr_train_tc_supported(static_cast<int>(ctx->de), static_cast<int>(ctx->dr)) &&
                     !tr_no_plan;
  for (auto& sl : ctx->slots) {
    sl.order.ensure(ctx->M + 1);
    if (!ctx->shard) sl.plan.reserve(6 * (ctx->dp ? es.Mg : ctx->M) + 6, es.nb);
    sl.th_on = th_on;
    sl.tr_on = tr_on;
    if (tr_on) {
      const int64_t mtr = relation_max_tiles(2 * es.B, ctx->R);
      sl.tr_seg.ensure(es.nb * mtr);
      sl.tr_p0.ensure(es.nb * mtr);
      sl.tr_total.ensure(2 * es.nb);
      sl.tr_segtiles.ensure(es.nb * (ctx->R + 2));
    }
    if (th_on) {
      sl.th_meta.ensure(es.nb * th_mt);
      sl.th_rows.ensure(es.nb * th_mt * 32);
      sl.th_pos.ensure(es.nb * th_mt * 32);
      sl.th_info.ensure(es.nb * (4 + 3 * ctx->R));
    }
  }
  ctx->shuffle.reserve(ctx->M);
  if (ctx->quad_version != ctx->data_version || ctx->quad.n < ctx->M + 1) {  // packed ids for the plan
    ctx->quad.ensure(ctx->M + 1);
    pack_triple_quads(ctx->H.p, ctx->T.p, ctx->NH.p, ctx->NT.p, ctx->M, ctx->quad.p, ctx->stream);
    ctx->quad_version = ctx->data_version;
  }
  if (ctx->shard) {  // plan buffers of both slots sized before any capture (owned entries per epoch are fixed)
    const int64_t E = shard_entry_count(ctx);
    for (auto& p : ctx->shard->plan) p.reserve(es.Mg, 2 * ctx->M, E, es.nb);
  }
  ensure_workspace(ctx, 2 * es.B, es.kind);
  if (is_ht(cfg)) ctx->ht_work.ensure(ht_work_floats(es.kind, 2 * es.B, ctx->de, ctx->dr, ctx->R));
  ctx->batch_loss.ensure(es.nb);
  ctx->stamps.ensure(2 * es.nb);
  if (ctx->h_stamps_cap < es.nb) {
    if (ctx->h_stamps) cudaFreeHost(ctx->h_stamps);
    SKG_CUDA(cudaMallocHost(&ctx->h_stamps, sizeof(unsigned long long) * 2 * es.nb));
    ctx->h_stamps_cap = es.nb;
  }
  if (ctx->h_loss_cap < es.nb) {
    if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
    SKG_CUDA(cudaMallocHost(&ctx->h_loss, sizeof(float) * es.nb));
    ctx->h_loss_cap = es.nb;
  }
}

// Keys are the raw bytes of the values they depend on (built every epoch on
// the host critical path: no formatting).
template <class... T>
std::string raw_key(const T&... v) {
  std::string k;
  k.reserve((sizeof(T) + ... + 0));
  (k.append(reinterpret_cast<const char*>(&v), sizeof(T)), ...);
  return k;
}

std::string graph_key(skg_ctx* ctx, const EpochShape& es, float margin) {
  return raw_key(es.B, es.nb, es.shuffle, es.kind, ctx->M, ctx->tables.p, ctx->H.p, ctx->NH.p, ctx->quad.p,
                 ctx->slots[0].order.p,
                 ctx->slots[1].order.p, ctx->perm[0].p, ctx->perm[1].p, ctx->res.p, ctx->ht_work.p, ctx->slots[0].plan.cap_entries,
                 ctx->slots[1].plan.cap_entries, ctx->shuffle.cap_n, es.world, es.rank, ctx->dp_grad.p,
                 ctx->slots[0].order_g.p, ctx->slots[1].order_g.p, ctx->proj.p, ctx->normals.p, margin,
                 // shapes baked into the captured launches (strides, relation offset, plan id space)
                 ctx->N, ctx->R, ctx->de, ctx->dr, ctx->cfg.dim_entity, ctx->proj.n, ctx->normals.n, dp_comm_tag(ctx),
                 ctx->phase_timers, ctx->stamps.p, ctx->shard, shard_tag(ctx), ctx->slots[0].th_meta.p,
                 ctx->slots[1].th_meta.p, ctx->slots[0].th_rows.p, ctx->slots[1].th_rows.p, ctx->slots[0].th_pos.p,
                 ctx->slots[1].th_pos.p, ctx->slots[0].th_info.p, ctx->slots[1].th_info.p, ctx->slots[0].th_on,
                 ctx->slots[0].tr_seg.p, ctx->slots[1].tr_seg.p, ctx->slots[0].tr_p0.p, ctx->slots[1].tr_p0.p,
                 ctx->slots[0].tr_total.p, ctx->slots[1].tr_total.p, ctx->slots[0].tr_segtiles.p,
                 ctx->slots[1].tr_segtiles.p, ctx->slots[0].tr_on, ctx->spec_graph, ctx->backup.p);
}

// Identity of an epoch plan: everything it depends on.
std::string plan_key(skg_ctx* ctx, const EpochShape& es, const skg_train_config& tc, int64_t epoch) {
  const uint64_t seed = es.shuffle ? tc.seed : 0;
  return raw_key(epoch, seed, es.shuffle, es.B, ctx->M, ctx->data_version, es.world, es.rank, ctx->H.p, ctx->NH.p,
                 ctx->N, ctx->R, dp_comm_tag(ctx), ctx->slots[0].th_on,  // the plan carries TransH / TransR tiles
                 ctx->slots[0].tr_on);
}

// The epoch's results (batch losses, error words, the speculative upload
// check's flags) written by one kernel into the pinned host buffers, which
// are device-addressable under UVA: one node after the epoch instead of up to
// three D2H copies, each a separate DMA round trip on the critical path.
__global__ void publish_kernel(const float* __restrict__ loss, int64_t nb, float* h_loss,
                               const uint32_t* __restrict__ err, uint32_t* h_err,
                               const uint32_t* __restrict__ spec, uint32_t* h_spec) {
  const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t i = i0; i < nb; i += static_cast<int64_t>(gridDim.x) * blockDim.x) h_loss[i] = loss[i];
  if (i0 < 4) {
    h_err[i0] = err[i0];
    if (spec) h_spec[i0] = spec[i0];
  }
}

void finish_epoch(skg_ctx* ctx, const EpochShape& es, int64_t epoch, skg_epoch_report* rep) {
  {
    const uint32_t* spec = ctx->pub_spec;
    ctx->pub_spec = nullptr;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((es.nb + 255) / 256, 64)));
    publish_kernel<<<grid, 256, 0, ctx->stream>>>(ctx->batch_loss.p, es.nb, ctx->h_loss, ctx->err_words.p,
                                                  ctx->h_err, spec, ctx->h_spec);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
  if (ctx->phase_timers)
    SKG_CUDA(cudaMemcpyAsync(ctx->h_stamps, ctx->stamps.p, sizeof(unsigned long long) * 2 * es.nb,
                             cudaMemcpyDeviceToHost, ctx->stream));
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  raise_device_error(ctx->h_err, epoch);
  // training.cpp:141, 163: loss_sum += loss * Real(hi - lo); loss = loss_sum / Real(m)
  float loss_sum = 0.f;
  for (int64_t b = 0; b < es.nb; ++b) {
    const int64_t lo = b * es.B, hi = std::min(ctx->M, lo + es.B);
    const volatile float prod = ctx->h_loss[b] * static_cast<float>(hi - lo);
    loss_sum = loss_sum + prod;
  }
  rep->epoch = epoch;
  rep->loss = static_cast<double>(loss_sum / static_cast<float>(ctx->M));
}

void set_epoch_params(skg_ctx* ctx, const skg_train_config& tc, float lr) {
  ctx->h_lr[0] = lr;
  ctx->h_lr[1] = tc.margin;
  SKG_CUDA(cudaMemcpyAsync(ctx->lr_dev.p, ctx->h_lr, sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
}

// First node of every epoch graph: this epoch's lr and the seed of the
// permutation the graph shuffles (arguments replaced in the instantiated graph
// before each launch, see set_graph_params).
struct EpochParams {
  float* lr_dev;
  uint64_t* seed_dst;
  float lr;
  uint64_t seed;
};
__global__ void epoch_params_kernel(EpochParams p) {
  *p.lr_dev = p.lr;
  *p.seed_dst = p.seed;
}

EpochParams epoch_params_of(skg_ctx* ctx, int cur) {
  return EpochParams{ctx->lr_dev.p, ctx->seed_eff.p + 2 + cur, ctx->h_lr[0], ctx->h_seed[2 + cur]};
}

void set_graph_params(skg_ctx* ctx, int cur) {
  EpochParams ep = epoch_params_of(ctx, cur);
  void* args[1] = {&ep};
  cudaKernelNodeParams kp{};
  kp.func = reinterpret_cast<void*>(epoch_params_kernel);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  SKG_CUDA(cudaGraphExecKernelNodeSetParams(ctx->graphs[cur], ctx->param_node[cur], &kp));
}

void set_slot_seed(skg_ctx* ctx, int slot, uint64_t seed_eff) {
  ctx->h_seed[slot] = seed_eff;
  SKG_CUDA(cudaMemcpyAsync(ctx->seed_eff.p + slot, ctx->h_seed + slot, sizeof(uint64_t), cudaMemcpyHostToDevice,
                           ctx->stream));
}

// L2 residency of the parameter tables. The per-batch streams (residual / dU
// rows, plan entries) together with a mid-size table exceed the 126 MB L2 (C4:
// 63 MB table + 67 MB dU rows), so without a hint every minibatch re-reads the
// table from HBM at gather latency. When the stacked table fits the
// persisting carve-out, every kernel node of the epoch graph gets an access
// policy window over it (hits persist, misses stream). SKG_L2_PERSIST=0 turns
// it off.
void apply_l2_policy(skg_ctx* ctx, cudaGraph_t g) {
  static const bool enabled = [] {
    const char* e = std::getenv("SKG_L2_PERSIST");
    return !(e && e[0] == '0');
  }();
  const size_t bytes = sizeof(float) * static_cast<size_t>(ctx->tables.n);
  if (!enabled || bytes < (size_t(16) << 20)) return;  // small tables stay L2-resident on their own
  int max_persist = 0, max_win = 0;
  SKG_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
  SKG_CUDA(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
  if (bytes > static_cast<size_t>(max_persist) || bytes > static_cast<size_t>(max_win)) return;
  size_t cur = 0;
  SKG_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  if (cur < bytes) SKG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
  cudaLaunchAttributeValue v{};
  v.accessPolicyWindow.base_ptr = ctx->tables.p;
  v.accessPolicyWindow.num_bytes = bytes;
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  size_t n = 0;
  SKG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  SKG_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    SKG_CUDA(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel)
      SKG_CUDA(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributeAccessPolicyWindow, &v));
  }
}

// One captured graph per plan slot: the main branch trains every minibatch on
// slot `cur`; a side branch builds the next epoch's plan into the other slot.
void capture_epoch_graph(skg_ctx* ctx, const EpochShape& es, int cur) {
  const int nxt = 1 - cur;
  const int64_t before = kernel_launches();
  cudaGraph_t g = nullptr;
  SKG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  try {
    epoch_params_kernel<<<1, 1, 0, ctx->stream>>>(epoch_params_of(ctx, cur));
    count_launch();
    SKG_LAUNCH_CHECK();
    if (ctx->spec_graph) {  // speculative epoch: parameter snapshot on a branch (joined at batch 0's first write)
      SKG_CUDA(cudaEventRecord(ctx->fork_up_ev, ctx->stream));
      SKG_CUDA(cudaStreamWaitEvent(ctx->up, ctx->fork_up_ev, 0));
      snapshot_params(ctx, false, ctx->up);
      SKG_CUDA(cudaEventRecord(ctx->snap_cap_ev, ctx->up));
    }
    SKG_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
    SKG_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
    SKG_CUDA(cudaStreamWaitEvent(ctx->side2, ctx->fork_ev, 0));
    // side: epoch + 1's plan from its permutation (shuffled during the previous epoch)
    copy_floats(reinterpret_cast<const float*>(ctx->perm[nxt].p), reinterpret_cast<float*>(ctx->slots[nxt].order.p),
                ctx->M, ctx->num_sms, ctx->side);
    build_plan_from_order(ctx, es, nxt, ctx->side);
    SKG_CUDA(cudaEventRecord(ctx->join_ev, ctx->side));
    // side2: epoch + 2's permutation (seed slot 2 + cur)
    gen_perm(ctx, es, ctx->seed_eff.p + 2 + cur, ctx->perm[cur].p, ctx->side2);
    SKG_CUDA(cudaEventRecord(ctx->join2_ev, ctx->side2));
    enqueue_batches(ctx, es, cur, ctx->stream, nullptr);
    SKG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
    SKG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join2_ev, 0));
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  SKG_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  try {
    apply_l2_policy(ctx, g);
  } catch (...) {
    cudaGraphDestroy(g);
    throw;
  }
  if (ctx->graphs[cur]) cudaGraphExecDestroy(ctx->graphs[cur]);
  ctx->graphs[cur] = nullptr;
  if (ctx->graph_src[cur]) cudaGraphDestroy(ctx->graph_src[cur]);
  ctx->graph_src[cur] = nullptr;
  ctx->param_node[cur] = nullptr;
  try {
    size_t n = 0;
    SKG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    SKG_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      SKG_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      SKG_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == reinterpret_cast<void*>(epoch_params_kernel)) ctx->param_node[cur] = nd;
    }
    if (!ctx->param_node[cur]) throw CudaError("epoch graph: parameter node not found");
    SKG_CUDA(cudaGraphInstantiate(&ctx->graphs[cur], g, 0));
  } catch (...) {
    cudaGraphDestroy(g);
    ctx->param_node[cur] = nullptr;
    throw;
  }
  ctx->graph_src[cur] = g;  // owns param_node[cur]
  ctx->graph_launches_k[cur] = kernel_launches() - before;
}

}  // namespace

void skg::drop_graphs(skg_ctx* ctx) {
  for (int k = 0; k < 2; ++k) {
    if (ctx->graphs[k]) cudaGraphExecDestroy(ctx->graphs[k]);
    ctx->graphs[k] = nullptr;
    if (ctx->graph_src[k]) cudaGraphDestroy(ctx->graph_src[k]);
    ctx->graph_src[k] = nullptr;
    ctx->param_node[k] = nullptr;
    ctx->graph_keys[k].clear();
    ctx->slots[k].key.clear();
    ctx->perm_key[k].clear();
  }
}

namespace {

// Does any positive or negative triple have head == tail? (cached per data version)
bool has_self_loops(skg_ctx* ctx) {
  if (ctx->loops_version == ctx->data_version) return ctx->has_loops;
  ctx->bad_idx.ensure(3);
  SKG_CUDA(cudaMemsetAsync(ctx->bad_idx.p, 0xFF, sizeof(uint32_t) * 2, ctx->stream));
  first_loop_kernel<<<grid_for(ctx->M), 256, 0, ctx->stream>>>(nullptr, ctx->H.p, ctx->T.p, ctx->NH.p, ctx->NT.p,
                                                               ctx->M, ctx->bad_idx.p);
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->bad_idx.p, sizeof(uint32_t) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->has_loops = ctx->h_err[0] != 0xFFFFFFFFu || ctx->h_err[1] != 0xFFFFFFFFu;
  ctx->loops_version = ctx->data_version;
  return ctx->has_loops;
}

// training.cpp:117-125 with a self-loop triple in the epoch: the batches before
// the first one containing it train normally, then score_batch throws (the
// positive sub-batch is scored before the negative one).
[[noreturn]] void train_until_degenerate(skg_ctx* ctx, EpochShape es, int64_t epoch, int cur) {
  SKG_CUDA(cudaMemsetAsync(ctx->bad_idx.p, 0xFF, sizeof(uint32_t) * 2, ctx->stream));
  first_loop_kernel<<<grid_for(ctx->M), 256, 0, ctx->stream>>>(ctx->slots[cur].order.p, ctx->H.p, ctx->T.p,
                                                               ctx->NH.p, ctx->NT.p, ctx->M, ctx->bad_idx.p);
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->bad_idx.p, sizeof(uint32_t) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  const int64_t kp = ctx->h_err[0], kn = ctx->h_err[1];
  const int64_t kmin = std::min(kp, kn);
  const int64_t bf = kmin / es.B;
  const int64_t i = (kp / es.B == bf ? kp : kn) - bf * es.B;
  ctx->slots[1 - cur].key.clear();
  es.nb_run = bf;
  if (bf > 0) {
    enqueue_batches(ctx, es, cur, ctx->stream, nullptr);
    SKG_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->err_words.p, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    raise_device_error(ctx->h_err, epoch);
  }
  throw DegenerateTripleError("triple " + std::to_string(i) +
                              ": head == tail is not representable in the multiplicative incidence layout");
}

// One epoch in three steps, so a driver of several sharded contexts can stage
// every rank (allocations, plan, graph capture: host work that may block)
// before firing any graph whose barriers wait for the others.
struct StagedEpoch {
  EpochShape es;
  int cur = 0, nxt = 1;
  int64_t eager = 0;
  int64_t epoch = 0;
  std::string next_key, perm_key;
};

StagedEpoch stage_epoch(skg_ctx* ctx, const skg_model_config& cfg, const skg_train_config& tc, int64_t epoch,
                        float lr) {
  StagedEpoch sg;
  EpochShape& es = sg.es;
  sg.epoch = epoch;
  prepare_epoch(ctx, cfg, tc, es);
  // lr (and margin, baked in at capture) on the host side only: the graph's
  // parameter node writes lr to the device (set_graph_params)
  ctx->h_lr[0] = lr;
  ctx->h_lr[1] = tc.margin;
  const int cur = ctx->cur, nxt = 1 - cur;
  sg.cur = cur;
  sg.nxt = nxt;
  // The plan of this epoch was normally built by the previous epoch's graph;
  // otherwise (first epoch, new data, other schedule) build it now.
  const std::string pk = plan_key(ctx, es, tc, epoch);
  if (ctx->slots[cur].key != pk) {
    set_slot_seed(ctx, cur, epoch_seed(tc.seed, epoch));
    const int64_t before = kernel_launches();
    enqueue_plan(ctx, es, cur, ctx->stream);
    sg.eager = kernel_launches() - before;
    ctx->slots[cur].key = pk;
  }
  if (is_mult(cfg) && has_self_loops(ctx)) {
    set_epoch_params(ctx, tc, lr);                // eager batches read lr from the device
    train_until_degenerate(ctx, es, epoch, cur);  // always throws
  }
  // Speculatively build epoch + 1's plan (same data and schedule) alongside,
  // from its permutation (normally shuffled by the previous epoch's graph),
  // and shuffle epoch + 2's permutation beside it.
  const std::string pk1 = plan_key(ctx, es, tc, epoch + 1);
  if (ctx->perm_key[nxt] != pk1) {
    set_slot_seed(ctx, nxt, epoch_seed(tc.seed, epoch + 1));
    const int64_t before = kernel_launches();
    gen_perm(ctx, es, ctx->seed_eff.p + nxt, ctx->perm[nxt].p, ctx->stream);
    sg.eager += kernel_launches() - before;
    ctx->perm_key[nxt] = pk1;
  }
  ctx->h_seed[2 + cur] = epoch_seed(tc.seed, epoch + 2);  // written by the graph's parameter node
  ctx->perm_key[cur].clear();
  ctx->slots[nxt].key.clear();
  // Margin is baked into the forward launches, so it is part of the graph key.
  const std::string gk = graph_key(ctx, es, tc.margin);
  if (!ctx->graphs[cur] || ctx->graph_keys[cur] != gk) {
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));  // margin in h_lr[1] is read at capture
    capture_epoch_graph(ctx, es, cur);
    ctx->graph_keys[cur] = gk;
  } else {
    set_graph_params(ctx, cur);
  }
  sg.next_key = pk1;
  sg.perm_key = plan_key(ctx, es, tc, epoch + 2);
  return sg;
}

void fire_epoch(skg_ctx* ctx, const StagedEpoch& sg) {
  SKG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  SKG_CUDA(cudaGraphLaunch(ctx->graphs[sg.cur], ctx->stream));
  SKG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->last_launches = ctx->graph_launches_k[sg.cur] + sg.eager;
  ctx->last_slot = sg.cur;
  ctx->slots[sg.nxt].key = sg.next_key;
  ctx->perm_key[sg.cur] = sg.perm_key;
  ctx->cur = sg.nxt;
}

void complete_epoch(skg_ctx* ctx, const StagedEpoch& sg, skg_epoch_report* rep) {
  const EpochShape& es = sg.es;
  try {
    finish_epoch(ctx, es, sg.epoch, rep);
  } catch (...) {
    ctx->slots[sg.nxt].key.clear();  // a failed epoch leaves no reusable prefetch
    ctx->perm_key[sg.cur].clear();
    throw;
  }
  float ms = 0.f;
  SKG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  // PhaseTimer buckets (training.cpp:126, 141, 158). Forward: gather, score,
  // hinge, loss of every batch. Backward: the transposed-SpMM reduce with the
  // SGD step fused into it (touched rows), so the step has no kernel of its own
  // and t_step_s stays 0; graph overhead outside the batches (error-word reset,
  // the join with the next epoch's plan) is counted in the backward bucket so
  // the buckets sum to the epoch's device time.
  double fwd = 0.0;
  if (ctx->phase_timers)
    for (int64_t b = 0; b < es.nb; ++b) {
      const unsigned long long t0 = ctx->h_stamps[2 * b], t1 = ctx->h_stamps[2 * b + 1];
      if (t1 > t0) fwd += static_cast<double>(t1 - t0) * 1e-6;  // ns -> ms
    }
  fwd = std::min<double>(fwd, ms);
  rep->t_forward_s = fwd * 1e-3;
  rep->t_backward_s = std::max(0.0, ms - fwd) * 1e-3;
  rep->t_step_s = 0.0;
  ctx->last_epoch_ms = ms;
}


void train_epoch_impl(skg_ctx* ctx, const skg_model_config& cfg, const skg_train_config& tc,
                      int64_t epoch, float lr, skg_epoch_report* rep,
                      const std::function<void()>* after_launch = nullptr) {
  static const bool dbg = std::getenv("SKG_EPOCH_DEBUG") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const StagedEpoch sg = stage_epoch(ctx, cfg, tc, epoch, lr);
  const auto t1 = clk::now();
  fire_epoch(ctx, sg);
  const auto t2 = clk::now();
  if (after_launch) (*after_launch)();
  const auto t3 = clk::now();
  complete_epoch(ctx, sg, rep);
  if (dbg) {
    const auto t4 = clk::now();
    auto us = [](clk::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
    std::fprintf(stderr, "epoch: stage %.1f us, launch %.1f us, after-launch %.1f us, complete %.1f us (graph %.1f us)\n",
                 us(t1 - t0), us(t2 - t1), us(t3 - t2), us(t4 - t3), ctx->last_epoch_ms * 1e3);
  }
}

void negative_sample_impl(skg_ctx* ctx, uint64_t seed, bool avoid) {  // training.cpp:51-71
  const int64_t n = ctx->tN;
  if (n < 2) throw ConfigError("negative sampling needs at least two entities");
  if (avoid && n < 3) throw ConfigError("self-loop-free negative sampling needs at least three entities");
  ctx->NH.ensure(ctx->M + 1);
  ctx->NT.ensure(ctx->M + 1);
  if (!device_negative_sample(ctx->H.p, ctx->T.p, ctx->M, n, seed, avoid, ctx->NH.p, ctx->NT.p, ctx->negw,
                              ctx->stream))
    throw CudaError("negative_sample: device RNG window exhausted");
  ctx->has_neg = true;
  ++ctx->data_version;
  ctx->neg_valid_version = ctx->data_version;
}

// ------------------------------------------------------ per-op kernels (small)

__global__ void incidence_count_kernel(const int32_t* __restrict__ ids, int64_t m, int layout,
                                       uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool self = ids[i] == ids[2 * m + i];
    cnt[i] = layout >= SKG_LAYOUT_MULT ? 3u : (self ? 0u : 2u) + (layout == SKG_LAYOUT_HRT ? 1u : 0u);
  }
}

// Canonical CSR rows (coo_to_csr on build_ht / build_hrt): ascending columns,
// +1/-1 merged away on self-loops; the relation column N + r is always last.
__global__ void incidence_fill_kernel(const int32_t* __restrict__ ids, int64_t m, int layout, int64_t N,
                                      const uint32_t* __restrict__ off, int64_t* __restrict__ row_ptr,
                                      int64_t* __restrict__ col, float* __restrict__ val) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t h = ids[i], r = ids[m + i], t = ids[2 * m + i];
    int64_t p = off[i];
    row_ptr[i] = p;
    if (layout >= SKG_LAYOUT_MULT) {  // build_multiplicative (incidence.hpp:93-121), h != t checked on the host
      const float tail_marker = layout == SKG_LAYOUT_MULT_CONJ ? -1.f : 1.f;
      const bool hf = h < t;
      col[p] = hf ? h : t;
      val[p++] = hf ? 1.f : tail_marker;
      col[p] = hf ? t : h;
      val[p++] = hf ? tail_marker : 1.f;
      col[p] = N + r;
      val[p++] = 1.f;
      if (i == m - 1) row_ptr[m] = p;
      continue;
    }
    if (h != t) {
      const bool hf = h < t;
      col[p] = hf ? h : t;
      val[p++] = hf ? 1.f : -1.f;
      col[p] = hf ? t : h;
      val[p++] = hf ? -1.f : 1.f;
    }
    if (layout == SKG_LAYOUT_HRT) {
      col[p] = N + r;
      val[p++] = 1.f;
    }
    if (i == m - 1) row_ptr[m] = p;
  }
}

__global__ void hinge_kernel(const float* __restrict__ p, const float* __restrict__ n, int64_t m, float margin,
                             float* __restrict__ dp, float* __restrict__ dn, float* __restrict__ term) {
  const float unit = 1.0f / static_cast<float>(m);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float t = __fsub_rn(__fadd_rn(margin, p[i]), n[i]);
    const bool act = t > 0.f;
    dp[i] = act ? unit : 0.f;
    dn[i] = act ? -unit : 0.f;
    term[i] = act ? t : 0.f;
  }
}

// Sequential sum in index order: the reference's exact loss (training.cpp:87-93).
__global__ void seq_sum_kernel(const float* __restrict__ x, int64_t m, float* __restrict__ out) {
  float s = 0.f;
  for (int64_t i = 0; i < m; ++i) s = __fadd_rn(s, x[i]);
  *out = __fdiv_rn(s, static_cast<float>(m));
}

__global__ void finite_check_kernel(const float* __restrict__ g, int64_t n, uint32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !(fabsf(g[i]) <= 3.402823466e38f);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void sgd_dense_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
}

// row /= ||row|| (Eigen row.norm(): the reduction order is Eigen's; ours is a
// fixed warp tree). collapse_flag: normals must not collapse (embedding.cpp:185).
__global__ void row_normalize_kernel(float* __restrict__ x, int64_t rows, int d, int mode,
                                     uint32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    float* row = x + r * d;
    float s = 0.f;
    for (int j = lane; j < d; j += 32) s = __fadd_rn(s, __fmul_rn(row[j], row[j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(kFull, s, o));
    const float n = __fsqrt_rn(s);
    if (!(n > 0.f)) {
      if (mode == 1 && lane == 0 && atomicCAS(&err[0], 0u, static_cast<uint32_t>(kErrNormalCollapsed)) == 0u)
        err[2] = static_cast<uint32_t>(r);
      continue;
    }
    for (int j = lane; j < d; j += 32) row[j] = __fdiv_rn(row[j], n);
  }
}

// embedding.cpp:192-198 on the rows this context holds (all of them, or the
// owned shard of a sharded context: the renorm is per row).
void renormalize_entities_impl(skg_ctx* ctx) {
  float* rows = ctx->shard ? ctx->shard->peers.ent[ctx->shard->rank] : ctx->tables.p;
  const int64_t n = ctx->shard ? ctx->shard->NEo : ctx->N;
  if (n == 0) return;
  row_normalize_kernel<<<grid_for(n * 32), 256, 0, ctx->stream>>>(rows, n, static_cast<int>(ctx->de), 0,
                                                                 ctx->err_words.p);
  count_launch();
  SKG_LAUNCH_CHECK();
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

// One id array to narrow: int64 source (HBM or UVA-mapped pinned host), int32
// destination, exclusive upper bound and the slot of its first-bad index.
struct NarrowJob {
  const int64_t* src;
  int32_t* dst;
  int64_t limit;
  uint32_t* bad;
};
struct NarrowJobs {
  NarrowJob j[3];
};

// Every array of one set_* call in one launch (blockIdx.y = array): 16-byte
// loads, four in flight per thread, so the pinned-host reads keep enough PCIe
// requests outstanding to run at DMA speed; validation (TripleBatch::validate,
// incidence.hpp:18-31), narrowing and the changed-data check in the same pass.
__global__ void __launch_bounds__(256) narrow_ids_kernel(NarrowJobs jobs, int64_t m, uint32_t* __restrict__ changed) {
  const NarrowJob J = jobs.j[blockIdx.y];
  bool diff = false;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(J.src) | reinterpret_cast<uintptr_t>(J.dst) * 2) & 15) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t n2 = m / 2;
    const longlong2* s2 = reinterpret_cast<const longlong2*>(J.src);
    int2* d2 = reinterpret_cast<int2*>(J.dst);
    constexpr int U = 4;
    for (int64_t base = tid; base < n2; base += U * stride) {
      longlong2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = base + u * stride;
        if (k < n2) v[u] = s2[k];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = base + u * stride;
        if (k >= n2) break;
        int2 w;
        if (v[u].x < 0 || v[u].x >= J.limit) atomicMin(J.bad, static_cast<uint32_t>(2 * k));
        if (v[u].y < 0 || v[u].y >= J.limit) atomicMin(J.bad, static_cast<uint32_t>(2 * k + 1));
        w.x = static_cast<int32_t>(v[u].x);
        w.y = static_cast<int32_t>(v[u].y);
        const int2 old = d2[k];
        diff |= old.x != w.x || old.y != w.y;
        d2[k] = w;
      }
    }
    done = 2 * n2;
  }
  for (int64_t i = done + tid; i < m; i += stride) {
    const int64_t v = J.src[i];
    if (v < 0 || v >= J.limit) atomicMin(J.bad, static_cast<uint32_t>(i));
    const int32_t w = static_cast<int32_t>(v);
    diff |= J.dst[i] != w;
    J.dst[i] = w;
  }
  if (diff) *changed = 0;
}

}  // namespace

// =================================================================== C ABI

extern "C" {

const char* skg_version(void) { return "skge-b200 0.1 (sm_100a)"; }

skg_status skg_create(int device, skg_ctx** out) {
  if (!out) return SKG_ERR_CONFIG;
  *out = nullptr;
  skg_ctx* ctx = new skg_ctx();
  ctx->device = device;
  const skg_status st = guard(ctx, [&] {
    int n = 0;
    SKG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw CudaError("no CUDA device " + std::to_string(device));
    cudaDeviceProp prop;
    SKG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError(std::string("skge-b200 is built for sm_100a; device is ") + prop.name);
    ctx->num_sms = prop.multiProcessorCount;
    SKG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    SKG_CUDA(cudaEventCreate(&ctx->ev0));
    SKG_CUDA(cudaEventCreate(&ctx->ev1));
    SKG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    SKG_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    SKG_CUDA(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->snap_ev, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->snap_cap_ev, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->fork_up_ev, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->join2_ev, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->aux_join, cudaEventDisableTiming));
    SKG_CUDA(cudaStreamCreateWithFlags(&ctx->up, cudaStreamNonBlocking));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->up_ev, cudaEventDisableTiming));

    ctx->speculate = false;  // opt-in: skg_set_deferred_uploads
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    SKG_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    ctx->err_words.ensure(4);
    ctx->counter.ensure(1);
    ctx->seed_eff.ensure(4);
    ctx->lr_dev.ensure(2);
    SKG_CUDA(cudaMallocHost(&ctx->h_seed, sizeof(uint64_t) * 4));
    SKG_CUDA(cudaMallocHost(&ctx->h_lr, sizeof(float) * 2));
    SKG_CUDA(cudaMallocHost(&ctx->h_err, sizeof(uint32_t) * 4));
    SKG_CUDA(cudaMallocHost(&ctx->h_spec, sizeof(uint32_t) * 4));
    SKG_CUDA(cudaMemset(ctx->err_words.p, 0, sizeof(uint32_t) * 4));
    SKG_CUDA(cudaMemset(ctx->counter.p, 0, sizeof(unsigned)));
    configure_hrt_kernels();
    configure_ht_kernels();
    configure_eval_kernels();
    configure_mult_kernels();
  });
  if (st != SKG_OK) {
    g_create_err = ctx->err;
    skg_destroy(ctx);
    return st;
  }
  *out = ctx;
  return SKG_OK;
}

void skg_destroy(skg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  dp_destroy(ctx);
  drop_graphs(ctx);
  if (ctx->h_stamps) cudaFreeHost(ctx->h_stamps);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->side2) cudaStreamDestroy(ctx->side2);
  if (ctx->snap_ev) cudaEventDestroy(ctx->snap_ev);
  if (ctx->snap_cap_ev) cudaEventDestroy(ctx->snap_cap_ev);
  if (ctx->fork_up_ev) cudaEventDestroy(ctx->fork_up_ev);
  if (ctx->join2_ev) cudaEventDestroy(ctx->join2_ev);
  if (ctx->aux_fork) cudaEventDestroy(ctx->aux_fork);
  if (ctx->aux_join) cudaEventDestroy(ctx->aux_join);
  if (ctx->up) {
    cudaStreamSynchronize(ctx->up);
    cudaStreamDestroy(ctx->up);
  }
  if (ctx->up_ev) cudaEventDestroy(ctx->up_ev);

  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->h_seed) cudaFreeHost(ctx->h_seed);
  if (ctx->h_lr) cudaFreeHost(ctx->h_lr);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->h_spec) cudaFreeHost(ctx->h_spec);
  destroy_host_narrow(ctx->narrow);
  ctx->narrow = nullptr;
  if (ctx->h_stage32) cudaFreeHost(ctx->h_stage32);
  if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* skg_last_error(const skg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
int skg_num_sms(const skg_ctx* ctx) { return ctx ? ctx->num_sms : 0; }
int64_t skg_last_launch_count(const skg_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

skg_status skg_synchronize(skg_ctx* ctx) {
  return guard(ctx, [&] {
    resolve_pending(ctx);
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_store_upload(skg_ctx* ctx, const skg_model_config* cfg, int64_t n_ent, int64_t n_rel,
                            const float* entity, const float* relation, const float* proj,
                            const float* normals) {
  return guard(ctx, [&] {
    if (!cfg) throw ConfigError("null model config");
    validate_model(*cfg);
    if (n_ent < 1 || n_rel < 1) throw ConfigError("store needs at least one entity and one relation");
    if (!entity || !relation) throw ShapeError("store: entity and relation tables are required");
    ctx->cfg = *cfg;
    ctx->N = n_ent;
    ctx->R = n_rel;
    ctx->de = width(cfg->model, cfg->dim_entity);  // complex: interleaved (re, im) pairs
    ctx->dr = width(cfg->model, cfg->dim_relation);
    ctx->tables.ensure(n_ent * ctx->de + n_rel * ctx->dr);
    SKG_CUDA(cudaMemcpyAsync(ctx->tables.p, entity, sizeof(float) * n_ent * ctx->de, cudaMemcpyHostToDevice,
                             ctx->stream));
    SKG_CUDA(cudaMemcpyAsync(ctx->tables.p + n_ent * ctx->de, relation, sizeof(float) * n_rel * ctx->dr,
                             cudaMemcpyHostToDevice, ctx->stream));
    ctx->proj.release();
    ctx->normals.release();
    if (proj) {
      ctx->proj.ensure(n_rel * ctx->dr * ctx->de);
      SKG_CUDA(cudaMemcpyAsync(ctx->proj.p, proj, sizeof(float) * ctx->proj.n, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (normals) {
      ctx->normals.ensure(n_rel * ctx->de);
      SKG_CUDA(cudaMemcpyAsync(ctx->normals.p, normals, sizeof(float) * ctx->normals.n, cudaMemcpyHostToDevice,
                               ctx->stream));
    }
    ctx->has_store = true;
    if (ctx->shard) {  // sharded: this rank keeps its owned rows and the relation replica
      if (n_ent != ctx->N || ctx->de != ctx->shard->d || n_rel * ctx->dr != static_cast<int64_t>(ctx->R) * ctx->shard->d)
        throw ConfigError("sharded context: store shape changed since init (release the shard first)");
      SKG_CUDA(cudaStreamSynchronize(ctx->stream));
      shard_scatter_store(ctx);
    }
    if (ctx->speculate)  // parameter snapshot of a speculative epoch (tables, proj, normals, aligned sections)
      ctx->backup.ensure(ctx->tables.n + ctx->proj.n + ctx->normals.n + 12);
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_store_download(skg_ctx* ctx, float* entity, float* relation, float* proj, float* normals) {
  return guard(ctx, [&] {
    if (!ctx->has_store) throw ConfigError("no parameter store uploaded");
    if (ctx->shard) shard_gather_store(ctx);  // every rank's owned rows (peer reads) into the full table
    if (entity)
      SKG_CUDA(cudaMemcpyAsync(entity, ctx->tables.p, sizeof(float) * ctx->N * ctx->de, cudaMemcpyDeviceToHost,
                               ctx->stream));
    if (relation)
      SKG_CUDA(cudaMemcpyAsync(relation, ctx->tables.p + ctx->N * ctx->de, sizeof(float) * ctx->R * ctx->dr,
                               cudaMemcpyDeviceToHost, ctx->stream));
    if (proj && ctx->proj.n)
      SKG_CUDA(cudaMemcpyAsync(proj, ctx->proj.p, sizeof(float) * ctx->proj.n, cudaMemcpyDeviceToHost, ctx->stream));
    if (normals && ctx->normals.n)
      SKG_CUDA(cudaMemcpyAsync(normals, ctx->normals.p, sizeof(float) * ctx->normals.n, cudaMemcpyDeviceToHost,
                               ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// Copies caller id arrays (int64, pinned or pageable) straight to HBM, then
// validates and narrows them on device (TripleBatch::validate semantics).
void upload_narrow(skg_ctx* ctx, const int64_t* const* srcs, int32_t* const* dsts, const int64_t* limits,
                   const int* slots, int count, int64_t m, uint32_t* bad_out) {
  ctx->stage_i64.ensure(3 * m + 1);
  ctx->bad_idx.ensure(3);
  SKG_CUDA(cudaMemsetAsync(ctx->bad_idx.p, 0xFF, sizeof(uint32_t) * 3, ctx->stream));
  NarrowJobs jobs{};
  for (int k = 0; k < count; ++k) {
    // Pinned (page-locked, UVA-mapped) caller arrays are read by the narrowing
    // kernel straight over PCIe: copy, validation and narrowing in one pass.
    // Pageable arrays are staged with a plain H2D copy first.
    const int64_t* src = nullptr;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, srcs[k]) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      src = static_cast<const int64_t*>(pa.devicePointer);
    else
      cudaGetLastError();
    if (!src) {
      SKG_CUDA(cudaMemcpyAsync(ctx->stage_i64.p + k * m, srcs[k], sizeof(int64_t) * m, cudaMemcpyHostToDevice,
                               ctx->stream));
      src = ctx->stage_i64.p + k * m;
    }
    jobs.j[k] = NarrowJob{src, dsts[k], limits[k], ctx->bad_idx.p + slots[k]};
  }
  const int64_t per = (m / 2 + 255) / 256;  // blocks for one 16-byte load per thread
  const int gx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(per, 4L * ctx->num_sms)));
  narrow_ids_kernel<<<dim3(gx, count), 256, 0, ctx->stream>>>(jobs, m, ctx->bad_idx.p + 2);
  count_launch();
  SKG_LAUNCH_CHECK();
  SKG_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->bad_idx.p, sizeof(uint32_t) * 3, cudaMemcpyDeviceToHost, ctx->stream));
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  bad_out[0] = ctx->h_err[0];
  bad_out[1] = ctx->h_err[1];
  bad_out[2] = ctx->h_err[2];
}

}  // extern "C"

namespace {

void set_triples_sync(skg_ctx* ctx, int64_t m, const int64_t* h, const int64_t* r, const int64_t* t, int64_t n_ent,
                      int64_t n_rel) {
    if (m > 0 && (!h || !r || !t)) throw ShapeError("triple batch: heads/relations/tails length mismatch");
    if (n_ent > INT32_MAX || n_rel > INT32_MAX || m > INT32_MAX) throw ShapeError("id space exceeds 32-bit device ids");
    // Re-uploading identical triples keeps data_version, so an epoch plan
    // prefetched inside the previous epoch's graph stays valid.
    bool same = ctx->triples_valid && m == ctx->M && n_ent == ctx->tN && n_rel == ctx->tR && ctx->H.n >= m + 1 &&
                ctx->Rl.n >= m + 1 && ctx->T.n >= m + 1;
    ctx->triples_valid = false;
    ctx->M = 0;
    ctx->has_neg = false;
    ctx->tN = n_ent;
    ctx->tR = n_rel;
    ctx->H.ensure(m + 1);
    ctx->Rl.ensure(m + 1);
    ctx->T.ensure(m + 1);
    if (m > 0) {
      const int64_t* srcs[3] = {h, r, t};
      int32_t* dsts[3] = {ctx->H.p, ctx->Rl.p, ctx->T.p};
      const int64_t lim[3] = {n_ent, n_rel, n_ent};
      const int slots[3] = {0, 1, 0};
      uint32_t bad[3];
      upload_narrow(ctx, srcs, dsts, lim, slots, 3, m, bad);
      same = same && bad[2] == 0xFFFFFFFFu;
      if (!same) ++ctx->data_version;
      if (bad[0] != 0xFFFFFFFFu && bad[0] <= bad[1])  // incidence.hpp:26-29: entity check first
        throw ShapeError("triple " + std::to_string(bad[0]) + ": entity id out of range");
      if (bad[1] != 0xFFFFFFFFu) throw ShapeError("triple " + std::to_string(bad[1]) + ": relation id out of range");
    } else if (!same) {
      ++ctx->data_version;
    }
    ctx->M = m;
    ctx->triples_valid = true;
    if (ctx->speculate && m > 0) {  // buffers of a later deferred re-upload, allocated outside any timed epoch
      ctx->stage_i64.ensure(5 * m + 1);
      ctx->spec_flags.ensure(4);
    }
}

void set_negatives_sync(skg_ctx* ctx, int64_t m, const int64_t* nh, const int64_t* nt) {
    if (m != ctx->M) throw ShapeError("negative set is not aligned with the positive triples");
    // negatives as they were when the triples were set: no new data_version for an identical re-upload
    bool same = ctx->neg_valid_version == ctx->data_version && ctx->NH.n >= m + 1 && ctx->NT.n >= m + 1;
    ctx->has_neg = false;
    ctx->NH.ensure(m + 1);
    ctx->NT.ensure(m + 1);
    if (m > 0) {
      const int64_t* srcs[2] = {nh, nt};
      int32_t* dsts[2] = {ctx->NH.p, ctx->NT.p};
      const int64_t lim[2] = {ctx->tN, ctx->tN};
      const int slots[2] = {0, 0};
      uint32_t bad[3];
      upload_narrow(ctx, srcs, dsts, lim, slots, 2, m, bad);
      same = same && bad[2] == 0xFFFFFFFFu;
      if (!same) ++ctx->data_version;
      if (bad[0] != 0xFFFFFFFFu) {
        ctx->neg_valid_version = ~0ull;
        throw ShapeError("triple " + std::to_string(bad[0]) + ": entity id out of range");
      }
    } else if (!same) {
      ++ctx->data_version;
    }
    ctx->has_neg = true;
    ctx->neg_valid_version = ctx->data_version;
}

// Page-locked caller array? Asked every time (no address cache: a pageable
// buffer re-allocated at a freed pinned address must not be deferred).
bool is_pinned(const void* p) {
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return pa.type == cudaMemoryTypeHost && pa.devicePointer != nullptr;
}

// Applies a deferred upload synchronously (every entry point other than
// set_triples / set_negatives / train_epoch sees the uploaded data).
void resolve_pending(skg_ctx* ctx) {
  if (!ctx->pend_tri) return;
  const int64_t* p[5];
  for (int k = 0; k < 5; ++k) p[k] = ctx->pend_ptr[k];
  const bool neg = ctx->pend_neg;
  ctx->pend_tri = ctx->pend_neg = false;
  set_triples_sync(ctx, ctx->M, p[0], p[1], p[2], ctx->tN, ctx->tR);
  if (neg) set_negatives_sync(ctx, ctx->M, p[3], p[4]);
}

// Deferred upload check: the caller's int64 ids (copied by DMA into
// stage_i64) against the device ids the speculative epoch used, with the
// validation of set_triples / set_negatives. flags: [0] first bad entity
// (h / t), [1] first bad relation, [2] first bad negative, [3] changed.
__global__ void spec_check_kernel(const int64_t* __restrict__ src, int64_t m, int64_t n_ent, int64_t n_rel,
                                  const int32_t* __restrict__ H, const int32_t* __restrict__ Rl,
                                  const int32_t* __restrict__ T, const int32_t* __restrict__ NH,
                                  const int32_t* __restrict__ NT, uint32_t* __restrict__ flags) {
  // Read-only and evict-first on the staged copy: the epoch running alongside
  // keeps its L2-resident tables (the staged ids are dead after this pass;
  // they are re-narrowed from HBM only when they differ).
  bool diff = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v[5] = {__ldcs(src + i), __ldcs(src + m + i), __ldcs(src + 2 * m + i), __ldcs(src + 3 * m + i),
                          __ldcs(src + 4 * m + i)};
    const int32_t* cur[5] = {H, Rl, T, NH, NT};
    if (v[0] < 0 || v[0] >= n_ent || v[2] < 0 || v[2] >= n_ent) atomicMin(flags, static_cast<uint32_t>(i));
    if (v[1] < 0 || v[1] >= n_rel) atomicMin(flags + 1, static_cast<uint32_t>(i));
    if (v[3] < 0 || v[3] >= n_ent || v[4] < 0 || v[4] >= n_ent) atomicMin(flags + 2, static_cast<uint32_t>(i));
#pragma unroll
    for (int k = 0; k < 5; ++k) diff |= __ldg(cur[k] + i) != static_cast<int32_t>(v[k]);
  }
  if (__any_sync(kFull, diff) && (threadIdx.x & 31) == 0) atomicOr(flags + 3, 1u);
}

__global__ void narrow_staged_kernel(const int64_t* __restrict__ src, int64_t m, int32_t* __restrict__ H,
                                     int32_t* __restrict__ Rl, int32_t* __restrict__ T, int32_t* __restrict__ NH,
                                     int32_t* __restrict__ NT) {
  int32_t* dst[5] = {H, Rl, T, NH, NT};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
#pragma unroll
    for (int k = 0; k < 5; ++k) dst[k][i] = static_cast<int32_t>(src[k * m + i]);
}

// Parameter snapshot / restore on the SMs (a D2D cudaMemcpy could queue
// behind the deferred upload's H2D transfer on a shared copy engine). Plain
// loads: an evict-first (streaming) read of the tables would demote the very
// L2 lines the epoch's gathers hit next (C1 epoch 0.73 -> 0.89 ms measured).
__global__ void copy_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  const int64_t n4 = n >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t done = 0;
  if (vec) {
    for (int64_t i = tid; i < n4; i += stride)
      reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
    done = 4 * n4;
  }
  for (int64_t i = done + tid; i < n; i += stride) dst[i] = src[i];
}

// Up to three float copies in one launch (blockIdx.y = segment): the
// speculative epoch's parameter snapshot / restore of tables, proj, normals.
struct CopySegs {
  const float* src[3];
  float* dst[3];
  int64_t n[3];
};
__global__ void copy_segs_kernel(const CopySegs c) {
  const int k = blockIdx.y;
  const float* __restrict__ src = c.src[k];
  float* __restrict__ dst = c.dst[k];
  const int64_t n = c.n[k], n4 = n >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t done = 0;
  if (vec) {
    for (int64_t i = tid; i < n4; i += stride)
      reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
    done = 4 * n4;
  }
  for (int64_t i = done + tid; i < n; i += stride) dst[i] = src[i];
}

void copy_float_segs(const float* const* src, float* const* dst, const int64_t* n, int num_sms, cudaStream_t s) {
  CopySegs c{};
  int k = 0;
  int64_t most = 0;
  for (int i = 0; i < 3; ++i)
    if (n[i] > 0) {
      c.src[k] = src[i];
      c.dst[k] = dst[i];
      c.n[k] = n[i];
      most = std::max(most, n[i]);
      ++k;
    }
  if (k == 0) return;
  const int64_t blocks = std::min<int64_t>((most / 4 + 255) / 256 + 1, 8LL * num_sms);
  copy_segs_kernel<<<dim3(static_cast<unsigned>(blocks), k), 256, 0, s>>>(c);
  count_launch();
  SKG_LAUNCH_CHECK();
}

// The parameters a speculative epoch mutates ([entity; relation], proj,
// normals) to / from ctx->backup (16-byte aligned sections).
void snapshot_params(skg_ctx* ctx, bool restore, cudaStream_t s) {
  const int64_t nt = ctx->tables.n, np = ctx->proj.n, nn = ctx->normals.n;
  const int64_t op = (nt + 3) / 4 * 4, on = op + (np + 3) / 4 * 4;
  ctx->backup.ensure(on + nn + 4);
  float* live[3] = {ctx->tables.p, ctx->proj.p, ctx->normals.p};
  float* saved[3] = {ctx->backup.p, ctx->backup.p + op, ctx->backup.p + on};
  const int64_t lens[3] = {nt, np, nn};
  if (restore)
    copy_float_segs(saved, live, lens, ctx->num_sms, s);
  else
    copy_float_segs(live, saved, lens, ctx->num_sms, s);
}

void copy_floats(const float* src, float* dst, int64_t n, int num_sms, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t blocks = std::min<int64_t>((n / 4 + 255) / 256 + 1, 8LL * num_sms);
  copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(src, dst, n);
  count_launch();
  SKG_LAUNCH_CHECK();
}

// ---- host-narrowed deferred uploads
// The caller's five int64 id arrays are narrowed to int32 by host threads in
// kWaves waves (triples [w L, (w + 1) L), L = ceil(m / kWaves)), wave-major in a
// pinned buffer: wave w holds its five arrays back to back. Each wave is
// DMA'd as soon as every thread has finished it, so the copy of half the
// bytes overlaps the narrowing of the next wave and the running epoch. The
// threads also do set_triples' / set_negatives' range checks (first bad
// index per category, like spec_check_kernel). SKG_SPEC_I64=1 keeps the int64 DMA.
constexpr int kWaves = 4;
}  // namespace

struct skg::HostNarrow {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv;
  uint64_t gen = 0;
  bool stop = false;
  int nt = 1;
  // job
  const int64_t* src[5] = {};
  void* dst = nullptr;
  bool w16 = false;  // ids fit 16 bits (every table <= 65536 rows): uint16 wire format
  int64_t m = 0, L = 0, n_ent = 0, n_rel = 0;
  std::atomic<int> wave_done[kWaves];
  std::atomic<uint32_t> bad[3];
  explicit HostNarrow(int n) : nt(n) {
    for (auto& w : wave_done) w = 0;
    for (int t = 0; t < nt; ++t) th.emplace_back([this, t] { loop(t); });
  }
  ~HostNarrow() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
      }
      work(t);
    }
  }
  static void atomic_min(std::atomic<uint32_t>& a, uint32_t v) {
    uint32_t cur = a.load(std::memory_order_relaxed);
    while (v < cur && !a.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
    }
  }
  void work(int t) {
    if (w16)
      work_t<uint16_t>(t);
    else
      work_t<int32_t>(t);
  }
  template <typename D>
  void work_t(int t) {
    for (int w = 0; w < kWaves; ++w) {
      const int64_t a = std::min<int64_t>(m, w * L), b = std::min<int64_t>(m, a + L), lw = b - a;
      const int64_t i0 = a + lw * t / nt, i1 = a + lw * (t + 1) / nt;
      D* base = static_cast<D*>(dst) + 5 * a;
      for (int k = 0; k < 5; ++k) {
        const int64_t* s = src[k];
        D* d = base + k * lw - a;
        const int64_t lim = k == 1 ? n_rel : n_ent;
        bool any = false;
        for (int64_t i = i0; i < i1; ++i) {  // vectorizable: narrow and flag, the index search only on a miss
          const int64_t v = s[i];
          any |= static_cast<uint64_t>(v) >= static_cast<uint64_t>(lim);
          d[i] = static_cast<D>(v);
        }
        if (any)
          for (int64_t i = i0; i < i1; ++i)
            if (static_cast<uint64_t>(s[i]) >= static_cast<uint64_t>(lim)) {
              atomic_min(bad[k == 1 ? 1 : (k <= 2 ? 0 : 2)], static_cast<uint32_t>(i));
              break;
            }
      }
      wave_done[w].fetch_add(1, std::memory_order_release);
    }
  }
  void start(const int64_t* const* s, void* d, bool narrow16, int64_t mm, int64_t ne, int64_t nr) {
    for (int k = 0; k < 5; ++k) src[k] = s[k];
    dst = d;
    w16 = narrow16;
    m = mm;
    L = (mm + kWaves - 1) / kWaves;
    n_ent = ne;
    n_rel = nr;
    for (auto& w : wave_done) w.store(0, std::memory_order_relaxed);
    for (auto& x : bad) x.store(0xFFFFFFFFu, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(mu);
      ++gen;
    }
    cv.notify_all();
  }
  void wait_wave(int w) {
    while (wave_done[w].load(std::memory_order_acquire) < nt) std::this_thread::yield();
  }
};

namespace {

void destroy_host_narrow(skg::HostNarrow* h) { delete h; }

// Compare the narrowed (wave-major) ids with the device ids the epoch used.
template <typename S>
__global__ void spec_check32_kernel(const S* __restrict__ st, int64_t m, int64_t L,
                                    const int32_t* __restrict__ H, const int32_t* __restrict__ Rl,
                                    const int32_t* __restrict__ T, const int32_t* __restrict__ NH,
                                    const int32_t* __restrict__ NT, uint32_t* __restrict__ flags) {
  bool diff = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = (i / L) * L, lw = min(L, m - a);
    const S* b = st + 5 * a + (i - a);
    diff |= (static_cast<int32_t>(__ldcs(b)) != __ldg(H + i)) | (static_cast<int32_t>(__ldcs(b + lw)) != __ldg(Rl + i)) |
            (static_cast<int32_t>(__ldcs(b + 2 * lw)) != __ldg(T + i)) |
            (static_cast<int32_t>(__ldcs(b + 3 * lw)) != __ldg(NH + i)) |
            (static_cast<int32_t>(__ldcs(b + 4 * lw)) != __ldg(NT + i));
  }
  if (__any_sync(kFull, diff) && (threadIdx.x & 31) == 0) atomicOr(flags + 3, 1u);
}

template <typename S>
__global__ void adopt_staged32_kernel(const S* __restrict__ st, int64_t m, int64_t L, int32_t* __restrict__ H,
                                      int32_t* __restrict__ Rl, int32_t* __restrict__ T, int32_t* __restrict__ NH,
                                      int32_t* __restrict__ NT) {
  int32_t* dst[5] = {H, Rl, T, NH, NT};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = (i / L) * L, lw = min(L, m - a);
#pragma unroll
    for (int k = 0; k < 5; ++k) dst[k][i] = static_cast<int32_t>(st[5 * a + k * lw + (i - a)]);
  }
}

// train_epoch with a deferred (pinned, identical-shape) upload pending: the
// copy runs on the DMA engines while the epoch trains on the current device
// ids; identical data (the common per-epoch re-upload) keeps the result.
// Otherwise the parameters are restored and the reference semantics apply:
// invalid ids throw set_triples' / set_negatives' ShapeError, new ids are
// adopted and the epoch is trained on them.
void train_epoch_speculative(skg_ctx* ctx, const skg_model_config& cfg, const skg_train_config& tc, int64_t epoch,
                             float lr, skg_epoch_report* rep) {
  static const bool dbg = std::getenv("SKG_SPEC_DEBUG") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int64_t m = ctx->M;
  const int64_t* src[5];
  for (int k = 0; k < 5; ++k) src[k] = ctx->pend_ptr[k];
  ctx->pend_tri = ctx->pend_neg = false;
  ctx->stage_i64.ensure(5 * m + 1);
  ctx->spec_flags.ensure(4);
  // the copy + check are enqueued right after the epoch graph is launched
  bool launched = false;
  static const bool i64 = [] {
    const char* v = std::getenv("SKG_SPEC_I64");
    return v && v[0] == '1';
  }();
  const bool narrowed = !i64 && m > 0;
  // wire format of the narrowed ids: uint16 when every id fits (C1-C3 tables),
  // else int32 (range-checked on the host either way)
  static const bool no16 = [] {
    const char* v = std::getenv("SKG_SPEC_NO16");
    return v && v[0] == '1';
  }();
  const bool w16 = narrowed && !no16 && ctx->tN <= 65536 && ctx->tR <= 65536;
  const int64_t wsz = w16 ? 2 : 4;
  if (narrowed) {
    if (!ctx->narrow) {
      // at most half the host's cores: a wave waits for its slowest thread, and
      // with every core busy one preempted thread costs a scheduler timeslice
      // (measured: 15 threads on 16 cores gave 1.1-1.4 ms step outliers, 8 none)
      const unsigned hc = std::thread::hardware_concurrency();
      int nt = static_cast<int>(std::max(1u, std::min(8u, hc / 2)));
      if (const char* e = std::getenv("SKG_NARROW_THREADS")) nt = std::max(1, std::atoi(e));
      ctx->narrow = new HostNarrow(nt);
    }
    if (ctx->h_stage32_cap < 5 * m) {
      if (ctx->h_stage32) cudaFreeHost(ctx->h_stage32);
      ctx->h_stage32 = nullptr;
      SKG_CUDA(cudaMallocHost(&ctx->h_stage32, sizeof(int32_t) * 5 * m));
      ctx->h_stage32_cap = 5 * m;
    }
    ctx->stage_i32.ensure(5 * m + 1);
  }
  bool in_epoch = true;
  // until the flags are read back, the check counts as a miss (changed data:
  // roll back and adopt), never as a stale hit
  ctx->h_spec[0] = ctx->h_spec[1] = ctx->h_spec[2] = 0xFFFFFFFFu;
  ctx->h_spec[3] = 1u;
  const std::function<void()> upload = [&]() {
    SKG_CUDA(cudaMemsetAsync(ctx->spec_flags.p, 0xFF, sizeof(uint32_t) * 3, ctx->up));
    SKG_CUDA(cudaMemsetAsync(ctx->spec_flags.p + 3, 0, sizeof(uint32_t), ctx->up));
    if (narrowed) {
      HostNarrow& hn = *ctx->narrow;
      hn.start(src, ctx->h_stage32, w16, m, ctx->tN, ctx->tR);
      char* hst = reinterpret_cast<char*>(ctx->h_stage32);
      char* dst = reinterpret_cast<char*>(ctx->stage_i32.p);
      for (int w = 0; w < kWaves; ++w) {
        const int64_t a = std::min<int64_t>(m, w * hn.L), b = std::min<int64_t>(m, a + hn.L);
        hn.wait_wave(w);
        if (b > a)
          SKG_CUDA(cudaMemcpyAsync(dst + wsz * 5 * a, hst + wsz * 5 * a, wsz * 5 * (b - a), cudaMemcpyHostToDevice,
                                   ctx->up));
      }
      ctx->upload_bytes += wsz * 5 * m;
      const unsigned g = static_cast<unsigned>(std::min<int64_t>(grid_for(m), 2LL * ctx->num_sms));
      if (w16)
        spec_check32_kernel<<<g, 256, 0, ctx->up>>>(reinterpret_cast<const uint16_t*>(ctx->stage_i32.p), m, hn.L,
                                                    ctx->H.p, ctx->Rl.p, ctx->T.p, ctx->NH.p, ctx->NT.p,
                                                    ctx->spec_flags.p);
      else
        spec_check32_kernel<<<g, 256, 0, ctx->up>>>(ctx->stage_i32.p, m, hn.L, ctx->H.p, ctx->Rl.p, ctx->T.p,
                                                    ctx->NH.p, ctx->NT.p, ctx->spec_flags.p);
    } else {
      for (int k = 0; k < 5; ++k)
        SKG_CUDA(cudaMemcpyAsync(ctx->stage_i64.p + k * m, src[k], sizeof(int64_t) * m, cudaMemcpyHostToDevice, ctx->up));
      ctx->upload_bytes += static_cast<int64_t>(sizeof(int64_t)) * 5 * m;
      spec_check_kernel<<<static_cast<unsigned>(std::min<int64_t>(grid_for(m), 2LL * ctx->num_sms)), 256, 0, ctx->up>>>(
          ctx->stage_i64.p, m, ctx->tN, ctx->tR, ctx->H.p, ctx->Rl.p, ctx->T.p, ctx->NH.p, ctx->NT.p, ctx->spec_flags.p);
    }
    count_launch();
    SKG_LAUNCH_CHECK();
    SKG_CUDA(cudaEventRecord(ctx->up_ev, ctx->up));
    // the epoch's own final sync also covers the check: its flags are read
    // back on the main stream after the upload's event
    SKG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->up_ev, 0));
    if (in_epoch)  // finish_epoch's publish kernel copies the flags with the losses
      ctx->pub_spec = ctx->spec_flags.p;
    else
      SKG_CUDA(cudaMemcpyAsync(ctx->h_spec, ctx->spec_flags.p, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost,
                               ctx->stream));
    launched = true;
  };
  // Parameter snapshot: a branch of the epoch graph itself (spec_graph: no
  // launches ahead of the graph), taken at the graph's start; batch 0 waits
  // for it before writing any parameter. Sharded contexts and the
  // multiplicative models (whose degenerate-batch path trains eagerly before
  // any graph launch, then throws) snapshot ahead of the launch.
  {
    const int64_t nt = ctx->tables.n, np = ctx->proj.n, nn = ctx->normals.n;  // backup sized before any capture
    ctx->backup.ensure((nt + 3) / 4 * 4 + (np + 3) / 4 * 4 + nn + 4);
  }
  const bool in_graph_snapshot = ctx->shard == nullptr && !is_mult(cfg);
  ctx->spec_graph = in_graph_snapshot;
  if (!in_graph_snapshot) {
    SKG_CUDA(cudaEventRecord(ctx->fork_up_ev, ctx->stream));
    SKG_CUDA(cudaStreamWaitEvent(ctx->up, ctx->fork_up_ev, 0));
    snapshot_params(ctx, false, ctx->up);
    SKG_CUDA(cudaEventRecord(ctx->snap_ev, ctx->up));
  }
  const auto t1 = clk::now();
  std::exception_ptr failed;
  try {
    train_epoch_impl(ctx, cfg, tc, epoch, lr, rep, &upload);
  } catch (...) {
    failed = std::current_exception();
  }
  ctx->spec_graph = false;
  // an in-graph snapshot exists iff the graph ran, i.e. the upload was enqueued after its launch
  const bool snapshot_taken = !in_graph_snapshot || launched;
  ctx->pub_spec = nullptr;
  in_epoch = false;
  if (!launched) upload();  // the epoch failed before its launch: still check the upload
  const auto t2 = clk::now();
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  uint32_t f[4];
  if (dbg) {
    const auto t3 = clk::now();
    auto us = [](clk::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
    std::fprintf(stderr, "spec: enqueue %.1f us, epoch %.1f us, upload wait %.1f us (graph %.1f us)\n", us(t1 - t0),
                 us(t2 - t1), us(t3 - t2), rep->t_backward_s * 1e6);
  }
  for (int k = 0; k < 4; ++k) f[k] = ctx->h_spec[k];
  if (narrowed)  // range checks ran on the host threads
    for (int k = 0; k < 3; ++k) f[k] = ctx->narrow->bad[k].load(std::memory_order_relaxed);
  const bool bad_tri = f[0] != 0xFFFFFFFFu || f[1] != 0xFFFFFFFFu, bad_neg = f[2] != 0xFFFFFFFFu;
  if (!bad_tri && !bad_neg && f[3] == 0) {  // identical re-upload: the speculative epoch stands
    ++ctx->spec_hits;
    if (failed) std::rethrow_exception(failed);
    return;
  }
  ++ctx->spec_misses;
  if (snapshot_taken) snapshot_params(ctx, true, ctx->stream);  // else the epoch never ran: nothing to undo
  for (auto& sl : ctx->slots) sl.key.clear();
  for (auto& k : ctx->perm_key) k.clear();
  ctx->has_neg = false;
  if (bad_tri) {  // set_triples' error (incidence.hpp:26-29: entity check first)
    ctx->triples_valid = false;
    ctx->M = 0;
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (f[0] != 0xFFFFFFFFu && f[0] <= f[1])
      throw ShapeError("triple " + std::to_string(f[0]) + ": entity id out of range");
    throw ShapeError("triple " + std::to_string(f[1]) + ": relation id out of range");
  }
  // adopt the uploaded ids (data changed, or the negatives are invalid)
  if (narrowed && w16)
    adopt_staged32_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(reinterpret_cast<const uint16_t*>(ctx->stage_i32.p),
                                                                m, ctx->narrow->L, ctx->H.p, ctx->Rl.p, ctx->T.p,
                                                                ctx->NH.p, ctx->NT.p);
  else if (narrowed)
    adopt_staged32_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(ctx->stage_i32.p, m, ctx->narrow->L, ctx->H.p,
                                                                ctx->Rl.p, ctx->T.p, ctx->NH.p, ctx->NT.p);
  else
    narrow_staged_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(ctx->stage_i64.p, m, ctx->H.p, ctx->Rl.p, ctx->T.p,
                                                              ctx->NH.p, ctx->NT.p);
  count_launch();
  SKG_LAUNCH_CHECK();
  ++ctx->data_version;
  SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (bad_neg) {  // set_negatives' error
    ctx->neg_valid_version = ~0ull;
    throw ShapeError("triple " + std::to_string(f[2]) + ": entity id out of range");
  }
  ctx->neg_valid_version = ctx->data_version;
  ctx->has_neg = true;
  train_epoch_impl(ctx, cfg, tc, epoch, lr, rep);
}

}  // namespace

extern "C" {

skg_status skg_set_deferred_uploads(skg_ctx* ctx, int32_t enable) {
  return guard(ctx, [&] {
    resolve_pending(ctx);
    ctx->speculate = enable != 0;
    if (ctx->speculate && ctx->M > 0) {  // buffers of a later deferred re-upload, allocated now
      ctx->stage_i64.ensure(5 * ctx->M + 1);
      ctx->spec_flags.ensure(4);
    }
    if (ctx->speculate && ctx->has_store)
      ctx->backup.ensure(ctx->tables.n + ctx->proj.n + ctx->normals.n + 12);
  });
}

skg_status skg_set_phase_timers(skg_ctx* ctx, int32_t enable) {
  return guard(ctx, [&] { ctx->phase_timers = enable != 0; });
}

skg_status skg_profile_shuffle_ms(skg_ctx* ctx, double* shuffle_ms) {
  return guard(ctx, [&] {
    if (shuffle_ms) *shuffle_ms = ctx->last_shuffle_ms;
  });
}

skg_status skg_upload_bytes(skg_ctx* ctx, int64_t* bytes) {
  return guard(ctx, [&] {
    if (bytes) *bytes = ctx->upload_bytes;
  });
}

skg_status skg_upload_stats(skg_ctx* ctx, int64_t* hits, int64_t* misses) {
  return guard(ctx, [&] {
    if (hits) *hits = ctx->spec_hits;
    if (misses) *misses = ctx->spec_misses;
  });
}

skg_status skg_set_triples(skg_ctx* ctx, int64_t m, const int64_t* h, const int64_t* r, const int64_t* t,
                           int64_t n_ent, int64_t n_rel) {
  return guard(ctx, [&] {
    if (m > 0 && (!h || !r || !t)) throw ShapeError("triple batch: heads/relations/tails length mismatch");
    // An identical-shape re-upload of pinned arrays (the per-epoch e2e loop)
    // is deferred to the next train_epoch, which copies it while it trains.
    if (ctx->speculate && !ctx->dp && !ctx->pend_tri && ctx->triples_valid && m > 0 && m == ctx->M &&
        n_ent == ctx->tN && n_rel == ctx->tR && ctx->neg_valid_version == ctx->data_version && is_pinned(h) &&
        is_pinned(r) && is_pinned(t)) {
      ctx->pend_tri = true;
      ctx->pend_neg = false;
      ctx->pend_ptr[0] = h;
      ctx->pend_ptr[1] = r;
      ctx->pend_ptr[2] = t;
      ctx->has_neg = false;  // as after any set_triples: negatives must follow
      return;
    }
    resolve_pending(ctx);
    set_triples_sync(ctx, m, h, r, t, n_ent, n_rel);
  });
}

skg_status skg_set_negatives(skg_ctx* ctx, int64_t m, const int64_t* nh, const int64_t* nt) {
  return guard(ctx, [&] {
    if (ctx->pend_tri && !ctx->pend_neg && m == ctx->M && m > 0 && is_pinned(nh) && is_pinned(nt)) {
      ctx->pend_neg = true;
      ctx->pend_ptr[3] = nh;
      ctx->pend_ptr[4] = nt;
      ctx->has_neg = true;
      return;
    }
    resolve_pending(ctx);
    set_negatives_sync(ctx, m, nh, nt);
  });
}

skg_status skg_negative_sample(skg_ctx* ctx, uint64_t seed, int32_t avoid, int64_t* out_h, int64_t* out_t) {
  return guard(ctx, [&] {
    resolve_pending(ctx);
    negative_sample_impl(ctx, seed, avoid != 0);
    if (out_h || out_t) {
      std::vector<int32_t> a(ctx->M), b(ctx->M);
      SKG_CUDA(cudaMemcpyAsync(a.data(), ctx->NH.p, sizeof(int32_t) * ctx->M, cudaMemcpyDeviceToHost, ctx->stream));
      SKG_CUDA(cudaMemcpyAsync(b.data(), ctx->NT.p, sizeof(int32_t) * ctx->M, cudaMemcpyDeviceToHost, ctx->stream));
      SKG_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int64_t i = 0; i < ctx->M; ++i) {
        if (out_h) out_h[i] = a[i];
        if (out_t) out_t[i] = b[i];
      }
    }
  });
}

skg_status skg_epoch_order(skg_ctx* ctx, int64_t m, uint64_t seed, int32_t shuffle, int64_t epoch,
                           int64_t* out_order) {
  return guard(ctx, [&] {
    if (m < 0) throw ShapeError("negative length");
    ctx->order.ensure(m + 1);
    if (shuffle) {
      ctx->h_seed[0] = epoch_seed(seed, epoch);
      SKG_CUDA(cudaMemcpyAsync(ctx->seed_eff.p, ctx->h_seed, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
      device_shuffle(ctx->seed_eff.p, m, ctx->order.p, ctx->shuffle, ctx->stream);
    } else {
      device_iota(ctx->order.p, m, ctx->stream);
    }
    std::vector<int32_t> o(m);
    if (m > 0)
      SKG_CUDA(cudaMemcpyAsync(o.data(), ctx->order.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < m; ++i) out_order[i] = o[i];
  });
}

skg_status skg_build_incidence(skg_ctx* ctx, int32_t layout, int64_t m, const int64_t* h, const int64_t* r,
                               const int64_t* t, int64_t n_ent, int64_t n_rel, int64_t* row_ptr,
                               int64_t* col_idx, float* vals, int64_t* nnz) {
  return guard(ctx, [&] {
    if (layout < SKG_LAYOUT_HT || layout > SKG_LAYOUT_MULT_CONJ) throw ConfigError("unknown incidence layout");
    upload_ids(ctx, m, h, r, t, n_ent, n_rel);
    if (layout >= SKG_LAYOUT_MULT) reject_self_loops(m, h, t);
    DevBuf<uint32_t> cnt, off;
    DevBuf<int64_t> drp, dcol;
    DevBuf<float> dval;
    DevBuf<uint32_t> tot;
    cnt.ensure(m + 1);
    off.ensure(m + 1);
    drp.ensure(m + 1);
    dcol.ensure(3 * m + 1);
    dval.ensure(3 * m + 1);
    tot.ensure(1);
    ScanPlan sp;
    if (m > 0) {
      incidence_count_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(ctx->tmp_i32.p, m, layout, cnt.p);
      exclusive_scan_u32(cnt.p, off.p, m, tot.p, sp, ctx->stream);
      incidence_fill_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(ctx->tmp_i32.p, m, layout, n_ent, off.p, drp.p,
                                                                 dcol.p, dval.p);
      count_launch(2);
      SKG_LAUNCH_CHECK();
    } else {
      SKG_CUDA(cudaMemsetAsync(drp.p, 0, sizeof(int64_t), ctx->stream));
    }
    SKG_CUDA(cudaMemcpyAsync(row_ptr, drp.p, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t z = row_ptr[m];
    if (z > 0) {
      SKG_CUDA(cudaMemcpyAsync(col_idx, dcol.p, sizeof(int64_t) * z, cudaMemcpyDeviceToHost, ctx->stream));
      SKG_CUDA(cudaMemcpyAsync(vals, dval.p, sizeof(float) * z, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    *nnz = z;
  });
}

}  // extern "C"

namespace {

// CsrMatrix::validate (sparse.hpp:54-68) on the host copy: the device kernels
// index through row_ptr / col_idx, so a malformed matrix is rejected up front.
void validate_csr(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci) {
  if (rows < 0 || cols < 0) throw ShapeError("csr: negative shape");
  if (rows > INT32_MAX || cols > INT32_MAX) throw ShapeError("csr: shape exceeds 32-bit device indices");
  if (rp[0] != 0) throw ShapeError("csr: row_ptr endpoints");
  for (int64_t r = 0; r < rows; ++r) {
    if (rp[r] > rp[r + 1]) throw ShapeError("csr: row_ptr decreasing");
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p)
      if (ci[p] < 0 || ci[p] >= cols) throw ShapeError("csr: column out of range");
  }
  if (rp[rows] > INT32_MAX) throw ShapeError("csr: nnz exceeds 32-bit device indices");
}

template <class T>
T* dev_copy(DevBuf<T>& b, const T* host, int64_t n, cudaStream_t s) {
  b.ensure(n + 1);
  if (n > 0) SKG_CUDA(cudaMemcpyAsync(b.p, host, sizeof(T) * n, cudaMemcpyHostToDevice, s));
  return b.p;
}

}  // namespace

extern "C" {

skg_status skg_coo_to_csr(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, int64_t nnz, const int64_t* rows,
                          const int64_t* cols, const float* vals, int64_t* row_ptr, int64_t* col_idx,
                          float* out_vals, int64_t* out_nnz) {
  return guard(ctx, [&] {
    if (nnz < 0 || (nnz > 0 && (!rows || !cols || !vals))) throw ShapeError("coo: rows/cols/vals length mismatch");
    for (int64_t i = 0; i < nnz; ++i)  // CooMatrix::validate (sparse.hpp:30-37)
      if (rows[i] < 0 || rows[i] >= num_rows || cols[i] < 0 || cols[i] >= num_cols)
        throw ShapeError("coo: entry " + std::to_string(i) + " outside declared shape");
    if (num_rows > INT32_MAX || num_cols > INT32_MAX || nnz > INT32_MAX)
      throw ShapeError("coo: shape exceeds 32-bit device indices");
    DevBuf<int64_t> dr, dc, orp, oc;
    DevBuf<float> dv, ov;
    const int64_t* r = dev_copy(dr, rows, nnz, ctx->stream);
    const int64_t* c = dev_copy(dc, cols, nnz, ctx->stream);
    const float* v = dev_copy(dv, vals, nnz, ctx->stream);
    orp.ensure(num_rows + 1);
    oc.ensure(nnz + 1);
    ov.ensure(nnz + 1);
    int64_t z = 0;
    sparse_coo_to_csr(num_rows, num_cols, nnz, r, c, v, orp.p, oc.p, ov.p, &z, ctx->stream);
    SKG_CUDA(cudaMemcpyAsync(row_ptr, orp.p, sizeof(int64_t) * (num_rows + 1), cudaMemcpyDeviceToHost, ctx->stream));
    if (z > 0) {
      SKG_CUDA(cudaMemcpyAsync(col_idx, oc.p, sizeof(int64_t) * z, cudaMemcpyDeviceToHost, ctx->stream));
      SKG_CUDA(cudaMemcpyAsync(out_vals, ov.p, sizeof(float) * z, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out_nnz = z;
  });
}

skg_status skg_csr_transpose(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                             const int64_t* col_idx, const float* vals, int64_t* t_row_ptr, int64_t* t_col_idx,
                             float* t_vals) {
  return guard(ctx, [&] {
    validate_csr(num_rows, num_cols, row_ptr, col_idx);
    const int64_t nnz = row_ptr[num_rows];
    DevBuf<int64_t> drp, dc, trp, tc;
    DevBuf<float> dv, tv;
    const int64_t* rp = dev_copy(drp, row_ptr, num_rows + 1, ctx->stream);
    const int64_t* c = dev_copy(dc, col_idx, nnz, ctx->stream);
    const float* v = dev_copy(dv, vals, nnz, ctx->stream);
    trp.ensure(num_cols + 1);
    tc.ensure(nnz + 1);
    tv.ensure(nnz + 1);
    sparse_transpose(num_rows, num_cols, nnz, rp, c, v, trp.p, tc.p, tv.p, ctx->stream);
    SKG_CUDA(cudaMemcpyAsync(t_row_ptr, trp.p, sizeof(int64_t) * (num_cols + 1), cudaMemcpyDeviceToHost,
                             ctx->stream));
    if (nnz > 0) {
      SKG_CUDA(cudaMemcpyAsync(t_col_idx, tc.p, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
      SKG_CUDA(cudaMemcpyAsync(t_vals, tv.p, sizeof(float) * nnz, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_spmm(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr, const int64_t* col_idx,
                    const float* vals, int64_t x_rows, int64_t d, const float* x, float* out) {
  return guard(ctx, [&] {
    if (num_cols != x_rows)  // sparse.hpp:244-246
      throw ShapeError("spmm: inner dimensions " + std::to_string(num_cols) + " vs " + std::to_string(x_rows));
    validate_csr(num_rows, num_cols, row_ptr, col_idx);
    if (d < 0 || d > INT32_MAX) throw ShapeError("spmm: bad dense width");
    const int64_t nnz = row_ptr[num_rows];
    DevBuf<int64_t> drp, dc;
    DevBuf<float> dv, dx, dout;
    const int64_t* rp = dev_copy(drp, row_ptr, num_rows + 1, ctx->stream);
    const int64_t* c = dev_copy(dc, col_idx, nnz, ctx->stream);
    const float* v = dev_copy(dv, vals, nnz, ctx->stream);
    const float* X = dev_copy(dx, x, x_rows * d, ctx->stream);
    dout.ensure(num_rows * d + 1);
    sparse_spmm(num_rows, rp, c, v, static_cast<int>(d), X, dout.p, ctx->num_sms, ctx->stream);
    if (num_rows * d > 0)
      SKG_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(float) * num_rows * d, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_spmm_transpose_add(skg_ctx* ctx, int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                                  const int64_t* col_idx, const float* vals, int64_t g_rows, int64_t d,
                                  const float* g, float* sink) {
  return guard(ctx, [&] {
    if (num_rows != g_rows) throw ShapeError("spmm_transpose: row count mismatch");  // sparse.hpp:275
    validate_csr(num_rows, num_cols, row_ptr, col_idx);
    if (d < 0 || d > INT32_MAX) throw ShapeError("spmm_transpose: bad dense width");
    const int64_t nnz = row_ptr[num_rows];
    DevBuf<int64_t> drp, dc;
    DevBuf<float> dv, dg, ds;
    const int64_t* rp = dev_copy(drp, row_ptr, num_rows + 1, ctx->stream);
    const int64_t* c = dev_copy(dc, col_idx, nnz, ctx->stream);
    const float* v = dev_copy(dv, vals, nnz, ctx->stream);
    const float* G = dev_copy(dg, g, g_rows * d, ctx->stream);
    float* S = dev_copy(ds, static_cast<const float*>(sink), num_cols * d, ctx->stream);
    sparse_spmm_transpose_add(num_rows, num_cols, nnz, rp, c, v, static_cast<int>(d), G, S, ctx->num_sms,
                              ctx->stream);
    if (num_cols * d > 0)
      SKG_CUDA(cudaMemcpyAsync(sink, S, sizeof(float) * num_cols * d, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_score_batch(skg_ctx* ctx, const skg_model_config* cfg, int64_t m, const int64_t* h,
                           const int64_t* r, const int64_t* t, float* scores, float* residual) {
  return guard(ctx, [&] {
    if (ctx->shard) shard_gather_store(ctx);  // per-op calls read the full tables
    check_config(ctx, *cfg, ctx->N, ctx->R);
    upload_ids(ctx, m, h, r, t, ctx->N, ctx->R);
    if (is_mult(*cfg)) reject_self_loops(m, h, t);
    if (m == 0) return;
    const int kind = kind_of(*cfg);
    ensure_workspace(ctx, m, kind);
    reset_err(ctx);
    FwdArgs a = base_fwd(ctx);
    a.H = ctx->tmp_i32.p;
    a.Rl = ctx->tmp_i32.p + m;
    a.T = ctx->tmp_i32.p + 2 * m;
    a.B = static_cast<int>(m);
    if (is_mult(*cfg)) {
      a.de = static_cast<int>(cfg->dim_entity);
      a.plane_rows = m;
      a.res_u = (residual && kind == kRotatE) ? ctx->res_u.p : nullptr;  // RotatE keeps q (ScoreBatch::v)
      launch_mult_forward(kind, false, a, ctx->num_sms, ctx->stream);
    } else if (is_ht(*cfg)) {
      ctx->ht_work.ensure(ht_work_floats(kind, m, ctx->de, ctx->dr, ctx->R));
      build_batch_plan(a.H, a.Rl, a.T, m, ctx->N, ctx->R, SKG_LAYOUT_HRT, ctx->plan, ctx->stream);
      BwdArgs ba{};
      ba.N = ctx->N;
      ba.d = static_cast<int>(ctx->de);
      ba.ent_val = ctx->plan.sorted_val;
      ba.seg_start = ctx->plan.seg_start;
      ba.seg_col = ctx->plan.seg_col;
      ba.seg_base = ctx->plan.seg_base;
      ba.batch = 0;
      ba.lr = ctx->lr_dev.p;
      ba.err = ctx->err_words.p;
      ht_score(kind, a, ba, ctx->ht_work.p, ctx->num_sms, ctx->stream, ctx->R);
    } else {
      launch_hrt_forward(kind, false, a, ctx->num_sms, ctx->stream);
    }
    SKG_CUDA(cudaMemcpyAsync(scores, ctx->scores.p, sizeof(float) * m, cudaMemcpyDeviceToHost, ctx->stream));
    if (residual && kind == kRotatE) {
      SKG_CUDA(cudaMemcpyAsync(residual, ctx->res_u.p, sizeof(float) * m * ctx->de, cudaMemcpyDeviceToHost,
                               ctx->stream));
    } else if (residual && !is_mult(*cfg)) {
      const int64_t d = cfg->model == SKG_TORUSE || cfg->model == SKG_TRANSE ? ctx->de : ctx->dr;
      SKG_CUDA(cudaMemcpyAsync(residual, ctx->res.p, sizeof(float) * m * d, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_score_backward(skg_ctx* ctx, const skg_model_config* cfg, int64_t m, const int64_t* h,
                              const int64_t* r, const int64_t* t, const float* up, float* g_entity,
                              float* g_relation, float* g_proj, float* g_normals) {
  return guard(ctx, [&] {
    if (ctx->shard) shard_gather_store(ctx);
    check_config(ctx, *cfg, ctx->N, ctx->R);
    upload_ids(ctx, m, h, r, t, ctx->N, ctx->R);
    if (is_mult(*cfg)) reject_self_loops(m, h, t);
    if (m == 0) return;
    const int kind = kind_of(*cfg);
    ensure_workspace(ctx, m, kind);
    reset_err(ctx);
    const int64_t ne = ctx->N * ctx->de, nr = ctx->R * ctx->dr;
    const int64_t np = ctx->proj.n, nn = ctx->normals.n;
    ctx->grad_sink.ensure(ne + nr + np + nn + 1);
    float* G = ctx->grad_sink.p;
    auto up_tab = [&](float* host, float* dev, int64_t n) {
      if (n == 0) return;
      if (host)
        SKG_CUDA(cudaMemcpyAsync(dev, host, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
      else
        SKG_CUDA(cudaMemsetAsync(dev, 0, sizeof(float) * n, ctx->stream));
    };
    up_tab(g_entity, G, ne);
    up_tab(g_relation, G + ne, nr);
    up_tab(g_proj, G + ne + nr, np);
    up_tab(g_normals, G + ne + nr + np, nn);
    ctx->tmp_f32.ensure(m);
    SKG_CUDA(cudaMemcpyAsync(ctx->tmp_f32.p, up, sizeof(float) * m, cudaMemcpyHostToDevice, ctx->stream));
    FwdArgs a = base_fwd(ctx);
    a.H = ctx->tmp_i32.p;
    a.Rl = ctx->tmp_i32.p + m;
    a.T = ctx->tmp_i32.p + 2 * m;
    a.B = static_cast<int>(m);
    a.upstream = ctx->tmp_f32.p;
    BwdArgs ba{};
    ba.X = G;
    ba.Xrel = G + ne;
    ba.scal = ctx->scal.p;
    ba.N = ctx->N;
    ba.d = static_cast<int>(ctx->de);
    ba.batch = 0;
    ba.lr = ctx->lr_dev.p;
    ba.err = ctx->err_words.p;
    if (is_mult(*cfg)) {
      a.de = static_cast<int>(cfg->dim_entity);
      a.plane_rows = m;
      a.res_u = nullptr;
      launch_mult_forward(kind, false, a, ctx->num_sms, ctx->stream);
      build_batch_plan(a.H, a.Rl, a.T, m, ctx->N, ctx->R, SKG_LAYOUT_HRT, ctx->plan, ctx->stream);
      ba.res = ctx->res.p;
      ba.plane_rows = m;
      ba.ent_val = ctx->plan.sorted_val;
      ba.seg_start = ctx->plan.seg_start;
      ba.seg_col = ctx->plan.seg_col;
      ba.seg_base = ctx->plan.seg_base;
      launch_segment_backward(kMultRows, false, ba, ctx->num_sms, ctx->stream);
    } else if (is_ht(*cfg)) {
      ctx->ht_work.ensure(ht_work_floats(kind, m, ctx->de, ctx->dr, ctx->R));
      build_batch_plan(a.H, a.Rl, a.T, m, ctx->N, ctx->R, SKG_LAYOUT_HRT, ctx->plan, ctx->stream);
      ba.res = ctx->res_u.p;
      ba.ent_val = ctx->plan.sorted_val;
      ba.seg_start = ctx->plan.seg_start;
      ba.seg_col = ctx->plan.seg_col;
      ba.seg_base = ctx->plan.seg_base;
      ht_score_backward(kind, a, ba, ctx->ht_work.p, G + ne + nr, G + ne + nr + np, ctx->num_sms, ctx->stream, ctx->R);
    } else {
      launch_hrt_forward(kind, false, a, ctx->num_sms, ctx->stream);
      build_batch_plan(a.H, a.Rl, a.T, m, ctx->N, ctx->R, SKG_LAYOUT_HRT, ctx->plan, ctx->stream);
      ba.res = ctx->res.p;
      ba.ent_val = ctx->plan.sorted_val;
      ba.seg_start = ctx->plan.seg_start;
      ba.seg_col = ctx->plan.seg_col;
      ba.seg_base = ctx->plan.seg_base;
      launch_segment_backward(kind, false, ba, ctx->num_sms, ctx->stream);
    }
    auto down = [&](float* host, const float* dev, int64_t n) {
      if (host && n) SKG_CUDA(cudaMemcpyAsync(host, dev, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
    };
    down(g_entity, G, ne);
    down(g_relation, G + ne, nr);
    down(g_proj, G + ne + nr, np);
    down(g_normals, G + ne + nr + np, nn);
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_margin_ranking_loss(skg_ctx* ctx, int64_t m, const float* pos, const float* neg, float margin,
                                   float* loss, float* d_pos, float* d_neg) {
  return guard(ctx, [&] {
    if (m < 0) throw ShapeError("margin_ranking_loss: length mismatch");
    if (m == 0) {
      *loss = 0.f;
      return;
    }
    DevBuf<float> buf;
    buf.ensure(5 * m + 1);
    float *p = buf.p, *n = buf.p + m, *dp = buf.p + 2 * m, *dn = buf.p + 3 * m, *term = buf.p + 4 * m;
    DevBuf<float> o;
    o.ensure(1);
    SKG_CUDA(cudaMemcpyAsync(p, pos, sizeof(float) * m, cudaMemcpyHostToDevice, ctx->stream));
    SKG_CUDA(cudaMemcpyAsync(n, neg, sizeof(float) * m, cudaMemcpyHostToDevice, ctx->stream));
    hinge_kernel<<<grid_for(m), 256, 0, ctx->stream>>>(p, n, m, margin, dp, dn, term);
    seq_sum_kernel<<<1, 1, 0, ctx->stream>>>(term, m, o.p);
    count_launch(2);
    SKG_LAUNCH_CHECK();
    SKG_CUDA(cudaMemcpyAsync(d_pos, dp, sizeof(float) * m, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaMemcpyAsync(d_neg, dn, sizeof(float) * m, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaMemcpyAsync(loss, o.p, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_sgd_step(skg_ctx* ctx, const float* g_entity, const float* g_relation, const float* g_proj,
                        const float* g_normals, float lr) {
  return guard(ctx, [&] {
    if (!ctx->has_store) throw ConfigError("no parameter store uploaded");
    if (ctx->shard) throw ConfigError("sgd_step on a sharded context: download, step and re-upload the store");
    const int64_t ne = ctx->N * ctx->de, nr = ctx->R * ctx->dr, np = ctx->proj.n, nn = ctx->normals.n;
    ctx->grad_sink.ensure(ne + nr + np + nn + 1);
    float* G = ctx->grad_sink.p;
    const float* hosts[4] = {g_entity, g_relation, g_proj, g_normals};
    const int64_t sizes[4] = {ne, nr, np, nn};
    int64_t off = 0;
    DevBuf<uint32_t> flags;
    flags.ensure(4);
    SKG_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(uint32_t) * 4, ctx->stream));
    for (int k = 0; k < 4; ++k) {
      if (sizes[k] && !hosts[k]) throw ShapeError("sgd_step: gradient shapes do not match the store");
      if (sizes[k]) {
        SKG_CUDA(cudaMemcpyAsync(G + off, hosts[k], sizeof(float) * sizes[k], cudaMemcpyHostToDevice, ctx->stream));
        finite_check_kernel<<<grid_for(sizes[k]), 256, 0, ctx->stream>>>(G + off, sizes[k], flags.p + k);
        count_launch();
      }
      off += sizes[k];
    }
    SKG_LAUNCH_CHECK();
    uint32_t hf[4];
    SKG_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    static const char* names[4] = {"entity embeddings", "relation embeddings", "relation projections",
                                   "hyperplane normals"};
    for (int k = 0; k < 4; ++k)
      if (hf[k]) throw TrainingError(std::string("non-finite gradient in ") + names[k]);
    float* params[4] = {ctx->tables.p, ctx->tables.p + ne, ctx->proj.p, ctx->normals.p};
    off = 0;
    for (int k = 0; k < 4; ++k) {
      if (sizes[k]) {
        sgd_dense_kernel<<<grid_for(sizes[k]), 256, 0, ctx->stream>>>(params[k], G + off, sizes[k], lr);
        count_launch();
      }
      off += sizes[k];
    }
    reset_err(ctx);
    if (nn) {
      row_normalize_kernel<<<grid_for(ctx->R * 32), 256, 0, ctx->stream>>>(ctx->normals.p, ctx->R,
                                                                          static_cast<int>(ctx->de), 1,
                                                                          ctx->err_words.p);
      count_launch();
    }
    SKG_LAUNCH_CHECK();
    SKG_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->err_words.p, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    raise_device_error(ctx->h_err, 0);
  });
}

skg_status skg_renormalize_entities(skg_ctx* ctx) {
  return guard(ctx, [&] {
    if (!ctx->has_store) throw ConfigError("no parameter store uploaded");
    renormalize_entities_impl(ctx);
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_train_epoch(skg_ctx* ctx, const skg_model_config* cfg, const skg_train_config* tc, int64_t epoch,
                           float lr, skg_epoch_report* rep) {
  return guard(ctx, [&] {
    if (ctx->pend_tri && ctx->pend_neg) {
      train_epoch_speculative(ctx, *cfg, *tc, epoch, lr, rep);
      return;
    }
    resolve_pending(ctx);
    train_epoch_impl(ctx, *cfg, *tc, epoch, lr, rep);
  });
}

skg_status skg_profile_epoch(skg_ctx* ctx, const skg_model_config* cfg, const skg_train_config* tc,
                             int64_t epoch, float lr, skg_epoch_report* rep, double* fwd_ms, double* bwd_ms,
                             double* plan_ms) {
  return guard(ctx, [&] {
    resolve_pending(ctx);
    EpochShape es{};
    prepare_epoch(ctx, *cfg, *tc, es);
    set_epoch_params(ctx, *tc, lr);
    set_slot_seed(ctx, ctx->cur, epoch_seed(tc->seed, epoch));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<cudaEvent_t> ev;
    // The plan, then every batch, each phase bracketed by event record nodes, in
    // one captured graph: the phase times are the kernels' own, without the host
    // launch gaps an eagerly enqueued epoch leaves between them (no overlap).
    cudaGraph_t g = nullptr;
    cudaGraphExec_t gx = nullptr;
    SKG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_epoch(ctx, es, &ev);
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &g);
      if (g) cudaGraphDestroy(g);
      for (auto x : ev) cudaEventDestroy(x);
      throw;
    }
    SKG_CUDA(cudaStreamEndCapture(ctx->stream, &g));
    struct Cleanup {  // graph, its instance and the events, on every exit
      cudaGraph_t& g;
      cudaGraphExec_t& gx;
      std::vector<cudaEvent_t>& ev;
      ~Cleanup() {
        if (gx) cudaGraphExecDestroy(gx);
        if (g) cudaGraphDestroy(g);
        for (auto x : ev) cudaEventDestroy(x);
      }
    } cleanup{g, gx, ev};
    apply_l2_policy(ctx, g);
    SKG_CUDA(cudaGraphInstantiate(&gx, g, 0));
    SKG_CUDA(cudaGraphLaunch(gx, ctx->stream));
    ctx->last_slot = ctx->cur;
    ctx->slots[0].key.clear();
    ctx->slots[1].key.clear();
    ctx->perm_key[0].clear();
    ctx->perm_key[1].clear();
    finish_epoch(ctx, es, epoch, rep);
    auto el = [&](size_t a, size_t b) {
      float ms = 0.f;
      SKG_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
      return static_cast<double>(ms);
    };
    ctx->last_shuffle_ms = el(0, 1);  // the epoch's permutation (two epochs ahead in the graphs)
    *plan_ms = el(1, 2);              // the transposed-incidence plan of the epoch
    double f = 0, b = 0;
    const size_t per = (ev.size() - 3) / es.nb;  // marks per batch
    for (int64_t k = 0; k < es.nb; ++k) {
      const size_t s0 = 2 + k * per;
      f += el(s0, s0 + 1);
      b += el(s0 + 1, s0 + per);
    }
    *fwd_ms = f / es.nb;
    *bwd_ms = b / es.nb;
    rep->t_forward_s = f * 1e-3;
    rep->t_backward_s = b * 1e-3;
    rep->t_step_s = 0.0;
  });
}

}  // extern "C"

namespace {
// Random-row gather probe (the roofline denominator for L2-resident tables):
// every warp gathers rows of `rf` floats at pseudo-random indices with 128-bit
// loads, 4 rows in flight per warp, full occupancy. Returns nothing useful; the
// XOR of the loaded words defeats dead-code elimination.
__global__ void __launch_bounds__(256) gather_probe_kernel(const float4* __restrict__ X, int64_t nrows, int rf4,
                                                           int64_t total_rows, uint32_t* __restrict__ sink) {
  // unit = one 512-byte chunk of a row (32 lanes x 16 B); 8 units in flight per warp
  constexpr int kU = 8;
  const int lane = threadIdx.x & 31;
  const int per_row = rf4 / 32;
  const int lg = per_row == 1 ? 0 : per_row == 2 ? 1 : per_row == 4 ? 2 : 3;
  const int64_t total_units = total_rows * per_row;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int64_t i = gw * kU; i < total_units; i += nw * kU) {
    float4 v[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {  // cheap index math: the probe must be bound by the loads
      const uint32_t u = static_cast<uint32_t>(i + q);
      const uint32_t r = u >> lg;
      const uint32_t h = r * 0x9E3779B9u;
      const uint32_t row = __umulhi(h, static_cast<uint32_t>(nrows));
      v[q] = (i + q) < total_units ? __ldg(X + static_cast<size_t>(row) * rf4 + ((u & ((1u << lg) - 1)) << 5) + lane)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < kU; ++q)
      acc ^= __float_as_uint(v[q].x) ^ __float_as_uint(v[q].y) ^ __float_as_uint(v[q].z) ^ __float_as_uint(v[q].w);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}
}  // namespace

extern "C" skg_status skg_measure_gather(skg_ctx* ctx, int64_t table_bytes, int32_t row_floats, double* gbs) {
  return guard(ctx, [&] {
    if (row_floats != 128 && row_floats != 256 && row_floats != 512 && row_floats != 1024)
      throw ConfigError("measure_gather: row_floats 128, 256, 512 or 1024");
    const int64_t nrows = std::max<int64_t>(1, table_bytes / (4LL * row_floats));
    DevBuf<float> tab;
    tab.ensure(nrows * row_floats);
    SKG_CUDA(cudaMemsetAsync(tab.p, 0, sizeof(float) * nrows * row_floats, ctx->stream));
    DevBuf<uint32_t> sink;
    sink.ensure(1);
    const int64_t total = std::max<int64_t>(4LL << 20, nrows);  // rows gathered per launch
    const int grid = ctx->num_sms * 8;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {  // first launch warms the table into L2 (or not, if it is larger)
      SKG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
      gather_probe_kernel<<<grid, 256, 0, ctx->stream>>>(reinterpret_cast<const float4*>(tab.p), nrows,
                                                         row_floats / 4, total, sink.p);
      SKG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
      SKG_LAUNCH_CHECK();
      SKG_CUDA(cudaEventSynchronize(ctx->ev1));
      float ms = 0.f;
      SKG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      if (rep > 0) best = std::min(best, ms);
    }
    *gbs = static_cast<double>(total) * row_floats * 4.0 / (best * 1e-3) / 1e9;
  });
}

extern "C" {

skg_status skg_flush_l2(skg_ctx* ctx) {
  return guard(ctx, [&] {
    ctx->flush_buf.ensure(256ll << 20);
    SKG_CUDA(cudaMemsetAsync(ctx->flush_buf.p, 0x5a, 256ull << 20, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

skg_status skg_plan_stats(skg_ctx* ctx, int64_t batch, int64_t* segments, int64_t* entries,
                          int64_t* relation_segments) {
  return guard(ctx, [&] {
    resolve_pending(ctx);
    if (ctx->shard) {  // this rank's owned-column plan (shard.cu)
      const ShardPlanBufs& p = ctx->shard->plan[ctx->last_slot];
      if (batch < 0 || batch >= p.nb || !p.seg_base) throw ShapeError("plan_stats: no such batch");
      uint32_t sb[2];
      SKG_CUDA(cudaMemcpy(sb, p.seg_base + batch, sizeof(sb), cudaMemcpyDeviceToHost));
      uint32_t e0 = 0, e1 = 0;
      if (sb[1] > sb[0]) {
        SKG_CUDA(cudaMemcpy(&e0, p.seg_start + sb[0], sizeof(uint32_t), cudaMemcpyDeviceToHost));
        SKG_CUDA(cudaMemcpy(&e1, p.seg_start + sb[1], sizeof(uint32_t), cudaMemcpyDeviceToHost));
      }
      std::vector<uint32_t> cols(sb[1] - sb[0]);
      if (!cols.empty())
        SKG_CUDA(cudaMemcpy(cols.data(), p.seg_col + sb[0], sizeof(uint32_t) * cols.size(), cudaMemcpyDeviceToHost));
      int64_t nrel = 0;
      for (uint32_t c : cols) nrel += (c & 0x80000000u) != 0;
      *segments = sb[1] - sb[0];
      *entries = static_cast<int64_t>(e1) - e0;
      *relation_segments = nrel;
      return;
    }
    if (batch < 0 || batch >= ctx->slots[ctx->last_slot].plan.nb || !ctx->slots[ctx->last_slot].plan.seg_base) throw ShapeError("plan_stats: no such batch");
    uint32_t sb[2];
    SKG_CUDA(cudaMemcpy(sb, ctx->slots[ctx->last_slot].plan.seg_base + batch, sizeof(sb), cudaMemcpyDeviceToHost));
    uint32_t e0 = 0, e1 = 0;
    SKG_CUDA(cudaMemcpy(&e0, ctx->slots[ctx->last_slot].plan.seg_start + sb[0], sizeof(uint32_t), cudaMemcpyDeviceToHost));
    SKG_CUDA(cudaMemcpy(&e1, ctx->slots[ctx->last_slot].plan.seg_start + sb[1], sizeof(uint32_t), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> cols(sb[1] - sb[0]);
    if (!cols.empty())
      SKG_CUDA(cudaMemcpy(cols.data(), ctx->slots[ctx->last_slot].plan.seg_col + sb[0], sizeof(uint32_t) * cols.size(),
                          cudaMemcpyDeviceToHost));
    int64_t nrel = 0;
    for (uint32_t c : cols) nrel += c >= ctx->N;
    *segments = sb[1] - sb[0];
    *entries = static_cast<int64_t>(e1) - e0;
    *relation_segments = nrel;
  });
}

skg_status skg_fit(skg_ctx* ctx, const skg_model_config* cfg, const skg_train_config* tc,
                   skg_epoch_report* reports) {
  return guard(ctx, [&] {
    resolve_pending(ctx);  // training.cpp:166-195
    validate_model(*cfg);
    validate_train(*tc);
    if (tc->epochs == 0) return;
    const bool no_self_loops = is_mult(*cfg);  // training.cpp:176
    negative_sample_impl(ctx, tc->seed, no_self_loops);
    for (int64_t e = 0; e < tc->epochs; ++e) {
      if (tc->resample_negatives && e > 0)
        negative_sample_impl(ctx, tc->seed + static_cast<uint64_t>(e) * 0x9E3779B9ULL, no_self_loops);
      float lr = tc->lr;
      if (tc->has_scheduler)
        lr = tc->lr * static_cast<float>(std::pow(tc->decay_factor, double(e / tc->decay_every)));
      skg_epoch_report rep{};
      train_epoch_impl(ctx, *cfg, *tc, e, lr, &rep);
      if (tc->renorm_entities) renormalize_entities_impl(ctx);
      reports[e] = rep;
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"

extern "C" skg_status skg_dp_shard(int64_t m, int64_t batch_size, int32_t world, int32_t rank, int64_t* out) {
  if (m < 1 || batch_size < 1 || world < 1 || rank < 0 || rank >= world || batch_size % world != 0)
    return SKG_ERR_CONFIG;
  dp_shard(m, std::min(batch_size, m), world, rank, out);
  return SKG_OK;
}

// rank_entity / evaluate (eval.cpp:16-96) on device for the translational
// hrt models: ranks[2i] = tail-side rank, ranks[2i + 1] = head-side rank.
extern "C" skg_status skg_rank_entities(skg_ctx* ctx, const skg_model_config* cfg, int64_t q, const int64_t* heads,
                                        const int64_t* relations, const int64_t* tails, int32_t protocol,
                                        int64_t nf, const int64_t* fh, const int64_t* fr, const int64_t* ft,
                                        int64_t* ranks) {
  return guard(ctx, [&] {
    if (ctx->shard) shard_gather_store(ctx);
    check_config(ctx, *cfg, ctx->N, ctx->R);
    const int kind = kind_of(*cfg);
    if (!eval_supported(kind)) throw ConfigError("rank_entities: model not supported");
    if (protocol != 0 && protocol != 1) throw ConfigError("rank_entities: protocol must be 0 (raw) or 1 (filtered)");
    for (int64_t i = 0; i < q; ++i)
      if (heads[i] < 0 || heads[i] >= ctx->N || tails[i] < 0 || tails[i] >= ctx->N || relations[i] < 0 ||
          relations[i] >= ctx->R)
        throw ShapeError("rank_entity: query ids out of range");  // eval.cpp:21
    if (q == 0) return;
    std::vector<int32_t> host;
    validate_ids(q, heads, relations, tails, ctx->N, ctx->R, host);
    DevBuf<int32_t> qd, fd;
    qd.ensure(3 * q);
    DevBuf<uint64_t> table;
    uint64_t cap = 0;
    if (protocol == 1) {
      std::vector<int32_t> fhost;
      validate_ids(nf, fh, fr, ft, ctx->N, ctx->R, fhost);
      cap = eval_filter_capacity(nf);
      table.ensure(static_cast<int64_t>(cap));
      fd.ensure(3 * nf + 1);
      if (nf > 0)
        SKG_CUDA(cudaMemcpyAsync(fd.p, fhost.data(), sizeof(int32_t) * 3 * nf, cudaMemcpyHostToDevice, ctx->stream));
      eval_build_filter(fd.p, fd.p + nf, fd.p + 2 * nf, nf, ctx->N, ctx->R, table.p, cap, ctx->stream);
    }
    DevBuf<uint32_t> better;
    DevBuf<float> te;
    better.ensure(2 * q);
    te.ensure(2 * q);
    const uint64_t* tp = protocol == 1 ? table.p : nullptr;
    std::vector<uint32_t> b(2 * q);
    if (eval_exact(kind)) {  // TransE / TorusE: the stacked tables as they are
      SKG_CUDA(cudaMemcpyAsync(qd.p, host.data(), sizeof(int32_t) * 3 * q, cudaMemcpyHostToDevice, ctx->stream));
      eval_rank(kind, ctx->tables.p, ctx->tables.p + ctx->N * ctx->de, ctx->N, ctx->R,
                static_cast<int>(is_mult(*cfg) ? cfg->dim_entity : ctx->de),
                qd.p, qd.p + q, qd.p + 2 * q, q, tp, cap, better.p, te.p, ctx->num_sms, ctx->stream);
      SKG_CUDA(cudaMemcpyAsync(b.data(), better.p, sizeof(uint32_t) * 2 * q, cudaMemcpyDeviceToHost, ctx->stream));
    } else {  // TransH / TransR: per relation, rank against the projected entity table
      const int dr = static_cast<int>(ctx->dr);
      DevBuf<float> pe;
      pe.ensure(ctx->N * dr);
      std::vector<std::vector<int64_t>> by_rel(static_cast<size_t>(ctx->R));
      for (int64_t i = 0; i < q; ++i) by_rel[static_cast<size_t>(relations[i])].push_back(i);
      std::vector<int32_t> sub;
      std::vector<uint32_t> bs;
      for (int64_t r = 0; r < ctx->R; ++r) {
        const auto& ids = by_rel[static_cast<size_t>(r)];
        if (ids.empty()) continue;
        const int64_t m = static_cast<int64_t>(ids.size());
        sub.resize(3 * m);
        for (int64_t k = 0; k < m; ++k) {
          sub[k] = host[ids[k]];
          sub[m + k] = host[q + ids[k]];
          sub[2 * m + k] = host[2 * q + ids[k]];
        }
        SKG_CUDA(cudaMemcpyAsync(qd.p, sub.data(), sizeof(int32_t) * 3 * m, cudaMemcpyHostToDevice, ctx->stream));
        eval_project(kind, ctx->tables.p, ctx->proj.p, ctx->normals.p, r, ctx->N, static_cast<int>(ctx->de), dr, pe.p,
                     ctx->stream);
        eval_rank(kind, pe.p, ctx->tables.p + ctx->N * ctx->de, ctx->N, ctx->R, dr, qd.p, qd.p + m, qd.p + 2 * m, m,
                  tp, cap, better.p, te.p, ctx->num_sms, ctx->stream);
        bs.resize(2 * m);
        SKG_CUDA(cudaMemcpyAsync(bs.data(), better.p, sizeof(uint32_t) * 2 * m, cudaMemcpyDeviceToHost, ctx->stream));
        SKG_CUDA(cudaStreamSynchronize(ctx->stream));  // qd / better are reused by the next relation
        for (int64_t k = 0; k < m; ++k) {
          b[2 * ids[k]] = bs[2 * k];
          b[2 * ids[k] + 1] = bs[2 * k + 1];
        }
      }
    }
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < 2 * q; ++i) ranks[i] = static_cast<int64_t>(b[i]) + 1;
  });
}

extern "C" int32_t skg_debug_mt_jump_selftest(uint64_t seed, int64_t jump) {
  try {
    return skg::mt_jump_selftest(seed, jump) ? 1 : 0;
  } catch (...) {
    return 0;
  }
}

extern "C" int64_t skg_debug_transr_trace(int32_t enable, unsigned long long* out, int64_t cap) {
  try {
    return transr_trace(enable, out, cap);
  } catch (...) {
    return -1;
  }
}

extern "C" int64_t skg_debug_bwd_trace(int32_t enable, unsigned long long* out, uint32_t* info, int64_t cap) {
  try {
    return skg::bwd_trace(enable, out, info, cap);
  } catch (...) {
    return -1;
  }
}

extern "C" int64_t skg_debug_transh_trace(int32_t enable, unsigned long long* out, int64_t cap) {
  try {
    return transh_trace(enable, out, cap);
  } catch (...) {
    return -1;
  }
}

extern "C" skg_status skg_debug_tc_gemm(skg_ctx* ctx, int32_t mode, const float* A, const float* B, float* D) {
  return guard(ctx, [&] {
    if (mode < 0 || mode > 2) throw ConfigError("debug_tc_gemm: mode 0..2");
    DevBuf<float> buf;
    buf.ensure(3 * 128 * 128);
    SKG_CUDA(cudaMemcpyAsync(buf.p, A, sizeof(float) * 128 * 128, cudaMemcpyHostToDevice, ctx->stream));
    SKG_CUDA(cudaMemcpyAsync(buf.p + 128 * 128, B, sizeof(float) * 128 * 128, cudaMemcpyHostToDevice, ctx->stream));
    transr_tc_selftest(mode, buf.p, buf.p + 128 * 128, buf.p + 2 * 128 * 128, ctx->stream);
    SKG_CUDA(cudaMemcpyAsync(D, buf.p + 2 * 128 * 128, sizeof(float) * 128 * 128, cudaMemcpyDeviceToHost, ctx->stream));
    SKG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// =================================================================== row-sharded data parallel

namespace {
struct ShardHandle {  // what one rank publishes to the others (skg_shard_export)
  cudaIpcMemHandle_t mem;
  int32_t device, rank, world, pad;
  uint64_t arena_bytes;
};
static_assert(sizeof(ShardHandle) <= SKG_SHARD_HANDLE_BYTES, "shard handle size");

template <class F>
skg_status guard_group(skg_ctx* const* ctxs, int world, F&& f) {
  if (!ctxs || world < 1) return SKG_ERR_CONFIG;
  for (int k = 0; k < world; ++k)
    if (!ctxs[k]) return SKG_ERR_CONFIG;
  int failed = 0;
  const skg_status st = guard(ctxs[0], [&] { f(failed); });
  if (st != SKG_OK && failed != 0) ctxs[failed]->err = ctxs[0]->err;
  return st;
}
}  // namespace

extern "C" {

skg_status skg_shard_group_init(skg_ctx* const* ctxs, int world, int64_t batch_size) {
  return guard_group(ctxs, world, [&](int& failed) {
    for (int k = 0; k < world; ++k) {
      skg_ctx* c = ctxs[k];
      if (c->shard) throw ConfigError("sharded tables already initialised on this context");
      if (c->dp) throw ConfigError("context already joined a replicated (NCCL) data-parallel group");
      if (k > 0 && (c->N != ctxs[0]->N || c->R != ctxs[0]->R || c->de != ctxs[0]->de || c->M != ctxs[0]->M))
        throw ConfigError("sharded group: contexts hold different stores or triples");
    }
    // Ranks sharing a device run their epoch graphs concurrently and wait for
    // each other in barrier kernels: each rank's streams need their own
    // hardware queue, or a spinning barrier can block a peer queued behind it.
    int per_dev = 1;
    for (int k = 0; k < world; ++k) {
      int c = 0;
      for (int j = 0; j < world; ++j) c += ctxs[j]->device == ctxs[k]->device;
      per_dev = std::max(per_dev, c);
    }
    // Measured on one B200: 2 and 4 ranks per device run; 8 ranks per device
    // stall in the barriers even with 32 hardware queues (the epoch graphs'
    // internal branch streams add to the 3 per rank).
    if (per_dev > 4) throw ConfigError("sharded group: at most 4 ranks may share one device");
    if (per_dev > 1) {
      const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
      const int conns = e ? std::atoi(e) : 8;
      if (conns < 3 * per_dev)
        throw ConfigError("sharded group with " + std::to_string(per_dev) +
                          " ranks on one device needs CUDA_DEVICE_MAX_CONNECTIONS >= " + std::to_string(3 * per_dev) +
                          " (set before the first CUDA call)");
    }
    std::vector<void*> bases(static_cast<size_t>(world));
    try {
      for (int k = 0; k < world; ++k) {
        failed = k;
        SKG_CUDA(cudaSetDevice(ctxs[k]->device));
        resolve_pending(ctxs[k]);
        shard_alloc(ctxs[k], k, world, batch_size);
        bases[k] = ctxs[k]->shard->arena;
      }
      for (int k = 0; k < world; ++k)  // peer access between distinct devices (same device: plain pointers)
        for (int j = 0; j < world; ++j) {
          if (ctxs[k]->device == ctxs[j]->device) continue;
          SKG_CUDA(cudaSetDevice(ctxs[k]->device));
          const cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[j]->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SKG_CUDA(e);
          cudaGetLastError();
        }
      for (int k = 0; k < world; ++k) {
        failed = k;
        SKG_CUDA(cudaSetDevice(ctxs[k]->device));
        shard_link(ctxs[k], bases.data());
      }
    } catch (...) {
      for (int k = 0; k < world; ++k) shard_destroy(ctxs[k]);
      SKG_CUDA(cudaSetDevice(ctxs[0]->device));
      throw;
    }
    SKG_CUDA(cudaSetDevice(ctxs[0]->device));
  });
}

skg_status skg_shard_group_train_epoch(skg_ctx* const* ctxs, int world, const skg_model_config* cfg,
                                       const skg_train_config* tc, int64_t epoch, float lr,
                                       skg_epoch_report* reports) {
  return guard_group(ctxs, world, [&](int& failed) {
    std::vector<StagedEpoch> sg(static_cast<size_t>(world));
    for (int k = 0; k < world; ++k) {  // host-side work of every rank first (no barrier is running yet)
      failed = k;
      if (!ctxs[k]->shard || ctxs[k]->shard->world != world || ctxs[k]->shard->rank != k)
        throw ConfigError("sharded group: contexts are not ranks 0..world-1 of one group");
      SKG_CUDA(cudaSetDevice(ctxs[k]->device));
      resolve_pending(ctxs[k]);
      sg[k] = stage_epoch(ctxs[k], *cfg, *tc, epoch, lr);
    }
    static const bool dbg = std::getenv("SKG_SHARD_DEBUG") != nullptr;
    for (int k = 0; k < world; ++k) {
      SKG_CUDA(cudaSetDevice(ctxs[k]->device));
      const auto t0 = std::chrono::steady_clock::now();
      fire_epoch(ctxs[k], sg[k]);
      if (dbg)
        std::fprintf(stderr, "shard group: fired rank %d in %.1f us\n", k,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::exception_ptr first;
    for (int k = 0; k < world; ++k) {  // every rank completes (and syncs) even if one failed
      try {
        SKG_CUDA(cudaSetDevice(ctxs[k]->device));
        complete_epoch(ctxs[k], sg[k], reports + k);
      } catch (...) {
        if (!first) {
          first = std::current_exception();
          failed = k;
        }
      }
    }
    SKG_CUDA(cudaSetDevice(ctxs[0]->device));
    if (first) std::rethrow_exception(first);
  });
}

skg_status skg_shard_export(skg_ctx* ctx, int rank, int world, int64_t batch_size, void* handle) {
  return guard(ctx, [&] {
    if (!handle) throw ConfigError("shard_export: null handle buffer");
    if (ctx->dp) throw ConfigError("context already joined a replicated (NCCL) data-parallel group");
    resolve_pending(ctx);
    shard_alloc(ctx, rank, world, batch_size);
    ShardHandle h{};
    SKG_CUDA(cudaIpcGetMemHandle(&h.mem, ctx->shard->arena));
    h.device = ctx->device;
    h.rank = rank;
    h.world = world;
    h.arena_bytes = ctx->shard->arena_bytes;
    std::memset(handle, 0, SKG_SHARD_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof(h));
  });
}

skg_status skg_shard_import(skg_ctx* ctx, const void* handles) {
  return guard(ctx, [&] {
    ShardState* st = ctx->shard;
    if (!st) throw ConfigError("shard_import: call skg_shard_export first");
    if (st->linked) throw ConfigError("shard_import: peers already linked");
    std::vector<void*> bases(static_cast<size_t>(st->world));
    for (int k = 0; k < st->world; ++k) {
      ShardHandle h;
      std::memcpy(&h, static_cast<const char*>(handles) + static_cast<size_t>(k) * SKG_SHARD_HANDLE_BYTES, sizeof(h));
      if (h.rank != k || h.world != st->world || h.arena_bytes != st->arena_bytes)
        throw ConfigError("shard_import: handle " + std::to_string(k) + " does not belong to this group");
      if (k == st->rank) {
        bases[k] = st->arena;
        continue;
      }
      void* p = nullptr;
      SKG_CUDA(cudaIpcOpenMemHandle(&p, h.mem, cudaIpcMemLazyEnablePeerAccess));
      st->opened[k] = p;
      bases[k] = p;
    }
    shard_link(ctx, bases.data());
  });
}

skg_status skg_shard_release(skg_ctx* ctx) {
  return guard(ctx, [&] { shard_destroy(ctx); });
}

}  // extern "C"
