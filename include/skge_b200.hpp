// skge_b200.hpp — reference-signature C++ shim over the C ABI (skge_b200.h).
//
// A caller of libsparsekge (/root/reference/proj) switches by including this
// header instead of sparsekge/{training,models,embedding}.hpp and linking
// libskge_b200.so. Types keep the reference names and meaning; the Eigen
// matrices become a minimal row-major Matrix (row(i) pointer access). The
// functions keep the reference signatures and throw the same exception types
// with the same messages. `Engine` is accepted and ignored: there is one
// device engine, no dispatch (training.hpp:19).
//
// Device residency: every function runs on a per-thread default context
// (device 0, or skge::use_device). EmbeddingStore stays a host object like
// the reference; train_epoch / fit upload it, run on device and download the
// result. Callers that want the store to stay in HBM across epochs use fit()
// (one upload, one download) or the C ABI directly.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "skge_b200.h"

namespace skge {

using Real = float;  // engine computes in fp32 (SPARSEKGE_REAL32 semantics)
using Index = std::int64_t;
using IndexVector = std::vector<Index>;

struct ShapeError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct DegenerateTripleError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct TrainingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

enum class ModelKind : std::uint32_t {
  TransE = 0, TransR = 1, TransH = 2, TorusE = 3, DistMult = 4, ComplEx = 5, RotatE = 6
};
enum class NormKind : std::uint32_t { L1 = 0, L2 = 1 };
// common.hpp:74-82, models.hpp:32-38
inline bool is_complex_model(ModelKind m) { return m == ModelKind::ComplEx || m == ModelKind::RotatE; }
inline bool is_multiplicative_model(ModelKind m) {
  return m == ModelKind::DistMult || m == ModelKind::ComplEx || m == ModelKind::RotatE;
}
inline bool higher_is_better(ModelKind m) { return m == ModelKind::DistMult || m == ModelKind::ComplEx; }
inline Real energy_sign(ModelKind m) { return higher_is_better(m) ? Real(-1) : Real(1); }
enum class Engine { Sparse, Dense };

struct Matrix {  // row-major, one embedding per row
  Index r = 0, c = 0;
  std::vector<Real> a;
  Matrix() = default;
  Matrix(Index rows, Index cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), Real(0)) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  Real* data() { return a.data(); }
  const Real* data() const { return a.data(); }
  Real* row(Index i) { return a.data() + i * c; }
  const Real* row(Index i) const { return a.data() + i * c; }
  Real& operator()(Index i, Index j) { return a[static_cast<size_t>(i * c + j)]; }
  Real operator()(Index i, Index j) const { return a[static_cast<size_t>(i * c + j)]; }
};
using RealMatrix = Matrix;
using RealVector = std::vector<Real>;

struct TripleBatch {  // incidence.hpp:14-33
  IndexVector heads, relations, tails;
  Index num_entities = 0, num_relations = 0;
  Index size() const { return static_cast<Index>(heads.size()); }
};

struct ModelConfig {  // models.hpp:17-30
  ModelKind model = ModelKind::TransE;
  Index dim_entity = 0, dim_relation = 0;
  NormKind norm = NormKind::L2;
};

// embedding.hpp:15-31. ComplEx / RotatE stores (EmbeddingStoreT<Complex> in the
// reference) hold dim interleaved (re, im) pairs per row: 2 * dim columns here,
// the same bytes as a row-major std::complex<float> matrix.
struct EmbeddingStore {
  Matrix entity, relation, proj, normals;
  Index num_entities() const { return entity.rows(); }
  Index num_relations() const { return relation.rows(); }
  Index dim_entity() const { return entity.cols(); }
  Index dim_relation() const { return relation.cols(); }
  bool has_proj() const { return proj.size() > 0; }
  bool has_normals() const { return normals.size() > 0; }
};
using Gradients = EmbeddingStore;

struct StepDecay {
  Index every_epochs = 50;
  Real factor = Real(0.5);
};
struct TrainConfig {  // training.hpp:29-50
  Real lr = Real(4e-4);
  Real margin = Real(0.5);
  Index epochs = 200;
  Index batch_size = 1024;
  std::uint64_t seed = 0;
  std::optional<StepDecay> scheduler;
  bool shuffle = true;
  bool resample_negatives = false;
  bool renorm_entities = false;
};
struct NegativeSet {
  TripleBatch corrupted;
};
struct LossGrad {
  Real loss = 0;
  RealVector d_pos, d_neg;
};
struct EpochReport {
  Index epoch = 0;
  Real loss = 0;
  double t_forward_s = 0, t_backward_s = 0, t_step_s = 0;
};
struct TrainingRun {
  std::vector<EpochReport> epochs;
  double t_forward_s = 0, t_backward_s = 0, t_step_s = 0;
  Real final_loss() const { return epochs.empty() ? Real(0) : epochs.back().loss; }
};
struct ScoreBatch {  // the subset of ScoreBatchT callers read
  RealVector scores;
  Matrix v;  // residual rows (v, or delta for TorusE)
};

namespace detail {
struct Ctx {
  skg_ctx* h = nullptr;
  explicit Ctx(int dev) {
    if (skg_create(dev, &h) != SKG_OK) throw DeviceError(skg_last_error(nullptr));
  }
  ~Ctx() { skg_destroy(h); }
};
inline int& device_ref() {
  static thread_local int d = 0;
  return d;
}
inline skg_ctx* ctx() {
  static thread_local std::unique_ptr<Ctx> c;
  if (!c) c = std::make_unique<Ctx>(device_ref());
  return c->h;
}
[[noreturn]] inline void rethrow(skg_status st) {
  const std::string m = skg_last_error(ctx());
  switch (st) {
    case SKG_ERR_SHAPE: throw ShapeError(m);
    case SKG_ERR_CONFIG: throw ConfigError(m);
    case SKG_ERR_DEGENERATE: throw DegenerateTripleError(m);
    case SKG_ERR_TRAINING: throw TrainingError(m);
    case SKG_ERR_PARSE: throw ParseError(m);
    default: throw DeviceError(m);
  }
}
inline void check(skg_status st) {
  if (st != SKG_OK) rethrow(st);
}
inline skg_model_config cfg(const ModelConfig& m) {
  return skg_model_config{static_cast<uint32_t>(m.model), static_cast<uint32_t>(m.norm), m.dim_entity,
                          m.dim_relation};
}
inline skg_train_config tcfg(const TrainConfig& t) {
  skg_train_config c{};
  c.lr = t.lr;
  c.margin = t.margin;
  c.epochs = t.epochs;
  c.batch_size = t.batch_size;
  c.seed = t.seed;
  c.has_scheduler = t.scheduler.has_value();
  c.decay_every = t.scheduler ? t.scheduler->every_epochs : 50;
  c.decay_factor = t.scheduler ? t.scheduler->factor : Real(0.5);
  c.shuffle = t.shuffle;
  c.resample_negatives = t.resample_negatives;
  c.renorm_entities = t.renorm_entities;
  return c;
}
inline void upload(const ModelConfig& mc, const EmbeddingStore& s) {
  skg_model_config c = cfg(mc);
  const Index w = is_complex_model(mc.model) ? 2 : 1;
  c.dim_entity = s.dim_entity() / w;
  c.dim_relation = s.dim_relation() / w;
  check(skg_store_upload(ctx(), &c, s.num_entities(), s.num_relations(), s.entity.data(), s.relation.data(),
                         s.has_proj() ? s.proj.data() : nullptr, s.has_normals() ? s.normals.data() : nullptr));
}
inline void download(EmbeddingStore& s) {
  check(skg_store_download(ctx(), s.entity.data(), s.relation.data(), s.has_proj() ? s.proj.data() : nullptr,
                           s.has_normals() ? s.normals.data() : nullptr));
}
inline void fill_uniform(Matrix& m, double bound, std::mt19937_64& rng) {  // embedding.cpp:17-30
  std::uniform_real_distribution<double> dist(-bound, bound);
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) m(i, j) = static_cast<Real>(dist(rng));
}
}  // namespace detail

inline void use_device(int device) { detail::device_ref() = device; }

// embedding.cpp:129-163 (host-side setup; same libstdc++ stream as the reference)
inline EmbeddingStore init_store(ModelKind model, Index n_ent, Index n_rel, Index de, Index dr,
                                 std::uint64_t seed) {
  if (de < 1 || dr < 1) throw ConfigError("embedding dimensions must be at least 1");
  if (n_ent < 1 || n_rel < 1) throw ConfigError("store needs at least one entity and one relation");
  std::mt19937_64 rng(seed);
  EmbeddingStore s;
  const Index w = is_complex_model(model) ? 2 : 1;  // re then im per coordinate (embedding.cpp:21-25)
  s.entity = Matrix(n_ent, w * de);
  detail::fill_uniform(s.entity, 6.0 / std::sqrt(static_cast<double>(de)), rng);
  s.relation = Matrix(n_rel, w * dr);
  detail::fill_uniform(s.relation, 6.0 / std::sqrt(static_cast<double>(dr)), rng);
  if (model == ModelKind::TransR) {
    s.proj = Matrix(n_rel, dr * de);
    for (Index r = 0; r < n_rel; ++r)
      for (Index k = 0; k < std::min(dr, de); ++k) s.proj(r, k * de + k) = Real(1);
  }
  if (model == ModelKind::TransH) {
    s.normals = Matrix(n_rel, de);
    detail::fill_uniform(s.normals, 6.0 / std::sqrt(static_cast<double>(de)), rng);
    for (Index r = 0; r < n_rel; ++r) {
      Real n = 0;
      for (Index j = 0; j < de; ++j) n += s.normals(r, j) * s.normals(r, j);
      n = std::sqrt(n);
      if (n > Real(0))
        for (Index j = 0; j < de; ++j) s.normals(r, j) /= n;
      else
        s.normals(r, 0) = Real(1);
    }
  }
  return s;
}

// training.cpp:51-71 (device, bit-exact)
inline NegativeSet negative_sample(const TripleBatch& pos, std::uint64_t seed, bool avoid_self_loops = false) {
  detail::check(skg_set_triples(detail::ctx(), pos.size(), pos.heads.data(), pos.relations.data(),
                                pos.tails.data(), pos.num_entities, pos.num_relations));
  NegativeSet out;
  out.corrupted = pos;
  detail::check(skg_negative_sample(detail::ctx(), seed, avoid_self_loops, out.corrupted.heads.data(),
                                    out.corrupted.tails.data()));
  return out;
}

// training.cpp:73-94
inline LossGrad margin_ranking_loss(const RealVector& pos, const RealVector& neg, Real margin) {
  if (pos.size() != neg.size()) throw ShapeError("margin_ranking_loss: length mismatch");
  LossGrad lg;
  lg.d_pos.resize(pos.size());
  lg.d_neg.resize(pos.size());
  detail::check(skg_margin_ranking_loss(detail::ctx(), static_cast<int64_t>(pos.size()), pos.data(), neg.data(),
                                        margin, &lg.loss, lg.d_pos.data(), lg.d_neg.data()));
  return lg;
}

// models.cpp:267-289 (scores + residual rows)
inline ScoreBatch score_batch(const ModelConfig& cfg, const EmbeddingStore& store, const TripleBatch& b) {
  detail::upload(cfg, store);
  skg_model_config c = detail::cfg(cfg);
  ScoreBatch sb;
  sb.scores.resize(static_cast<size_t>(b.size()));
  const Index d = (cfg.model == ModelKind::TransE || cfg.model == ModelKind::TorusE) ? cfg.dim_entity
                  : cfg.model == ModelKind::RotatE                                    ? 2 * cfg.dim_entity
                  : is_multiplicative_model(cfg.model)                                ? 0
                                                                                      : cfg.dim_relation;
  sb.v = Matrix(b.size(), d);  // DistMult / ComplEx keep no residual (models.cpp:203-231)
  detail::check(skg_score_batch(detail::ctx(), &c, b.size(), b.heads.data(), b.relations.data(), b.tails.data(),
                                sb.scores.data(), d ? sb.v.data() : nullptr));
  return sb;
}

// models.cpp:291-325: accumulates d(sum up_i score_i) into grads
inline void score_backward(const ModelConfig& cfg, const EmbeddingStore& store, const TripleBatch& b,
                           const RealVector& upstream, Gradients& grads) {
  if (static_cast<Index>(upstream.size()) != b.size())
    throw ShapeError("score_backward: upstream length does not match the batch");
  detail::upload(cfg, store);
  skg_model_config c = detail::cfg(cfg);
  detail::check(skg_score_backward(detail::ctx(), &c, b.size(), b.heads.data(), b.relations.data(),
                                   b.tails.data(), upstream.data(), grads.entity.data(), grads.relation.data(),
                                   grads.has_proj() ? grads.proj.data() : nullptr,
                                   grads.has_normals() ? grads.normals.data() : nullptr));
}

// training.cpp:96-164
inline EpochReport train_epoch(const ModelConfig& mc, EmbeddingStore& store, const TripleBatch& pos,
                               const NegativeSet& neg, const TrainConfig& tc, Engine /*ignored*/, Index epoch,
                               Real lr) {
  if (neg.corrupted.size() != pos.size()) throw ShapeError("negative set is not aligned with the positive triples");
  detail::upload(mc, store);
  detail::check(skg_set_triples(detail::ctx(), pos.size(), pos.heads.data(), pos.relations.data(), pos.tails.data(),
                                pos.num_entities, pos.num_relations));
  detail::check(skg_set_negatives(detail::ctx(), pos.size(), neg.corrupted.heads.data(), neg.corrupted.tails.data()));
  skg_model_config c = detail::cfg(mc);
  skg_train_config t = detail::tcfg(tc);
  skg_epoch_report r{};
  detail::check(skg_train_epoch(detail::ctx(), &c, &t, epoch, lr, &r));
  detail::download(store);
  return EpochReport{r.epoch, static_cast<Real>(r.loss), r.t_forward_s, r.t_backward_s, r.t_step_s};
}

// training.cpp:166-195
inline TrainingRun fit(const ModelConfig& mc, EmbeddingStore& store, const TripleBatch& train, const TrainConfig& tc,
                       Engine /*ignored*/ = Engine::Sparse,
                       const std::function<void(const EpochReport&)>& on_epoch = nullptr) {
  TrainingRun run;
  if (tc.epochs == 0) return run;
  detail::upload(mc, store);
  detail::check(skg_set_triples(detail::ctx(), train.size(), train.heads.data(), train.relations.data(),
                                train.tails.data(), train.num_entities, train.num_relations));
  skg_model_config c = detail::cfg(mc);
  skg_train_config t = detail::tcfg(tc);
  std::vector<skg_epoch_report> reps(static_cast<size_t>(tc.epochs));
  detail::check(skg_fit(detail::ctx(), &c, &t, reps.data()));
  detail::download(store);
  for (const auto& r : reps) {
    EpochReport e{r.epoch, static_cast<Real>(r.loss), r.t_forward_s, r.t_backward_s, r.t_step_s};
    run.t_forward_s += e.t_forward_s;
    run.t_backward_s += e.t_backward_s;
    run.t_step_s += e.t_step_s;
    run.epochs.push_back(e);
    if (on_epoch) on_epoch(e);
  }
  return run;
}

// ---- checkpoints (embedding.hpp:134-152, embedding.cpp:200-251) -----------
struct CheckpointHeader {
  ModelKind model = ModelKind::TransE;
  Index num_entities = 0, num_relations = 0, dim_entity = 0, dim_relation = 0;
};

namespace detail {
[[noreturn]] inline void rethrow_ckpt(skg_status st) {
  const std::string msg = skg_checkpoint_last_error();
  if (st == SKG_ERR_CONFIG) throw ConfigError(msg);
  throw ParseError(msg);
}
}  // namespace detail

inline CheckpointHeader peek_checkpoint(const std::string& path) {
  skg_checkpoint_header h{};
  const skg_status st = skg_peek_checkpoint(path.c_str(), &h);
  if (st != SKG_OK) detail::rethrow_ckpt(st);
  return CheckpointHeader{static_cast<ModelKind>(h.model), h.num_entities, h.num_relations, h.dim_entity,
                          h.dim_relation};
}

inline void save_checkpoint(const std::string& path, ModelKind model, const EmbeddingStore& s) {
  const Index w = is_complex_model(model) ? 2 : 1;
  const skg_status st = skg_save_checkpoint(path.c_str(), static_cast<std::uint32_t>(model), s.entity.rows(),
                                            s.relation.rows(), s.entity.cols() / w, s.relation.cols() / w, s.entity.data(),
                                            s.relation.data(), s.proj.size() ? s.proj.data() : nullptr,
                                            s.normals.size() ? s.normals.data() : nullptr);
  if (st != SKG_OK) detail::rethrow_ckpt(st);
}

inline EmbeddingStore load_checkpoint(const std::string& path, ModelKind expected) {
  const CheckpointHeader h = peek_checkpoint(path);
  EmbeddingStore s;
  const Index w = is_complex_model(h.model) ? 2 : 1;
  s.entity = Matrix(h.num_entities, w * h.dim_entity);
  s.relation = Matrix(h.num_relations, w * h.dim_relation);
  if (h.model == ModelKind::TransR) s.proj = Matrix(h.num_relations, h.dim_relation * h.dim_entity);
  if (h.model == ModelKind::TransH) s.normals = Matrix(h.num_relations, h.dim_entity);
  const skg_status st = skg_load_checkpoint(path.c_str(), static_cast<std::uint32_t>(expected), s.entity.data(),
                                            s.relation.data(), s.proj.size() ? s.proj.data() : nullptr,
                                            s.normals.size() ? s.normals.data() : nullptr);
  if (st != SKG_OK) detail::rethrow_ckpt(st);
  return s;
}

// ---- link prediction (eval.hpp / eval.cpp) --------------------------------
enum class Protocol { Raw, Filtered };
enum class Side { Head, Tail };
inline const char* protocol_name(Protocol p) { return p == Protocol::Raw ? "raw" : "filtered"; }

// eval.hpp:25-45: the known-true triples; kept as id lists, hashed on device.
class TripleFilter {
 public:
  TripleFilter(Index n_entities = 0, Index n_relations = 0) : n_(n_entities), r_(n_relations) {}
  void insert(Index h, Index r, Index t) {
    h_.push_back(h);
    r_ids_.push_back(r);
    t_.push_back(t);
  }
  void insert(const TripleBatch& b) {
    for (Index i = 0; i < b.size(); ++i) insert(b.heads[i], b.relations[i], b.tails[i]);
  }
  Index size() const { return static_cast<Index>(h_.size()); }
  const std::vector<Index>& heads() const { return h_; }
  const std::vector<Index>& relations() const { return r_ids_; }
  const std::vector<Index>& tails() const { return t_; }

 private:
  Index n_, r_;
  std::vector<Index> h_, r_ids_, t_;
};

struct EvalReport {  // eval.hpp:50-55
  std::map<Index, double> hits_at;
  double mrr = 0;
  Index n_queries = 0;
  Protocol protocol = Protocol::Raw;
};

namespace detail {
inline std::vector<Index> ranks(const ModelConfig& mc, const EmbeddingStore& store, const TripleBatch& q,
                                const TripleFilter* filter) {
  detail::upload(mc, store);
  skg_model_config c = detail::cfg(mc);
  std::vector<Index> out(2 * static_cast<size_t>(q.size()));
  static const std::vector<Index> none(1, 0);
  detail::check(skg_rank_entities(detail::ctx(), &c, q.size(), q.heads.data(), q.relations.data(), q.tails.data(),
                                  filter ? 1 : 0, filter ? filter->size() : 0,
                                  filter ? filter->heads().data() : none.data(),
                                  filter ? filter->relations().data() : none.data(),
                                  filter ? filter->tails().data() : none.data(), out.data()));
  return out;
}
}  // namespace detail

// eval.cpp:16-63
inline Index rank_entity(const ModelConfig& mc, const EmbeddingStore& store, Index h, Index r, Index t, Side side,
                         const TripleFilter* filter) {
  TripleBatch q;
  q.heads = {h};
  q.relations = {r};
  q.tails = {t};
  q.num_entities = store.entity.rows();
  q.num_relations = store.relation.rows();
  const auto rk = detail::ranks(mc, store, q, filter);
  return side == Side::Tail ? rk[0] : rk[1];
}

// eval.cpp:5-12 + 65-96 (filter over every split; MRR / Hits@k accumulated in
// the reference's order: tail then head per test triple)
inline EvalReport evaluate(const ModelConfig& mc, const EmbeddingStore& store, const TripleBatch& train,
                           const TripleBatch& valid, const TripleBatch& test, Protocol protocol,
                           const std::vector<Index>& ks = {1, 3, 10}) {
  if (test.size() < 1) throw ConfigError("evaluation needs a nonempty test split");
  TripleFilter filter(store.entity.rows(), store.relation.rows());
  if (protocol == Protocol::Filtered) {
    filter.insert(train);
    filter.insert(valid);
    filter.insert(test);
  }
  const auto rk = detail::ranks(mc, store, test, protocol == Protocol::Filtered ? &filter : nullptr);
  EvalReport rep;
  rep.protocol = protocol;
  std::vector<Index> hit_counts(ks.size(), 0);
  double mrr_sum = 0;
  for (size_t i = 0; i < rk.size(); ++i) {
    mrr_sum += 1.0 / double(rk[i]);
    for (size_t k = 0; k < ks.size(); ++k)
      if (rk[i] <= ks[k]) ++hit_counts[k];
    ++rep.n_queries;
  }
  for (size_t k = 0; k < ks.size(); ++k) rep.hits_at[ks[k]] = double(hit_counts[k]) / double(rep.n_queries);
  rep.mrr = mrr_sum / double(rep.n_queries);
  return rep;
}

// embedding.cpp:165-190
inline void sgd_step(EmbeddingStore& store, const Gradients& g, Real lr, const ModelConfig& mc) {
  detail::upload(mc, store);
  detail::check(skg_sgd_step(detail::ctx(), g.entity.data(), g.relation.data(),
                             g.has_proj() ? g.proj.data() : nullptr, g.has_normals() ? g.normals.data() : nullptr, lr));
  detail::download(store);
}

}  // namespace skge
