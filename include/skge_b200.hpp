// skge_b200.hpp — reference-signature C++ shim over the C ABI (skge_b200.h).
//
// A caller of libsparsekge (/root/reference/proj) switches by including this
// header instead of sparsekge/{training,models,embedding}.hpp and linking
// libskge_b200.so. Types keep the reference names and meaning; the Eigen
// matrices become a minimal row-major Matrix / RealVector carrying the subset
// of the Eigen API the reference's callers use (brace and comma
// initialisation, operator(), ==, -, cwiseAbs, maxCoeff). The
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

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <initializer_list>
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
using Complex = std::complex<float>;  // tag type: complex stores hold interleaved (re, im) floats
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
inline const char* model_name(ModelKind m) {  // common.hpp:82-93
  switch (m) {
    case ModelKind::TransE: return "transe";
    case ModelKind::TransR: return "transr";
    case ModelKind::TransH: return "transh";
    case ModelKind::TorusE: return "toruse";
    case ModelKind::DistMult: return "distmult";
    case ModelKind::ComplEx: return "complex";
    case ModelKind::RotatE: return "rotate";
  }
  return "unknown";
}
// common.hpp:74-82, models.hpp:32-38
inline bool is_complex_model(ModelKind m) { return m == ModelKind::ComplEx || m == ModelKind::RotatE; }
inline bool is_multiplicative_model(ModelKind m) {
  return m == ModelKind::DistMult || m == ModelKind::ComplEx || m == ModelKind::RotatE;
}
inline bool higher_is_better(ModelKind m) { return m == ModelKind::DistMult || m == ModelKind::ComplEx; }
inline Real energy_sign(ModelKind m) { return higher_is_better(m) ? Real(-1) : Real(1); }
enum class Engine { Sparse, Dense };

// ---- dense host types: the subset of the Eigen API the reference's callers use
// (row-major matrix, column vector, brace / comma initialisation, cwise helpers).
template <class V>
struct CommaInit {  // Eigen-style `v << a, b, c;`
  V& v;
  Index i;
  CommaInit& operator,(Real x) {
    if (i >= v.size()) throw ShapeError("comma initializer: too many coefficients");
    v.coeff_at(i++) = x;
    return *this;
  }
};

class RealVector : public std::vector<Real> {
 public:
  RealVector() = default;
  explicit RealVector(Index n) : std::vector<Real>(static_cast<size_t>(n), Real(0)) {}
  RealVector(std::initializer_list<Real> v) : std::vector<Real>(v) {}
  Index size() const { return static_cast<Index>(std::vector<Real>::size()); }
  Real& coeff_at(Index i) { return (*this)[static_cast<size_t>(i)]; }
  CommaInit<RealVector> operator<<(Real x) {
    if (size() < 1) throw ShapeError("comma initializer: empty vector");
    (*this)[0] = x;
    return CommaInit<RealVector>{*this, 1};
  }
  void setZero() { std::fill(begin(), end(), Real(0)); }
  RealVector operator-(const RealVector& o) const {
    if (o.size() != size()) throw ShapeError("vector size mismatch");
    RealVector r(size());
    for (Index i = 0; i < size(); ++i) r[i] = (*this)[i] - o[i];
    return r;
  }
  RealVector cwiseAbs() const {
    RealVector r(size());
    for (Index i = 0; i < size(); ++i) r[i] = std::abs((*this)[i]);
    return r;
  }
  Real maxCoeff() const { return empty() ? Real(0) : *std::max_element(begin(), end()); }
  Real sum() const {
    Real s = 0;
    for (Real x : *this) s += x;
    return s;
  }
};
inline RealVector operator*(Real s, const RealVector& v) {
  RealVector r(v.size());
  for (Index i = 0; i < v.size(); ++i) r[i] = s * v[i];
  return r;
}

struct Matrix {  // row-major, one embedding per row
  Index r = 0, c = 0;
  std::vector<Real> a;
  Matrix() = default;
  Matrix(Index rows, Index cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), Real(0)) {}
  Matrix(std::initializer_list<std::initializer_list<Real>> rows_init) {  // RealMatrix{{1, 2}, {3, 4}}
    r = static_cast<Index>(rows_init.size());
    c = r ? static_cast<Index>(rows_init.begin()->size()) : 0;
    for (const auto& row : rows_init) {
      if (static_cast<Index>(row.size()) != c) throw ShapeError("matrix initializer: ragged rows");
      a.insert(a.end(), row.begin(), row.end());
    }
  }
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Constant(Index rows, Index cols, Real v) {
    Matrix m(rows, cols);
    m.setConstant(v);
    return m;
  }
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  Real* data() { return a.data(); }
  const Real* data() const { return a.data(); }
  Real* row(Index i) { return a.data() + i * c; }
  const Real* row(Index i) const { return a.data() + i * c; }
  Real& operator()(Index i, Index j) { return a[static_cast<size_t>(i * c + j)]; }
  Real operator()(Index i, Index j) const { return a[static_cast<size_t>(i * c + j)]; }
  Real& coeff_at(Index k) { return a[static_cast<size_t>(k)]; }
  CommaInit<Matrix> operator<<(Real x) {
    if (size() < 1) throw ShapeError("comma initializer: empty matrix");
    a[0] = x;
    return CommaInit<Matrix>{*this, 1};
  }
  void setZero() { std::fill(a.begin(), a.end(), Real(0)); }
  void setConstant(Real v) { std::fill(a.begin(), a.end(), v); }
  bool operator==(const Matrix& o) const { return r == o.r && c == o.c && a == o.a; }
  bool operator!=(const Matrix& o) const { return !(*this == o); }
  Matrix operator-(const Matrix& o) const { return zip(o, [](Real x, Real y) { return x - y; }); }
  Matrix operator+(const Matrix& o) const { return zip(o, [](Real x, Real y) { return x + y; }); }
  Matrix cwiseAbs() const {
    Matrix m(r, c);
    for (size_t k = 0; k < a.size(); ++k) m.a[k] = std::abs(a[k]);
    return m;
  }
  Real maxCoeff() const { return a.empty() ? Real(0) : *std::max_element(a.begin(), a.end()); }

 private:
  template <class F>
  Matrix zip(const Matrix& o, F f) const {
    if (r != o.r || c != o.c) throw ShapeError("matrix shape mismatch");
    Matrix m(r, c);
    for (size_t k = 0; k < a.size(); ++k) m.a[k] = f(a[k], o.a[k]);
    return m;
  }
};
using RealMatrix = Matrix;
template <class S>
using DenseMatrix = Matrix;  // complex matrices: interleaved (re, im) columns

// ---- incidence and sparse types (incidence.hpp:14-33, sparse.hpp:23-70)
struct TripleBatch {  // incidence.hpp:14-33
  IndexVector heads, relations, tails;
  Index num_entities = 0, num_relations = 0;
  Index size() const { return static_cast<Index>(heads.size()); }
  void validate() const {
    if (heads.size() != relations.size() || heads.size() != tails.size())
      throw ShapeError("triple batch: heads/relations/tails length mismatch");
    for (size_t i = 0; i < heads.size(); ++i) {
      if (heads[i] < 0 || heads[i] >= num_entities || tails[i] < 0 || tails[i] >= num_entities)
        throw ShapeError("triple " + std::to_string(i) + ": entity id out of range");
      if (relations[i] < 0 || relations[i] >= num_relations)
        throw ShapeError("triple " + std::to_string(i) + ": relation id out of range");
    }
  }
};

template <class Scalar = Real>
struct CooMatrix {
  IndexVector rows, cols;
  std::vector<Scalar> vals;
  Index num_rows = 0, num_cols = 0;
  Index nnz() const { return static_cast<Index>(vals.size()); }
};
template <class Scalar = Real>
struct CsrMatrix {
  IndexVector row_ptr, col_idx;
  std::vector<Scalar> vals;
  Index num_rows = 0, num_cols = 0;
  Index nnz() const { return static_cast<Index>(vals.size()); }
};

struct ModelConfig {  // models.hpp:17-30
  ModelKind model = ModelKind::TransE;
  Index dim_entity = 0, dim_relation = 0;
  NormKind norm = NormKind::L2;
  void validate() const {
    if (dim_entity < 1 || dim_relation < 1) throw ConfigError("embedding dimensions must be at least 1");
    if (model != ModelKind::TransR && dim_relation != dim_entity)
      throw ConfigError(std::string(model_name(model)) + " requires dim_relation == dim_entity");
  }
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
template <class S>
using EmbeddingStoreT = EmbeddingStore;
using ComplexEmbeddingStore = EmbeddingStore;

struct Gradients {  // GradientsT, embedding.hpp:36-49
  Matrix entity, relation, proj, normals;
  void set_zero() {
    entity.setZero();
    relation.setZero();
    proj.setZero();
    normals.setZero();
  }
  bool has_proj() const { return proj.size() > 0; }
  bool has_normals() const { return normals.size() > 0; }
};
template <class S>
using GradientsT = Gradients;
inline Gradients make_gradients(const EmbeddingStore& s) {  // embedding.hpp:51-59
  Gradients g;
  g.entity = Matrix(s.entity.rows(), s.entity.cols());
  g.relation = Matrix(s.relation.rows(), s.relation.cols());
  g.proj = Matrix(s.proj.rows(), s.proj.cols());
  g.normals = Matrix(s.normals.rows(), s.normals.cols());
  return g;
}

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
  void validate() const {
    if (batch_size < 1) throw ConfigError("batch_size must be at least 1");
    if (!(margin >= Real(0))) throw ConfigError("margin must be nonnegative");
    if (!(lr >= Real(0)) || !std::isfinite(lr)) throw ConfigError("lr must be finite and >= 0");
    if (epochs < 0) throw ConfigError("epochs must be nonnegative");
    if (scheduler && (scheduler->every_epochs < 1 || !(scheduler->factor > Real(0))))
      throw ConfigError("scheduler needs every_epochs >= 1 and a positive factor");
  }
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
// ScoreBatchT (models.hpp:41-49): the forward result and what the backward needs.
struct ScoreBatch {
  RealVector scores;     // model-native polarity
  CsrMatrix<Real> a;     // the incidence operand (canonical CSR; ComplEx / RotatE: real parts of the markers)
  TripleBatch batch;     // ids, for the backward
  Matrix v;              // pre-norm residual rows (translational models, RotatE: interleaved complex)
  Matrix u;              // head - tail rows (TransH / TransR)
  Matrix delta;          // wrapped residual rows (TorusE)
};
template <class S>
using ScoreBatchT = ScoreBatch;
using ComplexScoreBatch = ScoreBatch;

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
// models.hpp:65-76 (the C ABI checks the same against the uploaded store; the
// batch's own id space is only visible here)
inline void check_config(const ModelConfig& cfg, const EmbeddingStore& store, const TripleBatch& b) {
  cfg.validate();
  const Index w = is_complex_model(cfg.model) ? 2 : 1;
  if (store.dim_entity() != w * cfg.dim_entity || store.dim_relation() != w * cfg.dim_relation)
    throw ConfigError("store dimensions do not match the model config");
  if (store.num_entities() != b.num_entities || store.num_relations() != b.num_relations)
    throw ConfigError("store table sizes do not match the batch id space");
  if (cfg.model == ModelKind::TransR && !store.has_proj())
    throw ConfigError("transr store is missing the projection table");
  if (cfg.model == ModelKind::TransH && !store.has_normals())
    throw ConfigError("transh store is missing the hyperplane normals");
}
// sgd_step / renormalize_entities take no ModelConfig (embedding.hpp:127-132):
// the table set decides the tag the device store is uploaded under.
inline void upload_tables(const EmbeddingStore& s) {
  skg_model_config c{};
  c.model = s.has_normals() ? SKG_TRANSH : (s.has_proj() || s.dim_entity() != s.dim_relation()) ? SKG_TRANSR : SKG_TRANSE;
  c.norm = SKG_L2;
  c.dim_entity = s.dim_entity();
  c.dim_relation = s.dim_relation();
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

// embedding.cpp:129-163 (host-side setup; same libstdc++ stream as the reference).
// init_store<Real> / init_store<Complex> as in the reference (the scalar type is
// implied by the model tag: complex models get interleaved (re, im) columns).
template <class S = Real>
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

// ---- incidence builders (incidence.hpp:38-121), host-side like the reference:
// they only list entries; coo_to_csr canonicalises them on the device.
template <class Scalar = Real>
inline CooMatrix<Scalar> build_ht(const TripleBatch& b) {
  b.validate();
  CooMatrix<Scalar> out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities;
  for (Index i = 0; i < b.size(); ++i) {
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Scalar(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(Scalar(-1));
  }
  return out;
}
template <class Scalar = Real>
inline CooMatrix<Scalar> build_hrt(const TripleBatch& b) {
  b.validate();
  CooMatrix<Scalar> out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities + b.num_relations;
  for (Index i = 0; i < b.size(); ++i) {
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Scalar(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(Scalar(-1));
    out.rows.push_back(i), out.cols.push_back(b.num_entities + b.relations[i]), out.vals.push_back(Scalar(1));
  }
  return out;
}
template <class Scalar = Real>
inline CooMatrix<Scalar> build_multiplicative(const TripleBatch& b, bool conjugate_tail) {
  b.validate();
  CooMatrix<Scalar> out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities + b.num_relations;
  for (Index i = 0; i < b.size(); ++i) {
    if (b.heads[i] == b.tails[i])
      throw DegenerateTripleError("triple " + std::to_string(i) +
                                  ": head == tail is not representable in the multiplicative incidence layout");
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Scalar(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(Scalar(conjugate_tail ? -1 : 1));
    out.rows.push_back(i), out.cols.push_back(b.num_entities + b.relations[i]), out.vals.push_back(Scalar(1));
  }
  return out;
}

// ---- the plus-times sparse layer on device (sparse.hpp:110-306)
inline CsrMatrix<Real> coo_to_csr(const CooMatrix<Real>& m) {
  if (m.rows.size() != m.cols.size() || m.rows.size() != m.vals.size())
    throw ShapeError("coo: rows/cols/vals length mismatch");
  CsrMatrix<Real> out;
  out.num_rows = m.num_rows;
  out.num_cols = m.num_cols;
  out.row_ptr.assign(static_cast<size_t>(m.num_rows) + 1, 0);
  out.col_idx.resize(m.vals.size());
  out.vals.resize(m.vals.size());
  int64_t nnz = 0;
  detail::check(skg_coo_to_csr(detail::ctx(), m.num_rows, m.num_cols, m.nnz(), m.rows.data(), m.cols.data(),
                               m.vals.data(), out.row_ptr.data(), out.col_idx.data(), out.vals.data(), &nnz));
  out.col_idx.resize(static_cast<size_t>(nnz));
  out.vals.resize(static_cast<size_t>(nnz));
  return out;
}
inline CsrMatrix<Real> transpose(const CsrMatrix<Real>& a) {
  CsrMatrix<Real> out;
  out.num_rows = a.num_cols;
  out.num_cols = a.num_rows;
  out.row_ptr.assign(static_cast<size_t>(a.num_cols) + 1, 0);
  out.col_idx.resize(a.vals.size());
  out.vals.resize(a.vals.size());
  detail::check(skg_csr_transpose(detail::ctx(), a.num_rows, a.num_cols, a.row_ptr.data(), a.col_idx.data(),
                                  a.vals.data(), out.row_ptr.data(), out.col_idx.data(), out.vals.data()));
  return out;
}
inline Matrix spmm(const CsrMatrix<Real>& a, const Matrix& x) {
  Matrix out(a.num_rows, x.cols());
  detail::check(skg_spmm(detail::ctx(), a.num_rows, a.num_cols, a.row_ptr.data(), a.col_idx.data(), a.vals.data(),
                         x.rows(), x.cols(), x.data(), out.data()));
  return out;
}
inline void spmm_transpose_add(const CsrMatrix<Real>& a, const Matrix& g, Matrix& out) {
  if (out.rows() != a.num_cols || out.cols() != g.cols()) throw ShapeError("spmm_transpose: sink shape mismatch");
  detail::check(skg_spmm_transpose_add(detail::ctx(), a.num_rows, a.num_cols, a.row_ptr.data(), a.col_idx.data(),
                                       a.vals.data(), g.rows(), g.cols(), g.data(), out.data()));
}
inline Matrix spmm_transpose(const CsrMatrix<Real>& a, const Matrix& g) {
  Matrix out(a.num_cols, g.cols());
  spmm_transpose_add(a, g, out);
  return out;
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
  lg.d_pos = RealVector(pos.size());
  lg.d_neg = RealVector(pos.size());
  detail::check(skg_margin_ranking_loss(detail::ctx(), static_cast<int64_t>(pos.size()), pos.data(), neg.data(),
                                        margin, &lg.loss, lg.d_pos.data(), lg.d_neg.data()));
  return lg;
}

// models.cpp:267-289: scores, the incidence operand and the residual rows the
// backward pass reads (v / delta from the device forward; u = h - t, exact).
inline ScoreBatch score_batch(const ModelConfig& cfg, const EmbeddingStore& store, const TripleBatch& b) {
  detail::check_config(cfg, store, b);
  detail::upload(cfg, store);
  skg_model_config c = detail::cfg(cfg);
  ScoreBatch sb;
  sb.batch = b;
  sb.scores = RealVector(b.size());
  const bool ht = cfg.model == ModelKind::TransH || cfg.model == ModelKind::TransR;
  const Index d = (cfg.model == ModelKind::TransE || cfg.model == ModelKind::TorusE) ? cfg.dim_entity
                  : cfg.model == ModelKind::RotatE                                    ? 2 * cfg.dim_entity
                  : is_multiplicative_model(cfg.model)                                ? 0
                                                                                      : cfg.dim_relation;
  Matrix res(b.size(), d);  // DistMult / ComplEx keep no residual (models.cpp:203-231)
  detail::check(skg_score_batch(detail::ctx(), &c, b.size(), b.heads.data(), b.relations.data(), b.tails.data(),
                                sb.scores.data(), d ? res.data() : nullptr));
  if (cfg.model == ModelKind::TorusE)
    sb.delta = std::move(res);
  else
    sb.v = std::move(res);
  if (ht) {  // u = A_ht E: (+1) h + (-1) t = h - t exactly; self-loops give the empty row 0
    sb.u = Matrix(b.size(), cfg.dim_entity);
    for (Index i = 0; i < b.size(); ++i)
      if (b.heads[i] != b.tails[i])
        for (Index j = 0; j < cfg.dim_entity; ++j)
          sb.u(i, j) = store.entity(b.heads[i], j) - store.entity(b.tails[i], j);
  }
  // the operand the forward used (models.cpp:15, 75, 114, 162, 207, 222, 239)
  const int layout = ht ? SKG_LAYOUT_HT
                     : cfg.model == ModelKind::DistMult                                   ? SKG_LAYOUT_MULT
                     : (cfg.model == ModelKind::ComplEx || cfg.model == ModelKind::RotatE) ? SKG_LAYOUT_MULT_CONJ
                                                                                          : SKG_LAYOUT_HRT;
  sb.a.num_rows = b.size();
  sb.a.num_cols = b.num_entities + (layout == SKG_LAYOUT_HT ? 0 : b.num_relations);
  sb.a.row_ptr.assign(static_cast<size_t>(b.size()) + 1, 0);
  sb.a.col_idx.resize(static_cast<size_t>(3 * b.size()));
  sb.a.vals.resize(static_cast<size_t>(3 * b.size()));
  int64_t nnz = 0;
  detail::check(skg_build_incidence(detail::ctx(), layout, b.size(), b.heads.data(), b.relations.data(),
                                    b.tails.data(), b.num_entities, b.num_relations, sb.a.row_ptr.data(),
                                    sb.a.col_idx.data(), sb.a.vals.data(), &nnz));
  sb.a.col_idx.resize(static_cast<size_t>(nnz));
  sb.a.vals.resize(static_cast<size_t>(nnz));
  return sb;
}

// models.cpp:291-325: accumulates d(sum up_i score_i) into grads
inline void score_backward(const ModelConfig& cfg, const EmbeddingStore& store, const ScoreBatch& sb,
                           const RealVector& upstream, Gradients& grads) {
  const TripleBatch& b = sb.batch;
  detail::check_config(cfg, store, b);
  if (upstream.size() != b.size()) throw ShapeError("score_backward: upstream length does not match the batch");
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
  tc.validate();
  if (pos.size() < 1) throw ConfigError("training requires at least one triple");
  if (neg.corrupted.size() != pos.size()) throw ShapeError("negative set is not aligned with the positive triples");
  detail::upload(mc, store);
  skg_model_config c = detail::cfg(mc);
  skg_train_config t = detail::tcfg(tc);
  skg_epoch_report r{};
  skg_status st = skg_set_triples(detail::ctx(), pos.size(), pos.heads.data(), pos.relations.data(),
                                  pos.tails.data(), pos.num_entities, pos.num_relations);
  if (st == SKG_OK)
    st = skg_set_negatives(detail::ctx(), pos.size(), neg.corrupted.heads.data(), neg.corrupted.tails.data());
  if (st == SKG_OK) st = skg_train_epoch(detail::ctx(), &c, &t, epoch, lr, &r);
  if (st != SKG_OK) {
    // the reference has already updated the caller's store for the batches
    // before a failing one (training.cpp:120-161): hand back the same state
    if (st == SKG_ERR_TRAINING || st == SKG_ERR_DEGENERATE) detail::download(store);
    detail::rethrow(st);
  }
  detail::download(store);
  return EpochReport{r.epoch, static_cast<Real>(r.loss), r.t_forward_s, r.t_backward_s, r.t_step_s};
}

// training.cpp:166-195: negatives once (or per epoch), the lr schedule, optional
// entity renorm, on_epoch after every epoch. The store stays in HBM between
// epochs and is written back to the caller's tables when fit returns (or throws).
inline TrainingRun fit(const ModelConfig& mc, EmbeddingStore& store, const TripleBatch& train, const TrainConfig& tc,
                       Engine /*ignored*/ = Engine::Sparse,
                       const std::function<void(const EpochReport&)>& on_epoch = nullptr) {
  mc.validate();
  tc.validate();
  TrainingRun run;
  if (tc.epochs == 0) return run;
  detail::upload(mc, store);
  detail::check(skg_set_triples(detail::ctx(), train.size(), train.heads.data(), train.relations.data(),
                                train.tails.data(), train.num_entities, train.num_relations));
  skg_model_config c = detail::cfg(mc);
  skg_train_config t = detail::tcfg(tc);
  const bool no_self_loops = is_multiplicative_model(mc.model);
  bool trained = false;
  try {
    detail::check(skg_negative_sample(detail::ctx(), tc.seed, no_self_loops, nullptr, nullptr));
    for (Index e = 0; e < tc.epochs; ++e) {
      if (tc.resample_negatives && e > 0)
        detail::check(skg_negative_sample(detail::ctx(), tc.seed + static_cast<std::uint64_t>(e) * 0x9E3779B9ULL,
                                          no_self_loops, nullptr, nullptr));
      Real lr = tc.lr;
      if (tc.scheduler)
        lr = tc.lr * static_cast<Real>(std::pow(tc.scheduler->factor, double(e / tc.scheduler->every_epochs)));
      skg_epoch_report r{};
      trained = true;
      detail::check(skg_train_epoch(detail::ctx(), &c, &t, e, lr, &r));
      if (tc.renorm_entities) detail::check(skg_renormalize_entities(detail::ctx()));
      const EpochReport rep{r.epoch, static_cast<Real>(r.loss), r.t_forward_s, r.t_backward_s, r.t_step_s};
      run.t_forward_s += rep.t_forward_s;
      run.t_backward_s += rep.t_backward_s;
      run.t_step_s += rep.t_step_s;
      run.epochs.push_back(rep);
      if (on_epoch) on_epoch(rep);
    }
  } catch (...) {
    if (trained) detail::download(store);  // the epochs before the failure stand, as in the reference
    throw;
  }
  detail::download(store);
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

// embedding.cpp:165-190: store -= lr * grads on every table, normals renormalized
inline void sgd_step(EmbeddingStore& store, const Gradients& g, Real lr) {
  auto same = [](const Matrix& x, const Matrix& y) { return x.rows() == y.rows() && x.cols() == y.cols(); };
  if (!same(g.entity, store.entity) || !same(g.relation, store.relation) || !same(g.proj, store.proj) ||
      !same(g.normals, store.normals))
    throw ShapeError("sgd_step: gradient shapes do not match the store");
  detail::upload_tables(store);
  detail::check(skg_sgd_step(detail::ctx(), g.entity.data(), g.relation.data(),
                             g.has_proj() ? g.proj.data() : nullptr, g.has_normals() ? g.normals.data() : nullptr, lr));
  detail::download(store);
}

// embedding.cpp:192-198: entity rows onto the unit sphere, zero rows left alone
inline void renormalize_entities(EmbeddingStore& store) {
  detail::upload_tables(store);
  detail::check(skg_renormalize_entities(detail::ctx()));
  detail::download(store);
}

// kge.cpp:181-247: the `kge train` artifacts (train_log.jsonl, loss.log,
// summary.json) written through the C ABI; pass log.callback() as fit's on_epoch.
class RunLog {
 public:
  explicit RunLog(const std::string& out_dir) {
    if (skg_run_log_open(out_dir.c_str(), &h_) != SKG_OK) throw ParseError(skg_run_log_last_error());
  }
  ~RunLog() { skg_run_log_close(h_); }
  RunLog(const RunLog&) = delete;
  RunLog& operator=(const RunLog&) = delete;
  void epoch(const EpochReport& r) {
    const skg_epoch_report c{r.epoch, static_cast<double>(r.loss), r.t_forward_s, r.t_backward_s, r.t_step_s};
    if (skg_run_log_epoch(h_, &c) != SKG_OK) throw ParseError(skg_run_log_last_error());
  }
  std::function<void(const EpochReport&)> callback() {
    return [this](const EpochReport& r) { epoch(r); };
  }
  void summary(const ModelConfig& mc, const TrainConfig& tc, const TrainingRun& run, const skg_run_summary& info) {
    skg_model_config c = detail::cfg(mc);
    skg_train_config t = detail::tcfg(tc);
    skg_run_summary s = info;
    s.epochs_run = static_cast<int64_t>(run.epochs.size());
    s.final_loss = run.final_loss();
    s.t_forward_s = run.t_forward_s;
    s.t_backward_s = run.t_backward_s;
    s.t_step_s = run.t_step_s;
    if (skg_run_log_summary(h_, &c, &t, &s) != SKG_OK) throw ParseError(skg_run_log_last_error());
  }

 private:
  skg_run_log* h_ = nullptr;
};

}  // namespace skge
