// TEST INFRASTRUCTURE ONLY — see skge_oracle.hpp for scope and pinning.
// Every function cites the reference file:line (under /root/reference/proj)
// whose arithmetic and ordering it restates.
#include "skge_oracle.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <numeric>
#include <random>
#include <unordered_set>

namespace orc {

namespace {
int g_threads = 1;
}
void set_num_threads(int n) { g_threads = n < 1 ? 1 : n; }
int num_threads() { return g_threads; }

const char* model_name(ModelKind m) {
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

// ---------------------------------------------------------------- sparse.hpp

void CooMatrix::validate() const {  // sparse.hpp:30-37
  if (rows.size() != cols.size() || rows.size() != vals.size())
    throw ShapeError("coo: rows/cols/vals length mismatch");
  for (size_t i = 0; i < rows.size(); ++i)
    if (rows[i] < 0 || rows[i] >= num_rows || cols[i] < 0 || cols[i] >= num_cols)
      throw ShapeError("coo: entry " + std::to_string(i) + " outside declared shape");
}

void CsrMatrix::validate() const {  // sparse.hpp:52-68
  if (static_cast<Index>(row_ptr.size()) != num_rows + 1)
    throw ShapeError("csr: row_ptr length != num_rows + 1");
  if (row_ptr.front() != 0 || row_ptr.back() != nnz()) throw ShapeError("csr: row_ptr endpoints");
  if (col_idx.size() != vals.size()) throw ShapeError("csr: col/val length mismatch");
  for (Index r = 0; r < num_rows; ++r) {
    if (row_ptr[r] > row_ptr[r + 1]) throw ShapeError("csr: row_ptr decreasing");
    for (Index p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= num_cols) throw ShapeError("csr: column out of range");
      if (p > row_ptr[r] && col_idx[p] <= col_idx[p - 1])
        throw ShapeError("csr: columns not strictly increasing within row");
    }
  }
}

// sparse.hpp:110-161: bucket by row (stable), sort each row by column, merge
// duplicates left to right, drop exact zeros.
CsrMatrix coo_to_csr(const CooMatrix& m) {
  m.validate();
  const Index nnz = m.nnz();
  CsrMatrix out;
  out.num_rows = m.num_rows;
  out.num_cols = m.num_cols;
  out.row_ptr.assign(static_cast<size_t>(m.num_rows) + 1, 0);
  IndexVector start(static_cast<size_t>(m.num_rows) + 1, 0);
  for (Index i = 0; i < nnz; ++i) ++start[m.rows[i] + 1];
  for (Index r = 0; r < m.num_rows; ++r) start[r + 1] += start[r];
  IndexVector cols(static_cast<size_t>(nnz));
  std::vector<Real> vals(static_cast<size_t>(nnz));
  {
    IndexVector cursor(start.begin(), start.end() - 1);
    for (Index i = 0; i < nnz; ++i) {
      const Index p = cursor[m.rows[i]]++;
      cols[p] = m.cols[i];
      vals[p] = m.vals[i];
    }
  }
  IndexVector perm;
  for (Index r = 0; r < m.num_rows; ++r) {
    const Index lo = start[r], n = start[r + 1] - lo;
    perm.resize(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), lo);
    std::sort(perm.begin(), perm.end(), [&](Index a, Index b) { return cols[a] < cols[b]; });
    for (Index p = 0; p < n;) {
      const Index c = cols[perm[p]];
      Real v = vals[perm[p]];
      for (++p; p < n && cols[perm[p]] == c; ++p) v += vals[perm[p]];
      if (v != Real(0)) {
        out.col_idx.push_back(c);
        out.vals.push_back(v);
      }
    }
    out.row_ptr[r + 1] = static_cast<Index>(out.col_idx.size());
  }
  return out;
}

// sparse.hpp:164-183: counting sort over columns, rows visited ascending.
CsrMatrix transpose(const CsrMatrix& a) {
  CsrMatrix out;
  out.num_rows = a.num_cols;
  out.num_cols = a.num_rows;
  out.row_ptr.assign(static_cast<size_t>(a.num_cols) + 1, 0);
  for (Index c : a.col_idx) ++out.row_ptr[c + 1];
  for (Index c = 0; c < a.num_cols; ++c) out.row_ptr[c + 1] += out.row_ptr[c];
  out.col_idx.resize(static_cast<size_t>(a.nnz()));
  out.vals.resize(static_cast<size_t>(a.nnz()));
  IndexVector cursor(out.row_ptr.begin(), out.row_ptr.end() - 1);
  for (Index r = 0; r < a.num_rows; ++r)
    for (Index p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p) {
      const Index q = cursor[a.col_idx[p]]++;
      out.col_idx[q] = r;
      out.vals[q] = a.vals[p];
    }
  return out;
}

namespace {

// Row source over [entity; relation] (embedding.hpp:63-83).
struct Stacked {
  const Mat* top;
  const Mat* bottom;
  Index rows() const { return top->rows + (bottom ? bottom->rows : 0); }
  Index cols() const { return top->cols; }
  const Real* row(Index k) const { return k < top->rows ? top->row(k) : bottom->row(k - top->rows); }
};
struct StackedMut {
  Mat* top;
  Mat* bottom;
  Real* row(Index k) { return k < top->rows ? top->row(k) : bottom->row(k - top->rows); }
};

// sparse.hpp:211-237: short rows combine terms left to right in stored order;
// longer rows zero then accumulate. coeff * x is formed first, then added.
void spmm_row(const CsrMatrix& a, const Stacked& x, Index i, Real* out) {
  const Index d = x.cols();
  const Index b = a.row_ptr[i], n = a.row_ptr[i + 1] - b;
  if (n == 0) {
    for (Index j = 0; j < d; ++j) out[j] = Real(0);
    return;
  }
  if (n <= 3) {
    const Real* r0 = x.row(a.col_idx[b]);
    for (Index j = 0; j < d; ++j) {
      Real acc = a.vals[b] * r0[j];
      for (Index p = 1; p < n; ++p) {
        const Real t = a.vals[b + p] * x.row(a.col_idx[b + p])[j];
        acc = acc + t;
      }
      out[j] = acc;
    }
    return;
  }
  for (Index j = 0; j < d; ++j) out[j] = Real(0);
  for (Index p = b; p < b + n; ++p) {
    const Real* xr = x.row(a.col_idx[p]);
    for (Index j = 0; j < d; ++j) {
      const Real t = a.vals[p] * xr[j];
      out[j] += t;
    }
  }
}

// Lazy rows for the transposed SpMM (models.cpp:37-60); `row_into` writes
// g_i, the value each coefficient is multiplied with.
struct DenseRows {
  const Mat& g;
  Index rows() const { return g.rows; }
  void row_into(Index i, Real* out) const {
    for (Index j = 0; j < g.cols; ++j) out[j] = g.row(i)[j];
  }
};
struct L2DirectionRows {  // models.cpp:37-47: inv recomputed on every access
  const Mat& v;
  const std::vector<Real>& up;
  Index rows() const { return v.rows; }
  void row_into(Index i, Real* out) const {
    const Real inv = up[i] / std::sqrt(squared_sum(v.row(i), v.cols) + kNormEps);
    for (Index j = 0; j < v.cols; ++j) out[j] = v.row(i)[j] * inv;
  }
};
struct L1DirectionRows {  // models.cpp:49-60
  const Mat& v;
  const std::vector<Real>& up;
  Index rows() const { return v.rows; }
  void row_into(Index i, Real* out) const {
    const Real w = up[i];
    for (Index j = 0; j < v.cols; ++j) {
      const Real x = v.row(i)[j];
      out[j] = x > Real(0) ? w : (x < Real(0) ? -w : Real(0));
    }
  }
};

// sparse.hpp:273-306: out_k += sum_i a_ik g_i, each output row accumulated in
// ascending source-row order ((row + a0 g0) + a1 g1) + ...
template <class GSrc, class Sink>
void spmm_transpose_add_impl(const CsrMatrix& a, const GSrc& g, Index d, Sink&& out) {
  if (a.num_rows != g.rows()) throw ShapeError("spmm_transpose: row count mismatch");
  const CsrMatrix at = transpose(a);
  parallel_for(at.num_rows, [&](Index lo, Index hi) {
    std::vector<Real> gr(static_cast<size_t>(d));
    for (Index k = lo; k < hi; ++k) {
      Real* row = out.row(k);
      for (Index p = at.row_ptr[k]; p < at.row_ptr[k + 1]; ++p) {
        g.row_into(at.col_idx[p], gr.data());
        const Real c = at.vals[p];
        for (Index j = 0; j < d; ++j) {
          const Real t = c * gr[j];
          row[j] = row[j] + t;
        }
      }
    }
  });
}

}  // namespace

Mat spmm(const CsrMatrix& a, const Mat& x) {  // sparse.hpp:242-266 (plus-times)
  if (a.num_cols != x.rows)
    throw ShapeError("spmm: inner dimensions " + std::to_string(a.num_cols) + " vs " +
                     std::to_string(x.rows));
  Mat out(a.num_rows, x.cols);
  Stacked xs{&x, nullptr};
  parallel_for(a.num_rows, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) spmm_row(a, xs, i, out.row(i));
  });
  return out;
}

void spmm_transpose_add(const CsrMatrix& a, const Mat& g, Mat& out) {
  spmm_transpose_add_impl(a, DenseRows{g}, g.cols, out);
}

// -------------------------------------------------------------- incidence.hpp

void TripleBatch::validate() const {  // incidence.hpp:23-32
  if (heads.size() != relations.size() || heads.size() != tails.size())
    throw ShapeError("triple batch: heads/relations/tails length mismatch");
  for (size_t i = 0; i < heads.size(); ++i) {
    if (heads[i] < 0 || heads[i] >= num_entities || tails[i] < 0 || tails[i] >= num_entities)
      throw ShapeError("triple " + std::to_string(i) + ": entity id out of range");
    if (relations[i] < 0 || relations[i] >= num_relations)
      throw ShapeError("triple " + std::to_string(i) + ": relation id out of range");
  }
}

CooMatrix build_ht(const TripleBatch& b) {  // incidence.hpp:38-57
  b.validate();
  CooMatrix out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities;
  for (Index i = 0; i < b.size(); ++i) {
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Real(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(Real(-1));
  }
  return out;
}

CooMatrix build_hrt(const TripleBatch& b) {  // incidence.hpp:62-85
  b.validate();
  CooMatrix out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities + b.num_relations;
  for (Index i = 0; i < b.size(); ++i) {
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Real(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(Real(-1));
    out.rows.push_back(i), out.cols.push_back(b.num_entities + b.relations[i]),
        out.vals.push_back(Real(1));
  }
  return out;
}

// incidence.hpp:93-121: +1 at head and relation, the tail +1 or the -1
// conjugate marker; head == tail is not representable.
CooMatrix build_multiplicative(const TripleBatch& b, bool conjugate_tail) {
  b.validate();
  CooMatrix out;
  out.num_rows = b.size();
  out.num_cols = b.num_entities + b.num_relations;
  const Real tail_marker = conjugate_tail ? Real(-1) : Real(1);
  for (Index i = 0; i < b.size(); ++i) {
    if (b.heads[i] == b.tails[i])
      throw DegenerateTripleError("triple " + std::to_string(i) +
                                  ": head == tail is not representable in the "
                                  "multiplicative incidence layout");
    out.rows.push_back(i), out.cols.push_back(b.heads[i]), out.vals.push_back(Real(1));
    out.rows.push_back(i), out.cols.push_back(b.tails[i]), out.vals.push_back(tail_marker);
    out.rows.push_back(i), out.cols.push_back(b.num_entities + b.relations[i]),
        out.vals.push_back(Real(1));
  }
  return out;
}

// ------------------------------------------------------------------ norms.hpp

Real squared_sum(const Real* v, Index n) {  // norms.hpp:19-36
  if (n < 8) {
    Real s = 0;
    for (Index j = 0; j < n; ++j) s += v[j] * v[j];
    return s;
  }
  Real s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  Index j = 0;
  for (; j + 4 <= n; j += 4) {
    s0 += v[j] * v[j];
    s1 += v[j + 1] * v[j + 1];
    s2 += v[j + 2] * v[j + 2];
    s3 += v[j + 3] * v[j + 3];
  }
  Real s = (s0 + s1) + (s2 + s3);
  for (; j < n; ++j) s += v[j] * v[j];
  return s;
}

Real abs_sum(const Real* v, Index n) {  // norms.hpp:38-55
  if (n < 8) {
    Real s = 0;
    for (Index j = 0; j < n; ++j) s += std::abs(v[j]);
    return s;
  }
  Real s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  Index j = 0;
  for (; j + 4 <= n; j += 4) {
    s0 += std::abs(v[j]);
    s1 += std::abs(v[j + 1]);
    s2 += std::abs(v[j + 2]);
    s3 += std::abs(v[j + 3]);
  }
  Real s = (s0 + s1) + (s2 + s3);
  for (; j < n; ++j) s += std::abs(v[j]);
  return s;
}

Real score_norm(const Real* v, Index n, NormKind norm) {  // norms.hpp:57-62
  if (norm == NormKind::L1) return abs_sum(v, n);
  return std::sqrt(squared_sum(v, n));
}

void norm_direction(const Real* v, Index n, NormKind norm, Real weight, Real* out) {  // :66-74
  if (norm == NormKind::L1) {
    for (Index j = 0; j < n; ++j) out[j] = v[j] > Real(0) ? weight : (v[j] < Real(0) ? -weight : Real(0));
    return;
  }
  const Real inv = weight / std::sqrt(squared_sum(v, n) + kNormEps);
  for (Index j = 0; j < n; ++j) out[j] = v[j] * inv;
}

Real torus_wrap(Real x) {  // norms.hpp:96-100
  Real d = x - std::nearbyint(x);
  if (d >= Real(0.5)) d -= Real(1);
  return d;
}

Real torus_score_from_delta(const Real* delta, Index n, NormKind norm) {  // norms.hpp:107-115
  Real s = 0;
  if (norm == NormKind::L1) {
    for (Index j = 0; j < n; ++j) s += std::abs(delta[j]);
    return s;
  }
  for (Index j = 0; j < n; ++j) s += delta[j] * delta[j];
  return s;
}

void torus_direction(const Real* delta, Index n, NormKind norm, Real weight, Real* out) {  // :119-126
  if (norm == NormKind::L1) {
    for (Index j = 0; j < n; ++j)
      out[j] = delta[j] > Real(0) ? weight : (delta[j] < Real(0) ? -weight : Real(0));
    return;
  }
  for (Index j = 0; j < n; ++j) out[j] = weight * Real(2) * delta[j];
}

namespace {
// Stand-in for Eigen's dot redux (models.hpp:101, 109-110): left to right.
Real dot(const Real* a, const Real* b, Index n) {
  Real s = 0;
  for (Index j = 0; j < n; ++j) s += a[j] * b[j];
  return s;
}
// Stand-in for Eigen row.norm() (embedding.cpp:309, 338, 349).
Real row_norm(const Real* a, Index n) { return std::sqrt(dot(a, a, n)); }
}  // namespace

// ----------------------------------------------------------------- models.cpp

void ModelConfig::validate() const {  // models.hpp:23-29
  if (dim_entity < 1 || dim_relation < 1) throw ConfigError("embedding dimensions must be at least 1");
  if (model != ModelKind::TransR && dim_relation != dim_entity)
    throw ConfigError(std::string(model_name(model)) + " requires dim_relation == dim_entity");
}

Gradients make_gradients(const Store& s) {  // embedding.hpp:51-59
  Gradients g;
  g.entity = Mat(s.entity.rows, s.entity.cols);
  g.relation = Mat(s.relation.rows, s.relation.cols);
  g.proj = Mat(s.proj.rows, s.proj.cols);
  g.normals = Mat(s.normals.rows, s.normals.cols);
  return g;
}

namespace {

void check_config(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.hpp:65-76
  cfg.validate();
  if (store.dim_entity() != cfg.width_entity() || store.dim_relation() != cfg.width_relation())
    throw ConfigError("store dimensions do not match the model config");
  if (store.num_entities() != b.num_entities || store.num_relations() != b.num_relations)
    throw ConfigError("store table sizes do not match the batch id space");
  if (cfg.model == ModelKind::TransR && !store.has_proj())
    throw ConfigError("transr store is missing the projection table");
  if (cfg.model == ModelKind::TransH && !store.has_normals())
    throw ConfigError("transh store is missing the hyperplane normals");
}

ScoreBatch transe_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:11-30
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_hrt(b));
  const Index m = b.size(), d = cfg.dim_entity;
  const Stacked x{&store.entity, &store.relation};
  sb.v = Mat(m, d);
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      spmm_row(sb.a, x, i, sb.v.row(i));
      sb.scores[i] = score_norm(sb.v.row(i), d, cfg.norm);
    }
  });
  return sb;
}

void transe_backward(const ModelConfig& cfg, const ScoreBatch& sb, const std::vector<Real>& up,
                     Gradients& g) {  // models.cpp:62-69
  StackedMut sink{&g.entity, &g.relation};
  if (cfg.norm == NormKind::L1)
    spmm_transpose_add_impl(sb.a, L1DirectionRows{sb.v, up}, sb.v.cols, sink);
  else
    spmm_transpose_add_impl(sb.a, L2DirectionRows{sb.v, up}, sb.v.cols, sink);
}

ScoreBatch toruse_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:71-92
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_hrt(b));
  const Index m = b.size(), d = cfg.dim_entity;
  const Stacked x{&store.entity, &store.relation};
  sb.delta = Mat(m, d);
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    std::vector<Real> raw(static_cast<size_t>(d));
    for (Index i = lo; i < hi; ++i) {
      spmm_row(sb.a, x, i, raw.data());
      for (Index j = 0; j < d; ++j) sb.delta.row(i)[j] = torus_wrap(raw[j]);
      sb.scores[i] = torus_score_from_delta(sb.delta.row(i), d, cfg.norm);
    }
  });
  return sb;
}

void toruse_backward(const ModelConfig& cfg, const ScoreBatch& sb, const std::vector<Real>& up,
                     Gradients& g) {  // models.cpp:94-105
  const Index m = sb.batch.size(), d = cfg.dim_entity;
  Mat dmat(m, d);
  parallel_for(m, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) torus_direction(sb.delta.row(i), d, cfg.norm, up[i], dmat.row(i));
  });
  StackedMut sink{&g.entity, &g.relation};
  spmm_transpose_add_impl(sb.a, DenseRows{dmat}, d, sink);
}

ScoreBatch transr_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:110-134
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_ht(b));
  sb.u = spmm(sb.a, store.entity);
  const Index m = b.size(), de = cfg.dim_entity, dr = cfg.dim_relation;
  sb.v = Mat(m, dr);
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      const Index r = b.relations[i];
      const Real* u = sb.u.row(i);
      const Real* mr = store.proj.row(r);  // d_r x d_e row-major (models.cpp:127)
      Real* v = sb.v.row(i);
      for (Index n = 0; n < dr; ++n) v[n] = dot(mr + n * de, u, de);  // project_forward, models.hpp:82-86
      for (Index n = 0; n < dr; ++n) v[n] += store.relation.row(r)[n];
      sb.scores[i] = score_norm(v, dr, cfg.norm);
    }
  });
  return sb;
}

void transr_backward(const ModelConfig& cfg, const Store& store, const ScoreBatch& sb,
                     const std::vector<Real>& up, Gradients& g) {  // models.cpp:136-156
  const Index m = sb.batch.size(), de = cfg.dim_entity, dr = cfg.dim_relation;
  Mat dumat(m, de);
  std::vector<Real> dz(static_cast<size_t>(dr));
  for (Index i = 0; i < m; ++i) {  // sequential: relation rows collide across triples
    norm_direction(sb.v.row(i), dr, cfg.norm, up[i], dz.data());
    const Index r = sb.batch.relations[i];
    Real* gr = g.relation.row(r);
    for (Index n = 0; n < dr; ++n) gr[n] += dz[n];
    const Real* u = sb.u.row(i);
    Real* gm = g.proj.row(r);
    for (Index n = 0; n < dr; ++n)  // project_back_mr, models.hpp:94-96
      for (Index k = 0; k < de; ++k) gm[n * de + k] += dz[n] * u[k];
    const Real* mr = store.proj.row(r);
    Real* du = dumat.row(i);
    for (Index k = 0; k < de; ++k) {  // project_back_u, models.hpp:89-91
      Real s = 0;
      for (Index n = 0; n < dr; ++n) s += dz[n] * mr[n * de + k];
      du[k] = s;
    }
  }
  spmm_transpose_add_impl(sb.a, DenseRows{dumat}, de, g.entity);
}

ScoreBatch transh_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:158-181
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_ht(b));
  sb.u = spmm(sb.a, store.entity);
  const Index m = b.size(), d = cfg.dim_entity;
  sb.v = Mat(m, d);
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      const Index r = b.relations[i];
      const Real* u = sb.u.row(i);
      const Real* rel = store.relation.row(r);
      const Real* w = store.normals.row(r);
      Real* v = sb.v.row(i);
      const Real wu = dot(w, u, d);  // hyperplane_forward, models.hpp:99-103
      for (Index j = 0; j < d; ++j) {
        const Real a = u[j] + rel[j];
        const Real c = wu * w[j];
        v[j] = a - c;
      }
      sb.scores[i] = score_norm(v, d, cfg.norm);
    }
  });
  return sb;
}

void transh_backward(const ModelConfig& cfg, const Store& store, const ScoreBatch& sb,
                     const std::vector<Real>& up, Gradients& g) {  // models.cpp:183-199
  const Index m = sb.batch.size(), d = cfg.dim_entity;
  Mat dumat(m, d);
  std::vector<Real> dz(static_cast<size_t>(d));
  for (Index i = 0; i < m; ++i) {
    norm_direction(sb.v.row(i), d, cfg.norm, up[i], dz.data());
    const Index r = sb.batch.relations[i];
    Real* gr = g.relation.row(r);
    for (Index j = 0; j < d; ++j) gr[j] += dz[j];
    const Real* u = sb.u.row(i);
    const Real* w = store.normals.row(r);
    Real* gw = g.normals.row(r);
    const Real dzw = dot(dz.data(), w, d);  // hyperplane_backward, models.hpp:106-113
    const Real wu = dot(w, u, d);
    Real* du = dumat.row(i);
    for (Index j = 0; j < d; ++j) {
      const Real c = dzw * w[j];
      du[j] = dz[j] - c;
      const Real a = dzw * u[j];
      const Real e = wu * dz[j];
      gw[j] -= a + e;
    }
  }
  spmm_transpose_add_impl(sb.a, DenseRows{dumat}, d, g.entity);
}

}  // namespace

// ---- multiplicative family (models.cpp:201-263) ----
//
// Complex arithmetic is restated on interleaved (re, im) Real pairs with the
// operation order of std::complex / Eigen's packet product (no FMA):
// (a * b).re = a.re*b.re - a.im*b.im, (a * b).im = a.re*b.im + a.im*b.re.
// semiring_detail::selects (sparse.hpp:72-77): a marker with positive real
// part selects the operand, a negative one its conjugate.

namespace {

inline bool selects(Real marker) { return marker > Real(0); }

// acc *= x (or conj(x)) elementwise over d coordinates (TimesTimes, sparse.hpp:94-106)
void times_row(Real* acc, const Real* x, Index d, bool cplx, bool conj) {
  if (!cplx) {
    for (Index j = 0; j < d; ++j) acc[j] = acc[j] * x[j];
    return;
  }
  for (Index j = 0; j < d; ++j) {
    const Real ar = acc[2 * j], ai = acc[2 * j + 1];
    const Real br = x[2 * j], bi = conj ? -x[2 * j + 1] : x[2 * j + 1];
    const Real t0 = ar * br, t1 = ai * bi, t2 = ar * bi, t3 = ai * br;
    acc[2 * j] = t0 - t1;
    acc[2 * j + 1] = t2 + t3;
  }
}

void set_identity(Real* acc, Index d, bool cplx) {
  for (Index j = 0; j < d; ++j) {
    if (cplx) {
      acc[2 * j] = Real(1);
      acc[2 * j + 1] = Real(0);
    } else {
      acc[j] = Real(1);
    }
  }
}

// spmm<TimesTimes> row (sparse.hpp:254-262): identity, then every entry in stored order.
void times_spmm_row(const CsrMatrix& a, const Stacked& x, Index i, Index d, bool cplx, Real* out) {
  set_identity(out, d, cplx);
  for (Index p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p)
    times_row(out, x.row(a.col_idx[p]), d, cplx, !selects(a.vals[p]));
}

Real sum_row(const Real* v, Index n) {  // norms.hpp:76-80
  Real s = 0;
  for (Index j = 0; j < n; ++j) s += v[j];
  return s;
}
Real sum_real(const Real* v, Index n) {  // norms.hpp:82-86 (v interleaved)
  Real s = 0;
  for (Index j = 0; j < n; ++j) s += v[2 * j];
  return s;
}
Real cabs(Real re, Real im) { return std::abs(std::complex<Real>(re, im)); }
Real sum_abs(const Real* v, Index n) {  // norms.hpp:88-92
  Real s = 0;
  for (Index j = 0; j < n; ++j) s += cabs(v[2 * j], v[2 * j + 1]);
  return s;
}

ScoreBatch product_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:203-231
  const bool cplx = cfg.model == ModelKind::ComplEx;
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_multiplicative(b, cplx));
  const Index m = b.size(), d = cfg.dim_entity;
  const Stacked x{&store.entity, &store.relation};
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    std::vector<Real> prow(static_cast<size_t>(cfg.width_entity()));
    for (Index i = lo; i < hi; ++i) {
      times_spmm_row(sb.a, x, i, d, cplx, prow.data());
      sb.scores[i] = cplx ? sum_real(prow.data(), d) : sum_row(prow.data(), d);
    }
  });
  return sb;
}

ScoreBatch rotate_forward(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:233-248
  ScoreBatch sb;
  sb.batch = b;
  sb.a = coo_to_csr(build_multiplicative(b, true));
  const Index m = b.size(), d = cfg.dim_entity;
  const Stacked x{&store.entity, &store.relation};
  sb.v = Mat(m, 2 * d);
  sb.scores.assign(static_cast<size_t>(m), Real(0));
  parallel_for(m, [&](Index lo, Index hi) {
    std::vector<Real> prod(static_cast<size_t>(2 * d)), sub(static_cast<size_t>(2 * d));
    for (Index i = lo; i < hi; ++i) {  // spmm_mulsub, sparse.hpp:345-365
      set_identity(prod.data(), d, true);
      for (Index j = 0; j < 2 * d; ++j) sub[j] = Real(0);
      for (Index p = sb.a.row_ptr[i]; p < sb.a.row_ptr[i + 1]; ++p) {
        const Real* xr = x.row(sb.a.col_idx[p]);
        if (selects(sb.a.vals[p])) {
          times_row(prod.data(), xr, d, true, false);
        } else {
          for (Index j = 0; j < 2 * d; ++j) sub[j] = sub[j] + xr[j];
        }
      }
      Real* q = sb.v.row(i);
      for (Index j = 0; j < 2 * d; ++j) q[j] = prod[j] - sub[j];
      sb.scores[i] = sum_abs(q, d);
    }
  });
  return sb;
}

// spmm_product_grad_add (sparse.hpp:315-339): entry p of row i receives
// upstream_i * (product of the row's other operands), conjugated when p selects.
// Sequential over rows and entries (output rows collide across triples).
void product_backward(const ModelConfig& cfg, const Store& store, const ScoreBatch& sb,
                      const std::vector<Real>& up, Gradients& g) {
  const bool cplx = cfg.model == ModelKind::ComplEx;
  const Index d = cfg.dim_entity, w = cfg.width_entity();
  const Stacked x{&store.entity, &store.relation};
  StackedMut sink{&g.entity, &g.relation};
  const CsrMatrix& a = sb.a;
  std::vector<Real> others(static_cast<size_t>(w));
  for (Index i = 0; i < a.num_rows; ++i) {
    const Index lo = a.row_ptr[i], hi = a.row_ptr[i + 1];
    for (Index p = lo; p < hi; ++p) {
      set_identity(others.data(), d, cplx);
      for (Index q = lo; q < hi; ++q) {
        if (q == p) continue;
        times_row(others.data(), x.row(a.col_idx[q]), d, cplx, !selects(a.vals[q]));
      }
      Real* out = sink.row(a.col_idx[p]);
      const bool conj = cplx && selects(a.vals[p]);
      for (Index j = 0; j < w; ++j) {
        const Real o = (conj && (j & 1)) ? -others[j] : others[j];
        const Real t = up[i] * o;
        out[j] = out[j] + t;
      }
    }
  }
}

// modulus_direction (norms.hpp:129-135) + spmm_mulsub_grad_add (sparse.hpp:367-391)
void rotate_backward(const ModelConfig& cfg, const Store& store, const ScoreBatch& sb,
                     const std::vector<Real>& up, Gradients& g) {
  const Index d = cfg.dim_entity, m = sb.batch.size();
  Mat dq(m, 2 * d);
  parallel_for(m, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      const Real* q = sb.v.row(i);
      Real* o = dq.row(i);
      for (Index j = 0; j < d; ++j) {
        const Real re = q[2 * j], im = q[2 * j + 1];
        const Real m2 = re * re + im * im;
        const Real inv = up[i] / std::sqrt(m2 + kNormEps);
        o[2 * j] = re * inv;
        o[2 * j + 1] = im * inv;
      }
    }
  });
  const Stacked x{&store.entity, &store.relation};
  StackedMut sink{&g.entity, &g.relation};
  const CsrMatrix& a = sb.a;
  std::vector<Real> others(static_cast<size_t>(2 * d));
  for (Index i = 0; i < a.num_rows; ++i) {
    const Index lo = a.row_ptr[i], hi = a.row_ptr[i + 1];
    const Real* dqi = dq.row(i);
    for (Index p = lo; p < hi; ++p) {
      Real* out = sink.row(a.col_idx[p]);
      if (!selects(a.vals[p])) {
        for (Index j = 0; j < 2 * d; ++j) out[j] = out[j] - dqi[j];
        continue;
      }
      set_identity(others.data(), d, true);
      for (Index q = lo; q < hi; ++q) {
        if (q == p || !selects(a.vals[q])) continue;
        times_row(others.data(), x.row(a.col_idx[q]), d, true, false);
      }
      for (Index j = 0; j < d; ++j) {  // out += dq * conj(others)
        const Real ar = dqi[2 * j], ai = dqi[2 * j + 1];
        const Real br = others[2 * j], bi = -others[2 * j + 1];
        const Real t0 = ar * br, t1 = ai * bi, t2 = ar * bi, t3 = ai * br;
        const Real re = t0 - t1, im = t2 + t3;
        out[2 * j] = out[2 * j] + re;
        out[2 * j + 1] = out[2 * j + 1] + im;
      }
    }
  }
}

}  // namespace

ScoreBatch score_batch(const ModelConfig& cfg, const Store& store, const TripleBatch& b) {  // models.cpp:267-289
  check_config(cfg, store, b);
  switch (cfg.model) {
    case ModelKind::TransE: return transe_forward(cfg, store, b);
    case ModelKind::TransR: return transr_forward(cfg, store, b);
    case ModelKind::TransH: return transh_forward(cfg, store, b);
    case ModelKind::TorusE: return toruse_forward(cfg, store, b);
    case ModelKind::DistMult:
    case ModelKind::ComplEx: return product_forward(cfg, store, b);
    case ModelKind::RotatE: return rotate_forward(cfg, store, b);
  }
  throw ConfigError("unknown model");
}

void score_backward(const ModelConfig& cfg, const Store& store, const ScoreBatch& sb,
                    const std::vector<Real>& up, Gradients& g) {  // models.cpp:291-325
  check_config(cfg, store, sb.batch);
  if (static_cast<Index>(up.size()) != sb.batch.size())
    throw ShapeError("score_backward: upstream length does not match the batch");
  switch (cfg.model) {
    case ModelKind::TransE: transe_backward(cfg, sb, up, g); return;
    case ModelKind::TransR: transr_backward(cfg, store, sb, up, g); return;
    case ModelKind::TransH: transh_backward(cfg, store, sb, up, g); return;
    case ModelKind::TorusE: toruse_backward(cfg, sb, up, g); return;
    case ModelKind::DistMult:
    case ModelKind::ComplEx: product_backward(cfg, store, sb, up, g); return;
    case ModelKind::RotatE: rotate_backward(cfg, store, sb, up, g); return;
  }
}

// -------------------------------------------------------------- embedding.cpp

namespace {
void fill_uniform(Mat& m, double bound, std::mt19937_64& rng) {  // embedding.cpp:17-30
  std::uniform_real_distribution<double> dist(-bound, bound);
  for (Index i = 0; i < m.rows; ++i)
    for (Index j = 0; j < m.cols; ++j) m.row(i)[j] = static_cast<Real>(dist(rng));
}
bool all_finite(const Mat& g) {
  for (Index i = 0; i < g.size(); ++i)
    if (!std::isfinite(g.p[i])) return false;
  return true;
}
}  // namespace

Store init_store(ModelKind model, Index n_ent, Index n_rel, Index de, Index dr, std::uint64_t seed) {  // embedding.cpp:129-163
  if (de < 1 || dr < 1) throw ConfigError("embedding dimensions must be at least 1");
  if (n_ent < 1 || n_rel < 1) throw ConfigError("store needs at least one entity and one relation");
  std::mt19937_64 rng(seed);
  Store s;
  // complex coefficients: re then im per coordinate (embedding.cpp:21-25)
  const Index wc = is_complex_model(model) ? 2 : 1;
  s.entity = Mat(n_ent, wc * de);
  fill_uniform(s.entity, 6.0 / std::sqrt(static_cast<double>(de)), rng);
  s.relation = Mat(n_rel, wc * dr);
  fill_uniform(s.relation, 6.0 / std::sqrt(static_cast<double>(dr)), rng);
  if (model == ModelKind::TransR) {
    s.proj = Mat(n_rel, dr * de);
    for (Index r = 0; r < n_rel; ++r)
      for (Index k = 0; k < std::min(dr, de); ++k) s.proj.row(r)[k * de + k] = Real(1);
  }
  if (model == ModelKind::TransH) {
    s.normals = Mat(n_rel, de);
    fill_uniform(s.normals, 6.0 / std::sqrt(static_cast<double>(de)), rng);
    for (Index r = 0; r < n_rel; ++r) {
      const Real n = row_norm(s.normals.row(r), de);
      if (n > Real(0))
        for (Index j = 0; j < de; ++j) s.normals.row(r)[j] /= n;
      else
        s.normals.row(r)[0] = Real(1);
    }
  }
  return s;
}

void sgd_step(Store& s, const Gradients& g, Real lr) {  // embedding.cpp:165-190
  if (g.entity.rows != s.entity.rows || g.entity.cols != s.entity.cols ||
      g.relation.rows != s.relation.rows || g.relation.cols != s.relation.cols ||
      g.proj.rows != s.proj.rows || g.proj.cols != s.proj.cols ||
      g.normals.rows != s.normals.rows || g.normals.cols != s.normals.cols)
    throw ShapeError("sgd_step: gradient shapes do not match the store");
  if (!all_finite(g.entity)) throw TrainingError("non-finite gradient in entity embeddings");
  if (!all_finite(g.relation)) throw TrainingError("non-finite gradient in relation embeddings");
  if (!all_finite(g.proj)) throw TrainingError("non-finite gradient in relation projections");
  if (!all_finite(g.normals)) throw TrainingError("non-finite gradient in hyperplane normals");
  auto step = [lr](Mat& p, const Mat& gm) {
    for (Index i = 0; i < p.size(); ++i) {
      const Real t = lr * gm.p[i];
      p.p[i] = p.p[i] - t;
    }
  };
  step(s.entity, g.entity);
  step(s.relation, g.relation);
  if (s.has_proj()) step(s.proj, g.proj);
  if (s.has_normals()) {
    step(s.normals, g.normals);
    for (Index r = 0; r < s.normals.rows; ++r) {
      const Real n = row_norm(s.normals.row(r), s.normals.cols);
      if (!(n > Real(0))) throw TrainingError("hyperplane normal " + std::to_string(r) + " collapsed to zero");
      for (Index j = 0; j < s.normals.cols; ++j) s.normals.row(r)[j] /= n;
    }
  }
}

void renormalize_entities(Store& s) {  // embedding.cpp:192-198
  for (Index i = 0; i < s.entity.rows; ++i) {
    const Real n = row_norm(s.entity.row(i), s.entity.cols);
    if (n > Real(0))
      for (Index j = 0; j < s.entity.cols; ++j) s.entity.row(i)[j] /= n;
  }
}

// --------------------------------------------------------------- training.cpp

void TrainConfig::validate() const {  // training.hpp:42-49
  if (batch_size < 1) throw ConfigError("batch_size must be at least 1");
  if (!(margin >= Real(0))) throw ConfigError("margin must be nonnegative");
  if (!(lr >= Real(0)) || !std::isfinite(lr)) throw ConfigError("lr must be finite and >= 0");
  if (epochs < 0) throw ConfigError("epochs must be nonnegative");
  if (has_scheduler && (decay_every < 1 || !(decay_factor > Real(0))))
    throw ConfigError("scheduler needs every_epochs >= 1 and a positive factor");
}

namespace {
// training.cpp:22-31 — uniform over [0, n) minus up to two excluded ids.
Index draw_excluding(std::mt19937_64& rng, Index n, Index ex0, Index ex1) {
  const Index lo = std::min(ex0, ex1), hi = std::max(ex0, ex1);
  const Index k = lo == hi ? 1 : 2;
  std::uniform_int_distribution<Index> dist(0, n - 1 - k);
  Index v = dist(rng);
  if (v >= lo) ++v;
  if (k == 2 && v >= hi) ++v;
  return v;
}

std::vector<Real> signed_scores(Real sign, const std::vector<Real>& v) {  // sign * RealVector
  std::vector<Real> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = sign * v[i];
  return out;
}

TripleBatch take(const TripleBatch& b, const IndexVector& order, Index lo, Index hi) {  // training.cpp:33-47
  TripleBatch out;
  out.num_entities = b.num_entities;
  out.num_relations = b.num_relations;
  for (Index k = lo; k < hi; ++k) {
    const Index i = order[k];
    out.heads.push_back(b.heads[i]);
    out.relations.push_back(b.relations[i]);
    out.tails.push_back(b.tails[i]);
  }
  return out;
}

using Clock = std::chrono::steady_clock;
struct PhaseTimer {  // training.cpp:15-20
  double& bucket;
  Clock::time_point t0 = Clock::now();
  explicit PhaseTimer(double& b) : bucket(b) {}
  ~PhaseTimer() { bucket += std::chrono::duration<double>(Clock::now() - t0).count(); }
};
}  // namespace

TripleBatch negative_sample(const TripleBatch& pos, std::uint64_t seed, bool avoid) {  // training.cpp:51-71
  pos.validate();
  const Index n = pos.num_entities;
  if (n < 2) throw ConfigError("negative sampling needs at least two entities");
  if (avoid && n < 3) throw ConfigError("self-loop-free negative sampling needs at least three entities");
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> coin(0, 1);
  TripleBatch out = pos;
  for (Index i = 0; i < pos.size(); ++i) {
    const bool corrupt_head = coin(rng) == 0;
    const Index original = corrupt_head ? pos.heads[i] : pos.tails[i];
    const Index other = corrupt_head ? pos.tails[i] : pos.heads[i];
    const Index rep = avoid ? draw_excluding(rng, n, original, other) : draw_excluding(rng, n, original, original);
    (corrupt_head ? out.heads[i] : out.tails[i]) = rep;
  }
  return out;
}

IndexVector epoch_order(Index m, const TrainConfig& tc, Index epoch) {  // training.cpp:106-112
  IndexVector order(static_cast<size_t>(m));
  std::iota(order.begin(), order.end(), Index{0});
  if (tc.shuffle) {
    std::mt19937_64 rng(tc.seed ^ (0x9E3779B97F4A7C15ULL * static_cast<std::uint64_t>(epoch + 1)));
    std::shuffle(order.begin(), order.end(), rng);
  }
  return order;
}

LossGrad margin_ranking_loss(const std::vector<Real>& p, const std::vector<Real>& n, Real margin) {  // training.cpp:73-94
  if (p.size() != n.size()) throw ShapeError("margin_ranking_loss: length mismatch");
  const Index m = static_cast<Index>(p.size());
  LossGrad lg;
  lg.d_pos.assign(static_cast<size_t>(m), Real(0));
  lg.d_neg.assign(static_cast<size_t>(m), Real(0));
  if (m == 0) return lg;
  const Real unit = Real(1) / Real(m);
  Real sum = 0;
  for (Index i = 0; i < m; ++i) {
    const Real term = margin + p[i] - n[i];
    if (term > Real(0)) {
      sum += term;
      lg.d_pos[i] = unit;
      lg.d_neg[i] = -unit;
    }
  }
  lg.loss = sum / Real(m);
  return lg;
}

EpochReport train_epoch(const ModelConfig& mc, Store& store, const TripleBatch& pos,
                        const TripleBatch& neg, const TrainConfig& tc, Index epoch, Real lr) {  // training.cpp:96-164
  tc.validate();
  const Index m = pos.size();
  if (m < 1) throw ConfigError("training requires at least one triple");
  if (neg.size() != m) throw ShapeError("negative set is not aligned with the positive triples");
  const IndexVector order = epoch_order(m, tc, epoch);
  const Real sign = energy_sign(mc.model);  // models.hpp:35-38
  EpochReport rep;
  rep.epoch = epoch;
  Gradients grads = make_gradients(store);
  Real loss_sum = 0;
  for (Index lo = 0; lo < m; lo += tc.batch_size) {
    const Index hi = std::min(m, lo + tc.batch_size);
    ScoreBatch ps, ns;
    LossGrad lg;
    {
      PhaseTimer t(rep.t_forward_s);
      const TripleBatch pb = take(pos, order, lo, hi);
      const TripleBatch nb = take(neg, order, lo, hi);
      ps = score_batch(mc, store, pb);
      ns = score_batch(mc, store, nb);
      lg = margin_ranking_loss(signed_scores(sign, ps.scores), signed_scores(sign, ns.scores), tc.margin);
    }
    if (!std::isfinite(lg.loss))
      throw TrainingError("non-finite loss at epoch " + std::to_string(epoch) + ", batch " +
                          std::to_string(lo / tc.batch_size));
    loss_sum += lg.loss * Real(hi - lo);
    {
      PhaseTimer t(rep.t_backward_s);
      grads.entity.set_zero();
      grads.relation.set_zero();
      grads.proj.set_zero();
      grads.normals.set_zero();
      score_backward(mc, store, ps, signed_scores(sign, lg.d_pos), grads);
      score_backward(mc, store, ns, signed_scores(sign, lg.d_neg), grads);
      ps = ScoreBatch{};
      ns = ScoreBatch{};
    }
    {
      PhaseTimer t(rep.t_step_s);
      sgd_step(store, grads, lr);
    }
  }
  rep.loss = loss_sum / Real(m);
  return rep;
}

std::vector<EpochReport> fit(const ModelConfig& mc, Store& store, const TripleBatch& train,
                             const TrainConfig& tc) {  // training.cpp:166-195
  mc.validate();
  tc.validate();
  std::vector<EpochReport> run;
  if (tc.epochs == 0) return run;
  const bool no_self_loops = is_multiplicative_model(mc.model);
  TripleBatch neg = negative_sample(train, tc.seed, no_self_loops);
  for (Index e = 0; e < tc.epochs; ++e) {
    if (tc.resample_negatives && e > 0)
      neg = negative_sample(train, tc.seed + static_cast<std::uint64_t>(e) * 0x9E3779B9ULL, no_self_loops);
    Real lr = tc.lr;
    if (tc.has_scheduler)
      lr = tc.lr * static_cast<Real>(std::pow(tc.decay_factor, double(e / tc.decay_every)));
    EpochReport rep = train_epoch(mc, store, train, neg, tc, e, lr);
    if (tc.renorm_entities) renormalize_entities(store);
    run.push_back(rep);
  }
  return run;
}

// ---------------------------------------------------------------- data_io.cpp

TripleBatch generate_synthetic(Index n_entities, Index n_relations, Index n_triples,
                               std::uint64_t seed) {  // data_io.cpp:128-211
  if (n_entities < 4 || n_relations < 1 || n_triples < 3)
    throw ConfigError("synthetic dataset needs >= 4 entities, >= 1 relation, >= 3 triples");
  const Index side = static_cast<Index>(std::ceil(std::cbrt(double(n_entities))));
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> step(-2, 2);
  std::vector<std::array<int, 3>> disp(static_cast<size_t>(n_relations));
  for (auto& d : disp) {
    do {
      d = {step(rng), step(rng), step(rng)};
    } while (d[0] == 0 && d[1] == 0 && d[2] == 0);
  }
  std::uniform_int_distribution<Index> ent(0, n_entities - 1);
  std::uniform_int_distribution<Index> rel(0, n_relations - 1);
  std::unordered_set<std::uint64_t> seen;
  TripleBatch all;
  all.num_entities = n_entities;
  all.num_relations = n_relations;
  const std::uint64_t max_attempts = static_cast<std::uint64_t>(n_triples) * 1000;
  std::uint64_t attempts = 0;
  while (all.size() < n_triples) {
    if (++attempts > max_attempts)
      throw ConfigError("cannot plant " + std::to_string(n_triples) +
                        " unique triples on this lattice; lower n_triples");
    const Index h = ent(rng);
    const Index r = rel(rng);
    const Index cx = h % side, cy = (h / side) % side, cz = h / (side * side);
    const auto& d = disp[static_cast<size_t>(r)];
    const Index x = cx + d[0], y = cy + d[1], z = cz + d[2];
    if (x < 0 || x >= side || y < 0 || y >= side || z < 0 || z >= side) continue;
    const Index t = x + side * (y + side * z);
    if (t >= n_entities || t == h) continue;
    const std::uint64_t key = static_cast<std::uint64_t>(h) * n_relations + r;
    if (!seen.insert(key).second) continue;
    all.heads.push_back(h);
    all.relations.push_back(r);
    all.tails.push_back(t);
  }
  return all;  // split: [0,n_test) test, next n_valid valid, rest train (data_io.cpp:189-203)
}

}  // namespace orc
