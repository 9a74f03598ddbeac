// TEST INFRASTRUCTURE ONLY — flat C entry points over the oracle restatement so
// pytest (ctypes) and bench.py's CPU legs can drive it. Real is float in
// liboracle_f32.so and double in liboracle_f64.so. Errors come back as status
// codes mirroring skg_status (include/skge_b200.h) plus orc_last_error().
#include <chrono>
#include <algorithm>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

#include "skge_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

enum { OK = 0, E_SHAPE = 1, E_CONFIG = 2, E_DEGENERATE = 3, E_TRAINING = 4, E_PARSE = 5, E_OTHER = 7 };

template <class F>
int guard(F&& f) {
  try {
    f();
    return OK;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return E_SHAPE;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return E_CONFIG;
  } catch (const DegenerateTripleError& e) {
    g_err = e.what();
    return E_DEGENERATE;
  } catch (const TrainingError& e) {
    g_err = e.what();
    return E_TRAINING;
  } catch (const ParseError& e) {
    g_err = e.what();
    return E_PARSE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_OTHER;
  }
}

TripleBatch mk_batch(Index m, const Index* h, const Index* r, const Index* t, Index n, Index nr) {
  TripleBatch b;
  b.heads.assign(h, h + m);
  b.relations.assign(r, r + m);
  b.tails.assign(t, t + m);
  b.num_entities = n;
  b.num_relations = nr;
  return b;
}
}  // namespace

extern "C" {

struct orc_model_config {
  std::uint32_t model, norm;
  std::int64_t dim_entity, dim_relation;
};
struct orc_store {  // caller-owned row-major tables; proj/normals may be null
  std::int64_t num_entities, num_relations, dim_entity, dim_relation;
  Real* entity;
  Real* relation;
  Real* proj;
  Real* normals;
};
struct orc_train_config {
  Real lr, margin;
  std::int64_t epochs, batch_size;
  std::uint64_t seed;
  std::int32_t has_scheduler;
  std::int64_t decay_every;
  Real decay_factor;
  std::int32_t shuffle, resample_negatives, renorm_entities;
};
struct orc_epoch_report {
  std::int64_t epoch;
  double loss;
  double t_forward_s, t_backward_s, t_step_s;
};

}  // extern "C"

namespace {
ModelConfig mk_cfg(const orc_model_config* c) {
  ModelConfig m;
  m.model = static_cast<ModelKind>(c->model);
  m.norm = static_cast<NormKind>(c->norm);
  m.dim_entity = c->dim_entity;
  m.dim_relation = c->dim_relation;
  return m;
}
Store view_store(const orc_store* s) {
  Store st;
  st.entity = Mat::view(s->entity, s->num_entities, s->dim_entity);
  st.relation = Mat::view(s->relation, s->num_relations, s->dim_relation);
  if (s->proj) st.proj = Mat::view(s->proj, s->num_relations, s->dim_relation * s->dim_entity);
  if (s->normals) st.normals = Mat::view(s->normals, s->num_relations, s->dim_entity);
  return st;
}
TrainConfig mk_tc(const orc_train_config* c) {
  TrainConfig t;
  t.lr = c->lr;
  t.margin = c->margin;
  t.epochs = c->epochs;
  t.batch_size = c->batch_size;
  t.seed = c->seed;
  t.has_scheduler = c->has_scheduler != 0;
  t.decay_every = c->decay_every;
  t.decay_factor = c->decay_factor;
  t.shuffle = c->shuffle != 0;
  t.resample_negatives = c->resample_negatives != 0;
  t.renorm_entities = c->renorm_entities != 0;
  return t;
}
void copy_mat(const Mat& src, Real* dst) {
  if (dst && src.size() > 0) std::memcpy(dst, src.p, sizeof(Real) * static_cast<size_t>(src.size()));
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_real_bytes() { return static_cast<int>(sizeof(Real)); }
void orc_set_num_threads(int n) { set_num_threads(n); }

// n-th (0-based) output of std::mt19937_64(seed): known-answer checks.
std::uint64_t orc_mt19937_64_nth(std::uint64_t seed, std::int64_t n) {
  std::mt19937_64 g(seed);
  std::uint64_t v = 0;
  for (std::int64_t i = 0; i <= n; ++i) v = g();
  return v;
}

// Triples in generation order; split sizes per data_io.cpp:189-190.
int orc_generate_synthetic(Index n_ent, Index n_rel, Index n_triples, std::uint64_t seed, Index* h,
                           Index* r, Index* t) {
  return guard([&] {
    TripleBatch b = generate_synthetic(n_ent, n_rel, n_triples, seed);
    std::memcpy(h, b.heads.data(), sizeof(Index) * b.heads.size());
    std::memcpy(r, b.relations.data(), sizeof(Index) * b.heads.size());
    std::memcpy(t, b.tails.data(), sizeof(Index) * b.heads.size());
  });
}

int orc_init_store(std::uint32_t model, Index n_ent, Index n_rel, Index de, Index dr,
                   std::uint64_t seed, Real* ent, Real* rel, Real* proj, Real* normals) {
  return guard([&] {
    Store s = init_store(static_cast<ModelKind>(model), n_ent, n_rel, de, dr, seed);
    copy_mat(s.entity, ent);
    copy_mat(s.relation, rel);
    copy_mat(s.proj, proj);
    copy_mat(s.normals, normals);
  });
}

int orc_negative_sample(Index m, const Index* h, const Index* r, const Index* t, Index n_ent,
                        Index n_rel, std::uint64_t seed, int avoid, Index* out_h, Index* out_t) {
  return guard([&] {
    TripleBatch neg = negative_sample(mk_batch(m, h, r, t, n_ent, n_rel), seed, avoid != 0);
    std::memcpy(out_h, neg.heads.data(), sizeof(Index) * static_cast<size_t>(m));
    std::memcpy(out_t, neg.tails.data(), sizeof(Index) * static_cast<size_t>(m));
  });
}

int orc_epoch_order(Index m, std::uint64_t seed, int shuffle, Index epoch, Index* out) {
  return guard([&] {
    TrainConfig tc;
    tc.seed = seed;
    tc.shuffle = shuffle != 0;
    IndexVector o = epoch_order(m, tc, epoch);
    std::memcpy(out, o.data(), sizeof(Index) * static_cast<size_t>(m));
  });
}

// kind 0 = ht (incidence.hpp:38), 1 = hrt (:62), 2 = multiplicative, 3 = multiplicative
// with the conjugate tail marker (:93). row_ptr has m+1 slots, col/val 3m.
int orc_build_incidence(int kind, Index m, const Index* h, const Index* r, const Index* t,
                        Index n_ent, Index n_rel, Index* row_ptr, Index* col, Real* val, Index* nnz) {
  return guard([&] {
    TripleBatch b = mk_batch(m, h, r, t, n_ent, n_rel);
    CsrMatrix c = coo_to_csr(kind == 0 ? build_ht(b) : kind == 1 ? build_hrt(b) : build_multiplicative(b, kind == 3));
    std::memcpy(row_ptr, c.row_ptr.data(), sizeof(Index) * c.row_ptr.size());
    std::memcpy(col, c.col_idx.data(), sizeof(Index) * c.col_idx.size());
    std::memcpy(val, c.vals.data(), sizeof(Real) * c.vals.size());
    *nnz = c.nnz();
  });
}

// Generic COO -> canonical CSR (sparse.hpp:110). Outputs sized nnz_in (+rows+1).
int orc_coo_to_csr(Index rows, Index cols, Index nnz_in, const Index* ri, const Index* ci,
                   const Real* vi, Index* row_ptr, Index* col, Real* val, Index* nnz) {
  return guard([&] {
    CooMatrix c;
    c.num_rows = rows;
    c.num_cols = cols;
    c.rows.assign(ri, ri + nnz_in);
    c.cols.assign(ci, ci + nnz_in);
    c.vals.assign(vi, vi + nnz_in);
    CsrMatrix s = coo_to_csr(c);
    std::memcpy(row_ptr, s.row_ptr.data(), sizeof(Index) * s.row_ptr.size());
    std::memcpy(col, s.col_idx.data(), sizeof(Index) * s.col_idx.size());
    std::memcpy(val, s.vals.data(), sizeof(Real) * s.vals.size());
    *nnz = s.nnz();
  });
}

namespace {
CsrMatrix mk_csr(Index rows, Index cols, const Index* rp, const Index* ci, const Real* v) {
  CsrMatrix a;
  a.num_rows = rows;
  a.num_cols = cols;
  a.row_ptr.assign(rp, rp + rows + 1);
  a.col_idx.assign(ci, ci + rp[rows]);
  a.vals.assign(v, v + rp[rows]);
  return a;
}
}  // namespace

int orc_transpose(Index rows, Index cols, const Index* rp, const Index* ci, const Real* v,
                  Index* out_rp, Index* out_ci, Real* out_v) {
  return guard([&] {
    CsrMatrix t = transpose(mk_csr(rows, cols, rp, ci, v));
    std::memcpy(out_rp, t.row_ptr.data(), sizeof(Index) * t.row_ptr.size());
    std::memcpy(out_ci, t.col_idx.data(), sizeof(Index) * t.col_idx.size());
    std::memcpy(out_v, t.vals.data(), sizeof(Real) * t.vals.size());
  });
}

int orc_spmm(Index rows, Index cols, const Index* rp, const Index* ci, const Real* v,
             Index x_rows, Index d, const Real* x, Real* out) {
  return guard([&] {
    Mat xm = Mat::view(const_cast<Real*>(x), x_rows, d);
    Mat z = spmm(mk_csr(rows, cols, rp, ci, v), xm);
    copy_mat(z, out);
  });
}

int orc_spmm_transpose_add(Index rows, Index cols, const Index* rp, const Index* ci, const Real* v,
                           Index d, const Real* g, Real* sink) {
  return guard([&] {
    Mat gm = Mat::view(const_cast<Real*>(g), rows, d);
    Mat out = Mat::view(sink, cols, d);
    spmm_transpose_add(mk_csr(rows, cols, rp, ci, v), gm, out);
  });
}

// scores (m), and optionally the residual rows the backward uses:
// v (m x d_r; translational/projection models), u (m x d_e), delta (m x d).
int orc_score_batch(const orc_model_config* cfg, const orc_store* st, Index m, const Index* h,
                    const Index* r, const Index* t, Real* scores, Real* v, Real* u, Real* delta) {
  return guard([&] {
    Store s = view_store(st);
    ScoreBatch sb = score_batch(mk_cfg(cfg), s, mk_batch(m, h, r, t, st->num_entities, st->num_relations));
    std::memcpy(scores, sb.scores.data(), sizeof(Real) * sb.scores.size());
    copy_mat(sb.v, v);
    copy_mat(sb.u, u);
    copy_mat(sb.delta, delta);
  });
}

// rank_entity (eval.cpp:16-63) for q queries, Tail then Head side per query
// (the order evaluate() visits them, eval.cpp:80-86): ranks[2i] = tail rank,
// ranks[2i+1] = head rank. filtered != 0: competing candidates whose triple is
// in the nf filter triples (TripleFilter, eval.hpp:25-45) are skipped; the
// query's own entity never is. Multiplicative models exclude the self-loop
// candidate (energy +inf, eval.cpp:36-37); energies carry energy_sign.
int orc_rank_entities(const orc_model_config* cfg, const orc_store* st, Index q, const Index* qh,
                      const Index* qr, const Index* qt, int filtered, Index nf, const Index* fh,
                      const Index* fr, const Index* ft, Index* ranks) {
  return guard([&] {
    Store s = view_store(st);
    const ModelConfig mc = mk_cfg(cfg);
    const Index n = st->num_entities, nr = st->num_relations;
    auto key = [&](Index h, Index r, Index t) {
      return (static_cast<std::uint64_t>(h) * static_cast<std::uint64_t>(nr) + static_cast<std::uint64_t>(r)) *
                 static_cast<std::uint64_t>(n) + static_cast<std::uint64_t>(t);
    };
    std::unordered_set<std::uint64_t> known;
    if (filtered)
      for (Index i = 0; i < nf; ++i) known.insert(key(fh[i], fr[i], ft[i]));
    const bool no_self = is_multiplicative_model(mc.model);  // eval.cpp:24, 36-37
    const Real sign = energy_sign(mc.model);
    std::vector<Index> ch, cr, ct, cand;
    std::vector<Real> energy(static_cast<size_t>(n));
    for (Index i = 0; i < q; ++i) {
      const Index h = qh[i], r = qr[i], t = qt[i];
      if (h < 0 || h >= n || t < 0 || t >= n || r < 0 || r >= nr) throw ShapeError("rank_entity: query ids out of range");
      for (int side = 0; side < 2; ++side) {  // 0 = Tail, 1 = Head
        const Index fixed = side == 0 ? h : t;
        ch.clear(), cr.clear(), ct.clear(), cand.clear();
        for (Index c = 0; c < n; ++c) {
          if (no_self && c == fixed) continue;  // unrepresentable candidate, ranks worst
          cand.push_back(c);
          ch.push_back(side == 0 ? h : c);
          cr.push_back(r);
          ct.push_back(side == 0 ? c : t);
        }
        ScoreBatch sb = score_batch(mc, s, mk_batch(static_cast<Index>(cand.size()), ch.data(), cr.data(), ct.data(), n, nr));
        std::fill(energy.begin(), energy.end(), std::numeric_limits<Real>::infinity());
        for (size_t k = 0; k < cand.size(); ++k) energy[cand[k]] = sign * sb.scores[k];
        const Index truth = side == 0 ? t : h;
        const Real te = energy[truth];
        Index better = 0;
        for (Index c = 0; c < n; ++c) {
          if (c == truth) continue;
          if (filtered && known.count(side == 0 ? key(h, r, c) : key(c, r, t))) continue;
          if (energy[c] < te) ++better;
        }
        ranks[2 * i + side] = better + 1;
      }
    }
  });
}

// Accumulates d(sum_i up_i * score_i) into the grads tables (caller zeroes).
int orc_score_backward(const orc_model_config* cfg, const orc_store* st, Index m, const Index* h,
                       const Index* r, const Index* t, const Real* up, orc_store* grads) {
  return guard([&] {
    Store s = view_store(st);
    ModelConfig mc = mk_cfg(cfg);
    TripleBatch b = mk_batch(m, h, r, t, st->num_entities, st->num_relations);
    ScoreBatch sb = score_batch(mc, s, b);
    Store g = view_store(grads);
    std::vector<Real> upv(up, up + m);
    score_backward(mc, s, sb, upv, g);
  });
}

int orc_margin_ranking_loss(Index m, Index m_neg, const Real* p, const Real* n, Real margin,
                            Real* loss, Real* d_pos, Real* d_neg) {
  return guard([&] {
    LossGrad lg = margin_ranking_loss(std::vector<Real>(p, p + m), std::vector<Real>(n, n + m_neg), margin);
    *loss = lg.loss;
    std::memcpy(d_pos, lg.d_pos.data(), sizeof(Real) * static_cast<size_t>(m));
    std::memcpy(d_neg, lg.d_neg.data(), sizeof(Real) * static_cast<size_t>(m));
  });
}

int orc_sgd_step(orc_store* st, const orc_store* grads, Real lr) {
  return guard([&] {
    Store s = view_store(st);
    Store g = view_store(grads);
    sgd_step(s, g, lr);
  });
}

int orc_renormalize_entities(orc_store* st) {
  return guard([&] {
    Store s = view_store(st);
    renormalize_entities(s);
  });
}

int orc_train_epoch(const orc_model_config* cfg, orc_store* st, Index m, const Index* ph,
                    const Index* pr, const Index* pt, const Index* nh, const Index* nt,
                    const orc_train_config* tc, Index epoch, Real lr, orc_epoch_report* rep) {
  return guard([&] {
    Store s = view_store(st);
    TripleBatch pos = mk_batch(m, ph, pr, pt, st->num_entities, st->num_relations);
    TripleBatch neg = mk_batch(m, nh, pr, nt, st->num_entities, st->num_relations);
    EpochReport e = train_epoch(mk_cfg(cfg), s, pos, neg, mk_tc(tc), epoch, lr);
    rep->epoch = e.epoch;
    rep->loss = e.loss;
    rep->t_forward_s = e.t_forward_s;
    rep->t_backward_s = e.t_backward_s;
    rep->t_step_s = e.t_step_s;
  });
}

// Bounded-sample training for the CPU baseline: batches [b0, b0+nb) of the
// epoch's order, exactly as train_epoch would run them. Returns seconds.
int orc_train_batches(const orc_model_config* cfg, orc_store* st, Index m, const Index* ph,
                      const Index* pr, const Index* pt, const Index* nh, const Index* nt,
                      const orc_train_config* tc, Index epoch, Real lr, Index b0, Index nb,
                      double* seconds, double* loss_sum) {
  return guard([&] {
    Store s = view_store(st);
    TrainConfig t = mk_tc(tc);
    TripleBatch pos = mk_batch(m, ph, pr, pt, st->num_entities, st->num_relations);
    TripleBatch neg = mk_batch(m, nh, pr, nt, st->num_entities, st->num_relations);
    // Same per-batch body as train_epoch, restricted to a window of batches.
    const auto t0 = std::chrono::steady_clock::now();
    const IndexVector order = epoch_order(m, t, epoch);
    Gradients grads = make_gradients(s);
    ModelConfig mc = mk_cfg(cfg);
    Real ls = 0;
    for (Index b = b0; b < b0 + nb && b * t.batch_size < m; ++b) {
      const Index lo = b * t.batch_size, hi = std::min(m, lo + t.batch_size);
      TripleBatch pb, nb2;
      pb.num_entities = nb2.num_entities = st->num_entities;
      pb.num_relations = nb2.num_relations = st->num_relations;
      for (Index k = lo; k < hi; ++k) {
        const Index i = order[k];
        pb.heads.push_back(pos.heads[i]), pb.relations.push_back(pos.relations[i]), pb.tails.push_back(pos.tails[i]);
        nb2.heads.push_back(neg.heads[i]), nb2.relations.push_back(neg.relations[i]), nb2.tails.push_back(neg.tails[i]);
      }
      ScoreBatch ps = score_batch(mc, s, pb), ns = score_batch(mc, s, nb2);
      const Real sign = energy_sign(mc.model);
      auto sg = [sign](const std::vector<Real>& v) {
        std::vector<Real> o(v.size());
        for (size_t k = 0; k < v.size(); ++k) o[k] = sign * v[k];
        return o;
      };
      LossGrad lg = margin_ranking_loss(sg(ps.scores), sg(ns.scores), t.margin);
      ls += lg.loss * Real(hi - lo);
      grads.entity.set_zero(), grads.relation.set_zero(), grads.proj.set_zero(), grads.normals.set_zero();
      score_backward(mc, s, ps, sg(lg.d_pos), grads);
      score_backward(mc, s, ns, sg(lg.d_neg), grads);
      sgd_step(s, grads, lr);
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *loss_sum = ls;
  });
}

int orc_fit(const orc_model_config* cfg, orc_store* st, Index m, const Index* h, const Index* r,
            const Index* t, const orc_train_config* tc, orc_epoch_report* reports) {
  return guard([&] {
    Store s = view_store(st);
    auto run = fit(mk_cfg(cfg), s, mk_batch(m, h, r, t, st->num_entities, st->num_relations), mk_tc(tc));
    for (size_t e = 0; e < run.size(); ++e) {
      reports[e].epoch = run[e].epoch;
      reports[e].loss = run[e].loss;
      reports[e].t_forward_s = run[e].t_forward_s;
      reports[e].t_backward_s = run[e].t_backward_s;
      reports[e].t_step_s = run[e].t_step_s;
    }
  });
}

}  // extern "C"
