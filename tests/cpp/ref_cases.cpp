// Reference unit-test case bodies (/root/reference/proj/tests/unit/*.cpp),
// adapted to the fp32 engine and compiled against include/skge_b200.hpp
// instead of sparsekge/*.hpp. Adaptations, all mechanical:
//  - the include line and the doctest runner (tests/cpp/mini_doctest.hpp);
//  - tolerances written for the reference's f64 default (1e-12 .. 1e-15)
//    become fp32 ones (1e-6), since the engine computes in f32 (the
//    reference's SPARSEKGE_REAL32 build);
//  - Eigen row expressions (row(r).norm(), stacked.topRows) are spelled out
//    as loops; the shim's Matrix::row returns a pointer.
// Each case cites the reference case it restates.
#include <cmath>
#include <limits>
#include <random>

#include "mini_doctest.hpp"
#include "skge_b200.hpp"

namespace skge {
namespace {

using Rng = std::mt19937_64;

// test_models.cpp:26-50
ModelConfig mk_cfg(ModelKind m, Index de, Index dr, NormKind norm = NormKind::L2) {
  ModelConfig c;
  c.model = m;
  c.dim_entity = de;
  c.dim_relation = dr;
  c.norm = norm;
  return c;
}
ModelConfig transe_cfg(Index d) { return mk_cfg(ModelKind::TransE, d, d); }
TripleBatch mk_batch(IndexVector h, IndexVector r, IndexVector t, Index n, Index nr) {
  TripleBatch b;
  b.heads = std::move(h);
  b.relations = std::move(r);
  b.tails = std::move(t);
  b.num_entities = n;
  b.num_relations = nr;
  return b;
}
EmbeddingStore mk_store(RealMatrix ent, RealMatrix rel) {
  EmbeddingStore s;
  s.entity = std::move(ent);
  s.relation = std::move(rel);
  return s;
}
// test_util.hpp:25-32, 62-78
RealMatrix random_dense(Rng& rng, Index rows, Index cols, Real lo = Real(-1), Real hi = Real(1)) {
  std::uniform_real_distribution<Real> dist(lo, hi);
  RealMatrix m(rows, cols);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < cols; ++j) m(i, j) = dist(rng);
  return m;
}
TripleBatch random_batch(Rng& rng, Index m, Index n, Index r, bool allow_self_loops = false) {
  TripleBatch b;
  b.num_entities = n;
  b.num_relations = r;
  std::uniform_int_distribution<Index> ent(0, n - 1);
  std::uniform_int_distribution<Index> rel(0, r - 1);
  for (Index i = 0; i < m; ++i) {
    const Index h = ent(rng);
    Index t = ent(rng);
    while (!allow_self_loops && t == h && n > 1) t = ent(rng);
    b.heads.push_back(h);
    b.relations.push_back(rel(rng));
    b.tails.push_back(t);
  }
  return b;
}
double max_abs_diff(const RealMatrix& a, const RealMatrix& b) {
  double m = 0;
  for (Index i = 0; i < a.size(); ++i) m = std::max(m, std::abs(double(a.a[i]) - double(b.a[i])));
  return m;
}
constexpr double kTol = 1e-6;  // fp32 engine (the reference cases use 1e-12 for f64)

// ---------------------------------------------------------------- test_models.cpp
TEST_CASE("transe: perfect translation scores exactly zero") {  // test_models.cpp:54-61
  auto s = mk_store(RealMatrix{{1, 0}, {1, 1}}, RealMatrix{{0, 1}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  for (auto norm : {NormKind::L2, NormKind::L1}) {
    auto sb = score_batch(mk_cfg(ModelKind::TransE, 2, 2, norm), s, b);
    CHECK(sb.scores[0] == 0.0);
  }
}

TEST_CASE("transe: residual [1,2] scores sqrt(5) under l2 and 3 under l1") {  // :63-70
  auto s = mk_store(RealMatrix{{1, 2}, {0, 0}}, RealMatrix{{0, 0}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  auto l2 = score_batch(mk_cfg(ModelKind::TransE, 2, 2, NormKind::L2), s, b);
  CHECK(l2.scores[0] == std::sqrt(Real(5)));
  auto l1 = score_batch(mk_cfg(ModelKind::TransE, 2, 2, NormKind::L1), s, b);
  CHECK(l1.scores[0] == 3.0);
}

TEST_CASE("transe backward: l2 direction v/|v| lands on h and r, negated on t") {  // :72-88
  auto s = mk_store(RealMatrix{{3, 4}, {0, 0}}, RealMatrix{{0, 0}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  auto cfg = mk_cfg(ModelKind::TransE, 2, 2, NormKind::L2);
  auto sb = score_batch(cfg, s, b);
  REQUIRE(sb.scores[0] == 5.0);
  auto g = make_gradients(s);
  RealVector up(1);
  up << 1;
  score_backward(cfg, s, sb, up, g);
  CHECK(std::abs(g.entity(0, 0) - 0.6) <= kTol);
  CHECK(std::abs(g.entity(0, 1) - 0.8) <= kTol);
  CHECK(std::abs(g.entity(1, 0) + 0.6) <= kTol);
  CHECK(std::abs(g.entity(1, 1) + 0.8) <= kTol);
  CHECK(std::abs(g.relation(0, 0) - 0.6) <= kTol);
  CHECK(std::abs(g.relation(0, 1) - 0.8) <= kTol);
}

TEST_CASE("transe backward: l1 direction is the sign, zero at kinks") {  // :90-102
  auto s = mk_store(RealMatrix{{3, -4, 0}, {0, 0, 0}}, RealMatrix{{0, 0, 0}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  auto cfg = mk_cfg(ModelKind::TransE, 3, 3, NormKind::L1);
  auto sb = score_batch(cfg, s, b);
  auto g = make_gradients(s);
  RealVector up(1);
  up << 1;
  score_backward(cfg, s, sb, up, g);
  CHECK(g.relation(0, 0) == 1.0);
  CHECK(g.relation(0, 1) == -1.0);
  CHECK(g.relation(0, 2) == 0.0);
}

TEST_CASE("transr: identity projection reproduces the translational score") {  // :104-112
  Rng rng(41);
  auto store = init_store<Real>(ModelKind::TransR, 12, 4, 5, 5, 41);
  auto b = random_batch(rng, 20, 12, 4);
  auto tr = score_batch(mk_cfg(ModelKind::TransR, 5, 5), store, b);
  auto plain = mk_store(store.entity, store.relation);
  auto te = score_batch(mk_cfg(ModelKind::TransE, 5, 5), plain, b);
  // the reference's Eigen GEMV by an identity block is exact; the engine's
  // tensor-core / FMA projection is fp32-exact on an identity too
  CHECK((tr.scores - te.scores).cwiseAbs().maxCoeff() <= kTol);
}

TEST_CASE("transr: zero projection leaves only the relation vector") {  // :114-121
  auto store = init_store<Real>(ModelKind::TransR, 4, 1, 3, 2, 1);
  store.proj.setZero();
  store.relation = RealMatrix{{3, 4}};
  auto b = mk_batch({0}, {0}, {2}, 4, 1);
  auto sb = score_batch(mk_cfg(ModelKind::TransR, 3, 2), store, b);
  CHECK(sb.scores[0] == 5.0);
}

TEST_CASE("transh: normal orthogonal to the residual changes nothing") {  // :123-130
  auto store = mk_store(RealMatrix{{1, 2, 0}, {0, 0, 0}}, RealMatrix{{0.5, -1, 0}});
  store.normals = RealMatrix{{0, 0, 1}};
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  auto sb = score_batch(mk_cfg(ModelKind::TransH, 3, 3), store, b);
  CHECK(sb.scores[0] == std::sqrt(Real(1.5 * 1.5 + 1.0)));
}

TEST_CASE("transh: difference parallel to the normal projects to zero") {  // :132-138
  auto store = mk_store(RealMatrix{{2, 0}, {0, 0}}, RealMatrix{{0, 0}});
  store.normals = RealMatrix{{1, 0}};
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  auto sb = score_batch(mk_cfg(ModelKind::TransH, 2, 2), store, b);
  CHECK(sb.scores[0] == 0.0);
}

TEST_CASE("toruse: wrapped residual goldens") {  // :140-151
  auto s = mk_store(RealMatrix{{0.75}, {0}}, RealMatrix{{0}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  CHECK(score_batch(mk_cfg(ModelKind::TorusE, 1, 1, NormKind::L2), s, b).scores[0] == 0.0625);
  CHECK(score_batch(mk_cfg(ModelKind::TorusE, 1, 1, NormKind::L1), s, b).scores[0] == 0.25);
  auto s2 = mk_store(RealMatrix{{1.5}, {0}}, RealMatrix{{0}});
  CHECK(score_batch(mk_cfg(ModelKind::TorusE, 1, 1, NormKind::L2), s2, b).scores[0] == 0.25);
  CHECK(score_batch(mk_cfg(ModelKind::TorusE, 1, 1, NormKind::L1), s2, b).scores[0] == 0.5);
}

TEST_CASE("toruse: integer shifts of the embeddings leave scores unchanged") {  // :153-172
  Rng rng(7);
  const Index n = 8, nr = 3, d = 4;
  RealMatrix ent = random_dense(rng, n, d), rel = random_dense(rng, nr, d);
  for (auto* m : {&ent, &rel})  // dyadic coefficients: the shifts stay exact
    for (auto& x : m->a) x = std::round(x * 64) / 64;
  auto s = mk_store(ent, rel);
  auto b = random_batch(rng, 12, n, nr);
  auto cfg = mk_cfg(ModelKind::TorusE, d, d, NormKind::L2);
  auto base = score_batch(cfg, s, b);
  std::uniform_int_distribution<int> shift(-3, 3);
  auto s2 = s;
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < d; ++j) s2.entity(i, j) += shift(rng);
  for (Index i = 0; i < nr; ++i)
    for (Index j = 0; j < d; ++j) s2.relation(i, j) += shift(rng);
  auto shifted = score_batch(cfg, s2, b);
  CHECK((base.scores - shifted.scores).cwiseAbs().maxCoeff() == 0.0);
}

TEST_CASE("distmult: factor product golden") {  // :174-181
  auto s = mk_store(RealMatrix{{2}, {5}}, RealMatrix{{3}});
  auto b = mk_batch({0}, {0}, {1}, 2, 1);
  CHECK(score_batch(mk_cfg(ModelKind::DistMult, 1, 1), s, b).scores[0] == 30.0);
}

TEST_CASE("config errors: mismatched dims and missing tables") {  // :438-472
  auto s = init_store<Real>(ModelKind::TransE, 4, 2, 3, 3, 1);
  auto b = mk_batch({0}, {0}, {1}, 4, 2);
  CHECK_THROWS_AS(score_batch(mk_cfg(ModelKind::TransE, 3, 4), s, b), ConfigError);
  CHECK_THROWS_AS(score_batch(mk_cfg(ModelKind::TransE, 4, 4), s, b), ConfigError);
  CHECK_THROWS_AS(score_batch(mk_cfg(ModelKind::TransR, 3, 3), s, b), ConfigError);
  CHECK_THROWS_AS(score_batch(mk_cfg(ModelKind::TransH, 3, 3), s, b), ConfigError);
  auto b_bad = mk_batch({0}, {0}, {1}, 5, 2);
  CHECK_THROWS_AS(score_batch(mk_cfg(ModelKind::TransE, 3, 3), s, b_bad), ConfigError);
}

TEST_CASE("score_backward: upstream length must match the batch") {
  auto s = init_store<Real>(ModelKind::TransE, 4, 2, 3, 3, 1);
  auto cfg = transe_cfg(3);
  auto sb = score_batch(cfg, s, mk_batch({0, 1}, {0, 1}, {1, 2}, 4, 2));
  auto g = make_gradients(s);
  RealVector up(3);
  CHECK_THROWS_AS(score_backward(cfg, s, sb, up, g), ShapeError);
}

TEST_CASE("score_batch keeps the incidence operand and the ids") {  // models.hpp:41-49
  auto s = init_store<Real>(ModelKind::TransE, 20, 3, 4, 4, 2);
  auto b = mk_batch({5, 3}, {2, 0}, {15, 3}, 20, 3);
  auto sb = score_batch(transe_cfg(4), s, b);
  CHECK(sb.a.row_ptr == IndexVector{0, 3, 4});
  CHECK(sb.a.col_idx == IndexVector{5, 15, 22, 20});
  CHECK(sb.batch.heads == b.heads);
  CHECK(sb.v.rows() == 2);
}

// ---------------------------------------------------------------- test_incidence.cpp
TEST_CASE("build_ht: one triple places +1 at head and -1 at tail") {  // test_incidence.cpp:30-37
  auto c = coo_to_csr(build_ht(mk_batch({5}, {0}, {15}, 22, 1)));
  CHECK(c.num_rows == 1);
  CHECK(c.num_cols == 22);
  CHECK(c.row_ptr == IndexVector{0, 2});
  CHECK(c.col_idx == IndexVector{5, 15});
  CHECK(c.vals == std::vector<Real>{1.0, -1.0});
}

TEST_CASE("build_ht: self-loop cancels to an empty row and a zero difference") {  // :39-45
  auto c = coo_to_csr(build_ht(mk_batch({3}, {0}, {3}, 8, 1)));
  CHECK(c.nnz() == 0);
  Rng rng(5);
  RealMatrix e = random_dense(rng, 8, 4);
  CHECK(spmm(c, e).cwiseAbs().maxCoeff() == 0.0);
}

TEST_CASE("build_hrt: relation column is offset by the entity count") {  // :58-64
  auto coo = build_hrt(mk_batch({5}, {2}, {15}, 20, 3));
  CHECK(coo.num_cols == 23);
  auto c = coo_to_csr(coo);
  CHECK(c.col_idx == IndexVector{5, 15, 22});
  CHECK(c.vals == std::vector<Real>{1.0, -1.0, 1.0});
}

TEST_CASE("build_hrt: batch rows equal gathered h + r - t") {  // :79-95
  Rng rng(43);
  const Index m = 16, n = 10, r = 4, d = 6;
  auto b = random_batch(rng, m, n, r);
  auto coo = build_hrt(b);
  CHECK(coo.nnz() == 3 * m);
  RealMatrix ent = random_dense(rng, n, d), rel = random_dense(rng, r, d);
  RealMatrix stacked(n + r, d);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < d; ++j) stacked(i, j) = ent(i, j);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < d; ++j) stacked(n + i, j) = rel(i, j);
  RealMatrix z = spmm(coo_to_csr(coo), stacked);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < d; ++j)
      CHECK(std::abs(z(i, j) - (ent(b.heads[i], j) + rel(b.relations[i], j) - ent(b.tails[i], j))) < kTol);
}

// ---------------------------------------------------------------- test_sparse.cpp
TEST_CASE("transpose: worked example") {  // test_sparse.cpp:114-130
  CooMatrix<Real> m;
  m.num_rows = 2;
  m.num_cols = 3;
  m.rows = {0, 0, 1};
  m.cols = {0, 2, 1};
  m.vals = {1.0, -1.0, 1.0};
  auto at = transpose(coo_to_csr(m));
  CHECK(at.num_rows == 3);
  CHECK(at.num_cols == 2);
  CHECK(at.row_ptr == IndexVector{0, 1, 2, 3});
  CHECK(at.col_idx == IndexVector{0, 1, 0});
  CHECK(at.vals == std::vector<Real>{1.0, 1.0, -1.0});
}

TEST_CASE("spmm: plus-times worked example and spmm_transpose") {  // :156-163, 245-257
  CooMatrix<Real> m;
  m.num_rows = 2;
  m.num_cols = 3;
  m.rows = {0, 0, 1};
  m.cols = {0, 2, 1};
  m.vals = {1.0, -1.0, 1.0};
  auto a = coo_to_csr(m);
  RealMatrix x(3, 2);
  x << 1, 2, 3, 4, 5, 6;
  RealMatrix expect(2, 2);
  expect << -4, -4, 3, 4;
  CHECK(max_abs_diff(spmm(a, x), expect) == 0.0);
  CooMatrix<Real> m1;
  m1.num_rows = 1;
  m1.num_cols = 3;
  m1.rows = {0, 0};
  m1.cols = {0, 2};
  m1.vals = {1.0, -1.0};
  RealMatrix g1(1, 2);
  g1 << 1, 1;
  RealMatrix e3(3, 2);
  e3 << 1, 1, 0, 0, -1, -1;
  CHECK(max_abs_diff(spmm_transpose(coo_to_csr(m1), g1), e3) == 0.0);
  RealMatrix bad = RealMatrix::Zero(4, 2);
  CHECK_THROWS_AS(spmm(a, bad), ShapeError);
}

TEST_CASE("coo_to_csr: duplicates merge, cancellations drop, bad entries throw") {  // :69-93
  CooMatrix<Real> m;
  m.num_rows = 1;
  m.num_cols = 3;
  m.rows = {0, 0, 0};
  m.cols = {1, 0, 1};
  m.vals = {2.5, 1.0, 1.5};
  auto c = coo_to_csr(m);
  CHECK(c.col_idx == IndexVector{0, 1});
  CHECK(c.vals == std::vector<Real>{1.0, 4.0});
  m.cols = {1, 1, 2};
  m.vals = {1.0, -1.0, 2.0};
  CHECK(coo_to_csr(m).col_idx == IndexVector{2});
  m.cols = {3, 0, 0};
  CHECK_THROWS_AS(coo_to_csr(m), ShapeError);
}

// ---------------------------------------------------------------- test_training.cpp
TEST_CASE("margin_ranking_loss: hinge goldens") {  // test_training.cpp:103-123
  RealVector p(1), n(1);
  p << 0.2, n << 1.0;
  auto lg = margin_ranking_loss(p, n, 0.5);
  CHECK(lg.loss == 0.0);
  CHECK(lg.d_pos[0] == 0.0);
  CHECK(lg.d_neg[0] == 0.0);
  p << 1.0, n << 0.2;
  lg = margin_ranking_loss(p, n, 0.5);
  CHECK(lg.loss == doctest::Approx(1.3).epsilon(kTol));
  CHECK(lg.d_pos[0] == 1.0);
  CHECK(lg.d_neg[0] == -1.0);
  p << 0.7, n << 0.7;
  lg = margin_ranking_loss(p, n, 0.0);
  CHECK(lg.loss == 0.0);
  CHECK(lg.d_pos[0] == 0.0);
}

TEST_CASE("margin_ranking_loss: mean reduction and per-term gradients") {  // :125-136
  RealVector p(2), n(2);
  p << 1.0, 0.0;
  n << 0.2, 5.0;
  auto lg = margin_ranking_loss(p, n, 0.5);
  CHECK(lg.loss == doctest::Approx(1.3 / 2).epsilon(kTol));
  CHECK(lg.d_pos[0] == 0.5);
  CHECK(lg.d_pos[1] == 0.0);
  CHECK(lg.d_neg[0] == -0.5);
  RealVector bad(3);
  CHECK_THROWS_AS(margin_ranking_loss(p, bad, 0.5), ShapeError);
}

TEST_CASE("train_epoch: lr 0 freezes the parameters but reports the loss") {  // :151-164
  auto store = init_store<Real>(ModelKind::TransE, 20, 4, 8, 8, 5);
  auto before = store;
  Rng rng(5);
  auto pos = random_batch(rng, 100, 20, 4);
  auto neg = negative_sample(pos, 6);
  TrainConfig tc;
  tc.batch_size = 32;
  tc.margin = 1.0;
  auto rep = train_epoch(transe_cfg(8), store, pos, neg, tc, Engine::Sparse, 0, Real(0));
  CHECK(store.entity == before.entity);
  CHECK(store.relation == before.relation);
  CHECK(rep.loss > 0.0);
}

TEST_CASE("train_epoch: misaligned negatives are rejected") {  // :166-175
  auto store = init_store<Real>(ModelKind::TransE, 10, 2, 4, 4, 1);
  Rng rng(1);
  auto pos = random_batch(rng, 20, 10, 2);
  NegativeSet neg;
  neg.corrupted = random_batch(rng, 19, 10, 2);
  TrainConfig tc;
  CHECK_THROWS_AS(train_epoch(transe_cfg(4), store, pos, neg, tc, Engine::Sparse, 0, Real(0.1)), ShapeError);
}

TEST_CASE("fit: one triple against its negative trains monotonically") {  // :177-196
  auto store = init_store<Real>(ModelKind::TransE, 2, 1, 8, 8, 3);
  TripleBatch pos;
  pos.num_entities = 2;
  pos.num_relations = 1;
  pos.heads = {0};
  pos.relations = {0};
  pos.tails = {1};
  TrainConfig tc;
  tc.lr = 0.01;
  tc.margin = 2.0;
  tc.epochs = 6;
  tc.batch_size = 1;
  tc.seed = 4;
  auto run = fit(transe_cfg(8), store, pos, tc);
  REQUIRE(run.epochs.size() == 6);
  CHECK(run.epochs[0].loss > 0.0);
  for (size_t e = 0; e + 1 < 6; ++e) CHECK(run.epochs[e + 1].loss < run.epochs[e].loss);
}

TEST_CASE("fit: zero epochs leave the store untouched, bad configs still throw") {  // :198-208
  auto store = init_store<Real>(ModelKind::TransE, 10, 2, 4, 4, 9);
  auto before = store;
  Rng rng(2);
  auto pos = random_batch(rng, 30, 10, 2);
  TrainConfig tc;
  tc.epochs = 0;
  auto run = fit(transe_cfg(4), store, pos, tc);
  CHECK(run.epochs.empty());
  CHECK(store.entity == before.entity);
  tc.batch_size = 0;  // training.cpp:169-170: validation precedes the zero-epoch return
  CHECK_THROWS_AS(fit(transe_cfg(4), store, pos, tc), ConfigError);
}

TEST_CASE("fit: fixed seed reproduces the loss series bitwise") {  // :209-224
  Rng rng(8);
  auto pos = random_batch(rng, 120, 25, 5);
  TrainConfig tc;
  tc.lr = 0.05;
  tc.epochs = 5;
  tc.batch_size = 32;
  tc.seed = 99;
  auto s1 = init_store<Real>(ModelKind::TransE, 25, 5, 8, 8, 1);
  auto s2 = s1;
  auto r1 = fit(transe_cfg(8), s1, pos, tc);
  auto r2 = fit(transe_cfg(8), s2, pos, tc);
  for (Index e = 0; e < 5; ++e) CHECK(r1.epochs[e].loss == r2.epochs[e].loss);
  CHECK(s1.entity == s2.entity);
}

TEST_CASE("fit: scheduler halves the rate on schedule") {  // :244-266
  Rng rng(15);
  auto pos = random_batch(rng, 60, 12, 3);
  TrainConfig tc;
  tc.lr = 0.2;
  tc.epochs = 2;
  tc.batch_size = 20;
  tc.seed = 5;
  tc.scheduler = StepDecay{1, Real(0.5)};
  auto s1 = init_store<Real>(ModelKind::TransE, 12, 3, 4, 4, 2);
  auto s2 = s1;
  auto run = fit(transe_cfg(4), s1, pos, tc);
  auto neg = negative_sample(pos, tc.seed);
  auto cfg = transe_cfg(4);
  auto e0 = train_epoch(cfg, s2, pos, neg, tc, Engine::Sparse, 0, Real(0.2));
  auto e1 = train_epoch(cfg, s2, pos, neg, tc, Engine::Sparse, 1, Real(0.1));
  CHECK(run.epochs[0].loss == e0.loss);
  CHECK(run.epochs[1].loss == e1.loss);
  CHECK(s1.entity == s2.entity);
}

TEST_CASE("fit: per-epoch resampling changes the negatives after epoch 0") {  // :268-286
  Rng rng(16);
  auto pos = random_batch(rng, 60, 20, 4);
  TrainConfig tc;
  tc.lr = 0.05;
  tc.epochs = 3;
  tc.batch_size = 60;
  tc.seed = 31;
  auto s1 = init_store<Real>(ModelKind::TransE, 20, 4, 6, 6, 8);
  auto s2 = s1;
  auto fixed = fit(transe_cfg(6), s1, pos, tc);
  tc.resample_negatives = true;
  auto resampled = fit(transe_cfg(6), s2, pos, tc);
  CHECK(fixed.epochs[0].loss == resampled.epochs[0].loss);
  bool diverged = false;
  for (Index e = 1; e < 3; ++e) diverged |= fixed.epochs[e].loss != resampled.epochs[e].loss;
  CHECK(diverged);
}

TEST_CASE("fit: on_epoch fires after every epoch, in order") {  // training.cpp:190-192
  Rng rng(3);
  auto pos = random_batch(rng, 50, 10, 2);
  TrainConfig tc;
  tc.epochs = 4;
  tc.batch_size = 16;
  auto s = init_store<Real>(ModelKind::TransE, 10, 2, 4, 4, 3);
  std::vector<Index> seen;
  fit(transe_cfg(4), s, pos, tc, Engine::Sparse, [&](const EpochReport& r) { seen.push_back(r.epoch); });
  CHECK(seen == IndexVector{0, 1, 2, 3});
}

TEST_CASE("negative_sample: exactly one side changes, ids stay in range") {  // :25-60
  Rng rng(4);
  auto pos = random_batch(rng, 500, 30, 3);
  auto neg = negative_sample(pos, 11);
  for (Index i = 0; i < pos.size(); ++i) {
    const bool h = neg.corrupted.heads[i] != pos.heads[i], t = neg.corrupted.tails[i] != pos.tails[i];
    CHECK(h != t);
    CHECK(neg.corrupted.relations[i] == pos.relations[i]);
    CHECK(neg.corrupted.heads[i] >= 0);
    CHECK(neg.corrupted.heads[i] < 30);
  }
  TripleBatch one = mk_batch({0}, {0}, {0}, 1, 1);
  CHECK_THROWS_AS(negative_sample(one, 0), ConfigError);
}

// ---------------------------------------------------------------- test_embedding.cpp
TEST_CASE("sgd_step: p=1, g=2, lr=0.1 gives 0.8") {  // test_embedding.cpp:128-136
  EmbeddingStore s;
  s.entity = RealMatrix::Constant(1, 1, 1.0);
  s.relation = RealMatrix::Zero(1, 1);
  auto g = make_gradients(s);
  g.entity(0, 0) = 2.0;
  sgd_step(s, g, Real(0.1));
  CHECK(s.entity(0, 0) == doctest::Approx(0.8).epsilon(kTol));
}

TEST_CASE("sgd_step: zero gradients leave the store bitwise unchanged") {  // :138-146
  auto s = init_store<Real>(ModelKind::TransR, 6, 2, 5, 3, 21);
  auto before = s;
  auto g = make_gradients(s);
  sgd_step(s, g, Real(0.5));
  CHECK(s.entity == before.entity);
  CHECK(s.relation == before.relation);
  CHECK(s.proj == before.proj);
}

TEST_CASE("sgd_step: updates every table") {  // :148-160
  auto s = init_store<Real>(ModelKind::TransR, 4, 2, 3, 3, 2);
  auto g = make_gradients(s);
  g.entity.setConstant(1.0);
  g.relation.setConstant(1.0);
  g.proj.setConstant(1.0);
  auto before = s;
  sgd_step(s, g, Real(0.25));
  CHECK(max_abs_diff(RealMatrix(before.entity - s.entity), RealMatrix::Constant(4, 3, 0.25)) <= kTol);
  CHECK(max_abs_diff(RealMatrix(before.proj - s.proj), RealMatrix::Constant(2, 9, 0.25)) <= kTol);
}

TEST_CASE("sgd_step: hyperplane normals come back unit length") {  // :162-170
  auto s = init_store<Real>(ModelKind::TransH, 5, 3, 8, 8, 13);
  auto g = make_gradients(s);
  Rng rng(99);
  g.normals = random_dense(rng, 3, 8);
  sgd_step(s, g, Real(0.3));
  for (Index r = 0; r < 3; ++r) {
    double n = 0;
    for (Index j = 0; j < 8; ++j) n += double(s.normals(r, j)) * s.normals(r, j);
    CHECK(std::abs(std::sqrt(n) - 1.0) <= kTol);
  }
}

TEST_CASE("sgd_step: non-finite and mismatched gradients are rejected") {  // :172-188
  auto s = init_store<Real>(ModelKind::TransE, 3, 2, 4, 4, 1);
  auto g = make_gradients(s);
  g.entity(1, 2) = std::numeric_limits<Real>::quiet_NaN();
  CHECK_THROWS_AS(sgd_step(s, g, Real(0.1)), TrainingError);
  g.entity(1, 2) = std::numeric_limits<Real>::infinity();
  CHECK_THROWS_AS(sgd_step(s, g, Real(0.1)), TrainingError);
  auto g2 = make_gradients(s);
  g2.relation = RealMatrix::Zero(2, 5);
  CHECK_THROWS_AS(sgd_step(s, g2, Real(0.1)), ShapeError);
}

TEST_CASE("sgd_step: two steps equal one step with summed gradients") {  // :190-207
  auto s1 = init_store<Real>(ModelKind::TransE, 8, 3, 6, 6, 31);
  auto s2 = s1;
  Rng rng(5);
  auto g1 = make_gradients(s1);
  auto g2 = make_gradients(s1);
  g1.entity = random_dense(rng, 8, 6);
  g1.relation = random_dense(rng, 3, 6);
  g2.entity = random_dense(rng, 8, 6);
  g2.relation = random_dense(rng, 3, 6);
  const Real lr = 0.07;
  sgd_step(s1, g1, lr);
  sgd_step(s1, g2, lr);
  auto gsum = make_gradients(s2);
  gsum.entity = g1.entity + g2.entity;
  gsum.relation = g1.relation + g2.relation;
  sgd_step(s2, gsum, lr);
  CHECK(max_abs_diff(s1.entity, s2.entity) <= kTol);
  CHECK(max_abs_diff(s1.relation, s2.relation) <= kTol);
}

TEST_CASE("renormalize_entities: rows project onto the unit sphere") {  // :209-218
  EmbeddingStore s;
  s.entity = RealMatrix{{3, 4}, {0, 0}, {0.5, 0}};
  s.relation = RealMatrix::Zero(1, 2);
  renormalize_entities(s);
  CHECK(s.entity(0, 0) == doctest::Approx(0.6).epsilon(kTol));
  CHECK(s.entity(0, 1) == doctest::Approx(0.8).epsilon(kTol));
  CHECK(s.entity(1, 0) == 0.0);
  CHECK(s.entity(1, 1) == 0.0);
  CHECK(s.entity(2, 0) == doctest::Approx(1.0).epsilon(kTol));
}

}  // namespace
}  // namespace skge

int main() { return mini::run_all(); }
