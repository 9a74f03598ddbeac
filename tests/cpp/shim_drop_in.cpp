// Drop-in check: a reference-style caller (the shape of test_training.cpp's
// "fit: loss on a lattice dataset drops" case, tests/unit/test_training.cpp:322)
// written against include/skge_b200.hpp instead of sparsekge/training.hpp.
#include <cmath>
#include <cstdio>
#include <random>

#include "skge_b200.hpp"

int main() {
  using namespace skge;
  // planted-lattice style data: tails are fixed offsets of heads per relation
  TripleBatch train;
  train.num_entities = 125;
  train.num_relations = 6;
  std::mt19937_64 rng(18);
  for (int i = 0; i < 150; ++i) {
    const Index h = static_cast<Index>(rng() % 125), r = static_cast<Index>(rng() % 6);
    train.heads.push_back(h);
    train.relations.push_back(r);
    train.tails.push_back((h + 1 + r) % 125);
  }
  ModelConfig mc;
  mc.model = ModelKind::TransE;
  mc.dim_entity = mc.dim_relation = 16;
  TrainConfig tc;
  tc.lr = 0.1f;
  tc.epochs = 100;
  tc.batch_size = 16;
  tc.seed = 20;
  auto store = init_store(ModelKind::TransE, 125, 6, 16, 16, 6);
  TrainingRun run = fit(mc, store, train, tc);
  Real first = 0, last = 0;
  for (int e = 0; e < 5; ++e) first += run.epochs[e].loss, last += run.epochs[95 + e].loss;
  std::printf("shim fit: first5 %.6f last5 %.6f\n", first / 5, last / 5);
  try {
    TrainConfig bad = tc;
    bad.batch_size = 0;
    fit(mc, store, train, bad);
    return 2;
  } catch (const ConfigError&) {
  }
  // link prediction through the shim (test_eval.cpp:47-79)
  {
    ModelConfig pc;
    pc.model = ModelKind::TransE;
    pc.dim_entity = pc.dim_relation = 2;
    auto plane = init_store(ModelKind::TransE, 5, 1, 2, 2, 0);
    const Real xy[5][2] = {{0, 0}, {0, 1}, {1, 0}, {2, 0}, {0.5f, 0}};
    for (int i = 0; i < 5; ++i) plane.entity(i, 0) = xy[i][0], plane.entity(i, 1) = xy[i][1];
    plane.relation(0, 0) = 1, plane.relation(0, 1) = 0;
    TripleFilter filter(5, 1);
    filter.insert(0, 0, 2);
    filter.insert(0, 0, 4);
    filter.insert(0, 0, 3);
    const Index raw = rank_entity(pc, plane, 0, 0, 3, Side::Tail, nullptr);
    const Index fil = rank_entity(pc, plane, 0, 0, 3, Side::Tail, &filter);
    std::printf("shim rank_entity: raw %lld filtered %lld\n", static_cast<long long>(raw), static_cast<long long>(fil));
    if (raw != 3 || fil != 1) return 3;
  }
  // multiplicative family through the shim (test_models.cpp:174-211, test_training.cpp:290-320)
  {
    ModelConfig dm;
    dm.model = ModelKind::DistMult;
    dm.dim_entity = dm.dim_relation = 1;
    EmbeddingStore s;
    s.entity = Matrix(2, 1);
    s.relation = Matrix(1, 1);
    s.entity(0, 0) = 2, s.entity(1, 0) = 5, s.relation(0, 0) = 3;
    TripleBatch b;
    b.heads = {0}, b.relations = {0}, b.tails = {1}, b.num_entities = 2, b.num_relations = 1;
    if (score_batch(dm, s, b).scores[0] != 30.0f) return 4;
    ModelConfig rc;
    rc.model = ModelKind::RotatE;
    rc.dim_entity = rc.dim_relation = 1;
    EmbeddingStore c;  // interleaved (re, im): h = 1, t = i, r = i
    c.entity = Matrix(2, 2);
    c.relation = Matrix(1, 2);
    c.entity(0, 0) = 1, c.entity(1, 1) = 1, c.relation(0, 1) = 1;
    if (score_batch(rc, c, b).scores[0] != 0.0f) return 5;
    for (ModelKind m : {ModelKind::DistMult, ModelKind::ComplEx, ModelKind::RotatE}) {
      ModelConfig mm;
      mm.model = m;
      mm.dim_entity = mm.dim_relation = 6;
      auto st = init_store(m, 125, 6, 6, 6, 3);
      TrainConfig t2 = tc;
      t2.epochs = 2;
      TrainingRun r2 = fit(mm, st, train, t2);
      if (r2.epochs.size() != 2 || !std::isfinite(r2.epochs.back().loss)) return 6;
    }
    try {
      b.tails = {0};
      score_batch(dm, s, b);
      return 7;
    } catch (const DegenerateTripleError&) {
    }
  }
  return last < 0.5f * first ? 0 : 1;
}
