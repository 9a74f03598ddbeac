// Drop-in check: a reference-style caller (the shape of test_training.cpp's
// "fit: loss on a lattice dataset drops" case, tests/unit/test_training.cpp:322)
// written against include/skge_b200.hpp instead of sparsekge/training.hpp.
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
  return last < 0.5f * first ? 0 : 1;
}
