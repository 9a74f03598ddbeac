// Host-side setup utilities of the engine's C ABI (not on the hot path):
// the reference's synthetic lattice generator (the benchmark-graph format,
// data_io.cpp:128-211) and parameter initialization (embedding.cpp:129-163).
// Both run once per job and use the same libstdc++ <random> templates the
// reference instantiates, so graphs and initial tables are the reference's own.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/skge_b200.h"

namespace {
thread_local std::string g_err;

void fill_uniform(float* m, int64_t rows, int64_t cols, double bound, std::mt19937_64& rng) {
  std::uniform_real_distribution<double> dist(-bound, bound);
  for (int64_t i = 0; i < rows * cols; ++i) m[i] = static_cast<float>(dist(rng));
}
}  // namespace

extern "C" {

const char* skg_host_last_error(void) { return g_err.c_str(); }

skg_status skg_generate_synthetic(int64_t n_entities, int64_t n_relations, int64_t n_triples, uint64_t seed,
                                  int64_t* heads, int64_t* relations, int64_t* tails) {
  if (n_entities < 4 || n_relations < 1 || n_triples < 3) {
    g_err = "synthetic dataset needs >= 4 entities, >= 1 relation, >= 3 triples";
    return SKG_ERR_CONFIG;
  }
  const int64_t side = static_cast<int64_t>(std::ceil(std::cbrt(double(n_entities))));
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> step(-2, 2);
  std::vector<std::array<int, 3>> disp(static_cast<size_t>(n_relations));
  for (auto& d : disp) {
    do {
      d = {step(rng), step(rng), step(rng)};
    } while (d[0] == 0 && d[1] == 0 && d[2] == 0);
  }
  std::uniform_int_distribution<int64_t> ent(0, n_entities - 1);
  std::uniform_int_distribution<int64_t> rel(0, n_relations - 1);
  std::unordered_set<uint64_t> seen;
  seen.reserve(static_cast<size_t>(n_triples) * 2);
  const uint64_t max_attempts = static_cast<uint64_t>(n_triples) * 1000;
  uint64_t attempts = 0;
  int64_t k = 0;
  while (k < n_triples) {
    if (++attempts > max_attempts) {
      g_err = "cannot plant " + std::to_string(n_triples) + " unique triples on this lattice; lower n_triples";
      return SKG_ERR_CONFIG;
    }
    const int64_t h = ent(rng);
    const int64_t r = rel(rng);
    const int64_t cx = h % side, cy = (h / side) % side, cz = h / (side * side);
    const auto& d = disp[static_cast<size_t>(r)];
    const int64_t x = cx + d[0], y = cy + d[1], z = cz + d[2];
    if (x < 0 || x >= side || y < 0 || y >= side || z < 0 || z >= side) continue;
    const int64_t t = x + side * (y + side * z);
    if (t >= n_entities || t == h) continue;
    const uint64_t key = static_cast<uint64_t>(h) * n_relations + r;
    if (!seen.insert(key).second) continue;
    heads[k] = h;
    relations[k] = r;
    tails[k] = t;
    ++k;
  }
  return SKG_OK;  // split: [0, n/20) test, next n/20 valid, rest train (data_io.cpp:189-203)
}

skg_status skg_init_store(uint32_t model, int64_t n_ent, int64_t n_rel, int64_t de, int64_t dr, uint64_t seed,
                          float* entity, float* relation, float* proj, float* normals) {
  if (de < 1 || dr < 1) {
    g_err = "embedding dimensions must be at least 1";
    return SKG_ERR_CONFIG;
  }
  if (n_ent < 1 || n_rel < 1) {
    g_err = "store needs at least one entity and one relation";
    return SKG_ERR_CONFIG;
  }
  std::mt19937_64 rng(seed);
  // complex stores draw re then im per coordinate (embedding.cpp:21-25): the
  // same stream order as a real table of twice the width, bound 6 / sqrt(dim)
  const int64_t w = (model == SKG_COMPLEX || model == SKG_ROTATE) ? 2 : 1;
  fill_uniform(entity, n_ent, w * de, 6.0 / std::sqrt(static_cast<double>(de)), rng);
  fill_uniform(relation, n_rel, w * dr, 6.0 / std::sqrt(static_cast<double>(dr)), rng);
  if (model == SKG_TRANSR && proj) {
    std::memset(proj, 0, sizeof(float) * n_rel * dr * de);
    for (int64_t r = 0; r < n_rel; ++r)
      for (int64_t k = 0; k < std::min(dr, de); ++k) proj[r * dr * de + k * de + k] = 1.f;
  }
  if (model == SKG_TRANSH && normals) {
    fill_uniform(normals, n_rel, de, 6.0 / std::sqrt(static_cast<double>(de)), rng);
    for (int64_t r = 0; r < n_rel; ++r) {
      float* w = normals + r * de;
      float s = 0.f;
      for (int64_t j = 0; j < de; ++j) s += w[j] * w[j];
      const float n = std::sqrt(s);
      if (n > 0.f)
        for (int64_t j = 0; j < de; ++j) w[j] /= n;
      else
        w[0] = 1.f;
    }
  }
  return SKG_OK;
}

}  // extern "C"
