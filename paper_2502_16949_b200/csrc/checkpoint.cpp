// Binary checkpoints: the reference's SKGECKPT v1 format
// (embedding.cpp:35-125, 200-251): 8-byte magic, u32 version, u32 model tag,
// four u64 dims, then little-endian f64 row-major blocks in the order entity,
// relation, projections (TransR), normals (TransH). The engine's fp32 tables
// are written as doubles exactly like the reference's 32-bit build
// (write_block) and read back with static_cast<float> (read_block). Complex
// models (ComplEx, RotatE) carry dim interleaved (re, im) pairs per row in
// both the fp32 tables and the f64 payload (std::complex layout), so the
// header dims count complex coordinates. Host code: the caller downloads /
// uploads the device store around these calls.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/skge_b200.h"

namespace {
thread_local std::string g_err;
constexpr char kMagic[8] = {'S', 'K', 'G', 'E', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kMaxTag = 6;  // RotatE (common.hpp:62-70)
const char* kNames[] = {"transe", "transr", "transh", "toruse", "distmult", "complex", "rotate"};

bool is_complex(uint32_t tag) { return tag == 5 || tag == 6; }  // common.hpp:74-76
struct Fail {
  skg_status st;
  std::string msg;
};

void write_block(std::ofstream& out, const float* m, int64_t n) {
  std::vector<double> buf(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) buf[i] = static_cast<double>(m[i]);
  out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(sizeof(double) * buf.size()));
}

void read_block(std::ifstream& in, float* m, int64_t n) {
  std::vector<double> buf(static_cast<size_t>(n));
  in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(sizeof(double) * buf.size()));
  if (!in) throw Fail{SKG_ERR_PARSE, "checkpoint: truncated parameter block"};
  for (int64_t i = 0; i < n; ++i) m[i] = static_cast<float>(buf[i]);
}

skg_checkpoint_header read_header(std::ifstream& in, const std::string& path) {
  char magic[8] = {};
  in.read(magic, sizeof(magic));
  if (!in || std::memcmp(magic, kMagic, sizeof(kMagic)) != 0) throw Fail{SKG_ERR_PARSE, "not a checkpoint file: " + path};
  uint32_t version = 0, tag = 0;
  in.read(reinterpret_cast<char*>(&version), 4);
  if (version != kVersion) throw Fail{SKG_ERR_PARSE, "unsupported checkpoint version " + std::to_string(version)};
  in.read(reinterpret_cast<char*>(&tag), 4);
  if (tag > kMaxTag) throw Fail{SKG_ERR_PARSE, "checkpoint carries unknown model tag " + std::to_string(tag)};
  uint64_t d[4] = {};
  in.read(reinterpret_cast<char*>(d), sizeof(d));
  if (!in) throw Fail{SKG_ERR_PARSE, "checkpoint: truncated header in " + path};
  skg_checkpoint_header h{};
  h.model = tag;
  h.num_entities = static_cast<int64_t>(d[0]);
  h.num_relations = static_cast<int64_t>(d[1]);
  h.dim_entity = static_cast<int64_t>(d[2]);
  h.dim_relation = static_cast<int64_t>(d[3]);
  return h;
}

template <class F>
skg_status guard(F&& f) {
  try {
    f();
    return SKG_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.st;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SKG_ERR_PARSE;
  }
}
}  // namespace

extern "C" {

const char* skg_checkpoint_last_error(void) { return g_err.c_str(); }

skg_status skg_peek_checkpoint(const char* path, skg_checkpoint_header* out) {
  return guard([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Fail{SKG_ERR_PARSE, std::string("cannot open checkpoint: ") + path};
    *out = read_header(in, path);
  });
}

skg_status skg_save_checkpoint(const char* path, uint32_t model, int64_t num_entities, int64_t num_relations,
                               int64_t dim_entity, int64_t dim_relation, const float* entity, const float* relation,
                               const float* proj, const float* normals) {
  return guard([&] {
    if (model > kMaxTag) throw Fail{SKG_ERR_CONFIG, "unknown model tag " + std::to_string(model)};
    if ((model == 1) != (proj != nullptr))
      throw Fail{SKG_ERR_CONFIG, "projection table presence does not match the model tag"};
    if ((model == 2) != (normals != nullptr))
      throw Fail{SKG_ERR_CONFIG, "normals table presence does not match the model tag"};
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw Fail{SKG_ERR_PARSE, std::string("cannot open checkpoint for writing: ") + path};
    out.write(kMagic, sizeof(kMagic));
    out.write(reinterpret_cast<const char*>(&kVersion), 4);
    out.write(reinterpret_cast<const char*>(&model), 4);
    const uint64_t d[4] = {static_cast<uint64_t>(num_entities), static_cast<uint64_t>(num_relations),
                           static_cast<uint64_t>(dim_entity), static_cast<uint64_t>(dim_relation)};
    out.write(reinterpret_cast<const char*>(d), sizeof(d));
    const int64_t w = is_complex(model) ? 2 : 1;
    write_block(out, entity, num_entities * dim_entity * w);
    write_block(out, relation, num_relations * dim_relation * w);
    if (proj) write_block(out, proj, num_relations * dim_relation * dim_entity);
    if (normals) write_block(out, normals, num_relations * dim_entity);
    if (!out) throw Fail{SKG_ERR_PARSE, std::string("short write while saving checkpoint: ") + path};
  });
}

skg_status skg_load_checkpoint(const char* path, uint32_t expected_model, float* entity, float* relation,
                               float* proj, float* normals) {
  return guard([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Fail{SKG_ERR_PARSE, std::string("cannot open checkpoint: ") + path};
    const skg_checkpoint_header h = read_header(in, path);
    if (h.model != expected_model)
      throw Fail{SKG_ERR_CONFIG, std::string("checkpoint holds a ") + kNames[h.model] + " model, expected " +
                                     (expected_model <= kMaxTag ? kNames[expected_model] : "unknown")};
    const int64_t w = is_complex(h.model) ? 2 : 1;
    read_block(in, entity, h.num_entities * h.dim_entity * w);
    read_block(in, relation, h.num_relations * h.dim_relation * w);
    if (h.model == 1) read_block(in, proj, h.num_relations * h.dim_relation * h.dim_entity);
    if (h.model == 2) read_block(in, normals, h.num_relations * h.dim_entity);
    in.peek();
    if (!in.eof()) throw Fail{SKG_ERR_PARSE, std::string("trailing bytes after checkpoint payload: ") + path};
  });
}

}  // extern "C"
