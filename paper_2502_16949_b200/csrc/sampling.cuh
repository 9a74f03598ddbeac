// Bit-exact device replicas of the reference's two random streams:
//  - negative_sample (training.cpp:51-71): per triple one coin draw and one
//    Lemire-bounded replacement draw from std::mt19937_64(seed);
//  - the per-epoch std::shuffle (training.cpp:106-112, libstdc++
//    bits/stl_algo.h shuffle with paired draws via __gen_two_uniform_ints).
// Both read a raw MT19937-64 stream generated on device; Lemire rejections
// (libstdc++ uniform_int_dist.h _S_nd) are located exactly and the stream
// offsets shifted accordingly, so results equal the sequential reference.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "primitives.cuh"

namespace skg {

// Raw tempered outputs 0..n-1 of std::mt19937_64(seed), one CTA, in order.
void mt19937_64_generate(uint64_t seed, uint64_t* out, int64_t n, cudaStream_t s);

struct ShuffleWork {
  int64_t cap_n = 0;
  uint64_t* raw = nullptr;     // raw draws
  uint64_t* cand = nullptr;    // rejection candidates (call << 8 | shift)
  uint32_t* ncand = nullptr;   // [0] count, [1] overflow flag
  uint64_t* shifts = nullptr;  // resolved (call << 8 | shift) table
  uint32_t* nshift = nullptr;
  uint32_t* jkey = nullptr;    // swap positions j_i, then sort keys
  uint32_t* jval = nullptr;
  uint32_t* jkey_alt = nullptr;
  uint32_t* jval_alt = nullptr;
  uint32_t* jpos = nullptr;    // j_i kept unsorted
  uint32_t* gstart = nullptr;
  uint32_t* nextsame = nullptr;
  SortPlan sort;
  void reserve(int64_t n);
  void release();
  ~ShuffleWork() { release(); }
};

// order[0..n) = permutation of train_epoch for `seed_eff` (already mixed with
// the epoch: seed ^ 0x9E3779B97F4A7C15*(epoch+1)); seed_eff is read from device
// memory so the launch sequence can live in a CUDA graph.
void device_shuffle(const uint64_t* d_seed_eff, int64_t n, int32_t* order, ShuffleWork& w,
                    cudaStream_t s);
void device_iota(int32_t* order, int64_t n, cudaStream_t s);

struct NegWork {
  int64_t cap = 0;
  uint64_t* raw = nullptr;
  uint32_t* first_reject = nullptr;
  void reserve(int64_t m);
  void release();
  ~NegWork() { release(); }
};

// out_h/out_t: corrupted heads/tails (relation unchanged). Returns false on an
// internal RNG-window overflow (reported as a CUDA error by the caller).
bool device_negative_sample(const int32_t* h, const int32_t* t, int64_t m, int64_t n_ent,
                            uint64_t seed, bool avoid_self_loops, int32_t* out_h, int32_t* out_t,
                            NegWork& w, cudaStream_t s);

}  // namespace skg
