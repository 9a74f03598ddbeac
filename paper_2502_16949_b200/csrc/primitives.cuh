// Device primitives shared by the epoch planner, the shuffle and the sampler:
// an exclusive scan and a stable LSD radix sort of (u32 key, u32 value) pairs.
// Stability is what makes the transposed incidence deterministic: entries are
// generated in reference accumulation order (pos rows ascending, then neg rows
// ascending, sparse.hpp:268-272 + training.cpp:146-147) and sorting by column
// keeps that order inside every column segment.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace skg {

// Exclusive scan of n u32 values (out may alias in). Writes the grand total to
// *total when total != nullptr. Scratch is owned by the ScanPlan.
struct ScanPlan {
  std::vector<uint32_t*> level;  // per-level block partials
  std::vector<int64_t> level_n;
  int64_t capacity = 0;
  void reserve(int64_t n);
  void release();
  ~ScanPlan() { release(); }
};
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                        ScanPlan& plan, cudaStream_t s);

// Stable radix sort on the low `key_bits` bits. Returns true when the sorted
// result ended up in (keys_alt, vals_alt), false when in (keys, vals).
struct SortPlan {
  uint32_t* counts = nullptr;
  int64_t counts_cap = 0;
  ScanPlan scan;
  void reserve(int64_t n);
  void release();
  ~SortPlan() { release(); }
};
// seg_items > 0 (a multiple of the sort block, see radix_segment_ok): the
// input is a sequence of seg_items-long segments that must keep their order;
// only the low key_bits are sorted, stably, inside each segment.
bool radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits, SortPlan& plan, cudaStream_t s, int64_t seg_items = 0);
bool radix_segment_ok(int64_t seg_items, int64_t n);

// Number of kernel launches the last radix_sort_pairs / exclusive_scan_u32 issued
// on this thread (for the launch accounting bench.py reports).
int64_t kernel_launches();
void reset_kernel_launches();
void count_launch(int n = 1);

}  // namespace skg
