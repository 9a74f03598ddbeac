// Exclusive scan and stable LSD radix sort (see primitives.cuh).
//
// Radix sort layout: a block owns kSortWarps consecutive "subtiles" of
// kSubItems entries; each warp ranks its subtile strictly in order, 32 entries
// at a time, matching equal digits with per-bit ballots. Per-(digit, block) counts are laid out
// digit-major so one exclusive scan yields every block's output base per digit.
#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "primitives.cuh"

#ifndef SKG_PLAN_STREAMING
#define SKG_PLAN_STREAMING 1  // sort passes stream through L2 (evict-first): the concurrent minibatch chain keeps its tables and residual rows
#endif

namespace skg {

namespace {
std::atomic<int64_t> g_launches{0};

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr int kSortWarps = 8;
// Chunks of 32 entries per warp subtile: CH (template) in {1, ..., 32},
// picked per sort so small sorts still spread over every SM.
constexpr int kMaxChunks = 32;
constexpr int kMaxBits = 8;

__device__ __forceinline__ uint32_t block_exclusive_sum(uint32_t v, uint32_t* warp_tot,
                                                        uint32_t* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t t = lane < nw ? warp_tot[lane] : 0;
    uint32_t s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_tot[lane] = s - t;
    if (lane == nw - 1) *block_total = s;
  }
  __syncthreads();
  return warp_tot[warp] + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                   int64_t n,
                                                                   uint32_t* __restrict__ partial) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t total;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  block_exclusive_sum(s, warp_tot, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

// Exclusive scan of one tile (thread-contiguous items) plus the tile offset.
__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(const uint32_t* __restrict__ in,
                                                                 uint32_t* __restrict__ out,
                                                                 int64_t n,
                                                                 const uint32_t* __restrict__ offs,
                                                                 uint32_t* __restrict__ total) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t btotal;
  __shared__ uint32_t tile[kScanTile];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  // coalesced load into smem, then each thread scans kScanItems contiguous items
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    tile[k * kScanThreads + threadIdx.x] = i < n ? in[i] : 0u;
  }
  __syncthreads();
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = tile[threadIdx.x * kScanItems + k];
    s += v[k];
  }
  uint32_t run = block_exclusive_sum(s, warp_tot, &btotal) + (offs ? offs[blockIdx.x] : 0u);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    tile[threadIdx.x * kScanItems + k] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    if (i < n) out[i] = tile[k * kScanThreads + threadIdx.x];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
    *total = (offs ? offs[blockIdx.x] : 0u) + btotal;
}

// Radix pass over blocks of kSortWarps subtiles (8192 entries). The hist
// kernel counts each block's digits (counts laid out digit-major over blocks,
// so one exclusive scan gives every block's first output slot per digit). The
// scatter kernel ranks the block stably (warps own consecutive subtiles,
// chunks in order, lanes in order), stages keys/values in shared memory in
// sorted order and writes each digit's run contiguously (coalesced stores).
template <int CH>
struct SortGeom {
  static constexpr int kSubItems = CH * 32;
  static constexpr int kBlockItems = kSortWarps * kSubItems;
  static constexpr size_t kScatterSmem =
      sizeof(uint32_t) * (2 * kBlockItems + kSortWarps * (1 << kMaxBits) + 2 * (1 << kMaxBits));
};

// Lanes of `active` whose digit equals this lane's d (bits-wide): one ballot
// per digit bit, cheaper than MATCH.ANY for <= 8-bit digits.
__device__ __forceinline__ unsigned match_digit(unsigned active, uint32_t d, int bits) {
  unsigned m = active;
#pragma unroll
  for (int b = 0; b < kMaxBits; ++b) {
    if (b >= bits) break;
    const bool on = (d >> b) & 1u;
    const unsigned x = __ballot_sync(kFull, on);
    m &= on ? x : ~x;
  }
  return m;
}

// Digit-count slot of block blk: segment-major, then digit, then block within
// the segment (bpb blocks per segment; bpb = all blocks when unsegmented).
__device__ __forceinline__ int64_t count_slot(int64_t blk, int64_t bpb, int nd, int d) {
  return ((blk / bpb) * nd + d) * bpb + (blk % bpb);
}

template <int CH>
__device__ __forceinline__ void load_subtile(const uint32_t* __restrict__ src, int64_t base, int64_t n, int lane,
                                             uint32_t* r) {
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int64_t e = base + c * 32 + lane;
#if SKG_PLAN_STREAMING
    r[c] = e < n ? __ldcs(src + e) : 0u;
#else
    r[c] = e < n ? __ldg(src + e) : 0u;
#endif
  }
}

// Per-warp digit counts of the warp's subtile into h[digit] (zeroed by the caller).
template <int CH>
__device__ __forceinline__ void count_subtile(const uint32_t* k, int64_t base, int64_t n, int lane, int shift,
                                              int bits, uint32_t* h) {
  const uint32_t mask = (1u << bits) - 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const bool valid = base + c * 32 + lane < n;
    const unsigned active = __ballot_sync(kFull, valid);
    const uint32_t d = (k[c] >> shift) & mask;
    const unsigned peers = match_digit(active, d, bits);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(&h[d], static_cast<uint32_t>(__popc(peers)));
  }
}

template <int CH>
__global__ void __launch_bounds__(kSortWarps * 32)
    radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift, int bits,
                      uint32_t* __restrict__ counts, int64_t bpb) {
  __shared__ uint32_t hist[kSortWarps][1 << kMaxBits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nd = 1 << bits;
  for (int d = threadIdx.x; d < kSortWarps * (1 << kMaxBits); d += blockDim.x) (&hist[0][0])[d] = 0;
  __syncthreads();
  using G = SortGeom<CH>;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * G::kBlockItems + static_cast<int64_t>(warp) * G::kSubItems;
  uint32_t k[CH];
  load_subtile<CH>(keys, base, n, lane, k);
  count_subtile<CH>(k, base, n, lane, shift, bits, hist[warp]);
  __syncthreads();
  for (int d = threadIdx.x; d < nd; d += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) t += hist[w][d];
    counts[count_slot(blockIdx.x, bpb, nd, d)] = t;
  }
}

template <int CH>
__global__ void __launch_bounds__(kSortWarps * 32, 2)
    radix_scatter_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                         uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n,
                         int shift, int bits, const uint32_t* __restrict__ offsets, int64_t bpb) {
  using G = SortGeom<CH>;
  constexpr int kBlockItems = G::kBlockItems;
  extern __shared__ uint32_t sm_sort[];
  uint32_t* sk = sm_sort;           // [kBlockItems]
  uint32_t* sv = sk + kBlockItems;  // [kBlockItems]
  uint32_t* run = sv + kBlockItems;  // [kSortWarps][256]
  uint32_t* lstart = run + kSortWarps * (1 << kMaxBits);
  uint32_t* gbase = lstart + (1 << kMaxBits);
  __shared__ uint32_t wtot[kSortWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nd = 1 << bits;
  const uint32_t mask = nd - 1;
  const int64_t bbase = static_cast<int64_t>(blockIdx.x) * kBlockItems;
  const int64_t base = bbase + static_cast<int64_t>(warp) * G::kSubItems;
  const int bn = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(kBlockItems), n - bbase)));
  uint32_t k[CH], v[CH];
  load_subtile<CH>(kin, base, n, lane, k);
  load_subtile<CH>(vin, base, n, lane, v);
  for (int d = threadIdx.x; d < kSortWarps * (1 << kMaxBits); d += blockDim.x) run[d] = 0;
  __syncthreads();
  count_subtile<CH>(k, base, n, lane, shift, bits, run + warp * (1 << kMaxBits));
  __syncthreads();
  {  // thread d: block count of digit d, exclusive scan over digits, per-warp bases
    const int d = threadIdx.x;  // blockDim == 256 == max digits
    uint32_t c = 0;
    if (d < nd)
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) c += run[w * (1 << kMaxBits) + d];
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint32_t t = lane < kSortWarps ? wtot[lane] : 0u;
      uint32_t sc = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, sc, o);
        if (lane >= o) sc += y;
      }
      if (lane < kSortWarps) wtot[lane] = sc - t;
    }
    __syncthreads();
    if (d < nd) {
      const uint32_t ls = wtot[warp] + x - c;
      lstart[d] = ls;
      gbase[d] = offsets[count_slot(blockIdx.x, bpb, nd, d)];
      uint32_t r = ls;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t cw = run[w * (1 << kMaxBits) + d];
        run[w * (1 << kMaxBits) + d] = r;
        r += cw;
      }
    }
  }
  __syncthreads();
  // stable ranking of this warp's subtile into the block's sorted staging
  uint32_t* wrun = run + warp * (1 << kMaxBits);
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const bool valid = base + c * 32 + lane < n;
    const unsigned active = __ballot_sync(kFull, valid);
    const uint32_t d = (k[c] >> shift) & mask;
    const unsigned peers = match_digit(active, d, bits);
    if (valid) {
      const uint32_t pos = wrun[d] + __popc(peers & lt);
      sk[pos] = k[c];
      sv[pos] = v[c];
    }
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wrun[d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // coalesced write-out: entry j of the sorted block -> gbase[d] + (j - lstart[d])
  for (int j = threadIdx.x; j < bn; j += blockDim.x) {
    const uint32_t key = sk[j];
    const uint32_t d = (key >> shift) & mask;
    const uint32_t pos = gbase[d] + (static_cast<uint32_t>(j) - lstart[d]);
#if SKG_PLAN_STREAMING
    __stcs(kout + pos, key);
    __stcs(vout + pos, sv[j]);
#else
    kout[pos] = key;
    vout[pos] = sv[j];
#endif
  }
}

// Chunks per warp for an n-entry sort: about two blocks per SM, 1..32.
int sort_chunks(int64_t n) {
  int ch = 1;
  while (ch < kMaxChunks && n / (static_cast<int64_t>(kSortWarps) * 32 * ch) > 2 * 148) ch <<= 1;
  return ch;
}

}  // namespace

int64_t kernel_launches() { return g_launches.load(); }
void reset_kernel_launches() { g_launches.store(0); }
void count_launch(int n) { g_launches.fetch_add(n); }

void ScanPlan::reserve(int64_t n) {
  if (n <= capacity) return;
  release();
  int64_t m = n;
  while (m > kScanTile) {
    m = (m + kScanTile - 1) / kScanTile;
    uint32_t* p = nullptr;
    SKG_CUDA(cudaMalloc(&p, sizeof(uint32_t) * (m + 1)));
    level.push_back(p);
    level_n.push_back(m);
  }
  capacity = n;
}

void ScanPlan::release() {
  for (auto* p : level) cudaFree(p);
  level.clear();
  level_n.clear();
  capacity = 0;
}

namespace {
void scan_rec(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, ScanPlan& plan,
              size_t lvl, cudaStream_t s) {
  const int nb = ceil_div(n, kScanTile);
  if (nb <= 1) {
    scan_tile_kernel<<<1, kScanThreads, 0, s>>>(in, out, n, nullptr, total);
    count_launch();
    SKG_LAUNCH_CHECK();
    return;
  }
  uint32_t* part = plan.level.at(lvl);
  scan_reduce_kernel<<<nb, kScanThreads, 0, s>>>(in, n, part);
  count_launch();
  SKG_LAUNCH_CHECK();
  scan_rec(part, part, nb, nullptr, plan, lvl + 1, s);
  scan_tile_kernel<<<nb, kScanThreads, 0, s>>>(in, out, n, part, total);
  count_launch();
  SKG_LAUNCH_CHECK();
}
}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total,
                        ScanPlan& plan, cudaStream_t s) {
  if (n <= 0) {
    if (total) SKG_CUDA(cudaMemsetAsync(total, 0, sizeof(uint32_t), s));
    return;
  }
  plan.reserve(n);
  scan_rec(in, out, n, total, plan, 0, s);
}

void SortPlan::reserve(int64_t n) {
  // segmented sorts pad the last segment with empty blocks: at most 2x blocks.
  // The block count is not monotone in n (a longer sort uses longer chunks), so
  // size for every n' <= n: the largest n' of each chunk length up to n's.
  int64_t nblk = 0;
  const int top = sort_chunks(n);
  for (int ch = 1; ch <= top; ch <<= 1) {
    const int64_t bi = static_cast<int64_t>(kSortWarps) * 32 * ch;
    const int64_t m = ch == top ? n : std::min<int64_t>(n, (2 * 148 + 1) * bi - 1);
    nblk = std::max<int64_t>(nblk, 2 * ((m + bi - 1) / bi));
  }
  const int64_t need = nblk * (1 << kMaxBits);
  if (need > counts_cap) {
    if (counts) cudaFree(counts);
    SKG_CUDA(cudaMalloc(&counts, sizeof(uint32_t) * need));
    counts_cap = need;
  }
  scan.reserve(need);
}

void SortPlan::release() {
  if (counts) cudaFree(counts);
  counts = nullptr;
  counts_cap = 0;
  scan.release();
}

namespace {
template <int CH>
bool sort_t(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n, int key_bits,
            SortPlan& plan, cudaStream_t s, int64_t seg_items) {
  using G = SortGeom<CH>;
  static bool configured = false;
  if (!configured) {
    SKG_CUDA(cudaFuncSetAttribute(radix_scatter_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(G::kScatterSmem)));
    configured = true;
  }
  const int64_t nblk = (n + G::kBlockItems - 1) / G::kBlockItems;
  const bool seg = seg_items > 0 && seg_items % G::kBlockItems == 0;
  const int64_t bpb = seg ? std::min<int64_t>(seg_items / G::kBlockItems, nblk) : nblk;
  const int64_t slots = (nblk + bpb - 1) / bpb * bpb;  // blocks incl. the last segment's empty tail
  const int passes = (key_bits + kMaxBits - 1) / kMaxBits;
  uint32_t *kin = keys, *vin = vals, *kout = keys_alt, *vout = vals_alt;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const int bits = (key_bits - shift + (passes - p) - 1) / (passes - p);
    radix_hist_kernel<CH><<<static_cast<unsigned>(slots), kSortWarps * 32, 0, s>>>(kin, n, shift, bits, plan.counts,
                                                                                 bpb);
    count_launch();
    SKG_LAUNCH_CHECK();
    exclusive_scan_u32(plan.counts, plan.counts, slots << bits, nullptr, plan.scan, s);
    radix_scatter_kernel<CH><<<static_cast<unsigned>(nblk), kSortWarps * 32, G::kScatterSmem, s>>>(
        kin, vin, kout, vout, n, shift, bits, plan.counts, bpb);
    count_launch();
    SKG_LAUNCH_CHECK();
    shift += bits;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  return kin == keys_alt;
}
}  // namespace

bool radix_segment_ok(int64_t seg_items, int64_t n) {
  return seg_items > 0 && seg_items % (static_cast<int64_t>(kSortWarps) * 32 * sort_chunks(n)) == 0;
}

bool radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits, SortPlan& plan, cudaStream_t s, int64_t seg_items) {
  if (n <= 1 || key_bits <= 0) return false;
  plan.reserve(n);  // no-op once the owner reserved (graph capture forbids allocation)
  switch (sort_chunks(n)) {
    case 1: return sort_t<1>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
    case 2: return sort_t<2>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
    case 4: return sort_t<4>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
    case 8: return sort_t<8>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
    case 16: return sort_t<16>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
    default: return sort_t<32>(keys, vals, keys_alt, vals_alt, n, key_bits, plan, s, seg_items);
  }
}

}  // namespace skg
