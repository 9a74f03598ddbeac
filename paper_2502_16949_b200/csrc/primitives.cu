// Exclusive scan and stable LSD radix sort (see primitives.cuh).
//
// Radix sort layout: each warp owns a contiguous "subtile" of kSubItems
// entries and processes it strictly in order, 32 entries at a time, ranking
// equal digits with __match_any_sync. Per-(digit, subtile) counts are laid out
// digit-major so one exclusive scan yields every subtile's output base.
#include <atomic>

#include "common.cuh"
#include "primitives.cuh"

namespace skg {

namespace {
std::atomic<int64_t> g_launches{0};

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr int kSortWarps = 8;
constexpr int kSubChunks = 32;                 // 32 chunks of 32 entries
constexpr int kSubItems = kSubChunks * 32;     // entries per warp subtile
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

__global__ void __launch_bounds__(kSortWarps * 32)
    radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift, int bits,
                      uint32_t* __restrict__ counts, int64_t nsub) {
  __shared__ uint32_t hist[kSortWarps][1 << kMaxBits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sub = static_cast<int64_t>(blockIdx.x) * kSortWarps + warp;
  const int nd = 1 << bits;
  const uint32_t mask = nd - 1;
  for (int d = lane; d < nd; d += 32) hist[warp][d] = 0;
  __syncwarp();
  if (sub < nsub) {
    const int64_t base = sub * kSubItems;
#pragma unroll 4
    for (int c = 0; c < kSubChunks; ++c) {
      const int64_t e = base + c * 32 + lane;
      if (e < n) atomicAdd(&hist[warp][(keys[e] >> shift) & mask], 1u);
    }
    __syncwarp();
    for (int d = lane; d < nd; d += 32) counts[static_cast<int64_t>(d) * nsub + sub] = hist[warp][d];
  }
}

__global__ void __launch_bounds__(kSortWarps * 32)
    radix_scatter_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                         uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n,
                         int shift, int bits, const uint32_t* __restrict__ offsets, int64_t nsub) {
  __shared__ uint32_t run[kSortWarps][1 << kMaxBits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sub = static_cast<int64_t>(blockIdx.x) * kSortWarps + warp;
  if (sub >= nsub) return;
  const int nd = 1 << bits;
  const uint32_t mask = nd - 1;
  for (int d = lane; d < nd; d += 32) run[warp][d] = offsets[static_cast<int64_t>(d) * nsub + sub];
  __syncwarp();
  const unsigned lt = lanemask_lt();
  const int64_t base = sub * kSubItems;
  for (int c = 0; c < kSubChunks; ++c) {
    const int64_t e = base + c * 32 + lane;
    const bool valid = e < n;
    const unsigned active = __ballot_sync(kFull, valid);
    if (active == 0) break;
    uint32_t key = 0, val = 0, d = 0, peers = 0;
    if (valid) {
      key = kin[e];
      val = vin[e];
      d = (key >> shift) & mask;
      peers = __match_any_sync(active, d);
      const uint32_t pos = run[warp][d] + __popc(peers & lt);
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) run[warp][d] += __popc(peers);
    __syncwarp();
  }
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
  const int64_t nsub = (n + kSubItems - 1) / kSubItems;
  const int64_t need = nsub * (1 << kMaxBits);
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

bool radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      int64_t n, int key_bits, SortPlan& plan, cudaStream_t s) {
  if (n <= 1 || key_bits <= 0) return false;
  plan.reserve(n);
  const int passes = (key_bits + kMaxBits - 1) / kMaxBits;
  const int64_t nsub = (n + kSubItems - 1) / kSubItems;
  const int blocks = ceil_div(nsub, kSortWarps);
  uint32_t *kin = keys, *vin = vals, *kout = keys_alt, *vout = vals_alt;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const int bits = (key_bits - shift + (passes - p) - 1) / (passes - p);
    radix_hist_kernel<<<blocks, kSortWarps * 32, 0, s>>>(kin, n, shift, bits, plan.counts, nsub);
    count_launch();
    SKG_LAUNCH_CHECK();
    const int64_t nc = nsub << bits;
    exclusive_scan_u32(plan.counts, plan.counts, nc, nullptr, plan.scan, s);
    radix_scatter_kernel<<<blocks, kSortWarps * 32, 0, s>>>(kin, vin, kout, vout, n, shift, bits,
                                                           plan.counts, nsub);
    count_launch();
    SKG_LAUNCH_CHECK();
    shift += bits;
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  return kin == keys_alt;
}

}  // namespace skg
