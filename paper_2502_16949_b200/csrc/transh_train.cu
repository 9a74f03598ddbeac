// TransH training step on relation-grouped tiles (sm_100a), d = 128.
//
// The epoch plan's relation segments list a relation's positive rows, then the
// same pairs' negatives; a CTA owns 64 such (pos, neg) pairs = 128 rows of ONE
// relation r (models.cpp:158-199, models.hpp:99-113), so the normal w_r and
// the relation row d_r are loaded once per tile and the relation-side
// gradients are summed inside the tile:
//   u = h - t, wu = w.u, v = (u + d_r) - wu w          (hyperplane_forward)
//   score = ||v|| in the reference's squared_sum / abs_sum order, pair hinge
//   dz = dir(v) * up, dzw = dz.w
//   du  = dz - dzw w          -> res_u rows (sorted entity segments, no atomics)
//   sum dz, sum (dzw u + wu dz) -> one partial per tile (relation gradient and
//                                  negated normal gradient, models.hpp:112)
// The CTA that finishes a relation's last tile adds its tile partials in tile
// order and applies SGD; the normals are then renormalized (embedding.cpp:181-189). Compared with
// the row-wise path (ht.cu) no dz / nrm rows go through HBM and w_r, d_r are
// not re-gathered per row. Dot products use a fixed warp tree (the reference
// reduces them with Eigen's redux; TransH parity is tolerance-only).
#include <algorithm>

#include "common.cuh"
#include "tc.cuh"
#include "ht.cuh"
#include "plan.cuh"
#include "primitives.cuh"
#include "refmath.cuh"

namespace skg {

namespace {

constexpr int kD = 128;
#ifndef SKG_TRANSH_PAIRS
#define SKG_TRANSH_PAIRS 32
#endif
constexpr int kPairs = SKG_TRANSH_PAIRS;
constexpr int kRows = 2 * kPairs;
#ifndef SKG_TRANSH_RPW
#define SKG_TRANSH_RPW 4
#endif
constexpr int kRowsPerWarp = SKG_TRANSH_RPW;  // rows 0 .. RPW/2-1: positives of the warp's pairs, then their negatives
constexpr int kHalf = kRowsPerWarp / 2;       // pairs per compute warp
constexpr int kLanesPerRow = 32 / kRowsPerWarp;
constexpr int kLaneRowShift = kRowsPerWarp == 8 ? 2 : 3;
static_assert(kRowsPerWarp == 4 || kRowsPerWarp == 8, "4 or 8 rows per compute warp");
static_assert(kPairs == 32, "a tile is 32 pairs");
constexpr int kStride = kD;        // staged rows (float4 row reads are conflict-free)

constexpr int kMaxRelSeg = 1024;  // relation segments per batch handled in shared memory

struct TArgs {
  FwdArgs f;
  const uint32_t* ent_val;
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* seg_base;
  int batch;
  int64_t mt;                 // tile capacity of `partial`
  float* partial;             // [tile][2][kD]
  uint32_t* info;             // [0] relation runs, [1] tiles, then per run {r, first tile, end tile}
  float* rel;                 // relation table (SGD), or the relation gradient sink
  const float* lr;
  float* nrm_sink;            // data parallel: normals gradient sink (null: SGD in place)
  int64_t R;
  // the epoch plan's precomputed tiles of this batch (transh_tile_plan), or null: chase them here
  const int4* tp_meta;   // per tile {relation run k, relation r, pairs np, 0}
  const int4* tp_rows;   // per tile x pair {h, t, neg h, neg t}
  const int32_t* tp_pos; // per tile x pair: batch position (-1: padding)
};

__device__ __forceinline__ float4 f4sub(float4 a, float4 b) {
  return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z), __fsub_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4scale(float s, float4 a) {
  return make_float4(__fmul_rn(s, a.x), __fmul_rn(s, a.y), __fmul_rn(s, a.z), __fmul_rn(s, a.w));
}
__device__ __forceinline__ float f4dot(float4 a, float4 b) {
  float acc = __fmul_rn(a.x, b.x);
  acc = fmaf(a.y, b.y, acc);
  acc = fmaf(a.z, b.z, acc);
  return fmaf(a.w, b.w, acc);
}

template <bool L2>
__device__ __forceinline__ float dirf(float v, float sc) {
  return L2 ? __fmul_rn(v, sc) : (v > 0.f ? sc : (v < 0.f ? -sc : 0.f));
}
template <bool L2>
__device__ __forceinline__ float4 dir4(float4 v, float sc) {
  return make_float4(dirf<L2>(v.x, sc), dirf<L2>(v.y, sc), dirf<L2>(v.z, sc), dirf<L2>(v.w, sc));
}

// Relation tiles of the batch, enumerated by warp 0 of every CTA: the batch's
// relation segments lead its segment list (relation column keys sort first);
// first[k] = first tile of relation segment k, first[nrel] = tile count.
struct RelTiles {
  uint32_t first[kMaxRelSeg + 1];
  uint32_t seg[kMaxRelSeg];
  uint32_t nrel;
};

__device__ void enumerate_rel_tiles(const TArgs& a, RelTiles& rt) {
  const int lane = threadIdx.x & 31;
  const uint32_t s0 = a.seg_base[a.batch], s1 = a.seg_base[a.batch + 1];
  uint32_t carry = 0, k0 = 0;
  for (uint32_t base = s0; base < s1 && k0 < kMaxRelSeg; base += 32) {
    const uint32_t s = base + lane;
    const uint32_t col = s < s1 ? __ldg(a.seg_col + s) : kDummyCol;
    const bool rel = col >= static_cast<uint32_t>(a.f.N) && col != kDummyCol;
    uint32_t n = 0;
    if (rel) n = ((__ldg(a.seg_start + s + 1) - __ldg(a.seg_start + s)) / 2 + kPairs - 1) / kPairs;
    const unsigned m = __ballot_sync(kFull, rel);
    const int nr = __popc(~m) == 0 ? 32 : __ffs(~m) - 1;  // relation segments form a prefix
    uint32_t x = lane < nr ? n : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane < nr && k0 + lane < kMaxRelSeg) {
      rt.first[k0 + lane] = carry + x - n;
      rt.seg[k0 + lane] = s;
    }
    carry += __shfl_sync(kFull, x, 31);
    k0 += static_cast<uint32_t>(nr);
    if (nr < 32) break;
  }
  if (lane == 0) {
    rt.nrel = min(k0, static_cast<uint32_t>(kMaxRelSeg));
    rt.first[rt.nrel] = carry;
  }
}

__device__ __forceinline__ uint32_t rel_of_tile(const RelTiles& rt, uint32_t t) {
  uint32_t lo = 0, hi = rt.nrel;
  while (lo + 1 < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rt.first[mid] <= t) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Pipelined relation tiles. One persistent CTA per SM walks a contiguous range
// of the batch's tiles [T b / G, T (b + 1) / G): a loader warp chases each
// tile's row ids and streams the head / tail rows into a kStages-deep shared
// ring with 16-byte cp.async (no registers held across the copy latency); 8
// compute warps own 4 (pos, neg) pairs each, so a pair's hinge never leaves
// its warp. Relation-side sums are accumulated per warp over the CTA's run of
// one relation and flushed once per (CTA, relation run) to slot b + k (unique:
// CTA ranges are ordered); the run that completes a relation sums the slots in
// CTA order, applies SGD to d_r / w_r and renormalizes w_r.
constexpr int kCompute = kPairs / kHalf;       // compute warps
#ifndef SKG_TRANSH_LOADERS
#define SKG_TRANSH_LOADERS 4
#endif
constexpr int kLoaders = SKG_TRANSH_LOADERS;   // copy warps (one warp's cp.async stream cannot fill an SM's L2 bandwidth)
constexpr int kPipeThreads = (kCompute + kLoaders) * 32;
constexpr int kLoaderWarp = kCompute;          // first loader: enumerates the tiles, writes the stage metadata
#ifndef SKG_TH_STAGES
#define SKG_TH_STAGES 2  // 2: the ring leaves shared memory for plan-branch blocks on the same SM (CTAs start together)
#endif
constexpr int kStages = SKG_TH_STAGES;
static_assert(kPairs % kLoaders == 0, "loaders split a tile's pairs evenly");

struct PipeMeta {
  int4 rows[kRows];  // warp-major: rows 8w..8w+3 = pos of pairs 4w..4w+3, 8w+4.. = their negatives
  float wr[kD], dr[kD];  // w_r and d_r rows (copied with the stage)
  int k, r, np;
};
struct PipeSmem {
  float H[kStages][kRows * kStride];  // head rows (v overwrites them)
  float Tl[kStages][kRows * kStride]; // tail rows
  PipeMeta meta[kStages];
  float4 wpart[kCompute][2][32];
  RelTiles rt;
  float wl[kCompute];
  uint64_t full[kStages], empty[kStages];
  uint32_t ntile, t0, T;
  int last_cta;
};

// CTA b's tiles start at range_start(b): T b / G when every CTA gets a tile,
// else one tile each for b < T, so the CTAs meeting a relation are always a
// contiguous run of non-empty ranges.
__device__ __forceinline__ uint32_t range_start(uint32_t b, uint32_t T, uint32_t G) {
  return T >= G ? static_cast<uint32_t>((static_cast<uint64_t>(T) * b) / G) : min(b, T);
}
// Transpose-reduce of kRowsPerWarp per-lane partials (one per row) over the
// warp in a fixed tree: each level hands half of the rows to the partner lane,
// then the remaining lanes of a row are summed; afterwards p[0] on lane L holds
// row (L >> kLaneRowShift)'s total, bitwise equal on that row's lanes.
// 9 (8 rows) / 6 (4 rows) shuffles instead of rows x 5.
__device__ __forceinline__ void warp_reduce_rows(float (&p)[kRowsPerWarp]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int n = kRowsPerWarp / 2, m = 16; n >= 1; n >>= 1, m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int q = 0; q < n; ++q) {
      const float send = up ? p[q] : p[q + n];
      const float keep = up ? p[q + n] : p[q];
      p[q] = __fadd_rn(keep, __shfl_xor_sync(kFull, send, m));
    }
  }
#pragma unroll
  for (int m = kLanesPerRow / 2; m >= 1; m >>= 1) p[0] = __fadd_rn(p[0], __shfl_xor_sync(kFull, p[0], m));
}

// embedding.cpp:181-189 on one normal, by a warp (normals_renorm_kernel's order:
// lane-strided squares, then the warp tree)
__device__ __forceinline__ void renorm_normal(float* normals, int64_t r, int d, int lane, uint32_t* err) {
  float* row = normals + r * d;
  float x[kD / 32];
  float ss = 0.f;
#pragma unroll
  for (int q = 0; q < kD / 32; ++q) {
    x[q] = lane + 32 * q < d ? row[lane + 32 * q] : 0.f;
    ss = __fadd_rn(ss, __fmul_rn(x[q], x[q]));
  }
  const float nn = __fsqrt_rn(warp_sum_bcast(ss));
  if (!(nn > 0.f)) {
    if (lane == 0 && atomicCAS(&err[0], 0u, static_cast<uint32_t>(kErrNormalCollapsed)) == 0u)
      err[2] = static_cast<uint32_t>(r);
    return;
  }
#pragma unroll
  for (int q = 0; q < kD / 32; ++q)
    if (lane + 32 * q < d) row[lane + 32 * q] = __fdiv_rn(x[q], nn);
}

__device__ __forceinline__ uint32_t cta_of_tile(uint32_t t, uint32_t T, uint32_t G) {  // max j: range_start(j) <= t
  return T >= G ? static_cast<uint32_t>(((static_cast<uint64_t>(t) + 1) * G - 1) / T) : t;
}

// Debug phase stamps (globaltimer ns) of one chosen minibatch, off unless
// enabled through skg_debug_transh_trace: [CTA < 160][event < 32].
constexpr int kThTrCtas = 160, kThTrEvents = 32;
__device__ unsigned long long g_thtrace[kThTrCtas * kThTrEvents];
__device__ int g_thtrace_on;
__device__ __forceinline__ void th_stamp(bool on, int ev) {
  if (on && blockIdx.x < kThTrCtas && ev < kThTrEvents) stamp_now(&g_thtrace[blockIdx.x * kThTrEvents + ev]);
}

template <bool L2, bool FULL>  // FULL: d == kD (compile-time row strides)
__global__ void __launch_bounds__(kPipeThreads, 1) transh_pipe_kernel(const TArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  PipeSmem& S = *reinterpret_cast<PipeSmem*>(smem_raw);
  const FwdArgs& f = a.f;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (f.stamp_start && blockIdx.x == 0 && tid == 0) stamp_now(f.stamp_start);
  const bool alive = f.err[0] == 0;
  const uint32_t G = gridDim.x;
  const bool tr = g_thtrace_on == f.batch + 1;
  if (tid == 0) th_stamp(tr, 0);
  const int d = FULL ? kD : f.de, d4 = d >> 2;  // row width (<= kD); staged rows are zero-padded to kD columns
  if constexpr (!FULL) if (d < kD && warp < kCompute) {  // the copies never write the padding: clear it once
    for (int i = tid; i < kStages * 2 * kRows * (kD - d) / 4; i += kCompute * 32) {
      const int c4 = d4 + i % (kD / 4 - d4), rr = i / (kD / 4 - d4);  // rr over stages x {H, T} x rows
      const int st = rr / (2 * kRows), ht = (rr / kRows) & 1, row = rr % kRows;
      reinterpret_cast<float4*>((ht ? S.Tl[st] : S.H[st]) + row * kStride)[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int i = tid; i < kStages * 2 * (kD - d); i += kCompute * 32) {
      const int c = d + i % (kD - d), rr = i / (kD - d);
      (rr & 1 ? S.meta[rr >> 1].dr : S.meta[rr >> 1].wr)[c] = 0.f;
    }
  }
  if (warp == kLoaderWarp && a.tp_meta) {  // tiles precomputed by the plan (a.info is the plan's)
    if (lane == 0) {
      const uint32_t T = alive ? a.info[1] : 0u;
      const uint32_t t0 = range_start(blockIdx.x, T, G), t1 = range_start(blockIdx.x + 1, T, G);
      S.T = T;
      S.t0 = t0;
      S.ntile = t1 - t0;
      for (int i = 0; i < kStages; ++i) {
        tc::mbar_init(&S.full[i], 32 * kLoaders + 1);
        tc::mbar_init(&S.empty[i], kCompute);
      }
      tc::fence_barrier_init();
    }
  } else if (warp == kLoaderWarp) {
    if (alive) enumerate_rel_tiles(a, S.rt);
    __syncwarp();
    if (blockIdx.x == 0 && alive)
      for (uint32_t q = lane; q < S.rt.nrel; q += 32) {
        a.info[4 + 3 * q] = static_cast<uint32_t>(__ldg(a.seg_col + S.rt.seg[q]) - static_cast<uint32_t>(a.f.N));
        a.info[5 + 3 * q] = S.rt.first[q];
        a.info[6 + 3 * q] = S.rt.first[q + 1];
      }
    if (lane == 0) {
      const uint32_t T = alive ? static_cast<uint32_t>(min(static_cast<int64_t>(S.rt.first[S.rt.nrel]), a.mt)) : 0u;
      const uint32_t t0 = range_start(blockIdx.x, T, G), t1 = range_start(blockIdx.x + 1, T, G);
      S.T = T;
      S.t0 = t0;
      S.ntile = t1 - t0;
      if (blockIdx.x == 0 && alive) {  // the batch's relation runs, for transh_rel_finalize_kernel
        a.info[0] = S.rt.nrel;
        a.info[1] = T;
      }
      for (int i = 0; i < kStages; ++i) {
        tc::mbar_init(&S.full[i], 32 * kLoaders + 1);  // cp.async arrivals of every loader lane + the metadata arrive
        tc::mbar_init(&S.empty[i], kCompute);
      }
      tc::fence_barrier_init();
    }
  }
  __syncthreads();
  if (tid == 0) th_stamp(tr, 1);
  const uint32_t ntile = S.ntile, t0 = S.t0;
  uint32_t pend = 0;

  if (warp >= kLoaderWarp) {
    // ------------------------------------------------------------ loaders
    // Row ids of kChase tiles are chased together (lane = pair; their
    // dependent ent_val -> pair record loads overlap), then each tile's rows
    // are copied into its stage as the stage frees up. Every loader warp
    // chases the same ids (L1 hits) and copies kPairs / kLoaders pairs.
    const int lw = warp - kLoaderWarp;
    const bool lead = lw == 0;
    constexpr int kChase = 4;
    for (uint32_t g = 0; g < ntile; g += kChase) {
      int pos[kChase], np[kChase];
      uint32_t kq[kChase];
      int rr_[kChase];
      int4 pr_[kChase];
      if (a.tp_meta) {  // the plan's tile records: one load per pair, no chase
#pragma unroll
        for (int c = 0; c < kChase; ++c) {
          pos[c] = -1;
          np[c] = 0;
          kq[c] = 0;
          rr_[c] = 0;
          pr_[c] = make_int4(0, 0, 0, 0);
          if (g + c < ntile) {
            const uint32_t t = t0 + g + c;
            const int4 mt = __ldg(a.tp_meta + t);
            kq[c] = static_cast<uint32_t>(mt.x);
            rr_[c] = mt.y;
            np[c] = mt.z;
            pos[c] = __ldg(a.tp_pos + static_cast<size_t>(t) * kPairs + lane);
            pr_[c] = __ldg(a.tp_rows + static_cast<size_t>(t) * kPairs + lane);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kChase; ++c) {
        if (a.tp_meta) break;
        pos[c] = -1;
        np[c] = 0;
        kq[c] = 0;
        if (g + c < ntile) {
          const uint32_t t = t0 + g + c;
          kq[c] = rel_of_tile(S.rt, t);
          const uint32_t sq = S.rt.seg[kq[c]], pq = (t - S.rt.first[kq[c]]) * kPairs;
          const uint32_t e0 = __ldg(a.seg_start + sq), len = __ldg(a.seg_start + sq + 1) - e0;
          np[c] = static_cast<int>(min(static_cast<uint32_t>(kPairs), len / 2 - pq));
          if (lane < np[c]) pos[c] = static_cast<int>(__ldg(a.ent_val + e0 + pq + lane) & 0x7fffffffu);
        }
      }
      if (lead && lane == 0 && g == 0) th_stamp(tr, 2);
      int4 pr[kChase], ng[kChase];
#pragma unroll
      for (int c = 0; c < kChase; ++c) {
        pr[c] = make_int4(0, 0, -1, 0);
        ng[c] = make_int4(0, 0, -1, 0);
        if (pos[c] >= 0 && a.tp_meta) {
          pr[c] = make_int4(pr_[c].x, pr_[c].y, pos[c], 0);
          ng[c] = make_int4(pr_[c].z, pr_[c].w, pos[c] + f.B, 0);
        } else if (pos[c] >= 0) {
          int h, tt, nh, nt;
          if (f.pair_ht) {
            const int4 x = __ldg(f.pair_ht + pos[c]);
            h = x.x, tt = x.y, nh = x.z, nt = x.w;
          } else {
            const int id = __ldg(f.order + pos[c]);
            h = __ldg(f.H + id), tt = __ldg(f.T + id), nh = __ldg(f.NH + id), nt = __ldg(f.NT + id);
          }
          pr[c] = make_int4(h, tt, pos[c], 0);
          ng[c] = make_int4(nh, nt, pos[c] + f.B, 0);
        }
      }
#pragma unroll
      for (int c = 0; c < kChase; ++c) {
        const uint32_t i = g + c;
        if (i >= ntile) break;
        const int s = static_cast<int>(i % kStages);
        if (i >= kStages) tc::mbar_wait(&S.empty[s], ((i / kStages) - 1) & 1);
        PipeMeta& M = S.meta[s];
        if (lead) {
          const int mp = kRowsPerWarp * (lane / kHalf) + lane % kHalf;  // warp-major slot of pair `lane`
          M.rows[mp] = pr[c];
          M.rows[mp + kHalf] = ng[c];
          const int64_t r = a.tp_meta ? rr_[c] : static_cast<int64_t>(__ldg(a.seg_col + S.rt.seg[kq[c]])) - f.N;
          if (lane == 0) {
            M.k = static_cast<int>(kq[c]);
            M.r = static_cast<int>(r);
            M.np = np[c];
          }
          if (lane < d4) {
            tc::cp_async16(M.wr + 4 * lane, f.normals + r * d + 4 * lane);
            tc::cp_async16(M.dr + 4 * lane, f.X + f.N * d + r * d + 4 * lane);
          }
        }
        // rows: lane = 16-byte chunk of a 512-byte row
        float* Hs = S.H[s];
        float* Ts = S.Tl[s];
#pragma unroll 4
        for (int p = lw * (kPairs / kLoaders); p < (lw + 1) * (kPairs / kLoaders); ++p) {
          const int hp = __shfl_sync(kFull, pr[c].x, p), tp = __shfl_sync(kFull, pr[c].y, p);
          const int hn = __shfl_sync(kFull, ng[c].x, p), tn = __shfl_sync(kFull, ng[c].y, p);
          const int m = kRowsPerWarp * (p / kHalf) + p % kHalf;
          if (lane < d4) {  // columns >= d stay zero (cleared once at kernel start)
            tc::cp_async16(Hs + m * kStride + 4 * lane, f.X + static_cast<size_t>(hp) * d + 4 * lane);
            tc::cp_async16(Ts + m * kStride + 4 * lane, f.X + static_cast<size_t>(tp) * d + 4 * lane);
            tc::cp_async16(Hs + (m + kHalf) * kStride + 4 * lane, f.X + static_cast<size_t>(hn) * d + 4 * lane);
            tc::cp_async16(Ts + (m + kHalf) * kStride + 4 * lane, f.X + static_cast<size_t>(tn) * d + 4 * lane);
          }
        }
        tc::cp_async_mbar_arrive(&S.full[s]);
        __syncwarp();
        if (lead && lane == 0) {
          tc::mbar_arrive(&S.full[s]);
          if (i < 4) th_stamp(tr, 3 + static_cast<int>(i));
        }
      }
    }
  } else {
    // ------------------------------------------------------------ compute
    const int m0 = warp * kRowsPerWarp;
    float lw = 0.f;  // this warp's loss terms, tile order
    float4 acc_dz = make_float4(0.f, 0.f, 0.f, 0.f), acc_n = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 w = make_float4(0.f, 0.f, 0.f, 0.f), drv = w;
    int run = -1, run_r = 0;
    // (CTA, run) flush: warps in order -> slot b + k; the run completing relation
    // k sums the slots in CTA order and applies SGD (+ renormalization of w_r)
    auto flush = [&]() {
      S.wpart[warp][0][lane] = acc_dz;
      S.wpart[warp][1][lane] = acc_n;
      tc::named_sync(1, kCompute * 32);
      if (tid < 64) {
        const int which = tid >> 5;
        float4 sum = S.wpart[0][which][lane];
#pragma unroll
        for (int q = 1; q < kCompute; ++q) sum = f4add(sum, S.wpart[q][which][lane]);
        reinterpret_cast<float4*>(a.partial + (static_cast<size_t>(blockIdx.x + run) * 2 + which) * kD)[lane] = sum;
      }
      tc::named_sync(1, kCompute * 32);  // wpart free for the next run
      acc_dz = make_float4(0.f, 0.f, 0.f, 0.f);
      acc_n = acc_dz;
    };
    for (uint32_t i = 0; i < ntile; ++i) {
      const int s = static_cast<int>(i % kStages);
      tc::mbar_wait(&S.full[s], (i / kStages) & 1);
      if (tid == 0 && i < 4) th_stamp(tr, 7 + static_cast<int>(i));
      const PipeMeta& M = S.meta[s];
      if (M.k != run) {
        if (run >= 0) flush();
        run = M.k;
        run_r = M.r;
        w = reinterpret_cast<const float4*>(M.wr)[lane];
        drv = reinterpret_cast<const float4*>(M.dr)[lane];
      }
      const int np = M.np;
      float* Hs = S.H[s] + m0 * kStride;
      const float* Ts = S.Tl[s] + m0 * kStride;
      // ---- u, wu, v for the warp's 8 rows, all in registers (lane = 4 columns)
      float4 u[kRowsPerWarp], v[kRowsPerWarp];
      float wu[kRowsPerWarp];
      int rz[kRowsPerWarp];  // incidence row of each row (-1: padding)
      {
        float part[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          const float4 xh = *reinterpret_cast<const float4*>(Hs + q * kStride + 4 * lane);
          const float4 xt = *reinterpret_cast<const float4*>(Ts + q * kStride + 4 * lane);
          rz[q] = M.rows[m0 + q].z;
          u[q] = f4sub(xh, xt);
        }
        // everything this warp needs from the stage is in registers: release it
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&S.empty[s]);
        if (tid == 0 && i < 2) th_stamp(tr, 19 + 4 * static_cast<int>(i));
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          if (rz[q] < 0) u[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          part[q] = f4dot(w, u[q]);
        }
        warp_reduce_rows(part);
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          wu[q] = __shfl_sync(kFull, part[0], kLanesPerRow * q);
          v[q] = f4sub(f4add(u[q], drv), f4scale(wu[q], w));
        }
      }
      if (tid == 0 && i < 2) th_stamp(tr, 20 + 4 * static_cast<int>(i));
      // ---- score: squared / absolute sums reduced in a fixed tree (lane 4q.. holds row q)
      float ssum;
      unsigned nfbits = 0;
      {
        float part[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          const float4 x = v[q];
          if (nonfinite(x.x) | nonfinite(x.y) | nonfinite(x.z) | nonfinite(x.w)) nfbits |= 1u << q;
          part[q] = __fadd_rn(__fadd_rn(norm_term<L2>(x.x), norm_term<L2>(x.y)),
                              __fadd_rn(norm_term<L2>(x.z), norm_term<L2>(x.w)));
        }
        warp_reduce_rows(part);
        ssum = part[0];
      }
      nfbits = __reduce_or_sync(kFull, nfbits);
      const int qrow = lane >> kLaneRowShift;     // this lane's row (its lanes hold identical sums)
      const float score = L2 ? __fsqrt_rn(ssum) : ssum;
      // ---- pair hinge (training.cpp:73-94): rows 0-3 pos of pairs 4w..4w+3, rows 4-7 their negatives
      const int jq = qrow % kHalf;
      const int pidx = kHalf * warp + jq;
      const float sother = __shfl_xor_sync(kFull, score, 16);
      const bool is_pos = qrow < kHalf;
      const bool valid = pidx < np;
      const float term = valid ? (is_pos ? __fsub_rn(__fadd_rn(f.margin, score), sother)
                                         : __fsub_rn(__fadd_rn(f.margin, sother), score))
                               : 0.f;
      const bool act = valid && term > 0.f;
      const float up = act ? (is_pos ? f.unit : -f.unit) : 0.f;
      const float sc = act ? (L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(ssum, kNormEpsF))) : up) : 0.f;
      if (lane % kLanesPerRow == 0) {
        int row2 = rz[0];
#pragma unroll
        for (int q = 1; q < kRowsPerWarp; ++q) row2 = qrow == q ? rz[q] : row2;
        if (valid) f.scal[row2] = act ? 1.f : 0.f;
        if (valid && ((nfbits >> qrow) & 1u) && (L2 || act)) pend |= kPendEntity;
      }
      {
        float tk = (act && is_pos && lane % kLanesPerRow == 0) ? term : 0.f;  // first lane of each pos row
#pragma unroll
        for (int o = 8; o >= kLanesPerRow; o >>= 1) tk = __fadd_rn(tk, __shfl_down_sync(kFull, tk, o));
        lw = __fadd_rn(lw, __shfl_sync(kFull, tk, 0));
      }
      if (tid == 0 && i < 2) th_stamp(tr, 21 + 4 * static_cast<int>(i));
      // ---- backward rows (hyperplane_backward, models.hpp:106-113)
      const unsigned amask = __ballot_sync(kFull, act);  // row q active <=> bit kLanesPerRow * q
      if (amask) {
        float4 dz[kRowsPerWarp];
        float part[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          const float scq = __shfl_sync(kFull, sc, kLanesPerRow * q);
          dz[q] = ((amask >> (kLanesPerRow * q)) & 1u) ? dir4<L2>(v[q], scq) : make_float4(0.f, 0.f, 0.f, 0.f);
          part[q] = f4dot(dz[q], w);
        }
        warp_reduce_rows(part);
        if (tid == 0 && i < 2) th_stamp(tr, 22 + 4 * static_cast<int>(i));
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          const float dzw = __shfl_sync(kFull, part[0], kLanesPerRow * q);
          if (!((amask >> (kLanesPerRow * q)) & 1u)) continue;
          const int r2 = rz[q];
          if (lane < d4)
            reinterpret_cast<float4*>(f.res_u + static_cast<size_t>(r2) * d)[lane] = f4sub(dz[q], f4scale(dzw, w));
          acc_dz = f4add(acc_dz, dz[q]);
          acc_n = f4add(acc_n, f4add(f4scale(dzw, u[q]), f4scale(wu[q], dz[q])));
        }
      }
      if (tid == 0 && i < 4) th_stamp(tr, 11 + static_cast<int>(i));
    }
    if (tid == 0) th_stamp(tr, 15);
    if (run >= 0) flush();
    if (tid == 0) th_stamp(tr, 16);
    if (lane == 0) S.wl[warp] = lw;
  }
  // ---- loss: warps in order -> one partial per CTA, the last CTA finalizes
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&f.err[3], pend);
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) th_stamp(tr, 17);
  if (!alive) return;
  if (tid == 0) {
    float lsum = 0.f;
    for (int q = 0; q < kCompute; ++q) lsum = __fadd_rn(lsum, S.wl[q]);
    f.block_partial[blockIdx.x] = lsum;
    S.last_cta = ticket_acq_rel(f.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (S.last_cta && warp == 0) {
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, f.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, f.loss_div > 0.f ? f.loss_div : static_cast<float>(f.B));
      f.batch_loss[f.batch] = loss;
      if (f.stamp_end) stamp_now(f.stamp_end);
      const uint32_t pflags = *reinterpret_cast<volatile uint32_t*>(&f.err[3]);
      if (nonfinite(loss)) {
        f.err[1] = f.batch;
        atomicCAS(&f.err[0], 0u, static_cast<uint32_t>(kErrLossNonFinite));
      } else if (pflags) {
        f.err[1] = f.batch;
        atomicCAS(&f.err[0], 0u, static_cast<uint32_t>(kErrGradEntity));
      }
      f.err[3] = 0;
      *f.counter = 0;
    }
  }
  if (tid == 0) th_stamp(tr, 18);
}

// Relation side of the batch (runs beside the entity segment pass; both read
// only the forward's outputs): block k < runs sums relation run k's (CTA, run)
// slots in CTA order (cta_of_tile's partition), applies SGD to d_r and w_r and
// renormalizes w_r; block b also renormalizes normal b when relation b is
// absent from the batch (embedding.cpp:165-190 steps every row, then
// renormalizes every normal). Data parallel (nrm_sink): the slot sums go to
// the sinks and the dense step + renormalization follow the all-reduce.
__global__ void __launch_bounds__(2 * kD) transh_rel_finalize_kernel(const TArgs a, uint32_t G) {
  const FwdArgs& f = a.f;
  if (f.err[0] != 0) return;  // nothing is applied for a failing batch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t b = blockIdx.x, nrel = a.info[0], T = a.info[1];
  if (b < nrel) {
    const int64_t r = a.info[4 + 3 * b];
    const uint32_t j0 = cta_of_tile(a.info[5 + 3 * b], T, G), j1 = cta_of_tile(a.info[6 + 3 * b] - 1, T, G);
    const int c = tid & (kD - 1), v = tid / kD;  // (column, vector)
    const int d = f.de;
    const float* src = a.partial + static_cast<size_t>(v) * kD + c;
    float g = 0.f;
    uint32_t j = j0;
    for (; j + 8 <= j1 + 1; j += 8) {
      float x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = __ldcg(src + static_cast<size_t>(j + e + b) * 2 * kD);
#pragma unroll
      for (int e = 0; e < 8; ++e) g = __fadd_rn(g, x[e]);
    }
    for (; j <= j1; ++j) g = __fadd_rn(g, __ldcg(src + static_cast<size_t>(j + b) * 2 * kD));
    if (a.nrm_sink) {  // data parallel: this rank's gradient rows (summed over ranks, then one dense step)
      if (c < d) {
        if (v == 0) a.rel[r * d + c] = g;
        else a.nrm_sink[r * d + c] = -g;
      }
      return;
    }
    const float step = *a.lr;
    if (c < d) {
      float* p = v == 0 ? a.rel + r * d + c : const_cast<float*>(f.normals) + r * d + c;
      *p = __fsub_rn(*p, __fmul_rn(step, v == 0 ? g : -g));  // grads.normals -= nrm (models.hpp:112)
    }
    __syncthreads();
    if (warp == 0) renorm_normal(const_cast<float*>(f.normals), r, f.de, lane, f.err);
  }
  if (a.nrm_sink || static_cast<int64_t>(b) >= a.R || warp != 0) return;
  bool present = false;
  for (uint32_t q0 = 0; q0 < nrel && !present; q0 += 32) {
    const uint32_t q = q0 + lane;
    present = __any_sync(kFull, q < nrel && a.info[4 + 3 * q] == b);
  }
  if (!present) renorm_normal(const_cast<float*>(f.normals), b, f.de, lane, f.err);
}

// Per minibatch b of the epoch plan (one block each, on the plan branch):
// the batch's relation tiles as the forward walks them -- per tile {run k,
// relation r, pairs}, per pair its ids and batch position -- and the run table
// transh_rel_finalize_kernel reads ({runs, tiles, 0, 0, then r, first, end per
// run}). The forward then loads each tile's records directly instead of
// chasing seg_start -> ent_val -> pair record at the start of every batch.
__global__ void __launch_bounds__(256) transh_tile_plan_kernel(TArgs a, int64_t B_full, int64_t nb, int64_t M,
                                                               int64_t mt, int4* meta, int4* rows, int32_t* pos,
                                                               uint32_t* info) {
  __shared__ RelTiles rt;
  const int64_t b = blockIdx.x;  // batch; blockIdx.y: slice of its tiles
  if (b >= nb) return;
  a.batch = static_cast<int>(b);
  const int tid = threadIdx.x;
  if (tid < 32) enumerate_rel_tiles(a, rt);
  __syncthreads();
  const uint32_t T = static_cast<uint32_t>(min(static_cast<int64_t>(rt.first[rt.nrel]), mt));
  const int64_t lo = b * B_full, Bb = min(B_full, M - lo);
  const int4* pair_ht = a.f.pair_ht + lo;
  uint32_t* inf = info + b * (4 + 3 * a.R);
  int4* mb = meta + b * mt;
  int4* rb = rows + b * mt * kPairs;
  int32_t* pb = pos + b * mt * kPairs;
  if (blockIdx.y == 0) {
    for (uint32_t q = tid; q < rt.nrel; q += blockDim.x) {
      inf[4 + 3 * q] = static_cast<uint32_t>(__ldg(a.seg_col + rt.seg[q]) - static_cast<uint32_t>(a.f.N));
      inf[5 + 3 * q] = rt.first[q];
      inf[6 + 3 * q] = rt.first[q + 1];
    }
    if (tid == 0) {
      inf[0] = rt.nrel;
      inf[1] = T;
    }
  }
  for (uint32_t i = blockIdx.y * blockDim.x + tid; i < T * kPairs; i += gridDim.y * blockDim.x) {
    const uint32_t t = i / kPairs, p = i % kPairs;
    const uint32_t kq = rel_of_tile(rt, t);
    const uint32_t sq = rt.seg[kq], pq = (t - rt.first[kq]) * kPairs;
    const uint32_t e0 = __ldg(a.seg_start + sq), len = __ldg(a.seg_start + sq + 1) - e0;
    const int np = static_cast<int>(min(static_cast<uint32_t>(kPairs), len / 2 - pq));
    int ps = -1;
    int4 q4 = make_int4(0, 0, 0, 0);
    if (static_cast<int>(p) < np) {
      ps = static_cast<int>(__ldg(a.ent_val + e0 + pq + p) & 0x7fffffffu);
      if (ps < Bb) q4 = __ldg(pair_ht + ps);
    }
    rb[i] = q4;
    pb[i] = ps;
    if (p == 0) mb[t] = make_int4(static_cast<int>(kq), static_cast<int>(__ldg(a.seg_col + sq) - static_cast<uint32_t>(a.f.N)), np, 0);
  }
}

}  // namespace

// any width up to 128 in 16-byte chunks: rows are staged zero-padded to 128 columns
bool transh_tiles_supported(int de, int dr, int64_t R) {
  return de == dr && de >= 4 && de <= kD && de % 4 == 0 && R <= kMaxRelSeg;
}

int64_t transh_trace(int enable, unsigned long long* out, int64_t cap) {
  SKG_CUDA(cudaMemcpyToSymbol(g_thtrace_on, &enable, sizeof(int)));
  const int64_t n = static_cast<int64_t>(kThTrCtas) * kThTrEvents;
  if (enable) {
    static const unsigned long long zeros[kThTrCtas * kThTrEvents] = {};
    SKG_CUDA(cudaMemcpyToSymbol(g_thtrace, zeros, sizeof(zeros)));
  }
  if (out && cap >= n) SKG_CUDA(cudaMemcpyFromSymbol(out, g_thtrace, sizeof(unsigned long long) * n));
  return n;
}

int64_t transh_tile_plan_tiles(int64_t B, int64_t R) { return relation_max_tiles(2 * B, R); }

void transh_tile_plan(const FwdArgs& fa, const BwdArgs& ba, int64_t B, int64_t nb, int64_t M, int64_t R,
                      const ThTilePlan& tp, cudaStream_t s) {
  TArgs a{};
  a.f = fa;
  a.ent_val = ba.ent_val;
  a.seg_start = ba.seg_start;
  a.seg_col = ba.seg_col;
  a.seg_base = ba.seg_base;
  a.R = R;
  const int64_t mt = transh_tile_plan_tiles(B, R);
  // (batch, slice) blocks: the records' dependent loads spread over the SMs
  const unsigned slices = static_cast<unsigned>(std::min<int64_t>(64, std::max<int64_t>(1, mt * kPairs / 2048)));
  transh_tile_plan_kernel<<<dim3(static_cast<unsigned>(nb), slices), 256, 0, s>>>(a, B, nb, M, mt, tp.meta, tp.rows,
                                                                                   tp.pos, tp.info);
  count_launch();
  SKG_LAUNCH_CHECK();
}

int64_t transh_tiles_work_floats(int64_t rows, int64_t R) {
  const int64_t mt = relation_max_tiles(rows, R);
  return (mt + R + 1) * 2 * kD + 3 * R + 64;  // run info, then (CTA, relation run) slots b + k, b < grid <= mt
}

void configure_transh_tiles_kernels() {
  const int smem = static_cast<int>(sizeof(PipeSmem));
  SKG_CUDA(cudaFuncSetAttribute(transh_pipe_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  SKG_CUDA(cudaFuncSetAttribute(transh_pipe_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  SKG_CUDA(cudaFuncSetAttribute(transh_pipe_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  SKG_CUDA(cudaFuncSetAttribute(transh_pipe_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
}

void transh_tiles_train_batch(bool l2, const FwdArgs& fa, const BwdArgs& ba, float* work, int64_t R, int num_sms,
                              cudaStream_t s, const std::function<void()>* mark, const HtSinks* sinks,
                              const Branch* br, const ThTilePlan* tp) {
  const int64_t mt = relation_max_tiles(2 * static_cast<int64_t>(fa.B), R);
  // run info leads the workspace (a fixed address for every batch size), the
  // float4 run partials follow
  uint32_t* info = reinterpret_cast<uint32_t*>(work);
  float* partial = work + ((4 + 3 * R + 3) & ~static_cast<int64_t>(3));
  TArgs a{};
  a.f = fa;
  a.ent_val = ba.ent_val;
  a.seg_start = ba.seg_start;
  a.seg_col = ba.seg_col;
  a.seg_base = ba.seg_base;
  a.batch = ba.batch;
  a.mt = mt;
  a.partial = partial;
  a.info = info;
  a.rel = sinks ? sinks->rel : const_cast<float*>(fa.X) + fa.N * static_cast<int64_t>(fa.de);
  a.lr = ba.lr;
  a.nrm_sink = sinks ? sinks->normals : nullptr;
  a.R = R;
  if (tp && tp->meta) {  // this batch's slice of the plan's tile records
    const int64_t mtp = transh_tile_plan_tiles(tp->B, R);
    a.tp_meta = tp->meta + ba.batch * mtp;
    a.tp_rows = tp->rows + ba.batch * mtp * kPairs;
    a.tp_pos = tp->pos + ba.batch * mtp * kPairs;
    a.info = tp->info + ba.batch * (4 + 3 * R);
    a.mt = mtp;
  }
  const size_t smem = sizeof(PipeSmem);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(mt, num_sms));  // persistent, one CTA per SM
  const bool full = fa.de == kD;
  if (l2 && full) transh_pipe_kernel<true, true><<<grid, kPipeThreads, smem, s>>>(a);
  else if (l2) transh_pipe_kernel<true, false><<<grid, kPipeThreads, smem, s>>>(a);
  else if (full) transh_pipe_kernel<false, true><<<grid, kPipeThreads, smem, s>>>(a);
  else transh_pipe_kernel<false, false><<<grid, kPipeThreads, smem, s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
  if (mark) (*mark)();
  // relation side on a forked branch, beside the entity segment pass
  cudaStream_t rs = s;
#ifdef SKG_TH_NOBRANCH
  br = nullptr;
#endif
  if (br) {
    SKG_CUDA(cudaEventRecord(br->fork, s));
    SKG_CUDA(cudaStreamWaitEvent(br->aux, br->fork, 0));
    rs = br->aux;
  }
  transh_rel_finalize_kernel<<<static_cast<unsigned>(std::max<int64_t>(R, 1)), 2 * kD, 0, rs>>>(a, grid);
  count_launch();
  SKG_LAUNCH_CHECK();
  if (br) SKG_CUDA(cudaEventRecord(br->join, br->aux));
  BwdArgs eb = ba;
  eb.entity_only = 1;
  launch_segment_backward(kPlainRows, sinks == nullptr, eb, num_sms, s);  // sink: ba.X is the entity gradient
  if (br) SKG_CUDA(cudaStreamWaitEvent(s, br->join, 0));
}

}  // namespace skg
