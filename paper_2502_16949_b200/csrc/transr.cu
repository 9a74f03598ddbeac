// TransR on device: relation-grouped projection tiles
// (models.cpp:110-156, models.hpp:82-96).
//
// Every minibatch row of relation r needs M_r (d_r x d_e). The epoch plan
// already groups rows by relation (the relation column's segment lists the
// positive rows, then the same pairs' negative rows, ascending). A CTA owns a
// tile of up to 64 (pos, neg) pairs of one relation = 128 rows:
//   U  = h - t                       (128 x d_e, exact ht CSR row)
//   V  = U M_r^T + r                 (projection, models.hpp:82-86)
//   score = ||V_row|| in the reference's squared_sum order, hinge on the pair
//   DZ = dir(V) * up                 (norm_direction)
//   dU = DZ M_r                      (project_back_u, models.hpp:89-91)
//   dM_r partial = DZ^T U, dr partial = sum DZ   (project_back_mr, :94-96)
// M_r, U and V/DZ stay in shared memory for the three products. dU rows go
// through the sorted entity segments (no atomics); per-tile dM_r / dr partials
// are summed per relation in tile order and applied with SGD in one kernel.
//
// The three products run as 128x128x128 register-tiled FP32 FMA blocks in this
// version; the projection has d_r*d_e*2 FLOP per row, so the tile is the unit a
// tcgen05 (3xTF32) MMA version replaces without changing the data flow.
#include <algorithm>

#include "common.cuh"
#include "ht.cuh"
#include "plan.cuh"
#include "primitives.cuh"
#include "refmath.cuh"

namespace skg {

namespace {

constexpr int kTileRows = 128;
constexpr int kTilePairs = 64;
constexpr int kTrThreads = 256;

enum Mode : int { kTrain = 0, kRows = 1 };

struct TrArgs {
  FwdArgs f;
  const uint32_t* ent_val;
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* seg_base;
  int batch;
  const uint32_t* tile_seg;   // tile -> relation segment
  const uint32_t* tile_p0;    // tile -> first pair (kTrain) / row (kRows) in the segment
  const uint32_t* tile_total;
  float* dm_part;             // [tile][dr*de]
  float* dr_part;             // [tile][dr]
  bool want_grads;            // kRows: produce dU / partials (score_backward)
};

// One CTA enumerates the batch's relation segments into tiles; seg_tiles[k]
// is the first tile of the k-th relation segment ([nrel] = total). Relation
// segments lead the batch's segment list (relation column keys sort first).
// Thread per segment, block scan of the tile counts, then every thread
// writes its own segment's tiles.
constexpr int kTilesThreads = 1024;
__device__ __forceinline__ void tiles_body(const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ seg_col,
                                           const uint32_t* __restrict__ seg_base, int batch, int64_t N, int paired,
                                           uint32_t* __restrict__ tile_seg, uint32_t* __restrict__ tile_p0,
                                           uint32_t* __restrict__ tile_total, uint32_t* __restrict__ seg_tiles,
                                           const uint32_t* __restrict__ err) {
  __shared__ uint32_t wsum[kTilesThreads / 32];
  __shared__ uint32_t carry_t, nrel;
  __shared__ int stop;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t s0 = seg_base[batch], s1 = seg_base[batch + 1];
  const uint32_t per = paired ? kTilePairs : kTileRows;
  if (tid == 0) {
    carry_t = 0;
    nrel = 0;
    stop = err ? err[0] != 0 : 0;
  }
  __syncthreads();
  for (uint32_t base = s0; base < s1 && !stop; base += kTilesThreads) {
    const uint32_t s = base + tid;
    const bool rel = s < s1 && seg_col[s] >= static_cast<uint32_t>(N) && seg_col[s] != kDummyCol;
    uint32_t n = 0, units = 0;
    if (rel) {
      const uint32_t len = seg_start[s + 1] - seg_start[s];
      units = paired ? len / 2 : len;
      n = (units + per - 1) / per;
    }
    // relation segments are a prefix: count them in this chunk
    const int nr = __syncthreads_count(rel);
    uint32_t x = n;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t v = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const uint32_t first = carry_t + (w > 0 ? wsum[w - 1] : 0u) + x - n;
    if (rel) {
      const uint32_t k = nrel + tid;
      seg_tiles[k] = first;
      for (uint32_t q = 0; q < n; ++q) {
        tile_seg[first + q] = s;
        tile_p0[first + q] = q * per;
      }
    }
    __syncthreads();
    if (tid == 0) {
      carry_t += wsum[kTilesThreads / 32 - 1];
      nrel += static_cast<uint32_t>(nr);
      if (nr < kTilesThreads) stop = 1;
    }
    __syncthreads();
  }
  if (tid == 0) {
    seg_tiles[nrel] = carry_t;
    tile_total[0] = carry_t;
    tile_total[1] = nrel;
  }
}

__global__ void __launch_bounds__(kTilesThreads) transr_tiles_kernel(
    const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ seg_col, const uint32_t* __restrict__ seg_base,
    int batch, int64_t N, int paired, uint32_t* __restrict__ tile_seg, uint32_t* __restrict__ tile_p0,
    uint32_t* __restrict__ tile_total, uint32_t* __restrict__ seg_tiles, const uint32_t* __restrict__ err,
    uint32_t* __restrict__ zero = nullptr, int nzero = 0, unsigned long long* stamp = nullptr) {
  if (stamp && threadIdx.x == 0) stamp_now(stamp);
  for (int i = threadIdx.x; i < nzero; i += blockDim.x) zero[i] = 0u;  // per-relation tickets of the next kernel
  tiles_body(seg_start, seg_col, seg_base, batch, N, paired, tile_seg, tile_p0, tile_total, seg_tiles, err);
}

// Every minibatch's relation tiles of an epoch plan at once (block b = batch b),
// on the plan branch: the training step then starts with its projection kernel.
__global__ void __launch_bounds__(kTilesThreads) transr_tiles_plan_kernel(
    const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ seg_col, const uint32_t* __restrict__ seg_base,
    int64_t N, int64_t mt, int64_t R, uint32_t* __restrict__ tile_seg, uint32_t* __restrict__ tile_p0,
    uint32_t* __restrict__ tile_total, uint32_t* __restrict__ seg_tiles) {
  const int64_t b = blockIdx.x;
  tiles_body(seg_start, seg_col, seg_base, static_cast<int>(b), N, 1, tile_seg + b * mt, tile_p0 + b * mt,
             tile_total + 2 * b, seg_tiles + b * (R + 2), nullptr);
}

template <bool L2, int MODE>
__global__ void __launch_bounds__(kTrThreads, 1) transr_tile_kernel(const TrArgs a) {
  extern __shared__ float smem[];
  __shared__ float warp_loss[kTrThreads / 32];
  __shared__ float rs[kTileRows], rsc[kTileRows];
  __shared__ int rrow[kTileRows];
  __shared__ float tile_loss;
  const FwdArgs& f = a.f;
  if (f.err[0] != 0) return;
  if (f.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) stamp_now(f.stamp_start);
  const int de = f.de, dr = f.dr;
  const int SE = de + 1, SR = dr + 1;
  float* Ms = smem;                 // dr x SE
  float* Us = Ms + dr * SE;         // 128 x SE
  float* Vs = Us + kTileRows * SE;  // 128 x SR
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const uint32_t ntiles = *a.tile_total;
  float lsum = 0.f;
  uint32_t pend = 0;
  if (blockIdx.x < ntiles) {
    const uint32_t s = a.tile_seg[blockIdx.x], p0 = a.tile_p0[blockIdx.x];
    const uint32_t e0 = a.seg_start[s], len = a.seg_start[s + 1] - e0;
    const int64_t r = static_cast<int64_t>(a.seg_col[s]) - f.N;
    const uint32_t units = MODE == kTrain ? len / 2 : len;
    const int np = static_cast<int>(min(static_cast<uint32_t>(MODE == kTrain ? kTilePairs : kTileRows), units - p0));
    // ---- row ids (row k of the tile)
    if (tid < kTileRows) {
      int row2 = -1;
      if (MODE == kTrain) {
        const int k = tid & 63;
        if (k < np) row2 = static_cast<int>(a.ent_val[e0 + (tid < 64 ? 0 : units) + p0 + k] & 0x7fffffffu);
      } else if (tid < np) {
        row2 = static_cast<int>(a.ent_val[e0 + p0 + tid] & 0x7fffffffu);
      }
      rrow[tid] = row2;
    }
    // ---- M_r -> smem
    const float* M = f.proj + r * static_cast<int64_t>(dr) * de;
    for (int i = tid; i < dr * de; i += kTrThreads) Ms[(i / de) * SE + (i % de)] = __ldg(M + i);
    __syncthreads();
    // ---- U = h - t (warp per row)
    const int warp = tid >> 5, lane = tid & 31;
    for (int k = warp; k < kTileRows; k += kTrThreads / 32) {
      const int row2 = rrow[k];
      int h = 0, t = 0;
      if (row2 >= 0) {
        if (MODE == kTrain) {
          const bool neg = row2 >= f.B;
          const int id = f.order[neg ? row2 - f.B : row2];
          h = neg ? f.NH[id] : f.H[id];
          t = neg ? f.NT[id] : f.T[id];
        } else {
          h = f.H[row2];
          t = f.T[row2];
        }
      }
      for (int c = lane; c < de; c += 32)
        Us[k * SE + c] = row2 >= 0 ? __fsub_rn(__ldg(f.X + static_cast<int64_t>(h) * de + c),
                                               __ldg(f.X + static_cast<int64_t>(t) * de + c))
                                   : 0.f;
    }
    __syncthreads();
    // ---- V = U M^T + rel  (thread: rows ty+16i, cols tx+16j)
    const float* rel = f.X + f.N * static_cast<int64_t>(de) + r * dr;
    for (int jb = 0; jb < dr; jb += 128) {
      float acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
      for (int k = 0; k < de; ++k) {
        float av[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = Us[(ty + 16 * i) * SE + k];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = jb + tx + 16 * j;
          bv[j] = n < dr ? Ms[n * SE + k] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = jb + tx + 16 * j;
          if (n < dr) Vs[(ty + 16 * i) * SR + n] = __fadd_rn(acc[i][j], __ldg(rel + n));
        }
    }
    __syncthreads();
    // ---- scores in the reference order (thread per row)
    if (tid < kTileRows) {
      bool bad = false;
      const float sq = ref_norm_sum<L2, 1>(Vs + tid * SR, dr, bad);
      rs[tid] = sq;
      if (bad && rrow[tid] >= 0) pend |= kPendEntity;
    }
    __syncthreads();
    if (tid < kTileRows) {
      const int row2 = rrow[tid];
      float up = 0.f;
      const float score = L2 ? __fsqrt_rn(rs[tid]) : rs[tid];
      if (MODE == kTrain) {
        const int k = tid & 63;
        if (k < np) {
          const float ps = L2 ? __fsqrt_rn(rs[k]) : rs[k];
          const float ns = L2 ? __fsqrt_rn(rs[64 + k]) : rs[64 + k];
          const float term = __fsub_rn(__fadd_rn(f.margin, ps), ns);
          if (term > 0.f) up = tid < 64 ? f.unit : -f.unit;
        }
      } else if (row2 >= 0) {
        f.scores[row2] = score;
        if (a.want_grads) up = f.upstream[row2];
      }
      rsc[tid] = up == 0.f ? 0.f : (L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(rs[tid], kNormEpsF))) : up);
      if (row2 >= 0 && (MODE == kTrain || a.want_grads)) f.scal[row2] = up != 0.f ? 1.f : 0.f;
    }
    if (MODE == kTrain && tid == 0) {  // tile loss, pairs in order
      float tl = 0.f;
      for (int k = 0; k < np; ++k) {
        const float ps = L2 ? __fsqrt_rn(rs[k]) : rs[k];
        const float ns = L2 ? __fsqrt_rn(rs[64 + k]) : rs[64 + k];
        const float term = __fsub_rn(__fadd_rn(f.margin, ps), ns);
        if (term > 0.f) tl = __fadd_rn(tl, term);
      }
      tile_loss = tl;
    }
    __syncthreads();
    if (MODE == kRows && !a.want_grads) {
      // score_batch: v and u rows out
      for (int k = warp; k < kTileRows; k += kTrThreads / 32) {
        const int row2 = rrow[k];
        if (row2 < 0) continue;
        for (int c = lane; c < dr; c += 32) f.res[static_cast<int64_t>(row2) * dr + c] = Vs[k * SR + c];
        for (int c = lane; c < de; c += 32) f.res_u[static_cast<int64_t>(row2) * de + c] = Us[k * SE + c];
      }
    } else {
      // ---- DZ in place of V
      for (int i = tid; i < kTileRows * dr; i += kTrThreads) {
        const int k = i / dr, n = i % dr;
        const float sc = rsc[k];
        const float v = Vs[k * SR + n];
        Vs[k * SR + n] = sc == 0.f ? 0.f : (L2 ? __fmul_rn(v, sc) : (v > 0.f ? sc : (v < 0.f ? -sc : 0.f)));
      }
      __syncthreads();
      // ---- dU = DZ M  (rows ty+16i, cols tx+16j of d_e) -> entity scatter rows
      for (int jb = 0; jb < de; jb += 128) {
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int n = 0; n < dr; ++n) {
          float av[8], bv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) av[i] = Vs[(ty + 16 * i) * SR + n];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = jb + tx + 16 * j;
            bv[j] = c < de ? Ms[n * SE + c] : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = ty + 16 * i;
          const int row2 = rrow[k];
          if (row2 < 0 || rsc[k] == 0.f) continue;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = jb + tx + 16 * j;
            if (c < de) f.res_u[static_cast<int64_t>(row2) * de + c] = acc[i][j];
          }
        }
      }
      // ---- dM partial = DZ^T U (rows n = ty+16i of d_r, cols tx+16j of d_e); dr partial
      float* dmp = a.dm_part + static_cast<int64_t>(blockIdx.x) * dr * de;
      for (int ib = 0; ib < dr; ib += 128)
        for (int jb = 0; jb < de; jb += 128) {
          float acc[8][8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
          for (int k = 0; k < kTileRows; ++k) {
            if (rsc[k] == 0.f) continue;
            float av[8], bv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int n = ib + ty + 16 * i;
              av[i] = n < dr ? Vs[k * SR + n] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int c = jb + tx + 16 * j;
              bv[j] = c < de ? Us[k * SE + c] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int n = ib + ty + 16 * i, c = jb + tx + 16 * j;
              if (n < dr && c < de) dmp[n * de + c] = acc[i][j];
            }
        }
      for (int n = tid; n < dr; n += kTrThreads) {
        float sdr = 0.f;
        for (int k = 0; k < kTileRows; ++k) sdr = __fadd_rn(sdr, Vs[k * SR + n]);
        a.dr_part[static_cast<int64_t>(blockIdx.x) * dr + n] = sdr;
      }
    }
    if (MODE == kTrain) lsum = tile_loss;
  }
  // ---- loss: one partial per CTA (tile order), last CTA finalizes
  if (MODE != kTrain) {
    pend = __reduce_or_sync(kFull, pend);
    if ((tid & 31) == 0 && pend) atomicOr(&f.err[3], pend);
    return;
  }
  pend = __reduce_or_sync(kFull, pend);
  if ((tid & 31) == 0 && pend) {
    atomicOr(&f.err[3], pend);
    __threadfence();
  }
  if ((tid & 31) == 0) warp_loss[tid >> 5] = tid == 0 ? lsum : 0.f;
  __syncthreads();
  __shared__ bool last;
  if (tid == 0) {
    f.block_partial[blockIdx.x] = lsum;
    last = ticket_acq_rel(f.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && tid < 32) {
    float acc = 0.f;
    for (int b = tid; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, f.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (tid == 0) {
      const float loss = __fdiv_rn(acc, static_cast<float>(f.B));
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
}

// Per relation segment: sum tile partials in tile order, then SGD on the
// projection block and the relation row (or accumulate into sinks).
__global__ void transr_apply_kernel(const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_total,
                                    const uint32_t* __restrict__ seg_tiles, const uint32_t* __restrict__ seg_col,
                                    int64_t N, const float* __restrict__ dm_part, const float* __restrict__ dr_part,
                                    int de, int dr, float* __restrict__ proj, float* __restrict__ rel,
                                    const float* __restrict__ lr, bool sgd, const uint32_t* __restrict__ err) {
  if (err[0] != 0) return;
  if (blockIdx.x >= tile_total[1]) return;
  const uint32_t lo = seg_tiles[blockIdx.x], hi = seg_tiles[blockIdx.x + 1];
  if (hi <= lo) return;
  const int64_t r = static_cast<int64_t>(seg_col[tile_seg[lo]]) - N;
  const float step = *lr;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < dr * de + dr; i += gridDim.y * blockDim.x) {
    float g = 0.f;
    if (i < dr * de) {
      for (uint32_t t = lo; t < hi; ++t) g = __fadd_rn(g, dm_part[static_cast<int64_t>(t) * dr * de + i]);
      float* p = proj + r * static_cast<int64_t>(dr) * de + i;
      *p = sgd ? __fsub_rn(*p, __fmul_rn(step, g)) : __fadd_rn(*p, g);
    } else {
      const int n = i - dr * de;
      for (uint32_t t = lo; t < hi; ++t) g = __fadd_rn(g, dr_part[static_cast<int64_t>(t) * dr + n]);
      float* p = rel + r * dr + n;
      *p = sgd ? __fsub_rn(*p, __fmul_rn(step, g)) : __fadd_rn(*p, g);
    }
  }
}

size_t tile_smem(int de, int dr) {
  return sizeof(float) * (static_cast<size_t>(dr) * (de + 1) + kTileRows * (de + 1) + kTileRows * (dr + 1));
}

struct Work {
  uint32_t *tile_seg, *tile_p0, *tile_total, *seg_tiles;
  float *dm_part, *dr_part, *mr_chunks;
};

int64_t max_tiles(int64_t rows, int64_t R) { return rows / kTilePairs + 2 * R + 2; }

// dM partial of one (CTA, run) slot: the tcgen05 training kernel writes 128 x 128 (zero-padded
// for narrower M_r), the FP32 tile kernel d_r x d_e.
int64_t part_floats(int64_t de, int64_t dr) {
  return transr_train_tc_supported(static_cast<int>(de), static_cast<int>(dr)) ? std::max<int64_t>(dr * de, 128 * 128)
                                                                               : dr * de;
}

Work carve(float* work, int64_t rows, int64_t de, int64_t dr, int64_t R) {
  const int64_t mt = max_tiles(rows, R);
  Work w;
  // the split M_r chunks come first: their offset must not depend on the batch
  // size (the training apply of batch b refreshes them for batch b + 1, and the
  // last batch of an epoch is shorter)
  w.mr_chunks = work;
  float* rest = work + ((std::max(transr_tc_mr_floats(R), transr_train_tc_mr_floats(R)) + 31) / 32) * 32;
  w.tile_seg = reinterpret_cast<uint32_t*>(rest);
  w.tile_p0 = w.tile_seg + mt;
  w.tile_total = w.tile_p0 + mt;
  w.seg_tiles = w.tile_total + 2;
  w.dm_part = rest + ((3 * mt + 2 * R + 8 + 31) / 32) * 32;  // 128 B aligned (float4 stores)
  w.dr_part = w.dm_part + std::max<int64_t>(mt, transr_tc_slots(256, R)) * part_floats(de, dr);
  return w;
}

template <bool L2, int MODE>
void launch_tile(const TrArgs& a, int64_t rows, int64_t R, cudaStream_t s) {
  const int grid = static_cast<int>(max_tiles(rows, R));
  transr_tile_kernel<L2, MODE><<<grid, kTrThreads, tile_smem(a.f.de, a.f.dr), s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void run_tiles(int kind, bool train, const FwdArgs& fa, const BwdArgs& ba, const Work& w, bool want_grads,
               int64_t rows, int64_t R, cudaStream_t s) {
  if (fa.de > 128 || fa.dr > 128 || tile_smem(fa.de, fa.dr) > 220 * 1024)
    throw CudaError("transr: dimensions above 128 are not supported by the projection tile");
  transr_tiles_kernel<<<1, kTilesThreads, 0, s>>>(ba.seg_start, ba.seg_col, ba.seg_base, ba.batch, ba.N, train ? 1 : 0, w.tile_seg,
                                       w.tile_p0, w.tile_total, w.seg_tiles, ba.err);
  count_launch();
  TrArgs a{};
  a.f = fa;
  a.ent_val = ba.ent_val;
  a.seg_start = ba.seg_start;
  a.seg_col = ba.seg_col;
  a.seg_base = ba.seg_base;
  a.batch = ba.batch;
  a.tile_seg = w.tile_seg;
  a.tile_p0 = w.tile_p0;
  a.tile_total = w.tile_total;
  a.dm_part = w.dm_part;
  a.dr_part = w.dr_part;
  a.want_grads = want_grads;
  const bool l2 = kind == kTransR_L2;
  if (train) {
    if (l2) launch_tile<true, kTrain>(a, rows, R, s);
    else launch_tile<false, kTrain>(a, rows, R, s);
  } else {
    if (l2) launch_tile<true, kRows>(a, rows, R, s);
    else launch_tile<false, kRows>(a, rows, R, s);
  }
}

void apply(const FwdArgs& fa, const BwdArgs& ba, const Work& w, float* proj, float* rel, bool sgd, int64_t R,
           cudaStream_t s) {
  transr_apply_kernel<<<dim3(static_cast<unsigned>(R), 16), 256, 0, s>>>(
      w.tile_seg, w.tile_total, w.seg_tiles, ba.seg_col, ba.N, w.dm_part, w.dr_part, fa.de, fa.dr, proj, rel, ba.lr, sgd, ba.err);
  count_launch();
  SKG_LAUNCH_CHECK();
}

template <bool L2, int MODE>
void configure_one() {
  SKG_CUDA(cudaFuncSetAttribute(transr_tile_kernel<L2, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                220 * 1024));
}

}  // namespace

int64_t relation_max_tiles(int64_t rows, int64_t R) { return max_tiles(rows, R); }

void transr_tile_plan(const BwdArgs& ba, int64_t B, int64_t nb, int64_t R, const TrTilePlan& tp, cudaStream_t s) {
  transr_tiles_plan_kernel<<<static_cast<unsigned>(nb), kTilesThreads, 0, s>>>(
      ba.seg_start, ba.seg_col, ba.seg_base, ba.N, max_tiles(2 * B, R), R, tp.tile_seg, tp.tile_p0, tp.tile_total,
      tp.seg_tiles);
  count_launch();
  SKG_LAUNCH_CHECK();
}

void launch_relation_tiles(const BwdArgs& ba, int paired, uint32_t* tile_seg, uint32_t* tile_p0, uint32_t* tile_total,
                           uint32_t* seg_tiles, cudaStream_t s, uint32_t* zero, int nzero) {
  transr_tiles_kernel<<<1, kTilesThreads, 0, s>>>(ba.seg_start, ba.seg_col, ba.seg_base, ba.batch, ba.N, paired,
                                                  tile_seg, tile_p0, tile_total, seg_tiles, ba.err, zero, nzero);
  count_launch();
  SKG_LAUNCH_CHECK();
}

int64_t transr_work_floats(int64_t rows, int64_t de, int64_t dr, int64_t R) {
  const int64_t mt = max_tiles(rows, R);
  const int64_t parts = std::max<int64_t>(mt, transr_tc_slots(256, R));  // tc path: (CTA, relation) runs
  return ((std::max(transr_tc_mr_floats(R), transr_train_tc_mr_floats(R)) + 31) / 32) * 32 +
         ((3 * mt + 2 * R + 8 + 31) / 32) * 32 + parts * part_floats(de, dr) +
         ((parts * std::max<int64_t>(dr, 128) + 31) / 32) * 32 + 64;
}

void configure_transr_kernels() {
  configure_one<true, kTrain>();
  configure_one<true, kRows>();
  configure_one<false, kTrain>();
  configure_one<false, kRows>();
  configure_transr_tc_kernels();
  configure_transr_train_tc_kernels();
}

namespace {
// tcgen05 path (d_e = d_r = 128): tile list, persistent projection CTAs.
void run_tc(int kind, int mode, const FwdArgs& fa, const BwdArgs& ba, const Work& w, int num_sms, cudaStream_t s,
            int64_t R) {
  transr_tiles_kernel<<<1, kTilesThreads, 0, s>>>(ba.seg_start, ba.seg_col, ba.seg_base, ba.batch, ba.N, mode == 0 ? 1 : 0,
                                       w.tile_seg, w.tile_p0, w.tile_total, w.seg_tiles, ba.err);
  count_launch();
  SKG_LAUNCH_CHECK();
  launch_transr_tc(kind == kTransR_L2, mode, fa, ba.ent_val, ba.seg_start, ba.seg_col, w.tile_seg, w.tile_p0,
                   w.tile_total, w.seg_tiles, w.dm_part, w.dr_part, w.mr_chunks, R, num_sms, s);
}
}  // namespace

void transr_train_batch(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                        const std::function<void()>* mark, int64_t R, const HtSinks* sinks, const Branch* br,
                        const TrTilePlan* tp) {
  Work w = carve(work, 2 * static_cast<int64_t>(fa.B), fa.de, fa.dr, R);
  // data parallel (sinks): entity rows accumulate into ba.X, proj / relation
  // gradients land in the sinks, and the engine applies one dense step
  float* proj_dst = sinks ? sinks->proj : const_cast<float*>(fa.proj);
  float* rel_dst = sinks ? sinks->rel : const_cast<float*>(fa.X) + fa.N * static_cast<int64_t>(fa.de);
  if (transr_train_tc_supported(fa.de, fa.dr)) {
    FwdArgs fa_tc = fa;
    if (tp && tp->tile_seg) {  // tiles from the epoch plan: this batch's slice
      const int64_t mtp = max_tiles(2 * tp->B, R);
      w.tile_seg = tp->tile_seg + ba.batch * mtp;
      w.tile_p0 = tp->tile_p0 + ba.batch * mtp;
      w.tile_total = tp->tile_total + 2 * static_cast<int64_t>(ba.batch);
      w.seg_tiles = tp->seg_tiles + ba.batch * (R + 2);
    } else {
      transr_tiles_kernel<<<1, kTilesThreads, 0, s>>>(ba.seg_start, ba.seg_col, ba.seg_base, ba.batch, ba.N, 1,
                                                      w.tile_seg, w.tile_p0, w.tile_total, w.seg_tiles, ba.err,
                                                      nullptr, 0, fa.stamp_start);
      count_launch();
      SKG_LAUNCH_CHECK();
      fa_tc.stamp_start = nullptr;  // stamped by the tiles kernel, the batch's first launch
    }
    launch_transr_train_tc(kind == kTransR_L2, fa_tc, ba.ent_val, ba.seg_start, ba.seg_col, w.tile_seg, w.tile_p0,
                           w.tile_total, w.seg_tiles, w.dm_part, w.dr_part, w.mr_chunks, R, num_sms, s,
                           sinks != nullptr);
    if (mark) (*mark)();
    // relation side (M_r and relation rows) on a forked branch beside the entity segment pass:
    // disjoint parameters, both read only the projection kernel's outputs
    cudaStream_t as = s;
    if (br) {
      SKG_CUDA(cudaEventRecord(br->fork, s));
      SKG_CUDA(cudaStreamWaitEvent(br->aux, br->fork, 0));
      as = br->aux;
    }
    launch_transr_train_apply(w.tile_total, w.seg_tiles, w.tile_seg, ba.seg_col, ba.N, num_sms, w.dm_part, w.dr_part,
                              proj_dst, rel_dst, ba.lr, ba.err, w.mr_chunks, R, as, sinks != nullptr, fa.dr, fa.de);
    if (br) SKG_CUDA(cudaEventRecord(br->join, br->aux));
    BwdArgs eb = ba;
    eb.entity_only = 1;
    eb.d = fa.de;
    launch_segment_backward(kTileSlotRows, sinks == nullptr, eb, num_sms, s);
    if (br) SKG_CUDA(cudaStreamWaitEvent(s, br->join, 0));
    if (mark) (*mark)();
    return;
  }
  run_tiles(kind, true, fa, ba, w, true, 2 * static_cast<int64_t>(fa.B), R, s);
  if (mark) (*mark)();
  BwdArgs eb = ba;
  eb.entity_only = 1;
  eb.d = fa.de;
  launch_segment_backward(kPlainRows, sinks == nullptr, eb, num_sms, s);
  apply(fa, ba, w, proj_dst, rel_dst, sinks == nullptr, R, s);
  if (mark) (*mark)();
}

void transr_score(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                  int64_t R) {
  const Work w = carve(work, fa.B, fa.de, fa.dr, R);
  if (transr_tc_supported(fa.de, fa.dr)) {
    run_tc(kind, 1, fa, ba, w, num_sms, s, R);
    return;
  }
  run_tiles(kind, false, fa, ba, w, false, fa.B, R, s);
}

void transr_score_backward(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, float* g_proj, int num_sms,
                           cudaStream_t s, int64_t R) {
  const Work w = carve(work, fa.B, fa.de, fa.dr, R);
  if (transr_tc_supported(fa.de, fa.dr)) {
    run_tc(kind, 2, fa, ba, w, num_sms, s, R);
    BwdArgs eb = ba;
    eb.entity_only = 1;
    eb.d = fa.de;
    launch_segment_backward(kPlainRows, false, eb, num_sms, s);
    launch_transr_tc_apply(w.tile_total, w.seg_tiles, w.tile_seg, ba.seg_col, ba.N, num_sms, w.dm_part, w.dr_part,
                           g_proj, ba.Xrel, ba.lr, false, ba.err, R, s);
    return;
  }
  run_tiles(kind, false, fa, ba, w, true, fa.B, R, s);
  BwdArgs eb = ba;
  eb.entity_only = 1;
  eb.d = fa.de;
  launch_segment_backward(kPlainRows, false, eb, num_sms, s);
  apply(fa, ba, w, g_proj, ba.Xrel, false, R, s);
}

}  // namespace skg
