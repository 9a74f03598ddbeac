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
// 32 pairs = 64 rows per tile, 8 warps x 8 rows, two CTAs per SM: twice the
// tiles of a 64-pair tile, so the persistent grid ends more evenly and one
// CTA's barrier waits overlap the other's work.
constexpr int kPairs = SKG_TRANSH_PAIRS;
constexpr int kRows = 2 * kPairs;
constexpr int kRowsPerWarp = 8;
constexpr int kThreads = kRows / kRowsPerWarp * 32;
constexpr int kCtasPerSm = 64 / kPairs;
static_assert(kThreads >= 2 * 128, "the relation reduction uses one thread per (column, vector)");
constexpr int kStride = kD + 4;    // staged v rows (16-byte aligned, conflict-free row reads)

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
  uint32_t* rel_ticket;       // per relation segment: tiles finished (zeroed by the tile enumerator)
  float* rel;                 // relation table (SGD), or the relation gradient sink
  const float* lr;
  float* nrm_sink;            // data parallel: normals gradient sink (null: SGD in place)
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

template <bool L2>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) transh_tile_kernel(const TArgs a) {
  extern __shared__ float4 smv[];
  float* Vs = reinterpret_cast<float*>(smv);  // [kRows][kStride]
  __shared__ int4 rows[kRows];                 // {head, tail, incidence row (-1: padding), 0}
  __shared__ float score[kRows];
  __shared__ float wloss[kThreads / 32];
  __shared__ float4 accs[2][kThreads / 32][32];
  __shared__ bool last, rel_last;
  __shared__ RelTiles rt;
  const FwdArgs& f = a.f;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (f.stamp_start && blockIdx.x == 0 && tid == 0) stamp_now(f.stamp_start);
  const bool alive = f.err[0] == 0;
  if (warp == 0 && alive) enumerate_rel_tiles(a, rt);
  __syncthreads();
  const uint32_t T = alive ? static_cast<uint32_t>(min(static_cast<int64_t>(rt.first[rt.nrel]), a.mt)) : 0u;
  float lsum = 0.f;
  uint32_t pend = 0;
  // Row ids of tile tt for pair kk = tid < 64: stage 1 reads the relation
  // segment entry (positive row = batch position), stage 2 its pair record.
  // The next tile's chase is issued while the current tile computes.
  auto stage1 = [&](uint32_t tt, int kk) -> int {
    const uint32_t kq = rel_of_tile(rt, tt);
    const uint32_t sq = rt.seg[kq], pq = (tt - rt.first[kq]) * kPairs;
    const uint32_t e0q = __ldg(a.seg_start + sq), lenq = __ldg(a.seg_start + sq + 1) - e0q;
    const int npq = static_cast<int>(min(static_cast<uint32_t>(kPairs), lenq / 2 - pq));
    return kk < npq ? static_cast<int>(__ldg(a.ent_val + e0q + pq + kk) & 0x7fffffffu) : -1;
  };
  auto stage2 = [&](int pos, int4& pr, int4& ng) {
    pr = make_int4(0, 0, -1, 0);
    ng = make_int4(0, 0, -1, 0);
    if (pos < 0) return;
    int h, tt, nh, nt;
    if (f.pair_ht) {
      const int4 x = __ldg(f.pair_ht + pos);
      h = x.x, tt = x.y, nh = x.z, nt = x.w;
    } else {
      const int id = __ldg(f.order + pos);
      h = __ldg(f.H + id), tt = __ldg(f.T + id), nh = __ldg(f.NH + id), nt = __ldg(f.NT + id);
    }
    pr = make_int4(h, tt, pos, 0);
    ng = make_int4(nh, nt, pos + f.B, 0);
  };
  int4 pr_next = make_int4(0, 0, -1, 0), ng_next = make_int4(0, 0, -1, 0);
  int pos_next = -1;
  if (tid < kPairs && blockIdx.x < T) stage2(stage1(blockIdx.x, tid), pr_next, ng_next);
  for (uint32_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint32_t k = rel_of_tile(rt, t);
    const uint32_t sseg = rt.seg[k], p0 = (t - rt.first[k]) * kPairs;
    const uint32_t e0 = __ldg(a.seg_start + sseg), len = __ldg(a.seg_start + sseg + 1) - e0;
    const int64_t r = static_cast<int64_t>(__ldg(a.seg_col + sseg)) - f.N;
    const int np = static_cast<int>(min(static_cast<uint32_t>(kPairs), len / 2 - p0));
    (void)e0;
    const float4 w = __ldg(reinterpret_cast<const float4*>(f.normals + r * kD) + lane);
    const float4 drv = __ldg(reinterpret_cast<const float4*>(f.X + (f.N + r) * kD) + lane);
    if (tid < kPairs) {
      rows[tid] = pr_next;
      rows[kPairs + tid] = ng_next;
    }
    __syncthreads();
    const uint32_t tn = t + gridDim.x;
    if (tid < kPairs && tn < T) pos_next = stage1(tn, tid);  // in flight during this tile
    // ---- u, wu, v for this warp's 8 rows, all 16 row loads in flight
    const int m0 = warp * kRowsPerWarp;
    float4 u[kRowsPerWarp];
    float wu[kRowsPerWarp];
    {
      float4 xh[kRowsPerWarp], xt[kRowsPerWarp];
#pragma unroll
      for (int q = 0; q < kRowsPerWarp; ++q) {
        const int4 rw = rows[m0 + q];
        xh[q] = __ldg(reinterpret_cast<const float4*>(f.X + static_cast<size_t>(rw.x) * kD) + lane);
        xt[q] = __ldg(reinterpret_cast<const float4*>(f.X + static_cast<size_t>(rw.y) * kD) + lane);
      }
      float part[kRowsPerWarp];
#pragma unroll
      for (int q = 0; q < kRowsPerWarp; ++q) {
        u[q] = rows[m0 + q].z >= 0 ? f4sub(xh[q], xt[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
        part[q] = f4dot(w, u[q]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) part[q] = __fadd_rn(part[q], __shfl_xor_sync(kFull, part[q], o));
#pragma unroll
      for (int q = 0; q < kRowsPerWarp; ++q) {
        wu[q] = part[q];
        const float4 v = f4sub(f4add(u[q], drv), f4scale(wu[q], w));
        *reinterpret_cast<float4*>(Vs + (m0 + q) * kStride + 4 * lane) = v;
      }
    }
    __syncwarp();
    // ---- score (lane j < 8 owns row m0 + j): reference-order squared_sum / abs_sum
    float ssum = 0.f;
    bool bad = false;
    const int mj = m0 + (lane & 7);
    const int row2 = rows[mj].z;
    {  // whole warp, reference association (warp_norm8); row j lands on lane j
      bool b = false;
      const float sj = warp_norm8<L2>(Vs + m0 * kStride, kStride, kD, lane, b);
      if (lane < kRowsPerWarp) {
        ssum = sj;
        bad = b;
        score[mj] = L2 ? __fsqrt_rn(ssum) : ssum;
      }
    }
    __syncthreads();
    if (tid < kPairs && tn < T) stage2(pos_next, pr_next, ng_next);
    // ---- pair hinge (training.cpp:73-94)
    const int kk = mj & (kPairs - 1);
    const bool valid = lane < kRowsPerWarp && kk < np;
    float term = 0.f;
    if (valid) term = __fsub_rn(__fadd_rn(f.margin, score[kk]), score[kPairs + kk]);
    const bool act = valid && term > 0.f;
    const float up = act ? (mj < kPairs ? f.unit : -f.unit) : 0.f;
    const float sc = act ? (L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(ssum, kNormEpsF))) : up) : 0.f;
    if (valid) f.scal[row2] = act ? 1.f : 0.f;
    if (valid && bad && (L2 || act)) pend |= kPendEntity;
    {
      float tk = (act && mj < kPairs) ? term : 0.f;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) tk = __fadd_rn(tk, __shfl_down_sync(kFull, tk, o));
      if (lane == 0) wloss[warp] = tk;
    }
    // ---- backward rows (hyperplane_backward, models.hpp:106-113)
    const unsigned amask = __ballot_sync(kFull, act);
    float4 acc_dz = make_float4(0.f, 0.f, 0.f, 0.f), acc_n = make_float4(0.f, 0.f, 0.f, 0.f);
    if (amask) {
      float4 dz[kRowsPerWarp];
      float part[kRowsPerWarp];
#pragma unroll
      for (int q = 0; q < kRowsPerWarp; ++q) {
        const float scq = __shfl_sync(kFull, sc, q);
        dz[q] = dir4<L2>(*reinterpret_cast<const float4*>(Vs + (m0 + q) * kStride + 4 * lane), scq);
        if (!((amask >> q) & 1u)) dz[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        part[q] = f4dot(dz[q], w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) part[q] = __fadd_rn(part[q], __shfl_xor_sync(kFull, part[q], o));
#pragma unroll
      for (int q = 0; q < kRowsPerWarp; ++q) {
        if (!((amask >> q) & 1u)) continue;
        const float dzw = part[q];
        const int r2 = rows[m0 + q].z;
        reinterpret_cast<float4*>(f.res_u + static_cast<size_t>(r2) * kD)[lane] = f4sub(dz[q], f4scale(dzw, w));
        acc_dz = f4add(acc_dz, dz[q]);
        acc_n = f4add(acc_n, f4add(f4scale(dzw, u[q]), f4scale(wu[q], dz[q])));
      }
    }
    accs[0][warp][lane] = acc_dz;
    accs[1][warp][lane] = acc_n;
    __syncthreads();
    if (tid < 64) {  // tile partial: warps in order
      const int which = tid >> 5;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < kThreads / 32; ++q) s = f4add(s, accs[which][q][lane]);
      reinterpret_cast<float4*>(a.partial + (static_cast<size_t>(t) * 2 + which) * kD)[lane] = s;
      __threadfence();
    }
    if (tid == 0)
      for (int q = 0; q < kPairs / kRowsPerWarp; ++q) lsum = __fadd_rn(lsum, wloss[q]);
    __syncthreads();
    // the CTA finishing a relation's last tile sums its tile partials in tile
    // order and applies SGD to the relation row and the normal
    // (grads.normals -= nrm, models.hpp:112; embedding.cpp:165-190)
    const uint32_t lo = rt.first[k], hi = rt.first[k + 1];
    if (tid == 0) {
      rel_last = atomicAdd(a.rel_ticket + k, 1u) == hi - lo - 1;
      if (rel_last) a.rel_ticket[k] = 0;  // every tile of k has arrived: ready for the next batch
    }
    __syncthreads();
    if (rel_last && tid < 2 * kD) {
      // thread (c, v): column c of the relation gradient (v = 0) or of the
      // normal's (v = 1); 16 tiles' loads in flight, added in tile order
      __threadfence();
      const int c = tid & (kD - 1), v = tid / kD;
      const float* src = a.partial + static_cast<size_t>(v) * kD + c;
      float g = 0.f;
      uint32_t q = lo;
      for (; q + 16 <= hi; q += 16) {
        float x[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __ldcg(src + static_cast<size_t>(q + e) * 2 * kD);
#pragma unroll
        for (int e = 0; e < 16; ++e) g = __fadd_rn(g, x[e]);
      }
      for (; q < hi; ++q) g = __fadd_rn(g, __ldcg(src + static_cast<size_t>(q) * 2 * kD));
      if (a.nrm_sink) {  // data parallel: this rank's gradient rows (summed over ranks, then one dense step)
        if (v == 0) a.rel[r * kD + c] = g;
        else a.nrm_sink[r * kD + c] = -g;
      } else {
        const float step = *a.lr;
        float* p = v == 0 ? a.rel + r * kD + c : const_cast<float*>(f.normals) + r * kD + c;
        *p = __fsub_rn(*p, __fmul_rn(step, v == 0 ? g : -g));
      }
    }
    __syncthreads();  // rows / score / accs reuse by the next tile
  }
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&f.err[3], pend);
    __threadfence();
  }
  if (!alive) return;
  // ---- loss: one partial per tile (tile order), the last CTA finalizes
  if (tid == 0) {
    f.block_partial[blockIdx.x] = lsum;
    __threadfence();
    last = atomicAdd(f.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && warp == 0) {
    __threadfence();
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, f.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, f.loss_div > 0.f ? f.loss_div : static_cast<float>(f.B));
      f.batch_loss[f.batch] = loss;
      if (f.stamp_end) stamp_now(f.stamp_end);
      const uint32_t pflags = atomicOr(&f.err[3], 0u);
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

}  // namespace

bool transh_tiles_supported(int de, int dr, int64_t R) { return de == kD && dr == kD && R <= kMaxRelSeg; }

int64_t transh_tiles_work_floats(int64_t rows, int64_t R) {
  const int64_t mt = relation_max_tiles(rows, R);
  return mt * 2 * kD + R + 64;
}

void configure_transh_tiles_kernels() {
  const int smem = static_cast<int>(sizeof(float) * kRows * kStride);
  SKG_CUDA(cudaFuncSetAttribute(transh_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  SKG_CUDA(cudaFuncSetAttribute(transh_tile_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
}

void transh_tiles_train_batch(bool l2, const FwdArgs& fa, const BwdArgs& ba, float* work, int64_t R, int num_sms,
                              cudaStream_t s, const std::function<void()>* mark, const HtSinks* sinks) {
  const int64_t mt = relation_max_tiles(2 * static_cast<int64_t>(fa.B), R);
  // tickets lead the workspace (a fixed address for every batch size), the
  // float4 tile partials follow
  uint32_t* ticket = reinterpret_cast<uint32_t*>(work);
  float* partial = work + ((R + 1 + 3) & ~static_cast<int64_t>(3));
  // per-relation tickets: zeroed at the epoch's first batch, then reset by the
  // CTA that retires each relation (no memset node between the batch kernels)
  if (ba.batch == 0) SKG_CUDA(cudaMemsetAsync(ticket, 0, sizeof(uint32_t) * (R + 1), s));
  TArgs a{};
  a.f = fa;
  a.ent_val = ba.ent_val;
  a.seg_start = ba.seg_start;
  a.seg_col = ba.seg_col;
  a.seg_base = ba.seg_base;
  a.batch = ba.batch;
  a.mt = mt;
  a.partial = partial;
  a.rel_ticket = ticket;
  a.rel = sinks ? sinks->rel : const_cast<float*>(fa.X) + fa.N * static_cast<int64_t>(fa.de);
  a.lr = ba.lr;
  a.nrm_sink = sinks ? sinks->normals : nullptr;
  const size_t smem = sizeof(float) * kRows * kStride;
  const unsigned grid =
      static_cast<unsigned>(std::min<int64_t>(mt, static_cast<int64_t>(num_sms) * kCtasPerSm));  // persistent
  if (l2) transh_tile_kernel<true><<<grid, kThreads, smem, s>>>(a);
  else transh_tile_kernel<false><<<grid, kThreads, smem, s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
  if (mark) (*mark)();
  BwdArgs eb = ba;
  eb.entity_only = 1;
  launch_segment_backward(kPlainRows, sinks == nullptr, eb, num_sms, s);  // sink: ba.X is the entity gradient
}

}  // namespace skg
