// TransE / TorusE hot path: fused forward (gather + distance + hinge + loss)
// and the fused transposed-SpMM backward + SGD step.
//
// Forward (models.cpp:11-30, 71-92; norms.hpp:19-126; training.cpp:73-94).
// A warp owns a tile of 8 (pos, neg) pairs = 16 incidence rows. For each row
// the lanes gather the h, t and r embedding rows with 128-bit loads and form
// v = (h - t) + r, which is bitwise the CSR row sum a_h x_h + a_t x_t + x_r in
// canonical column order (sparse.hpp:211-237; a = +-1 makes every product
// exact and (-t) + h == h - t). Rows are staged in shared memory with a
// (d + 4)-float stride so that in the reduction phase lane l can read row l
// with conflict-free float4 loads and evaluate squared_sum / abs_sum with the
// reference's exact 4-accumulator order. The pair's hinge is formed in
// registers; only rows of active pairs write their residual to HBM, with one
// per-row scale (the L2 1/||v|| weight, or the L1/torus weight). The batch
// loss is reduced deterministically (warp -> block -> last-block).
//
// Backward (sparse.hpp:273-306 + embedding.cpp:165-190). Entries of the
// batch's incidence are pre-sorted by column (stable, so in ascending row
// order with all positive rows before all negative rows, exactly the order in
// which the reference accumulates spmm_transpose_add(pos) then (neg)). A warp
// owns one column segment, accumulates a * D_row in that order in registers
// (no atomics) and applies p -= lr * g to the touched row in the same kernel.
// Rows never touched keep p - lr*0 == p, so touching only the segment rows is
// bitwise the reference's dense step.
#include <cstdlib>

#include "common.cuh"
#include "plan.cuh"
#include "kernels.cuh"
#include "primitives.cuh"
#include "tc.cuh"

namespace skg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr float kEps = 1e-6f;  // kNormEps for 32-bit reals, common.hpp:34
#ifndef SKG_BWD_KB
#define SKG_BWD_KB 4
#endif

__device__ __forceinline__ float torus_wrap(float x) {  // norms.hpp:96-100
  float d = __fsub_rn(x, rintf(x));
  if (d >= 0.5f) d = __fsub_rn(d, 1.0f);
  return d;
}

template <int KIND>
__device__ __forceinline__ float4 hrt_combine(float4 h, float4 t, float4 r, bool self_loop) {
  float4 v;
  if (self_loop) {
    v = r;
  } else {
    v.x = __fadd_rn(__fsub_rn(h.x, t.x), r.x);
    v.y = __fadd_rn(__fsub_rn(h.y, t.y), r.y);
    v.z = __fadd_rn(__fsub_rn(h.z, t.z), r.z);
    v.w = __fadd_rn(__fsub_rn(h.w, t.w), r.w);
  }
  if (KIND == kTorusE_L2 || KIND == kTorusE_L1) {
    v.x = torus_wrap(v.x);
    v.y = torus_wrap(v.y);
    v.z = torus_wrap(v.z);
    v.w = torus_wrap(v.w);
  }
  return v;
}

template <int KIND>
__device__ __forceinline__ float hrt_combine1(float h, float t, float r, bool self_loop) {
  float v = self_loop ? r : __fadd_rn(__fsub_rn(h, t), r);
  if (KIND == kTorusE_L2 || KIND == kTorusE_L1) v = torus_wrap(v);
  return v;
}

__device__ __forceinline__ float term_of(int KIND, float x) {
  return (KIND == kTransE_L2) ? __fmul_rn(x, x) : fabsf(x);
}

// squared_sum / abs_sum (norms.hpp:19-55) and the torus sums (:107-115) in the
// reference's exact association; `bad` collects non-finite elements.
template <int KIND, int VEC>
__device__ float ref_reduce(const float* v, int n, bool& bad) {
  bool nf = false;
  float s;
  if (KIND == kTorusE_L2 || KIND == kTorusE_L1) {
    s = 0.f;
    for (int j = 0; j < n; ++j) {
      const float x = v[j];
      s = __fadd_rn(s, KIND == kTorusE_L2 ? __fmul_rn(x, x) : fabsf(x));
    }
    // terms are >= 0 or NaN: a finite sum proves every element finite
    if (!(fabsf(s) <= 3.402823466e38f))
      for (int j = 0; j < n; ++j) nf |= !(fabsf(v[j]) <= 3.402823466e38f);
  } else if (n < 8) {
    s = 0.f;
    for (int j = 0; j < n; ++j) {
      nf |= !(fabsf(v[j]) <= 3.402823466e38f);
      s = __fadd_rn(s, term_of(KIND, v[j]));
    }
  } else {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
      float4 q;
      if (VEC == 4) {
        q = *reinterpret_cast<const float4*>(v + j);
      } else {
        q = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      nf |= !(fabsf(q.x) <= 3.402823466e38f) | !(fabsf(q.y) <= 3.402823466e38f) |
            !(fabsf(q.z) <= 3.402823466e38f) | !(fabsf(q.w) <= 3.402823466e38f);
      s0 = __fadd_rn(s0, term_of(KIND, q.x));
      s1 = __fadd_rn(s1, term_of(KIND, q.y));
      s2 = __fadd_rn(s2, term_of(KIND, q.z));
      s3 = __fadd_rn(s3, term_of(KIND, q.w));
    }
    s = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
    for (; j < n; ++j) {
      nf |= !(fabsf(v[j]) <= 3.402823466e38f);
      s = __fadd_rn(s, term_of(KIND, v[j]));
    }
  }
  bad = nf;
  return s;
}

// TransE rows (d >= 8, d % 4 == 0) reduced by the whole warp: lane 2 r + h
// runs accumulators 2h and 2h + 1 of row r over float2 steps, then
// (s0 + s1) + (s2 + s3) — ref_reduce's association with every lane busy
// (lanes 0-15 / 16-31 read 16 distinct bank pairs per half-warp request).
// Row j's sum lands on lane j < 16.
template <int KIND>
__device__ __forceinline__ float warp_reduce16(const float* rows, int S, int d, int lane, bool& bad) {
  const int r = lane >> 1, hb = lane & 1;
  const float* v = rows + r * S + 2 * hb;
  float sa = 0.f, sb = 0.f;
#pragma unroll 8
  for (int j = 0; j < d; j += 4) {
    const float2 x = *reinterpret_cast<const float2*>(v + j);
    sa = __fadd_rn(sa, term_of(KIND, x.x));
    sb = __fadd_rn(sb, term_of(KIND, x.y));
  }
  const float pair = __fadd_rn(sa, sb);                // s0 + s1 (h = 0) or s2 + s3 (h = 1)
  // Terms are >= 0 or NaN, so a finite sum proves every element finite; only a
  // non-finite sum (a non-finite element, or overflow) rescans its elements.
  bool nf = false;
  if (!(fabsf(pair) <= 3.402823466e38f))
    for (int j = 0; j < d; j += 4) {
      const float2 x = *reinterpret_cast<const float2*>(v + j);
      nf |= !(fabsf(x.x) <= 3.402823466e38f) | !(fabsf(x.y) <= 3.402823466e38f);
    }
  const float tot = __fadd_rn(pair, __shfl_down_sync(kFull, pair, 1));  // on h == 0 lanes
  const unsigned nfm = __ballot_sync(kFull, nf);
  bad = ((nfm >> (2 * (lane & 15))) & 3u) != 0u;
  return __shfl_sync(kFull, tot, 2 * (lane & 15));
}

// Eight TransE rows per warp (4-pair tiles, d > 128): lane 4 r + k runs
// accumulator k of row r, then (s0 + s1) + (s2 + s3); row j lands on lane j.
// S = 4 (mod 32) keeps each step's 32 scalar reads on 32 banks.
template <int KIND>
__device__ __forceinline__ float warp_reduce8(const float* rows, int S, int d, int lane, bool& bad) {
  const int r = lane >> 2, k = lane & 3;
  const float* v = rows + r * S + k;
  float sacc = 0.f;
#pragma unroll 8
  for (int j = 0; j < d; j += 4) sacc = __fadd_rn(sacc, term_of(KIND, v[j]));
  bool nf = false;  // a finite sum proves every element finite (see warp_reduce16)
  if (!(fabsf(sacc) <= 3.402823466e38f))
    for (int j = 0; j < d; j += 4) nf |= !(fabsf(v[j]) <= 3.402823466e38f);
  const float s1 = __shfl_down_sync(kFull, sacc, 1), s2 = __shfl_down_sync(kFull, sacc, 2),
              s3 = __shfl_down_sync(kFull, sacc, 3);
  const float tot = __fadd_rn(__fadd_rn(sacc, s1), __fadd_rn(s2, s3));  // on k == 0 lanes
  const unsigned nfm = __ballot_sync(kFull, nf);
  bad = ((nfm >> (4 * (lane & 7))) & 0xFu) != 0u;
  return __shfl_sync(kFull, tot, 4 * (lane & 7));
}

// Per-row gradient scale: D_row = dir(residual, scale) in the backward.
template <int KIND>
__device__ __forceinline__ float row_scale(float up, float s) {
  if (KIND == kTransE_L2) return __fdiv_rn(up, __fsqrt_rn(__fadd_rn(s, kEps)));  // norms.hpp:71-73
  if (KIND == kTorusE_L2) return __fmul_rn(up, 2.0f);                            // norms.hpp:125
  return up;                                                                     // L1 sign weight
}

// TRAIN-mode gather of a tile's 8 (pos, neg) pairs: lanes k and k + 8 hold
// the ids of pair k's positive and negative row (same relation).
// Row addressing: the stacked [entity; relation] table, or (SH) entity rows
// on their owner rank's shard (peer memory) and relation rows in the local
// replica (shard.cu).
template <bool SH>
struct RowSrc {
  const float4* X4;
  const float* const* peer;  // SH: per-rank entity shards
  const float4* rel4;        // SH: relation replica
  int glog;
  int64_t N;
  __device__ __forceinline__ const float4* ent(int e, int d4) const {
    if (SH)
      return reinterpret_cast<const float4*>(peer[e & ((1 << glog) - 1)]) + static_cast<size_t>(e >> glog) * d4;
    return X4 + static_cast<size_t>(e) * d4;
  }
  __device__ __forceinline__ const float4* rel(int r, int d4) const {
    return SH ? rel4 + static_cast<size_t>(r) * d4 : X4 + static_cast<size_t>(N + r) * d4;
  }
};

template <int KIND, int P, int TP = 8, bool SH = false>
__device__ __forceinline__ void gather_pairs(const RowSrc<SH>& src, int d4, int h, int t, int r,
                                             float* rows, int S, int lane) {
#pragma unroll
  for (int k0 = 0; k0 < TP; k0 += P) {
    int hp[P], tp[P], hn[P], tn[P], rr[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      hp[q] = __shfl_sync(kFull, h, k0 + q);
      tp[q] = __shfl_sync(kFull, t, k0 + q);
      hn[q] = __shfl_sync(kFull, h, k0 + q + TP);
      tn[q] = __shfl_sync(kFull, t, k0 + q + TP);
      rr[q] = __shfl_sync(kFull, r, k0 + q);
    }
    for (int c = lane; c < d4; c += 32) {
      float4 xa[P], xb[P], xe[P], xf[P], xr[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        xa[q] = __ldg(src.ent(hp[q], d4) + c);
        xb[q] = __ldg(src.ent(tp[q], d4) + c);
        xe[q] = __ldg(src.ent(hn[q], d4) + c);
        xf[q] = __ldg(src.ent(tn[q], d4) + c);
        xr[q] = __ldg(src.rel(rr[q], d4) + c);
      }
#pragma unroll
      for (int q = 0; q < P; ++q) {
        *reinterpret_cast<float4*>(rows + (k0 + q) * S + 4 * c) = hrt_combine<KIND>(xa[q], xb[q], xr[q], hp[q] == tp[q]);
        *reinterpret_cast<float4*>(rows + (k0 + q + TP) * S + 4 * c) =
            hrt_combine<KIND>(xe[q], xf[q], xr[q], hn[q] == tn[q]);
      }
    }
  }
}

#ifndef SKG_FWD_MINB
#define SKG_FWD_MINB 2
#endif
#ifndef SKG_FWD_P128
#define SKG_FWD_P128 4  // pairs gathered together when d <= 128 (5 row loads each)
#endif
#ifndef SKG_FWD_MINB_SMALL
#define SKG_FWD_MINB_SMALL 3
#endif
#ifndef SKG_FWD_P256
#define SKG_FWD_P256 2  // ... when d <= 256
#endif
template <int KIND, bool TRAIN, int VEC, int MINB = SKG_FWD_MINB, int TP = 8, bool SH = false>
__global__ void __launch_bounds__(kThreads, MINB) hrt_forward_kernel(const FwdArgs a) {
  extern __shared__ float4 smem4[];
  __shared__ float warp_loss[kWarps];
  __shared__ const float* s_peer[8];
  if (a.err[0] != 0) return;  // sticky error: nothing runs after the failing batch
  if (SH) {
    if (threadIdx.x < 8) s_peer[threadIdx.x] = a.ent_peer[threadIdx.x];
    __syncthreads();
  }
  if (a.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) stamp_now(a.stamp_start);
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = a.de;
  const int S = VEC == 4 ? d + 4 : d + 1;
  constexpr int RW = TRAIN ? 2 * TP : 16;  // rows per warp tile
  float* rows = smem + warp * RW * S;
  constexpr int kUnits = TRAIN ? TP : 16;
  const int ntiles = (a.B + kUnits - 1) / kUnits;
  const int64_t N = a.N;
  float lsum = 0.f;
  uint32_t pend = 0;

  const int nwarps = blockDim.x >> 5;
  // epoch-plan pair records of the warp's next tile, loaded while the current
  // tile is processed (one load per pair, no order -> id chase)
  int4 pq_next = make_int4(0, 0, 0, 0);
  int pr_next = 0;
  auto prefetch = [&](int tl) {
    if (TRAIN && a.pair_ht && lane < RW) {
      const int p = tl * TP + (lane & (TP - 1));
      if (tl < ntiles && p < a.B) {
        pq_next = __ldg(a.pair_ht + p);
        pr_next = __ldg(a.pair_r + p);
      }
    }
  };
  prefetch(blockIdx.x * nwarps + warp);
  for (int tile = blockIdx.x * nwarps + warp; tile < ntiles; tile += gridDim.x * nwarps) {
    // ---- row ids: lane j < 16 describes row j of the tile
    int h = 0, t = 0, r = 0, row2 = 0;
    bool valid = false;
    const int4 pq = pq_next;
    const int prr = pr_next;
    prefetch(tile + gridDim.x * nwarps);
    if (lane < RW) {
      if (TRAIN) {
        const int p = tile * TP + (lane & (TP - 1));
        const bool neg = lane >= TP;
        valid = p < a.B;
        if (valid) {
          if (a.pair_ht) {
            h = neg ? pq.z : pq.x;
            t = neg ? pq.w : pq.y;
            r = prr;
          } else {
            const int id = a.order[p];
            h = neg ? a.NH[id] : a.H[id];
            t = neg ? a.NT[id] : a.T[id];
            r = a.Rl[id];
          }
          row2 = neg ? a.B + p : p;
        }
      } else {
        const int i = tile * 16 + lane;
        valid = i < a.B;
        if (valid) {
          h = a.H[i];
          t = a.T[i];
          r = a.Rl[i];
          row2 = i;
        }
      }
    }
    const unsigned vmask = __ballot_sync(kFull, valid);

    // ---- gather 16 residual rows into shared memory
    if (TRAIN && VEC == 4) {
      // pair-grouped: a pair's positive (row k) and negative (row k + 8) share
      // the relation row, so P pairs need 5P row loads, all in flight at once
      const int d4 = d >> 2;
      constexpr int P128 = SKG_FWD_P128 < TP ? SKG_FWD_P128 : TP, P256 = SKG_FWD_P256 < TP ? SKG_FWD_P256 : TP;
      const RowSrc<SH> src{reinterpret_cast<const float4*>(a.X), s_peer, reinterpret_cast<const float4*>(a.rel_rows),
                           a.glog, N};
      if (d4 <= 32) gather_pairs<KIND, P128, TP, SH>(src, d4, h, t, r, rows, S, lane);
      else if (d4 <= 64) gather_pairs<KIND, P256, TP, SH>(src, d4, h, t, r, rows, S, lane);
      else gather_pairs<KIND, 1, TP, SH>(src, d4, h, t, r, rows, S, lane);
    } else if (VEC == 4) {
      const float4* X4 = reinterpret_cast<const float4*>(a.X);
      const int d4 = d >> 2;
#pragma unroll
      for (int j0 = 0; j0 < 16; j0 += 4) {
        int hj[4], tj[4], rj[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hj[q] = __shfl_sync(kFull, h, j0 + q);
          tj[q] = __shfl_sync(kFull, t, j0 + q);
          rj[q] = __shfl_sync(kFull, r, j0 + q);
        }
        for (int c = lane; c < d4; c += 32) {
          float4 xh[4], xt[4], xr[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            xh[q] = __ldg(X4 + static_cast<size_t>(hj[q]) * d4 + c);
            xt[q] = __ldg(X4 + static_cast<size_t>(tj[q]) * d4 + c);
            xr[q] = __ldg(X4 + static_cast<size_t>(N + rj[q]) * d4 + c);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(rows + (j0 + q) * S + 4 * c) =
                hrt_combine<KIND>(xh[q], xt[q], xr[q], hj[q] == tj[q]);
        }
      }
    } else {
      for (int j = 0; j < 16; ++j) {
        const int hj = __shfl_sync(kFull, h, j), tj = __shfl_sync(kFull, t, j),
                  rj = __shfl_sync(kFull, r, j);
        for (int c = lane; c < d; c += 32)
          rows[j * S + c] = hrt_combine1<KIND>(__ldg(a.X + static_cast<size_t>(hj) * d + c),
                                               __ldg(a.X + static_cast<size_t>(tj) * d + c),
                                               __ldg(a.X + static_cast<size_t>(N + rj) * d + c),
                                               hj == tj);
      }
    }
    __syncwarp();

    // ---- exact-order reduction: lane j reduces row j
    float s = 0.f, score = 0.f;
    bool bad = false;
    if ((KIND == kTransE_L2 || KIND == kTransE_L1) && VEC == 4 && d >= 8) {
      bool b = false;
      const float sw = RW == 8 ? warp_reduce8<KIND>(rows, S, d, lane, b) : warp_reduce16<KIND>(rows, S, d, lane, b);
      if (lane < RW && valid) {
        s = sw;
        bad = b;
        score = (KIND == kTransE_L2) ? __fsqrt_rn(s) : s;  // norms.hpp:57-62
      }
    } else if (lane < RW && valid) {
      s = ref_reduce<KIND, VEC>(rows + lane * S, d, bad);
      score = (KIND == kTransE_L2) ? __fsqrt_rn(s) : s;  // norms.hpp:57-62, 107-115
    }

    float up = 0.f;
    bool act = false;
    if (TRAIN) {
      // ---- margin hinge on (pos = lane k, neg = lane k + 8), training.cpp:86-96
      const float ns = __shfl_down_sync(kFull, score, TP);
      float term = 0.f;
      if (lane < TP && valid) {
        term = __fsub_rn(__fadd_rn(a.margin, score), ns);
        act = term > 0.f;  // strict
      }
      const float tk = act ? term : 0.f;
      float tsum = 0.f;
#pragma unroll
      for (int k = 0; k < TP; ++k) tsum = __fadd_rn(tsum, __shfl_sync(kFull, tk, k));
      lsum = __fadd_rn(lsum, tsum);
      act = __shfl_sync(kFull, act, lane & (TP - 1)) && lane < RW && valid;
      up = act ? (lane < TP ? a.unit : -a.unit) : 0.f;
    } else {
      act = lane < 16 && valid;
      up = (act && a.upstream) ? a.upstream[row2] : 0.f;
    }
    const float sc = (up != 0.f) ? row_scale<KIND>(up, s) : 0.f;
    // A non-finite residual turns into a non-finite gradient for L2 / torus-L2
    // even at zero upstream (v * 0); the reference rejects it in sgd_step.
    if ((KIND == kTransE_L2 || KIND == kTorusE_L2) && bad && (TRAIN || a.upstream))
      pend |= (h != t) ? kPendEntity : kPendRelation;

    if (lane < RW && valid) {
      a.scal[row2] = sc;
      if (!TRAIN) a.scores[row2] = score;
    }
    // ---- residual rows of active pairs (all rows in SCORE mode) to HBM
    const unsigned wmask = __ballot_sync(kFull, TRAIN ? (sc != 0.f) : (lane < 16 && valid)) & vmask;
    if (TRAIN && VEC == 4 && d <= 128) {  // one 16-byte chunk per lane per row; row k of the tile is
      const int d4 = d >> 2;              // pair tile * TP + k (positive) or B + that (negative)
      float4* pos = reinterpret_cast<float4*>(a.res) + static_cast<size_t>(tile) * TP * d4 + lane;
      float4* neg = pos + static_cast<size_t>(a.B) * d4;
      if (lane < d4) {
#pragma unroll
        for (int q = 0; q < RW; ++q)
          if ((wmask >> q) & 1u)
            (q < TP ? pos : neg)[(q & (TP - 1)) * d4] = *reinterpret_cast<const float4*>(rows + q * S + 4 * lane);
      }
      __syncwarp();
      continue;
    }
    for (unsigned m = wmask; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const int r2 = __shfl_sync(kFull, row2, j);  // uniform: every lane executes
      if (VEC == 4) {
        float4* dst = reinterpret_cast<float4*>(a.res + static_cast<size_t>(r2) * d);
        for (int c = lane; c < (d >> 2); c += 32) dst[c] = *reinterpret_cast<const float4*>(rows + j * S + 4 * c);
      } else {
        float* dst = a.res + static_cast<size_t>(r2) * d;
        for (int c = lane; c < d; c += 32) dst[c] = rows[j * S + c];
      }
    }
    __syncwarp();
  }

  // ---- deterministic loss reduction and batch finalization
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&a.err[3], pend);
    __threadfence();
  }
  if (!TRAIN) return;
  if (lane == 0) warp_loss[warp] = lsum;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w = 0; w < nwarps; ++w) b = __fadd_rn(b, warp_loss[w]);
    a.block_partial[blockIdx.x] = b;
    last = ticket_acq_rel(a.counter) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && warp == 0) {
    float acc = 0.f;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) acc = __fadd_rn(acc, a.block_partial[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_down_sync(kFull, acc, o));
    if (lane == 0) {
      const float loss = __fdiv_rn(acc, a.loss_div > 0.f ? a.loss_div : static_cast<float>(a.B));  // training.cpp:93
      a.batch_loss[a.batch] = loss;
      if (a.stamp_end) stamp_now(a.stamp_end);
      const uint32_t pflags = *reinterpret_cast<volatile uint32_t*>(&a.err[3]);
      if (!(fabsf(loss) <= 3.402823466e38f)) {
        a.err[1] = a.batch;
        atomicCAS(&a.err[0], 0u, static_cast<uint32_t>(kErrLossNonFinite));
      } else if (pflags) {
        a.err[1] = a.batch;
        atomicCAS(&a.err[0], 0u,
                  static_cast<uint32_t>((pflags & kPendEntity) ? kErrGradEntity : kErrGradRelation));
      }
      a.err[3] = 0;
      *a.counter = 0;
    }
  }
}

// D_row coefficient for one residual element (models.cpp:37-60, norms.hpp:119-126):
// L2: v * (up / ||v||_eps); torus-L2: (up * 2) * delta; L1 / torus-L1: sign weight.
template <int KIND>
__device__ __forceinline__ float dir1(float r, float sc) {
  if (KIND == kPlainRows || KIND == kMultRows || KIND == kTileSlotRows) return r;
  if (KIND == kTransE_L2 || KIND == kTorusE_L2) return __fmul_rn(r, sc);
  return r > 0.f ? sc : (r < 0.f ? -sc : 0.f);
}

// acc + a * D with a = +-1 (exact negation), sparse.hpp:284-296 association.
template <int KIND>
__device__ __forceinline__ void acc_add(float& acc, float r, float sc, bool neg) {
  const float x = dir1<KIND>(r, sc);
  acc = __fadd_rn(acc, neg ? -x : x);
}
template <int KIND>
__device__ __forceinline__ void acc_add(float4& acc, float4 r, float sc, bool neg) {
  acc_add<KIND>(acc.x, r.x, sc, neg);
  acc_add<KIND>(acc.y, r.y, sc, neg);
  acc_add<KIND>(acc.z, r.z, sc, neg);
  acc_add<KIND>(acc.w, r.w, sc, neg);
}

__device__ __forceinline__ float sgd1(float p, float g, float lr) {  // embedding.cpp:177-178
  return __fsub_rn(p, __fmul_rn(lr, g));
}
__device__ __forceinline__ float4 sgd1(float4 p, float4 g, float lr) {
  return make_float4(sgd1(p.x, g.x, lr), sgd1(p.y, g.y, lr), sgd1(p.z, g.z, lr), sgd1(p.w, g.w, lr));
}

template <int VEC> struct VecT;
template <> struct VecT<4> { using T = float4; };
template <> struct VecT<1> { using T = float; };

// One column segment [e0, e1) of column `col`, by one warp; CH vector chunks
// per lane per pass (CH = 1 covers d <= 128 with float4 lanes). Up to KB
// residual rows are in flight per round; the adds stay in the segment's entry
// order. `single`: a one-entry segment whose entry v0 and scale sc0 the
// caller already holds.
template <int KIND, bool SGD, int VEC, int CH, int KB>
__device__ __forceinline__ void segment_rows(const BwdArgs& a, uint32_t col, uint32_t e0, uint32_t e1, bool single,
                                             uint32_t v0, float sc0, int lane) {
  using V = typename VecT<VEC>::T;
  const int dv = a.d / VEC;
  const V* RV = reinterpret_cast<const V*>(a.res);
  V* P = reinterpret_cast<V*>(a.X) + static_cast<size_t>(col) * dv;
  for (int cb = 0; cb < dv; cb += 32 * CH) {
    int c[CH];
    bool has[CH];
    V acc[CH], p[CH];
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      c[h] = cb + 32 * h + lane;
      has[h] = c[h] < dv;
      acc[h] = V{};
      p[h] = V{};
      // the owner warp is the only writer of this row: load it up front
      if (has[h]) p[h] = P[c[h]];
      if (!SGD) acc[h] = p[h];  // accumulate into an existing sink (score_backward)
    }
    for (uint32_t eb = e0; eb < e1; eb += 32) {
      const int cnt = min(32u, e1 - eb);
      uint32_t myv = 0;
      float mysc = 0.f;
      if (lane < cnt) {
        if (single) {
          myv = v0;
          mysc = sc0;
        } else {
          myv = a.ent_val[eb + lane];
          mysc = a.scal[myv & 0x7fffffffu];
        }
      }
      const bool on = KIND == kTileSlotRows ? __float_as_uint(mysc) != 0u : mysc != 0.f;
      unsigned live = __ballot_sync(kFull, lane < cnt && on);
      while (live) {
        int k[KB];
        int n = 0;
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          k[q] = live ? __ffs(live) - 1 : 0;
          if (live) {
            live &= live - 1;
            ++n;
          }
        }
        uint32_t vq[KB];
        float scq[KB];
        V rv[KB][CH];
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          vq[q] = __shfl_sync(kFull, myv, k[q]);
          scq[q] = __shfl_sync(kFull, mysc, k[q]);
          size_t rowoff = static_cast<size_t>(vq[q] & 0x7fffffffu) * dv;
          if (KIND == kTileSlotRows) {  // d = 128, float4 lanes: chunk c of slot s
            const uint32_t sl = __float_as_uint(scq[q]) - 1u;
            rowoff = (static_cast<size_t>(sl >> 7) * 128 * 128 + (sl & 127u) * kDuGroup) / 4;
            scq[q] = 1.f;
          }
          if (KIND == kMultRows) {  // the entry's own gradient plane: head, tail or relation
            const uint32_t slot = col >= static_cast<uint32_t>(a.N) ? 2u : (vq[q] >> 31);
            rowoff += static_cast<size_t>(slot) * a.plane_rows * dv;
          }
#pragma unroll
          for (int h = 0; h < CH; ++h)
            if (q < n && has[h])
              rv[q][h] = __ldg(RV + rowoff +
                               (KIND == kTileSlotRows ? (c[h] / (kDuGroup / 4)) * (32 * kDuGroup) + c[h] % (kDuGroup / 4)
                                                      : c[h]));
        }
#pragma unroll
        for (int q = 0; q < KB; ++q)
          if (q < n) {
            const bool neg = KIND != kMultRows && (vq[q] >> 31) != 0;
#pragma unroll
            for (int h = 0; h < CH; ++h)
              if (has[h]) acc_add<KIND>(acc[h], rv[q][h], scq[q], neg);
          }
      }
    }
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      if (!has[h]) continue;
      if (SGD) P[c[h]] = sgd1(p[h], acc[h], *a.lr);
      else P[c[h]] = acc[h];
    }
  }
}

// The TransH / TransR entity pass at d <= 128 (float4 rows; one warp per
// column segment, segment_rows): the warp's segments s = s0 + gw + i nw are
// taken 32 at a time, lane j loading segment j's column and entry range and,
// for a one-entry segment, its entry and scale into shared memory, so each
// segment starts with its row loads instead of four dependent metadata loads
// (C2: most entity segments hold one entry; epoch -3 %, C4 -1.8 %). The other
// passes keep segment_backward_kernel: the staging measured slower there
// (C1 backward 22.3 -> 30.8 us, M1 26.8 -> 29.4 us).
template <bool SGD, int KIND = kPlainRows, int KB = SKG_BWD_KB>
__global__ void __launch_bounds__(kThreads) segment_backward_staged_kernel(const BwdArgs a) {
  if (a.err[0] != 0) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t s0 = a.seg_base[a.batch], s1 = a.seg_base[a.batch + 1];
  auto skip = [&](uint32_t col) {
    return col == kDummyCol || (a.entity_only && col >= static_cast<uint32_t>(a.N));
  };
  __shared__ uint4 seg_q[kThreads / 32][32];  // {column, e0, e1, entry of a one-entry segment}
  __shared__ float seg_sc[kThreads / 32][32];
  uint4* myq = seg_q[threadIdx.x >> 5];
  float* mysc = seg_sc[threadIdx.x >> 5];
  for (uint32_t sb = s0 + gw; sb < s1; sb += 32u * static_cast<uint32_t>(nw)) {
    const uint32_t sj = sb + static_cast<uint32_t>(lane) * static_cast<uint32_t>(nw);
    uint4 q = make_uint4(kDummyCol, 0u, 0u, 0u);
    float sc = 0.f;
    if (sj < s1) {
      q.x = a.seg_col[sj];
      q.y = a.seg_start[sj];
      q.z = a.seg_start[sj + 1];
    }
    const bool use = !skip(q.x);
    if (use && q.z - q.y == 1) {
      q.w = a.ent_val[q.y];
      sc = a.scal[q.w & 0x7fffffffu];
    }
    __syncwarp();
    myq[lane] = q;
    mysc[lane] = sc;
    for (unsigned m = __ballot_sync(kFull, use); m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const uint4 qj = myq[j];
      segment_rows<KIND, SGD, 4, 1, KB>(a, qj.x, qj.y, qj.z, qj.z - qj.y == 1, qj.w, mysc[j], lane);
    }
  }
}

// One warp per column segment; CH vector chunks per lane per pass (CH = 1
// covers d <= 128 with float4 lanes). Up to KB residual rows are in flight
// per round; the adds stay in the segment's entry order.
// Debug: per-warp start / end stamps (globaltimer) and segment mix of one
// chosen minibatch, off unless enabled through skg_debug_bwd_trace.
constexpr int kBwTrWarps = 148 * 64;
__device__ unsigned long long g_bwtrace[kBwTrWarps * 2];
__device__ uint32_t g_bwtrace_info[kBwTrWarps];  // relation segments << 16 | entries
__device__ int g_bwtrace_on;

template <int KIND, bool SGD, int VEC, int CH, int KB = SKG_BWD_KB>
__global__ void __launch_bounds__(kThreads) segment_backward_kernel(const BwdArgs a) {
  using V = typename VecT<VEC>::T;
  if (a.err[0] != 0) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
#ifdef SKG_BWD_TRACE  // debug build only: the stamps cost registers (C5: 80 -> 87, one block per SM less)
  const bool trc = g_bwtrace_on == a.batch + 1 && gw < kBwTrWarps;
  uint32_t tr_info = 0;
  if (trc && lane == 0) stamp_now(&g_bwtrace[2 * gw]);
#endif
  const uint32_t s0 = a.seg_base[a.batch], s1 = a.seg_base[a.batch + 1];
  const int dv = a.d / VEC;
  const V* RV = reinterpret_cast<const V*>(a.res);
  for (uint32_t s = s0 + gw; s < s1; s += nw) {
    const uint32_t col = a.seg_col[s];
#ifdef SKG_BWD_TRACE
    if (trc) tr_info += (col >= static_cast<uint32_t>(a.N) && col != kDummyCol ? (1u << 16) : 0u) +
                        (col != kDummyCol ? a.seg_start[s + 1] - a.seg_start[s] : 0u);
#endif
    if (col == kDummyCol || (a.entity_only && col >= static_cast<uint32_t>(a.N))) continue;
    const uint32_t e0 = a.seg_start[s], e1 = a.seg_start[s + 1];
    V* P = reinterpret_cast<V*>(a.X) + static_cast<size_t>(col) * dv;
    for (int cb = 0; cb < dv; cb += 32 * CH) {
      int c[CH];
      bool has[CH];
      V acc[CH], p[CH];
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        c[h] = cb + 32 * h + lane;
        has[h] = c[h] < dv;
        acc[h] = V{};
        p[h] = V{};
        // the owner warp is the only writer of this row: load it up front
        if (has[h]) p[h] = P[c[h]];
        if (!SGD) acc[h] = p[h];  // accumulate into an existing sink (score_backward)
      }
      for (uint32_t eb = e0; eb < e1; eb += 32) {
        const int cnt = min(32u, e1 - eb);
        uint32_t myv = 0;
        float mysc = 0.f;
        if (lane < cnt) {
          myv = a.ent_val[eb + lane];
          mysc = a.scal[myv & 0x7fffffffu];
        }
        unsigned live = __ballot_sync(kFull, lane < cnt && mysc != 0.f);
        while (live) {
          int k[KB];
          int n = 0;
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            k[q] = live ? __ffs(live) - 1 : 0;
            if (live) {
              live &= live - 1;
              ++n;
            }
          }
          uint32_t vq[KB];
          float scq[KB];
          V rv[KB][CH];
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            vq[q] = __shfl_sync(kFull, myv, k[q]);
            scq[q] = __shfl_sync(kFull, mysc, k[q]);
            size_t rowoff = static_cast<size_t>(vq[q] & 0x7fffffffu) * dv;
            if (KIND == kMultRows) {  // the entry's own gradient plane: head, tail or relation
              const uint32_t slot = col >= static_cast<uint32_t>(a.N) ? 2u : (vq[q] >> 31);
              rowoff += static_cast<size_t>(slot) * a.plane_rows * dv;
            }
#pragma unroll
            for (int h = 0; h < CH; ++h)
              if (q < n && has[h]) rv[q][h] = __ldg(RV + rowoff + c[h]);
          }
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (q < n) {
              const bool neg = KIND != kMultRows && (vq[q] >> 31) != 0;
#pragma unroll
              for (int h = 0; h < CH; ++h)
                if (has[h]) acc_add<KIND>(acc[h], rv[q][h], scq[q], neg);
            }
        }
      }
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        if (!has[h]) continue;
        if (SGD) P[c[h]] = sgd1(p[h], acc[h], *a.lr);
        else P[c[h]] = acc[h];
      }
    }
  }
#ifdef SKG_BWD_TRACE
  if (trc && lane == 0) {
    stamp_now(&g_bwtrace[2 * gw + 1]);
    g_bwtrace_info[gw] = tr_info;
  }
#endif
}


template <int KIND, bool TRAIN, int VEC>
void launch_fwd_t(const FwdArgs& a, int num_sms, cudaStream_t s) {
  constexpr size_t kSmemCap = 200 * 1024;
  // d > 128 (DRAM-resident wide tables, C5): 4-pair tiles, half the shared
  // memory per warp, so twice the warps (and row loads) in flight per SM
  // (TransE only: the torus sums are lane-serial, so their 16-row tiles stay)
  const bool small_tile = TRAIN && VEC == 4 && (KIND == kTransE_L2 || KIND == kTransE_L1) && a.de > 128 &&
                          std::getenv("SKG_FWD_TILE8") == nullptr;
  const int S = VEC == 4 ? a.de + 4 : a.de + 1;
  const size_t per_warp = static_cast<size_t>(small_tile ? 8 : 16) * S * sizeof(float);
  if (per_warp > kSmemCap) throw CudaError("hrt_forward: embedding dimension too large for the staged tile");
  int wpb = static_cast<int>(kSmemCap / 3 / per_warp);  // aim for >= 3 resident blocks per SM
  wpb = wpb < 1 ? 1 : (wpb > kWarps ? kWarps : wpb);
  const size_t smem = wpb * per_warp;
  const int units = TRAIN ? (small_tile ? 4 : 8) : 16;
  const int ntiles = (a.B + units - 1) / units;
  int per_sm = static_cast<int>(kSmemCap / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  int grid = (ntiles + wpb - 1) / wpb;
  if (grid > num_sms * per_sm) grid = num_sms * per_sm;
  if (grid < 1) grid = 1;
  // d > 128: three blocks' worth of registers per SM (more rows in flight for
  // the DRAM-resident wide tables; C5 +3 %), d <= 128: two (C1 -1.5 % with three)
  const bool sharded = a.ent_peer[0] != nullptr;
  if (sharded && !(TRAIN && VEC == 4)) throw CudaError("hrt_forward: sharded tables need training mode and d % 4 == 0");
  if (sharded && TRAIN && VEC == 4) {
    if (small_tile) hrt_forward_kernel<KIND, true, 4, SKG_FWD_MINB_SMALL, 4, true><<<grid, wpb * 32, smem, s>>>(a);
    else if (a.de > 128) hrt_forward_kernel<KIND, true, 4, 3, 8, true><<<grid, wpb * 32, smem, s>>>(a);
    else hrt_forward_kernel<KIND, true, 4, SKG_FWD_MINB, 8, true><<<grid, wpb * 32, smem, s>>>(a);
  } else if (small_tile) hrt_forward_kernel<KIND, TRAIN, VEC, SKG_FWD_MINB_SMALL, 4><<<grid, wpb * 32, smem, s>>>(a);
  else if (a.de > 128) hrt_forward_kernel<KIND, TRAIN, VEC, 3><<<grid, wpb * 32, smem, s>>>(a);
  else hrt_forward_kernel<KIND, TRAIN, VEC><<<grid, wpb * 32, smem, s>>>(a);
  count_launch();
  SKG_LAUNCH_CHECK();
}

template <int KIND>
void launch_fwd_k(bool train, const FwdArgs& a, int num_sms, cudaStream_t s) {
  const bool v4 = (a.de % 4) == 0;
  if (train) {
    if (v4) launch_fwd_t<KIND, true, 4>(a, num_sms, s);
    else launch_fwd_t<KIND, true, 1>(a, num_sms, s);
  } else {
    if (v4) launch_fwd_t<KIND, false, 4>(a, num_sms, s);
    else launch_fwd_t<KIND, false, 1>(a, num_sms, s);
  }
}

// Grid of a grid-stride backward kernel. The warp-per-segment kernel launches
// 64 warps per SM in 128-thread blocks: about two waves, and the second wave's
// blocks take over SMs as first-wave blocks finish, which balances the uneven
// segments better than a resident grid (measured: C1 23.0 vs 26.7 us, C5 313
// vs 516 us); 4-warp blocks hand SMs over sooner than 8-warp ones (epoch C3
// 0.754 -> 0.732 ms, C1 0.653 -> 0.647, M1-M3 -0.7 %; SKG_BWD_TPB=256 restores).
// The staged ht entity pass (mostly one-entry segments) runs every block at
// once (C2 17.9 -> 16.5 us).
template <class K>
int resident_grid(K kernel, int num_sms) {
  int per_sm = 0;
  SKG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
  return num_sms * (per_sm > 0 ? per_sm : 1);
}

inline int bwd_tpb() {
  static const int v = [] {
    const char* e = std::getenv("SKG_BWD_TPB");
    const int t = e ? std::atoi(e) : 128;
    return (t == 64 || t == 128 || t == 256) ? t : kThreads;
  }();
  return v;
}

template <class K>
void run_bwd(K kernel, const BwdArgs& a, int num_sms, cudaStream_t s, bool resident = false) {
  if (resident) {
    kernel<<<resident_grid(kernel, num_sms), kThreads, 0, s>>>(a);
    return;
  }
  const int tpb = bwd_tpb();
  kernel<<<num_sms * 8 * (kThreads / tpb), tpb, 0, s>>>(a);
}

template <int KIND>
void launch_bwd_k(bool sgd, const BwdArgs& a, int num_sms, cudaStream_t s) {
  const bool v4 = (a.d % 4) == 0;
  const bool narrow = v4 ? a.d <= 128 : a.d <= 32;
  if constexpr (KIND == kTileSlotRows) {
    if (a.d > 128 || a.d % kDuGroup != 0) throw CudaError("tile-blocked dU rows need d <= 128, a multiple of 16");
    if (sgd) run_bwd(segment_backward_staged_kernel<true, kTileSlotRows>, a, num_sms, s, true);
    else run_bwd(segment_backward_staged_kernel<false, kTileSlotRows>, a, num_sms, s, true);
  } else if (KIND == kPlainRows && v4 && narrow) {
    if (sgd) run_bwd(segment_backward_staged_kernel<true>, a, num_sms, s, true);
    else run_bwd(segment_backward_staged_kernel<false>, a, num_sms, s, true);
  } else if (sgd) {
    if (v4) {
      if (narrow) run_bwd(segment_backward_kernel<KIND, true, 4, 1>, a, num_sms, s);
      else if (KIND == kTorusE_L2 || KIND == kTorusE_L1)  // L2-resident wide rows: 8 in flight (C3 -9%)
        run_bwd(segment_backward_kernel<KIND, true, 4, 2, 8>, a, num_sms, s);
      else run_bwd(segment_backward_kernel<KIND, true, 4, 2>, a, num_sms, s);
    } else {
      if (narrow) run_bwd(segment_backward_kernel<KIND, true, 1, 1>, a, num_sms, s);
      else run_bwd(segment_backward_kernel<KIND, true, 1, 2>, a, num_sms, s);
    }
  } else {
    if (v4) {
      if (narrow) run_bwd(segment_backward_kernel<KIND, false, 4, 1>, a, num_sms, s);
      else run_bwd(segment_backward_kernel<KIND, false, 4, 2>, a, num_sms, s);
    } else {
      if (narrow) run_bwd(segment_backward_kernel<KIND, false, 1, 1>, a, num_sms, s);
      else run_bwd(segment_backward_kernel<KIND, false, 1, 2>, a, num_sms, s);
    }
  }
  count_launch();
  SKG_LAUNCH_CHECK();
}

template <int KIND, bool TRAIN, int VEC>
void configure_one() {
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, TRAIN, VEC>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, TRAIN, VEC, 3>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, TRAIN, VEC, SKG_FWD_MINB_SMALL, 4>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
}
template <int KIND>
void configure_kind() {
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, true, 4, SKG_FWD_MINB, 8, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, true, 4, 3, 8, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SKG_CUDA(cudaFuncSetAttribute(hrt_forward_kernel<KIND, true, 4, SKG_FWD_MINB_SMALL, 4, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  configure_one<KIND, true, 4>();
  configure_one<KIND, true, 1>();
  configure_one<KIND, false, 4>();
  configure_one<KIND, false, 1>();
}

}  // namespace

// Opt every staged-tile kernel into > 48 KB dynamic shared memory. Called once
// per context at creation, outside any stream capture.
int64_t bwd_trace(int enable, unsigned long long* out, uint32_t* info, int64_t cap) {
  SKG_CUDA(cudaMemcpyToSymbol(g_bwtrace_on, &enable, sizeof(int)));
  if (enable) {
    static const unsigned long long z[kBwTrWarps * 2] = {};
    static const uint32_t zi[kBwTrWarps] = {};
    SKG_CUDA(cudaMemcpyToSymbol(g_bwtrace, z, sizeof(z)));
    SKG_CUDA(cudaMemcpyToSymbol(g_bwtrace_info, zi, sizeof(zi)));
  }
  if (out && cap >= kBwTrWarps) {
    SKG_CUDA(cudaMemcpyFromSymbol(out, g_bwtrace, sizeof(unsigned long long) * 2 * kBwTrWarps));
    SKG_CUDA(cudaMemcpyFromSymbol(info, g_bwtrace_info, sizeof(uint32_t) * kBwTrWarps));
  }
  return kBwTrWarps;
}

void configure_hrt_kernels() {
  configure_kind<kTransE_L2>();
  configure_kind<kTransE_L1>();
  configure_kind<kTorusE_L2>();
  configure_kind<kTorusE_L1>();
}

void launch_hrt_forward(int kind, bool train, const FwdArgs& a, int num_sms, cudaStream_t s) {
  switch (kind) {
    case kTransE_L2: launch_fwd_k<kTransE_L2>(train, a, num_sms, s); break;
    case kTransE_L1: launch_fwd_k<kTransE_L1>(train, a, num_sms, s); break;
    case kTorusE_L2: launch_fwd_k<kTorusE_L2>(train, a, num_sms, s); break;
    case kTorusE_L1: launch_fwd_k<kTorusE_L1>(train, a, num_sms, s); break;
    default: throw CudaError("launch_hrt_forward: not an hrt kind");
  }
}

void launch_segment_backward(int kind, bool sgd, const BwdArgs& a, int num_sms, cudaStream_t s) {
  switch (kind) {
    case kTransE_L2: launch_bwd_k<kTransE_L2>(sgd, a, num_sms, s); break;
    case kTransE_L1: launch_bwd_k<kTransE_L1>(sgd, a, num_sms, s); break;
    case kTorusE_L2: launch_bwd_k<kTorusE_L2>(sgd, a, num_sms, s); break;
    case kTorusE_L1: launch_bwd_k<kTorusE_L1>(sgd, a, num_sms, s); break;
    case kPlainRows: launch_bwd_k<kPlainRows>(sgd, a, num_sms, s); break;
    case kMultRows: launch_bwd_k<kMultRows>(sgd, a, num_sms, s); break;
    case kTileSlotRows: launch_bwd_k<kTileSlotRows>(sgd, a, num_sms, s); break;
    default: throw CudaError("launch_segment_backward: unsupported kind");
  }
}

}  // namespace skg
