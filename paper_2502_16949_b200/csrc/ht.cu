// ht-layout models on device.
//
// TransH (models.cpp:158-199, models.hpp:99-113). A warp owns a tile of 8
// (pos, neg) pairs = 16 rows. Per row it gathers h, t (entity), d_r (relation)
// and w_r (normal), forms u = h - t (bitwise the ht CSR row, sparse.hpp:211-237),
// wu = w.u (fixed warp tree; the reference uses Eigen's redux, so TransH parity
// is tolerance-only) and v = (u + d_r) - wu w. The score reduction uses the
// reference's exact squared_sum / abs_sum order on v staged in shared memory.
// After the hinge each active row emits
//   du  = dz - (dz.w) w                   -> entity scatter (sorted ht segments)
//   dz                                    -> relation gradient
//   nrm = (dz.w) u + (w.u) dz             -> normal gradient (subtracted)
// with dz = v / ||v||_eps * up (L2) or sign(v) * up (L1). Relation-side sums
// are deterministic two-level reductions over the relation's rows (plan
// segments, rows ascending); SGD on relation rows and normals is fused into the
// second level, followed by the renormalization of every normal
// (embedding.cpp:181-189).
//
// TransR (models.cpp:110-156, models.hpp:82-96) lives in transr.cu.
#include <algorithm>

#include "common.cuh"
#include "ht.cuh"
#include "plan.cuh"
#include "primitives.cuh"
#include "refmath.cuh"

namespace skg {

namespace {

constexpr int kHtThreads = 128;
constexpr int kRelParts = 64;  // first-level partial blocks per relation segment

enum Mode : int { kTrain = 0, kScore = 1, kPrep = 2 };

template <int VEC>
struct V;
template <>
struct V<4> {
  using T = float4;
};
template <>
struct V<1> {
  using T = float;
};

__device__ __forceinline__ float4 ld(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float ld(const float* p) { return __ldg(p); }
__device__ __forceinline__ float dot_acc(float acc, float4 a, float4 b) {
  acc = fmaf(a.x, b.x, acc);
  acc = fmaf(a.y, b.y, acc);
  acc = fmaf(a.z, b.z, acc);
  return fmaf(a.w, b.w, acc);
}
__device__ __forceinline__ float dot_acc(float acc, float a, float b) { return fmaf(a, b, acc); }
__device__ __forceinline__ float4 sub(float4 a, float4 b) {
  return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z), __fsub_rn(a.w, b.w));
}
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float4 add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float4 scale(float s, float4 a) {
  return make_float4(__fmul_rn(s, a.x), __fmul_rn(s, a.y), __fmul_rn(s, a.z), __fmul_rn(s, a.w));
}
__device__ __forceinline__ float scale(float s, float a) { return __fmul_rn(s, a); }
template <bool L2>
__device__ __forceinline__ float dir(float v, float sc) {
  return L2 ? __fmul_rn(v, sc) : (v > 0.f ? sc : (v < 0.f ? -sc : 0.f));
}
template <bool L2>
__device__ __forceinline__ float4 dir(float4 v, float sc) {
  return make_float4(dir<L2>(v.x, sc), dir<L2>(v.y, sc), dir<L2>(v.z, sc), dir<L2>(v.w, sc));
}

// Shared deterministic loss finalization (warp -> block -> last block).
__device__ void finalize_loss(const FwdArgs& a, float lsum, float* warp_loss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
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
      const float loss = __fdiv_rn(acc, static_cast<float>(a.B));
      a.batch_loss[a.batch] = loss;
      if (a.stamp_end) stamp_now(a.stamp_end);
      const uint32_t pflags = *reinterpret_cast<volatile uint32_t*>(&a.err[3]);
      if (nonfinite(loss)) {
        a.err[1] = a.batch;
        atomicCAS(&a.err[0], 0u, static_cast<uint32_t>(kErrLossNonFinite));
      } else if (pflags) {
        a.err[1] = a.batch;
        const uint32_t code = (pflags & kPendEntity)     ? kErrGradEntity
                              : (pflags & kPendRelation) ? kErrGradRelation
                              : (pflags & kPendProj)     ? kErrGradProj
                                                         : kErrGradNormals;
        atomicCAS(&a.err[0], 0u, code);
      }
      a.err[3] = 0;
      *a.counter = 0;
    }
  }
}

template <bool L2, int MODE, int VEC>
__global__ void __launch_bounds__(kHtThreads) transh_forward_kernel(const FwdArgs a, float* __restrict__ nrm_out) {
  using T = typename V<VEC>::T;
  extern __shared__ float4 sm4[];
  __shared__ float warp_loss[kHtThreads / 32];
  if (a.err[0] != 0) return;
  if (a.stamp_start && blockIdx.x == 0 && threadIdx.x == 0) stamp_now(a.stamp_start);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int d = a.de;
  const int dv = d / VEC;
  const int S = VEC == 4 ? d + 4 : d + 1;
  float* U = reinterpret_cast<float*>(sm4) + warp * 32 * S;
  float* Vt = U + 16 * S;
  const T* E = reinterpret_cast<const T*>(a.X);
  const T* RELT = reinterpret_cast<const T*>(a.X + a.N * static_cast<int64_t>(d));
  const T* W = reinterpret_cast<const T*>(a.normals);
  constexpr int kUnits = MODE == kTrain ? 8 : 16;
  const int ntiles = (a.B + kUnits - 1) / kUnits;
  float lsum = 0.f;
  uint32_t pend = 0;

  for (int tile = blockIdx.x * nwarps + warp; tile < ntiles; tile += gridDim.x * nwarps) {
    int h = 0, t = 0, r = 0, row2 = 0;
    bool valid = false;
    if (lane < 16) {
      if (MODE == kTrain) {
        const int p = tile * 8 + (lane & 7);
        const bool neg = lane >= 8;
        valid = p < a.B;
        if (valid) {
          const int id = a.order[p];
          h = neg ? a.NH[id] : a.H[id];
          t = neg ? a.NT[id] : a.T[id];
          r = a.Rl[id];
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
    float my_wu = 0.f;
    // ---- u, wu, v for the 16 rows (hyperplane_forward, models.hpp:99-103)
    for (int j = 0; j < 16; ++j) {
      const int hj = __shfl_sync(kFull, h, j), tj = __shfl_sync(kFull, t, j), rj = __shfl_sync(kFull, r, j);
      float part = 0.f;
      for (int c = lane; c < dv; c += 32) {
        const T u = sub(ld(E + static_cast<size_t>(hj) * dv + c), ld(E + static_cast<size_t>(tj) * dv + c));
        *reinterpret_cast<T*>(U + j * S + VEC * c) = u;
        part = dot_acc(part, ld(W + static_cast<size_t>(rj) * dv + c), u);
      }
      const float wu = warp_sum_bcast(part);
      if (lane == j) my_wu = wu;
      for (int c = lane; c < dv; c += 32) {
        const T u = *reinterpret_cast<const T*>(U + j * S + VEC * c);
        const T w = ld(W + static_cast<size_t>(rj) * dv + c);
        *reinterpret_cast<T*>(Vt + j * S + VEC * c) = sub(add(u, ld(RELT + static_cast<size_t>(rj) * dv + c)), scale(wu, w));
      }
    }
    __syncwarp();
    float s = 0.f, score = 0.f;
    bool bad = false;
    if (lane < 16 && valid) {
      s = ref_norm_sum<L2, VEC>(Vt + lane * S, d, bad);
      score = L2 ? __fsqrt_rn(s) : s;
    }
    float up = 0.f;
    bool act = false;
    if (MODE == kTrain) {
      const float ns = __shfl_down_sync(kFull, score, 8);
      float term = 0.f;
      if (lane < 8 && valid) {
        term = __fsub_rn(__fadd_rn(a.margin, score), ns);
        act = term > 0.f;
      }
      const float tk = act ? term : 0.f;
      float tsum = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) tsum = __fadd_rn(tsum, __shfl_sync(kFull, tk, k));
      lsum = __fadd_rn(lsum, tsum);
      act = __shfl_sync(kFull, act, lane & 7) && lane < 16 && valid;
      up = act ? (lane < 8 ? a.unit : -a.unit) : 0.f;
    } else if (MODE == kPrep) {
      act = lane < 16 && valid;
      up = act ? a.upstream[row2] : 0.f;
      act = act && up != 0.f;
    }
    float sc = 0.f;
    if (act) sc = L2 ? __fdiv_rn(up, __fsqrt_rn(__fadd_rn(s, kNormEpsF))) : up;
    if (bad && (L2 || act)) pend |= kPendEntity;

    if (MODE == kScore) {
      if (lane < 16 && valid) a.scores[row2] = score;
      for (unsigned m = vmask; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const int r2 = __shfl_sync(kFull, row2, j);
        for (int c = lane; c < dv; c += 32) {
          reinterpret_cast<T*>(a.res + static_cast<size_t>(r2) * d)[c] = *reinterpret_cast<const T*>(Vt + j * S + VEC * c);
          reinterpret_cast<T*>(a.res_u + static_cast<size_t>(r2) * d)[c] = *reinterpret_cast<const T*>(U + j * S + VEC * c);
        }
      }
    } else {
      if (lane < 16 && valid) a.scal[row2] = act ? 1.f : 0.f;
      const unsigned amask = __ballot_sync(kFull, act);
      for (unsigned m = amask; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const int r2 = __shfl_sync(kFull, row2, j), rj = __shfl_sync(kFull, r, j);
        const float scj = __shfl_sync(kFull, sc, j), wuj = __shfl_sync(kFull, my_wu, j);
        float part = 0.f;
        for (int c = lane; c < dv; c += 32)
          part = dot_acc(part, dir<L2>(*reinterpret_cast<const T*>(Vt + j * S + VEC * c), scj),
                         ld(W + static_cast<size_t>(rj) * dv + c));
        const float dzw = warp_sum_bcast(part);  // hyperplane_backward, models.hpp:106-113
        for (int c = lane; c < dv; c += 32) {
          const T dz = dir<L2>(*reinterpret_cast<const T*>(Vt + j * S + VEC * c), scj);
          const T w = ld(W + static_cast<size_t>(rj) * dv + c);
          const T u = *reinterpret_cast<const T*>(U + j * S + VEC * c);
          reinterpret_cast<T*>(a.res_u + static_cast<size_t>(r2) * d)[c] = sub(dz, scale(dzw, w));
          reinterpret_cast<T*>(a.res + static_cast<size_t>(r2) * d)[c] = dz;
          reinterpret_cast<T*>(nrm_out + static_cast<size_t>(r2) * d)[c] = add(scale(dzw, u), scale(wuj, dz));
        }
      }
    }
    __syncwarp();
  }
  pend = __reduce_or_sync(kFull, pend);
  if (lane == 0 && pend) {
    atomicOr(&a.err[3], pend);
    __threadfence();
  }
  if (MODE == kTrain) finalize_loss(a, lsum, warp_loss);
}

// First level of the relation-side reduction: block (k, part) sums rows of
// its slice of relation segment k (entries ascending), for two row sources.
struct RelArgs {
  const uint32_t* ent_val;
  const uint32_t* seg_start;
  const uint32_t* seg_col;
  const uint32_t* seg_base;
  int batch;
  int64_t N;
  const float* scal;
  const float* srcA;  // dz rows -> relation gradient
  const float* srcB;  // nrm rows -> normal gradient (negated)
  int d;
  float* partial;  // [R][kRelParts][2][d]
  // second level
  float* rel;       // relation table (SGD) or sink (accumulate)
  float* normals;   // normals table (SGD) or sink
  const float* lr;
  bool sgd;
  const uint32_t* err;
};

__device__ __forceinline__ bool rel_segment(const RelArgs& a, int k, uint32_t& s) {
  const uint32_t s0 = a.seg_base[a.batch], s1 = a.seg_base[a.batch + 1];
  s = s0 + k;
  return s < s1 && a.seg_col[s] >= static_cast<uint32_t>(a.N) && a.seg_col[s] != kDummyCol;
}

__global__ void __launch_bounds__(128) rel_partial_kernel(const RelArgs a) {
  __shared__ float part[4][2][128];
  if (a.err[0] != 0) return;
  uint32_t s;
  if (!rel_segment(a, blockIdx.x, s)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t e0 = a.seg_start[s], e1 = a.seg_start[s + 1], len = e1 - e0;
  const uint32_t p0 = e0 + static_cast<uint32_t>((static_cast<uint64_t>(len) * blockIdx.y) / kRelParts);
  const uint32_t p1 = e0 + static_cast<uint32_t>((static_cast<uint64_t>(len) * (blockIdx.y + 1)) / kRelParts);
  const uint32_t w0 = p0 + static_cast<uint32_t>((static_cast<uint64_t>(p1 - p0) * warp) / 4);
  const uint32_t w1 = p0 + static_cast<uint32_t>((static_cast<uint64_t>(p1 - p0) * (warp + 1)) / 4);
  const int d = a.d;
  for (int cb = 0; cb < d; cb += 128) {
    float accA[4], accB[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) accA[q] = accB[q] = 0.f;
    // entries in order; row ids and activity fetched 32 at a time, rows of
    // four live entries loaded together (independent loads in flight)
    for (uint32_t g = w0; g < w1; g += 32) {
      const uint32_t cnt = min(32u, w1 - g);
      uint32_t myrow = 0;
      bool mylive = false;
      if (lane < cnt) {
        myrow = a.ent_val[g + lane] & 0x7fffffffu;
        mylive = a.scal[myrow] != 0.f;
      }
      unsigned live = __ballot_sync(kFull, mylive);
      while (live) {
        int n = 0;
        uint32_t rows[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = live ? __ffs(live) - 1 : 0;
          rows[q] = __shfl_sync(kFull, myrow, k);
          if (live) {
            live &= live - 1;
            ++n;
          }
        }
        float va[4][4], vb[4][4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = cb + lane + 32 * q;
            const bool ok = e < n && c < d;
            va[e][q] = ok ? __ldg(a.srcA + static_cast<size_t>(rows[e]) * d + c) : 0.f;
            vb[e][q] = ok ? __ldg(a.srcB + static_cast<size_t>(rows[e]) * d + c) : 0.f;
          }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < n)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              accA[q] = __fadd_rn(accA[q], va[e][q]);
              accB[q] = __fadd_rn(accB[q], vb[e][q]);
            }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      part[warp][0][lane + 32 * q] = accA[q];
      part[warp][1][lane + 32 * q] = accB[q];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 128 && cb + c < d; c += blockDim.x) {
      float x = 0.f, y = 0.f;
      for (int w = 0; w < 4; ++w) {
        x = __fadd_rn(x, part[w][0][c]);
        y = __fadd_rn(y, part[w][1][c]);
      }
      float* out = a.partial + ((static_cast<size_t>(blockIdx.x) * kRelParts + blockIdx.y) * 2) * d;
      out[cb + c] = x;
      out[d + cb + c] = y;
    }
    __syncthreads();
  }
}

// Second level: sum the parts in order, then SGD (or accumulate into sinks).
__global__ void rel_apply_kernel(const RelArgs a) {
  if (a.err[0] != 0) return;
  uint32_t s;
  if (!rel_segment(a, blockIdx.x, s)) return;
  const int64_t r = a.seg_col[s] - a.N;
  const int d = a.d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float gA = 0.f, gB = 0.f;
    for (int p = 0; p < kRelParts; ++p) {
      const float* in = a.partial + ((static_cast<size_t>(blockIdx.x) * kRelParts + p) * 2) * d;
      gA = __fadd_rn(gA, in[c]);
      gB = __fadd_rn(gB, in[d + c]);
    }
    float* pr = a.rel + r * d + c;
    float* pn = a.normals + r * d + c;
    if (a.sgd) {
      const float lr = *a.lr;
      *pr = __fsub_rn(*pr, __fmul_rn(lr, gA));
      *pn = __fsub_rn(*pn, __fmul_rn(lr, -gB));  // grads.normals -= nrm (models.hpp:112)
    } else {
      *pr = __fadd_rn(*pr, gA);
      *pn = __fsub_rn(*pn, gB);
    }
  }
}

// embedding.cpp:181-189: every normal back to unit length after the step.
__global__ void normals_renorm_kernel(float* __restrict__ w, int64_t rows, int d, uint32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  if (err[0] != 0) return;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    float* row = w + r * d;
    float s = 0.f;
    for (int j = lane; j < d; j += 32) s = __fadd_rn(s, __fmul_rn(row[j], row[j]));
    const float n = __fsqrt_rn(warp_sum_bcast(s));
    if (!(n > 0.f)) {
      if (lane == 0 && atomicCAS(&err[0], 0u, static_cast<uint32_t>(kErrNormalCollapsed)) == 0u)
        err[2] = static_cast<uint32_t>(r);
      continue;
    }
    for (int j = lane; j < d; j += 32) row[j] = __fdiv_rn(row[j], n);
  }
}

template <bool L2, int MODE, int VEC>
void launch_transh_t(const FwdArgs& a, float* nrm, int num_sms, cudaStream_t s) {
  const int S = VEC == 4 ? a.de + 4 : a.de + 1;
  const size_t per_warp = static_cast<size_t>(32) * S * sizeof(float);
  int wpb = static_cast<int>((64 * 1024) / per_warp);
  wpb = wpb < 1 ? 1 : (wpb > 4 ? 4 : wpb);
  const size_t smem = wpb * per_warp;
  if (smem > 200 * 1024) throw CudaError("transh: embedding dimension too large for the staged tile");
  const int units = MODE == kTrain ? 8 : 16;
  const int ntiles = (a.B + units - 1) / units;
  int grid = (ntiles + wpb - 1) / wpb;
  const int cap = num_sms * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  transh_forward_kernel<L2, MODE, VEC><<<grid, wpb * 32, smem, s>>>(a, nrm);
  count_launch();
  SKG_LAUNCH_CHECK();
}

template <int MODE>
void launch_transh(int kind, const FwdArgs& a, float* nrm, int num_sms, cudaStream_t s) {
  const bool l2 = kind == kTransH_L2;
  const bool v4 = a.de % 4 == 0;
  if (l2) {
    if (v4) launch_transh_t<true, MODE, 4>(a, nrm, num_sms, s);
    else launch_transh_t<true, MODE, 1>(a, nrm, num_sms, s);
  } else {
    if (v4) launch_transh_t<false, MODE, 4>(a, nrm, num_sms, s);
    else launch_transh_t<false, MODE, 1>(a, nrm, num_sms, s);
  }
}

template <bool L2, int MODE, int VEC>
void configure_transh_one() {
  SKG_CUDA(cudaFuncSetAttribute(transh_forward_kernel<L2, MODE, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                200 * 1024));
}

void launch_relation_side(const FwdArgs& fa, const BwdArgs& ba, float* partial, float* rel, float* normals,
                          bool sgd, int64_t R, const float* nrm, cudaStream_t s) {
  RelArgs ra{};
  ra.ent_val = ba.ent_val;
  ra.seg_start = ba.seg_start;
  ra.seg_col = ba.seg_col;
  ra.seg_base = ba.seg_base;
  ra.batch = ba.batch;
  ra.N = ba.N;
  ra.scal = ba.scal;
  ra.srcA = fa.res;
  ra.srcB = nrm;
  ra.d = fa.de;
  ra.partial = partial;
  ra.rel = rel;
  ra.normals = normals;
  ra.lr = ba.lr;
  ra.sgd = sgd;
  ra.err = ba.err;
  rel_partial_kernel<<<dim3(static_cast<unsigned>(R), kRelParts), 128, 0, s>>>(ra);
  rel_apply_kernel<<<static_cast<unsigned>(R), 128, 0, s>>>(ra);
  count_launch(2);
  SKG_LAUNCH_CHECK();
}

}  // namespace

void launch_normals_renorm(float* normals, int64_t R, int d, uint32_t* err, cudaStream_t s) {
  normals_renorm_kernel<<<static_cast<unsigned>((R * 32 + 127) / 128), 128, 0, s>>>(normals, R, d, err);
  count_launch();
  SKG_LAUNCH_CHECK();
}

// work layout (floats): [nrm rows: rows x d][partials: R x parts x 2 x d]
int64_t ht_work_floats(int kind, int64_t rows, int64_t de, int64_t dr, int64_t R) {
  if (kind == kTransR_L2 || kind == kTransR_L1) return transr_work_floats(rows, de, dr, R);
  return std::max<int64_t>(2 * rows * de + R * kRelParts * 2 * de + 64, transh_tiles_work_floats(rows, R));
}

void configure_ht_kernels() {
  configure_transh_tiles_kernels();
  configure_transh_one<true, kTrain, 4>();
  configure_transh_one<true, kTrain, 1>();
  configure_transh_one<true, kScore, 4>();
  configure_transh_one<true, kScore, 1>();
  configure_transh_one<true, kPrep, 4>();
  configure_transh_one<true, kPrep, 1>();
  configure_transh_one<false, kTrain, 4>();
  configure_transh_one<false, kTrain, 1>();
  configure_transh_one<false, kScore, 4>();
  configure_transh_one<false, kScore, 1>();
  configure_transh_one<false, kPrep, 4>();
  configure_transh_one<false, kPrep, 1>();
  configure_transr_kernels();
}

void ht_train_batch(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s,
                    const std::function<void()>* mark, int64_t R, const HtSinks* sinks, const Branch* br,
                    const ThTilePlan* tp, const TrTilePlan* trp) {
  if (kind == kTransR_L2 || kind == kTransR_L1) {
    transr_train_batch(kind, fa, ba, work, num_sms, s, mark, R, sinks, br, trp);
    return;
  }
  float* normals = const_cast<float*>(fa.normals);
  if (transh_tiles_supported(fa.de, fa.dr, R)) {  // relation-tiled path (transh_train.cu)
    // the tile kernel renormalizes the normals itself (data parallel: after the dense step)
    transh_tiles_train_batch(kind == kTransH_L2, fa, ba, work, R, num_sms, s, mark, sinks, br, tp);
    if (mark) (*mark)();
    return;
  }
  float* nrm = work;
  float* partial = work + static_cast<int64_t>(2 * fa.B) * fa.de;
  launch_transh<kTrain>(kind, fa, nrm, num_sms, s);
  if (mark) (*mark)();
  BwdArgs eb = ba;
  eb.entity_only = 1;
  launch_segment_backward(kPlainRows, sinks == nullptr, eb, num_sms, s);
  float* rel = sinks ? sinks->rel : const_cast<float*>(fa.X) + fa.N * static_cast<int64_t>(fa.de);
  launch_relation_side(fa, ba, partial, rel, sinks ? sinks->normals : normals, sinks == nullptr, R, nrm, s);
  if (!sinks) {
    normals_renorm_kernel<<<static_cast<unsigned>((R * 32 + 127) / 128), 128, 0, s>>>(normals, R, fa.de, ba.err);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
  if (mark) (*mark)();
}

void ht_score(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, int num_sms, cudaStream_t s, int64_t R) {
  if (kind == kTransR_L2 || kind == kTransR_L1) {
    transr_score(kind, fa, ba, work, num_sms, s, R);
    return;
  }
  launch_transh<kScore>(kind, fa, work, num_sms, s);
}

void ht_score_backward(int kind, const FwdArgs& fa, const BwdArgs& ba, float* work, float* g_proj, float* g_normals,
                       int num_sms, cudaStream_t s, int64_t R) {
  if (kind == kTransR_L2 || kind == kTransR_L1) {
    transr_score_backward(kind, fa, ba, work, g_proj, num_sms, s, R);
    return;
  }
  float* nrm = work;
  float* partial = work + static_cast<int64_t>(fa.B) * fa.de;
  launch_transh<kPrep>(kind, fa, nrm, num_sms, s);
  BwdArgs eb = ba;
  eb.entity_only = 1;
  launch_segment_backward(kPlainRows, false, eb, num_sms, s);
  launch_relation_side(fa, ba, partial, ba.Xrel, g_normals, false, R, nrm, s);
}

}  // namespace skg
