// Link-prediction ranking on device: rank_entity /
// evaluate (eval.cpp:16-96, TripleFilter eval.hpp:25-45).
//
// For a query (h, r, t) and a side, every entity c is a candidate: the tail
// side scores the incidence row (h, r, c), the head side (c, r, t). The
// candidate's energy is computed in the reference's exact arithmetic (the same
// as the training forward: v = (a - b) + r with the cancelled self-loop pair
// giving v = r, squared_sum / abs_sum with four strided accumulators for TransE,
// plain sequential sums of the wrapped residual for TorusE), so ranks are
// bit-exact with score_batch + the rank loop. rank = 1 + #{c != truth, not a
// known triple under the filtered protocol, energy(c) < energy(truth)}.
//
// Tiled kernel (d % 4 == 0): a CTA holds 16 queries' fixed and relation rows
// and streams 64 candidate rows at a time through shared memory; a thread
// scores 4 candidates against one query per 128-bit step (all arithmetic on
// the CUDA cores: the exact reference order rules out a GEMM reformulation).
// The filter is an open-addressing device hash set of the reference's triple
// key (h * R + r) * N + t, probed only for candidates that beat the truth.
#include <algorithm>

#include "common.cuh"
#include "ht.cuh"
#include "kernels.cuh"
#include "multmath.cuh"
#include "primitives.cuh"
#include "refmath.cuh"

namespace skg {

namespace {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kQB = 16;       // queries per CTA
constexpr int kCB = 64;       // candidates per shared-memory chunk
constexpr int kEvalThreads = 256;

__device__ __forceinline__ uint64_t triple_key(int64_t h, int64_t r, int64_t t, int64_t N, int64_t R) {
  return (static_cast<uint64_t>(h) * static_cast<uint64_t>(R) + static_cast<uint64_t>(r)) * static_cast<uint64_t>(N) +
         static_cast<uint64_t>(t);
}
__device__ __forceinline__ uint64_t mix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

__global__ void filter_insert_kernel(const int32_t* __restrict__ h, const int32_t* __restrict__ r,
                                     const int32_t* __restrict__ t, int64_t nf, int64_t N, int64_t R,
                                     uint64_t* __restrict__ table, uint64_t mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nf;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = triple_key(h[i], r[i], t[i], N, R);
    uint64_t slot = mix64(key) & mask;
    while (true) {
      const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + slot), kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) break;
      slot = (slot + 1) & mask;
    }
  }
}

__device__ __forceinline__ bool filter_contains(const uint64_t* __restrict__ table, uint64_t mask, uint64_t key) {
  uint64_t slot = mix64(key) & mask;
  while (true) {
    const uint64_t k = __ldg(reinterpret_cast<const unsigned long long*>(table + slot));
    if (k == key) return true;
    if (k == kEmptyKey) return false;
    slot = (slot + 1) & mask;
  }
}

constexpr bool is_torus(int K) { return K == kTorusE_L2 || K == kTorusE_L1; }

template <int KIND>
__device__ __forceinline__ float combine(float a, float b, float r, bool self_loop) {
  float v = self_loop ? r : __fadd_rn(__fsub_rn(a, b), r);
  if (is_torus(KIND)) v = torus_wrap(v);
  return v;
}
template <int KIND>
__device__ __forceinline__ float term(float x) {
  return (KIND == kTransE_L2 || KIND == kTorusE_L2) ? __fmul_rn(x, x) : fabsf(x);
}
template <int KIND>
__device__ __forceinline__ float finish(float s) {
  return KIND == kTransE_L2 ? __fsqrt_rn(s) : s;  // norms.hpp:57-62 (L2 sqrt), 107-115 (torus sums)
}

// Energy of the incidence row a - b + r read straight from the tables (any d):
// the reference's reduction order (ref_reduce in hrt.cu).
template <int KIND>
__device__ float row_energy(const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ r,
                            int d, bool self_loop) {
  if (is_torus(KIND) || d < 8) {
    float s = 0.f;
    for (int j = 0; j < d; ++j) s = __fadd_rn(s, term<KIND>(combine<KIND>(__ldg(a + j), __ldg(b + j), __ldg(r + j), self_loop)));
    return finish<KIND>(s);
  }
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int j = 0;
  for (; j + 4 <= d; j += 4) {
    s0 = __fadd_rn(s0, term<KIND>(combine<KIND>(__ldg(a + j), __ldg(b + j), __ldg(r + j), self_loop)));
    s1 = __fadd_rn(s1, term<KIND>(combine<KIND>(__ldg(a + j + 1), __ldg(b + j + 1), __ldg(r + j + 1), self_loop)));
    s2 = __fadd_rn(s2, term<KIND>(combine<KIND>(__ldg(a + j + 2), __ldg(b + j + 2), __ldg(r + j + 2), self_loop)));
    s3 = __fadd_rn(s3, term<KIND>(combine<KIND>(__ldg(a + j + 3), __ldg(b + j + 3), __ldg(r + j + 3), self_loop)));
  }
  float s = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
  for (; j < d; ++j) s = __fadd_rn(s, term<KIND>(combine<KIND>(__ldg(a + j), __ldg(b + j), __ldg(r + j), self_loop)));
  return finish<KIND>(s);
}

struct EvalArgs {
  const float* X;   // entity-side rows (the entity table, or a per-relation projected copy)
  const float* Rt;  // relation rows (R x d)
  int64_t N, R;
  int d;
  const int32_t *qh, *qr, *qt;
  int64_t q;
  int side;                  // 0 = tail (rows (h, r, c)), 1 = head (rows (c, r, t))
  const float* te;           // [q][2] true energies
  const uint64_t* table;     // filter hash set (null: raw protocol)
  uint64_t mask;
  uint32_t* better;          // [q][2]
};

template <int KIND>
__global__ void true_energy_kernel(EvalArgs a, float* __restrict__ te) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= 2 * a.q) return;
  const int64_t qi = i >> 1;
  const int side = static_cast<int>(i & 1);
  const int64_t h = a.qh[qi], r = a.qr[qi], t = a.qt[qi];
  const float* rel = a.Rt + r * a.d;
  // the truth row is the query itself on both sides: (h, r, t)
  te[i] = row_energy<KIND>(a.X + h * a.d, a.X + t * a.d, rel, a.d, h == t);
  (void)side;
}

// Generic path: thread per (query, candidate), tables read from L2.
template <int KIND>
__global__ void rank_simple_kernel(EvalArgs a) {
  const int64_t qi = blockIdx.y;
  const int64_t h = a.qh[qi], r = a.qr[qi], t = a.qt[qi];
  const int64_t fixed = a.side == 0 ? h : t, truth = a.side == 0 ? t : h;
  const float te = a.te[2 * qi + a.side];
  const float* rel = a.Rt + r * a.d;
  uint32_t cnt = 0;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < a.N;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (c == truth) continue;
    const float* pa = a.X + (a.side == 0 ? fixed : c) * a.d;
    const float* pb = a.X + (a.side == 0 ? c : fixed) * a.d;
    const float e = row_energy<KIND>(pa, pb, rel, a.d, c == fixed);
    if (!(e < te)) continue;
    if (a.table && filter_contains(a.table, a.mask, a.side == 0 ? triple_key(h, r, c, a.N, a.R)
                                                                 : triple_key(c, r, t, a.N, a.R)))
      continue;
    ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(kFull, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.better + 2 * qi + a.side, cnt);
}

// Tiled path (d % 4 == 0): 16 queries x 64-candidate chunks per CTA.
template <int KIND, int SIDE>
__global__ void __launch_bounds__(kEvalThreads) rank_tiled_kernel(EvalArgs a, int64_t cand_per_cta) {
  extern __shared__ float4 sm_eval[];
  const int d = a.d, S = d + 4;  // padded row stride (floats)
  float* F = reinterpret_cast<float*>(sm_eval);  // [kQB][S] fixed rows
  float* Rr = F + kQB * S;                       // [kQB][S] relation rows
  float* Cc = Rr + kQB * S;                      // [kCB][S] candidate rows
  __shared__ int64_t qfix[kQB], qtruth[kQB], qh[kQB], qr[kQB], qt[kQB];
  __shared__ float qte[kQB], qself[kQB];
  const int tid = threadIdx.x;
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kQB;
  const int nq = static_cast<int>(min(static_cast<int64_t>(kQB), a.q - q0));
  const int64_t c_lo = static_cast<int64_t>(blockIdx.y) * cand_per_cta;
  const int64_t c_hi = min(a.N, c_lo + cand_per_cta);
  if (tid < kQB) {
    const int64_t qi = q0 + min(tid, nq - 1);
    qh[tid] = a.qh[qi];
    qr[tid] = a.qr[qi];
    qt[tid] = a.qt[qi];
    qfix[tid] = SIDE == 0 ? qh[tid] : qt[tid];
    qtruth[tid] = SIDE == 0 ? qt[tid] : qh[tid];
    qte[tid] = a.te[2 * qi + SIDE];
    // the candidate equal to the fixed entity is the cancelled self-loop row
    // (energy of r alone); every other candidate skips that select in the loop
    qself[tid] = row_energy<KIND>(a.X + qfix[tid] * d, a.X + qfix[tid] * d, a.Rt + qr[tid] * d, d, true);
  }
  __syncthreads();
  const int d4 = d >> 2;
  for (int i = tid; i < kQB * d4; i += kEvalThreads) {
    const int qq = i / d4, c = i - qq * d4;
    reinterpret_cast<float4*>(F + qq * S)[c] = __ldg(reinterpret_cast<const float4*>(a.X + qfix[qq] * d) + c);
    reinterpret_cast<float4*>(Rr + qq * S)[c] =
        __ldg(reinterpret_cast<const float4*>(a.Rt + qr[qq] * d) + c);
  }
  const int qi = tid >> 4, cg = tid & 15;
  const float* fq = F + qi * S;
  const float* rq = Rr + qi * S;
  uint32_t cnt = 0;
  for (int64_t cb = c_lo; cb < c_hi; cb += kCB) {
    const int nc = static_cast<int>(min(static_cast<int64_t>(kCB), c_hi - cb));
    __syncthreads();  // previous chunk consumed (and the query rows on the first pass)
    for (int i = tid; i < nc * d4; i += kEvalThreads) {
      const int cc = i / d4, c = i - cc * d4;
      reinterpret_cast<float4*>(Cc + cc * S)[c] = __ldg(reinterpret_cast<const float4*>(a.X + (cb + cc) * d) + c);
    }
    __syncthreads();
    if (qi >= nq) continue;
    constexpr bool sl[4] = {false, false, false, false};
    float e[4];
    if (is_torus(KIND)) {
      float s[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < d; j += 4) {
        const float4 f = *reinterpret_cast<const float4*>(fq + j);
        const float4 r = *reinterpret_cast<const float4*>(rq + j);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 c = *reinterpret_cast<const float4*>(Cc + (cg + 16 * k) * S + j);
          const float4 A = SIDE == 0 ? f : c, B = SIDE == 0 ? c : f;
          s[k] = __fadd_rn(s[k], term<KIND>(combine<KIND>(A.x, B.x, r.x, sl[k])));
          s[k] = __fadd_rn(s[k], term<KIND>(combine<KIND>(A.y, B.y, r.y, sl[k])));
          s[k] = __fadd_rn(s[k], term<KIND>(combine<KIND>(A.z, B.z, r.z, sl[k])));
          s[k] = __fadd_rn(s[k], term<KIND>(combine<KIND>(A.w, B.w, r.w, sl[k])));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = finish<KIND>(s[k]);
    } else {  // d >= 8: four strided accumulators, (s0 + s1) + (s2 + s3)
      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      float s2[4] = {0.f, 0.f, 0.f, 0.f}, s3[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < d; j += 4) {
        const float4 f = *reinterpret_cast<const float4*>(fq + j);
        const float4 r = *reinterpret_cast<const float4*>(rq + j);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 c = *reinterpret_cast<const float4*>(Cc + (cg + 16 * k) * S + j);
          const float4 A = SIDE == 0 ? f : c, B = SIDE == 0 ? c : f;
          s0[k] = __fadd_rn(s0[k], term<KIND>(combine<KIND>(A.x, B.x, r.x, sl[k])));
          s1[k] = __fadd_rn(s1[k], term<KIND>(combine<KIND>(A.y, B.y, r.y, sl[k])));
          s2[k] = __fadd_rn(s2[k], term<KIND>(combine<KIND>(A.z, B.z, r.z, sl[k])));
          s3[k] = __fadd_rn(s3[k], term<KIND>(combine<KIND>(A.w, B.w, r.w, sl[k])));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) e[k] = finish<KIND>(__fadd_rn(__fadd_rn(s0[k], s1[k]), __fadd_rn(s2[k], s3[k])));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t c = cb + cg + 16 * k;
      if (c == qfix[qi]) e[k] = qself[qi];
      if (cg + 16 * k >= nc || c == qtruth[qi] || !(e[k] < qte[qi])) continue;
      if (a.table && filter_contains(a.table, a.mask, SIDE == 0 ? triple_key(qh[qi], qr[qi], c, a.N, a.R)
                                                                : triple_key(c, qr[qi], qt[qi], a.N, a.R)))
        continue;
      ++cnt;
    }
  }
  // 16 lanes share a query: reduce, one atomic per (query, CTA)
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) cnt += __shfl_down_sync(kFull, cnt, o, 16);
  if (cg == 0 && qi < nq && cnt) atomicAdd(a.better + 2 * (q0 + qi) + SIDE, cnt);
}

// Multiplicative family: energy_sign * score of the row (hc, r, tc), +inf for
// the unrepresentable self-loop candidate (eval.cpp:24, 36-37, 44-47).
template <int KIND>
__device__ float mult_energy(const float* __restrict__ X, const float* __restrict__ Rt, int64_t hc, int64_t r,
                             int64_t tc, int d) {
  if (hc == tc) return __int_as_float(0x7f800000);
  using U = Unit<KIND>;
  const int W = KIND == kDistMult ? d : 2 * d;
  const bool tail_lo = tc < hc;
  float s = 0.f;
  for (int j = 0; j < d; ++j)
    s = __fadd_rn(s, U::term(U::load(X, hc, W, j), U::load(X, tc, W, j), U::load(Rt, r, W, j), tail_lo));
  return KIND == kRotatE ? s : -s;  // DistMult / ComplEx score plausibility (models.hpp:32-38)
}

template <int KIND>
__global__ void mult_true_energy_kernel(EvalArgs a, float* __restrict__ te) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= 2 * a.q) return;
  const int64_t qi = i >> 1;
  te[i] = mult_energy<KIND>(a.X, a.Rt, a.qh[qi], a.qr[qi], a.qt[qi], a.d);
}

// Thread per (query, candidate); the fixed and relation rows are shared by
// the whole block (L1 broadcast), candidate rows stream from L2.
template <int KIND>
__global__ void mult_rank_kernel(EvalArgs a) {
  const int64_t qi = blockIdx.y;
  const int64_t h = a.qh[qi], r = a.qr[qi], t = a.qt[qi];
  const int64_t truth = a.side == 0 ? t : h;
  const float te = a.te[2 * qi + a.side];
  uint32_t cnt = 0;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < a.N;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (c == truth) continue;
    const float e = a.side == 0 ? mult_energy<KIND>(a.X, a.Rt, h, r, c, a.d) : mult_energy<KIND>(a.X, a.Rt, c, r, t, a.d);
    if (!(e < te)) continue;
    if (a.table && filter_contains(a.table, a.mask, a.side == 0 ? triple_key(h, r, c, a.N, a.R)
                                                                 : triple_key(c, r, t, a.N, a.R)))
      continue;
    ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(kFull, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(a.better + 2 * qi + a.side, cnt);
}

template <int KIND>
void launch_mult(EvalArgs a, float* te, int num_sms, cudaStream_t s) {
  mult_true_energy_kernel<KIND><<<ceil_div(2 * a.q, 256), 256, 0, s>>>(a, te);
  count_launch();
  SKG_LAUNCH_CHECK();
  a.te = te;
  const int64_t per_q = std::max<int64_t>(1, std::min<int64_t>((a.N + 255) / 256, (4 * num_sms + a.q - 1) / a.q));
  for (int side = 0; side < 2; ++side) {
    a.side = side;
    dim3 grid(static_cast<unsigned>(per_q), static_cast<unsigned>(a.q));
    mult_rank_kernel<KIND><<<grid, 256, 0, s>>>(a);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
}

template <int KIND>
void launch_kind(EvalArgs a, float* te, int num_sms, cudaStream_t s) {
  true_energy_kernel<KIND><<<ceil_div(2 * a.q, 256), 256, 0, s>>>(a, te);
  count_launch();
  SKG_LAUNCH_CHECK();
  a.te = te;
  const bool tiled = a.d % 4 == 0 && (is_torus(KIND) || a.d >= 8);
  for (int side = 0; side < 2; ++side) {
    a.side = side;
    if (tiled) {
      const int64_t qb = (a.q + kQB - 1) / kQB;
      // split the candidate range so the grid covers every SM at least twice
      int64_t splits = std::max<int64_t>(1, (2 * num_sms + qb - 1) / qb);
      splits = std::min<int64_t>(splits, (a.N + kCB - 1) / kCB);
      const int64_t per = ((a.N + splits - 1) / splits + kCB - 1) / kCB * kCB;
      const size_t smem = sizeof(float) * (2 * kQB + kCB) * (a.d + 4);
      dim3 grid(static_cast<unsigned>(qb), static_cast<unsigned>((a.N + per - 1) / per));
      if (side == 0) rank_tiled_kernel<KIND, 0><<<grid, kEvalThreads, smem, s>>>(a, per);
      else rank_tiled_kernel<KIND, 1><<<grid, kEvalThreads, smem, s>>>(a, per);
    } else {
      dim3 grid(static_cast<unsigned>(std::min<int64_t>(64, (a.N + 255) / 256)), static_cast<unsigned>(a.q));
      rank_simple_kernel<KIND><<<grid, 256, 0, s>>>(a);
    }
    count_launch();
    SKG_LAUNCH_CHECK();
  }
}

template <int KIND, int SIDE>
void configure_tiled() {
  SKG_CUDA(cudaFuncSetAttribute(rank_tiled_kernel<KIND, SIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                200 * 1024));
}

}  // namespace

bool eval_supported(int kind) { return (kind >= kTransE_L2 && kind <= kTransR_L1) || is_mult_kind(kind); }
bool eval_exact(int kind) { return kind <= kTorusE_L1 || is_mult_kind(kind); }

// TransH / TransR rank through per-relation projected entity tables: the ht
// row (a, r, b) scores ||P_r a - P_r b + r_vec|| with the linear map
// P_r x = x - (w_r.x) w_r (TransH, models.hpp:99-103) or M_r x (TransR,
// models.hpp:82-86) applied to both entities, which is the reference's
// v = P_r (a - b) + r_vec up to rounding (these models are tolerance-only).
__global__ void project_transh_kernel(const float* __restrict__ E, const float* __restrict__ w, int64_t N, int d,
                                      float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; row < N;
       row += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const float* x = E + row * d;
    float s = 0.f;
    for (int j = lane; j < d; j += 32) s = fmaf(__ldg(w + j), __ldg(x + j), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    for (int j = lane; j < d; j += 32) out[row * d + j] = __fsub_rn(__ldg(x + j), __fmul_rn(s, __ldg(w + j)));
  }
}

// out (N x dr) = E (N x de) M^T with M (dr x de) row-major: 64 x 64 output
// tiles, 16-wide K slabs through shared memory, 4 x 4 outputs per thread.
__global__ void __launch_bounds__(256) project_transr_kernel(const float* __restrict__ E, const float* __restrict__ M,
                                                              int64_t N, int de, int dr, float* __restrict__ out) {
  __shared__ float As[16][65], Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int c0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < de; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int rr = i / 16, kk = i % 16;
      As[kk][rr] = (r0 + rr < N && k0 + kk < de) ? __ldg(E + (r0 + rr) * de + k0 + kk) : 0.f;
      Bs[kk][rr] = (c0 + rr < dr && k0 + kk < de) ? __ldg(M + static_cast<int64_t>(c0 + rr) * de + k0 + kk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t rr = r0 + ty * 4 + i;
      const int cc = c0 + tx * 4 + j;
      if (rr < N && cc < dr) out[rr * dr + cc] = acc[i][j];
    }
}

void eval_project(int kind, const float* E, const float* proj, const float* normals, int64_t r, int64_t N, int de,
                  int dr, float* out, cudaStream_t s) {
  if (kind == kTransH_L2 || kind == kTransH_L1) {
    project_transh_kernel<<<ceil_div(N * 32, 256), 256, 0, s>>>(E, normals + r * de, N, de, out);
  } else {
    dim3 grid(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>((dr + 63) / 64));
    project_transr_kernel<<<grid, 256, 0, s>>>(E, proj + r * static_cast<int64_t>(dr) * de, N, de, dr, out);
  }
  count_launch();
  SKG_LAUNCH_CHECK();
}

void configure_eval_kernels() {
  configure_tiled<kTransE_L2, 0>();
  configure_tiled<kTransE_L2, 1>();
  configure_tiled<kTransE_L1, 0>();
  configure_tiled<kTransE_L1, 1>();
  configure_tiled<kTorusE_L2, 0>();
  configure_tiled<kTorusE_L2, 1>();
  configure_tiled<kTorusE_L1, 0>();
  configure_tiled<kTorusE_L1, 1>();
}

uint64_t eval_filter_capacity(int64_t nf) {
  uint64_t cap = 1024;
  while (cap < static_cast<uint64_t>(2 * nf)) cap <<= 1;
  return cap;
}

void eval_build_filter(const int32_t* h, const int32_t* r, const int32_t* t, int64_t nf, int64_t N, int64_t R,
                       uint64_t* table, uint64_t cap, cudaStream_t s) {
  SKG_CUDA(cudaMemsetAsync(table, 0xFF, sizeof(uint64_t) * cap, s));
  if (nf > 0) {
    filter_insert_kernel<<<ceil_div(nf, 256), 256, 0, s>>>(h, r, t, nf, N, R, table, cap - 1);
    count_launch();
    SKG_LAUNCH_CHECK();
  }
}

void eval_rank(int kind, const float* X, const float* Rt, int64_t N, int64_t R, int d, const int32_t* qh,
               const int32_t* qr, const int32_t* qt, int64_t q, const uint64_t* table, uint64_t cap, uint32_t* better,
               float* te, int num_sms, cudaStream_t s) {
  SKG_CUDA(cudaMemsetAsync(better, 0, sizeof(uint32_t) * 2 * q, s));
  if (q == 0) return;
  // The per-query kernels put queries on grid.y (at most 65535): chunk.
  constexpr int64_t kMaxQ = 65535;
  if (q > kMaxQ) {
    for (int64_t off = 0; off < q; off += kMaxQ)
      eval_rank(kind, X, Rt, N, R, d, qh + off, qr + off, qt + off, std::min(kMaxQ, q - off), table, cap,
                better + 2 * off, te + 2 * off, num_sms, s);
    return;
  }
  EvalArgs a{};
  a.X = X;
  a.Rt = Rt;
  a.N = N;
  a.R = R;
  a.d = d;
  a.qh = qh;
  a.qr = qr;
  a.qt = qt;
  a.q = q;
  a.table = table;
  a.mask = cap ? cap - 1 : 0;
  a.better = better;
  if (kind == kTransH_L2 || kind == kTransR_L2) kind = kTransE_L2;  // projected tables: ||P a - P b + r||
  if (kind == kTransH_L1 || kind == kTransR_L1) kind = kTransE_L1;
  switch (kind) {
    case kTransE_L2: launch_kind<kTransE_L2>(a, te, num_sms, s); break;
    case kTransE_L1: launch_kind<kTransE_L1>(a, te, num_sms, s); break;
    case kTorusE_L2: launch_kind<kTorusE_L2>(a, te, num_sms, s); break;
    case kTorusE_L1: launch_kind<kTorusE_L1>(a, te, num_sms, s); break;
    case kDistMult: launch_mult<kDistMult>(a, te, num_sms, s); break;
    case kComplEx: launch_mult<kComplEx>(a, te, num_sms, s); break;
    case kRotatE: launch_mult<kRotatE>(a, te, num_sms, s); break;
    default: throw CudaError("eval: model kind not supported on device");
  }
}

}  // namespace skg
