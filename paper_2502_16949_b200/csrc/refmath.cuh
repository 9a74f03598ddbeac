// Reference arithmetic on device, in the reference's exact float association
// (norms.hpp:19-126, compiled without FMA contraction; every op is _rn).
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace skg {

constexpr float kNormEpsF = 1e-6f;  // kNormEps for 32-bit reals, common.hpp:34

__device__ __forceinline__ float torus_wrap(float x) {  // norms.hpp:96-100
  float d = __fsub_rn(x, rintf(x));
  if (d >= 0.5f) d = __fsub_rn(d, 1.0f);
  return d;
}

__device__ __forceinline__ bool nonfinite(float x) { return !(fabsf(x) <= 3.402823466e38f); }

template <bool SQUARE>
__device__ __forceinline__ float norm_term(float x) {
  return SQUARE ? __fmul_rn(x, x) : fabsf(x);
}

// squared_sum (SQUARE) / abs_sum (norms.hpp:19-55): plain loop below 8
// elements, else four strided accumulators combined as (s0+s1)+(s2+s3).
template <bool SQUARE, int VEC>
__device__ float ref_norm_sum(const float* v, int n, bool& bad) {
  bool nf = false;
  float s;
  if (n < 8) {
    s = 0.f;
    for (int j = 0; j < n; ++j) {
      nf |= nonfinite(v[j]);
      s = __fadd_rn(s, norm_term<SQUARE>(v[j]));
    }
  } else {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
      const float4 q = VEC == 4 ? *reinterpret_cast<const float4*>(v + j)
                                : make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      nf |= nonfinite(q.x) | nonfinite(q.y) | nonfinite(q.z) | nonfinite(q.w);
      s0 = __fadd_rn(s0, norm_term<SQUARE>(q.x));
      s1 = __fadd_rn(s1, norm_term<SQUARE>(q.y));
      s2 = __fadd_rn(s2, norm_term<SQUARE>(q.z));
      s3 = __fadd_rn(s3, norm_term<SQUARE>(q.w));
    }
    s = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
    for (; j < n; ++j) {
      nf |= nonfinite(v[j]);
      s = __fadd_rn(s, norm_term<SQUARE>(v[j]));
    }
  }
  bad = nf;
  return s;
}

// squared_sum / abs_sum of 8 rows of n (>= 8, multiple of 4) floats with the
// whole warp: lane 4q + k runs accumulator k of row q (elements k, k + 4, ...
// in order), then (s0 + s1) + (s2 + s3) — the reference association
// (norms.hpp:19-55) with every lane busy. Returns row q's sum on lane q < 8;
// `bad` = a non-finite element in row q (lanes q < 8). Rows are `stride`
// floats apart; stride = 4 (mod 32) keeps the 32 reads of a step on 32 banks.
template <bool SQUARE>
__device__ __forceinline__ float warp_norm8(const float* rows, int stride, int n, int lane, bool& bad) {
  const int q = lane >> 2, k = lane & 3;
  const float* v = rows + q * stride + k;
  float s = 0.f;
  bool nf = false;
#pragma unroll 8
  for (int j = 0; j < n; j += 4) {
    const float x = v[j];
    nf |= nonfinite(x);
    s = __fadd_rn(s, norm_term<SQUARE>(x));
  }
  const unsigned full = 0xffffffffu;
  const float s1 = __shfl_down_sync(full, s, 1), s2 = __shfl_down_sync(full, s, 2), s3 = __shfl_down_sync(full, s, 3);
  const float tot = __fadd_rn(__fadd_rn(s, s1), __fadd_rn(s2, s3));  // valid on lanes k == 0
  const unsigned nfm = __ballot_sync(full, nf);
  const float out = __shfl_sync(full, tot, (lane & 7) * 4);
  bad = ((nfm >> ((lane & 7) * 4)) & 0xFu) != 0u;
  return out;
}

// Deterministic warp sum: tree down to lane 0, then broadcast (every lane gets
// the identical value, unlike an xor butterfly).
__device__ __forceinline__ float warp_sum_bcast(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_down_sync(kFull, v, o));
  return __shfl_sync(kFull, v, 0);
}

}  // namespace skg
